// train_planar.cu -- the fused tile kernel for planar tiles (every tile of a real
// slice): forward (Eq.5) + L1 + all analytic gradients of kernels.py:78-198.
//
// All pixels of a tile lie on the slice plane x = x_T + alpha a1 + beta a2
// (a1, a2 = Rc_s b1, Rc_s b2).  For each (tile, Gaussian) the observed Gaussian
// restricted to that plane factorises exactly into
//   * the in-plane 2D conditional: centre t* = (alpha_g, beta_g) and precision
//     G = B^T Sigma_obs^-1 B,  B = [a1 a2], and
//   * the through-plane marginal term c_min = d_perp^T Sigma_obs^-1 d_perp,
// so u = -1/2 v^T Sigma_obs^-1 v = -1/2 (c_min + dt^T G dt), dt = (alpha, beta) - t*.
// This is the reference's Mahalanobis form (kernels.py:113-122) rewritten, not an
// approximation; membership stays the K-NN set and the -80 cut is applied to u.
// Per pair the forward needs 7 floats of record and 7 flops instead of a 3x3
// inverse; the backward needs q = Sigma_obs^-1 v (scaled) = q0 + da m1 + db m2.
//
// Phases per CTA (one tile): (1) records in fp64 -> fp32 shared memory,
// (2) pixel-major forward over each pixel's K local ids (ascending, so lanes hit
// neighbouring records), (3) Gaussian-major backward: each thread owns a
// contiguous chunk of the tile's Gaussian-sorted pair list, keeps the current
// Gaussian's 10 gradient sums in registers and parks them in a shared-memory
// slot (chunk, Gaussian) -- no atomics -- (4) one combine per Gaussian and one
// global fp32 reduction set per (tile, Gaussian); slice gradients block-reduced.
#include <cub/block/block_reduce.cuh>

#include <algorithm>

#include "batch.cuh"

namespace gsvr {

constexpr int kPB = 256;              // threads per CTA (>= tile_points)
constexpr int kPCap = 1536;           // records staged per page
constexpr float kPCut2 = (float)(-80.0 * 1.4426950408889634);
constexpr float kPLn2 = 0.69314718055994531f;

struct PlanarParams {
  const int64_t *tstart;
  const int32_t *tn;
  const int32_t *tslice;
  const double *torigin;
  const double *tbasis;
  const float2 *ab;
  const float4 *d0obs;  // .w = observed intensity
  const int32_t *perm;
  int K;
  const uint16_t *nbr_local;
  const uint16_t *pair_pix;
  const int64_t *nl_off, *pp_off;
  const int32_t *uoff;
  const int32_t *gid;
  const uint16_t *csr;
  float4 *rec;  // (U, 5) float4, used when a tile's records exceed one page
  const double *mu, *cov6, *cvals;
  const double *Rc, *tvec, *psf6s, *sigma_s, *wdata_s;
  float delta;
  float *dfield;
  double *dslice;
  double *I_hat, *absres;
  unsigned long long *nonfinite_first;
};

// fp64 record of (tile, Gaussian j): forward F0, F1 and backward B0..B2.
__device__ inline void planar_record(const PlanarParams &a, int64_t j, const double xT[3], const double a1[3],
                                     const double a2[3], const double p6[6], float4 r[5]) {
  double S6[6], M[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) S6[e] = a.cov6[6 * j + e] + p6[e];
  inv_sym3<double>(S6, M);
  const double D[3] = {xT[0] - a.mu[3 * j], xT[1] - a.mu[3 * j + 1], xT[2] - a.mu[3 * j + 2]};
  auto mv = [&](const double x[3], double y[3]) {
    y[0] = M[0] * x[0] + M[1] * x[1] + M[2] * x[2];
    y[1] = M[1] * x[0] + M[3] * x[1] + M[4] * x[2];
    y[2] = M[2] * x[0] + M[4] * x[1] + M[5] * x[2];
  };
  double Ma1[3], Ma2[3], MD[3];
  mv(a1, Ma1);
  mv(a2, Ma2);
  mv(D, MD);
  const double G00 = a1[0] * Ma1[0] + a1[1] * Ma1[1] + a1[2] * Ma1[2];
  const double G01 = a1[0] * Ma2[0] + a1[1] * Ma2[1] + a1[2] * Ma2[2];
  const double G11 = a2[0] * Ma2[0] + a2[1] * Ma2[1] + a2[2] * Ma2[2];
  const double h0 = a1[0] * MD[0] + a1[1] * MD[1] + a1[2] * MD[2];
  const double h1 = a2[0] * MD[0] + a2[1] * MD[1] + a2[2] * MD[2];
  const double idet = 1.0 / (G00 * G11 - G01 * G01);
  const double t0 = -(G11 * h0 - G01 * h1) * idet;
  const double t1 = -(G00 * h1 - G01 * h0) * idet;
  double Dp[3], MDp[3];
  for (int d = 0; d < 3; ++d) {
    Dp[d] = D[d] + t0 * a1[d] + t1 * a2[d];
    MDp[d] = MD[d] + t0 * Ma1[d] + t1 * Ma2[d];
  }
  const double cmin = fmax(Dp[0] * MDp[0] + Dp[1] * MDp[1] + Dp[2] * MDp[2], 0.0);
  const double k = -0.5 * kLog2e;
  r[0] = make_float4((float)t0, (float)t1, (float)(k * cmin), (float)a.cvals[j]);
  r[1] = make_float4((float)(k * G00), (float)(2.0 * k * G01), (float)(k * G11), 0.f);
  r[2] = make_float4((float)(k * MDp[0]), (float)(k * MDp[1]), (float)(k * MDp[2]), (float)(k * Ma1[0]));
  r[3] = make_float4((float)(k * Ma1[1]), (float)(k * Ma1[2]), (float)(k * Ma2[0]), (float)(k * Ma2[1]));
  r[4] = make_float4((float)(k * Ma2[2]), 0.f, 0.f, 0.f);
}

// ---- TMA bulk copy (cp.async.bulk) + mbarrier helpers ----------------------
__device__ inline uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ inline void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count) : "memory");
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ inline void tma_load_1d(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}
__device__ inline void mbar_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
        : "=r"(done)
        : "r"(smem_u32(bar)), "r"(parity)
        : "memory");
}
// 2^x on the MUFU pipe (flush-to-zero is exact here: x >= -80 log2(e) > -126)
__device__ inline float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

extern __shared__ __align__(16) unsigned char g_planar_smem[];

struct PlanarSmem {
  float4 *F0, *F1, *B0, *B1;
  float *B2;
  uint16_t *nl;     // staged nbr_local of the tile (TMA), aliased by the slots
  float *slots;     // (10, nslot) gradient slots
  uint16_t *csr;    // staged csr (cap + 1)
  int nslot;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) / 16 * 16; }

__host__ __device__ inline size_t planar_smem_bytes(int cap, int tp, int K, PlanarSmem *L, unsigned char *base) {
  size_t off = 0;
  const size_t rec = (size_t)cap * 16;
  if (L) {
    L->F0 = reinterpret_cast<float4 *>(base + off);
    L->F1 = reinterpret_cast<float4 *>(base + off + rec);
    L->B0 = reinterpret_cast<float4 *>(base + off + 2 * rec);
    L->B1 = reinterpret_cast<float4 *>(base + off + 3 * rec);
    L->B2 = reinterpret_cast<float *>(base + off + 4 * rec);
  }
  off = align16(4 * rec + (size_t)cap * 4);
  const int nslot = cap + kPB;
  const size_t uni = std::max(align16((size_t)tp * K * 2), (size_t)nslot * 10 * 4);
  if (L) {
    L->nl = reinterpret_cast<uint16_t *>(base + off);
    L->slots = reinterpret_cast<float *>(base + off);
    L->nslot = nslot;
  }
  off = align16(off + uni);
  if (L) L->csr = reinterpret_cast<uint16_t *>(base + off);
  off = align16(off + (size_t)(cap + 1) * 2);
  return off;
}

#ifndef GSVR_PLANAR_MINB
#define GSVR_PLANAR_MINB 3
#endif
__global__ void __launch_bounds__(kPB, GSVR_PLANAR_MINB) k_train_planar(PlanarParams a, int cap, int tp) {
  using BR = cub::BlockReduce<float, kPB>;
  __shared__ typename BR::TempStorage red;
  __shared__ float4 spix[kPB];  // (alpha, beta, gnum, gden)
  __shared__ float sred[20];
  __shared__ __align__(8) uint64_t bar;

  PlanarSmem L;
  planar_smem_bytes(cap, tp, a.K, &L, g_planar_smem);

  const int t = blockIdx.x, tid = threadIdx.x;
  const int64_t ts = a.tstart[t];
  const int n = a.tn[t];
  const int s = a.tslice[t];
  const int K = a.K;
  const int m = n * K;
  const int u0 = a.uoff[t];
  const int nU = a.uoff[t + 1] - u0;
  const bool onepage = nU <= cap;
  const uint16_t *gcsr = a.csr + u0 + t;

  // stage this tile's pixel-major local ids with one TMA bulk copy; it lands
  // while the records below are being built
  if (tid == 0) {
    mbar_init(&bar, 1);
    tma_load_1d(L.nl, a.nbr_local + a.nl_off[t], (uint32_t)align16((size_t)m * 2), &bar);
  }

  double R[9], p6[6], xT[3], a1[3], a2[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) R[e] = a.Rc[9 * s + e];
#pragma unroll
  for (int e = 0; e < 6; ++e) p6[e] = a.psf6s[6 * s + e];
  {
    const double *o = a.torigin + 3 * t, *b = a.tbasis + 6 * t;
    for (int r = 0; r < 3; ++r) {
      xT[r] = R[3 * r] * o[0] + R[3 * r + 1] * o[1] + R[3 * r + 2] * o[2] + a.tvec[3 * s + r];
      a1[r] = R[3 * r] * b[0] + R[3 * r + 1] * b[1] + R[3 * r + 2] * b[2];
      a2[r] = R[3 * r] * b[3] + R[3 * r + 1] * b[4] + R[3 * r + 2] * b[5];
    }
  }
  const float sig = (float)a.sigma_s[s];
  const float wdat = (float)a.wdata_s[s];

  const int p = tid;
  float al = 0.f, be = 0.f, iobs = 0.f;
  if (p < n) {
    const float2 v = a.ab[ts + p];
    al = v.x;
    be = v.y;
    iobs = a.d0obs[ts + p].w;
  }
  if (onepage)
    for (int g = tid; g <= nU; g += kPB) L.csr[g] = gcsr[g];

  // ---- forward -----------------------------------------------------------
  float num = 0.f, den = a.delta;
  const int npages = onepage ? 1 : (nU + cap - 1) / cap;
  for (int page = 0; page < npages; ++page) {
    const int base = page * cap;
    const int cnt = min(cap, nU - base);
    if (page > 0) __syncthreads();
    for (int g = tid; g < cnt; g += kPB) {
      float4 r[5];
      planar_record(a, a.gid[u0 + base + g], xT, a1, a2, p6, r);
      L.F0[g] = r[0];
      L.F1[g] = r[1];
      L.B0[g] = r[2];
      L.B1[g] = r[3];
      L.B2[g] = r[4].x;
      if (!onepage) {
        float4 *gr = a.rec + 5 * (int64_t)(u0 + base + g);
        for (int e = 0; e < 5; ++e) gr[e] = r[e];
      }
    }
    if (page == 0) mbar_wait(&bar, 0);
    __syncthreads();
    if (p < n) {
      const uint16_t *nl = L.nl + p;
      if (onepage) {
#pragma unroll 5
        for (int k = 0; k < K; ++k) {
          const int lid = nl[k * n];
          const float4 f0 = L.F0[lid], f1 = L.F1[lid];
          const float da = al - f0.x, db = be - f0.y;
          const float u2 = fmaf(f1.z * db, db, fmaf(fmaf(f1.y, db, f1.x * da), da, f0.z));
          const float e = (u2 < kPCut2) ? 0.f : ex2(u2);
          num = fmaf(f0.w, e, num);
          den += e;
        }
      } else {
        for (int k = 0; k < K; ++k) {
          const unsigned lid = (unsigned)nl[k * n] - (unsigned)base;
          if (lid >= (unsigned)cnt) continue;
          const float4 f0 = L.F0[lid], f1 = L.F1[lid];
          const float da = al - f0.x, db = be - f0.y;
          const float u2 = fmaf(f1.z * db, db, fmaf(fmaf(f1.y, db, f1.x * da), da, f0.z));
          const float e = (u2 < kPCut2) ? 0.f : ex2(u2);
          num = fmaf(f0.w, e, num);
          den += e;
        }
      }
    }
  }

  float l1 = 0.f, dsig = 0.f;
  if (p < n) {
    const float ratio = num / den;
    const float ihat = sig * ratio;
    const float r = ihat - iobs;
    const int64_t dst = a.perm[ts + p];
    if (a.I_hat) a.I_hat[dst] = (double)ihat;
    if (a.absres) a.absres[dst] = (double)fabsf(r);
    if (a.nonfinite_first && !isfinite(ihat)) atomicMin(a.nonfinite_first, (unsigned long long)dst);
    l1 = fabsf(r);
    const float g = (r > 0.f) ? wdat : ((r < 0.f) ? -wdat : 0.f);
    dsig = g * ratio;
    const float gout = g * sig;
    spix[p] = make_float4(al, be, gout / den, -gout * ratio / den);
  }
  __syncthreads();  // spix complete; staged nbr_local dead -> slots may be written

  // ---- backward: Gaussian-major chunks (chunk = thread) --------------------
  const int C = (m + kPB - 1) / kPB;
  float Sa0 = 0.f, Sa1 = 0.f, Sa2 = 0.f, Sb0 = 0.f, Sb1 = 0.f, Sb2 = 0.f;
  {
    const int lo = tid * C;
    const int hi = min(lo + C, m);
    if (lo < hi) {
      const uint16_t *cs = onepage ? L.csr : gcsr;
      int lo_g = 0, hi_g = nU - 1;
      while (lo_g < hi_g) {
        const int mid = (lo_g + hi_g + 1) >> 1;
        if ((int)cs[mid] <= lo) lo_g = mid; else hi_g = mid - 1;
      }
      int g = lo_g;
      int gend = cs[g + 1];
      float4 f0, f1, b0, b1;
      float b2;
      auto load_rec = [&](int gg) {
        if (onepage) {
          f0 = L.F0[gg]; f1 = L.F1[gg]; b0 = L.B0[gg]; b1 = L.B1[gg]; b2 = L.B2[gg];
        } else {
          const float4 *gr = a.rec + 5 * (int64_t)(u0 + gg);
          f0 = gr[0]; f1 = gr[1]; b0 = gr[2]; b1 = gr[3]; b2 = gr[4].x;
        }
      };
      load_rec(g);
      float am0 = 0.f, am1 = 0.f, am2 = 0.f, ac0 = 0.f, ac1 = 0.f, ac2 = 0.f, ac3 = 0.f, ac4 = 0.f,
            ac5 = 0.f, adc = 0.f;
      auto flush = [&](int gg) {
        if (onepage) {
          float *sl = L.slots + gg + tid;
          const int ns = L.nslot;
          sl[0] = am0; sl[ns] = am1; sl[2 * ns] = am2; sl[3 * ns] = ac0; sl[4 * ns] = ac1;
          sl[5 * ns] = ac2; sl[6 * ns] = ac3; sl[7 * ns] = ac4; sl[8 * ns] = ac5; sl[9 * ns] = adc;
        } else {  // tiles beyond one page (rare): direct reductions
          float *df = a.dfield + 10 * (int64_t)a.gid[u0 + gg];
          atomicAdd(df + 0, am0); atomicAdd(df + 1, am1); atomicAdd(df + 2, am2);
          atomicAdd(df + 3, ac0); atomicAdd(df + 4, ac1); atomicAdd(df + 5, ac2);
          atomicAdd(df + 6, ac3); atomicAdd(df + 7, ac4); atomicAdd(df + 8, ac5);
          atomicAdd(df + 9, adc);
          double *dsl = a.dslice + 20 * (int64_t)s;
          atomicAdd(dsl + 0, -(double)am0); atomicAdd(dsl + 1, -(double)am1); atomicAdd(dsl + 2, -(double)am2);
          atomicAdd(dsl + 12, (double)ac0); atomicAdd(dsl + 13, (double)ac1); atomicAdd(dsl + 14, (double)ac2);
          atomicAdd(dsl + 15, (double)ac3); atomicAdd(dsl + 16, (double)ac4); atomicAdd(dsl + 17, (double)ac5);
          const double *o = a.torigin + 3 * t;  // (sum aw) o^T part of dRc
          const double amv[3] = {am0, am1, am2};
          for (int r = 0; r < 3; ++r)
            for (int c = 0; c < 3; ++c) atomicAdd(dsl + 3 + 3 * r + c, -amv[r] * o[c]);
        }
        am0 = am1 = am2 = ac0 = ac1 = ac2 = ac3 = ac4 = ac5 = adc = 0.f;
      };
      // pixel ids of the chunk, chunk-transposed (coalesced); prefetched one
      // group of kPre ahead so the global-load latency overlaps the math
      constexpr int kPre = 8;
      const uint16_t *pp = a.pair_pix + a.pp_off[t] + tid;
      uint32_t nxt[kPre];
#pragma unroll
      for (int j = 0; j < kPre; ++j) nxt[j] = (lo + j < hi) ? pp[j * kPB] : 0u;
      for (int i0 = lo; i0 < hi; i0 += kPre) {
        uint32_t cur[kPre];
#pragma unroll
        for (int j = 0; j < kPre; ++j) cur[j] = nxt[j];
#pragma unroll
        for (int j = 0; j < kPre; ++j) {
          const int ii = i0 + kPre + j;
          nxt[j] = (ii < hi) ? pp[(ii - lo) * kPB] : 0u;
        }
#pragma unroll
        for (int j = 0; j < kPre; ++j) {
          const int i = i0 + j;
          if (i >= hi) break;
          if (i >= gend) {
            flush(g);
            ++g;
            gend = cs[g + 1];
            load_rec(g);
          }
          const float4 px = spix[cur[j]];
          const float da = px.x - f0.x, db = px.y - f0.y;
          const float u2 = fmaf(f1.z * db, db, fmaf(fmaf(f1.y, db, f1.x * da), da, f0.z));
          if (u2 < kPCut2) continue;
          const float e = ex2(u2);
          adc = fmaf(px.z, e, adc);                                        // dc += gnum e
          const float aw_s = fmaf(px.z, f0.w, px.w) * e * (-2.f * kPLn2);  // a * (-2 ln 2)
          // q = Sigma_obs^-1 v * (-log2(e)/2) = q0 + da m1 + db m2;  w = q * (-2 ln 2)
          const float q0 = fmaf(db, b1.z, fmaf(da, b0.w, b0.x));
          const float q1 = fmaf(db, b1.w, fmaf(da, b1.x, b0.y));
          const float q2 = fmaf(db, b2, fmaf(da, b1.y, b0.z));
          const float aw0 = aw_s * q0, aw1 = aw_s * q1, aw2 = aw_s * q2;
          am0 += aw0; am1 += aw1; am2 += aw2;
          Sa0 = fmaf(aw0, px.x, Sa0); Sa1 = fmaf(aw1, px.x, Sa1); Sa2 = fmaf(aw2, px.x, Sa2);
          Sb0 = fmaf(aw0, px.y, Sb0); Sb1 = fmaf(aw1, px.y, Sb1); Sb2 = fmaf(aw2, px.y, Sb2);
          const float h0 = aw0 * (-kPLn2), h1 = aw1 * (-kPLn2), h2 = aw2 * (-kPLn2);  // (a/2) w_i
          ac0 = fmaf(h0, q0, ac0); ac1 = fmaf(h0, q1, ac1); ac2 = fmaf(h0, q2, ac2);
          ac3 = fmaf(h1, q1, ac3); ac4 = fmaf(h1, q2, ac4); ac5 = fmaf(h2, q2, ac5);
        }
      }
      flush(g);
    }
  }
  float St0 = 0.f, St1 = 0.f, St2 = 0.f;
  float P00 = 0.f, P01 = 0.f, P02 = 0.f, P11 = 0.f, P12 = 0.f, P22 = 0.f;
  if (onepage) {
    __syncthreads();
    // ---- combine the (chunk, Gaussian) slots: one reduction set per Gaussian
    const int ns = L.nslot;
    for (int g = tid; g < nU; g += kPB) {
      const int c0 = L.csr[g] / C, c1 = (L.csr[g + 1] - 1) / C;
      float v[10];
#pragma unroll
      for (int e = 0; e < 10; ++e) v[e] = 0.f;
      for (int c = c0; c <= c1; ++c)
#pragma unroll
        for (int e = 0; e < 10; ++e) v[e] += L.slots[e * ns + g + c];
      float *df = a.dfield + 10 * (int64_t)a.gid[u0 + g];
#pragma unroll
      for (int e = 0; e < 10; ++e) atomicAdd(df + e, v[e]);
      St0 += v[0]; St1 += v[1]; St2 += v[2];
      P00 += v[3]; P01 += v[4]; P02 += v[5]; P11 += v[6]; P12 += v[7]; P22 += v[8];
    }
  }

  // ---- slice gradients ----------------------------------------------------
  float vals[20] = {St0, St1, St2, Sa0, Sa1, Sa2, Sb0, Sb1, Sb2, 0.f, 0.f, 0.f,
                    P00, P01, P02, P11, P12, P22, dsig, l1};
#pragma unroll
  for (int e = 0; e < 20; ++e) {
    if (e >= 9 && e < 12) continue;
    const float tot = BR(red).Sum(vals[e]);
    if (tid == 0) sred[e] = tot;
    __syncthreads();
  }
  if (tid < 20) {
    double val;
    const double *o = a.torigin + 3 * t, *b = a.tbasis + 6 * t;
    if (tid < 3) {
      val = -(double)sred[tid];  // dt = sum_p gx_p = -sum aw
    } else if (tid < 12) {
      // dRc = -[(sum aw) o^T + (sum aw alpha) b1^T + (sum aw beta) b2^T]
      const int r = (tid - 3) / 3, c = (tid - 3) % 3;
      val = -((double)sred[r] * o[c] + (double)sred[3 + r] * b[c] + (double)sred[6 + r] * b[3 + c]);
    } else {
      val = (double)sred[tid];
    }
    atomicAdd(a.dslice + 20 * (int64_t)s + tid, val);
  }
}

int train_tiles_planar(const gsvr_batch *b, int64_t S, int64_t N, const double *Rc, const double *tvec,
                       const double *psf6s, const double *sigma_s, const double *wdata_s, const double *mu,
                       const double *cov6, const double *cvals, double delta, float *dfield, double *dslice,
                       double *I_hat, double *absres, unsigned long long *nonfinite_first, cudaStream_t st) {
  (void)S;
  (void)N;
  if (b->TP > kPB) return fail(GSVR_ERR_INVALID, "tile_points must be <= %d", kPB);
  PlanarParams a;
  a.tstart = b->tile_start; a.tn = b->tile_n; a.tslice = b->tile_slice; a.torigin = b->tile_origin;
  a.tbasis = b->tile_basis; a.ab = b->ab; a.d0obs = b->d0obs; a.perm = b->perm; a.K = (int)b->K;
  a.nbr_local = b->nbr_local; a.pair_pix = b->pair_pix; a.uoff = b->uoff; a.gid = b->gid; a.csr = b->csr;
  a.nl_off = b->nl_off; a.pp_off = b->pp_off;
  a.rec = b->rec;
  a.mu = mu; a.cov6 = cov6; a.cvals = cvals;
  a.Rc = Rc; a.tvec = tvec; a.psf6s = psf6s; a.sigma_s = sigma_s; a.wdata_s = wdata_s;
  a.delta = (float)delta;
  a.dfield = dfield; a.dslice = dslice; a.I_hat = I_hat; a.absres = absres;
  a.nonfinite_first = nonfinite_first;
  const int cap = std::max(1, std::min(b->max_unique, kPCap));
  const size_t smem = planar_smem_bytes(cap, b->TP, (int)b->K, nullptr, nullptr);
  static size_t attr = 0;
  if (smem > attr) {
    GSVR_CUDA(cudaFuncSetAttribute(k_train_planar, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = smem;
  }
  k_train_planar<<<(unsigned)b->T, kPB, smem, st>>>(a, cap, b->TP);
  GSVR_LAUNCH_CHECK("k_train_planar");
  return GSVR_OK;
}

}  // namespace gsvr
