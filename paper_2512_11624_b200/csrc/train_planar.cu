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
#include "tma.cuh"

namespace gsvr {

constexpr int kPB = 256;              // threads per CTA (>= tile_points)
constexpr int kPCap = 1536;           // records staged per page
static_assert(kPCap >= kMinRecordPage, "global record pages are sized from kMinRecordPage");
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
  const double2 *grec;  // (N, 5) double2 = [mu0 mu1] [mu2 c] [cov6 0..5]: one 80-byte gather per record
  const int32_t *gpos;  // row of Gaussian j in grec (spatial order), or null (row j)
  const int32_t *tlist;  // tiles of this launch (blockIdx.x -> tile), or null (all tiles)
  const double *Rc, *tvec, *psf6s, *sigma_s, *wdata_s;
  float delta;
  double delta64;
  // float64 inputs of the L1 sign refinement (pixel_l1, batch.cuh)
  const double *x0s, *iobs_s, *mu, *cov6, *cvals;
  float *gpart;  // (U, 10) per-(tile, Gaussian) partial gradients
  float4 *brec;  // (U, 3) backward record halves when they do not stay in shared memory, else null
  double *tpart;   // (T, 20) per-tile slice partials
  double *I_hat, *absres;
  unsigned long long *nonfinite_first;
};

// fp64 record of (tile, Gaussian j): forward F0, F1 and backward B0..B2.
__device__ inline void planar_record(const PlanarParams &a, int64_t j, const double xT[3], const double a1[3],
                                     const double a2[3], const double p6[6], float4 r[5]) {
  const double2 *gr = a.grec + 5 * (int64_t)(a.gpos ? a.gpos[j] : (int32_t)j);
  const double2 g0 = gr[0], g1 = gr[1], g2 = gr[2], g3 = gr[3], g4 = gr[4];
  const double cj[6] = {g2.x, g2.y, g3.x, g3.y, g4.x, g4.y};
  double S6[6], M[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) S6[e] = cj[e] + p6[e];
  inv_sym3<double>(S6, M);
  const double D[3] = {xT[0] - g0.x, xT[1] - g0.y, xT[2] - g1.x};
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
  r[0] = make_float4((float)t0, (float)t1, (float)(k * cmin), (float)g1.y);
  r[1] = make_float4((float)(k * G00), (float)(2.0 * k * G01), (float)(k * G11), 0.f);
  r[2] = make_float4((float)(k * MDp[0]), (float)(k * MDp[1]), (float)(k * MDp[2]), (float)(k * Ma1[0]));
  r[3] = make_float4((float)(k * Ma1[1]), (float)(k * Ma1[2]), (float)(k * Ma2[0]), (float)(k * Ma2[1]));
  r[4] = make_float4((float)(k * Ma2[2]), 0.f, 0.f, 0.f);
}

// 2^x on the MUFU pipe (flush-to-zero is exact here: x >= -80 log2(e) > -126)
__device__ inline float ex2(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}

extern __shared__ __align__(16) unsigned char g_planar_smem[];

struct PlanarSmem {
  float4 *F0, *B0, *B1;
  float2 *F1;   // (k G00, 2k G01): with F1c, the in-plane conic (24 B forward record:
  float *F1c;   // one 16-, one 8- and one 4-byte load instead of two 16-byte ones)
  float *B2;
  uint16_t *nl;     // staged nbr_local of the tile (TMA), aliased by the slots
  float *slots;     // (10, nslot) gradient slots
  uint16_t *csr;    // staged csr (cap + 1)
  int nslot;
};

__host__ __device__ inline size_t align16(size_t x) { return (x + 15) / 16 * 16; }

// bglob: the backward record halves (B0, B1, B2; 36 of the 64 bytes per
// record) live in global memory instead (large tiles: keeps 3 CTAs per SM)
__host__ __device__ inline size_t planar_smem_bytes(int cap, int tp, int K, PlanarSmem *L, unsigned char *base,
                                                    bool bglob = false) {
  size_t off = 0;
  const size_t rec = (size_t)cap * 16;
  const size_t nb = bglob ? 0 : 2;  // B0, B1 float4 arrays
  if (L) {
    L->F0 = reinterpret_cast<float4 *>(base + off);
    L->B0 = reinterpret_cast<float4 *>(base + off + rec);
    L->B1 = reinterpret_cast<float4 *>(base + off + 2 * rec);
    L->F1 = reinterpret_cast<float2 *>(base + off + (1 + nb) * rec);
    L->F1c = reinterpret_cast<float *>(base + off + (1 + nb) * rec + (size_t)cap * 8);
    L->B2 = reinterpret_cast<float *>(base + off + (1 + nb) * rec + (size_t)cap * 12);
  }
  off = align16((1 + nb) * rec + (size_t)cap * (bglob ? 12 : 16));
  const int nslot = cap + kPB;
  const size_t uni = std::max(align16((size_t)nl_len(tp, K) * 2), (size_t)nslot * 8 * 4);
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
// BG: backward record halves in global memory (a.brec); LIST: tiles through a.tlist
template <bool BG, bool LIST>
__global__ void __launch_bounds__(kPB, GSVR_PLANAR_MINB) k_train_planar(PlanarParams a, int cap, int tp) {
  __shared__ float4 spix[kPB];  // (alpha, beta, gnum, gden)
  __shared__ float swred[kPB / 32][20];
  __shared__ uint16_t cstart[kPB];  // first local Gaussian of every backward chunk
  __shared__ double sgeo[15];
  __shared__ unsigned s_amb[kPB / 32];  // per warp: pixels whose L1 sign needs float64
  __shared__ __align__(8) uint64_t bar;

  PlanarSmem L;
  planar_smem_bytes(cap, tp, a.K, &L, g_planar_smem, BG);

  const int t = LIST ? a.tlist[blockIdx.x] : (int)blockIdx.x, tid = threadIdx.x;
  const int64_t ts = a.tstart[t];
  const int n = a.tn[t];
  const int s = a.tslice[t];
  const int K = a.K;
  const int m = n * K;
  const int u0 = a.uoff[t];
  const int nU = a.uoff[t + 1] - u0;
  const bool onepage = nU <= cap;
  const uint16_t *gcsr = a.csr + u0 + t;

  // independent per-thread loads first (pixel inputs, slice scalars, this
  // thread's first record id), so their latency overlaps the setup below
  const int p = tid;
  float al = 0.f, be = 0.f, iobs = 0.f;
  if (p < n) {
    const float2 v = a.ab[ts + p];
    al = v.x;
    be = v.y;
    iobs = a.d0obs[ts + p].w;
  }
  const float sig = (float)a.sigma_s[s];
  const float wdat = (float)a.wdata_s[s];
  const int gid0 = tid < min(nU, cap) ? a.gid[u0 + tid] : 0;

  // stage this tile's pixel-major local ids with one TMA bulk copy; it lands
  // while the records below are being built
  if (tid == 0) {
    mbar_init(&bar, 1);
    tma_load_1d(L.nl, a.nbr_local + a.nl_off[t], (uint32_t)align16((size_t)nl_len(n, K) * 2), &bar);
  }
  __syncthreads();  // barrier initialised before anyone waits on it

  // per-tile fp64 geometry in shared memory (keeps it out of every thread's registers):
  // x_T = Rc o + t, a1 = Rc b1, a2 = Rc b2 (world in-plane axes), rotated PSF
  const double *xT = sgeo, *a1 = sgeo + 3, *a2 = sgeo + 6, *p6 = sgeo + 9;
  if (tid < 15) {
    double v;
    if (tid < 9) {
      const int r = tid % 3, which = tid / 3;  // which: 0 -> x_T, 1 -> a1, 2 -> a2
      const double *R = a.Rc + 9 * s + 3 * r;
      const double *src = which == 0 ? a.torigin + 3 * t : a.tbasis + 6 * t + 3 * (which - 1);
      v = R[0] * src[0] + R[1] * src[1] + R[2] * src[2] + (which == 0 ? a.tvec[3 * s + r] : 0.0);
      sgeo[3 * which + r] = v;
    } else {
      sgeo[tid] = a.psf6s[6 * s + (tid - 9)];
    }
  }
  if (onepage) {
    for (int g = tid; g <= nU; g += kPB) L.csr[g] = gcsr[g];
  } else {  // segments of one Gaussian are flushed by several threads: accumulate
    for (int e = tid; e < 10 * nU; e += kPB) a.gpart[10 * (int64_t)u0 + e] = 0.f;
  }
  __syncthreads();

  // ---- forward -----------------------------------------------------------
  float num = 0.f, den = a.delta;
  const int npages = onepage ? 1 : (nU + cap - 1) / cap;
  for (int page = 0; page < npages; ++page) {
    const int base = page * cap;
    const int cnt = min(cap, nU - base);
    if (page > 0) __syncthreads();
    for (int g = tid; g < cnt; g += kPB) {
      float4 r[5];
      planar_record(a, (page == 0 && g == tid) ? gid0 : a.gid[u0 + base + g], xT, a1, a2, p6, r);
      L.F0[g] = r[0];
      L.F1[g] = make_float2(r[1].x, r[1].y);
      L.F1c[g] = r[1].z;
      if (BG) {
        float4 *bg = a.brec + 3 * (int64_t)(u0 + base + g);
        bg[0] = r[2];
        bg[1] = r[3];
        bg[2] = r[4];
      } else {
        L.B0[g] = r[2];
        L.B1[g] = r[3];
        L.B2[g] = r[4].x;
      }
      if (!onepage) {
        float4 *gr = a.rec + 5 * (int64_t)(u0 + base + g);
        for (int e = 0; e < 5; ++e) gr[e] = r[e];
      }
    }
    if (page == 0 && onepage) {
      // chunk c of the backward starts inside the Gaussian whose pair range
      // holds c*C: scattered here once instead of a binary search per thread
      const int Cc = chunk_len(m);
      for (int g = tid; g < nU; g += kPB) {
        const int i0 = L.csr[g], i1 = L.csr[g + 1];
        for (int c = (i0 + Cc - 1) / Cc; c * Cc < i1; ++c) cstart[c] = (uint16_t)g;
      }
    }
    if (page == 0) mbar_wait(&bar, 0);
    __syncthreads();
    if (p < n) {
      // local ids of neighbours (2k, 2k+1) in one 32-bit word (nl_index)
      const uint32_t *nl2 = reinterpret_cast<const uint32_t *>(L.nl) + p;
      const uint16_t *nl = L.nl;
      auto fwd_pair = [&](int lid) {
        GSVR_DCHECK(lid < nU, "planar fwd lid", lid, nU);
        const float4 f0 = L.F0[lid];
        const float2 f1 = L.F1[lid];
        const float f1z = L.F1c[lid];
        const float da = al - f0.x, db = be - f0.y;
        const float u2 = fmaf(f1z * db, db, fmaf(fmaf(f1.y, db, f1.x * da), da, f0.z));
        const float e = (u2 < kPCut2) ? 0.f : ex2(u2);
        num = fmaf(f0.w, e, num);
        den += e;
      };
      if (onepage) {
        const int K2 = K >> 1;
#pragma unroll 1
        for (int kp = 0; kp < K2; ++kp) {
          const uint32_t two = nl2[kp * n];
          fwd_pair((int)(two & 0xffffu));
          fwd_pair((int)(two >> 16));
        }
        if (K & 1) fwd_pair((int)nl[nl_index(p, K - 1, n)]);
      } else {
        for (int k = 0; k < K; ++k) {
          const unsigned lid = (unsigned)nl[nl_index(p, k, n)] - (unsigned)base;
          if (lid >= (unsigned)cnt) continue;
          const float4 f0 = L.F0[lid];
          const float2 f1 = L.F1[lid];
          const float f1z = L.F1c[lid];
          const float da = al - f0.x, db = be - f0.y;
          const float u2 = fmaf(f1z * db, db, fmaf(fmaf(f1.y, db, f1.x * da), da, f0.z));
          const float e = (u2 < kPCut2) ? 0.f : ex2(u2);
          num = fmaf(f0.w, e, num);
          den += e;
        }
      }
    }
  }

  // residual, L1 subgradient (kernels.py:133-143), outputs.  Residuals within
  // the fp32 render tolerance are only flagged here; the warps that hold one
  // re-render those pixels in float64 after the barrier (refine_pixel_f64,
  // batch.cuh), before the backward reads spix -- the common path carries a
  // compare and a ballot.
  float l1 = 0.f, dsig = 0.f, ratio = 0.f;
  bool amb = false;
  if (p < n) {
    ratio = num / den;
    const float ihat = sig * ratio;
    const float r = ihat - iobs;
    amb = fabsf(r) <= kResidualFloorRel * fmaxf(fabsf(iobs), fabsf(ihat));
    const int64_t dst = a.perm[ts + p];
    if (a.I_hat) a.I_hat[dst] = (double)ihat;
    if (a.absres) a.absres[dst] = (double)fabsf(r);
    if (a.nonfinite_first && !isfinite(ihat)) atomicMin(a.nonfinite_first, (unsigned long long)dst);
    l1 = fabsf(r);
    const float g = (r > 0.f) ? wdat : -wdat;
    dsig = g * ratio;
    const float gout = g * sig;
    spix[p] = make_float4(al, be, gout / den, -gout * ratio / den);
  }
  {
    const unsigned wamb = __ballot_sync(0xffffffffu, amb);
    if ((tid & 31) == 0) s_amb[tid >> 5] = wamb;
  }
  __syncthreads();  // spix complete
  {
    unsigned any = 0;
#pragma unroll
    for (int w = 0; w < kPB / 32; ++w) any |= s_amb[w];
    if (any) {  // rare: float64 re-render of the ambiguous pixels (nbr_local still staged)
      unsigned ball = s_amb[tid >> 5];
      const int lane = tid & 31;
      while (ball) {
        const int src = __ffs(ball) - 1;
        ball &= ball - 1;
        const int q = (tid & ~31) + src;
        const double2 nd = refine_pixel_f64(lane, q, n, K, L.nl, a.gid + u0, a.x0s, ts + q, a.Rc + 9 * s,
                                            a.tvec + 3 * s, p6, a.mu, a.cov6, a.cvals);
        if (lane == src) {
          const double ratio64 = nd.x / (nd.y + a.delta64);
          const double ihat64 = a.sigma_s[s] * ratio64;
          const double io = a.iobs_s[ts + q];
          const double r64 = ihat64 - io;
          const float g = fabs(r64) <= kResidualZeroRel * fmax(fabs(io), fabs(ihat64)) ? 0.f
                          : (r64 > 0.0 ? wdat : -wdat);
          ratio = (float)ratio64;
          l1 = (float)fabs(r64);
          dsig = g * ratio;
          const float gout = g * sig;
          spix[q] = make_float4(al, be, gout / den, -gout * ratio / den);
          const int64_t dst = a.perm[ts + q];
          if (a.I_hat) a.I_hat[dst] = ihat64;
          if (a.absres) a.absres[dst] = fabs(r64);
        }
      }
      __syncthreads();  // refined spix visible; staged nbr_local dead -> slots may be written
    }
  }

  // ---- backward: Gaussian-major chunks (chunk = thread) --------------------
  // Per pair only 7 weighted moments about the Gaussian's in-plane centre are
  // accumulated (a = (gnum c + gden) e; dal, dbe = offsets from the centre):
  //   Sc = sum gnum e, S0 = sum a, S1 = sum a dal, S2 = sum a dbe,
  //   S11 = sum a dal^2, S12 = sum a dal dbe, S22 = sum a dbe^2.
  // Since Sigma_obs^-1 v = (q0 + dal m1 + dbe m2) / kappa is affine in (dal, dbe),
  // every gradient of kernels.py:157-198 is a fixed combination of these moments,
  // evaluated once per (tile, Gaussian) in the combine step below.
  const int C = chunk_len(m);
  float St0 = 0.f, St1 = 0.f, St2 = 0.f;                                  // sum a w
  float Sa0 = 0.f, Sa1 = 0.f, Sa2 = 0.f, Sb0 = 0.f, Sb1 = 0.f, Sb2 = 0.f;  // sum a w alpha, a w beta
  float P00 = 0.f, P01 = 0.f, P02 = 0.f, P11 = 0.f, P12 = 0.f, P22 = 0.f;
  // Moments of one (tile, Gaussian) -> gradients.  With B = [q0 m1 m2] (scaled
  // Sigma_obs^-1 applied to the plane frame) and the moment matrix
  // Sm = [[S0 S1 S2], [S1 S11 S12], [S2 S12 S22]]:  C = B Sm,
  //   sum a w           = ik C[:,0]            (dmu; dt = -sum)
  //   sum (a/2) w w^T   = (ik^2/2) C B^T       (dcov6; dpsf6 = sum)
  //   sum a w alpha     = alpha_g sum a w + ik C[:,1]   (dRc, with beta likewise)
  auto moments_to_grads = [&](const float4 &f0, const float4 &b0, const float4 &b1, float b2, const float M[7],
                              float out[10]) {
    const float ik = -2.f * kPLn2;  // 1 / kappa, kappa = -log2(e)/2
    const float q0[3] = {b0.x, b0.y, b0.z}, m1[3] = {b0.w, b1.x, b1.y}, m2[3] = {b1.z, b1.w, b2};
    float Cm[3][3];
#pragma unroll
    for (int d = 0; d < 3; ++d) {
      Cm[d][0] = fmaf(q0[d], M[1], fmaf(m1[d], M[2], m2[d] * M[3]));
      Cm[d][1] = fmaf(q0[d], M[2], fmaf(m1[d], M[4], m2[d] * M[5]));
      Cm[d][2] = fmaf(q0[d], M[3], fmaf(m1[d], M[5], m2[d] * M[6]));
    }
    const float h = 0.5f * ik * ik;
    const int ri[6] = {0, 0, 0, 1, 1, 2}, ci[6] = {0, 1, 2, 1, 2, 2};
#pragma unroll
    for (int e = 0; e < 6; ++e) {
      const int i = ri[e], j = ci[e];
      out[3 + e] = h * fmaf(Cm[i][0], q0[j], fmaf(Cm[i][1], m1[j], Cm[i][2] * m2[j]));
    }
#pragma unroll
    for (int d = 0; d < 3; ++d) out[d] = ik * Cm[d][0];
    out[9] = M[0];
    St0 += out[0]; St1 += out[1]; St2 += out[2];
    Sa0 += fmaf(f0.x, out[0], ik * Cm[0][1]); Sa1 += fmaf(f0.x, out[1], ik * Cm[1][1]);
    Sa2 += fmaf(f0.x, out[2], ik * Cm[2][1]);
    Sb0 += fmaf(f0.y, out[0], ik * Cm[0][2]); Sb1 += fmaf(f0.y, out[1], ik * Cm[1][2]);
    Sb2 += fmaf(f0.y, out[2], ik * Cm[2][2]);
    P00 += out[3]; P01 += out[4]; P02 += out[5]; P11 += out[6]; P12 += out[7]; P22 += out[8];
  };
  // one pair's moment contributions (a = (gnum c + gden) e about the centre)
#define GSVR_PAIR(PXID)                                                                         \
  do {                                                                                           \
    const float4 px = spix[(PXID)];                                                              \
    const float da = px.x - f0.x, db = px.y - f0.y;                                              \
    const float u2 = fmaf(f1.z * db, db, fmaf(fmaf(f1.y, db, f1.x * da), da, f0.z));             \
    const float e = (u2 < kPCut2) ? 0.f : ex2(u2);                                               \
    sc = fmaf(px.z, e, sc);                                                                      \
    const float av = fmaf(px.z, f0.w, px.w) * e;                                                 \
    s0 += av;                                                                                    \
    const float t1 = av * da, t2 = av * db;                                                      \
    s1 += t1;                                                                                    \
    s2 += t2;                                                                                    \
    s11 = fmaf(t1, da, s11);                                                                     \
    s12 = fmaf(t1, db, s12);                                                                     \
    s22 = fmaf(t2, db, s22);                                                                     \
  } while (0)
  const int lo = tid * C;
  const int hi = min(lo + C, m);
  if (onepage) {
    // each thread owns pairs [lo, hi) of the Gaussian-sorted list; a segment
    // ends at a Gaussian boundary or at the chunk end and parks its 7 moments in
    // slot (chunk, Gaussian) = g + tid: two 16-byte stores into SoA halves, so
    // neighbouring slots are neighbouring 16-byte words (conflict-free combine)
    if (lo < hi) {
      int g = cstart[tid];
      int gend = L.csr[g + 1];
      float4 f0 = L.F0[g], f1 = make_float4(L.F1[g].x, L.F1[g].y, L.F1c[g], 0.f);
      float4 *slot = reinterpret_cast<float4 *>(L.slots) + (g + tid);
      const int sh = L.nslot;  // offset of the second half
      float sc = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f, s11 = 0.f, s12 = 0.f, s22 = 0.f;
#define GSVR_NEXT_SEGMENT()                                       \
  do {                                                            \
    slot[0] = make_float4(sc, s0, s1, s2);                        \
    slot[sh] = make_float4(s11, s12, s22, 0.f);                   \
    slot += 1;                                                    \
    sc = s0 = s1 = s2 = s11 = s12 = s22 = 0.f;                    \
    ++g;                                                          \
    gend = L.csr[g + 1];                                          \
    f0 = L.F0[g];                                                 \
    f1 = make_float4(L.F1[g].x, L.F1[g].y, L.F1c[g], 0.f);        \
  } while (0)
      // pair pixel ids: 8 per 16-byte load (chunk-blocked layout), one group ahead
      const uint4 *pp4 = reinterpret_cast<const uint4 *>(a.pair_pix + a.pp_off[t]) + tid;
      uint4 nxt = pp4[0];
      int i0 = lo, q = 0;
      for (; i0 + 8 <= hi; i0 += 8, ++q) {
        const uint4 cur = nxt;
        if (i0 + 8 < hi) nxt = pp4[(q + 1) * kPB];
        const uint32_t ids[8] = {cur.x & 0xffffu, cur.x >> 16, cur.y & 0xffffu, cur.y >> 16,
                                 cur.z & 0xffffu, cur.z >> 16, cur.w & 0xffffu, cur.w >> 16};
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (i0 + j >= gend) GSVR_NEXT_SEGMENT();
          GSVR_PAIR(ids[j]);
        }
      }
      if (i0 < hi) {
        // remainder (< 8 pairs): ids shifted out of registers (a runtime-indexed
        // array would live in local memory)
        uint64_t lo64 = ((uint64_t)nxt.y << 32) | nxt.x, hi64 = ((uint64_t)nxt.w << 32) | nxt.z;
        for (int j = 0; i0 + j < hi; ++j) {
          if (i0 + j >= gend) GSVR_NEXT_SEGMENT();
          const uint32_t id = (uint32_t)lo64 & 0xffffu;
          lo64 = (lo64 >> 16) | (hi64 << 48);
          hi64 >>= 16;
          GSVR_PAIR(id);
        }
      }
      slot[0] = make_float4(sc, s0, s1, s2);
      slot[sh] = make_float4(s11, s12, s22, 0.f);
#undef GSVR_NEXT_SEGMENT
    }
    __syncthreads();
    // ---- combine the (chunk, Gaussian) moment slots; one partial set per Gaussian
    const float4 *slots4 = reinterpret_cast<const float4 *>(L.slots);
    for (int g = tid; g < nU; g += kPB) {
      const int c0 = L.csr[g] / C, c1 = (L.csr[g + 1] - 1) / C;
      float Mo[7];
#pragma unroll
      for (int e = 0; e < 7; ++e) Mo[e] = 0.f;
      for (int c = c0; c <= c1; ++c) {
        const float4 x = slots4[g + c], y = slots4[L.nslot + g + c];
        Mo[0] += x.x; Mo[1] += x.y; Mo[2] += x.z; Mo[3] += x.w; Mo[4] += y.x; Mo[5] += y.y; Mo[6] += y.z;
      }
      float out[10];
      if (BG) {
        const float4 *bg = a.brec + 3 * (int64_t)(u0 + g);
        moments_to_grads(L.F0[g], bg[0], bg[1], bg[2].x, Mo, out);
      } else {
        moments_to_grads(L.F0[g], L.B0[g], L.B1[g], L.B2[g], Mo, out);
      }
      float2 *df = reinterpret_cast<float2 *>(a.gpart + 10 * (int64_t)(u0 + g));
#pragma unroll
      for (int e = 0; e < 5; ++e) df[e] = make_float2(out[2 * e], out[2 * e + 1]);
    }
  } else if (lo < hi) {
    // tiles whose records exceed one page (rare): records from global memory,
    // each segment converted and accumulated into the tile's zeroed partials
    int glo = 0, ghi = nU - 1;
    while (glo < ghi) {
      const int mid = (glo + ghi + 1) >> 1;
      if ((int)gcsr[mid] <= lo) glo = mid; else ghi = mid - 1;
    }
    int g = glo, gend = gcsr[g + 1];
    const float4 *gr = a.rec + 5 * (int64_t)(u0 + g);
    float4 f0 = gr[0], f1 = gr[1];
    float sc = 0.f, s0 = 0.f, s1 = 0.f, s2 = 0.f, s11 = 0.f, s12 = 0.f, s22 = 0.f;
    auto flush = [&]() {
      const float4 *r = a.rec + 5 * (int64_t)(u0 + g);
      const float Mo[7] = {sc, s0, s1, s2, s11, s12, s22};
      float out[10];
      moments_to_grads(r[0], r[2], r[3], r[4].x, Mo, out);
      float *df = a.gpart + 10 * (int64_t)(u0 + g);
#pragma unroll
      for (int e = 0; e < 10; ++e) atomicAdd(df + e, out[e]);
      sc = s0 = s1 = s2 = s11 = s12 = s22 = 0.f;
    };
    const uint16_t *pp = a.pair_pix + a.pp_off[t];
    for (int i = lo; i < hi; ++i) {
      if (i >= gend) {
        flush();
        ++g;
        gend = gcsr[g + 1];
        gr = a.rec + 5 * (int64_t)(u0 + g);
        f0 = gr[0];
        f1 = gr[1];
      }
      const int r = i - lo;
      GSVR_PAIR(pp[(int64_t)(r >> 3) * kPB * 8 + tid * 8 + (r & 7)]);
    }
    flush();
  }
#undef GSVR_PAIR

  // ---- slice gradients: warp shuffles, one barrier, one fp64 add per component
  {
    const double *o = a.torigin + 3 * t, *b = a.tbasis + 6 * t;
    // transposed warp reduction: each butterfly step halves the vector a lane
    // carries (31 shuffles for 32 slots instead of 5 per value); lane l ends
    // with the warp total of slot l (slots 9-11 and 20-31 are zero padding)
    float v[32] = {St0, St1, St2, Sa0, Sa1, Sa2, Sb0, Sb1, Sb2, 0.f, 0.f, 0.f,
                   P00, P01, P02, P11, P12, P22, dsig, l1};
    const int warp = tid >> 5, lane = tid & 31;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) {
      const bool up = (lane & o) != 0;
#pragma unroll
      for (int e = 0; e < o; ++e) {
        const float send = up ? v[e] : v[e + o];
        const float keep = up ? v[e + o] : v[e];
        v[e] = keep + __shfl_xor_sync(0xffffffffu, send, o);
      }
    }
    if (lane < 20) swred[warp][lane] = v[0];
    __syncthreads();
    if (tid < 20) {
      double acc[9];
      for (int e = 0; e < 9; ++e) {
        double x = 0.0;
        for (int w = 0; w < kPB / 32; ++w) x += (double)swred[w][e];
        acc[e] = x;
      }
      double val;
      if (tid < 3) {
        val = -acc[tid];  // dt = sum_p gx_p = -sum aw
      } else if (tid < 12) {
        // dRc = -[(sum aw) o^T + (sum aw alpha) b1^T + (sum aw beta) b2^T]
        const int r = (tid - 3) / 3, c = (tid - 3) % 3;
        val = -(acc[r] * o[c] + acc[3 + r] * b[c] + acc[6 + r] * b[3 + c]);
      } else {
        val = 0.0;
        for (int w = 0; w < kPB / 32; ++w) val += (double)swred[w][tid];
      }
      a.tpart[20 * (int64_t)t + tid] = val;
    }
  }
}

// (mu, c, cov6) of every Gaussian packed into one 80-byte row (record gathers)
__global__ void k_pack_grec(int64_t N, const double *__restrict__ mu, const double *__restrict__ cov6,
                            const double *__restrict__ cvals, const int32_t *__restrict__ gpos,
                            double2 *__restrict__ out) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    double2 *o = out + 5 * (int64_t)(gpos ? gpos[j] : (int32_t)j);
    o[0] = make_double2(mu[3 * j], mu[3 * j + 1]);
    o[1] = make_double2(mu[3 * j + 2], cvals[j]);
    o[2] = make_double2(cov6[6 * j], cov6[6 * j + 1]);
    o[3] = make_double2(cov6[6 * j + 2], cov6[6 * j + 3]);
    o[4] = make_double2(cov6[6 * j + 4], cov6[6 * j + 5]);
  }
}

int train_tiles_planar(const gsvr_batch *b, int64_t S, int64_t N, const double *Rc, const double *tvec,
                       const double *psf6s, const double *sigma_s, const double *wdata_s, const double *mu,
                       const double *cov6, const double *cvals, double delta, float *dfield, double *dslice,
                       double *I_hat, double *absres, unsigned long long *nonfinite_first, cudaStream_t st) {
  (void)S;
  if (b->TP > kPB) return fail(GSVR_ERR_INVALID, "tile_points must be <= %d", kPB);
  GSVR_TRY(grow(b->ws_grec, b->ws_grec_cap, (size_t)N * 80, st));
  double2 *grec = reinterpret_cast<double2 *>(b->ws_grec);
  const int32_t *gpos = b->gpos && b->gpos_N == N ? b->gpos : nullptr;
  k_pack_grec<<<grid_for(N, 256), 256, 0, st>>>(N, mu, cov6, cvals, gpos, grec);
  GSVR_LAUNCH_CHECK("k_pack_grec");
  PlanarParams a;
  a.tstart = b->tile_start; a.tn = b->tile_n; a.tslice = b->tile_slice; a.torigin = b->tile_origin;
  a.tbasis = b->tile_basis; a.ab = b->ab; a.d0obs = b->d0obs; a.perm = b->perm; a.K = (int)b->K;
  a.nbr_local = b->nbr_local; a.pair_pix = b->pair_pix; a.uoff = b->uoff; a.gid = b->gid; a.csr = b->csr;
  a.nl_off = b->nl_off; a.pp_off = b->pp_off;
  a.rec = b->rec;
  a.grec = grec;
  a.gpos = gpos;
  a.Rc = Rc; a.tvec = tvec; a.psf6s = psf6s; a.sigma_s = sigma_s; a.wdata_s = wdata_s;
  a.delta = (float)delta;
  a.delta64 = delta;
  a.x0s = b->x0s; a.iobs_s = b->iobs_s; a.mu = mu; a.cov6 = cov6; a.cvals = cvals;
  a.gpart = b->gpart; a.tpart = b->tpart; a.I_hat = I_hat; a.absres = absres;
  a.nonfinite_first = nonfinite_first;
  a.tlist = nullptr;
  const int cap = std::max(1, std::min(b->max_unique, kPCap));
  const size_t static_smem = 6 * 1024;
  auto fits = [&](int c) {  // records in shared memory without costing residency
    return (planar_smem_bytes(c, b->TP, (int)b->K, nullptr, nullptr) + static_smem) * GSVR_PLANAR_MINB <=
           227 * 1024;
  };
  static const bool allow_bglob = [] {
    const char *v = std::getenv("GSVR_BREC_GLOBAL");
    return !(v && v[0] == '0');
  }();
  static const bool allow_buckets = [] {
    const char *v = std::getenv("GSVR_TILE_BUCKETS");
    return !(v && v[0] == '0');
  }();
  extern bool force_brec_global;
  // one launch: the page sized by the largest tile; large tiles move the
  // backward record halves to global memory when the page would cut residency
  // below GSVR_PLANAR_MINB CTAs per SM
  auto launch = [&](int c, unsigned blocks, bool may_bglob) -> int {
    size_t smem = planar_smem_bytes(c, b->TP, (int)b->K, nullptr, nullptr);
    a.brec = nullptr;
    if (force_brec_global || (may_bglob && allow_bglob && !fits(c))) {
      GSVR_TRY(grow(b->ws_brec, b->ws_brec_cap, (size_t)std::max<int64_t>(b->U, 1) * 48, st));
      a.brec = reinterpret_cast<float4 *>(b->ws_brec);
      smem = planar_smem_bytes(c, b->TP, (int)b->K, nullptr, nullptr, true);
    }
    if (a.brec && a.tlist) {
      GSVR_TRY(ensure_smem((const void *)k_train_planar<true, true>, smem));
      k_train_planar<true, true><<<blocks, kPB, smem, st>>>(a, c, b->TP);
    } else if (a.brec) {
      GSVR_TRY(ensure_smem((const void *)k_train_planar<true, false>, smem));
      k_train_planar<true, false><<<blocks, kPB, smem, st>>>(a, c, b->TP);
    } else if (a.tlist) {
      GSVR_TRY(ensure_smem((const void *)k_train_planar<false, true>, smem));
      k_train_planar<false, true><<<blocks, kPB, smem, st>>>(a, c, b->TP);
    } else {
      GSVR_TRY(ensure_smem((const void *)k_train_planar<false, false>, smem));
      k_train_planar<false, false><<<blocks, kPB, smem, st>>>(a, c, b->TP);
    }
    GSVR_LAUNCH_CHECK("k_train_planar");
    return GSVR_OK;
  };
  // tiles of very different unique counts (cfg4: median 526, max 899): two
  // launches, the tiles whose records fit a full-residency page first
  static const int forced_bucket_cap = [] {  // tests: bucket at a given page size
    const char *v = std::getenv("GSVR_TILE_BUCKET_CAP");
    return v ? std::max(1, std::atoi(v)) : 0;
  }();
  if (allow_buckets && (!fits(cap) || (forced_bucket_cap && forced_bucket_cap < cap)) &&
      (int64_t)b->h_nu.size() == b->T) {
    if (!b->buckets_valid) {
      int cs = cap;
      while (cs > 1 && !fits(cs)) --cs;
      if (forced_bucket_cap) cs = std::min(cs, forced_bucket_cap);
      std::vector<int32_t> lists;
      lists.reserve(b->T);
      for (int64_t t = 0; t < b->T; ++t)
        if (b->h_nu[t] <= cs) lists.push_back((int32_t)t);
      b->n_small = (int64_t)lists.size();
      for (int64_t t = 0; t < b->T; ++t)
        if (b->h_nu[t] > cs) lists.push_back((int32_t)t);
      b->n_large = (int64_t)lists.size() - b->n_small;
      b->bucket_cap = cs;
      GSVR_TRY(grow(b->tile_buckets, b->cap_tile_buckets, lists.size() * 4 + 16, st));
      GSVR_CUDA(cudaMemcpyAsync(b->tile_buckets, lists.data(), lists.size() * 4, cudaMemcpyHostToDevice, st));
      GSVR_CUDA(cudaStreamSynchronize(st));  // `lists` is pageable host memory
      b->buckets_valid = true;
    }
    kernel_timer().before(st);
    if (b->n_small > 0) {
      a.tlist = b->tile_buckets;
      GSVR_TRY(launch(b->bucket_cap, (unsigned)b->n_small, false));
    }
    if (b->n_large > 0) {
      a.tlist = b->tile_buckets + b->n_small;
      GSVR_TRY(launch(cap, (unsigned)b->n_large, true));
    }
    kernel_timer().after(st);
  } else {
    kernel_timer().before(st);
    GSVR_TRY(launch(cap, (unsigned)b->T, true));
    kernel_timer().after(st);
  }
  GSVR_TRY(gather_grads(b, dfield, dslice, st));
  return GSVR_OK;
}

}  // namespace gsvr
