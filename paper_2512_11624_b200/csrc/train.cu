// train.cu -- the fused tile kernel: forward (Eq.5) + L1 residual + all analytic
// gradients of kernels.py:78-198, restructured for B200.
//
// One CTA per (slice, tile).  Per tile:
//  1. Gaussian records (fp64 -> fp32), one per UNIQUE Gaussian of the tile:
//       Sigma_obs^-1 = (Sigma_j + Sigma_PSF,s)^-1, pre-scaled by -log2(e)/2, and
//       D_j = (Rc_s o_t + t_s) - mu_j   (o_t = tile origin)
//     so the per-pair form is u2 = v^T M' v with v = Rc_s d0_p + D_j, where d0_p is
//     the fp32 tile-relative nominal offset (|d0| ~ tile size): no large-magnitude
//     cancellation in fp32.  The reference recomputes the inverse per pair
//     (kernels.py:113-115); here it is hoisted to (slice, tile, Gaussian).
//     Records are staged in shared memory (SoA, 40 B) for the random gathers.
//  2. Pixel-major forward: thread per pixel, K gathers from shared memory,
//     exp2 on the MUFU pipe, num/den, ratio, residual, L1 sign (kernels.py:101-143).
//     Drop semantics: pairs with u < -80 contribute 0 (kernels.py:123-124).
//  3. Gaussian-major backward over the tile's pair list (sorted by Gaussian at
//     binning): each thread owns an equal chunk of pairs, keeps the current
//     Gaussian's record and its 10 gradient sums in registers and flushes them
//     with one fire-and-forget global reduction per (segment, component)
//     instead of 10 atomics per pair (kernels.py:157-186).  Slice gradients
//     (dt, dRc, dpsf6, dsigma, L1) are block-reduced and added once per tile.
#include <cub/block/block_reduce.cuh>
#include <atomic>
#include <condition_variable>
#include <mutex>
#include <thread>

#include "batch.cuh"

namespace gsvr {
// host_narrow.cpp: int64 neighbour ids -> int32 on the host (all cores) with
// the range check [0, N); nonzero if any id is out of range.
int narrow_ids_host(const int64_t *src, int32_t *dst, int64_t n, int64_t N, int threads);
void copy_host_parallel(void *dst, const void *src, int64_t bytes, int threads);
}  // namespace gsvr

namespace gsvr {


constexpr int kTrainBlock = 256;
constexpr int kRecCap = 2048;  // records staged in shared memory per page
static_assert(kRecCap >= kMinRecordPage, "global record pages are sized from kMinRecordPage");
constexpr float kCut2 = (float)(-80.0 * 1.4426950408889634);  // u < -80 in log2 units
constexpr float kLn2 = 0.69314718055994531f;

struct TileParams {
  const int64_t *tstart;
  const int32_t *tn;
  const int32_t *tslice;
  const double *torigin;
  const float4 *d0obs;
  const int32_t *perm;
  int K;
  const uint16_t *nbr_local;
  const uint16_t *pair_pix;
  const int64_t *nl_off, *pp_off;
  const int32_t *uoff;
  const int32_t *gid;
  const uint16_t *csr;
  float4 *rec;  // overflow pages: SoA in global, 3 float4 per record slot
  const double *mu, *cov6, *cvals;
  const double *Rc, *tvec, *psf6s, *sigma_s, *wdata_s;
  float delta;
  double delta64;
  const double *x0s, *iobs_s;  // float64 inputs of the L1 sign refinement (pixel_l1, batch.cuh)
  float *gpart;    // (U,10) per-(tile, Gaussian) partials [dmu dcov6 dc]
  double *tpart;   // (T, 20) per-tile slice partials  // (S,20) [dt dRc dpsf6 dsig l1]
  double *I_hat, *absres;
  unsigned long long *nonfinite_first;
};

__device__ inline void make_record(const TileParams &a, int64_t j, const double xT[3], const double p6[6],
                                   float4 &r0, float4 &r1, float2 &r2) {
  double S6[6], M[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) S6[e] = a.cov6[6 * j + e] + p6[e];
  inv_sym3<double>(S6, M);
  const double sc = -0.5 * kLog2e;
  r0 = make_float4((float)(xT[0] - a.mu[3 * j]), (float)(xT[1] - a.mu[3 * j + 1]),
                   (float)(xT[2] - a.mu[3 * j + 2]), (float)a.cvals[j]);
  r1 = make_float4((float)(M[0] * sc), (float)(M[1] * sc), (float)(M[2] * sc), (float)(M[3] * sc));
  r2 = make_float2((float)(M[4] * sc), (float)(M[5] * sc));
}

extern __shared__ float4 g_dyn_smem[];

__global__ void __launch_bounds__(kTrainBlock) k_train_tiles(TileParams a, int cap) {
  using BR = cub::BlockReduce<float, kTrainBlock>;
  __shared__ typename BR::TempStorage red;
  __shared__ float4 spix[2 * kTrainBlock];  // per pixel: (e.xyz, gnum), (d0.xyz, gden)
  __shared__ float sred[20];

  float4 *sA = g_dyn_smem;               // (D, c)
  float4 *sB = sA + cap;                 // M'0..3
  float2 *sC = reinterpret_cast<float2 *>(sB + cap);  // M'4..5

  const int t = blockIdx.x;
  const int tid = threadIdx.x;
  const int64_t ts = a.tstart[t];
  const int n = a.tn[t];
  const int s = a.tslice[t];
  const int K = a.K;
  const int u0 = a.uoff[t];
  const int nU = a.uoff[t + 1] - u0;
  const int npages = (nU + cap - 1) / cap;

  // slice parameters (fp64) and tile anchor x_T = Rc o + t
  double R[9], p6[6], xT[3];
#pragma unroll
  for (int e = 0; e < 9; ++e) R[e] = a.Rc[9 * s + e];
#pragma unroll
  for (int e = 0; e < 6; ++e) p6[e] = a.psf6s[6 * s + e];
  {
    const double o0 = a.torigin[3 * t], o1 = a.torigin[3 * t + 1], o2 = a.torigin[3 * t + 2];
    xT[0] = R[0] * o0 + R[1] * o1 + R[2] * o2 + a.tvec[3 * s];
    xT[1] = R[3] * o0 + R[4] * o1 + R[5] * o2 + a.tvec[3 * s + 1];
    xT[2] = R[6] * o0 + R[7] * o1 + R[8] * o2 + a.tvec[3 * s + 2];
  }
  const float sig = (float)a.sigma_s[s];
  const float wdat = (float)a.wdata_s[s];
  float Rf[9];
#pragma unroll
  for (int e = 0; e < 9; ++e) Rf[e] = (float)R[e];

  // ---- forward (pixel-major) -------------------------------------------
  const int p = tid;
  float4 d0o = make_float4(0.f, 0.f, 0.f, 0.f);
  float ex0 = 0.f, ex1 = 0.f, ex2 = 0.f;
  if (p < n) {
    d0o = a.d0obs[ts + p];
    ex0 = Rf[0] * d0o.x + Rf[1] * d0o.y + Rf[2] * d0o.z;
    ex1 = Rf[3] * d0o.x + Rf[4] * d0o.y + Rf[5] * d0o.z;
    ex2 = Rf[6] * d0o.x + Rf[7] * d0o.y + Rf[8] * d0o.z;
  }
  float num = 0.f, den = a.delta;
  const uint16_t *nl = a.nbr_local + a.nl_off[t];
  for (int page = 0; page < npages; ++page) {
    const int base = page * cap;
    const int cnt = min(cap, nU - base);
    if (page > 0) __syncthreads();
    for (int g = tid; g < cnt; g += kTrainBlock) {
      float4 r0, r1;
      float2 r2;
      make_record(a, a.gid[u0 + base + g], xT, p6, r0, r1, r2);
      sA[g] = r0;
      sB[g] = r1;
      sC[g] = r2;
      if (npages > 1) {
        float4 *gr = a.rec + 3 * (int64_t)(u0 + base + g);
        gr[0] = r0;
        gr[1] = r1;
        gr[2] = make_float4(r2.x, r2.y, 0.f, 0.f);
      }
    }
    __syncthreads();
    if (p < n) {
#pragma unroll 4
      for (int k = 0; k < K; ++k) {
        const unsigned lid = (unsigned)nl[nl_index(p, k, n)] - (unsigned)base;
        if (npages > 1 && lid >= (unsigned)cnt) continue;
        const float4 r0 = sA[lid], r1 = sB[lid];
        const float2 r2 = sC[lid];
        const float v0 = ex0 + r0.x, v1 = ex1 + r0.y, v2 = ex2 + r0.z;
        const float q0 = r1.x * v0 + r1.y * v1 + r1.z * v2;
        const float q1 = r1.y * v0 + r1.w * v1 + r2.x * v2;
        const float q2 = r1.z * v0 + r2.x * v1 + r2.y * v2;
        const float u2 = v0 * q0 + v1 * q1 + v2 * q2;
        const float e = (u2 < kCut2) ? 0.f : exp2f(u2);
        num = fmaf(r0.w, e, num);
        den += e;
      }
    }
  }

  // residual, L1 subgradient (kernels.py:133-143; fp64 sign refinement of
  // residuals within the fp32 render tolerance, batch.cuh pixel_l1), outputs
  float l1 = 0.f, dsig = 0.f;
  {
    const PixelL1 o = pixel_l1(p < n, num, den, d0o.w, sig, wdat, p, n, K, nl, a.gid + u0, a.x0s, ts, R,
                               a.tvec + 3 * s, p6, a.mu, a.cov6, a.cvals, a.sigma_s[s], a.delta64, a.iobs_s);
    if (p < n) {
      const int64_t dst = a.perm[ts + p];
      if (a.I_hat) a.I_hat[dst] = o.ihat_d;
      if (a.absres) a.absres[dst] = o.absr_d;
      if (a.nonfinite_first && !isfinite(o.ihat)) atomicMin(a.nonfinite_first, (unsigned long long)dst);
      l1 = fabsf(o.r);
      dsig = o.g * o.ratio;
      const float gout = o.g * sig;
      const float gnum = gout / den;
      const float gden = -gout * o.ratio / den;
      spix[2 * p] = make_float4(ex0, ex1, ex2, gnum);
      spix[2 * p + 1] = make_float4(d0o.x, d0o.y, d0o.z, gden);
    }
  }
  __syncthreads();

  // ---- backward (Gaussian-major) ----------------------------------------
  float dt0 = 0.f, dt1 = 0.f, dt2 = 0.f;
  float R00 = 0.f, R01 = 0.f, R02 = 0.f, R10 = 0.f, R11 = 0.f, R12 = 0.f, R20 = 0.f, R21 = 0.f, R22 = 0.f;
  float P00 = 0.f, P01 = 0.f, P02 = 0.f, P11 = 0.f, P12 = 0.f, P22 = 0.f;
  {
    const int m = n * K;
    const int chunk = (m + kTrainBlock - 1) / kTrainBlock;
    int i = tid * chunk;
    const int hi = min(i + chunk, m);
    if (i < hi) {
      const uint16_t *cs = a.csr + u0 + t;
      // last local Gaussian whose first pair is <= i
      int lo_g = 0, hi_g = nU - 1;
      while (lo_g < hi_g) {
        const int mid = (lo_g + hi_g + 1) >> 1;
        if ((int)cs[mid] <= i) lo_g = mid; else hi_g = mid - 1;
      }
      int g = lo_g;
      int gend = cs[g + 1];
      float4 r0, r1;
      float2 r2;
      auto load_rec = [&](int gg) {
        if (npages == 1) {
          r0 = sA[gg];
          r1 = sB[gg];
          r2 = sC[gg];
        } else {
          const float4 *gr = a.rec + 3 * (int64_t)(u0 + gg);
          r0 = gr[0];
          r1 = gr[1];
          const float4 t2 = gr[2];
          r2 = make_float2(t2.x, t2.y);
        }
      };
      load_rec(g);
      float am0 = 0.f, am1 = 0.f, am2 = 0.f, ac0 = 0.f, ac1 = 0.f, ac2 = 0.f, ac3 = 0.f, ac4 = 0.f,
            ac5 = 0.f, adc = 0.f;
      auto flush = [&](int gg) {
        float *df = a.gpart + 10 * (int64_t)(u0 + gg);
        atomicAdd(df + 0, am0); atomicAdd(df + 1, am1); atomicAdd(df + 2, am2);
        atomicAdd(df + 3, ac0); atomicAdd(df + 4, ac1); atomicAdd(df + 5, ac2);
        atomicAdd(df + 6, ac3); atomicAdd(df + 7, ac4); atomicAdd(df + 8, ac5);
        atomicAdd(df + 9, adc);
        P00 += ac0; P01 += ac1; P02 += ac2; P11 += ac3; P12 += ac4; P22 += ac5;
        am0 = am1 = am2 = ac0 = ac1 = ac2 = ac3 = ac4 = ac5 = adc = 0.f;
      };
      const uint16_t *pp = a.pair_pix + a.pp_off[t] + tid * 8;
      const int lo_i = i;
      for (; i < hi; ++i) {
        if (i >= gend) {
          flush(g);
          ++g;
          gend = cs[g + 1];
          load_rec(g);
        }
        const int r = i - lo_i;
        const int px = pp[(int64_t)(r >> 3) * kChunkThreads * 8 + (r & 7)];
        const float4 A = spix[2 * px], B = spix[2 * px + 1];
        const float v0 = A.x + r0.x, v1 = A.y + r0.y, v2 = A.z + r0.z;
        const float q0 = r1.x * v0 + r1.y * v1 + r1.z * v2;
        const float q1 = r1.y * v0 + r1.w * v1 + r2.x * v2;
        const float q2 = r1.z * v0 + r2.x * v1 + r2.y * v2;
        const float u2 = v0 * q0 + v1 * q1 + v2 * q2;
        if (u2 < kCut2) continue;
        const float e = exp2f(u2);
        adc = fmaf(A.w, e, adc);                         // dc += gnum e
        const float aa = (A.w * r0.w + B.w) * e;         // a = (gnum c + gden) e
        // w = Sigma_obs^-1 v = q * (-2 ln 2);  a w and (a/2) w w^T
        const float aw_s = aa * (-2.f * kLn2);
        const float aw0 = aw_s * q0, aw1 = aw_s * q1, aw2 = aw_s * q2;
        am0 += aw0; am1 += aw1; am2 += aw2;
        dt0 -= aw0; dt1 -= aw1; dt2 -= aw2;
        R00 = fmaf(-aw0, B.x, R00); R01 = fmaf(-aw0, B.y, R01); R02 = fmaf(-aw0, B.z, R02);
        R10 = fmaf(-aw1, B.x, R10); R11 = fmaf(-aw1, B.y, R11); R12 = fmaf(-aw1, B.z, R12);
        R20 = fmaf(-aw2, B.x, R20); R21 = fmaf(-aw2, B.y, R21); R22 = fmaf(-aw2, B.z, R22);
        const float h0 = aw0 * (-kLn2), h1 = aw1 * (-kLn2), h2 = aw2 * (-kLn2);  // (a/2) w_i
        ac0 = fmaf(h0, q0, ac0); ac1 = fmaf(h0, q1, ac1); ac2 = fmaf(h0, q2, ac2);
        ac3 = fmaf(h1, q1, ac3); ac4 = fmaf(h1, q2, ac4); ac5 = fmaf(h2, q2, ac5);
      }
      flush(g);
    }
  }

  // ---- slice gradients: block reduction, one fp64 add per tile ------------
  float vals[20] = {dt0, dt1, dt2, R00, R01, R02, R10, R11, R12, R20, R21, R22,
                    P00, P01, P02, P11, P12, P22, dsig, l1};
#pragma unroll
  for (int e = 0; e < 20; ++e) {
    float tot = BR(red).Sum(vals[e]);
    if (tid == 0) sred[e] = tot;
    __syncthreads();
  }
  if (tid < 20) {
    double val = (double)sred[tid];
    if (tid >= 3 && tid < 12) {
      // dRc = sum_p gx_p x0_p^T = sum gx d0^T + (sum gx) o^T
      const int r = (tid - 3) / 3, c = (tid - 3) % 3;
      val += (double)sred[r] * a.torigin[3 * t + c];
    }
    a.tpart[20 * (int64_t)t + tid] = val;
  }
}

bool force_general = false;  // diagnostics: run the general 3D kernel on planar batches
bool force_brec_global = false;  // diagnostics: planar kernel with backward records in global memory

int train_tiles(const gsvr_batch *b, int64_t S, int64_t N, const double *Rc, const double *tvec,
                const double *psf6s, const double *sigma_s, const double *wdata_s, const double *mu,
                const double *cov6, const double *cvals, double delta, float *dfield, double *dslice,
                double *I_hat, double *absres, unsigned long long *nonfinite_first, cudaStream_t st) {
  if (!b->nbr_local) return fail(GSVR_ERR_INVALID, "batch has no binned neighbour lists");
  if (b->N != N) return fail(GSVR_ERR_INVALID, "binning was built for %lld primitives, got %lld",
                             (long long)b->N, (long long)N);
  if (b->planar && !force_general)
    return train_tiles_planar(b, S, N, Rc, tvec, psf6s, sigma_s, wdata_s, mu, cov6, cvals, delta, dfield, dslice,
                              I_hat, absres, nonfinite_first, st);
  if (b->TP > kTrainBlock) return fail(GSVR_ERR_INVALID, "tile_points must be <= %d", kTrainBlock);
  if (b->N != N) return fail(GSVR_ERR_INVALID, "binning was built for %lld primitives, got %lld",
                             (long long)b->N, (long long)N);
  TileParams a;
  a.tstart = b->tile_start; a.tn = b->tile_n; a.tslice = b->tile_slice; a.torigin = b->tile_origin;
  a.d0obs = b->d0obs; a.perm = b->perm; a.K = (int)b->K;
  a.nbr_local = b->nbr_local; a.pair_pix = b->pair_pix; a.uoff = b->uoff; a.gid = b->gid; a.csr = b->csr;
  a.nl_off = b->nl_off; a.pp_off = b->pp_off;
  a.rec = b->rec;
  a.mu = mu; a.cov6 = cov6; a.cvals = cvals;
  a.Rc = Rc; a.tvec = tvec; a.psf6s = psf6s; a.sigma_s = sigma_s; a.wdata_s = wdata_s;
  a.delta = (float)delta;
  a.delta64 = delta;
  a.x0s = b->x0s;
  a.iobs_s = b->iobs_s;
  a.gpart = b->gpart; a.tpart = b->tpart; a.I_hat = I_hat; a.absres = absres;
  a.nonfinite_first = nonfinite_first;
  const int cap = std::max(1, std::min(b->max_unique, kRecCap));
  const size_t smem = (size_t)cap * 40;
  GSVR_TRY(ensure_smem((const void *)k_train_tiles, (size_t)kRecCap * 40));
  GSVR_CUDA(cudaMemsetAsync(b->gpart, 0, (size_t)b->U * 40, st));
  kernel_timer().before(st);
  k_train_tiles<<<(unsigned)b->T, kTrainBlock, smem, st>>>(a, cap);
  kernel_timer().after(st);
  GSVR_LAUNCH_CHECK("k_train_tiles");
  GSVR_TRY(gather_grads(b, dfield, dslice, st));
  return GSVR_OK;
}

// ---------------------------------------------------------------------------
// staleness (train.py:457-461): max_p |x_a(p) - x_b(p)|^2 with x = Rc x0 + t

__device__ inline double stale_d2(const double *A, const double *ta, const double *B, const double *tb,
                                  double a0, double a1, double a2) {
  double d2 = 0.0;
#pragma unroll
  for (int r = 0; r < 3; ++r) {
    double xa = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(A[3 * r], a0), __dmul_rn(A[3 * r + 1], a1)),
                                    __dmul_rn(A[3 * r + 2], a2)), ta[r]);
    double xb = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(B[3 * r], a0), __dmul_rn(B[3 * r + 1], a1)),
                                    __dmul_rn(B[3 * r + 2], a2)), tb[r]);
    double d = __dsub_rn(xa, xb);
    d2 = __dadd_rn(d2, __dmul_rn(d, d));
  }
  return d2;
}

// Pass 1 (one thread per tile): the exact value at the tile's first point (a
// lower bound of the max) and an upper bound over the whole tile,
// (|D o + c| + ||D||_F r)^2 with D = Ra - Rb, c = ta - tb, o / r the tile's
// centroid / radius, inflated well past fp64 rounding.
__global__ void __launch_bounds__(256) k_disp_bounds(int64_t T, const int64_t *__restrict__ tstart,
                                                     const int32_t *__restrict__ tslice,
                                                     const double *__restrict__ origin,
                                                     const double *__restrict__ radius,
                                                     const double *__restrict__ x0s, const double *Ra,
                                                     const double *ta, const double *Rb, const double *tb,
                                                     double *__restrict__ ub, double *lower, double *out) {
  using BR = cub::BlockReduce<double, 256>;
  __shared__ typename BR::TempStorage tmp;
  double lo = 0.0;
  for (int64_t t = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; t < T; t += (int64_t)gridDim.x * blockDim.x) {
    const int s = tslice[t];
    const double *A = Ra + 9 * s, *B = Rb + 9 * s;
    const int64_t i = tstart[t];
    lo = fmax(lo, stale_d2(A, ta + 3 * s, B, tb + 3 * s, x0s[3 * i], x0s[3 * i + 1], x0s[3 * i + 2]));
    double fro = 0.0, cn = 0.0;
#pragma unroll
    for (int r = 0; r < 3; ++r) {
      double v = ta[3 * s + r] - tb[3 * s + r];
#pragma unroll
      for (int k = 0; k < 3; ++k) {
        const double d = A[3 * r + k] - B[3 * r + k];
        fro += d * d;
        v += d * origin[3 * t + k];
      }
      cn += v * v;
    }
    const double u = sqrt(cn) + sqrt(fro) * radius[t];
    ub[t] = (u * (1.0 + 1e-9) + 1e-9) * (u * (1.0 + 1e-9) + 1e-9);
  }
  const double bl = BR(tmp).Reduce(lo, cub::Max());
  if (threadIdx.x == 0) {
    lower[blockIdx.x] = bl;  // per-block maxima: no zeroed accumulator needed
    if (blockIdx.x == 0) *out = 0.0;  // pass 2 max-accumulates into it
  }
}

// Pass 2 (one block per tile): every point of a tile whose bound reaches the
// lower bound, exactly as train.py:457-461 (x = Rc x0 + t at both states).
// Pass 2 (one warp per tile, grid-stride): every point of a tile whose bound
// reaches the lower bound, exactly as train.py:457-461 (x = Rc x0 + t at both
// states).
__global__ void __launch_bounds__(256) k_disp_points(int64_t T, const int64_t *__restrict__ tstart,
                                                     const int32_t *__restrict__ tn,
                                                     const int32_t *__restrict__ tslice,
                                                     const double *__restrict__ ub,
                                                     const double *__restrict__ x0s, const double *Ra,
                                                     const double *ta, const double *Rb, const double *tb,
                                                     const double *lower, int nlower, double *out) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t)gridDim.x * (blockDim.x >> 5);
  __shared__ double s_lo;
  if (threadIdx.x < 32) {
    double l = 0.0;
    for (int k = lane; k < nlower; k += 32) l = fmax(l, lower[k]);
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) l = fmax(l, __shfl_xor_sync(0xffffffffu, l, o));
    if (lane == 0) s_lo = l;
  }
  __syncthreads();
  const double lo = s_lo;
  double mx = 0.0;
  for (int64_t t = (blockIdx.x * (int64_t)blockDim.x + threadIdx.x) >> 5; t < T; t += warps) {
    if (ub[t] < lo) continue;  // no point of this tile can hold the maximum
    const int s = tslice[t];
    const int64_t s0 = tstart[t];
    for (int p = lane; p < tn[t]; p += 32) {
      const int64_t i = s0 + p;
      mx = fmax(mx, stale_d2(Ra + 9 * s, ta + 3 * s, Rb + 9 * s, tb + 3 * s, x0s[3 * i], x0s[3 * i + 1],
                             x0s[3 * i + 2]));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  if (lane == 0 && mx > 0.0) atomic_max_nonneg(out, mx);
}

// ---------------------------------------------------------------------------
// drop-in adapter: fp32 tile-reduced gradients -> the reference's fp64 buffers

__global__ void k_scatter_grads(int64_t N, int64_t S, const float *__restrict__ dfield,
                                const double *__restrict__ dslice, double *dmu, double *dcov6, double *dc,
                                double *dt, double *dRc, double *dpsf6, double *dsig) {
  const int64_t tot = N + S;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < tot; i += (int64_t)gridDim.x * blockDim.x) {
    if (i < N) {
      const float *f = dfield + 10 * i;
      for (int e = 0; e < 3; ++e) dmu[3 * i + e] += (double)f[e];
      for (int e = 0; e < 6; ++e) dcov6[6 * i + e] += (double)f[3 + e];
      dc[i] += (double)f[9];
    } else {
      const int64_t s = i - N;
      const double *d = dslice + 20 * s;
      for (int e = 0; e < 3; ++e) dt[3 * s + e] += d[e];
      for (int e = 0; e < 9; ++e) dRc[9 * s + e] += d[3 + e];
      for (int e = 0; e < 6; ++e) dpsf6[6 * s + e] += d[12 + e];
      dsig[s] += d[18];
    }
  }
}

// per-tile largest caller row (readiness of a tile during a chunked upload)
__global__ void k_tile_maxrow(const int64_t *__restrict__ tstart, const int32_t *__restrict__ tn,
                              const int32_t *__restrict__ perm, int32_t *__restrict__ out) {
  const int t = blockIdx.x;
  const int64_t s0 = tstart[t];
  int mx = -1;
  for (int p = threadIdx.x; p < tn[t]; p += blockDim.x) mx = max(mx, perm[s0 + p]);
  mx = __reduce_max_sync(0xffffffffu, mx);
  __shared__ int wm[8];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = mx;
  __syncthreads();
  if (threadIdx.x == 0) {
    for (int w = 1; w < (int)(blockDim.x >> 5); ++w) mx = max(mx, wm[w]);
    out[t] = max(mx, wm[0]);
  }
}

// tiles grouped by the upload chunk that completes them (one block; order
// within a chunk is irrelevant: tiles are binned independently)
// int64 -> int32 neighbour ids on the device with the range check (the chunks
// of the host drop-in that cross PCIe unnarrowed)
__global__ void k_narrow_ids(int64_t n, const int64_t *__restrict__ src, int32_t *__restrict__ dst, int64_t N,
                             int *bad) {
  for (int64_t e = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; e < n; e += (int64_t)gridDim.x * blockDim.x) {
    const int64_t v = src[e];
    if ((uint64_t)v >= (uint64_t)N) *bad = 1;
    dst[e] = (int32_t)v;
  }
}

constexpr int kReadyMaxChunks = 63;
__global__ void __launch_bounds__(1024) k_ready_order(int64_t T, const int32_t *__restrict__ maxrow, int64_t rows, int nch,
                              int32_t *__restrict__ order, int64_t *__restrict__ first) {
  __shared__ int cnt[kReadyMaxChunks + 1], pos[kReadyMaxChunks + 1];
  if (threadIdx.x <= nch) cnt[threadIdx.x] = 0;
  __syncthreads();
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) atomicAdd(&cnt[maxrow[t] / rows], 1);
  __syncthreads();
  if (threadIdx.x == 0) {
    int acc = 0;
    for (int c = 0; c < nch; ++c) {
      pos[c] = acc;
      first[c] = acc;
      acc += cnt[c];
    }
    first[nch] = acc;
  }
  __syncthreads();
  for (int64_t t = threadIdx.x; t < T; t += blockDim.x) order[atomicAdd(&pos[maxrow[t] / rows], 1)] = (int32_t)t;
}

}  // namespace gsvr

using namespace gsvr;

extern "C" {

int gsvr_train_tiles(const gsvr_batch *b, int64_t S, int64_t N, const double *Rc, const double *tvec,
                     const double *psf6s, const double *sigma_s, const double *wdata_s, const double *mu,
                     const double *cov6, const double *cvals, double delta, float *dfield, double *dslice,
                     double *I_hat, double *absres, unsigned long long *nonfinite_first, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (S != b->S) return fail(GSVR_ERR_INVALID, "slice count mismatch");
  return train_tiles(b, S, N, Rc, tvec, psf6s, sigma_s, wdata_s, mu, cov6, cvals, delta, dfield, dslice, I_hat,
                     absres, nonfinite_first, st);
}

int gsvr_batch_displacement(const gsvr_batch *b, const double *Rc_a, const double *t_a, const double *Rc_b,
                            const double *t_b, double *out, void *stream) {
  cudaStream_t st = as_stream(stream);
  // max over points of a convex function: only tiles whose bound reaches the
  // exact value at some point are scanned (same per-point formula -> same max)
  const int g1 = grid_for(b->T, 256);
  GSVR_TRY(grow(b->ws_disp, b->ws_disp_cap, (size_t)(b->T + g1) * 8, st));
  double *ub = reinterpret_cast<double *>(b->ws_disp), *lower = ub + b->T;
  k_disp_bounds<<<g1, 256, 0, st>>>(b->T, b->tile_start, b->tile_slice, b->tile_origin, b->tile_radius, b->x0s,
                                    Rc_a, t_a, Rc_b, t_b, ub, lower, out);
  k_disp_points<<<grid_for(b->T * 32, 256, 148 * 8), 256, 0, st>>>(b->T, b->tile_start, b->tile_n, b->tile_slice,
                                                                    ub, b->x0s, Rc_a, t_a, Rc_b, t_b, lower, g1,
                                                                    out);
  GSVR_LAUNCH_CHECK("k_displacement");
  return GSVR_OK;
}

int gsvr_train_step_backward(int64_t P, int64_t K, int64_t S, int64_t N, const double *x0pts,
                             const int32_t *sid, const double *Rc, const double *tvec, const double *psf6s,
                             const double *sigma_s, const double *wdata_s, const double *I_obs,
                             const void *nbr, int nbr_i64, const double *mu, const double *cov6,
                             const double *cvals, double delta, double *I_hat, double *absres, double *dmu,
                             double *dcov6, double *dc, double *dt, double *dRc, double *dpsf6,
                             double *dsigraw, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (P == 0) return GSVR_OK;
  if (P < 0 || K < 1 || S < 1 || N < 1) return fail(GSVR_ERR_INVALID, "bad train_step_backward sizes");
  const bool htrace = trace_enabled();
  const auto t_call = std::chrono::steady_clock::now();
  auto hmark = [&](const char *what) {
    if (htrace)
      std::fprintf(stderr, "[gsvr trace] dropin/%s at %.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count());
  };
  int tp = 256;
  while ((int64_t)tp * K > 65535 && tp > 1) tp >>= 1;
  if ((int64_t)tp * K > 65535) return fail(GSVR_ERR_INVALID, "K too large");
  gsvr_batch *b = nullptr;
  GSVR_TRY(batch_create(P, S, x0pts, sid, I_obs, tp, &b, st));
  struct Guard {
    gsvr_batch *b;
    ~Guard() { delete b; }
  } guard{b};
  GSVR_TRY(gsvr_batch_bin(b, K, N, nbr, nbr_i64, stream));
  Scratch df, ds;
  GSVR_TRY(df.alloc(N * 40, st));
  GSVR_TRY(ds.alloc(S * 160, st));
  GSVR_CUDA(cudaMemsetAsync(df.ptr, 0, N * 40, st));
  GSVR_CUDA(cudaMemsetAsync(ds.ptr, 0, S * 160, st));
  GSVR_TRY(train_tiles(b, S, N, Rc, tvec, psf6s, sigma_s, wdata_s, mu, cov6, cvals, delta, df.as<float>(),
                       ds.as<double>(), I_hat, absres, nullptr, st));
  k_scatter_grads<<<grid_for(N + S, 256), 256, 0, st>>>(N, S, df.as<float>(), ds.as<double>(), dmu, dcov6, dc, dt,
                                                        dRc, dpsf6, dsigraw);
  GSVR_LAUNCH_CHECK("k_scatter_grads");
  return GSVR_OK;
}

static int host_threads() {
  static const int n = [] {
    if (const char *v = std::getenv("GSVR_HOST_THREADS")) return std::max(1, std::atoi(v));
    // two per hardware thread: the narrowing pass is host-memory-latency bound
    // and more streams in flight measured faster (16-core host: 45.1 -> 42.7 ms/call)
    return (int)std::min(64u, 2 * std::max(1u, std::thread::hardware_concurrency()));
  }();
  return n;
}

// Host-buffer drop-in (numpy callers over an FFI): same arguments as
// gsvr_train_step_backward, every array a HOST pointer.  The neighbour lists
// (the bulk of the bytes) are uploaded in row chunks on a copy stream while the
// batch is planned; tiles are binned as soon as the rows they read have
// arrived, so the upload hides planning and binning.  int64 lists are narrowed
// to int32 by host threads into pinned staging slots first (ids are checked
// against N there), pipelined with the upload: the bus carries 4 B per id.  Gradients accumulate into
// the caller's buffers (kernels.py semantics), I_hat / absres are overwritten.
int gsvr_train_step_backward_host(int64_t P, int64_t K, int64_t S, int64_t N, const double *x0pts,
                                  const int32_t *sid, const double *Rc, const double *tvec, const double *psf6s,
                                  const double *sigma_s, const double *wdata_s, const double *I_obs,
                                  const void *nbr, int nbr_i64, const double *mu, const double *cov6,
                                  const double *cvals, double delta, double *I_hat, double *absres, double *dmu,
                                  double *dcov6, double *dc, double *dt, double *dRc, double *dpsf6,
                                  double *dsigraw, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (P == 0) return GSVR_OK;
  if (P < 0 || K < 1 || S < 1 || N < 1) return fail(GSVR_ERR_INVALID, "bad train_step_backward sizes");
  const bool htrace = trace_enabled();
  const auto t_call = std::chrono::steady_clock::now();
  auto hmark = [&](const char *what) {
    if (htrace)
      std::fprintf(stderr, "[gsvr trace] dropin/%s at %.3f ms\n", what,
                   std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_call).count());
  };
  int tp = 256;
  while ((int64_t)tp * K > 65535 && tp > 1) tp >>= 1;
  if ((int64_t)tp * K > 65535) return fail(GSVR_ERR_INVALID, "K too large");
  constexpr int kMaxChunks = 40, kSlots = 3;
  static_assert(kMaxChunks <= kReadyMaxChunks, "k_ready_order chunk table");
  // per-device copy stream, events and pinned staging (grow-only), guarded by
  // a per-device mutex held for the whole call: concurrent callers on one
  // device (ctypes releases the GIL) serialise instead of sharing the staging
  // slots and events; callers on different devices run in parallel
  struct HostDropinState {
    cudaStream_t cs = nullptr, cs2 = nullptr;  // small inputs / neighbour-id chunks
    cudaEvent_t ev[kMaxChunks + 2], slot_ev[kSlots], ev_raw, out_ev[8];
    char *stage = nullptr;
    size_t stage_cap = 0;
    char *stage_io = nullptr;  // pinned staging of pageable small inputs / outputs
    size_t stage_io_cap = 0;
  };
  constexpr int kMaxDevices = 64;
  static HostDropinState dstate[kMaxDevices];
  int cur_dev = 0;
  GSVR_CUDA(cudaGetDevice(&cur_dev));
  if (cur_dev < 0 || cur_dev >= kMaxDevices) return fail(GSVR_ERR_INVALID, "device ordinal %d unsupported", cur_dev);
  static std::mutex dmutex[kMaxDevices];
  std::lock_guard<std::mutex> call_lock(dmutex[cur_dev]);
  HostDropinState &hs = dstate[cur_dev];
  if (!hs.cs) {
    GSVR_CUDA(cudaStreamCreateWithFlags(&hs.cs, cudaStreamNonBlocking));
    GSVR_CUDA(cudaStreamCreateWithFlags(&hs.cs2, cudaStreamNonBlocking));
    for (auto &e : hs.ev) GSVR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    for (auto &e : hs.slot_ev) GSVR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    GSVR_CUDA(cudaEventCreateWithFlags(&hs.ev_raw, cudaEventDisableTiming));
    for (auto &e : hs.out_ev) GSVR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  cudaStream_t cs = hs.cs, cs2 = hs.cs2;
  cudaEvent_t *ev = hs.ev, *slot_ev = hs.slot_ev, ev_raw = hs.ev_raw;
  char *&stage = hs.stage;
  size_t &stage_cap = hs.stage_cap;
  cudaEvent_t ev_alloc = ev[kMaxChunks], ev_small = ev[kMaxChunks + 1];
  bool narrow = nbr_i64 != 0;  // device copy is int32 either way
  const size_t esz = 4, hsz = nbr_i64 ? 8 : 4;
  const size_t npar = (size_t)S * 20, nfld = (size_t)N * 10, ngr = (size_t)N * 10 + (size_t)S * 20;
  Scratch d_x0, d_sid, d_iobs, d_par, d_fld, d_nbr, d_out, d_gr, bad, d_raw;
  struct CopyFence {  // destroyed before the buffers: no upload may target freed memory
    cudaStream_t s, s2;
    ~CopyFence() {
      cudaStreamSynchronize(s);
      cudaStreamSynchronize(s2);
    }
  } fence{cs, cs2};
  GSVR_TRY(d_x0.alloc(P * 24, st));
  GSVR_TRY(d_sid.alloc(P * 4, st));
  GSVR_TRY(d_iobs.alloc(P * 8, st));
  GSVR_TRY(d_par.alloc(npar * 8, st));
  GSVR_TRY(d_fld.alloc(nfld * 8, st));
  GSVR_TRY(d_nbr.alloc(P * K * esz, st));
  GSVR_TRY(d_out.alloc(P * 16, st));
  GSVR_TRY(d_gr.alloc(ngr * 8, st));
  GSVR_TRY(bad.alloc(4, st));
  GSVR_CUDA(cudaMemsetAsync(bad.ptr, 0, 4, st));
  double *par = d_par.as<double>(), *fld = d_fld.as<double>(), *gr = d_gr.as<double>();
  double *pRc = par, *ptv = pRc + 9 * S, *pp6 = ptv + 3 * S, *psg = pp6 + 6 * S, *pw = psg + S;
  double *fmu = fld, *fcov = fmu + 3 * N, *fc = fcov + 6 * N;
  double *gmu = gr, *gcov = gmu + 3 * N, *gc = gcov + 6 * N, *gt = gc + N, *gR = gt + 3 * S, *gp6 = gR + 9 * S,
         *gsg = gp6 + 6 * S;
  GSVR_CUDA(cudaEventRecord(ev_alloc, st));
  GSVR_CUDA(cudaStreamWaitEvent(cs, ev_alloc, 0));
  GSVR_CUDA(cudaStreamWaitEvent(cs2, ev_alloc, 0));
  // pageable caller buffers (plain numpy, as train.py:254-260 passes them) go
  // through pinned staging copied by host threads; page-locked ones are DMA'd
  // directly
  auto pageable = [](const void *ptr) {
    cudaPointerAttributes at;
    if (cudaPointerGetAttributes(&at, ptr) != cudaSuccess) {
      cudaGetLastError();
      return true;
    }
    return at.type == cudaMemoryTypeUnregistered;
  };
  const size_t in_bytes = (size_t)P * 36 + npar * 8 + nfld * 8 + ngr * 8;
  const size_t out_bytes = (size_t)P * 16 + ngr * 8;
  const size_t io_need = in_bytes + out_bytes + 64 * 32;
  if (hs.stage_io_cap < io_need) {
    if (hs.stage_io) cudaFreeHost(hs.stage_io);
    hs.stage_io = nullptr;
    hs.stage_io_cap = 0;
    GSVR_CUDA(cudaHostAlloc((void **)&hs.stage_io, io_need + io_need / 4, cudaHostAllocDefault));
    hs.stage_io_cap = io_need + io_need / 4;
  }
  size_t io_off = 0;
  auto up = [&](void *dst, const void *src, size_t bytes) {
    if (bytes && pageable(src)) {
      char *slot = hs.stage_io + io_off;
      io_off += (bytes + 63) / 64 * 64;
      copy_host_parallel(slot, src, (int64_t)bytes, host_threads());
      src = slot;
    }
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, cs);
  };
  // pageable int32 lists also go through the host-thread staging slots
  const bool ids_pageable = pageable(nbr);
  narrow = narrow || ids_pageable;
  // neighbour lists in row chunks (~64 MB of caller bytes; GSVR_UPLOAD_CHUNK_MB overrides)
  const int64_t nbytes = P * K * (int64_t)hsz;
  int64_t chunk_bytes = 64ll << 20;
  if (const char *v = std::getenv("GSVR_UPLOAD_CHUNK_MB")) chunk_bytes = std::max(1ll, std::atoll(v)) << 20;
  const int nch = (int)std::min<int64_t>(kMaxChunks, std::max<int64_t>(1, nbytes / chunk_bytes));
  const int64_t rows = (P + nch - 1) / nch;
  std::atomic<int> produced{0}, host_bad{0};
  std::mutex mu_p;
  std::condition_variable cv_p;
  if (!narrow) {
    for (int c = 0; c < nch; ++c) {
      const int64_t r0 = c * rows, r1 = std::min(P, r0 + rows);
      if (r1 > r0)
        GSVR_CUDA(cudaMemcpyAsync(d_nbr.as<char>() + r0 * K * esz, (const char *)nbr + r0 * K * esz,
                                  (r1 - r0) * K * esz, cudaMemcpyHostToDevice, cs2));
      GSVR_CUDA(cudaEventRecord(ev[c], cs2));
    }
    produced.store(nch);
  } else {
    const size_t slot_bytes = ((size_t)rows * K * 4 + 4095) / 4096 * 4096;  // 32-byte streaming stores
    if (stage_cap < slot_bytes * kSlots) {
      if (stage) {
        for (int k = 0; k < kSlots; ++k) cudaEventSynchronize(slot_ev[k]);
        cudaFreeHost(stage);
        stage = nullptr;
        stage_cap = 0;
      }
      GSVR_CUDA(cudaHostAlloc((void **)&stage, slot_bytes * kSlots, cudaHostAllocDefault));
      stage_cap = slot_bytes * kSlots;
    }
  }
  // host narrowing runs at the host's memory bandwidth, the copy engine at
  // PCIe's: every raw_every-th chunk crosses unnarrowed (8 B per id) and is
  // narrowed on the device, balancing the two (GSVR_RAW_EVERY, 0 = never)
  // (pageable lists: the copy engine cannot read them directly at full speed,
  // so every chunk is narrowed / staged by host threads)
  int raw_every = ids_pageable || !nbr_i64 ? 0 : 3;
  if (const char *v = std::getenv("GSVR_RAW_EVERY"); v && !ids_pageable && nbr_i64) raw_every = std::max(0, std::atoi(v));
  if (narrow && raw_every > 0 && nch >= raw_every) {
    GSVR_TRY(d_raw.alloc((size_t)rows * K * 8, st));
    GSVR_CUDA(cudaEventRecord(ev_raw, st));  // stream-ordered allocation -> visible to cs2
    GSVR_CUDA(cudaStreamWaitEvent(cs2, ev_raw, 0));
  }
  const bool use_raw = d_raw.ptr != nullptr;
  const int dev = cur_dev;
  // producer: narrow chunk c into slot c % kSlots (once its previous upload has
  // drained), queue its upload, publish ev[c]
  auto produce = [&] {
    cudaSetDevice(dev);
    for (int c = 0; c < nch; ++c) {
      const int64_t r0 = c * rows, r1 = std::min(P, r0 + rows);
      const int slot = c % kSlots;
      if (r1 > r0 && use_raw && c % raw_every == raw_every - 1) {
        cudaMemcpyAsync(d_raw.ptr, reinterpret_cast<const int64_t *>(nbr) + r0 * K, (r1 - r0) * K * 8,
                        cudaMemcpyHostToDevice, cs2);
        k_narrow_ids<<<grid_for((r1 - r0) * K, 256), 256, 0, cs2>>>((r1 - r0) * K, d_raw.as<int64_t>(),
                                                                   d_nbr.as<int32_t>() + r0 * K, N, bad.as<int>());
      } else if (r1 > r0) {
        if (c >= kSlots) cudaEventSynchronize(slot_ev[slot]);
        int32_t *sl = reinterpret_cast<int32_t *>(stage + (size_t)slot * (stage_cap / kSlots));
        if (nbr_i64) {
          if (narrow_ids_host(reinterpret_cast<const int64_t *>(nbr) + r0 * K, sl, (r1 - r0) * K, N, host_threads()))
            host_bad.store(1);
        } else {  // pageable int32: plain staged copy (ids checked on the device by the binning)
          copy_host_parallel(sl, reinterpret_cast<const int32_t *>(nbr) + r0 * K, (r1 - r0) * K * 4, host_threads());
        }
        cudaMemcpyAsync(d_nbr.as<int32_t>() + r0 * K, sl, (r1 - r0) * K * 4, cudaMemcpyHostToDevice, cs2);
        cudaEventRecord(slot_ev[slot], cs2);
      }
      cudaEventRecord(ev[c], cs2);
      if (c == nch - 1) hmark("ids staged");
      {
        std::lock_guard<std::mutex> lk(mu_p);
        produced.store(c + 1);
      }
      cv_p.notify_all();
    }
  };
  struct Joiner {  // destroyed before the fence and the buffers
    std::thread t;
    ~Joiner() {
      if (t.joinable()) t.join();
    }
  } producer;
  if (narrow) producer.t = std::thread(produce);
  // planning inputs first, then parameters and the caller's gradient buffers
  // (staged by this thread while the producer narrows the id chunks)
  GSVR_CUDA(up(d_x0.ptr, x0pts, P * 24));
  GSVR_CUDA(up(d_sid.ptr, sid, P * 4));
  GSVR_CUDA(up(d_iobs.ptr, I_obs, P * 8));
  GSVR_CUDA(up(pRc, Rc, S * 72));
  GSVR_CUDA(up(ptv, tvec, S * 24));
  GSVR_CUDA(up(pp6, psf6s, S * 48));
  GSVR_CUDA(up(psg, sigma_s, S * 8));
  GSVR_CUDA(up(pw, wdata_s, S * 8));
  GSVR_CUDA(up(fmu, mu, N * 24));
  GSVR_CUDA(up(fcov, cov6, N * 48));
  GSVR_CUDA(up(fc, cvals, N * 8));
  GSVR_CUDA(up(gmu, dmu, N * 24));
  GSVR_CUDA(up(gcov, dcov6, N * 48));
  GSVR_CUDA(up(gc, dc, N * 8));
  GSVR_CUDA(up(gt, dt, S * 24));
  GSVR_CUDA(up(gR, dRc, S * 72));
  GSVR_CUDA(up(gp6, dpsf6, S * 48));
  GSVR_CUDA(up(gsg, dsigraw, S * 8));
  GSVR_CUDA(cudaEventRecord(ev_small, cs));
  hmark("small inputs staged");
  auto wait_chunk = [&](int c) {
    std::unique_lock<std::mutex> lk(mu_p);
    cv_p.wait(lk, [&] { return produced.load() > c; });
  };
  GSVR_CUDA(cudaStreamWaitEvent(st, ev_small, 0));
  gsvr_batch *b = nullptr;
  GSVR_TRY(batch_create(P, S, d_x0.as<double>(), d_sid.as<int32_t>(), d_iobs.as<double>(), tp, &b, st));
  struct Guard {
    gsvr_batch *b;
    ~Guard() { delete b; }
  } guard{b};
  BinPlan plan;
  GSVR_TRY(bin_prepare(b, K, N, st, &plan));
  const void *dn = d_nbr.ptr;
  if (plan.fast) {
    // tiles become ready when every caller row they read has arrived: bin them
    // straight from the uploaded rows (through perm), chunk by chunk
    BinSource src{dn, 0, b->perm, N, bad.as<int>()};
    std::vector<int64_t> first(nch + 1, 0);
    Scratch mr, list, fst;
    GSVR_TRY(mr.alloc(b->T * 4, st));
    GSVR_TRY(list.alloc(b->T * 4, st));
    GSVR_TRY(fst.alloc((nch + 1) * 8, st));
    k_tile_maxrow<<<(unsigned)b->T, 256, 0, st>>>(b->tile_start, b->tile_n, b->perm, mr.as<int32_t>());
    k_ready_order<<<1, 1024, 0, st>>>(b->T, mr.as<int32_t>(), rows, nch, list.as<int32_t>(), fst.as<int64_t>());
    GSVR_LAUNCH_CHECK("tile readiness");
    GSVR_CUDA(cudaMemcpyAsync(first.data(), fst.ptr, (nch + 1) * 8, cudaMemcpyDeviceToHost, st));
    GSVR_CUDA(cudaStreamSynchronize(st));
    Scratch ovl, ovc;  // overflow tiles of all chunks, handled once after the last
    GSVR_TRY(ovl.alloc((size_t)b->T * 4, st));
    GSVR_TRY(ovc.alloc(4, st));
    GSVR_CUDA(cudaMemsetAsync(ovc.ptr, 0, 4, st));
    plan.ov_list = ovl.as<int32_t>();
    plan.ov_count = ovc.as<int>();
    for (int c = 0; c < nch; ++c) {
      wait_chunk(c);
      GSVR_CUDA(cudaStreamWaitEvent(st, ev[c], 0));
      GSVR_TRY(bin_sort_tiles(b, K, plan, first[c], first[c + 1], st, list.as<int32_t>(), src));
    }
    GSVR_TRY(bin_flush_overflow(b, K, plan, st, src));
    GSVR_TRY(bin_finish(b, K, N, plan, st));
  } else {
    GSVR_CUDA(cudaMallocAsync((void **)&b->nbr_int, P * K * 4, st));
    wait_chunk(nch - 1);
    GSVR_CUDA(cudaStreamWaitEvent(st, ev[nch - 1], 0));
    GSVR_TRY(gather_nbr_rows(b, K, N, dn, 0, 0, P, bad.as<int>(), st));
    GSVR_TRY(batch_bin_internal(b, K, N, st));
  }
  int hbad = 0;
  GSVR_CUDA(cudaMemcpyAsync(&hbad, bad.ptr, 4, cudaMemcpyDeviceToHost, st));
  Scratch df, ds;
  GSVR_TRY(df.alloc(N * 40, st));
  GSVR_TRY(ds.alloc(S * 160, st));
  GSVR_CUDA(cudaMemsetAsync(df.ptr, 0, N * 40, st));
  GSVR_CUDA(cudaMemsetAsync(ds.ptr, 0, S * 160, st));
  double *oI = d_out.as<double>(), *oA = oI + P;
  GSVR_TRY(train_tiles(b, S, N, pRc, ptv, pp6, psg, pw, fmu, fcov, fc, delta, df.as<float>(), ds.as<double>(), oI,
                       oA, nullptr, st));
  k_scatter_grads<<<grid_for(N + S, 256), 256, 0, st>>>(N, S, df.as<float>(), ds.as<double>(), gmu, gcov, gc, gt,
                                                        gR, gp6, gsg);
  GSVR_LAUNCH_CHECK("k_scatter_grads");
  // pageable destinations: D2H into pinned staging, host threads copy out after the sync
  struct Pending {
    void *dst;
    const char *src;
    size_t bytes;
  };
  std::vector<Pending> copy_out;
  auto down = [&](void *dst, const void *src, size_t bytes) {
    if (bytes && pageable(dst)) {
      char *slot = hs.stage_io + io_off;
      io_off += (bytes + 63) / 64 * 64;
      copy_out.push_back({dst, slot, bytes});
      return cudaMemcpyAsync(slot, src, bytes, cudaMemcpyDeviceToHost, st);
    }
    return cudaMemcpyAsync(dst, src, bytes, cudaMemcpyDeviceToHost, st);
  };
  // the two per-pixel outputs (most of the bytes) leave in pieces: host threads
  // copy a landed piece into the caller's pageable array while the next one is
  // still crossing the bus
  struct Piece {
    void *dst;
    const char *src;
    size_t bytes;
    int ev;
  };
  std::vector<Piece> pieces;
  constexpr int kOutPieces = 4;
  auto down_pieces = [&](double *dst, const double *src, int64_t n) -> cudaError_t {
    if (n == 0) return cudaSuccess;
    if (!pageable(dst)) return cudaMemcpyAsync(dst, src, n * 8, cudaMemcpyDeviceToHost, st);
    char *slot = hs.stage_io + io_off;
    io_off += (n * 8 + 63) / 64 * 64;
    const int64_t per = (n + kOutPieces - 1) / kOutPieces;
    for (int64_t a0 = 0; a0 < n; a0 += per) {
      const int64_t len = std::min(per, n - a0);
      cudaError_t e = cudaMemcpyAsync(slot + a0 * 8, src + a0, len * 8, cudaMemcpyDeviceToHost, st);
      if (e == cudaSuccess) e = cudaEventRecord(hs.out_ev[pieces.size()], st);
      if (e != cudaSuccess) return e;
      pieces.push_back({dst + a0, slot + a0 * 8, (size_t)len * 8, (int)pieces.size()});
    }
    return cudaSuccess;
  };
  GSVR_CUDA(down_pieces(I_hat, oI, P));
  GSVR_CUDA(down_pieces(absres, oA, P));
  GSVR_CUDA(down(dmu, gmu, N * 24));
  GSVR_CUDA(down(dcov6, gcov, N * 48));
  GSVR_CUDA(down(dc, gc, N * 8));
  GSVR_CUDA(down(dt, gt, S * 24));
  GSVR_CUDA(down(dRc, gR, S * 72));
  GSVR_CUDA(down(dpsf6, gp6, S * 48));
  GSVR_CUDA(down(dsigraw, gsg, S * 8));
  hmark("all queued");
  for (const Piece &c : pieces) {
    GSVR_CUDA(cudaEventSynchronize(hs.out_ev[c.ev]));
    copy_host_parallel(c.dst, c.src, (int64_t)c.bytes, host_threads());
  }
  GSVR_CUDA(cudaStreamSynchronize(st));
  hmark("device done");
  if (producer.t.joinable()) producer.t.join();
  if (hbad || host_bad.load()) return fail(GSVR_ERR_INVALID, "neighbor id out of range");
  for (const Pending &c : copy_out) copy_host_parallel(c.dst, c.src, (int64_t)c.bytes, host_threads());
  hmark("outputs copied");
  return GSVR_OK;
}

// Device -> host copy into a caller buffer of any kind.  Pageable destinations
// (plain numpy) go through a ring of pinned staging pieces: the copy engine
// fills piece i + kRing while host threads move piece i out (streaming
// stores), instead of the driver's single-bounce-buffer pageable path.
int gsvr_copy_d2h(void *dst, const void *src, int64_t bytes, void *stream) {
  cudaStream_t st = as_stream(stream);
  if (bytes <= 0) return GSVR_OK;
  if (!dst || !src) return fail(GSVR_ERR_INVALID, "null pointer");
  cudaPointerAttributes at;
  bool pageable_dst = true;
  if (cudaPointerGetAttributes(&at, dst) == cudaSuccess) pageable_dst = at.type == cudaMemoryTypeUnregistered;
  else cudaGetLastError();
  if (!pageable_dst || bytes < (4 << 20)) {
    GSVR_CUDA(cudaMemcpyAsync(dst, src, (size_t)bytes, cudaMemcpyDeviceToHost, st));
    GSVR_CUDA(cudaStreamSynchronize(st));
    return GSVR_OK;
  }
  constexpr int kRing = 4;
  constexpr int64_t kPiece = 32 << 20;
  struct D2HState {
    char *stage = nullptr;
    cudaEvent_t ev[kRing];
    std::mutex mu;
  };
  static D2HState states[64];
  int dev = 0;
  GSVR_CUDA(cudaGetDevice(&dev));
  if (dev < 0 || dev >= 64) return fail(GSVR_ERR_INVALID, "device ordinal out of range");
  D2HState &ds = states[dev];
  std::lock_guard<std::mutex> lock(ds.mu);
  if (!ds.stage) {
    GSVR_CUDA(cudaHostAlloc((void **)&ds.stage, (size_t)kRing * kPiece, cudaHostAllocDefault));
    for (auto &e : ds.ev) GSVR_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
  }
  const int64_t npieces = (bytes + kPiece - 1) / kPiece;
  auto issue = [&](int64_t i) -> cudaError_t {
    const int64_t off = i * kPiece, len = std::min(kPiece, bytes - off);
    cudaError_t e = cudaMemcpyAsync(ds.stage + (i % kRing) * kPiece, static_cast<const char *>(src) + off,
                                    (size_t)len, cudaMemcpyDeviceToHost, st);
    if (e == cudaSuccess) e = cudaEventRecord(ds.ev[i % kRing], st);
    return e;
  };
  for (int64_t i = 0; i < std::min<int64_t>(kRing, npieces); ++i) GSVR_CUDA(issue(i));
  for (int64_t i = 0; i < npieces; ++i) {
    GSVR_CUDA(cudaEventSynchronize(ds.ev[i % kRing]));
    const int64_t off = i * kPiece, len = std::min(kPiece, bytes - off);
    copy_host_parallel(static_cast<char *>(dst) + off, ds.stage + (i % kRing) * kPiece, len, host_threads());
    if (i + kRing < npieces) GSVR_CUDA(issue(i + kRing));
  }
  return GSVR_OK;
}

int gsvr_set_kernel_variant(int general) {
  force_general = (general & 1) != 0;
  force_brec_global = (general & 2) != 0;
  return GSVR_OK;
}

int gsvr_batch_is_planar(const gsvr_batch *b) { return b && b->planar ? 1 : 0; }

}  // extern "C"
