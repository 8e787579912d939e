// field.cu -- per-primitive and per-slice O(N) / O(S) kernels around the hot pass:
//   * covariances from (log_scales, quaternions)            field.py:67-69, geometry.py:143-165
//   * scale-floor check                                      train.py:162-169
//   * covariance chain dcov6 -> (dls, dq) + regulariser      train.py:271-282
//   * slice inputs (Rc, R_eff, rotated PSF, sigma)           train.py:145-152
//   * slice chain (dRc, dpsf6, dsigraw) -> (dq_i, dlog_sigma) train.py:284-290
//   * AdamW fused with both chains (fit loop)                optim.py:69-88, train.py:470-479
// All float64, like the reference's parameter and optimiser state.
#include <cub/block/block_reduce.cuh>

#include "common.cuh"

namespace gsvr {

// ---------------------------------------------------------------------------
// primitive covariances (+ floor check, + scale-regulariser sum of squares)

__device__ inline void primitive_cov(const double *ls, const double *q, double c6[6],
                                     double R[9], double D[3]) {
  quat_to_rot(q, R);
  D[0] = exp(2.0 * ls[0]);
  D[1] = exp(2.0 * ls[1]);
  D[2] = exp(2.0 * ls[2]);
  rot_diag_rot_t(R, D, c6);
}

template <int BLOCK>
__global__ void __launch_bounds__(BLOCK) k_field_cov(int64_t N, const double *__restrict__ ls,
                                                     const double *__restrict__ q,
                                                     double *__restrict__ cov6, double s_target,
                                                     double *reg_sumsq,
                                                     unsigned long long *floor_first) {
  using BR = cub::BlockReduce<double, BLOCK>;
  __shared__ typename BR::TempStorage tmp;
  double acc = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)BLOCK + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * BLOCK) {
    double c6[6], R[9], D[3];
    primitive_cov(ls + 3 * j, q + 4 * j, c6, R, D);
#pragma unroll
    for (int e = 0; e < 6; ++e) cov6[6 * j + e] = c6[e];
    double s0 = exp(ls[3 * j]), s1 = exp(ls[3 * j + 1]), s2 = exp(ls[3 * j + 2]);
    double smin = fmin(fmin(s0, s1), s2);
    if (floor_first && smin * smin < kEigenFloor) atomicMin(floor_first, (unsigned long long)j);
    double d0 = s0 - s_target, d1 = s1 - s_target, d2 = s2 - s_target;
    acc += d0 * d0 + d1 * d1 + d2 * d2;
  }
  if (reg_sumsq) {
    double tot = BR(tmp).Sum(acc);
    if (threadIdx.x == 0) atomicAdd(reg_sumsq, tot);
  }
}

// train.py:271-282 for one primitive: G (packed, full-matrix convention) -> dls, dq.
__device__ inline void cov_chain(const double *ls, const double *q, const double g6[6],
                                 double lambda_reg, double s_target, double dls[3],
                                 double dq[4]) {
  double R[9], D[3], G[9], GR[9], dR[9];
  quat_to_rot(q, R);
  D[0] = exp(2.0 * ls[0]);
  D[1] = exp(2.0 * ls[1]);
  D[2] = exp(2.0 * ls[2]);
  unpack6(g6, G);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      GR[3 * i + k] = G[3 * i] * R[k] + G[3 * i + 1] * R[3 + k] + G[3 * i + 2] * R[6 + k];
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k) dR[3 * i + k] = 2.0 * GR[3 * i + k] * D[k];
  for (int k = 0; k < 3; ++k)
    dls[k] = 2.0 * D[k] * (R[k] * GR[k] + R[3 + k] * GR[3 + k] + R[6 + k] * GR[6 + k]);
  quat_vjp(q, dR, dq);
  if (lambda_reg > 0.0) {
    for (int k = 0; k < 3; ++k) {
      double s = exp(ls[k]);
      dls[k] = dls[k] + lambda_reg * 2.0 * (s - s_target) * s;
    }
  }
}

__global__ void k_field_chain(int64_t N, const double *__restrict__ ls, const double *__restrict__ q,
                              const double *__restrict__ dcov6, double lambda_reg,
                              double s_target, double *__restrict__ dls, double *__restrict__ dq) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * blockDim.x) {
    double g6[6], a[3], b[4];
    for (int e = 0; e < 6; ++e) g6[e] = dcov6[6 * j + e];
    cov_chain(ls + 3 * j, q + 4 * j, g6, lambda_reg, s_target, a, b);
    for (int e = 0; e < 3; ++e) dls[3 * j + e] = a[e];
    for (int e = 0; e < 4; ++e) dq[4 * j + e] = b[e];
  }
}

// optim.py:69-88 for one scalar (m, v in float64; decoupled weight decay).
struct AdamArgs {
  double beta1, beta2, eps, wd, bc1, bc2;
};
__device__ inline void adamw(double &p, double &m, double &v, double g, double lr,
                             const AdamArgs &a) {
  m = m * a.beta1;
  m = m + (1.0 - a.beta1) * g;
  v = v * a.beta2;
  v = v + (1.0 - a.beta2) * g * g;
  double upd = (m / a.bc1) / (sqrt(v / a.bc2) + a.eps);
  if (a.wd > 0.0) upd = upd + a.wd * p;
  p -= lr * upd;
}

// Deterministic grid sum: per-block partials, the last block to finish adds
// them in block order (no floating-point atomics -> bit-identical losses) and
// overwrites ws[0] (its previous value -> *prev_out when given).  The floor
// check's first index is reduced as max(~j) into ws[2] (0 = none), which the
// same last block publishes and re-arms, so the step needs no memsets.  All of
// it lives in the CALLER's workspace (kFieldWsDoubles doubles, zero-filled
// once): concurrent steps of different engines never share state.
//   ws[0] regulariser sum (f64 out)   ws[1] done-block counter (u32)
//   ws[2] floor flag max(~j) (u64)    ws[3 ..] per-block partials
constexpr int kMaxSumBlocks = 148 * 32;
constexpr int kFieldWsDoubles = 3 + kMaxSumBlocks;

template <int BLOCK>
__device__ inline void grid_sum_ordered(double block_total, double *ws, double *prev_out,
                                        unsigned long long *floor_out) {
  __shared__ bool last;
  double *partials = ws + 3;
  unsigned int *done = reinterpret_cast<unsigned int *>(ws + 1);
  unsigned long long *flag = reinterpret_cast<unsigned long long *>(ws + 2);
  if (threadIdx.x == 0) {
    partials[blockIdx.x] = block_total;
    __threadfence();
    last = atomicAdd(done, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (last && threadIdx.x == 0) {
    __threadfence();
    double s = 0.0;
    for (unsigned b = 0; b < gridDim.x; ++b) s += *(volatile double *)&partials[b];
    if (prev_out) *prev_out = ws[0];
    ws[0] = s;
    *floor_out = ~atomicExch(flag, 0ull);
    *done = 0;
  }
}

#ifndef GSVR_FIELD_MINB
#define GSVR_FIELD_MINB 3
#endif
// Fit-loop field step: chain the fp32 tile-reduced gradients, AdamW all 11
// parameters, zero the gradient buffer, then covariances / regulariser / floor
// check of the updated field (consumed by the next epoch).
template <int BLOCK>
__global__ void __launch_bounds__(BLOCK, GSVR_FIELD_MINB) k_field_step(
    int64_t N, double *__restrict__ mu, double *__restrict__ ls, double *__restrict__ q,
    double *__restrict__ c, double *__restrict__ m, double *__restrict__ v,
    float *__restrict__ dfield, double lambda_reg, double s_target, double4 lrs, double lr_scale,
    AdamArgs aa, int do_step, double *__restrict__ cov6, double *reg_sumsq, double *reg_prev,
    unsigned long long *floor_first) {
  using BR = cub::BlockReduce<double, BLOCK>;
  __shared__ typename BR::TempStorage tmp;
  double acc = 0.0;
  for (int64_t j = blockIdx.x * (int64_t)BLOCK + threadIdx.x; j < N;
       j += (int64_t)gridDim.x * BLOCK) {
    if (do_step) {
      float *df = dfield + 10 * j;
      double g6[6], dls[3], dq[4];
      for (int e = 0; e < 6; ++e) g6[e] = (double)df[3 + e];
      cov_chain(ls + 3 * j, q + 4 * j, g6, lambda_reg, s_target, dls, dq);
      double *mj = m + 11 * j, *vj = v + 11 * j;
      for (int e = 0; e < 3; ++e) adamw(mu[3 * j + e], mj[e], vj[e], (double)df[e], lrs.x * lr_scale, aa);
      for (int e = 0; e < 3; ++e) adamw(ls[3 * j + e], mj[3 + e], vj[3 + e], dls[e], lrs.y * lr_scale, aa);
      for (int e = 0; e < 4; ++e) adamw(q[4 * j + e], mj[6 + e], vj[6 + e], dq[e], lrs.z * lr_scale, aa);
      adamw(c[j], mj[10], vj[10], (double)df[9], lrs.w * lr_scale, aa);
#pragma unroll
      for (int e = 0; e < 10; ++e) df[e] = 0.f;
    }
    double c6[6], R[9], D[3];
    primitive_cov(ls + 3 * j, q + 4 * j, c6, R, D);
    for (int e = 0; e < 6; ++e) cov6[6 * j + e] = c6[e];
    double s0 = exp(ls[3 * j]), s1 = exp(ls[3 * j + 1]), s2 = exp(ls[3 * j + 2]);
    double smin = fmin(fmin(s0, s1), s2);
    if (smin * smin < kEigenFloor) atomicMax(reinterpret_cast<unsigned long long *>(reg_sumsq + 2), ~(unsigned long long)j);
    double d0 = s0 - s_target, d1 = s1 - s_target, d2 = s2 - s_target;
    acc += d0 * d0 + d1 * d1 + d2 * d2;
  }
  const double tot = BR(tmp).Sum(acc);
  grid_sum_ordered<BLOCK>(tot, reg_sumsq, reg_prev, floor_first);
}

// ---------------------------------------------------------------------------
// slices

// train.py:145-152 for one slice.
__device__ inline void slice_prep(const double q[4], const double Rs[9], const double pd[3],
                                  double Rc[9], double Reff[9], double p6[6]) {
  quat_to_rot(q, Rc);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      Reff[3 * i + k] = Rc[3 * i] * Rs[k] + Rc[3 * i + 1] * Rs[3 + k] + Rc[3 * i + 2] * Rs[6 + k];
  rot_diag_rot_t(Reff, pd, p6);
}

// train.py:284-289 for one slice: returns dq_i.
__device__ inline void slice_chain_one(const double q[4], const double Rs[9], const double pd[3],
                                       const double dRc[9], const double dp6[6], double dq[4]) {
  double Rc[9], Reff[9], p6[6], Gp[9], dReff[9], tot[9];
  slice_prep(q, Rs, pd, Rc, Reff, p6);
  unpack6(dp6, Gp);
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      dReff[3 * i + k] = 2.0 * (Gp[3 * i] * Reff[k] + Gp[3 * i + 1] * Reff[3 + k] +
                                Gp[3 * i + 2] * Reff[6 + k]) * pd[k];
  // dRc_total = dRc + dReff @ Rs^T
  for (int i = 0; i < 3; ++i)
    for (int k = 0; k < 3; ++k)
      tot[3 * i + k] = dRc[3 * i + k] + (dReff[3 * i] * Rs[3 * k] + dReff[3 * i + 1] * Rs[3 * k + 1] +
                                          dReff[3 * i + 2] * Rs[3 * k + 2]);
  quat_vjp(q, tot, dq);
}

__global__ void k_slice_inputs(int64_t S, const double *q, const double *Rs_all, const int32_t *s2t,
                               const double *log_sigma, const double *pdiag, double *Rc_out,
                               double *Reff_out, double *p6_out, double *sig_out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    double Rc[9], Reff[9], p6[6];
    slice_prep(q + 4 * s, Rs_all + 9 * s2t[s], pdiag + 3 * s, Rc, Reff, p6);
    if (Rc_out) for (int e = 0; e < 9; ++e) Rc_out[9 * s + e] = Rc[e];
    if (Reff_out) for (int e = 0; e < 9; ++e) Reff_out[9 * s + e] = Reff[e];
    if (p6_out) for (int e = 0; e < 6; ++e) p6_out[6 * s + e] = p6[e];
    if (sig_out) sig_out[s] = exp(log_sigma[s]);
  }
}

__global__ void k_slice_chain(int64_t S, const double *q, const double *Rs_all, const int32_t *s2t,
                              const double *log_sigma, const double *pdiag, const double *dRc,
                              const double *dp6, const double *dsig, double *dq_out,
                              double *dls_out) {
  for (int64_t s = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; s < S;
       s += (int64_t)gridDim.x * blockDim.x) {
    double dq[4];
    slice_chain_one(q + 4 * s, Rs_all + 9 * s2t[s], pdiag + 3 * s, dRc + 9 * s, dp6 + 6 * s, dq);
    for (int e = 0; e < 4; ++e) dq_out[4 * s + e] = dq[e];
    dls_out[s] = dsig[s] * exp(log_sigma[s]);
  }
}

// Fit-loop slice step (single block): loss terms of the current epoch, slice
// chain, masked AdamW (train.py:473-479), next-epoch slice inputs, zero grads.
// state (S,9) = [q(4) t(3) log_sigma eta]; dslice (S,20) = [dt dRc dpsf6 dsig l1].
constexpr int kSliceBlock = 256;
__global__ void __launch_bounds__(kSliceBlock) k_slice_step(
    int64_t S, double *state, double *m, double *v, double *dslice, const double *Rs_all,
    const int32_t *s2t, const double *pdiag, const double *counts, int outlier,
    double4 lrs, double lr_scale, AdamArgs aa, int step_mask, int64_t anchor, double *loss_out,
    double *Rc_out, double *t_out, double *p6_out, double *sig_out, double *w_out) {
  using BR = cub::BlockReduce<double, kSliceBlock>;
  __shared__ typename BR::TempStorage tmp;
  double data = 0.0, outl = 0.0, l1tot = 0.0;
  for (int64_t s = threadIdx.x; s < S; s += kSliceBlock) {
    double *st = state + 9 * s;
    double *ds = dslice + 20 * s;
    const double *Rs = Rs_all + 9 * s2t[s];
    const double *pd = pdiag + 3 * s;
    const double eta = st[8];
    const double wdat = outlier ? exp(-eta) : 1.0;
    const double l1 = ds[19];
    data += wdat * l1;
    l1tot += l1;
    if (outlier) outl += counts[s] * eta;
    if (step_mask & 1) {
      double g[9];
      slice_chain_one(st, Rs, pd, ds + 3, ds + 12, g);   // dq_i
      g[4] = ds[0]; g[5] = ds[1]; g[6] = ds[2];         // dt
      g[7] = ds[18] * exp(st[7]);                       // dlog_sigma
      g[8] = outlier ? (-wdat * l1 + counts[s]) : 0.0;  // deta
      if (step_mask & 2) g[0] = g[1] = g[2] = g[3] = 0.0;
      if (s == anchor) for (int e = 0; e < 9; ++e) g[e] = 0.0;
      const double lr[9] = {lrs.x, lrs.x, lrs.x, lrs.x, lrs.y, lrs.y, lrs.y, lrs.z, lrs.w};
      for (int e = 0; e < 9; ++e) adamw(st[e], m[9 * s + e], v[9 * s + e], g[e], lr[e] * lr_scale, aa);
    }
    for (int e = 0; e < 20; ++e) ds[e] = 0.0;
    double Rc[9], Reff[9], p6[6];
    slice_prep(st, Rs, pd, Rc, Reff, p6);
    for (int e = 0; e < 9; ++e) Rc_out[9 * s + e] = Rc[e];
    for (int e = 0; e < 3; ++e) t_out[3 * s + e] = st[4 + e];
    for (int e = 0; e < 6; ++e) p6_out[6 * s + e] = p6[e];
    sig_out[s] = exp(st[7]);
    w_out[s] = outlier ? exp(-st[8]) : 1.0;
  }
  double a = BR(tmp).Sum(data);
  __syncthreads();
  double b = BR(tmp).Sum(outl);
  __syncthreads();
  double c = BR(tmp).Sum(l1tot);
  if (threadIdx.x == 0) {
    loss_out[0] = a;
    loss_out[1] = b;
    loss_out[2] = c;
  }
}

}  // namespace gsvr

using namespace gsvr;

extern "C" {

int gsvr_field_covariances(int64_t N, const double *log_scales, const double *quats, double *cov6,
                           int check_floor, void *stream) {
  if (N < 0) return fail(GSVR_ERR_INVALID, "negative primitive count");
  if (N == 0) return GSVR_OK;
  cudaStream_t st = as_stream(stream);
  Scratch flag;
  unsigned long long *ff = nullptr;
  if (check_floor) {
    GSVR_TRY(flag.alloc(sizeof(unsigned long long), st));
    ff = flag.as<unsigned long long>();
    GSVR_CUDA(cudaMemsetAsync(ff, 0xff, sizeof(unsigned long long), st));
  }
  k_field_cov<256><<<grid_for(N, 256), 256, 0, st>>>(N, log_scales, quats, cov6, 0.0, nullptr, ff);
  GSVR_LAUNCH_CHECK("k_field_cov");
  if (check_floor) {
    unsigned long long h = 0;
    GSVR_CUDA(cudaMemcpyAsync(&h, ff, sizeof(h), cudaMemcpyDeviceToHost, st));
    GSVR_CUDA(cudaStreamSynchronize(st));
    if (h != ~0ull) {
      double l3[3];
      GSVR_CUDA(cudaMemcpy(l3, log_scales + 3 * h, sizeof(l3), cudaMemcpyDeviceToHost));
      double smin = fmin(fmin(exp(l3[0]), exp(l3[1])), exp(l3[2]));
      set_error(GSVR_ERR_DEGENERATE, "scale collapsed below the eigenvalue floor", (int64_t)h, smin);
      return GSVR_ERR_DEGENERATE;
    }
  }
  return GSVR_OK;
}

int gsvr_field_chain(int64_t N, const double *log_scales, const double *quats, const double *dcov6,
                     double lambda_reg, double s_target, double *dls, double *dq, void *stream) {
  if (N <= 0) return N == 0 ? GSVR_OK : fail(GSVR_ERR_INVALID, "negative primitive count");
  cudaStream_t st = as_stream(stream);
  k_field_chain<<<grid_for(N, 256), 256, 0, st>>>(N, log_scales, quats, dcov6, lambda_reg,
                                                   s_target, dls, dq);
  GSVR_LAUNCH_CHECK("k_field_chain");
  return GSVR_OK;
}

int gsvr_slice_inputs(int64_t S, const double *slice_quats, const double *stack_rots,
                      const int32_t *slice_to_stack, const double *log_sigma,
                      const double *psf_diags, double *Rc, double *R_eff, double *psf6s,
                      double *sigma_s, void *stream) {
  if (S <= 0) return S == 0 ? GSVR_OK : fail(GSVR_ERR_INVALID, "negative slice count");
  cudaStream_t st = as_stream(stream);
  k_slice_inputs<<<grid_for(S, 128), 128, 0, st>>>(S, slice_quats, stack_rots, slice_to_stack,
                                                    log_sigma, psf_diags, Rc, R_eff, psf6s, sigma_s);
  GSVR_LAUNCH_CHECK("k_slice_inputs");
  return GSVR_OK;
}

int gsvr_slice_chain(int64_t S, const double *slice_quats, const double *stack_rots,
                     const int32_t *slice_to_stack, const double *log_sigma,
                     const double *psf_diags, const double *dRc, const double *dpsf6,
                     const double *dsigraw, double *dq_slice, double *dlog_sigma, void *stream) {
  if (S <= 0) return S == 0 ? GSVR_OK : fail(GSVR_ERR_INVALID, "negative slice count");
  cudaStream_t st = as_stream(stream);
  k_slice_chain<<<grid_for(S, 128), 128, 0, st>>>(S, slice_quats, stack_rots, slice_to_stack,
                                                   log_sigma, psf_diags, dRc, dpsf6, dsigraw,
                                                   dq_slice, dlog_sigma);
  GSVR_LAUNCH_CHECK("k_slice_chain");
  return GSVR_OK;
}

int gsvr_field_adamw_step(int64_t N, double *means, double *log_scales, double *quats,
                          double *cvals, double *m, double *v, float *dfield, double lambda_reg,
                          double s_target, const double *lrs, double lr_scale, double beta1,
                          double beta2, double eps, double weight_decay, double bc1, double bc2,
                          int do_step, double *cov6_out, double *stats_out,
                          unsigned long long *floor_out, double *stats_prev_out, void *stream) {
  if (N <= 0) return fail(GSVR_ERR_INVALID, "need at least one primitive");
  cudaStream_t st = as_stream(stream);
  AdamArgs aa{beta1, beta2, eps, weight_decay, bc1, bc2};
  double4 lr4 = make_double4(lrs[0], lrs[1], lrs[2], lrs[3]);
  if (grid_for(N, 256) > (unsigned)kMaxSumBlocks) return fail(GSVR_ERR_INVALID, "field step grid too large");
  k_field_step<256><<<grid_for(N, 256), 256, 0, st>>>(N, means, log_scales, quats, cvals, m, v,
                                                       dfield, lambda_reg, s_target, lr4, lr_scale,
                                                       aa, do_step, cov6_out, stats_out, stats_prev_out,
                                                       floor_out);
  GSVR_LAUNCH_CHECK("k_field_step");
  return GSVR_OK;
}

int gsvr_slice_adamw_step(int64_t S, double *state, double *m, double *v, double *dslice,
                          const double *stack_rots, const int32_t *slice_to_stack,
                          const double *psf_diags, const double *slice_counts,
                          int outlier_weighting, const double *lrs, double lr_scale, double beta1,
                          double beta2, double eps, double weight_decay, double bc1, double bc2,
                          int step_mask, int64_t anchor, double *loss_out, double *Rc,
                          double *tvec, double *psf6s, double *sigma_s, double *wdata_s,
                          void *stream) {
  if (S <= 0) return fail(GSVR_ERR_INVALID, "need at least one slice");
  cudaStream_t st = as_stream(stream);
  AdamArgs aa{beta1, beta2, eps, weight_decay, bc1, bc2};
  double4 lr4 = make_double4(lrs[0], lrs[1], lrs[2], lrs[3]);
  k_slice_step<<<1, kSliceBlock, 0, st>>>(S, state, m, v, dslice, stack_rots, slice_to_stack,
                                          psf_diags, slice_counts, outlier_weighting, lr4, lr_scale,
                                          aa, step_mask, anchor, loss_out, Rc, tvec, psf6s, sigma_s,
                                          wdata_s);
  GSVR_LAUNCH_CHECK("k_slice_step");
  return GSVR_OK;
}

int64_t gsvr_field_workspace_bytes(void) { return (int64_t)kFieldWsDoubles * 8; }

}  // extern "C"
