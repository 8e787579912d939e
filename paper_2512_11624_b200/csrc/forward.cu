// forward.cu -- forward-only evaluations with arbitrary points:
//   gsvr_render_forward  kernels.py:41-75  observed intensities, per-point PSF, clamp at -80
//   gsvr_eval_field      field.py:93-135   PSF-free field values (HR export, reseed)
// These are not the training hot pass (that is train.cu); they serve the
// reference's render_observed / render_batch / compute_loss / evaluate_field /
// rasterize callers.  Templated on the arithmetic type so the float64 path keeps
// the reference's own precision (finite-difference gradient checks need it).
#include "common.cuh"

namespace gsvr {

template <class T, class I>
__global__ void k_render_forward(int64_t M, int K, const T *__restrict__ pts, const T *__restrict__ psf6,
                                 const T *__restrict__ sigma, const I *__restrict__ nbr, int64_t N,
                                 const T *__restrict__ mu, const T *__restrict__ cov6,
                                 const T *__restrict__ cvals, T delta, T *__restrict__ out, int *bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M; p += (int64_t)gridDim.x * blockDim.x) {
    const T x0 = pts[3 * p], x1 = pts[3 * p + 1], x2 = pts[3 * p + 2];
    T ps[6];
#pragma unroll
    for (int e = 0; e < 6; ++e) ps[e] = psf6[6 * p + e];
    T num = 0, den = delta;
    for (int k = 0; k < K; ++k) {
      int64_t j = (int64_t)nbr[p * K + k];
      if (j < 0 || j >= N) {
        atomicExch(bad, 1);
        continue;
      }
      T a[6], m[6];
#pragma unroll
      for (int e = 0; e < 6; ++e) a[e] = cov6[6 * j + e] + ps[e];
      inv_sym3<T>(a, m);
      const T v0 = x0 - mu[3 * j], v1 = x1 - mu[3 * j + 1], v2 = x2 - mu[3 * j + 2];
      const T w0 = m[0] * v0 + m[1] * v1 + m[2] * v2;
      const T w1 = m[1] * v0 + m[3] * v1 + m[4] * v2;
      const T w2 = m[2] * v0 + m[4] * v1 + m[5] * v2;
      T u = T(-0.5) * (v0 * w0 + v1 * w1 + v2 * w2);
      if (u < T(kExpClamp)) u = T(kExpClamp);
      const T e = exp(u);
      num += cvals[j] * e;
      den += e;
    }
    out[p] = sigma[p] * num / den;
  }
}

// Per-primitive inverse covariance (geometry.py:168-201 closed form) + floor check.
__global__ void k_inv_cov(int64_t N, const double *__restrict__ ls, const double *__restrict__ q,
                          double *__restrict__ inv6, unsigned long long *floor_first) {
  for (int64_t j = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; j < N; j += (int64_t)gridDim.x * blockDim.x) {
    double R[9], D[3], c6[6], m[6];
    quat_to_rot(q + 4 * j, R);
    for (int d = 0; d < 3; ++d) D[d] = exp(2.0 * ls[3 * j + d]);
    rot_diag_rot_t(R, D, c6);
    inv_sym3<double>(c6, m);
    for (int e = 0; e < 6; ++e) inv6[6 * j + e] = m[e];
    if (fmin(fmin(D[0], D[1]), D[2]) < kEigenFloor) atomicMin(floor_first, (unsigned long long)j);
  }
}

template <class I>
__global__ void k_eval_field(int64_t M, int K, const double *__restrict__ pts, const I *__restrict__ nbr,
                             int64_t N, const double *__restrict__ mu, const double *__restrict__ inv6,
                             const double *__restrict__ cvals, double delta, double *__restrict__ out, int *bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < M; p += (int64_t)gridDim.x * blockDim.x) {
    const double x0 = pts[3 * p], x1 = pts[3 * p + 1], x2 = pts[3 * p + 2];
    double num = 0.0, den = 0.0;
    for (int k = 0; k < K; ++k) {
      int64_t j = (int64_t)nbr[p * K + k];
      if (j < 0 || j >= N) {
        atomicExch(bad, 1);
        continue;
      }
      const double *m = inv6 + 6 * j;
      const double v0 = x0 - mu[3 * j], v1 = x1 - mu[3 * j + 1], v2 = x2 - mu[3 * j + 2];
      // field.py:125-130 symmetric expansion, same association order
      const double quad = m[0] * v0 * v0 + m[3] * v1 * v1 + m[5] * v2 * v2 +
                          2.0 * (m[1] * v0 * v1 + m[2] * v0 * v2 + m[4] * v1 * v2);
      const double w = exp(fmax(-0.5 * quad, kExpClamp));
      num += cvals[j] * w;
      den += w;
    }
    out[p] = num / (den + delta);
  }
}


// train.py:189-206 render_batch: x = Rc[s] x0 + t[s] (einsum order), per-slice PSF and
// sigma, clamp semantics, float64.
template <class I>
__global__ void k_render_slices(int64_t P, int K, const double *__restrict__ x0, const int32_t *__restrict__ sid,
                                const double *__restrict__ Rc, const double *__restrict__ tv,
                                const double *__restrict__ psf6s, const double *__restrict__ sig,
                                const I *__restrict__ nbr, int64_t N, const double *__restrict__ mu,
                                const double *__restrict__ cov6, const double *__restrict__ cvals, double delta,
                                double *__restrict__ out, int *bad) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int s = sid[p];
    const double a0 = x0[3 * p], a1 = x0[3 * p + 1], a2 = x0[3 * p + 2];
    double x[3];
    for (int r = 0; r < 3; ++r) {
      const double *R = Rc + 9 * s + 3 * r;
      x[r] = __dadd_rn(__dadd_rn(__dadd_rn(__dmul_rn(R[0], a0), __dmul_rn(R[1], a1)), __dmul_rn(R[2], a2)),
                       tv[3 * s + r]);
    }
    double num = 0.0, den = delta;
    for (int k = 0; k < K; ++k) {
      const int64_t j = (int64_t)nbr[p * K + k];
      if (j < 0 || j >= N) {
        atomicExch(bad, 1);
        continue;
      }
      double a[6], m[6];
      for (int e = 0; e < 6; ++e) a[e] = cov6[6 * j + e] + psf6s[6 * s + e];
      inv_sym3<double>(a, m);
      const double v0 = x[0] - mu[3 * j], v1 = x[1] - mu[3 * j + 1], v2 = x[2] - mu[3 * j + 2];
      const double w0 = m[0] * v0 + m[1] * v1 + m[2] * v2;
      const double w1 = m[1] * v0 + m[3] * v1 + m[4] * v2;
      const double w2 = m[2] * v0 + m[4] * v1 + m[5] * v2;
      double u = -0.5 * (v0 * w0 + v1 * w1 + v2 * w2);
      if (u < kExpClamp) u = kExpClamp;
      const double e = exp(u);
      num += cvals[j] * e;
      den += e;
    }
    out[p] = sig[s] * num / den;
  }
}

// train.py:305-309 corrected_points (einsum order, no FMA).
__global__ void k_corrected_points(int64_t P, const double *__restrict__ x0, const int32_t *__restrict__ sid,
                                   const double *__restrict__ Rc, const double *__restrict__ tv,
                                   double *__restrict__ out) {
  for (int64_t p = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; p < P; p += (int64_t)gridDim.x * blockDim.x) {
    const int s = sid[p];
    const double a0 = x0[3 * p], a1 = x0[3 * p + 1], a2 = x0[3 * p + 2];
    for (int r = 0; r < 3; ++r) {
      const double *R = Rc + 9 * s + 3 * r;
      out[3 * p + r] = __dadd_rn(
          __dadd_rn(__dadd_rn(__dmul_rn(R[0], a0), __dmul_rn(R[1], a1)), __dmul_rn(R[2], a2)), tv[3 * s + r]);
    }
  }
}

}  // namespace gsvr

using namespace gsvr;

extern "C" {

int gsvr_render_forward(int dtype, int64_t M, int64_t K, const void *points, const void *psf6, const void *sigma,
                        const void *nbr, int nbr_i64, int64_t N, const void *mu, const void *cov6,
                        const void *cvals, double delta, void *out, void *stream) {
  if (M == 0) return GSVR_OK;
  if (M < 0 || K < 0 || N < 1) return fail(GSVR_ERR_INVALID, "bad render_forward sizes");
  cudaStream_t st = as_stream(stream);
  Scratch flag;
  GSVR_TRY(flag.alloc(4, st));
  GSVR_CUDA(cudaMemsetAsync(flag.ptr, 0, 4, st));
  const int g = grid_for(M, 128, 148 * 64);
#define GSVR_RF(T, I)                                                                                        \
  k_render_forward<T, I><<<g, 128, 0, st>>>(M, (int)K, (const T *)points, (const T *)psf6, (const T *)sigma, \
                                            (const I *)nbr, N, (const T *)mu, (const T *)cov6,              \
                                            (const T *)cvals, (T)delta, (T *)out, flag.as<int>())
  if (dtype == GSVR_F64) {
    if (nbr_i64) GSVR_RF(double, int64_t); else GSVR_RF(double, int32_t);
  } else if (dtype == GSVR_F32) {
    if (nbr_i64) GSVR_RF(float, int64_t); else GSVR_RF(float, int32_t);
  } else {
    return fail(GSVR_ERR_INVALID, "unsupported dtype %d", dtype);
  }
#undef GSVR_RF
  GSVR_LAUNCH_CHECK("k_render_forward");
  int bad = 0;
  GSVR_CUDA(cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  if (bad) return fail(GSVR_ERR_INVALID, "neighbor id out of range");
  return GSVR_OK;
}

int gsvr_eval_field(int64_t M, int64_t K, const double *points, const void *nbr, int nbr_i64, int64_t N,
                    const double *mu, const double *log_scales, const double *quats, const double *cvals,
                    double delta, double *out, void *stream) {
  if (N < 1) return fail(GSVR_ERR_INVALID, "empty field");
  cudaStream_t st = as_stream(stream);
  Scratch inv, flag;
  GSVR_TRY(inv.alloc(N * 48, st));
  GSVR_TRY(flag.alloc(16, st));
  GSVR_CUDA(cudaMemsetAsync(flag.ptr, 0, 4, st));
  GSVR_CUDA(cudaMemsetAsync(flag.as<char>() + 8, 0xff, 8, st));
  unsigned long long *ff = reinterpret_cast<unsigned long long *>(flag.as<char>() + 8);
  k_inv_cov<<<grid_for(N, 256), 256, 0, st>>>(N, log_scales, quats, inv.as<double>(), ff);
  GSVR_LAUNCH_CHECK("k_inv_cov");
  if (M > 0) {
    const int g = grid_for(M, 128, 148 * 64);
    if (nbr_i64)
      k_eval_field<int64_t><<<g, 128, 0, st>>>(M, (int)K, points, (const int64_t *)nbr, N, mu, inv.as<double>(),
                                               cvals, delta, out, flag.as<int>());
    else
      k_eval_field<int32_t><<<g, 128, 0, st>>>(M, (int)K, points, (const int32_t *)nbr, N, mu, inv.as<double>(),
                                               cvals, delta, out, flag.as<int>());
    GSVR_LAUNCH_CHECK("k_eval_field");
  }
  int bad = 0;
  unsigned long long fl = 0;
  GSVR_CUDA(cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaMemcpyAsync(&fl, ff, 8, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  if (fl != ~0ull) {
    double l3[3];
    GSVR_CUDA(cudaMemcpy(l3, log_scales + 3 * fl, sizeof(l3), cudaMemcpyDeviceToHost));
    double ev = fmin(fmin(exp(2 * l3[0]), exp(2 * l3[1])), exp(2 * l3[2]));
    set_error(GSVR_ERR_DEGENERATE, "covariance eigenvalue below floor", (int64_t)fl, ev);
    return GSVR_ERR_DEGENERATE;
  }
  if (bad) return fail(GSVR_ERR_INVALID, "neighbor id out of range");
  return GSVR_OK;
}


int gsvr_render_batch(int64_t P, int64_t K, const double *x0, const int32_t *sid, const double *Rc,
                      const double *tvec, const double *psf6s, const double *sigma_s, const void *nbr, int nbr_i64,
                      int64_t N, const double *mu, const double *cov6, const double *cvals, double delta, double *out,
                      void *stream) {
  if (P == 0) return GSVR_OK;
  if (P < 0 || K < 0 || N < 1) return fail(GSVR_ERR_INVALID, "bad render_batch sizes");
  cudaStream_t st = as_stream(stream);
  Scratch flag;
  GSVR_TRY(flag.alloc(4, st));
  GSVR_CUDA(cudaMemsetAsync(flag.ptr, 0, 4, st));
  const int g = grid_for(P, 128, 148 * 64);
  if (nbr_i64)
    k_render_slices<int64_t><<<g, 128, 0, st>>>(P, (int)K, x0, sid, Rc, tvec, psf6s, sigma_s, (const int64_t *)nbr,
                                                N, mu, cov6, cvals, delta, out, flag.as<int>());
  else
    k_render_slices<int32_t><<<g, 128, 0, st>>>(P, (int)K, x0, sid, Rc, tvec, psf6s, sigma_s, (const int32_t *)nbr,
                                                N, mu, cov6, cvals, delta, out, flag.as<int>());
  GSVR_LAUNCH_CHECK("k_render_slices");
  int bad = 0;
  GSVR_CUDA(cudaMemcpyAsync(&bad, flag.ptr, 4, cudaMemcpyDeviceToHost, st));
  GSVR_CUDA(cudaStreamSynchronize(st));
  if (bad) return fail(GSVR_ERR_INVALID, "neighbor id out of range");
  return GSVR_OK;
}

int gsvr_corrected_points(int64_t P, const double *x0, const int32_t *sid, const double *Rc, const double *tvec,
                          double *out, void *stream) {
  if (P <= 0) return GSVR_OK;
  cudaStream_t st = as_stream(stream);
  k_corrected_points<<<grid_for(P, 256), 256, 0, st>>>(P, x0, sid, Rc, tvec, out);
  GSVR_LAUNCH_CHECK("k_corrected_points");
  return GSVR_OK;
}

}  // extern "C"
