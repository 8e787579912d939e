// common.cuh -- shared device helpers and status plumbing for libgsvr_b200.
//
// Maths helpers restate /root/reference/pkg/src/gsvr/geometry.py and the
// inline inverse of kernels.py:28-38; status codes are the ones declared in
// include/gsvr_b200.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <string>

#include "../../include/gsvr_b200.h"

namespace gsvr {

// Stage tracing: with GSVR_TRACE set, host entry points synchronise their
// stream at each mark and print the wall time of the stage to stderr.
inline bool trace_enabled() {
  static const bool on = [] {
    const char *v = std::getenv("GSVR_TRACE");
    return v && *v && !(v[0] == '0' && v[1] == 0);
  }();
  return on;
}
// Tile-kernel timing (gsvr_set_kernel_timing): CUDA events recorded on the
// launching stream right around each tile-kernel launch (not its gathers).
struct KernelTimer {
  static constexpr int kCap = 4096;
  bool on = false;
  int n = 0;
  cudaEvent_t ev[2 * kCap];
  bool made = false;
  void before(cudaStream_t st) {
    if (on && n < kCap) cudaEventRecord(ev[2 * n], st);
  }
  void after(cudaStream_t st) {
    if (on && n < kCap) cudaEventRecord(ev[2 * n + 1], st), ++n;
  }
};
KernelTimer &kernel_timer();

struct StageTrace {
  const char *scope;
  cudaStream_t st;
  bool on = trace_enabled();
  std::chrono::steady_clock::time_point t = std::chrono::steady_clock::now();
  StageTrace(const char *s, cudaStream_t stream) : scope(s), st(stream) {
    if (on) cudaStreamSynchronize(st), t = std::chrono::steady_clock::now();
  }
  void mark(const char *stage) {
    if (!on) return;
    cudaStreamSynchronize(st);
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "[gsvr trace] %s/%s %.3f ms\n", scope, stage,
                 std::chrono::duration<double, std::milli>(now - t).count());
    t = now;
  }
};

constexpr double kExpClamp = -80.0;          // kernels.py:25, geometry.py:22
constexpr double kEigenFloor = 1e-6;         // geometry.py:18
constexpr double kLog2e = 1.4426950408889634;  // log2(e)

// ---- thread-local status ---------------------------------------------------
void set_error(int code, const std::string &msg, int64_t index = -1, double value = 0.0);
int fail(int code, const char *fmt, ...);
// Maps a CUDA error to GSVR_ERR_CUDA (with a message); GSVR_OK otherwise.
int cuda_status(cudaError_t e, const char *what);

#define GSVR_CUDA(call)                                  \
  do {                                                   \
    cudaError_t _e = (call);                             \
    if (_e != cudaSuccess) return ::gsvr::cuda_status(_e, #call); \
  } while (0)

#define GSVR_LAUNCH_CHECK(what)                                       \
  do {                                                                \
    cudaError_t _e = cudaGetLastError();                              \
    if (_e != cudaSuccess) return ::gsvr::cuda_status(_e, what);      \
  } while (0)

#define GSVR_TRY(expr)          \
  do {                          \
    int _rc = (expr);           \
    if (_rc != GSVR_OK) return _rc; \
  } while (0)

inline cudaStream_t as_stream(void *s) { return reinterpret_cast<cudaStream_t>(s); }

inline int grid_for(int64_t n, int block, int cap = 148 * 32) {
  int64_t g = (n + block - 1) / block;
  if (g < 1) g = 1;
  return (int)(g < cap ? g : cap);
}

// Keep stream-ordered allocations cached in the device's default pool instead of
// returning them to the driver at every synchronisation (GB-sized scratch).
int ensure_pool();
// cudaFuncSetAttribute(MaxDynamicSharedMemorySize) for `kernel` on the current
// device, once per (kernel, device) and size high-water mark
int ensure_smem(const void *kernel, size_t bytes);

// Stream-ordered scratch allocation (cudaMallocAsync) with RAII release.
struct Scratch {
  void *ptr = nullptr;
  cudaStream_t stream = nullptr;
  Scratch() = default;
  Scratch(const Scratch &) = delete;
  Scratch &operator=(const Scratch &) = delete;
  ~Scratch() {
    if (ptr) cudaFreeAsync(ptr, stream);
  }
  int alloc(size_t bytes, cudaStream_t s) {
    ensure_pool();
    stream = s;
    if (ptr) cudaFreeAsync(ptr, stream), ptr = nullptr;
    if (bytes == 0) bytes = 16;
    GSVR_CUDA(cudaMallocAsync(&ptr, bytes, s));
    return GSVR_OK;
  }
  template <class T>
  T *as() const { return reinterpret_cast<T *>(ptr); }
};

// ---- symmetric 3x3 helpers (packed order 00,01,02,11,12,22; geometry.py:24) --

// kernels.py:28-38 cofactor inverse; T = float or double.
template <class T>
__host__ __device__ inline void inv_sym3(const T a[6], T m[6]) {
  T c00 = a[3] * a[5] - a[4] * a[4];
  T c01 = a[2] * a[4] - a[1] * a[5];
  T c02 = a[1] * a[4] - a[2] * a[3];
  T c11 = a[0] * a[5] - a[2] * a[2];
  T c12 = a[1] * a[2] - a[0] * a[4];
  T c22 = a[0] * a[3] - a[1] * a[1];
  T det = a[0] * c00 + a[1] * c01 + a[2] * c02;
  T idet = T(1) / det;
  m[0] = c00 * idet; m[1] = c01 * idet; m[2] = c02 * idet;
  m[3] = c11 * idet; m[4] = c12 * idet; m[5] = c22 * idet;
}

// geometry.py:28-55: normalise, then the scalar-first rotation matrix.
__host__ __device__ inline void quat_to_rot(const double q_in[4], double R[9]) {
  double n = sqrt(q_in[0] * q_in[0] + q_in[1] * q_in[1] + q_in[2] * q_in[2] + q_in[3] * q_in[3]);
  double w = q_in[0] / n, x = q_in[1] / n, y = q_in[2] / n, z = q_in[3] / n;
  R[0] = 1 - 2 * (y * y + z * z); R[1] = 2 * (x * y - w * z); R[2] = 2 * (x * z + w * y);
  R[3] = 2 * (x * y + w * z); R[4] = 1 - 2 * (x * x + z * z); R[5] = 2 * (y * z - w * x);
  R[6] = 2 * (x * z - w * y); R[7] = 2 * (y * z + w * x); R[8] = 1 - 2 * (x * x + y * y);
}

// geometry.py:58-85: dL/dR -> dL/dq through the normalisation.
__host__ __device__ inline void quat_vjp(const double q[4], const double G[9], double dq[4]) {
  double n = sqrt(q[0] * q[0] + q[1] * q[1] + q[2] * q[2] + q[3] * q[3]);
  double w = q[0] / n, x = q[1] / n, y = q[2] / n, z = q[3] / n;
  double g00 = G[0], g01 = G[1], g02 = G[2], g10 = G[3], g11 = G[4], g12 = G[5];
  double g20 = G[6], g21 = G[7], g22 = G[8];
  double gw = 2 * (-z * g01 + y * g02 + z * g10 - x * g12 - y * g20 + x * g21);
  double gx = 2 * (y * g01 + z * g02 + y * g10 - 2 * x * g11 - w * g12 + z * g20 + w * g21 - 2 * x * g22);
  double gy = 2 * (-2 * y * g00 + x * g01 + w * g02 + x * g10 + z * g12 - w * g20 + z * g21 - 2 * y * g22);
  double gz = 2 * (-2 * z * g00 - w * g01 + x * g02 + w * g10 - 2 * z * g11 + y * g12 + x * g20 + y * g21);
  double rad = gw * w + gx * x + gy * y + gz * z;
  dq[0] = (gw - w * rad) / n; dq[1] = (gx - x * rad) / n;
  dq[2] = (gy - y * rad) / n; dq[3] = (gz - z * rad) / n;
}

// R diag(d) R^T packed (geometry.py:143-157).
__host__ __device__ inline void rot_diag_rot_t(const double R[9], const double d[3], double c6[6]) {
  const int ri[6] = {0, 0, 0, 1, 1, 2}, ci[6] = {0, 1, 2, 1, 2, 2};
  for (int e = 0; e < 6; ++e) {
    const int i = ri[e], j = ci[e];
    c6[e] = R[3 * i] * d[0] * R[3 * j] + R[3 * i + 1] * d[1] * R[3 * j + 1] +
            R[3 * i + 2] * d[2] * R[3 * j + 2];
  }
}

__host__ __device__ inline void unpack6(const double v[6], double A[9]) {
  A[0] = v[0]; A[1] = v[1]; A[2] = v[2];
  A[3] = v[1]; A[4] = v[3]; A[5] = v[4];
  A[6] = v[2]; A[7] = v[4]; A[8] = v[5];
}

// Non-negative doubles order like their bit patterns as int64 -> atomicMax.
__device__ inline void atomic_max_nonneg(double *addr, double v) {
  atomicMax(reinterpret_cast<unsigned long long *>(addr), (unsigned long long)__double_as_longlong(v));
}

// Debug builds (-DGSVR_CHECKS): device-side bounds checks that print the
// failing site and trap.  Compiled out otherwise.
#ifdef GSVR_CHECKS
#define GSVR_DCHECK(cond, site, a, b)                                                          \
  do {                                                                                          \
    if (!(cond)) {                                                                              \
      printf("GSVR_DCHECK %s failed: %lld %lld (block %d thread %d)\n", site, (long long)(a),     \
             (long long)(b), (int)blockIdx.x, (int)threadIdx.x);                                \
      __trap();                                                                                 \
    }                                                                                           \
  } while (0)
#else
#define GSVR_DCHECK(cond, site, a, b) \
  do {                                \
  } while (0)
#endif

template <class T>
__device__ inline T warp_sum(T v) {
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}

}  // namespace gsvr
