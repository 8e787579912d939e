// status.cu -- thread-local error reporting behind gsvr_last_error*().
#include <cstdarg>
#include <cstdio>
#include <string>

#include <map>
#include <mutex>
#include <utility>

#include "common.cuh"

namespace gsvr {
namespace {
thread_local std::string g_msg;
thread_local int64_t g_index = -1;
thread_local double g_value = 0.0;
}  // namespace

void set_error(int code, const std::string &msg, int64_t index, double value) {
  (void)code;
  g_msg = msg;
  g_index = index;
  g_value = value;
}

int fail(int code, const char *fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  set_error(code, buf);
  return code;
}

int ensure_pool() {
  static thread_local int done_dev = -1;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GSVR_ERR_CUDA;
  if (done_dev == dev) return GSVR_OK;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t keep = ~0ull;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &keep);
  }
  done_dev = dev;
  return GSVR_OK;
}

int ensure_smem(const void *kernel, size_t bytes) {
  static std::mutex mu;
  static std::map<std::pair<const void *, int>, size_t> done;
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess) return GSVR_ERR_CUDA;
  std::lock_guard<std::mutex> lk(mu);
  size_t &have = done[{kernel, dev}];
  if (bytes <= have) return GSVR_OK;
  const cudaError_t e = cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bytes);
  if (e != cudaSuccess) return fail(GSVR_ERR_CUDA, "shared-memory attribute: %s", cudaGetErrorString(e));
  have = bytes;
  return GSVR_OK;
}

int cuda_status(cudaError_t e, const char *what) {
  if (e == cudaSuccess) return GSVR_OK;
  return fail(GSVR_ERR_CUDA, "%s: %s", what, cudaGetErrorString(e));
}

}  // namespace gsvr

extern "C" {
int gsvr_abi_version(void) { return 1; }
const char *gsvr_last_error(void) { return gsvr::g_msg.c_str(); }
int64_t gsvr_last_error_index(void) { return gsvr::g_index; }
double gsvr_last_error_value(void) { return gsvr::g_value; }
}

namespace gsvr {
KernelTimer &kernel_timer() {
  static KernelTimer t;
  return t;
}
}  // namespace gsvr

extern "C" {

int gsvr_set_kernel_timing(int on) {
  gsvr::KernelTimer &t = gsvr::kernel_timer();
  if (on && !t.made) {
    for (auto &e : t.ev) GSVR_CUDA(cudaEventCreate(&e));
    t.made = true;
  }
  t.on = on != 0;
  t.n = 0;
  return GSVR_OK;
}

double gsvr_kernel_time_ms(int64_t *launches) {
  gsvr::KernelTimer &t = gsvr::kernel_timer();
  double tot = 0.0;
  for (int i = 0; i < t.n; ++i) {
    float ms = 0.f;
    if (cudaEventSynchronize(t.ev[2 * i + 1]) == cudaSuccess &&
        cudaEventElapsedTime(&ms, t.ev[2 * i], t.ev[2 * i + 1]) == cudaSuccess)
      tot += ms;
  }
  if (launches) *launches = t.n;
  return tot;
}

}  // extern "C"
