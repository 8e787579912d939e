// probe.cu -- FP32 FMA-pipe peak probe (diagnostic, used by bench.py as the
// roofline denominator: MEASURED_PEAKS.json carries no FP32 CUDA-core figure).
#include "common.cuh"

namespace gsvr {

__global__ void __launch_bounds__(256) k_ffma_probe(float *out, int iters, float seed) {
  float a[8];
#pragma unroll
  for (int i = 0; i < 8; ++i) a[i] = seed + (float)(threadIdx.x + i);
  const float b = 0.999999f, c = 1e-7f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < 8; ++i) a[i] = fmaf(a[i], b, c);
  }
  float s = 0.f;
#pragma unroll
  for (int i = 0; i < 8; ++i) s += a[i];
  if (s == 12345.678f) out[blockIdx.x] = s;  // keep the chains alive
}

}  // namespace gsvr

extern "C" int gsvr_probe_fp32_peak(double *tflops_out, void *stream) {
  using namespace gsvr;
  cudaStream_t st = as_stream(stream);
  int dev = 0, sms = 0;
  GSVR_CUDA(cudaGetDevice(&dev));
  GSVR_CUDA(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  Scratch out;
  GSVR_TRY(out.alloc(4096 * 4, st));
  const int blocks = sms * 8, iters = 1 << 15;
  cudaEvent_t e0, e1;
  GSVR_CUDA(cudaEventCreate(&e0));
  GSVR_CUDA(cudaEventCreate(&e1));
  k_ffma_probe<<<blocks, 256, 0, st>>>(out.as<float>(), 256, 1.f);  // warm-up
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    GSVR_CUDA(cudaEventRecord(e0, st));
    k_ffma_probe<<<blocks, 256, 0, st>>>(out.as<float>(), iters, 1.f + r);
    GSVR_CUDA(cudaEventRecord(e1, st));
    GSVR_CUDA(cudaEventSynchronize(e1));
    float ms = 0.f;
    GSVR_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    best = ms < best ? ms : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  const double flops = (double)blocks * 256.0 * iters * 8.0 * 2.0;
  *tflops_out = flops / (best * 1e-3) / 1e12;
  return GSVR_OK;
}
