// peak.cu — FP32 FMA throughput probe: the measured denominator of the
// roofline fraction bench.py reports (the path is FP32-SIMT bound; the
// driver's MEASURED_PEAKS.json holds only HBM and bf16 tensor peaks).
#include <cuda_runtime.h>

#include "../../include/velan_gpu.h"

namespace {
__global__ void fma_probe(float* out, int iters, float seed) {
  float a0 = seed + threadIdx.x, a1 = a0 + 1, a2 = a0 + 2, a3 = a0 + 3;
  float a4 = a0 + 4, a5 = a0 + 5, a6 = a0 + 6, a7 = a0 + 7;
  const float b = 0.999999f, c = 1e-7f;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 16; ++u) {
      a0 = __fmaf_rn(a0, b, c); a1 = __fmaf_rn(a1, b, c);
      a2 = __fmaf_rn(a2, b, c); a3 = __fmaf_rn(a3, b, c);
      a4 = __fmaf_rn(a4, b, c); a5 = __fmaf_rn(a5, b, c);
      a6 = __fmaf_rn(a6, b, c); a7 = __fmaf_rn(a7, b, c);
    }
  }
  const float s = a0 + a1 + a2 + a3 + a4 + a5 + a6 + a7;
  if (s == 1234.5f) out[blockIdx.x] = s;  // keep the chains alive
}
}  // namespace

extern "C" int velan_gpu_measure_fp32_peak(int32_t device, double* tflops) {
  if (!tflops) return VELAN_GPU_EPARAM;
  if (cudaSetDevice(device) != cudaSuccess) return VELAN_GPU_ENODEV;
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
  float* out = nullptr;
  if (cudaMalloc(&out, 4 * 65536) != cudaSuccess) return VELAN_GPU_ERUNTIME;
  const int threads = 256, blocks = sms * 8, iters = 4096;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  fma_probe<<<blocks, threads>>>(out, 64, 1.0f);  // warm-up / clocks up
  double best = 0.0;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    fma_probe<<<blocks, threads>>>(out, iters, 1.0f + r);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms = 0.0f;
    cudaEventElapsedTime(&ms, e0, e1);
    const double flops = 2.0 * 8 * 16 * static_cast<double>(iters) * threads * blocks;
    if (ms > 0.0f) best = flops / (ms * 1e-3) / 1e12 > best ? flops / (ms * 1e-3) / 1e12 : best;
  }
  cudaEventDestroy(e0);
  cudaEventDestroy(e1);
  cudaFree(out);
  *tflops = best;
  return cudaGetLastError() == cudaSuccess ? VELAN_GPU_OK : VELAN_GPU_ERUNTIME;
}
