// pipe_probe.cu — FP32 pipe throughput probe (FFMA vs FFMA2, register
// operands vs immediates, with/without LDS traffic), per SM per cycle.
// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o pipe_probe pipe_probe.cu
#include <cstdio>
#include <cuda_runtime.h>

template <int MODE>
__global__ void probe(float* out, int iters, float seed, float bb, float cc) {
  __shared__ float2 sm[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) sm[i] = make_float2(i, i + 1);
  __syncthreads();
  float2 a[8];
  for (int u = 0; u < 8; ++u) a[u] = make_float2(seed + threadIdx.x + u, seed - u);
  float b = bb + threadIdx.x * 1e-9f, c = cc + threadIdx.x * 1e-12f;
  float2 b2 = make_float2(b, b * 0.5f), c2 = make_float2(c, c * 0.7f);
  unsigned addr = (threadIdx.x * 8) & 4095;
#pragma unroll 1
  for (int i = 0; i < iters; ++i) {
#pragma unroll
    for (int u = 0; u < 8; ++u) {
      if (MODE == 0) {  // scalar FFMA, register operands
        a[u].x = __fmaf_rn(a[u].x, b, c);
        a[u].y = __fmaf_rn(a[u].y, b, c);
      } else if (MODE == 1) {  // FFMA2 register operands
        a[u] = __ffma2_rn(a[u], b2, c2);
      } else if (MODE == 2) {  // FFMA2 + one LDS.64 per 2 FFMA2 (kernel-like mix)
        float2 v = sm[(addr + u * 33) & 1023];
        a[u] = __ffma2_rn(v, b2, a[u]);
        a[(u + 4) & 7] = __ffma2_rn(v, c2, a[(u + 4) & 7]);
      } else if (MODE == 3) {  // FADD2
        a[u] = __fadd2_rn(a[u], b2);
      }
    }
    addr += 17;
  }
  float s = 0;
  for (int u = 0; u < 8; ++u) s += a[u].x + a[u].y;
  if (s == 1234.5f) out[blockIdx.x] = s;
}

template <int MODE>
void run(const char* name, int threads, double flops_per_iter_thread) {
  int sms;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int clk;
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  float* out;
  cudaMalloc(&out, 4 * 65536);
  const int blocks = sms, iters = 1 << 16;
  probe<MODE><<<blocks, threads>>>(out, 256, 1.0f, 0.999f, 1e-7f);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    probe<MODE><<<blocks, threads>>>(out, iters, 1.0f + r, 0.999f, 1e-7f);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    if (ms < best) best = ms;
  }
  const double fl = flops_per_iter_thread * iters * threads * blocks;
  const double cyc = best * 1e-3 * 1965e6;
  printf("%-28s threads %4d: %.1f TFLOP/s  %.1f lane-FMA/cycle/SM  (%.3f ms)\n", name, threads,
         fl / (best * 1e-3) / 1e12, fl / 2 / cyc / sms, best);
  cudaFree(out);
}

int main() {
  for (int t : {128, 256, 512, 1024}) {
    run<0>("FFMA scalar reg", t, 2.0 * 16);
    run<1>("FFMA2 reg", t, 2.0 * 16);
    run<2>("FFMA2+LDS.64 (1 per 2)", t, 2.0 * 32);
    run<3>("FADD2 (counted as 1 flop)", t, 2.0 * 8);
  }
  return 0;
}
