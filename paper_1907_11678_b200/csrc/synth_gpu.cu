// synth_gpu.cu — the seeded synthetic generator of synth.cpp on the device
// (SURVEY.md §8f-3): samples are written straight into HBM, so multi-GPU
// weak-scaling runs never generate (or copy) tens of GB on the host.
//
// Same model and the same counter-based streams as the host generator: a
// splitmix64 stream per gather for its events (or the line's reflectors for
// CRS, drawn on the host — a handful of numbers) and per (gather, trace) for
// the Box-Muller noise, addressed by counter so any sample pair can be drawn
// independently.  Every sample accumulates its events in event order and
// then its noise, in double, rounded to float per term, exactly as the host
// loop does; results match the host generator to the last bit except where a
// double libm result (exp/log/sin/cos) differs by an ulp and that flips a
// float rounding (tests/test_gpu_synth.py bounds it).
#include <cuda_runtime.h>

#include <cmath>
#include <cstdint>
#include <vector>

#include "../../include/velan_gpu.h"

namespace {

__host__ __device__ inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}
// draw number `ctr` of the stream `key` (synth.cpp Stream::next)
__host__ __device__ inline uint64_t draw(uint64_t key, uint64_t ctr) {
  return mix64(key + ctr * 0xD1B54A32D192ED03ull);
}
__host__ __device__ inline double unit(uint64_t key, uint64_t ctr) {
  return static_cast<double>(draw(key, ctr) >> 11) * 0x1.0p-53;
}

struct DevEvent {
  double t0, v, amp, x, A, B;
};

constexpr int kMaxEvents = 64;
constexpr double kPi = 3.14159265358979323846;

// One CTA per (gather, trace); thread i owns sample pair (2i, 2i+1).
__global__ void synth_kernel(velan_gpu_synth p, const DevEvent* __restrict__ line_events,
                             float* __restrict__ samples) {
  __shared__ DevEvent evs[kMaxEvents];
  const int gl = blockIdx.y;
  const int m = blockIdx.x;
  const int g = p.gather_first + gl;
  const uint64_t key = mix64(p.seed ^ mix64(0x5EED000000000000ull + g));
  const int ne = min(p.n_events, kMaxEvents);
  if (threadIdx.x == 0) {
    if (p.kind == 0) {
      // synth.cpp gen_gather: eps, then per event t0, (v), amp in stream order
      uint64_t c = 0;
      const double eps = -p.v_perturb + 2.0 * p.v_perturb * unit(key, c++);
      for (int e = 0; e < ne; ++e) {
        DevEvent ev{};
        ev.t0 = p.t0_lo + (p.t0_hi - p.t0_lo) * unit(key, c++);
        ev.v = p.v_profile == 1 ? (p.v_trend_0 + p.v_trend_slope * ev.t0) * (1.0 + eps)
                                : p.v_lo + (p.v_hi - p.v_lo) * unit(key, c++);
        ev.amp = p.amp_lo + (p.amp_hi - p.amp_lo) * unit(key, c++);
        evs[e] = ev;
      }
    } else {
      for (int e = 0; e < ne; ++e) evs[e] = line_events[e];
    }
  }
  __syncthreads();
  const int ns = p.ns;
  const double dt = static_cast<double>(p.dt_us) * 1e-6;
  const double mx = g * p.spacing;
  const double h = p.h0 + m * p.dh;
  const double support = 4.0 / p.freq;
  float* tr = samples + (static_cast<size_t>(gl) * p.n_traces + m) * ns;
  const uint64_t nkey = mix64(key ^ mix64(0xA0000000ull + m));
  for (int i = threadIdx.x; 2 * i < ns; i += blockDim.x) {
    float acc[2] = {0.0f, 0.0f};
    for (int e = 0; e < ne; ++e) {
      const DevEvent& ev = evs[e];
      double t;
      if (p.kind == 0) {
        t = sqrt(ev.t0 * ev.t0 + 4.0 * h * h / (ev.v * ev.v));
      } else {
        const double dm = mx - ev.x;
        const double tau = ev.t0 + 2.0 * ev.A * dm;
        const double t2 = tau * tau + 2.0 * ev.t0 * ev.B * dm * dm + 4.0 * h * h / (ev.v * ev.v);
        if (!(t2 > 0.0)) continue;
        t = sqrt(t2);
      }
      // add_event's support window [lo, hi)
      const int lo = max(0, static_cast<int>(floor((t - support) / dt)));
      const int hi = min(ns, static_cast<int>(ceil((t + support) / dt)) + 1);
#pragma unroll
      for (int j = 0; j < 2; ++j) {
        const int s = 2 * i + j;
        if (s < lo || s >= hi || s >= ns) continue;
        const double a = kPi * p.freq * (s * dt - t);
        const double a2 = a * a;
        acc[j] += static_cast<float>(ev.amp * ((1.0 - 2.0 * a2) * exp(-a2)));
      }
    }
    if (p.sigma > 0.0) {
      const double u1 = (static_cast<double>(draw(nkey, 2ull * i) >> 11) + 1.0) * 0x1.0p-53;
      const double u2 = static_cast<double>(draw(nkey, 2ull * i + 1) >> 11) * 0x1.0p-53;
      const double r = sqrt(-2.0 * log(u1));
      const double th = 2.0 * kPi * u2;
      acc[0] += static_cast<float>(p.sigma * r * cos(th));
      acc[1] += static_cast<float>(p.sigma * r * sin(th));
    }
    tr[2 * i] = acc[0];
    if (2 * i + 1 < ns) tr[2 * i + 1] = acc[1];
  }
}

}  // namespace

// the host generator's CRS reflectors (synth.cpp, one stream per line)
extern "C" int velan_gpu_synth_line_events(const velan_gpu_synth* p, double* out6);

extern "C" int velan_gpu_synth_generate_device(const velan_gpu_synth* p, float* d_samples,
                                               void* stream) {
  if (!p || !d_samples) return VELAN_GPU_EPARAM;
  if (p->n_gathers < 0 || p->n_traces < 1 || p->ns < 2 || p->dt_us == 0 || p->freq <= 0.0 ||
      p->n_events < 0 || p->n_events > kMaxEvents)
    return VELAN_GPU_EPARAM;
  if (p->n_gathers == 0) return VELAN_GPU_OK;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  DevEvent* d_ev = nullptr;
  if (p->kind == 1 && p->n_events > 0) {
    std::vector<double> ev(6 * static_cast<size_t>(p->n_events));
    int rc = velan_gpu_synth_line_events(p, ev.data());
    if (rc) return rc;
    std::vector<DevEvent> de(p->n_events);
    for (int e = 0; e < p->n_events; ++e)
      de[e] = DevEvent{ev[6 * e + 0], ev[6 * e + 1], ev[6 * e + 2],
                       ev[6 * e + 3], ev[6 * e + 4], ev[6 * e + 5]};
    if (cudaMallocAsync(&d_ev, sizeof(DevEvent) * de.size(), st) != cudaSuccess)
      return VELAN_GPU_ERUNTIME;
    cudaMemcpyAsync(d_ev, de.data(), sizeof(DevEvent) * de.size(), cudaMemcpyHostToDevice, st);
  }
  dim3 grid(p->n_traces, p->n_gathers);
  synth_kernel<<<grid, 256, 0, st>>>(*p, d_ev, d_samples);
  cudaError_t e = cudaGetLastError();
  if (d_ev) cudaFreeAsync(d_ev, st);
  if (e == cudaSuccess) e = cudaStreamSynchronize(st);
  return e == cudaSuccess ? VELAN_GPU_OK : VELAN_GPU_ERUNTIME;
}
