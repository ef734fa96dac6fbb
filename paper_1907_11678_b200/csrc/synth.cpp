// synth.cpp — seeded synthetic inputs for the BASELINE.json configurations.
//
// Follows the reference generator's conventions (synthetic.hpp): Ricker
// wavelet (1 - 2a^2) e^{-a^2}, a = pi f tau (synthetic.hpp:39-43), summed
// over a support of +-4/f around each event (synthetic.hpp:102,131-139),
// Box-Muller Gaussian noise (synthetic.hpp:49-72), geometry through the
// Trace source/receiver coordinates (types.hpp:14-25) with sx = mx - h,
// gx = mx + h.  Deliberate deviations: a counter-based
// splitmix64 stream per (gather, trace) instead of one mt19937_64 stream,
// so generation is order-free, thread-count independent and shardable;
// per-gather random events (CMP) / global dipping reflectors (CRS line) as
// BASELINE.json describes, and a fixed noise sigma.
#include <algorithm>
#include <cmath>
#include <cstdint>
#include <thread>
#include <vector>

#include "../../include/velan_gpu.h"

namespace {

inline uint64_t mix64(uint64_t z) {
  z += 0x9E3779B97F4A7C15ull;
  z = (z ^ (z >> 30)) * 0xBF58476D1CE4E5B9ull;
  z = (z ^ (z >> 27)) * 0x94D049BB133111EBull;
  return z ^ (z >> 31);
}

struct Stream {
  uint64_t key;
  uint64_t ctr = 0;
  explicit Stream(uint64_t k) : key(k) {}
  uint64_t next() { return mix64(key + (ctr++) * 0xD1B54A32D192ED03ull); }
  double uniform() { return static_cast<double>(next() >> 11) * 0x1.0p-53; }
  double uniform(double lo, double hi) { return lo + (hi - lo) * uniform(); }
};

inline double ricker(double tau, double freq) {
  const double a = M_PI * freq * tau;
  const double a2 = a * a;
  return (1.0 - 2.0 * a2) * std::exp(-a2);
}

struct Event {
  double t0, v, amp, x, A, B;
};

void add_event(float* tr, int ns, double dt, double t, double amp,
               double freq) {
  const double support = 4.0 / freq;
  const int lo = std::max(0, static_cast<int>(std::floor((t - support) / dt)));
  const int hi =
      std::min(ns, static_cast<int>(std::ceil((t + support) / dt)) + 1);
  for (int s = lo; s < hi; ++s)
    tr[s] += static_cast<float>(amp * ricker(s * dt - t, freq));
}

// CRS: reflectors are global to the line, one stream
std::vector<Event> make_line_events(const velan_gpu_synth* p, int n_line) {
  std::vector<Event> line_events;
  Stream es(mix64(p->seed ^ 0xC0FFEE1234ull));
  const double L = (n_line - 1) * p->spacing;
  for (int e = 0; e < p->n_events; ++e) {
    Event ev;
    ev.x = es.uniform(0.0, L);
    ev.t0 = es.uniform(p->t0_lo, p->t0_hi);
    ev.A = es.uniform(-p->a_abs, p->a_abs);
    ev.B = es.uniform(0.0, p->b_max);
    ev.v = es.uniform(p->v_lo, p->v_hi);
    ev.amp = es.uniform(p->amp_lo, p->amp_hi);
    line_events.push_back(ev);
  }
  return line_events;
}

}  // namespace

// The line's reflectors as (t0, v, amp, x, A, B) per event, for the device
// generator (synth_gpu.cu).
extern "C" int velan_gpu_synth_line_events(const velan_gpu_synth* p, double* out6) {
  if (!p || !out6) return VELAN_GPU_EPARAM;
  const int n_line = p->n_line > 0 ? p->n_line : p->gather_first + p->n_gathers;
  const std::vector<Event> ev = make_line_events(p, n_line);
  for (size_t e = 0; e < ev.size(); ++e) {
    out6[6 * e + 0] = ev[e].t0;
    out6[6 * e + 1] = ev[e].v;
    out6[6 * e + 2] = ev[e].amp;
    out6[6 * e + 3] = ev[e].x;
    out6[6 * e + 4] = ev[e].A;
    out6[6 * e + 5] = ev[e].B;
  }
  return VELAN_GPU_OK;
}

extern "C" int velan_gpu_synth_generate(const velan_gpu_synth* p,
                                        float* samples, float* coords,
                                        int32_t* ntraces, uint32_t* cdp_id) {
  // samples may be NULL: geometry only (the device generator fills samples)
  if (!p || !coords || !ntraces || !cdp_id) return VELAN_GPU_EPARAM;
  if (p->n_gathers < 0 || p->n_traces < 1 || p->ns < 2 || p->dt_us == 0 ||
      p->freq <= 0.0 || p->n_events < 0)
    return VELAN_GPU_EPARAM;
  const int G = p->n_gathers, M = p->n_traces, ns = p->ns;
  const double dt = static_cast<double>(p->dt_us) * 1e-6;
  const int n_line = p->n_line > 0 ? p->n_line : p->gather_first + G;

  std::vector<Event> line_events;
  if (p->kind == 1) line_events = make_line_events(p, n_line);

  auto gen_gather = [&](int gl) {
    const int g = p->gather_first + gl;
    const uint64_t key = mix64(p->seed ^ mix64(0x5EED000000000000ull + g));
    Stream gs(key);
    std::vector<Event> evs;
    if (p->kind == 0) {
      const double eps = gs.uniform(-p->v_perturb, p->v_perturb);
      for (int e = 0; e < p->n_events; ++e) {
        Event ev{};
        ev.t0 = gs.uniform(p->t0_lo, p->t0_hi);
        ev.v = p->v_profile == 1
                   ? (p->v_trend_0 + p->v_trend_slope * ev.t0) * (1.0 + eps)
                   : gs.uniform(p->v_lo, p->v_hi);
        ev.amp = gs.uniform(p->amp_lo, p->amp_hi);
        evs.push_back(ev);
      }
    }
    const double mx = g * p->spacing;
    cdp_id[gl] = static_cast<uint32_t>(g);
    ntraces[gl] = M;
    for (int m = 0; m < M; ++m) {
      const double h = p->h0 + m * p->dh;
      float* c4 = coords + (static_cast<size_t>(gl) * M + m) * 4;
      c4[0] = static_cast<float>(mx - h);
      c4[1] = 0.0f;
      c4[2] = static_cast<float>(mx + h);
      c4[3] = 0.0f;
      if (!samples) continue;
      float* tr = samples + (static_cast<size_t>(gl) * M + m) * ns;
      std::fill(tr, tr + ns, 0.0f);
      if (p->kind == 0) {
        for (const Event& ev : evs) {
          const double t = std::sqrt(ev.t0 * ev.t0 + 4.0 * h * h / (ev.v * ev.v));
          add_event(tr, ns, dt, t, ev.amp, p->freq);
        }
      } else {
        for (const Event& ev : line_events) {
          const double dm = mx - ev.x;
          const double tau = ev.t0 + 2.0 * ev.A * dm;
          const double t2 = tau * tau + 2.0 * ev.t0 * ev.B * dm * dm +
                            4.0 * h * h / (ev.v * ev.v);
          if (t2 > 0.0) add_event(tr, ns, dt, std::sqrt(t2), ev.amp, p->freq);
        }
      }
      if (p->sigma > 0.0) {
        Stream ns_(mix64(key ^ mix64(0xA0000000ull + m)));
        for (int s = 0; s + 1 < ns + 1; s += 2) {
          const double u1 = (static_cast<double>(ns_.next() >> 11) + 1.0) * 0x1.0p-53;
          const double u2 = static_cast<double>(ns_.next() >> 11) * 0x1.0p-53;
          const double r = std::sqrt(-2.0 * std::log(u1));
          const double th = 2.0 * M_PI * u2;
          tr[s] += static_cast<float>(p->sigma * r * std::cos(th));
          if (s + 1 < ns) tr[s + 1] += static_cast<float>(p->sigma * r * std::sin(th));
        }
      }
    }
  };

  int nt = p->n_threads > 0 ? p->n_threads
                            : static_cast<int>(std::thread::hardware_concurrency());
  nt = std::max(1, std::min(nt, G));
  if (nt <= 1) {
    for (int g = 0; g < G; ++g) gen_gather(g);
  } else {
    std::vector<std::thread> th;
    for (int t = 0; t < nt; ++t)
      th.emplace_back([&, t] {
        for (int g = t; g < G; g += nt) gen_gather(g);
      });
    for (auto& x : th) x.join();
  }
  return VELAN_GPU_OK;
}
