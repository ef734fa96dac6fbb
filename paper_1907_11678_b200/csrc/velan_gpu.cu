// velan_gpu.cu — host runtime of the C-ABI (include/velan_gpu.h).
//
// Replaces the reference's pipeline layer (cmp_pipeline.hpp, crs_pipeline.hpp)
// for the hot path:
//   * validation before any device work (ScanConfig::validate, scan.hpp:61-78;
//     scan_sweep's ns > w + 1, scan.hpp:113-114; partition's apm > 0,
//     crs_pipeline.hpp:95-98);
//   * TraceSweep construction on the host: h2 per trace (traveltime.hpp:16-27),
//     midpoints (types.hpp:57-62), the CRS neighbourhood as a closed ball in
//     cdp_id order (crs_pipeline.hpp:162-180) with fp32 d2 (kernel.hpp:86-91);
//   * data parallelism: contiguous blocks of output rows per device, each
//     device receiving its rows' gathers plus the CRS halo (replicated, no
//     collective), one host thread per device — the B200 form of
//     parallel_for_indexed (cmp_pipeline.hpp:34-88) and of run_crs's shards;
//   * H2D staging overlapped with compute: rows are launched in waves, the
//     copy stream uploads the gathers a wave needs while the previous wave
//     computes;
//   * results in input order (CMP) or cdp_id order (CRS, crs_pipeline.hpp:
//     449-459), bitwise independent of the device count.
#include <cuda_runtime.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <cmath>
#include <cstddef>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <exception>
#include <memory>
#include <mutex>
#include <limits>
#include <numeric>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/velan_gpu.h"
#include "semblance_kernels.cuh"

namespace velan_gpu {
namespace {

thread_local std::string g_last_error;

struct ApiError : std::runtime_error {
  int code;
  ApiError(int c, const std::string& m) : std::runtime_error(m), code(c) {}
};

[[noreturn]] void throw_cuda(cudaError_t e, const char* what, const char* file,
                             int line) {
  char buf[512];
  std::snprintf(buf, sizeof buf, "CUDA error %s (%s) in %s at %s:%d",
                cudaGetErrorName(e), cudaGetErrorString(e), what, file, line);
  throw ApiError(VELAN_GPU_ERUNTIME, buf);
}
#define VG_CUDA(expr)                                              \
  do {                                                             \
    cudaError_t e_ = (expr);                                       \
    if (e_ != cudaSuccess) throw_cuda(e_, #expr, __FILE__, __LINE__); \
  } while (0)

constexpr int kMaxW = 32;
// device memory of one per-wave semblance panel (host matrix / top-k scans)
constexpr size_t kPanelBytes = size_t(4) << 30;

// ---------------------------------------------------------------------------
// Kernel dispatch: (operator kind, variant, window) -> instantiation.

using KernelFn = void (*)(ScanParams);

struct KernelChoice {
  KernelFn fn = nullptr;
  int cc = 0;
  int cap = 0;  // compile-time stage capacity (FAST), 0 = runtime (EXACT)
  size_t slot_bytes = 0;  // plan slots + per-warp moveout terms (dynamic smem)
  bool quad = false;      // FAST table layout: quads (16 B) instead of pairs (8 B)
  int wmax = 0;           // compiled window bound (sizes the split-group scratch)
};

// FAST stage capacities (entries): the default, and the one for traces
// longer than it holds (one CTA per SM)
#ifndef VELAN_FAST_CAP
#define VELAN_FAST_CAP 5120
#endif
constexpr int kFastCap = VELAN_FAST_CAP;
// large stages: kStages of them in ~190 KB (6080 entries, ns <= 6032, at
// two stages; an ABC scan with both traces this long and a CRS-large
// aperture exceeds the 227 KB budget and is refused before any launch)
constexpr int kFastCapBig = (190 * 1024 / (kStages * 16)) / 32 * 32;
constexpr int kFastMaxNs = kFastCapBig - 48;  // staging_need(ns) <= cap
// the quad layout's stage (24 B per entry: a float4 quad + the float2
// energies): two stages in ~166 KB, traces up to 3408 samples.  Experimental
// (-DVELAN_QUAD): half the window loads, but the LDS.128 destinations cost
// register moves at 128 registers and it measured 0.5 % slower on CMP large
// (profiles/round2/experiments.md), so the pair layout is the default.
#ifdef VELAN_QUAD
#error "the experimental quad layout is stale: it fails parity since the byte-offset / exact-quotient hits (profiles/round2/experiments.md); do not build with -DVELAN_QUAD"
#endif
#ifndef VELAN_QUAD_CAP
#define VELAN_QUAD_CAP 3456
#endif
constexpr int kQuadCap = VELAN_QUAD_CAP;

template <int OPK, int VAR, int WMAX, bool FIXED, int CAPF = 0, bool QUAD = false>
KernelChoice pick() {
  // FAST keeps two accumulator rows (P, R) per pair: half the pairs
  // candidates per warp (the group of a CTA is kWarps x CC candidates)
  // (CC = 1 everywhere at 3 CTAs/SM — 80 registers, 6 warps per scheduler —
  // measured 1.21x slower on CMP large: instruction count beats occupancy)
  constexpr int CC = WMAX > 16 ? 1 : 2;
  constexpr int CAP = VAR == VAR_FAST ? (CAPF ? CAPF : kFastCap) : 0;
  return KernelChoice{&semblance_scan_kernel<OPK, VAR, WMAX, FIXED, CC, CAP, QUAD>, CC, CAP,
                      2 * kStages * sizeof(PlanSlot) +
                          sizeof(float) * kWarps * kBatch * qs_row(CC, OpTraits<OPK>::NQ),
                      QUAD, WMAX};
}

template <int OPK, int VAR>
KernelChoice pick_w(int w, bool big, bool quad) {
#ifdef VELAN_QUAD
  if constexpr (VAR == VAR_FAST) {
    if (quad) {  // fixed windows, traces that fit the quad stage
      switch (w) {
        case 1: return pick<OPK, VAR, 1, true, kQuadCap, true>();
        case 2: return pick<OPK, VAR, 2, true, kQuadCap, true>();
        case 4: return pick<OPK, VAR, 4, true, kQuadCap, true>();
        case 8: return pick<OPK, VAR, 8, true, kQuadCap, true>();
        case 11: return pick<OPK, VAR, 11, true, kQuadCap, true>();
        case 15: return pick<OPK, VAR, 15, true, kQuadCap, true>();
        case 16: return pick<OPK, VAR, 16, true, kQuadCap, true>();
        default: break;
      }
    }
  }
#else
  (void)quad;
#endif
  if (VAR == VAR_FAST && big) {  // rare: generic windows only
    if (w <= 4) return pick<OPK, VAR, 4, false, kFastCapBig>();
    if (w <= 8) return pick<OPK, VAR, 8, false, kFastCapBig>();
    if (w <= 16) return pick<OPK, VAR, 16, false, kFastCapBig>();
    return pick<OPK, VAR, 32, false, kFastCapBig>();
  }
  switch (w) {
    case 1: return pick<OPK, VAR, 1, true>();
    case 2: return pick<OPK, VAR, 2, true>();
    case 4: return pick<OPK, VAR, 4, true>();
    case 8: return pick<OPK, VAR, 8, true>();
    case 11: return pick<OPK, VAR, 11, true>();
    case 15: return pick<OPK, VAR, 15, true>();
    case 16: return pick<OPK, VAR, 16, true>();
    default: break;
  }
  if (w <= 4) return pick<OPK, VAR, 4, false>();
  if (w <= 8) return pick<OPK, VAR, 8, false>();
  if (w <= 16) return pick<OPK, VAR, 16, false>();
  return pick<OPK, VAR, 32, false>();
}

bool is_fixed_window(int w) {
  return w == 1 || w == 2 || w == 4 || w == 8 || w == 11 || w == 15 || w == 16;
}

int staging_need(int ns, bool fast);

// FAST: the quad layout when the window is a compiled one and a trace fits
// its stage; the pair layout (larger stage) otherwise.
KernelChoice choose_kernel(int op, int variant, int w, int ns) {
  const bool fast = variant == VELAN_VARIANT_FAST;
  const bool quad = fast && is_fixed_window(w) && staging_need(ns, true) <= kQuadCap;
  const bool big = fast && staging_need(ns, true) > kFastCap;
  const int opk = op == VELAN_OP_CRS_ABC ? OPK_ABC : OPK_Q;
  if (opk == OPK_Q)
    return variant == VELAN_VARIANT_EXACT ? pick_w<OPK_Q, VAR_EXACT>(w, big, false)
                                          : pick_w<OPK_Q, VAR_FAST>(w, big, quad);
  return variant == VELAN_VARIANT_EXACT ? pick_w<OPK_ABC, VAR_EXACT>(w, big, false)
                                        : pick_w<OPK_ABC, VAR_FAST>(w, big, quad);
}

// ---------------------------------------------------------------------------
// Validation (before any device work).

std::string fmt(const char* f, long long a = 0, long long b = 0) {
  char buf[256];
  std::snprintf(buf, sizeof buf, f, a, b);
  return buf;
}

void validate(const velan_gpu_dataset* ds, const velan_gpu_scan* sc,
              bool crs) {
  if (!ds || !sc) throw ApiError(VELAN_GPU_EPARAM, "null dataset or scan");
  // ScanConfig::validate (scan.hpp:61-78)
  if (sc->w < 1) throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: w must be >= 1");
  if (sc->n_c < 1)
    throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: nc must be >= 1");
  if (sc->op != VELAN_OP_NMO && sc->op != VELAN_OP_CRS_D2 &&
      sc->op != VELAN_OP_CRS_ABC)
    throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: unknown moveout operator");
  if (sc->variant != VELAN_VARIANT_EXACT && sc->variant != VELAN_VARIANT_FAST)
    throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: unknown kernel variant");
  if (crs && sc->op == VELAN_OP_NMO)
    throw ApiError(VELAN_GPU_ECONFIG,
                   "velan_gpu_crs: operator must be CRS_D2 or CRS_ABC");
  if (!crs && sc->op != VELAN_OP_NMO)
    throw ApiError(VELAN_GPU_ECONFIG, "velan_gpu_cmp: operator must be NMO");
  if (sc->w > kMaxW)
    throw ApiError(VELAN_GPU_ECONFIG,
                   fmt("ScanConfig: w = %lld exceeds the GPU kernels' maximum "
                       "window of %lld samples",
                       sc->w, kMaxW));
  if (!sc->v) throw ApiError(VELAN_GPU_EPARAM, "velocity candidates are null");
  for (int c = 0; c < sc->n_c; ++c)
    if (!(sc->v[c] > 0.0f) || !std::isfinite(sc->v[c]))
      throw ApiError(VELAN_GPU_ECONFIG,
                     "ScanConfig: need 0 < v for every velocity candidate");
  if (sc->op == VELAN_OP_CRS_ABC) {
    if (sc->n_a < 1 || sc->n_b < 1 || !sc->a || !sc->b)
      throw ApiError(VELAN_GPU_ECONFIG,
                     "ScanConfig: CRS_ABC needs n_a >= 1 and n_b >= 1");
    for (int i = 0; i < sc->n_a; ++i)
      if (!std::isfinite(sc->a[i]))
        throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: non-finite A candidate");
    for (int i = 0; i < sc->n_b; ++i)
      if (!std::isfinite(sc->b[i]))
        throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: non-finite B candidate");
    const long long nc = 1LL * sc->n_a * sc->n_b * sc->n_c;
    if (nc > (1LL << 30))
      throw ApiError(VELAN_GPU_ECONFIG, "ScanConfig: too many candidates");
  }
  // dataset shape
  if (ds->n_gathers < 0) throw ApiError(VELAN_GPU_EPARAM, "n_gathers < 0");
  if (sc->row_first < 0 || sc->row_count < 0 ||
      static_cast<long long>(sc->row_first) + sc->row_count > ds->n_gathers ||
      (sc->row_count == 0 && sc->row_first != 0))
    throw ApiError(VELAN_GPU_EPARAM, "output row range outside the dataset");
  if (ds->n_gathers == 0) return;  // run_cmp / run_crs return {} (no error)
  if (crs && !(sc->apm > 0.0))
    throw ApiError(VELAN_GPU_ECONFIG, "partition: apm must be > 0");
  if (ds->max_traces < 1)
    throw ApiError(VELAN_GPU_EPARAM, "max_traces must be >= 1");
  if (ds->dt_us == 0) throw ApiError(VELAN_GPU_EPARAM, "dt must be > 0");
  if (!ds->ntraces || !ds->coords || !ds->samples || !ds->cdp_id)
    throw ApiError(VELAN_GPU_EPARAM, "dataset arrays are null");
  if (ds->samples_mem != VELAN_MEM_HOST && ds->samples_mem != VELAN_MEM_DEVICE)
    throw ApiError(VELAN_GPU_EPARAM, "samples_mem must be HOST or DEVICE");
  // scan_sweep: the window plus its interpolation neighbour must fit
  if (ds->ns <= sc->w + 1)
    throw ApiError(VELAN_GPU_ECONFIG,
                   "scan_sweep: window does not fit trace length");
  // one trace must fit a staging stage (kStages stages per CTA)
  if (ds->ns > (sc->variant == VELAN_VARIANT_FAST ? kFastMaxNs : 27000))
    throw ApiError(VELAN_GPU_ECONFIG,
                   fmt("ns exceeds the shared-memory staging capacity of the "
                       "kernel variant (FAST %lld, EXACT %lld samples)",
                       kFastMaxNs, 27000));
  for (int g = 0; g < ds->n_gathers; ++g) {
    if (ds->ntraces[g] < 0 || ds->ntraces[g] > ds->max_traces)
      throw ApiError(VELAN_GPU_EPARAM,
                     fmt("gather %lld: ntraces outside [0, max_traces]", g));
  }
  for (int g = 0; g < ds->n_gathers; ++g)
    if (ds->ntraces[g] == 0) {
      if (crs)  // partition -> midpoint_of throws (crs_pipeline.hpp:104)
        throw ApiError(VELAN_GPU_EPARAM, "midpoint_of: gather has no traces");
      // run_cmp: the worker's TraceSweep throws, the pool wraps it
      // (cmp_pipeline.hpp:77-85, kernel.hpp:100-101)
      throw ApiError(
          VELAN_GPU_ERUNTIME,
          fmt("worker pool failure after 0 of %lld jobs: TraceSweep: central "
              "gather has no traces (gather %lld)",
              ds->n_gathers, g));
    }
}

// ---------------------------------------------------------------------------
// Host-side sweep construction.

struct HostSweep {
  int G = 0, M = 0, ns = 0, rows = 0;
  int op = 0, w = 0, n_a = 1, n_b = 1, n_c = 1, ncand = 1;
  double dt = 0.0;
  std::vector<float> h2;          // [G][M]
  std::vector<float> mx, my;      // [G]
  std::vector<int> row_gather;    // [rows]
  std::vector<int> leg_off;       // [rows + 1]
  std::vector<int> leg_gather;    // global gather index
  std::vector<float> leg_d2, leg_dm;
  std::vector<long long> row_traces;  // traces per sweep
  std::vector<float> t0;          // [ns]
  std::vector<float> a, b, v;
};

HostSweep build_sweep(const velan_gpu_dataset* ds, const velan_gpu_scan* sc) {
  HostSweep h;
  h.G = ds->n_gathers;
  h.M = ds->max_traces;
  h.ns = ds->ns;
  h.op = sc->op;
  h.w = sc->w;
  h.n_a = sc->op == VELAN_OP_CRS_ABC ? sc->n_a : 1;
  h.n_b = sc->op == VELAN_OP_CRS_ABC ? sc->n_b : 1;
  h.n_c = sc->n_c;
  h.ncand = h.n_a * h.n_b * h.n_c;
  h.dt = static_cast<double>(ds->dt_us) * 1e-6;  // CdpGather::dt_seconds
  h.v.assign(sc->v, sc->v + sc->n_c);
  if (sc->op == VELAN_OP_CRS_ABC) {
    h.a.assign(sc->a, sc->a + sc->n_a);
    h.b.assign(sc->b, sc->b + sc->n_b);
  } else {
    h.a.assign(1, 0.0f);
    h.b.assign(1, 0.0f);
  }
  // t0_k = float(k * dt_s), scan.hpp:133
  h.t0.resize(h.ns);
  for (int k = 0; k < h.ns; ++k) h.t0[k] = static_cast<float>(k * h.dt);
  // compute_halfpoints (traveltime.hpp:16-27) and midpoint_of
  h.h2.assign(static_cast<size_t>(h.G) * h.M, 0.0f);
  h.mx.assign(h.G, 0.0f);
  h.my.assign(h.G, 0.0f);
  for (int g = 0; g < h.G; ++g) {
    for (int m = 0; m < ds->ntraces[g]; ++m) {
      const float* c4 = ds->coords + (static_cast<size_t>(g) * h.M + m) * 4;
      const float dx = c4[2] - c4[0];
      const float dy = c4[3] - c4[1];
      h.h2[static_cast<size_t>(g) * h.M + m] = (dx * dx + dy * dy) * 0.25f;
    }
    const float* c0 = ds->coords + static_cast<size_t>(g) * h.M * 4;
    h.mx[g] = (c0[0] + c0[2]) * 0.5f;
    h.my[g] = (c0[1] + c0[3]) * 0.5f;
  }
  // output rows
  h.rows = h.G;
  h.row_gather.resize(h.G);
  std::iota(h.row_gather.begin(), h.row_gather.end(), 0);
  if (sc->op != VELAN_OP_NMO)
    std::stable_sort(h.row_gather.begin(), h.row_gather.end(),
                     [&](int x, int y) { return ds->cdp_id[x] < ds->cdp_id[y]; });
  if (sc->row_count > 0) {  // a shard's own block; the rest is halo
    h.row_gather.erase(h.row_gather.begin(),
                       h.row_gather.begin() + sc->row_first);
    h.row_gather.resize(sc->row_count);
    h.rows = sc->row_count;
  }
  h.leg_off.assign(1, 0);
  h.row_traces.resize(h.rows);
  if (sc->op == VELAN_OP_NMO) {
    for (int r = 0; r < h.rows; ++r) {
      const int g = h.row_gather[r];
      h.leg_gather.push_back(g);
      h.leg_d2.push_back(0.0f);
      h.leg_dm.push_back(0.0f);
      h.leg_off.push_back(static_cast<int>(h.leg_gather.size()));
      h.row_traces[r] = ds->ntraces[g];
    }
    return h;
  }
  // CRS neighbourhoods: closed ball |dm| <= apm (double compare of the
  // fp32 difference, crs_pipeline.hpp:172-174), self excluded, empty
  // gathers skipped (kernel.hpp:87), cdp_id order (crs_pipeline.hpp:176-179)
  std::vector<int> by_x(h.G);
  std::iota(by_x.begin(), by_x.end(), 0);
  std::sort(by_x.begin(), by_x.end(),
            [&](int x, int y) { return h.mx[x] < h.mx[y]; });
  std::vector<double> xs(h.G);
  for (int i = 0; i < h.G; ++i) xs[i] = h.mx[by_x[i]];
  const double apm = sc->apm;
  const double margin = apm * 1e-5 + 1e-3;
  std::vector<int> nb;
  for (int r = 0; r < h.rows; ++r) {
    const int g = h.row_gather[r];
    nb.clear();
    const auto lo = std::lower_bound(xs.begin(), xs.end(),
                                     static_cast<double>(h.mx[g]) - apm - margin);
    const auto hi = std::upper_bound(xs.begin(), xs.end(),
                                     static_cast<double>(h.mx[g]) + apm + margin);
    for (auto it = lo; it != hi; ++it) {
      const int o = by_x[it - xs.begin()];
      if (o == g || ds->ntraces[o] == 0) continue;
      const double dx = static_cast<double>(h.mx[o] - h.mx[g]);
      const double dy = static_cast<double>(h.my[o] - h.my[g]);
      if (dx * dx + dy * dy <= apm * apm) nb.push_back(o);
    }
    std::sort(nb.begin(), nb.end(), [&](int x, int y) {
      return ds->cdp_id[x] != ds->cdp_id[y] ? ds->cdp_id[x] < ds->cdp_id[y]
                                            : x < y;
    });
    long long traces = ds->ntraces[g];
    h.leg_gather.push_back(g);
    h.leg_d2.push_back(0.0f);
    h.leg_dm.push_back(0.0f);
    for (int o : nb) {
      const float dx = h.mx[o] - h.mx[g];
      const float dy = h.my[o] - h.my[g];
      h.leg_gather.push_back(o);
      h.leg_d2.push_back(dx * dx + dy * dy);
      h.leg_dm.push_back(dx);
      traces += ds->ntraces[o];
    }
    h.leg_off.push_back(static_cast<int>(h.leg_gather.size()));
    h.row_traces[r] = traces;
  }
  return h;
}

// ---------------------------------------------------------------------------
// Device buffers.

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  void ensure(size_t n) {
    if (n <= bytes && p) return;
    if (p) VG_CUDA(cudaFree(p));
    p = nullptr;
    bytes = 0;
    if (n == 0) n = 16;
    VG_CUDA(cudaMalloc(&p, n));
    bytes = n;
  }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  template <class T>
  T* as() const {
    return static_cast<T*>(p);
  }
};

enum BufId {
  B_SAMPLES, B_EC, B_H2, B_NTR, B_LEGOFF, B_LEGG, B_LEGD2, B_LEGDM, B_T0, B_A, B_B,
  B_V, B_BIDX, B_BS, B_BST, B_MAT, B_VALID, B_TKI, B_TKS, B_COUNT
};

struct DeviceState {
  int dev = 0;
  cudaStream_t stream = nullptr, copy_stream = nullptr, d2h_stream = nullptr;
  DevBuf bufs[B_COUNT];
  std::vector<cudaEvent_t> events;
  cudaEvent_t ev(size_t i) {
    while (events.size() <= i) {
      cudaEvent_t e;
      VG_CUDA(cudaEventCreate(&e));
      events.push_back(e);
    }
    return events[i];
  }
  int n_sm = 148;
  void init(int d) {
    dev = d;
    VG_CUDA(cudaSetDevice(d));
    VG_CUDA(cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, d));
    VG_CUDA(cudaStreamCreateWithFlags(&stream, cudaStreamNonBlocking));
    VG_CUDA(cudaStreamCreateWithFlags(&copy_stream, cudaStreamNonBlocking));
    VG_CUDA(cudaStreamCreateWithFlags(&d2h_stream, cudaStreamNonBlocking));
  }
  void destroy() {
    cudaSetDevice(dev);
    for (auto& b : bufs) b.release();
    for (auto e : events) cudaEventDestroy(e);
    events.clear();
    if (stream) cudaStreamDestroy(stream);
    if (copy_stream) cudaStreamDestroy(copy_stream);
    if (d2h_stream) cudaStreamDestroy(d2h_stream);
    stream = copy_stream = d2h_stream = nullptr;
  }
};

// A shard: rows [r0, r1) of the global sweep on one device.
struct Shard {
  int r0 = 0, r1 = 0;
  std::vector<int> local_gathers;  // local -> global gather, ascending
  std::vector<int> leg_off, leg_gather;
  std::vector<float> leg_d2, leg_dm;
  std::vector<float> h2;
  std::vector<int> ntr;
  std::vector<int> wave_rows;  // wave boundaries (local rows)
  std::vector<int> wave_need;  // local gathers needed up to each wave
  std::vector<int> wave_lo;    // first local gather a wave's sweeps touch
  std::vector<int> wave_hi;    // one past the last
  int max_wave_rows = 0;
  int table_span = 0;          // max over waves of wave_hi - wave_lo
  long long nominal = 0;
};

// max_wave_rows caps the rows of one launch (the per-wave semblance panel
// of a matrix / top-k scan: rows x ns x ncand floats, never a whole shard).
Shard make_shard(const HostSweep& h, const velan_gpu_dataset* ds, int r0,
                 int r1, bool identity_gathers, long long max_wave_rows = 65535) {
  Shard s;
  s.r0 = r0;
  s.r1 = r1;
  const int lb = h.leg_off[r0], le = h.leg_off[r1];
  if (identity_gathers) {
    s.local_gathers.resize(h.G);
    std::iota(s.local_gathers.begin(), s.local_gathers.end(), 0);
  } else {
    s.local_gathers.assign(h.leg_gather.begin() + lb, h.leg_gather.begin() + le);
    std::sort(s.local_gathers.begin(), s.local_gathers.end());
    s.local_gathers.erase(
        std::unique(s.local_gathers.begin(), s.local_gathers.end()),
        s.local_gathers.end());
  }
  std::vector<int> g2l;
  if (!identity_gathers) {
    g2l.assign(h.G, -1);
    for (size_t i = 0; i < s.local_gathers.size(); ++i)
      g2l[s.local_gathers[i]] = static_cast<int>(i);
  }
  const int L = static_cast<int>(s.local_gathers.size());
  s.h2.resize(static_cast<size_t>(L) * h.M);
  s.ntr.resize(L);
  for (int l = 0; l < L; ++l) {
    const int g = s.local_gathers[l];
    std::memcpy(&s.h2[static_cast<size_t>(l) * h.M],
                &h.h2[static_cast<size_t>(g) * h.M], sizeof(float) * h.M);
    s.ntr[l] = ds->ntraces[g];
  }
  s.leg_off.resize(r1 - r0 + 1);
  for (int r = r0; r <= r1; ++r) s.leg_off[r - r0] = h.leg_off[r] - lb;
  s.leg_gather.resize(le - lb);
  for (int i = lb; i < le; ++i)
    s.leg_gather[i - lb] =
        identity_gathers ? h.leg_gather[i] : g2l[h.leg_gather[i]];
  s.leg_d2.assign(h.leg_d2.begin() + lb, h.leg_d2.begin() + le);
  s.leg_dm.assign(h.leg_dm.begin() + lb, h.leg_dm.begin() + le);
  for (int r = r0; r < r1; ++r)
    s.nominal += h.row_traces[r] * static_cast<long long>(h.ns) * h.ncand;
  // waves: ~equal nominal work, >= 2 waves of CTAs per launch when possible
  const long long per_row_ctas = (h.ns + kT0 - 1) / kT0;
  const long long rows = r1 - r0;
  long long total_work = 0;
  for (int r = r0; r < r1; ++r) total_work += h.row_traces[r];
  total_work *= static_cast<long long>(h.ns) * h.ncand * h.w;
  // target ~1.5e12 window evaluations per launch (~1 s), but at least
  // 8 waves worth of CTAs, and at most 65535 rows (grid.y)
  const long long target_evals = 1500000000000LL;
  long long rows_per_wave =
      std::max<long long>(1, rows * target_evals / std::max(total_work, 1LL));
  rows_per_wave = std::max<long long>(
      rows_per_wave, std::min<long long>(rows, (148LL * 4 * 8) / per_row_ctas + 1));
  const long long cap = std::max<long long>(1, std::min<long long>(max_wave_rows, 65535));
  rows_per_wave = std::min<long long>(rows_per_wave, cap);
  rows_per_wave = std::max<long long>(rows_per_wave, 1);
  // the first waves ramp up (1/8, 1/4, 1/2 of the target): the upload of
  // wave 0 is the only one not hidden behind a scan, so keep it small
  const long long min_rows =
      std::min(cap, std::min<long long>(rows, 148LL * 2 / per_row_ctas + 1));
  int need = 0;
  long long step = rows_per_wave;
  for (long long b = 0, i = 0; b < rows; b += step, ++i) {
    step = std::max(min_rows, rows_per_wave >> std::max<long long>(0, 3 - i));
    const long long e = std::min(rows, b + step);
    int lo = std::numeric_limits<int>::max(), hi = 0;
    for (long long i = s.leg_off[b]; i < s.leg_off[e]; ++i) {
      lo = std::min(lo, s.leg_gather[i]);
      hi = std::max(hi, s.leg_gather[i] + 1);
    }
    need = std::max(need, hi);
    s.wave_rows.push_back(static_cast<int>(b));
    s.wave_need.push_back(need);
    s.wave_lo.push_back(lo);
    s.wave_hi.push_back(hi);
    s.max_wave_rows = std::max<int>(s.max_wave_rows, static_cast<int>(e - b));
    s.table_span = std::max(s.table_span, hi - lo);
  }
  s.wave_rows.push_back(static_cast<int>(rows));
  return s;
}

template <class T>
void upload(DevBuf& b, const std::vector<T>& v, cudaStream_t st) {
  b.ensure(sizeof(T) * std::max<size_t>(v.size(), 1));
  if (!v.empty())
    VG_CUDA(cudaMemcpyAsync(b.p, v.data(), sizeof(T) * v.size(),
                            cudaMemcpyHostToDevice, st));
}

// Device-resident samples must live on the device that runs the scan: the
// pointer's owner (cudaPointerGetAttributes) and the declared samples_device
// both have to match, or the kernels would fault or read a peer over NVLink.
void check_device_samples(const velan_gpu_dataset* ds, int dev) {
  if (ds->samples_mem != VELAN_MEM_DEVICE || ds->n_gathers == 0) return;
  if (ds->samples_device != dev)
    throw ApiError(VELAN_GPU_ECONFIG,
                   fmt("device-resident samples declared on device %lld, the context "
                       "runs on device %lld",
                       ds->samples_device, dev));
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, ds->samples) != cudaSuccess) {
    cudaGetLastError();
    throw ApiError(VELAN_GPU_ECONFIG, "samples_mem is DEVICE but samples is not a CUDA pointer");
  }
  if (a.type != cudaMemoryTypeDevice && a.type != cudaMemoryTypeManaged)
    throw ApiError(VELAN_GPU_ECONFIG, "samples_mem is DEVICE but samples is host memory");
  if (a.type == cudaMemoryTypeDevice && a.device != dev)
    throw ApiError(VELAN_GPU_ECONFIG,
                   fmt("device-resident samples live on device %lld, the context runs on "
                       "device %lld",
                       a.device, dev));
}

void set_smem_attr(KernelFn fn, size_t smem) {
  VG_CUDA(cudaFuncSetAttribute(reinterpret_cast<const void*>(fn),
                               cudaFuncAttributeMaxDynamicSharedMemorySize,
                               static_cast<int>(smem)));
}

// Entries per staging stage: one 512-thread CTA per SM fits kStages
// stages.  FAST entries are 16 B (a sample pair and its window energies),
// EXACT entries fp32 samples.  A stage must hold one whole trace plus the
// zero pad.
int staging_need(int ns, bool fast) {
  return ((ns + 3) / 4) * 4 + 8 + (fast ? 40 : 0);
}
int staging_cap(int ns, bool fast) {
  if (fast) return staging_need(ns, true) <= kFastCap ? kFastCap : kFastCapBig;
  const int cap = std::max(8192, staging_need(ns, false));
  return (cap + 31) / 32 * 32;
}

void check_topk(const velan_gpu_result* res) {
  if (res->topk < 0 || res->topk > 8)
    throw ApiError(VELAN_GPU_EPARAM, "topk must be in [0, 8]");
  if (res->topk > 0 && (!res->topk_idx || !res->topk_semblance))
    throw ApiError(VELAN_GPU_EPARAM, "topk output arrays are null");
}

struct RunOut {
  uint64_t valid = 0;
  double kernel_ms = 0.0;
  int launches = 0;
};

// Run one shard on one device.  When out_host is true the result arrays are
// host memory and rows are copied back at the end; samples are uploaded
// from host (per wave) unless d_samples_ext is given.
//
// Memory is bounded per WAVE (a launch's rows), not per shard:
//   * FAST tables (16 B per sample) exist only for the gathers the current
//     wave's sweeps touch [wave_lo, wave_hi) — CRS waves recompute their
//     halo gathers; the scan kernel indexes the tables relative to
//     table_trace0;
//   * a requested semblance panel (host matrix or top-k) is per wave: the
//     kernel writes rows relative to mat_row0, top-k reduces the wave's panel
//     in place, and a host matrix leaves the device per wave on its own
//     stream (two panels alternate so the copy of wave i overlaps the scan
//     of wave i + 1).
RunOut run_shard(DeviceState& D, const HostSweep& h, const Shard& s,
                 const velan_gpu_dataset* ds, const velan_gpu_scan* sc,
                 velan_gpu_result* res, const float* d_samples_ext,
                 cudaStream_t user_stream, bool tables_resident,
                 bool samples_resident) {
  VG_CUDA(cudaSetDevice(D.dev));
  cudaStream_t st = user_stream ? user_stream : D.stream;
  const int rows = s.r1 - s.r0;
  RunOut out;
  if (rows <= 0) return out;
  const int L = static_cast<int>(s.local_gathers.size());
  const size_t trace_floats = static_cast<size_t>(h.M) * h.ns;

  if (!tables_resident) {
    upload(D.bufs[B_H2], s.h2, st);
    upload(D.bufs[B_NTR], s.ntr, st);
    upload(D.bufs[B_LEGOFF], s.leg_off, st);
    upload(D.bufs[B_LEGG], s.leg_gather, st);
    upload(D.bufs[B_LEGD2], s.leg_d2, st);
    upload(D.bufs[B_LEGDM], s.leg_dm, st);
    upload(D.bufs[B_T0], h.t0, st);
    upload(D.bufs[B_A], h.a, st);
    upload(D.bufs[B_B], h.b, st);
    upload(D.bufs[B_V], h.v, st);
  }
  const bool out_host = res->out_mem == VELAN_MEM_HOST;
  const size_t cells = static_cast<size_t>(rows) * h.ns;
  const size_t row_cells = static_cast<size_t>(h.ns);
  const size_t panel_row = row_cells * h.ncand;  // floats per row of a panel
  const int K = res->topk;
  int32_t* d_bidx;
  float *d_bs, *d_bst;
  int32_t* d_tki = nullptr;
  float* d_tks = nullptr;
  // the semblance panel: the caller's device matrix (device-out), or per-wave
  // internal panels (a host matrix: two alternating; top-k only: one)
  float* d_mat_user = nullptr;
  float* d_panel[2] = {nullptr, nullptr};
  const bool host_matrix = out_host && res->matrix;
  if (out_host) {
    if (K > 0) {
      D.bufs[B_TKI].ensure(cells * K * 4);
      D.bufs[B_TKS].ensure(cells * K * 4);
      d_tki = D.bufs[B_TKI].as<int32_t>();
      d_tks = D.bufs[B_TKS].as<float>();
    }
    D.bufs[B_BIDX].ensure(cells * 4);
    D.bufs[B_BS].ensure(cells * 4);
    D.bufs[B_BST].ensure(cells * 4);
    d_bidx = D.bufs[B_BIDX].as<int32_t>();
    d_bs = D.bufs[B_BS].as<float>();
    d_bst = D.bufs[B_BST].as<float>();
  } else {
    d_bidx = res->best_idx + static_cast<size_t>(s.r0) * h.ns;
    d_bs = res->best_semblance + static_cast<size_t>(s.r0) * h.ns;
    d_bst = res->best_stack + static_cast<size_t>(s.r0) * h.ns;
    if (res->matrix) d_mat_user = res->matrix + static_cast<size_t>(s.r0) * panel_row;
    if (K > 0) {
      d_tki = res->topk_idx + static_cast<size_t>(s.r0) * h.ns * K;
      d_tks = res->topk_semblance + static_cast<size_t>(s.r0) * h.ns * K;
    }
  }
  if (!d_mat_user && (host_matrix || K > 0)) {
    const size_t panel = static_cast<size_t>(s.max_wave_rows) * panel_row;
    const int np = host_matrix ? 2 : 1;
    D.bufs[B_MAT].ensure(panel * np * 4);
    d_panel[0] = D.bufs[B_MAT].as<float>();
    d_panel[1] = host_matrix ? d_panel[0] + panel : d_panel[0];
  }
  D.bufs[B_VALID].ensure(8);
  VG_CUDA(cudaMemsetAsync(D.bufs[B_VALID].p, 0, 8, st));

  // samples: external device pointer, resident, or uploaded per wave
  const float* d_samples = d_samples_ext;
  const bool upload_samples = !d_samples_ext && !samples_resident;
  if (!d_samples_ext) {
    if (upload_samples) D.bufs[B_SAMPLES].ensure(
        std::max<size_t>(1, static_cast<size_t>(L) * trace_floats * 4 + 64));
    d_samples = D.bufs[B_SAMPLES].as<float>();
  }

  const bool fast = sc->variant == VELAN_VARIANT_FAST;
  const KernelChoice kc = choose_kernel(h.op, sc->variant, h.w, h.ns);
  ScanParams p{};
  p.samples = d_samples;
  p.h2 = D.bufs[B_H2].as<float>();
  p.ntr = D.bufs[B_NTR].as<int>();
  p.leg_off = D.bufs[B_LEGOFF].as<int>();
  p.leg_gather = D.bufs[B_LEGG].as<int>();
  p.leg_d2 = D.bufs[B_LEGD2].as<float>();
  p.leg_dm = D.bufs[B_LEGDM].as<float>();
  p.t0 = D.bufs[B_T0].as<float>();
  p.cand_a = D.bufs[B_A].as<float>();
  p.cand_b = D.bufs[B_B].as<float>();
  p.cand_v = D.bufs[B_V].as<float>();
  p.n_a = h.n_a;
  p.n_b = h.n_b;
  p.n_c = h.n_c;
  p.ncand = h.ncand;
  p.Mmax = h.M;
  p.ns = h.ns;
  p.w = h.w;
  // TMA bulk copies need 16-byte aligned trace segments: EXACT stages the
  // samples (ns % 4), FAST its own pair/energy tables (ns % 2)
  p.vec4 = sc->variant == VELAN_VARIANT_FAST
               ? (h.ns % 2 == 0)
               : (h.ns % 4 == 0) &&
                     (reinterpret_cast<uintptr_t>(d_samples) % 16 == 0);
  p.cap = kc.cap ? kc.cap : staging_cap(h.ns, fast);
  char* d_tab = nullptr;
  float2* d_ec = nullptr;
  size_t tab_traces = 0;
  const size_t tab_b = kc.quad ? 16 : 8;  // table entry bytes
  if (fast) {
    // pairs (quads) then energies of one wave's gathers: 16 (24) B per sample
    tab_traces = static_cast<size_t>(std::max(s.table_span, 1)) * h.M;
    D.bufs[B_EC].ensure(tab_traces * h.ns * (tab_b + 8) + 64);
    d_tab = D.bufs[B_EC].as<char>();
    d_ec = reinterpret_cast<float2*>(d_tab + tab_traces * h.ns * tab_b);
    p.pairs = reinterpret_cast<const float2*>(d_tab);
    p.quads = reinterpret_cast<const float4*>(d_tab);
    p.ec = d_ec;
  }
  p.dt = h.dt;
  {
    const double inv = 1.0 / h.dt;
    p.inv_hi = static_cast<float>(inv);
    p.inv_lo = static_cast<float>(inv - static_cast<double>(p.inv_hi));
    p.amb_eps = static_cast<float>(std::ldexp(std::max(h.ns, 16), -40));
    // Exact quotient: 1/dt is an integer N (a float) and dt = (1 + e)/N with
    // |e| < 2^-54.  Then for every float t the double t N is exact (<= 24 +
    // 20 bits) and |t N e| is below half an ulp of it, so hit_for's
    // double(t) / dt (traveltime.hpp:66-80) rounds to t N itself: the FAST
    // hit (floor and fraction of the exact product) equals the reference's
    // bit for bit and needs no near-integer fix-up.  dt = 1, 2, 4 ms ...
    const double n = std::nearbyint(inv);
    p.exact_q = (inv == n && n >= 1.0 && n <= 1048576.0 &&
                 std::fabs(std::fma(h.dt, n, -1.0)) < std::ldexp(1.0, -54))
                    ? 1
                    : 0;
  }
  p.best_idx = d_bidx;
  p.best_s = d_bs;
  p.best_stack = d_bst;
  p.valid = D.bufs[B_VALID].as<unsigned long long>();
  // per-row metadata staged in shared memory by the kernel
  int max_legs = 1, max_sweep = 1;
  for (int r = 0; r < rows; ++r) {
    max_legs = std::max(max_legs, s.leg_off[r + 1] - s.leg_off[r]);
    max_sweep = std::max<long long>(max_sweep, h.row_traces[s.r0 + r]);
  }
  p.max_legs = max_legs;
  p.max_sweep = max_sweep;
  // + the consumers' per-tile argmax scratch [2][3][kWarps - 1][kT0]
  const size_t meta_floats = 5 * static_cast<size_t>(max_legs) + max_sweep +
                             h.n_a + h.n_b + h.n_c + 6 * (kWarps - 1) * kT0;
  size_t smem =
      (static_cast<size_t>(kStages) * p.cap * (fast ? (kc.quad ? 6 : 4) : 1) + meta_floats) *
          sizeof(float) +
      kc.slot_bytes;
  // A last candidate group that fills at most half of the consumer warps is
  // swept by two warps per candidate pair (half a batch each; FAST, two
  // candidates per warp): the helpers' partial sums go through a scratch of
  // [consumer warps / 2][2][w + 2][32] floats — when the budget has room
  p.tail_split = 0;
  if (fast && kc.cc == 2 && h.op != VELAN_OP_CRS_ABC) {
    const int cg = (kWarps - 1) * kc.cc;
    const int rem = h.ncand % cg ? h.ncand % cg : cg;
    const size_t merge_bytes =
        sizeof(float) * ((kWarps - 1) / 2) * kc.cc * (kc.wmax + 2) * kT0;
    cudaFuncAttributes fa0{};
    VG_CUDA(cudaFuncGetAttributes(&fa0, reinterpret_cast<const void*>(kc.fn)));
    if (2 * ((rem + kc.cc - 1) / kc.cc) <= kWarps - 1 &&
        smem + merge_bytes + fa0.sharedSizeBytes <= 227 * 1024) {
      p.tail_split = 1;
      smem += merge_bytes;
    }
  }
  // the kernel's static __shared__ (barriers, planner state) counts against
  // the same 227 KB opt-in limit as the dynamic allocation
  cudaFuncAttributes fa{};
  VG_CUDA(cudaFuncGetAttributes(&fa, reinterpret_cast<const void*>(kc.fn)));
  if (smem + fa.sharedSizeBytes > 227 * 1024)
    throw ApiError(VELAN_GPU_ECONFIG,
                   "scan exceeds the 227 KB shared-memory budget of a CTA "
                   "(too many traces per sweep or candidates)");
  set_smem_attr(kc.fn, smem);

  const int nwaves = static_cast<int>(s.wave_need.size());
  // event slots: [2 wv, 2 wv + 1] timing, [2 nw + wv] upload done,
  // [3 nw + wv] scan done (panel ready), [4 nw + b] panel b copied out
  int uploaded = 0;
  int tab_lo = 0, tab_hi = 0;  // gathers the FAST tables currently hold
  for (int wv = 0; wv < nwaves; ++wv) {
    if (upload_samples && s.wave_need[wv] > uploaded) {
      // contiguous runs of global gathers -> one copy each
      int l = uploaded;
      const int need = s.wave_need[wv];
      while (l < need) {
        int e = l + 1;
        while (e < need && s.local_gathers[e] == s.local_gathers[e - 1] + 1) ++e;
        VG_CUDA(cudaMemcpyAsync(
            D.bufs[B_SAMPLES].as<float>() + static_cast<size_t>(l) * trace_floats,
            ds->samples + static_cast<size_t>(s.local_gathers[l]) * trace_floats,
            sizeof(float) * trace_floats * (e - l), cudaMemcpyHostToDevice,
            D.copy_stream));
        l = e;
      }
      uploaded = need;
      VG_CUDA(cudaEventRecord(D.ev(2 * nwaves + wv), D.copy_stream));
      VG_CUDA(cudaStreamWaitEvent(st, D.ev(2 * nwaves + wv), 0));
    }
    if (fast && !(s.wave_lo[wv] >= tab_lo && s.wave_hi[wv] <= tab_hi)) {
      // window-energy tables of this wave's gathers (part of the scan)
      tab_lo = s.wave_lo[wv];
      tab_hi = s.wave_hi[wv];
      const long long ntr = static_cast<long long>(tab_hi - tab_lo) * h.M;
      dim3 eg(static_cast<unsigned>(ntr), (h.ns + 255) / 256);
      const size_t tsm = (256 + std::max(h.w, 2) + 1) * sizeof(float);
      if (kc.quad)
        pair_energy_kernel<true><<<eg, 256, tsm, st>>>(
            d_samples + static_cast<size_t>(tab_lo) * trace_floats, d_tab, d_ec, ntr, h.ns,
            h.w);
      else
        pair_energy_kernel<false><<<eg, 256, tsm, st>>>(
            d_samples + static_cast<size_t>(tab_lo) * trace_floats, d_tab, d_ec, ntr, h.ns,
            h.w);
      VG_CUDA(cudaGetLastError());
      p.table_trace0 = static_cast<long long>(tab_lo) * h.M;
      ++out.launches;
    }
    const int rb = s.wave_rows[wv], re = s.wave_rows[wv + 1];
    p.row_first = rb;
    p.n_rows = re - rb;
    float* panel = nullptr;
    if (d_mat_user) {
      p.matrix = d_mat_user;
      p.mat_row0 = 0;
      panel = d_mat_user + static_cast<size_t>(rb) * panel_row;
    } else if (d_panel[0]) {
      panel = d_panel[wv & 1];
      // the panel's previous contents (wave wv - 2) must have left the device
      if (host_matrix && wv >= 2) VG_CUDA(cudaStreamWaitEvent(st, D.ev(4 * nwaves + (wv & 1)), 0));
      p.matrix = panel;
      p.mat_row0 = rb;
    } else {
      p.matrix = nullptr;
      p.mat_row0 = 0;
    }
    // persistent CTAs, one per SM, striding over the wave's tiles
    const long long tiles = static_cast<long long>((h.ns + kT0 - 1) / kT0) * (re - rb);
    dim3 grid(static_cast<unsigned>(std::min<long long>(tiles, D.n_sm)));
    VG_CUDA(cudaEventRecord(D.ev(2 * wv), st));
    kc.fn<<<grid, kThreads, smem, st>>>(p);
    VG_CUDA(cudaGetLastError());
    VG_CUDA(cudaEventRecord(D.ev(2 * wv + 1), st));
    ++out.launches;
    const size_t wcells = static_cast<size_t>(re - rb) * row_cells;
    if (K > 0) {
      const long long nc = static_cast<long long>(wcells);
      topk_kernel<<<static_cast<unsigned>((nc + 7) / 8), 256, 0, st>>>(
          panel, nc, h.ncand, K, d_tks + static_cast<size_t>(rb) * row_cells * K,
          d_tki + static_cast<size_t>(rb) * row_cells * K);
      VG_CUDA(cudaGetLastError());
      ++out.launches;
    }
    if (host_matrix) {
      VG_CUDA(cudaEventRecord(D.ev(3 * nwaves + wv), st));
      VG_CUDA(cudaStreamWaitEvent(D.d2h_stream, D.ev(3 * nwaves + wv), 0));
      VG_CUDA(cudaMemcpyAsync(
          res->matrix + (static_cast<size_t>(s.r0) + rb) * panel_row, panel,
          wcells * h.ncand * 4, cudaMemcpyDeviceToHost, D.d2h_stream));
      VG_CUDA(cudaEventRecord(D.ev(4 * nwaves + (wv & 1)), D.d2h_stream));
    }
  }
  unsigned long long valid = 0;
  VG_CUDA(cudaMemcpyAsync(&valid, D.bufs[B_VALID].p, 8, cudaMemcpyDeviceToHost,
                          st));
  if (out_host) {
    VG_CUDA(cudaMemcpyAsync(res->best_idx + static_cast<size_t>(s.r0) * h.ns,
                            d_bidx, cells * 4, cudaMemcpyDeviceToHost, st));
    VG_CUDA(cudaMemcpyAsync(res->best_semblance + static_cast<size_t>(s.r0) * h.ns,
                            d_bs, cells * 4, cudaMemcpyDeviceToHost, st));
    VG_CUDA(cudaMemcpyAsync(res->best_stack + static_cast<size_t>(s.r0) * h.ns,
                            d_bst, cells * 4, cudaMemcpyDeviceToHost, st));
    if (K > 0) {
      VG_CUDA(cudaMemcpyAsync(res->topk_idx + static_cast<size_t>(s.r0) * h.ns * K, d_tki,
                              cells * K * 4, cudaMemcpyDeviceToHost, st));
      VG_CUDA(cudaMemcpyAsync(res->topk_semblance + static_cast<size_t>(s.r0) * h.ns * K,
                              d_tks, cells * K * 4, cudaMemcpyDeviceToHost, st));
    }
  }
  if (host_matrix) VG_CUDA(cudaStreamSynchronize(D.d2h_stream));
  VG_CUDA(cudaStreamSynchronize(st));
  out.valid = valid;
  for (int wv = 0; wv < nwaves; ++wv) {
    float ms = 0.0f;
    VG_CUDA(cudaEventElapsedTime(&ms, D.ev(2 * wv), D.ev(2 * wv + 1)));
    out.kernel_ms += ms;
  }
  return out;
}

// Balanced contiguous row blocks by nominal work.
std::vector<int> split_rows(const HostSweep& h, int parts) {
  std::vector<int> cuts(1, 0);
  long long total = 0;
  for (int r = 0; r < h.rows; ++r) total += h.row_traces[r];
  long long acc = 0;
  int r = 0;
  for (int p = 1; p < parts; ++p) {
    const long long target = total * p / parts;
    while (r < h.rows && acc + h.row_traces[r] <= target) acc += h.row_traces[r++];
    cuts.push_back(r);
  }
  cuts.push_back(h.rows);
  return cuts;
}

}  // namespace
}  // namespace velan_gpu

// ===========================================================================
// C ABI

using namespace velan_gpu;

struct velan_gpu_ctx {
  std::vector<DeviceState> devs;
  std::mutex lock;
};

struct velan_gpu_plan {
  velan_gpu_ctx* ctx = nullptr;
  DeviceState dev;
  HostSweep h;
  Shard shard;
  velan_gpu_dataset ds{};
  velan_gpu_scan sc{};
  const float* d_samples_ext = nullptr;
  int launches = 0;
};

// the thread's last-error message, shared with ssf_io.cpp
namespace velan_gpu {
void set_last_error(const std::string& msg) { g_last_error = msg; }
}  // namespace velan_gpu

#define VG_API_BEGIN try {
#define VG_API_END                                    \
  }                                                   \
  catch (const ApiError& e) {                         \
    g_last_error = e.what();                          \
    return e.code;                                    \
  }                                                   \
  catch (const std::exception& e) {                   \
    g_last_error = e.what();                          \
    return VELAN_GPU_ERUNTIME;                        \
  }                                                   \
  catch (...) {                                       \
    g_last_error = "unknown error";                   \
    return VELAN_GPU_ERUNTIME;                        \
  }

extern "C" {

int velan_gpu_abi_version(void) { return VELAN_GPU_ABI_VERSION; }

const char* velan_gpu_last_error(void) { return g_last_error.c_str(); }

int velan_gpu_abi_layout(int32_t* out8) {
  if (!out8) return VELAN_GPU_EPARAM;
  out8[0] = sizeof(velan_gpu_dataset);
  out8[1] = offsetof(velan_gpu_dataset, samples_device);
  out8[2] = sizeof(velan_gpu_scan);
  out8[3] = offsetof(velan_gpu_scan, row_count);
  out8[4] = sizeof(velan_gpu_result);
  out8[5] = offsetof(velan_gpu_result, topk_semblance);
  out8[6] = sizeof(velan_gpu_synth);
  out8[7] = offsetof(velan_gpu_synth, n_threads);
  return VELAN_GPU_OK;
}

int velan_gpu_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  int ok = 0;
  for (int d = 0; d < n; ++d) {
    cudaDeviceProp prop;
    if (cudaGetDeviceProperties(&prop, d) == cudaSuccess && prop.major == 10 &&
        prop.minor == 0)
      ++ok;
  }
  return ok;
}

int velan_gpu_create(const int32_t* device_ids, int32_t n_devices,
                     velan_gpu_ctx** out) {
  VG_API_BEGIN
  if (!out) throw ApiError(VELAN_GPU_EPARAM, "out is null");
  *out = nullptr;
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess || n == 0) {
    cudaGetLastError();
    throw ApiError(VELAN_GPU_ENODEV, "no CUDA device visible");
  }
  if (n_devices < 1) throw ApiError(VELAN_GPU_EPARAM, "n_devices must be >= 1");
  auto ctx = std::make_unique<velan_gpu_ctx>();
  ctx->devs.resize(n_devices);
  for (int i = 0; i < n_devices; ++i) {
    const int d = device_ids ? device_ids[i] : i;
    if (d < 0 || d >= n)
      throw ApiError(VELAN_GPU_ENODEV, fmt("device %lld not visible", d));
    cudaDeviceProp prop;
    VG_CUDA(cudaGetDeviceProperties(&prop, d));
    if (prop.major != 10 || prop.minor != 0)
      throw ApiError(VELAN_GPU_ENODEV,
                     fmt("device %lld is sm_%lld; kernels are built for "
                         "sm_100a only",
                         d, prop.major * 10 + prop.minor));
    ctx->devs[i].init(d);
  }
  *out = ctx.release();
  return VELAN_GPU_OK;
  VG_API_END
}

void velan_gpu_destroy(velan_gpu_ctx* ctx) {
  if (!ctx) return;
  for (auto& d : ctx->devs) d.destroy();
  delete ctx;
}

int velan_gpu_validate(const velan_gpu_dataset* ds, const velan_gpu_scan* sc) {
  VG_API_BEGIN
  validate(ds, sc, sc && sc->op != VELAN_OP_NMO);
  return VELAN_GPU_OK;
  VG_API_END
}

int velan_gpu_describe(const velan_gpu_dataset* ds, const velan_gpu_scan* sc,
                       int32_t* row_gather, int32_t* sweep_traces,
                       int32_t* leg_off, int32_t* leg_gather,
                       int64_t leg_capacity, int64_t* n_legs,
                       uint64_t* nominal) {
  VG_API_BEGIN
  validate(ds, sc, sc && sc->op != VELAN_OP_NMO);
  if (ds->n_gathers == 0) {
    if (n_legs) *n_legs = 0;
    if (nominal) *nominal = 0;
    if (leg_off) leg_off[0] = 0;
    return VELAN_GPU_OK;
  }
  const HostSweep h = build_sweep(ds, sc);
  uint64_t nom = 0;
  for (int r = 0; r < h.rows; ++r) {
    if (row_gather) row_gather[r] = h.row_gather[r];
    if (sweep_traces) sweep_traces[r] = static_cast<int32_t>(h.row_traces[r]);
    nom += static_cast<uint64_t>(h.row_traces[r]) * h.ns * h.ncand;
  }
  const int64_t nl = static_cast<int64_t>(h.leg_gather.size());
  if (n_legs) *n_legs = nl;
  if (nominal) *nominal = nom;
  if (leg_off)
    for (int r = 0; r <= h.rows; ++r) leg_off[r] = h.leg_off[r];
  if (leg_gather && leg_capacity >= nl)
    for (int64_t i = 0; i < nl; ++i) leg_gather[i] = h.leg_gather[i];
  return VELAN_GPU_OK;
  VG_API_END
}

static int run_oneshot(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                       const velan_gpu_scan* sc, velan_gpu_result* res,
                       bool crs) {
  VG_API_BEGIN
  const auto t_start = std::chrono::steady_clock::now();
  if (!ctx || !res) throw ApiError(VELAN_GPU_EPARAM, "null context or result");
  validate(ds, sc, crs);
  res->valid_intersections = 0;
  res->nominal_intersections = 0;
  res->kernel_ms = 0.0;
  if (ds->n_gathers == 0) {
    res->total_ms = 0.0;
    return VELAN_GPU_OK;
  }
  if (!res->best_idx || !res->best_semblance || !res->best_stack)
    throw ApiError(VELAN_GPU_EPARAM, "result arrays are null");
  check_topk(res);
  if (ds->samples_mem == VELAN_MEM_DEVICE && ctx->devs.size() != 1)
    throw ApiError(VELAN_GPU_ECONFIG,
                   "device-resident samples need a single-device context");
  if (res->out_mem == VELAN_MEM_DEVICE && ctx->devs.size() != 1)
    throw ApiError(VELAN_GPU_ECONFIG,
                   "device-resident outputs need a single-device context");
  check_device_samples(ds, ctx->devs[0].dev);
  std::lock_guard<std::mutex> guard(ctx->lock);
  const HostSweep h = build_sweep(ds, sc);
  const int nd = static_cast<int>(ctx->devs.size());
  const std::vector<int> cuts = split_rows(h, nd);
  std::vector<RunOut> outs(nd);
  std::vector<std::string> errs(nd);
  std::vector<int> codes(nd, 0);
  const bool dev_samples = ds->samples_mem == VELAN_MEM_DEVICE;
  // a semblance panel that is not the caller's device matrix is per wave:
  // cap a wave's rows so one panel stays within kPanelBytes
  long long wave_cap = 65535;
  const bool internal_panel =
      res->topk > 0 || (res->matrix && res->out_mem == VELAN_MEM_HOST);
  if (internal_panel)
    wave_cap = std::max<long long>(
        1, static_cast<long long>(kPanelBytes / (static_cast<size_t>(h.ns) * h.ncand * 4)));
  auto body = [&](int i) {
    try {
      const Shard s = make_shard(h, ds, cuts[i], cuts[i + 1], dev_samples, wave_cap);
      outs[i] = run_shard(ctx->devs[i], h, s, ds, sc, res,
                          dev_samples ? ds->samples : nullptr, nullptr, false,
                          false);
    } catch (const ApiError& e) {
      codes[i] = e.code;
      errs[i] = e.what();
    } catch (const std::exception& e) {
      codes[i] = VELAN_GPU_ERUNTIME;
      errs[i] = e.what();
    }
  };
  if (nd == 1) {
    body(0);
  } else {
    std::vector<std::thread> th;
    for (int i = 0; i < nd; ++i) th.emplace_back(body, i);
    for (auto& t : th) t.join();
  }
  for (int i = 0; i < nd; ++i)
    if (codes[i]) throw ApiError(codes[i], errs[i]);
  uint64_t valid = 0;
  double kms = 0.0;
  for (auto& o : outs) {
    valid += o.valid;
    kms = std::max(kms, o.kernel_ms);
  }
  uint64_t nominal = 0;
  for (int r = 0; r < h.rows; ++r)
    nominal += static_cast<uint64_t>(h.row_traces[r]) * h.ns * h.ncand;
  if (res->row_gather)
    for (int r = 0; r < h.rows; ++r) res->row_gather[r] = h.row_gather[r];
  res->valid_intersections = valid;
  res->nominal_intersections = nominal;
  res->kernel_ms = kms;
  res->total_ms = std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now() - t_start)
                      .count();
  return VELAN_GPU_OK;
  VG_API_END
}

int velan_gpu_cmp(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                  const velan_gpu_scan* sc, velan_gpu_result* res) {
  return run_oneshot(ctx, ds, sc, res, false);
}

int velan_gpu_crs(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                  const velan_gpu_scan* sc, velan_gpu_result* res) {
  return run_oneshot(ctx, ds, sc, res, true);
}

int velan_gpu_plan_create(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                          const velan_gpu_scan* sc, velan_gpu_plan** out) {
  VG_API_BEGIN
  if (!ctx || !out) throw ApiError(VELAN_GPU_EPARAM, "null context or out");
  *out = nullptr;
  validate(ds, sc, sc && sc->op != VELAN_OP_NMO);
  if (ctx->devs.size() != 1)
    throw ApiError(VELAN_GPU_ECONFIG, "plans need a single-device context");
  check_device_samples(ds, ctx->devs[0].dev);
  auto plan = std::make_unique<velan_gpu_plan>();
  plan->ctx = ctx;
  plan->ds = *ds;
  plan->sc = *sc;
  plan->dev.init(ctx->devs[0].dev);
  plan->h = build_sweep(ds, sc);
  const bool dev_samples = ds->samples_mem == VELAN_MEM_DEVICE;
  plan->shard = make_shard(plan->h, ds, 0, plan->h.rows, dev_samples);
  plan->d_samples_ext = dev_samples ? ds->samples : nullptr;
  if (ds->n_gathers > 0) {
    // resident tables + samples: one upload now, none per execute
    DeviceState& D = plan->dev;
    const Shard& s = plan->shard;
    const HostSweep& h = plan->h;
    upload(D.bufs[B_H2], s.h2, D.stream);
    upload(D.bufs[B_NTR], s.ntr, D.stream);
    upload(D.bufs[B_LEGOFF], s.leg_off, D.stream);
    upload(D.bufs[B_LEGG], s.leg_gather, D.stream);
    upload(D.bufs[B_LEGD2], s.leg_d2, D.stream);
    upload(D.bufs[B_LEGDM], s.leg_dm, D.stream);
    upload(D.bufs[B_T0], h.t0, D.stream);
    upload(D.bufs[B_A], h.a, D.stream);
    upload(D.bufs[B_B], h.b, D.stream);
    upload(D.bufs[B_V], h.v, D.stream);
    if (!dev_samples) {
      const size_t tf = static_cast<size_t>(h.M) * h.ns;
      const size_t L = s.local_gathers.size();
      D.bufs[B_SAMPLES].ensure(L * tf * 4 + 64);
      for (size_t l = 0; l < L; ++l)
        VG_CUDA(cudaMemcpyAsync(D.bufs[B_SAMPLES].as<float>() + l * tf,
                                ds->samples + static_cast<size_t>(s.local_gathers[l]) * tf,
                                tf * 4, cudaMemcpyHostToDevice, D.stream));
    }
    VG_CUDA(cudaStreamSynchronize(D.stream));
  }
  plan->ds.samples = nullptr;  // host pointers are not retained
  plan->ds.coords = nullptr;
  plan->ds.ntraces = nullptr;
  plan->ds.cdp_id = nullptr;
  plan->sc.a = plan->sc.b = plan->sc.v = nullptr;
  *out = plan.release();
  return VELAN_GPU_OK;
  VG_API_END
}

int velan_gpu_plan_execute(velan_gpu_plan* plan, velan_gpu_result* res,
                           void* stream) {
  VG_API_BEGIN
  const auto t_start = std::chrono::steady_clock::now();
  if (!plan || !res) throw ApiError(VELAN_GPU_EPARAM, "null plan or result");
  res->valid_intersections = 0;
  res->nominal_intersections = 0;
  res->kernel_ms = 0.0;
  if (plan->h.rows == 0) return VELAN_GPU_OK;
  if (!res->best_idx || !res->best_semblance || !res->best_stack)
    throw ApiError(VELAN_GPU_EPARAM, "result arrays are null");
  check_topk(res);
  const RunOut o =
      run_shard(plan->dev, plan->h, plan->shard, &plan->ds, &plan->sc, res,
                plan->d_samples_ext, static_cast<cudaStream_t>(stream), true,
                plan->d_samples_ext == nullptr);
  plan->launches = o.launches;
  if (res->row_gather)
    for (int r = 0; r < plan->h.rows; ++r) res->row_gather[r] = plan->h.row_gather[r];
  res->valid_intersections = o.valid;
  res->nominal_intersections = static_cast<uint64_t>(plan->shard.nominal);
  res->kernel_ms = o.kernel_ms;
  res->total_ms = std::chrono::duration<double, std::milli>(
                      std::chrono::steady_clock::now() - t_start)
                      .count();
  return VELAN_GPU_OK;
  VG_API_END
}

int velan_gpu_plan_launches(const velan_gpu_plan* plan) {
  if (!plan) return 0;
  // the last execute's kernel launches (scan waves + FAST table passes +
  // top-k); before any execute, the scan waves alone
  if (plan->launches > 0) return plan->launches;
  return static_cast<int>(plan->shard.wave_need.size());
}

void velan_gpu_plan_destroy(velan_gpu_plan* plan) {
  if (!plan) return;
  plan->dev.destroy();
  delete plan;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// hit_for test hook

namespace velan_gpu {
namespace {
__global__ void hit_batch_kernel(const float* t, int n, double dt, int ns,
                                 int w, int variant, float inv_hi,
                                 float inv_lo, float amb_eps, int32_t* k1,
                                 float* x, uint8_t* valid) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  int kk;
  float xx;
  bool vv;
  if (variant == VELAN_VARIANT_EXACT) {
    hit_exact(t[i], dt, ns, w, kk, xx, vv);
  } else {
    ScanParams p{};
    p.dt = dt;
    p.ns = ns;
    p.inv_hi = inv_hi;
    p.inv_lo = inv_lo;
    p.amb_eps = amb_eps;
    hit_fast(t[i], p, w, kk, xx, vv);
  }
  // the reference reports k1 even for invalid hits; recompute it exactly
  const double base = floor(__ddiv_rn(static_cast<double>(t[i]), dt));
  const bool in_range = base >= -2147483648.0 && base < 2147483648.0;
  k1[i] = in_range ? static_cast<int>(base) - (w >> 1)
                   : static_cast<int>(0x80000000u) - (w >> 1);
  if (vv) k1[i] = kk;
  x[i] = xx;
  valid[i] = vv ? 1 : 0;
}
}  // namespace
}  // namespace velan_gpu

namespace velan_gpu {
namespace {
// One block per (row, trace), threads over the output samples: the trace is
// read once into shared memory, every output sample interpolates it at the
// pick's traveltime with the reference's rounding (crs_traveltime, hit_for,
// interpolate — no contraction).
__global__ void __launch_bounds__(256)
    nmo_correct_kernel(const float* __restrict__ samples, const float* __restrict__ h2,
                       const int* __restrict__ ntr, const int* __restrict__ row_gather,
                       const int32_t* __restrict__ picks, const float* __restrict__ t0,
                       const float* __restrict__ v, int n_c, int Mmax, int ns, double dt,
                       float* __restrict__ out) {
  extern __shared__ float tr[];
  const int r = blockIdx.y, m = blockIdx.x;
  const int g = row_gather[r];
  float* o = out + (static_cast<size_t>(r) * Mmax + m) * ns;
  if (m >= ntr[g]) {
    for (int k = threadIdx.x; k < ns; k += blockDim.x) o[k] = 0.0f;
    return;
  }
  const float* a = samples + (static_cast<size_t>(g) * Mmax + m) * ns;
  for (int k = threadIdx.x; k < ns; k += blockDim.x) tr[k] = a[k];
  __syncthreads();
  const float hh = h2[static_cast<size_t>(g) * Mmax + m];
  for (int k = threadIdx.x; k < ns; k += blockDim.x) {
    const int c = picks[static_cast<size_t>(r) * ns + k];
    const float vv = v[((c % n_c) + n_c) % n_c];
    const float t = tt_q(__fmul_rn(t0[k], t0[k]), moveout_q(hh, 0.0f, vv));
    int k1;
    float x;
    bool valid;
    hit_exact(t, dt, ns, 1, k1, x, valid);
    o[k] = valid ? __fadd_rn(__fmul_rn(__fsub_rn(tr[k1 + 1], tr[k1]), x), tr[k1]) : 0.0f;
  }
}
}  // namespace
}  // namespace velan_gpu

extern "C" int velan_gpu_nmo_correct(velan_gpu_ctx* ctx, const velan_gpu_dataset* ds,
                                     const velan_gpu_scan* sc, const int32_t* picks,
                                     float* out) {
  VG_API_BEGIN
  if (!ctx) throw ApiError(VELAN_GPU_EPARAM, "null context");
  validate(ds, sc, sc && sc->op != VELAN_OP_NMO);
  if (ds->n_gathers == 0) return VELAN_GPU_OK;
  if (!picks || !out) throw ApiError(VELAN_GPU_EPARAM, "picks or out is null");
  if (ds->samples_mem != VELAN_MEM_HOST)
    throw ApiError(VELAN_GPU_EPARAM, "velan_gpu_nmo_correct: samples must be host memory");
  const HostSweep h = build_sweep(ds, sc);
  if (h.rows == 0) return VELAN_GPU_OK;
  for (size_t i = 0; i < static_cast<size_t>(h.rows) * h.ns; ++i)
    if (picks[i] < 0 || picks[i] >= h.ncand)
      throw ApiError(VELAN_GPU_EPARAM, "pick index outside the candidate grid");
  std::lock_guard<std::mutex> guard(ctx->lock);
  DeviceState& D = ctx->devs[0];
  VG_CUDA(cudaSetDevice(D.dev));
  cudaStream_t st = D.stream;
  const size_t tf = static_cast<size_t>(h.M) * h.ns;
  std::vector<int> ntr(ds->ntraces, ds->ntraces + h.G);
  D.bufs[B_SAMPLES].ensure(static_cast<size_t>(h.G) * tf * 4 + 64);
  VG_CUDA(cudaMemcpyAsync(D.bufs[B_SAMPLES].p, ds->samples, static_cast<size_t>(h.G) * tf * 4,
                          cudaMemcpyHostToDevice, st));
  upload(D.bufs[B_H2], h.h2, st);
  upload(D.bufs[B_NTR], ntr, st);
  upload(D.bufs[B_LEGG], h.row_gather, st);
  upload(D.bufs[B_T0], h.t0, st);
  upload(D.bufs[B_V], h.v, st);
  const size_t cells = static_cast<size_t>(h.rows) * h.ns;
  D.bufs[B_BIDX].ensure(cells * 4);
  VG_CUDA(cudaMemcpyAsync(D.bufs[B_BIDX].p, picks, cells * 4, cudaMemcpyHostToDevice, st));
  D.bufs[B_MAT].ensure(static_cast<size_t>(h.rows) * tf * 4);
  dim3 grid(static_cast<unsigned>(h.M), static_cast<unsigned>(h.rows));
  nmo_correct_kernel<<<grid, 256, h.ns * sizeof(float), st>>>(
      D.bufs[B_SAMPLES].as<float>(), D.bufs[B_H2].as<float>(), D.bufs[B_NTR].as<int>(),
      D.bufs[B_LEGG].as<int>(), D.bufs[B_BIDX].as<int32_t>(), D.bufs[B_T0].as<float>(),
      D.bufs[B_V].as<float>(), h.n_c, h.M, h.ns, h.dt, D.bufs[B_MAT].as<float>());
  VG_CUDA(cudaGetLastError());
  VG_CUDA(cudaMemcpyAsync(out, D.bufs[B_MAT].p, static_cast<size_t>(h.rows) * tf * 4,
                          cudaMemcpyDeviceToHost, st));
  VG_CUDA(cudaStreamSynchronize(st));
  return VELAN_GPU_OK;
  VG_API_END
}

extern "C" int velan_gpu_hit_batch(const float* t, int32_t n, double dt_s,
                                   int32_t ns, int32_t w, int32_t variant,
                                   int32_t* k1, float* x, uint8_t* valid) {
  VG_API_BEGIN
  if (n < 0 || (n > 0 && (!t || !k1 || !x || !valid)))
    throw ApiError(VELAN_GPU_EPARAM, "bad arguments");
  if (velan_gpu_device_count() == 0)
    throw ApiError(VELAN_GPU_ENODEV, "no sm_100 device visible");
  if (n == 0) return VELAN_GPU_OK;
  float* dt_ = nullptr;
  int32_t* dk = nullptr;
  float* dx = nullptr;
  uint8_t* dv = nullptr;
  VG_CUDA(cudaMalloc(&dt_, n * 4));
  VG_CUDA(cudaMalloc(&dk, n * 4));
  VG_CUDA(cudaMalloc(&dx, n * 4));
  VG_CUDA(cudaMalloc(&dv, n));
  VG_CUDA(cudaMemcpy(dt_, t, n * 4, cudaMemcpyHostToDevice));
  const double inv = 1.0 / dt_s;
  const float hi = static_cast<float>(inv);
  const float lo = static_cast<float>(inv - hi);
  const float eps = static_cast<float>(std::ldexp(std::max(ns, 16), -40));
  hit_batch_kernel<<<(n + 255) / 256, 256>>>(dt_, n, dt_s, ns, w, variant, hi,
                                             lo, eps, dk, dx, dv);
  VG_CUDA(cudaGetLastError());
  VG_CUDA(cudaMemcpy(k1, dk, n * 4, cudaMemcpyDeviceToHost));
  VG_CUDA(cudaMemcpy(x, dx, n * 4, cudaMemcpyDeviceToHost));
  VG_CUDA(cudaMemcpy(valid, dv, n, cudaMemcpyDeviceToHost));
  cudaFree(dt_);
  cudaFree(dk);
  cudaFree(dx);
  cudaFree(dv);
  return VELAN_GPU_OK;
  VG_API_END
}
