// velan_gpu/adapter.hpp — the drop-in: the reference's pipeline signatures,
// executed by the B200 kernels behind include/velan_gpu.h.
//
// A user of the reference library (velan, /root/reference/proj/include)
// replaces
//     velan::run_cmp(ds, cfg, workers, &stats)            cmp_pipeline.hpp:94
//     velan::run_crs(ds, cfg, dims, apm, opts, &info, &st) crs_pipeline.hpp:283
//     velan::scan_cdp(gather, cfg)                        cmp_pipeline.hpp:24
//     velan::scan_central_cdp(central, nbrs, cfg)         crs_pipeline.hpp:193
// by the same calls in namespace velan_gpu, linking libvelan_gpu.so.  Inputs
// are the reference's own types (Dataset, ScanConfig, ...); outputs are
// std::vector<velan::SemblanceMatrix> with values, best_velocity and
// stack_trace filled exactly like scan_sweep fills them.  With the default
// EXACT variant the matrices are bitwise identical to the reference's
// blocked kernel.  `workers` selects the number of GPUs (devices 0..n-1).
// Errors are rethrown as the reference's exception types (error.hpp).
//
// The CPU tuning knobs of ScanConfig (tile_size, lane_width, size_h,
// scratch_budget, range_cap, kernel_variant) do not apply to the GPU path
// and are ignored, after ScanConfig::validate() has checked them as the
// reference does.  CacheStats::naive_fetches is filled (the valid
// curve-trace intersections, bench.hpp:126); the CPU cache's other
// counters have no GPU equivalent and stay 0.
#pragma once

#include <cstdint>
#include <cstring>
#include <memory>
#include <mutex>
#include <span>
#include <string>
#include <vector>

#include "velan/cmp_pipeline.hpp"
#include "velan/crs_pipeline.hpp"
#include "velan/error.hpp"
#include "velan/scan.hpp"
#include "velan/types.hpp"
#include "velan_gpu.h"

namespace velan_gpu {

enum class Variant { exact = VELAN_VARIANT_EXACT, fast = VELAN_VARIANT_FAST };

// GPU-side options of a drop-in call.  A Variant converts implicitly, so
// run_cmp(ds, cfg, n, &stats, Variant::fast) keeps working.  values = false
// leaves SemblanceMatrix::values empty (picks and stack only, as an SMB1 file
// without matrices, io.hpp:170-194): the full ns x nc matrix is then never
// allocated, on the device or the host (CMP large: 26 GB).
struct Options {
  Variant variant = Variant::exact;
  bool values = true;
  Options() = default;
  Options(Variant v) : variant(v) {}  // NOLINT: implicit on purpose
  Options(Variant v, bool with_values) : variant(v), values(with_values) {}
};

// BASELINE's three-parameter CRS search (no reference implementation):
// candidates A [s/m] x B [s/m^2] x C, the C axis scanned as a velocity
// (C = 2 / (t0 v^2)); flat index (ia * nB + ib) * nC + ic.
struct AbcGrid {
  std::vector<float> a, b, v;
  int ncand() const { return static_cast<int>(a.size() * b.size() * v.size()); }
};

// BestPick for the ABC operator: the index triple of the pick (SURVEY.md
// §8b: BestPick carries one velocity, scan.hpp:81-103).
struct AbcPick {
  int32_t ia = 0, ib = 0, ic = 0;
  float semblance = 0.0f;
};

// SemblanceMatrix for the ABC operator: values [ns][ncand] sample-major
// (empty unless requested), the pick triple and the stack at the pick.
struct AbcMatrix {
  std::uint32_t cdp_id = 0;
  int ns = 0, nc = 0;
  std::vector<float> values;
  std::vector<AbcPick> best;
  std::vector<float> stack_trace;
};

namespace detail {

[[noreturn]] inline void rethrow(int code, const char* where) {
  const std::string msg = std::string(where) + ": " + velan_gpu_last_error();
  switch (code) {
    case VELAN_GPU_ECONFIG: throw velan::config_error(msg);
    case VELAN_GPU_EPARAM: throw velan::parameter_error(msg);
    default: throw velan::error(msg);
  }
}

// One context per device count, created on first use.
inline velan_gpu_ctx* context(int devices) {
  static std::mutex m;
  static std::vector<std::unique_ptr<velan_gpu_ctx, void (*)(velan_gpu_ctx*)>> ctx;
  std::lock_guard<std::mutex> g(m);
  if (devices < 1) throw velan::parameter_error("worker count must be >= 1");
  const int avail = velan_gpu_device_count();
  if (avail == 0) throw velan::error("velan_gpu: no sm_100 device visible");
  if (devices > avail) devices = avail;
  while (static_cast<int>(ctx.size()) < devices)
    ctx.emplace_back(nullptr, &velan_gpu_destroy);
  auto& slot = ctx[devices - 1];
  if (!slot) {
    velan_gpu_ctx* c = nullptr;
    const int code = velan_gpu_create(nullptr, devices, &c);
    if (code) rethrow(code, "velan_gpu_create");
    slot.reset(c);
  }
  return slot.get();
}

// Dataset (types.hpp:46-54) -> flat arrays of the C-ABI.
struct Flat {
  std::vector<float> samples, coords;
  std::vector<int32_t> ntraces;
  std::vector<uint32_t> cdp_id;
  velan_gpu_dataset ds{};
};

inline Flat flatten(std::span<const velan::CdpGather* const> gathers) {
  Flat f;
  const int G = static_cast<int>(gathers.size());
  int M = 1, ns = 0;
  uint32_t dt = 0;
  for (const velan::CdpGather* g : gathers) {
    M = std::max<int>(M, static_cast<int>(g->traces.size()));
    if (ns == 0 && g->ns) {
      ns = static_cast<int>(g->ns);
      dt = g->dt_us;
    }
    if (g->ns != 0 && static_cast<int>(g->ns) != ns)
      throw velan::parameter_error("TraceSweep: neighbor ns differs from central");
  }
  f.samples.assign(static_cast<size_t>(G) * M * ns, 0.0f);
  f.coords.assign(static_cast<size_t>(G) * M * 4, 0.0f);
  f.ntraces.resize(G);
  f.cdp_id.resize(G);
  for (int i = 0; i < G; ++i) {
    const velan::CdpGather& g = *gathers[i];
    f.ntraces[i] = static_cast<int32_t>(g.traces.size());
    f.cdp_id[i] = g.cdp_id;
    for (size_t m = 0; m < g.traces.size(); ++m) {
      const velan::Trace& t = g.traces[m];
      float* c4 = &f.coords[(static_cast<size_t>(i) * M + m) * 4];
      c4[0] = t.sx;
      c4[1] = t.sy;
      c4[2] = t.gx;
      c4[3] = t.gy;
      if (static_cast<int>(t.samples.size()) != ns)
        throw velan::parameter_error("trace sample count differs from ns");
      std::memcpy(&f.samples[(static_cast<size_t>(i) * M + m) * ns],
                  t.samples.data(), sizeof(float) * ns);
    }
  }
  f.ds.n_gathers = G;
  f.ds.max_traces = M;
  f.ds.ns = ns;
  f.ds.dt_us = dt;
  f.ds.cdp_id = f.cdp_id.data();
  f.ds.ntraces = f.ntraces.data();
  f.ds.coords = f.coords.data();
  f.ds.samples = f.samples.data();
  f.ds.samples_mem = VELAN_MEM_HOST;
  return f;
}

inline std::vector<const velan::CdpGather*> pointers(const velan::Dataset& ds) {
  std::vector<const velan::CdpGather*> p;
  p.reserve(ds.gathers.size());
  for (const auto& g : ds.gathers) p.push_back(&g);
  return p;
}

// Run one scan and repackage as SemblanceMatrix (scan.hpp:89-103, filled as
// scan_sweep fills it: values sample-major, best_velocity = grid value of
// the pick, stack_trace = stack at the pick).
inline std::vector<velan::SemblanceMatrix> run(
    std::span<const velan::CdpGather* const> gathers,
    const velan::ScanConfig& cfg, int op, double apm, int devices,
    Options opts, velan::CacheStats* stats, int32_t row_first = 0,
    int32_t row_count = 0) {
  cfg.validate();  // config_error before any compute (scan.hpp:61-78)
  if (gathers.empty()) return {};
  Flat f = flatten(gathers);
  const velan::VelocityGrid grid = cfg.grid();
  std::vector<float> v(cfg.nc);
  for (int c = 0; c < cfg.nc; ++c) v[c] = grid.value(c);
  velan_gpu_scan sc{};
  sc.op = op;
  sc.variant = static_cast<int32_t>(opts.variant);
  sc.w = cfg.w;
  sc.n_a = sc.n_b = 1;
  sc.n_c = cfg.nc;
  sc.v = v.data();
  sc.apm = apm;
  sc.row_first = row_first;
  sc.row_count = row_count;
  const int G = f.ds.n_gathers, ns = f.ds.ns, nc = cfg.nc;
  const int rows = row_count > 0 ? row_count : G;
  std::vector<int32_t> best(static_cast<size_t>(rows) * ns), order(rows);
  std::vector<float> sem(best.size()), stk(best.size());
  std::vector<float> matrix(opts.values ? static_cast<size_t>(rows) * ns * nc : 0);
  velan_gpu_result res{};
  res.out_mem = VELAN_MEM_HOST;
  res.best_idx = best.data();
  res.best_semblance = sem.data();
  res.best_stack = stk.data();
  res.matrix = opts.values ? matrix.data() : nullptr;
  res.row_gather = order.data();
  velan_gpu_ctx* ctx = context(devices);
  const int code = op == VELAN_OP_NMO ? velan_gpu_cmp(ctx, &f.ds, &sc, &res)
                                      : velan_gpu_crs(ctx, &f.ds, &sc, &res);
  if (code) rethrow(code, op == VELAN_OP_NMO ? "velan_gpu_cmp" : "velan_gpu_crs");
  if (stats) stats->naive_fetches += res.valid_intersections;
  std::vector<velan::SemblanceMatrix> out(rows);
  for (int r = 0; r < rows; ++r) {
    velan::SemblanceMatrix& m = out[r];
    m.cdp_id = f.cdp_id[order[r]];
    m.ns = ns;
    m.nc = nc;
    if (opts.values)
      m.values.assign(matrix.begin() + static_cast<size_t>(r) * ns * nc,
                      matrix.begin() + static_cast<size_t>(r + 1) * ns * nc);
    m.best_velocity.resize(ns);
    m.stack_trace.resize(ns);
    for (int k = 0; k < ns; ++k) {
      const size_t o = static_cast<size_t>(r) * ns + k;
      m.best_velocity[k] = velan::BestPick{grid.value(best[o]), sem[o]};
      m.stack_trace[k] = stk[o];
    }
  }
  return out;
}

}  // namespace detail

// run_cmp (cmp_pipeline.hpp:94-106).  workers = GPUs.
inline std::vector<velan::SemblanceMatrix> run_cmp(
    const velan::Dataset& dataset, const velan::ScanConfig& config,
    int workers, velan::CacheStats* stats_out = nullptr,
    Options options = {}) {
  config.validate();
  if (workers < 1) throw velan::parameter_error("worker count must be >= 1");
  const auto ptrs = detail::pointers(dataset);
  return detail::run(ptrs, config, VELAN_OP_NMO, 0.0, workers, options,
                     stats_out);
}

// run_crs (crs_pipeline.hpp:283-460).  The reference's 2-D shard grid is
// validated exactly as partition() does (apm <= half a shard edge,
// crs_pipeline.hpp:92-158) so the same configurations are rejected; the
// GPU then shards the cdp_id-ordered midpoints over workers devices with a
// replicated halo.  Results are in cdp_id order.  CrsRunInfo is left
// empty: there is no halo message protocol on the GPU path.
inline std::vector<velan::SemblanceMatrix> run_crs(
    const velan::Dataset& dataset, const velan::ScanConfig& config,
    velan::GridDims dims, double apm, const velan::CrsOptions& options = {},
    velan::CrsRunInfo* info = nullptr, velan::CacheStats* stats_out = nullptr,
    Options opts = {}) {
  config.validate();
  if (options.workers_per_shard < 1)
    throw velan::parameter_error("run_crs: workers_per_shard must be >= 1");
  if (dataset.gathers.empty()) return {};
  (void)velan::partition(dataset, dims, apm);  // reference validation
  if (info) info->shards.clear();
  const auto ptrs = detail::pointers(dataset);
  return detail::run(ptrs, config, VELAN_OP_CRS_D2, apm,
                     options.workers_per_shard, opts, stats_out);
}

// scan_cdp (cmp_pipeline.hpp:17-27).
inline velan::SemblanceMatrix scan_cdp(const velan::CdpGather& gather,
                                       const velan::ScanConfig& config,
                                       Options options = {}) {
  const velan::CdpGather* p = &gather;
  auto out = detail::run(std::span<const velan::CdpGather* const>(&p, 1),
                         config, VELAN_OP_NMO, 0.0, 1, options, nullptr);
  return std::move(out.front());
}

// scan_central_cdp (crs_pipeline.hpp:184-197): the central sweep extended
// by `neighbors` (passed in cdp_id order, as neighbors_of returns them).
inline velan::SemblanceMatrix scan_central_cdp(
    const velan::CdpGather& central,
    std::span<const velan::CdpGather* const> neighbors,
    const velan::ScanConfig& config, Options options = {}) {
  std::vector<const velan::CdpGather*> all;
  all.push_back(&central);
  double apm = 0.0;
  const velan::Midpoint c = velan::midpoint_of(central);
  for (const velan::CdpGather* g : neighbors) {
    if (g == &central || g->traces.empty()) continue;
    all.push_back(g);
    const velan::Midpoint m = velan::midpoint_of(*g);
    const double dx = m.mx - c.mx, dy = m.my - c.my;
    apm = std::max(apm, dx * dx + dy * dy);
  }
  apm = std::sqrt(apm) * (1.0 + 1e-9) + 1e-9;
  // output row of the central gather: cdp_id order, ties by input index
  int32_t row = 0;
  for (size_t i = 1; i < all.size(); ++i)
    if (all[i]->cdp_id < central.cdp_id) ++row;
  auto out = detail::run(all, config, VELAN_OP_CRS_D2, apm, 1, options,
                         nullptr, row, 1);
  return std::move(out.front());
}

// BASELINE's CRS search with the three-parameter operator
// t^2 = (t0 + 2 A dm)^2 + 2 t0 (B dm^2 + C h^2) over each midpoint's closed
// apm ball (neighbors_of, crs_pipeline.hpp:162-180), results in cdp_id order
// like run_crs.  w is the semblance window (ScanConfig::w); workers = GPUs.
inline std::vector<AbcMatrix> run_crs_abc(const velan::Dataset& dataset,
                                          const AbcGrid& grid, int w, double apm,
                                          int workers = 1,
                                          velan::CacheStats* stats_out = nullptr,
                                          Options opts = {}) {
  if (workers < 1) throw velan::parameter_error("worker count must be >= 1");
  if (w < 1) throw velan::config_error("ScanConfig: w must be >= 1");
  if (grid.a.empty() || grid.b.empty() || grid.v.empty())
    throw velan::config_error("ScanConfig: CRS_ABC needs non-empty A, B and C axes");
  if (dataset.gathers.empty()) return {};
  const auto ptrs = detail::pointers(dataset);
  detail::Flat f = detail::flatten(ptrs);
  velan_gpu_scan sc{};
  sc.op = VELAN_OP_CRS_ABC;
  sc.variant = static_cast<int32_t>(opts.variant);
  sc.w = w;
  sc.n_a = static_cast<int32_t>(grid.a.size());
  sc.n_b = static_cast<int32_t>(grid.b.size());
  sc.n_c = static_cast<int32_t>(grid.v.size());
  sc.a = grid.a.data();
  sc.b = grid.b.data();
  sc.v = grid.v.data();
  sc.apm = apm;
  const int G = f.ds.n_gathers, ns = f.ds.ns, nc = grid.ncand();
  std::vector<int32_t> best(static_cast<size_t>(G) * ns), order(G);
  std::vector<float> sem(best.size()), stk(best.size());
  std::vector<float> matrix(opts.values ? static_cast<size_t>(G) * ns * nc : 0);
  velan_gpu_result res{};
  res.out_mem = VELAN_MEM_HOST;
  res.best_idx = best.data();
  res.best_semblance = sem.data();
  res.best_stack = stk.data();
  res.matrix = opts.values ? matrix.data() : nullptr;
  res.row_gather = order.data();
  const int code = velan_gpu_crs(detail::context(workers), &f.ds, &sc, &res);
  if (code) detail::rethrow(code, "velan_gpu_crs");
  if (stats_out) stats_out->naive_fetches += res.valid_intersections;
  const int nB = sc.n_b, nC = sc.n_c;
  std::vector<AbcMatrix> out(G);
  for (int r = 0; r < G; ++r) {
    AbcMatrix& m = out[r];
    m.cdp_id = f.cdp_id[order[r]];
    m.ns = ns;
    m.nc = nc;
    if (opts.values)
      m.values.assign(matrix.begin() + static_cast<size_t>(r) * ns * nc,
                      matrix.begin() + static_cast<size_t>(r + 1) * ns * nc);
    m.best.resize(ns);
    m.stack_trace.resize(ns);
    for (int k = 0; k < ns; ++k) {
      const size_t o = static_cast<size_t>(r) * ns + k;
      const int flat = best[o];
      m.best[k] = AbcPick{flat / (nB * nC), (flat / nC) % nB, flat % nC, sem[o]};
      m.stack_trace[k] = stk[o];
    }
  }
  return out;
}

}  // namespace velan_gpu
