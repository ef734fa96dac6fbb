// ref_shim.cpp — C entry points onto the UNMODIFIED reference library.
//
// TEST / BASELINE INFRASTRUCTURE ONLY.  Compiled by oracle/Makefile against
// the reference headers where they lie (/root/reference/proj/include, not
// copied), with the reference's own flags (-O3 -ffp-contract=off,
// proj/CMakeLists.txt:15-20), into oracle/_ref/libvelan_ref.so.  It is used
// (a) to pin the C restatement in oracle/semblance_oracle.c, (b) to generate
// tests/golden fixtures, and (c) as the timed CPU baseline ("kind":
// "reference") of bench.py.  Nothing in the product path loads it.
//
// The reference API driven here:
//   velan::run_cmp                       cmp_pipeline.hpp:94-106
//   velan::run_crs                       crs_pipeline.hpp:283-460
//   velan::scan_tile_blocked / scan_pair_baseline / scan_tile_vectorized
//                                        kernel.hpp:244-409
//   velan::TraceSweep, neighbors_of      kernel.hpp:61-113,
//                                        crs_pipeline.hpp:162-180
//   velan::oracle::semblance_reference   oracle.hpp:64-113
//   velan::detail::parallel_for_indexed  cmp_pipeline.hpp:34-88
//   velan::write_dataset / read_dataset / write_picks / read_picks
//                                        io.hpp:95-224
// For an arbitrary candidate list (BASELINE's slowness-linear grid) the
// pairs are built exactly as scan_sweep builds them (scan.hpp:130-136) and
// tiled with ScanConfig::effective_tile_size (scan.hpp:53-59); the per-pair
// results are tile-invariant (test_kernel.cpp:278-309).

#include <algorithm>
#include <atomic>
#include <cstdint>
#include <cstring>
#include <exception>
#include <map>
#include <string>
#include <vector>

#include "velan/cmp_pipeline.hpp"
#include "velan/crs_pipeline.hpp"
#include "velan/io.hpp"
#include "velan/kernel.hpp"
#include "velan/oracle.hpp"
#include "velan/scan.hpp"
#include "velan/traveltime.hpp"

namespace {

thread_local std::string g_err;

velan::Dataset make_dataset(const float* samples, const float* coords,
                            const int32_t* ntraces, const uint32_t* cdp_id,
                            int G, int M, int ns, uint32_t dt_us) {
  velan::Dataset ds;
  ds.fold = static_cast<std::uint32_t>(M);
  ds.gathers.resize(G);
  for (int g = 0; g < G; ++g) {
    velan::CdpGather& cg = ds.gathers[g];
    cg.cdp_id = cdp_id[g];
    cg.ns = static_cast<std::uint32_t>(ns);
    cg.dt_us = dt_us;
    cg.traces.resize(ntraces[g]);
    for (int m = 0; m < ntraces[g]; ++m) {
      velan::Trace& t = cg.traces[m];
      const float* c4 = coords + (static_cast<size_t>(g) * M + m) * 4;
      t.sx = c4[0];
      t.sy = c4[1];
      t.gx = c4[2];
      t.gy = c4[3];
      const float* s = samples + (static_cast<size_t>(g) * M + m) * ns;
      t.samples.assign(s, s + ns);
    }
  }
  return ds;
}

void fill_matrix_out(const velan::SemblanceMatrix& m, int row, int ns, int nc,
                     const std::vector<float>& vgrid, int32_t* best_idx,
                     float* best_s, float* best_stack, float* matrix) {
  for (int k = 0; k < ns; ++k) {
    // recover the index of the picked velocity (values are distinct grid
    // points; the first equal one is the reference's pick under its tie rule)
    int idx = 0;
    for (int c = 0; c < nc; ++c)
      if (vgrid[c] == m.best_velocity[k].velocity) {
        idx = c;
        break;
      }
    best_idx[static_cast<size_t>(row) * ns + k] = idx;
    best_s[static_cast<size_t>(row) * ns + k] = m.best_velocity[k].semblance;
    best_stack[static_cast<size_t>(row) * ns + k] = m.stack_trace[k];
  }
  if (matrix)
    std::memcpy(matrix + static_cast<size_t>(row) * ns * nc, m.values.data(),
                sizeof(float) * static_cast<size_t>(ns) * nc);
}

}  // namespace

extern "C" {

const char* vref_last_error() { return g_err.c_str(); }

// velan::run_cmp with a v-linear ScanConfig grid (the reference pipeline
// verbatim).  Returns 0 ok, 1 config_error, 2 parameter_error, 3 error.
int vref_run_cmp(const float* samples, const float* coords,
                 const int32_t* ntraces, const uint32_t* cdp_id, int G, int M,
                 int ns, uint32_t dt_us, float vmin, float vmax, int nc, int w,
                 int variant, int workers, int32_t* best_idx, float* best_s,
                 float* best_stack, float* matrix, uint64_t* naive) {
  try {
    const velan::Dataset ds =
        make_dataset(samples, coords, ntraces, cdp_id, G, M, ns, dt_us);
    velan::ScanConfig cfg;
    cfg.vmin = vmin;
    cfg.vmax = vmax;
    cfg.nc = nc;
    cfg.w = w;
    cfg.kernel_variant = static_cast<velan::KernelVariant>(variant);
    velan::CacheStats stats;
    const auto res = velan::run_cmp(ds, cfg, workers, &stats);
    std::vector<float> vgrid(nc);
    for (int c = 0; c < nc; ++c) vgrid[c] = cfg.grid().value(c);
    for (size_t r = 0; r < res.size(); ++r)
      fill_matrix_out(res[r], static_cast<int>(r), ns, nc, vgrid, best_idx,
                      best_s, best_stack, matrix);
    if (naive) *naive = stats.naive_fetches;
    return 0;
  } catch (const velan::config_error& e) {
    g_err = e.what();
    return 1;
  } catch (const velan::parameter_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// velan::run_crs (d2 operator) on a gx x gy shard grid.
int vref_run_crs(const float* samples, const float* coords,
                 const int32_t* ntraces, const uint32_t* cdp_id, int G, int M,
                 int ns, uint32_t dt_us, float vmin, float vmax, int nc, int w,
                 int variant, int grid_x, int grid_y, double apm, int workers,
                 int32_t* best_idx, float* best_s, float* best_stack,
                 float* matrix, uint64_t* naive) {
  try {
    const velan::Dataset ds =
        make_dataset(samples, coords, ntraces, cdp_id, G, M, ns, dt_us);
    velan::ScanConfig cfg;
    cfg.vmin = vmin;
    cfg.vmax = vmax;
    cfg.nc = nc;
    cfg.w = w;
    cfg.kernel_variant = static_cast<velan::KernelVariant>(variant);
    velan::CrsOptions opts;
    opts.workers_per_shard = workers;
    velan::CacheStats stats;
    const auto res = velan::run_crs(ds, cfg, velan::GridDims{grid_x, grid_y},
                                    apm, opts, nullptr, &stats);
    std::vector<float> vgrid(nc);
    for (int c = 0; c < nc; ++c) vgrid[c] = cfg.grid().value(c);
    for (size_t r = 0; r < res.size(); ++r)
      fill_matrix_out(res[r], static_cast<int>(r), ns, nc, vgrid, best_idx,
                      best_s, best_stack, matrix);
    if (naive) *naive = stats.naive_fetches;
    return 0;
  } catch (const velan::config_error& e) {
    g_err = e.what();
    return 1;
  } catch (const velan::parameter_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// Output cells (row, k) of a scan over an explicit velocity list v[nc]
// with the reference's own kernels (NMO or the d2 CRS operator).
//   variant 0 baseline, 1 blocked (default production), 2 vectorized (L=4)
//   mode 0 = kernels, 1 = oracle::semblance_reference
// Rows follow run_cmp (input) / run_crs (cdp_id) order like the GPU ABI.
// A velan::Dataset built once (the bench's CPU arm keeps the copy out of its
// timed calls) and reused by vref_run_cells_ds.
void* vref_dataset_create(const float* samples, const float* coords,
                          const int32_t* ntraces, const uint32_t* cdp_id, int G,
                          int M, int ns, uint32_t dt_us) {
  try {
    return new velan::Dataset(
        make_dataset(samples, coords, ntraces, cdp_id, G, M, ns, dt_us));
  } catch (const std::exception& e) {
    g_err = e.what();
    return nullptr;
  }
}

void vref_dataset_destroy(void* ds) { delete static_cast<velan::Dataset*>(ds); }

int vref_run_cells_ds(const void* dsh, int op, int w, int nc, const float* v,
                      double apm, int variant, int mode,
                      const int32_t* cell_row, const int32_t* cell_k,
                      int n_cells, int workers, int32_t* best_idx,
                      float* best_s, float* best_stack, float* matrix,
                      uint64_t* naive) {
  try {
    if (!dsh) throw velan::error("null dataset");
    const velan::Dataset& ds = *static_cast<const velan::Dataset*>(dsh);
    const int G = static_cast<int>(ds.gathers.size());
    const int ns = G ? static_cast<int>(ds.gathers[0].ns) : 0;
    std::vector<uint32_t> cdp_id(G);
    for (int g = 0; g < G; ++g) cdp_id[g] = ds.gathers[g].cdp_id;
    velan::ScanConfig cfg;
    cfg.w = w;
    cfg.nc = nc;
    cfg.kernel_variant = static_cast<velan::KernelVariant>(variant);
    cfg.validate();
    if (ns <= w + 1)
      throw velan::config_error("scan_sweep: window does not fit trace length");

    // output row -> gather, as run_crs orders its results
    std::vector<int> row_gather(G);
    for (int i = 0; i < G; ++i) row_gather[i] = i;
    if (op != 0)
      std::stable_sort(row_gather.begin(), row_gather.end(),
                       [&](int a, int b) { return cdp_id[a] < cdp_id[b]; });
    for (int c = 0; c < n_cells; ++c)
      if (cell_row[c] < 0 || cell_row[c] >= G || cell_k[c] < 0 || cell_k[c] >= ns)
        throw velan::parameter_error("cell outside the dataset");
    std::vector<const velan::CdpGather*> all;
    for (const auto& g : ds.gathers) all.push_back(&g);

    // group the cells by row
    std::map<int, std::vector<int>> by_row;
    for (int c = 0; c < n_cells; ++c) by_row[cell_row[c]].push_back(c);
    std::vector<std::pair<int, std::vector<int>>> jobs(by_row.begin(),
                                                       by_row.end());
    const double dt_s = G ? ds.gathers[0].dt_seconds() : 0.0;
    const int tile = cfg.effective_tile_size();

    velan::CacheStats stats;
    std::atomic<uint64_t> oracle_valid{0};
    velan::detail::parallel_for_indexed(
        jobs.size(), workers, cfg.size_h, cfg.range_cap, &stats,
        [&](std::size_t j, velan::TraceCache& cache) {
          const velan::CdpGather& central =
              ds.gathers[row_gather[jobs[j].first]];
          const std::vector<int>& cells = jobs[j].second;
          std::vector<const velan::CdpGather*> nbrs;
          if (op != 0) nbrs = velan::neighbors_of(central, all, apm);
          const velan::TraceSweep sweep =
              op == 0 ? velan::TraceSweep::single(central)
                      : velan::TraceSweep::with_neighbors(
                            central, nbrs, velan::midpoint_of(central));
          std::vector<float> sem(static_cast<size_t>(cells.size()) * nc);
          std::vector<float> stk(sem.size());
          if (mode == 1) {
            for (size_t i = 0; i < cells.size(); ++i) {
              const float t0 = static_cast<float>(cell_k[cells[i]] * dt_s);
              for (int c = 0; c < nc; ++c) {
                const velan::SemblanceResult r =
                    velan::oracle::semblance_reference(
                        central,
                        op == 0 ? std::span<const velan::CdpGather* const>{}
                                : std::span<const velan::CdpGather* const>(all),
                        t0, v[c], w, op == 0 ? 0.0 : apm);
                sem[i * nc + c] = r.semblance;
                stk[i * nc + c] = r.stack;
                oracle_valid.fetch_add(static_cast<uint64_t>(r.m_used),
                                       std::memory_order_relaxed);
              }
            }
          } else {
            std::vector<velan::PairRequest> pairs;
            pairs.reserve(sem.size());
            for (size_t i = 0; i < cells.size(); ++i) {
              const float t0 = static_cast<float>(cell_k[cells[i]] * dt_s);
              for (int c = 0; c < nc; ++c)
                pairs.push_back(velan::PairRequest{t0, v[c]});
            }
            velan::TileAccumulators acc;
            for (size_t begin = 0; begin < pairs.size(); begin += tile) {
              const size_t count =
                  std::min<size_t>(tile, pairs.size() - begin);
              const std::span<const velan::PairRequest> tp(
                  pairs.data() + begin, count);
              if (variant == 0) {
                for (size_t i = 0; i < count; ++i) {
                  const velan::SemblanceResult r = velan::finalize(
                      velan::scan_pair_baseline(sweep, tp[i], w, cache));
                  sem[begin + i] = r.semblance;
                  stk[begin + i] = r.stack;
                }
                continue;
              }
              if (variant == 1)
                velan::scan_tile_blocked(sweep, tp, w, cache, acc);
              else
                velan::scan_tile_vectorized(sweep, tp, w, 4, cache, acc);
              for (size_t i = 0; i < count; ++i) {
                const velan::SemblanceResult r =
                    acc.result(static_cast<int>(i));
                sem[begin + i] = r.semblance;
                stk[begin + i] = r.stack;
              }
            }
          }
          // argmax: scan.hpp:167-179 (strict '>', lowest index wins)
          for (size_t i = 0; i < cells.size(); ++i) {
            const int cell = cells[i];
            int best_c = 0;
            float best = sem[i * nc];
            for (int c = 1; c < nc; ++c)
              if (sem[i * nc + c] > best) {
                best = sem[i * nc + c];
                best_c = c;
              }
            best_idx[cell] = best_c;
            best_s[cell] = best;
            best_stack[cell] = stk[i * nc + best_c];
            if (matrix)
              std::memcpy(matrix + static_cast<size_t>(cell) * nc,
                          sem.data() + i * nc, sizeof(float) * nc);
          }
        });
    if (naive)
      *naive = mode == 1 ? oracle_valid.load() : stats.naive_fetches;
    return 0;
  } catch (const velan::config_error& e) {
    g_err = e.what();
    return 1;
  } catch (const velan::parameter_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

int vref_run_cells(const float* samples, const float* coords,
                   const int32_t* ntraces, const uint32_t* cdp_id, int G,
                   int M, int ns, uint32_t dt_us, int op, int w, int nc,
                   const float* v, double apm, int variant, int mode,
                   const int32_t* cell_row, const int32_t* cell_k,
                   int n_cells, int workers, int32_t* best_idx, float* best_s,
                   float* best_stack, float* matrix, uint64_t* naive) {
  void* ds = vref_dataset_create(samples, coords, ntraces, cdp_id, G, M, ns, dt_us);
  if (!ds) return 3;
  const int code = vref_run_cells_ds(ds, op, w, nc, v, apm, variant, mode, cell_row,
                                     cell_k, n_cells, workers, best_idx, best_s,
                                     best_stack, matrix, naive);
  vref_dataset_destroy(ds);
  return code;
}

// Scalar hooks onto the reference's own inline functions.
void vref_hit_batch(const float* t, int n, double dt_s, int ns, int w,
                    int32_t* k1, float* x, uint8_t* valid) {
  for (int i = 0; i < n; ++i) {
    const velan::CurveHit h = velan::hit_for(t[i], dt_s, ns, w);
    k1[i] = h.k1;
    x[i] = h.x;
    valid[i] = h.valid ? 1 : 0;
  }
}

void vref_traveltime_batch(const float* t0, const float* h2, const float* d2,
                           const float* v, int n, float* out) {
  for (int i = 0; i < n; ++i)
    out[i] = velan::crs_traveltime(t0[i], h2[i], d2[i], v[i]);
}

void vref_halfpoint_batch(const float* coords, int n, float* h2) {
  velan::CdpGather g;
  g.ns = 2;
  g.traces.resize(n);
  for (int i = 0; i < n; ++i) {
    g.traces[i].sx = coords[4 * i + 0];
    g.traces[i].sy = coords[4 * i + 1];
    g.traces[i].gx = coords[4 * i + 2];
    g.traces[i].gy = coords[4 * i + 3];
  }
  const auto hps = velan::compute_halfpoints(g);
  for (int i = 0; i < n; ++i) h2[i] = hps[i].h2;
}

void vref_finalize(const float* num, int w, float den, float ac, int m_used,
                   float* semblance, float* stack) {
  velan::PairAccumulator acc;
  acc.num.assign(num, num + w);
  acc.den = den;
  acc.ac_linear = ac;
  acc.m_used = m_used;
  const velan::SemblanceResult r = velan::finalize(acc);
  *semblance = r.semblance;
  *stack = r.stack;
}

float vref_interpolate(float a, float b, float x) {
  return velan::interpolate(a, b, x);
}

// velan::write_dataset (io.hpp:95-122) of a flattened dataset.  Returns 0
// ok, 2 parameter_error, 3 error (messages via vref_last_error).
int vref_write_dataset(const char* path, const float* samples, const float* coords,
                       const int32_t* ntraces, const uint32_t* cdp_id, int G, int M,
                       int ns, uint32_t dt_us, const char* metadata) {
  try {
    velan::Dataset ds = make_dataset(samples, coords, ntraces, cdp_id, G, M, ns, dt_us);
    if (metadata) ds.metadata_json = metadata;
    velan::write_dataset(ds, path);
    return 0;
  } catch (const velan::parameter_error& e) {
    g_err = e.what();
    return 2;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// velan::read_dataset (io.hpp:124-166): dims first (out4 = ncdps, fold, ns,
// dt_us of gather 0; metadata length in *meta_len), then, with buffers, the
// flattened arrays.  Returns 0 ok, 1 format_error, 3 error.
int vref_read_dataset(const char* path, int32_t* out4, uint64_t* meta_len, float* samples,
                      float* coords, int32_t* ntraces, uint32_t* cdp_id, char* metadata) {
  try {
    const velan::Dataset ds = velan::read_dataset(path);
    const int G = static_cast<int>(ds.ncdps());
    const int M = static_cast<int>(ds.fold);
    const int ns = G ? static_cast<int>(ds.gathers[0].ns) : 0;
    out4[0] = G;
    out4[1] = M;
    out4[2] = ns;
    out4[3] = G ? static_cast<int32_t>(ds.gathers[0].dt_us) : 0;
    if (meta_len) *meta_len = ds.metadata_json.size();
    if (!samples) return 0;
    for (int g = 0; g < G; ++g) {
      const velan::CdpGather& cg = ds.gathers[g];
      cdp_id[g] = cg.cdp_id;
      ntraces[g] = static_cast<int32_t>(cg.traces.size());
      for (size_t m = 0; m < cg.traces.size(); ++m) {
        const velan::Trace& t = cg.traces[m];
        float* c4 = coords + (static_cast<size_t>(g) * M + m) * 4;
        c4[0] = t.sx;
        c4[1] = t.sy;
        c4[2] = t.gx;
        c4[3] = t.gy;
        std::memcpy(samples + (static_cast<size_t>(g) * M + m) * ns, t.samples.data(),
                    sizeof(float) * ns);
      }
    }
    if (metadata) std::memcpy(metadata, ds.metadata_json.data(), ds.metadata_json.size());
    return 0;
  } catch (const velan::format_error& e) {
    g_err = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

// velan::write_picks (io.hpp:170-194) of n records built from flat arrays.
int vref_write_picks(const char* path, int n, const uint32_t* cdp_id, int ns, int nc,
                     const float* velocity, const float* semblance, const float* matrix) {
  try {
    std::vector<velan::SemblanceMatrix> res(n);
    for (int r = 0; r < n; ++r) {
      velan::SemblanceMatrix& m = res[r];
      m.cdp_id = cdp_id[r];
      m.ns = ns;
      m.nc = nc;
      m.best_velocity.resize(ns);
      for (int k = 0; k < ns; ++k) {
        m.best_velocity[k].velocity = velocity[static_cast<size_t>(r) * ns + k];
        m.best_velocity[k].semblance = semblance[static_cast<size_t>(r) * ns + k];
      }
      if (matrix)
        m.values.assign(matrix + static_cast<size_t>(r) * ns * nc,
                        matrix + static_cast<size_t>(r + 1) * ns * nc);
    }
    velan::write_picks(res, path, matrix != nullptr);
    return 0;
  } catch (const std::exception& e) {
    g_err = e.what();
    return 3;
  }
}

}  // extern "C"
