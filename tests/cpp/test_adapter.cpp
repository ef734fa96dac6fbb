// test_adapter.cpp — the drop-in check: the reference pipeline and the GPU
// adapter (include/velan_gpu/adapter.hpp) on the same inputs, in one program.
//
// Built by oracle/Makefile against the UNMODIFIED reference headers into
// oracle/_ref/test_adapter (test infrastructure; needs a B200 to run).  Exit
// code = number of failed checks.
#include <sys/resource.h>

#include <cmath>
#include <cstdio>
#include <cstring>
#include <random>
#include <string>

#include "velan/velan.hpp"
#include "velan_gpu/adapter.hpp"

namespace {

int failures = 0;

void check(bool ok, const char* what, const std::string& detail = "") {
  std::printf("%s  %s %s\n", ok ? "PASS" : "FAIL", what, detail.c_str());
  if (!ok) ++failures;
}

bool same_bits(const std::vector<float>& a, const std::vector<float>& b) {
  return a.size() == b.size() &&
         (a.empty() || std::memcmp(a.data(), b.data(), a.size() * 4) == 0);
}

bool matrices_equal(const std::vector<velan::SemblanceMatrix>& a,
                    const std::vector<velan::SemblanceMatrix>& b) {
  if (a.size() != b.size()) return false;
  for (size_t i = 0; i < a.size(); ++i) {
    if (a[i].cdp_id != b[i].cdp_id || a[i].ns != b[i].ns || a[i].nc != b[i].nc)
      return false;
    if (!same_bits(a[i].values, b[i].values)) return false;
    if (!same_bits(a[i].stack_trace, b[i].stack_trace)) return false;
    for (int k = 0; k < a[i].ns; ++k)
      if (std::memcmp(&a[i].best_velocity[k], &b[i].best_velocity[k],
                      sizeof(velan::BestPick)))
        return false;
  }
  return true;
}

velan::Dataset synthetic(int ncdps, double snr, double spacing = 25.0,
                         int fold = 16) {
  velan::GenParams p;
  p.ncdps = ncdps;
  p.fold = fold;
  p.ns = 200;
  p.dt_us = 220;
  p.wavelet_freq = 300.0;
  p.max_offset = 160.0;
  p.cdp_spacing = spacing;
  p.snr = snr;
  p.seed = 1234;
  p.events = {velan::ReflectorEvent{0.0154, 2500.0f, 1.0f},
              velan::ReflectorEvent{0.033, 2700.0f, 0.8f}};
  return velan::generate_synthetic(p);
}

}  // namespace

// CMP large through the drop-in with values = false: 8192 gathers x 60 x
// 2000 samples (the reference's own containers, 3.9 GB), picks only.  Peak
// RSS stays far below the 26 GB the full matrix would take.
int large_picks_only() {
  velan::Dataset ds;
  ds.fold = 60;
  ds.gathers.resize(8192);
  std::mt19937 rng(5);
  std::uniform_real_distribution<float> u(-1.0f, 1.0f);
  std::vector<float> noise(1 << 16);
  for (float& x : noise) x = u(rng);
  for (int g = 0; g < 8192; ++g) {
    velan::CdpGather& cg = ds.gathers[g];
    cg.cdp_id = g;
    cg.ns = 2000;
    cg.dt_us = 2000;
    cg.traces.resize(60);
    for (int m = 0; m < 60; ++m) {
      velan::Trace& t = cg.traces[m];
      const float h = 25.0f * (m + 1), mx = 25.0f * g;
      t.sx = mx - h;
      t.gx = mx + h;
      t.samples.resize(2000);
      const size_t off = (static_cast<size_t>(g) * 60 + m) * 2000 % (noise.size() - 2000);
      std::memcpy(t.samples.data(), noise.data() + off, 2000 * 4);
    }
  }
  velan::ScanConfig cfg;
  cfg.nc = 401;
  cfg.w = 15;
  cfg.vmin = 1400.0f;
  cfg.vmax = 5000.0f;
  velan::CacheStats st;
  const auto out = velan_gpu::run_cmp(ds, cfg, 1, &st,
                                      velan_gpu::Options{velan_gpu::Variant::fast, false});
  struct rusage ru;
  getrusage(RUSAGE_SELF, &ru);
  const double rss_gb = ru.ru_maxrss / 1048576.0;
  check(out.size() == 8192 && out[0].values.empty() && out[8191].best_velocity.size() == 2000,
        "CMP large, values = false: 8192 picked gathers");
  check(rss_gb < 16.0, "peak RSS without the 26 GB matrix", std::to_string(rss_gb) + " GB");
  std::printf("%d failure(s)\n", failures);
  return failures;
}

int main(int argc, char** argv) {
  if (argc > 1 && std::string(argv[1]) == "large") return large_picks_only();
  // 1. run_cmp: bitwise equal to the reference pipeline (blocked kernel)
  {
    const velan::Dataset ds = synthetic(6, 3.0);
    velan::ScanConfig cfg;
    cfg.nc = 21;
    cfg.w = 4;
    velan::CacheStats s_ref, s_gpu;
    const auto ref = velan::run_cmp(ds, cfg, 4, &s_ref);
    const auto gpu = velan_gpu::run_cmp(ds, cfg, 1, &s_gpu);
    check(matrices_equal(ref, gpu), "run_cmp bitwise vs velan::run_cmp");
    check(s_ref.naive_fetches == s_gpu.naive_fetches, "run_cmp naive_fetches",
          std::to_string(s_ref.naive_fetches) + " vs " +
              std::to_string(s_gpu.naive_fetches));
  }
  // 2. scan_cdp with the default ScanConfig (v 2000..3000, nc 101, w 4)
  {
    const velan::Dataset ds = synthetic(1, 0.0);
    velan::ScanConfig cfg;
    const auto ref = velan::scan_cdp(ds.gathers[0], cfg);
    const auto gpu = velan_gpu::scan_cdp(ds.gathers[0], cfg);
    check(matrices_equal({ref}, {gpu}), "scan_cdp bitwise vs velan::scan_cdp");
    const int k1 = static_cast<int>(std::lround(0.0154 / 220e-6));
    check(gpu.best_velocity[k1].velocity == 2500.0f, "planted 2500 m/s pick");
  }
  // 3. run_crs on a 2x2 shard grid: same results as the sharded reference
  {
    const velan::Dataset ds = synthetic(25, 8.0, 12.5, 5);
    velan::ScanConfig cfg;
    cfg.nc = 11;
    cfg.w = 4;
    velan::CacheStats s_ref, s_gpu;
    const auto ref = velan::run_crs(ds, cfg, velan::GridDims{2, 2}, 12.5, {},
                                    nullptr, &s_ref);
    const auto gpu = velan_gpu::run_crs(ds, cfg, velan::GridDims{2, 2}, 12.5,
                                        {}, nullptr, &s_gpu);
    check(matrices_equal(ref, gpu), "run_crs bitwise vs velan::run_crs");
    check(s_ref.naive_fetches == s_gpu.naive_fetches, "run_crs naive_fetches");
  }
  // 4. scan_central_cdp with explicit neighbours
  {
    const velan::Dataset ds = synthetic(9, 8.0, 12.5, 6);
    std::vector<const velan::CdpGather*> all;
    for (const auto& g : ds.gathers) all.push_back(&g);
    velan::ScanConfig cfg;
    cfg.nc = 17;
    cfg.w = 5;
    const auto nbrs = velan::neighbors_of(ds.gathers[4], all, 12.5);
    const auto ref = velan::scan_central_cdp(ds.gathers[4], nbrs, cfg);
    const auto gpu = velan_gpu::scan_central_cdp(ds.gathers[4], nbrs, cfg);
    check(matrices_equal({ref}, {gpu}), "scan_central_cdp bitwise",
          "neighbours=" + std::to_string(nbrs.size()));
  }
  // 5. error behaviour: config errors before compute, worker failures
  {
    const velan::Dataset ds = synthetic(3, 0.0);
    velan::ScanConfig bad;
    bad.w = 0;
    bool ref_cfg = false, gpu_cfg = false;
    try { velan::run_cmp(ds, bad, 1); } catch (const velan::config_error&) { ref_cfg = true; }
    try { velan_gpu::run_cmp(ds, bad, 1); } catch (const velan::config_error&) { gpu_cfg = true; }
    check(ref_cfg && gpu_cfg, "w = 0 -> config_error (both)");
    velan::Dataset holes = synthetic(3, 0.0);
    holes.gathers[2].traces.clear();
    velan::ScanConfig cfg;
    cfg.nc = 5;
    std::string ref_msg, gpu_msg;
    try { velan::run_cmp(holes, cfg, 2); } catch (const velan::error& e) { ref_msg = e.what(); }
    try { velan_gpu::run_cmp(holes, cfg, 1); } catch (const velan::error& e) { gpu_msg = e.what(); }
    check(ref_msg.find("worker pool failure") != std::string::npos &&
              gpu_msg.find("worker pool failure") != std::string::npos,
          "empty gather -> worker pool failure (both)", gpu_msg);
    bool ref_apm = false, gpu_apm = false;
    const velan::Dataset grid = synthetic(25, 0.0, 12.5, 5);
    try { velan::run_crs(grid, cfg, velan::GridDims{2, 2}, 30.0); } catch (const velan::config_error&) { ref_apm = true; }
    try { velan_gpu::run_crs(grid, cfg, velan::GridDims{2, 2}, 30.0); } catch (const velan::config_error&) { gpu_apm = true; }
    check(ref_apm && gpu_apm, "apm > half shard -> config_error (both)");
    velan::Dataset empty;
    check(velan_gpu::run_cmp(empty, cfg, 1).empty(), "empty dataset -> {}");
  }
  // 6. FAST variant: identical picks, semblance within 1e-4
  {
    const velan::Dataset ds = synthetic(4, 5.0);
    velan::ScanConfig cfg;
    cfg.nc = 41;
    cfg.w = 4;
    const auto ref = velan::run_cmp(ds, cfg, 2);
    const auto gpu = velan_gpu::run_cmp(ds, cfg, 1, nullptr, velan_gpu::Variant::fast);
    double max_rel = 0.0;
    for (size_t i = 0; i < ref.size(); ++i)
      for (size_t j = 0; j < ref[i].values.size(); ++j)
        max_rel = std::max(max_rel, std::abs(static_cast<double>(gpu[i].values[j]) - ref[i].values[j]) /
                                        std::max(std::abs(static_cast<double>(ref[i].values[j])), 1e-12));
    const auto rep = velan::oracle::compare(gpu, ref);
    check(max_rel <= 1e-4 && rep.argmax_mismatches == 0, "FAST variant within 1e-4",
          "max_rel=" + std::to_string(max_rel));
  }
  // 7. values = false: the same picks and stack, no matrix anywhere
  {
    const velan::Dataset ds = synthetic(5, 5.0);
    velan::ScanConfig cfg;
    cfg.nc = 33;
    cfg.w = 4;
    const auto full = velan_gpu::run_cmp(ds, cfg, 1);
    velan::CacheStats st;
    const auto picks = velan_gpu::run_cmp(ds, cfg, 1, &st, velan_gpu::Options{velan_gpu::Variant::exact, false});
    bool ok = picks.size() == full.size();
    for (size_t i = 0; ok && i < full.size(); ++i) {
      ok = picks[i].values.empty() && picks[i].cdp_id == full[i].cdp_id &&
           same_bits(picks[i].stack_trace, full[i].stack_trace);
      for (int k = 0; ok && k < full[i].ns; ++k)
        ok = std::memcmp(&picks[i].best_velocity[k], &full[i].best_velocity[k],
                         sizeof(velan::BestPick)) == 0;
    }
    check(ok && st.naive_fetches > 0, "values = false: picks and stack only");
  }
  // 8. run_crs_abc: with the aperture holding only the central gather
  //    (dm = 0) the three-parameter operator is NMO bit for bit, so the
  //    picks equal velan::run_cmp's (ia = ib = 0 by the tie rule) and every
  //    (A, B) column of the matrix equals the reference's v column
  {
    const velan::Dataset ds = synthetic(4, 5.0, 200.0);
    velan::ScanConfig cfg;
    cfg.nc = 17;
    cfg.w = 5;
    const auto ref = velan::run_cmp(ds, cfg, 1);
    velan_gpu::AbcGrid grid;
    grid.a = {-2e-4f, 0.0f, 1e-4f};
    grid.b = {0.0f, 5e-8f};
    for (int c = 0; c < cfg.nc; ++c) grid.v.push_back(cfg.grid().value(c));
    velan::CacheStats st;
    const auto abc = velan_gpu::run_crs_abc(ds, grid, cfg.w, 1.0, 1, &st);
    bool ok = abc.size() == ref.size();
    const int nab = 6, nc = cfg.nc;
    for (size_t i = 0; ok && i < ref.size(); ++i) {
      ok = abc[i].cdp_id == ref[i].cdp_id && same_bits(abc[i].stack_trace, ref[i].stack_trace) &&
           abc[i].nc == nab * nc;
      for (int k = 0; ok && k < ref[i].ns; ++k) {
        const velan_gpu::AbcPick& p = abc[i].best[k];
        ok = p.ia == 0 && p.ib == 0 && grid.v[p.ic] == ref[i].best_velocity[k].velocity &&
             std::memcmp(&p.semblance, &ref[i].best_velocity[k].semblance, 4) == 0;
        for (int ab = 0; ok && ab < nab; ++ab)
          for (int c = 0; ok && c < nc; ++c)
            ok = std::memcmp(&abc[i].values[static_cast<size_t>(k) * nab * nc + ab * nc + c],
                             &ref[i].values[static_cast<size_t>(k) * nc + c], 4) == 0;
      }
    }
    check(ok && st.naive_fetches > 0, "run_crs_abc (dm = 0) == run_cmp bitwise, (ia, ib, ic) picks");
    bool cfg_err = false;
    try { velan_gpu::run_crs_abc(ds, velan_gpu::AbcGrid{}, 5, 1.0); } catch (const velan::config_error&) { cfg_err = true; }
    check(cfg_err, "run_crs_abc: empty axes -> config_error");
  }
  std::printf("%d failure(s)\n", failures);
  return failures;
}
