"""GPU parity: the sm_100a kernels through the C-ABI against the CPU oracle.

EXACT variant: bitwise equal to the reference arithmetic (semblance matrix,
picks, stack, valid-intersection count).  FAST variant: identical picks except
near-ties, semblance and stack within the north-star tolerance (1e-4 relative;
stack with an absolute floor).
"""
import numpy as np
import pytest

import oracle
from paper_1907_11678_b200 import (CrsAbcGrid, ScanConfig, configs,
                                    slowness_grid, velocity_grid)

pytestmark = pytest.mark.gpu

SEM_RTOL = 1e-4


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def assert_bitwise(gpu, ref_cells, ns, ncand=None):
    G = gpu.best_idx.shape[0]
    np.testing.assert_array_equal(gpu.best_idx.reshape(-1), ref_cells.best_idx)
    np.testing.assert_array_equal(bits(gpu.best_semblance).reshape(-1),
                                  bits(ref_cells.best_semblance))
    np.testing.assert_array_equal(bits(gpu.stack_trace).reshape(-1),
                                  bits(ref_cells.best_stack))
    if ncand is not None and ref_cells.matrix is not None:
        np.testing.assert_array_equal(bits(gpu.values).reshape(G * ns, ncand),
                                      bits(ref_cells.matrix))
    assert gpu.stats.naive_fetches == ref_cells.valid


def assert_close(gpu, ref_cells, ns, ncand, stack_floor, sem_floor=0.0):
    """FAST variant check.  sem_floor = 0: pure relative 1e-4 (the north-star
    bound, used on BASELINE-like data).  sem_floor > 0: relative 1e-4 plus an
    absolute floor on the semblance scale [0, M] for adversarial random data,
    where sum_j num_j cancels and any reassociation — the reference's own
    blocked vs oracle included — differs at ~eps*M (the reference's tests use
    the same kind of margin for its vectorized variant, test_kernel.cpp:221-226)."""
    G = gpu.best_idx.shape[0]
    m_gpu = gpu.values.reshape(G * ns, ncand)
    rep = oracle.compare(m_gpu, ref_cells.matrix)
    if sem_floor == 0.0:
        assert rep["max_rel_err"] <= SEM_RTOL, rep
    else:
        d = np.abs(m_gpu.astype(np.float64) - ref_cells.matrix)
        assert np.all(d <= SEM_RTOL * np.abs(ref_cells.matrix) + sem_floor), float(d.max())
    assert rep["argmax_mismatches"] == 0, rep
    same = gpu.best_idx.reshape(-1) == ref_cells.best_idx
    # stack at the pick: relative with an absolute floor (near-cancelling mean)
    d = np.abs(gpu.stack_trace.reshape(-1)[same] - ref_cells.best_stack[same])
    tol = SEM_RTOL * np.abs(ref_cells.best_stack[same]) + stack_floor
    assert np.all(d <= tol), float(np.max(d - tol))
    assert gpu.stats.naive_fetches == ref_cells.valid


@pytest.fixture(scope="module")
def cmp_small():
    w = configs.cmp_small()
    return w, w.spec.generate()


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_cmp_small_full(engine, cmp_small, variant):
    w, ds = cmp_small
    cfg = ScanConfig(w=w.config.w, velocities=w.config.grid(), kernel_variant=variant)
    r = engine.run_cmp(ds, cfg, emit_matrix=True)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "nmo", cfg.w, cfg.grid(), rows, ks, matrix=True)
    if variant == "exact":
        assert_bitwise(r, ref, ds.ns, len(cfg.grid()))
    else:
        assert_close(r, ref, ds.ns, len(cfg.grid()), 1e-6 * float(np.abs(ds.samples).max()))
    assert r.stats.nominal_intersections == ds.ncdps * ds.ns * 101 * 24


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_crs_d2_subset(engine, variant):
    w = configs.crs_small()
    ds = w.spec.generate(count=24)
    v = velocity_grid(1500.0, 3500.0, 21)
    cfg = ScanConfig(w=11, velocities=v, kernel_variant=variant)
    r = engine.run_crs(ds, cfg, 125.0, emit_matrix=True)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "d2", 11, v, rows, ks, apm=125.0, matrix=True)
    if variant == "exact":
        assert_bitwise(r, ref, ds.ns, 21)
    else:
        assert_close(r, ref, ds.ns, 21, 1e-6 * float(np.abs(ds.samples).max()))


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_crs_abc_subset(engine, variant):
    w = configs.crs_small()
    ds = w.spec.generate(count=16)
    grid = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 3),
                      np.linspace(1500, 3500, 7))
    cfg = ScanConfig(w=11, velocities=grid.v, kernel_variant=variant)
    r = engine.run_crs(ds, cfg, 125.0, abc=grid, emit_matrix=True)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "abc", 11, None, rows, ks, apm=125.0, abc=grid, matrix=True)
    if variant == "exact":
        assert_bitwise(r, ref, ds.ns, grid.ncand)
    else:
        assert_close(r, ref, ds.ns, grid.ncand, 1e-6 * float(np.abs(ds.samples).max()))


@pytest.mark.parametrize("w", [1, 2, 3, 4, 5, 8, 11, 13, 15, 16, 21, 32])
@pytest.mark.parametrize("ns,variant", [(131, "exact"), (132, "exact"),
                                        (131, "fast"), (132, "fast")])
def test_window_lengths(engine, w, ns, variant):
    """Every window length, through both staging paths (ns % 4 / ns % 2
    decide between TMA bulk copies and the synchronous fallback)."""
    rng = np.random.default_rng(100 + w)
    G, M = 3, 7
    samples = rng.uniform(-1, 1, (G, M, ns)).astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    coords[:, :, 2] = np.linspace(0, 40, M)[None, :]
    from paper_1907_11678_b200 import Dataset
    ds = Dataset(samples, coords, np.full(G, M, np.int32), np.arange(G, dtype=np.uint32), 244)
    v = velocity_grid(2000.0, 3000.0, 9)
    cfg = ScanConfig(w=w, velocities=v, kernel_variant=variant)
    if ns <= w + 1:
        pytest.skip("window does not fit")
    r = engine.run_cmp(ds, cfg, emit_matrix=True)
    rows, ks = oracle.all_cells(G, ns)
    ref = oracle.run_cells(ds, "nmo", w, v, rows, ks, matrix=True)
    if variant == "exact":
        assert_bitwise(r, ref, ns, len(v))
    else:
        # U[-1, 1] noise, M = 7: semblance scale M, floor 2e-6 * M
        assert_close(r, ref, ns, len(v), 1e-6, sem_floor=2e-6 * M)


@pytest.mark.parametrize("ns,w", [(2513, 15), (4001, 11), (5960, 21)])
def test_long_traces_fast(engine, ns, w):
    """Traces longer than the default FAST stage (2512 samples): the
    large-stage kernel (one CTA per SM), through TMA (even ns) and the
    synchronous fallback (odd ns), up to the FAST limit."""
    rng = np.random.default_rng(ns)
    G, M = 2, 6
    samples = rng.uniform(-1, 1, (G, M, ns)).astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    coords[:, :, 2] = np.linspace(0, 3000, M)[None, :]
    from paper_1907_11678_b200 import Dataset
    ds = Dataset(samples, coords, np.full(G, M, np.int32), np.arange(G, dtype=np.uint32), 1000)
    v = velocity_grid(1500.0, 4000.0, 5)
    r = engine.run_cmp(ds, ScanConfig(w=w, velocities=v, kernel_variant="fast"), emit_matrix=True)
    rng2 = np.random.default_rng(1)
    rows = rng2.integers(0, G, 600).astype(np.int32)
    ks = rng2.integers(0, ns, 600).astype(np.int32)
    ref = oracle.run_cells(ds, "nmo", w, v, rows, ks, matrix=True)
    got = r.values.reshape(G, ns, len(v))[rows, ks]
    rep = oracle.compare(got, ref.matrix)
    # U[-1, 1] noise: relative 1e-4 plus the 2e-6 * M semblance floor
    err = np.abs(got.astype(np.float64) - ref.matrix)
    assert np.all(err <= 1e-4 * np.abs(ref.matrix) + 2e-6 * M), rep
    ex = engine.run_cmp(ds, ScanConfig(w=w, velocities=v, kernel_variant="exact"))
    assert r.stats.naive_fetches == ex.stats.naive_fetches


def test_hit_exact_matches_reference_rule():
    from paper_1907_11678_b200 import _native as N
    import ctypes as C
    rng = np.random.default_rng(7)
    dt = 0.004
    ns, w = 1000, 11
    k = rng.integers(0, ns, 20000)
    t = np.concatenate([
        (k * dt).astype(np.float32),                      # on-sample t0 values
        rng.uniform(0, ns * dt, 20000).astype(np.float32),
        np.array([0.0, 1e-30, np.inf, np.nan, -1.0, 1e9], np.float32)])
    for variant in (0, 1):
        k1 = np.zeros(len(t), np.int32)
        x = np.zeros(len(t), np.float32)
        valid = np.zeros(len(t), np.uint8)
        code = N.load().velan_gpu_hit_batch(t.ctypes.data, len(t), dt, ns, w, variant,
                                            k1.ctypes.data, x.ctypes.data, valid.ctypes.data)
        assert code == 0
        ok1, ox, ov = oracle.hit_batch(t, dt, ns, w)
        np.testing.assert_array_equal(valid.astype(bool), ov)
        np.testing.assert_array_equal(k1[ov], ok1[ov])
        if variant == 0:
            np.testing.assert_array_equal(bits(x[ov]), bits(ox[ov]))
        else:
            assert np.max(np.abs(x[ov] - ox[ov])) <= 2 ** -23


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_run_cmp_matches_reference_pipeline(engine, cmp_small):
    """velan::run_cmp (v-linear ScanConfig grid) vs the GPU with the same grid."""
    _, ds = cmp_small
    sub = ds.subset(range(8))
    code, msg, ref = oracle.ref_run_pipeline(sub, "cmp", 1400.0, 4000.0, 41, 11, workers=4)
    assert code == 0, msg
    cfg = ScanConfig(vmin=1400.0, vmax=4000.0, nc=41, w=11)
    r = engine.run_cmp(sub, cfg, emit_matrix=True)
    np.testing.assert_array_equal(bits(r.values), bits(ref.matrix))
    np.testing.assert_array_equal(r.best_idx, ref.best_idx)
    np.testing.assert_array_equal(bits(r.stack_trace), bits(ref.best_stack))
    assert r.stats.naive_fetches == ref.valid


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_run_crs_matches_reference_pipeline(engine):
    w = configs.crs_small()
    ds = w.spec.generate(count=24)
    code, msg, ref = oracle.ref_run_pipeline(ds, "crs", 1500.0, 3500.0, 15, 11,
                                             grid=(2, 1), apm=125.0, workers=4)
    assert code == 0, msg
    cfg = ScanConfig(vmin=1500.0, vmax=3500.0, nc=15, w=11)
    r = engine.run_crs(ds, cfg, 125.0, emit_matrix=True)
    np.testing.assert_array_equal(bits(r.values), bits(ref.matrix))
    np.testing.assert_array_equal(r.best_idx, ref.best_idx)
    np.testing.assert_array_equal(bits(r.stack_trace), bits(ref.best_stack))
    assert r.stats.naive_fetches == ref.valid


@pytest.mark.parametrize("variant,k", [("exact", 1), ("exact", 5), ("fast", 8)])
def test_topk_matches_matrix(engine, variant, k):
    """Per-sample top-k (§8f-2) equals the k best entries of the full matrix
    (best first, ties to the lower flat index); entry 0 is the pick."""
    wl = configs.crs_small()
    ds = wl.spec.generate(count=12)
    grid = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 2),
                      np.linspace(1500, 3500, 5))
    cfg = ScanConfig(w=11, velocities=grid.v, kernel_variant=variant)
    r = engine.run_crs(ds, cfg, 125.0, abc=grid, emit_matrix=True, topk=k)
    m = r.values.reshape(-1, grid.ncand)
    # reference order: descending semblance, ascending index among equals
    order = np.lexsort((np.broadcast_to(np.arange(grid.ncand), m.shape), -m), axis=1)[:, :k]
    ti = r.topk_idx.reshape(-1, k)
    ts = r.topk_semblance.reshape(-1, k)
    np.testing.assert_array_equal(ti, order)
    np.testing.assert_array_equal(ts, np.take_along_axis(m, order, axis=1))
    np.testing.assert_array_equal(ti[:, 0], r.best_idx.reshape(-1))


def test_topk_more_than_candidates(engine, cmp_small):
    """k > n_cand: the tail entries are index -1."""
    ds = cmp_small[1].subset(range(2))
    cfg = ScanConfig(w=11, velocities=velocity_grid(1500.0, 3000.0, 3))
    r = engine.run_cmp(ds, cfg, topk=5)
    assert np.all(r.topk_idx[..., 3:] == -1)
    assert np.all(np.sort(r.topk_idx[..., :3], axis=-1) == np.arange(3))


def test_topk_crs_large_slice_bounded_panel(engine):
    """Top-k on a 64-midpoint CRS-large slice (18081 candidates): the
    semblance panel is per wave (<= 4 GB), not the shard's 9.3 GB; top-1 is
    the pick, the k entries are sorted, and the picks equal a run without
    top-k bit for bit."""
    import torch
    wl = configs.crs_large()
    wl.config.kernel_variant = "fast"
    halo = 10
    ds = wl.spec.generate(first=1000 - halo, count=64 + 2 * halo)
    plain = engine.run_crs(ds, wl.config, wl.apm, abc=wl.abc, rows=(halo, 64))
    torch.cuda.synchronize()
    free0, _ = torch.cuda.mem_get_info()
    r = engine.run_crs(ds, wl.config, wl.apm, abc=wl.abc, rows=(halo, 64), topk=4)
    free1, _ = torch.cuda.mem_get_info()
    whole = 64 * ds.ns * wl.ncand * 4
    assert free0 - free1 < 0.6 * whole, (free0 - free1, whole)
    np.testing.assert_array_equal(r.topk_idx[..., 0], plain.best_idx)
    np.testing.assert_array_equal(r.best_idx, plain.best_idx)
    np.testing.assert_array_equal(r.best_semblance.view(np.uint32),
                                  plain.best_semblance.view(np.uint32))
    ts = r.topk_semblance
    assert np.all(ts[..., :-1] >= ts[..., 1:])
    np.testing.assert_array_equal(ts[..., 0], plain.best_semblance)


@pytest.mark.parametrize("op", ["nmo", "abc"])
def test_nmo_corrected_gathers_match_oracle(engine, op):
    """NMO-corrected output gathers from the scan's own
    picks: bitwise equal to the oracle's restatement (crs_traveltime at the
    pick, hit_for with w = 1, interpolate), ragged traces zero."""
    if op == "nmo":
        wl = configs.cmp_small()
        ds = wl.spec.generate(count=6)
        ds.ntraces[2] = 17
        cfg = ScanConfig(w=11, velocities=wl.config.grid(), kernel_variant="fast")
        r = engine.run_cmp(ds, cfg)
        out = engine.nmo_correct(ds, cfg, r.best_idx)
        ref = oracle.nmo_correct(ds, "nmo", cfg.grid(), r.best_idx)
        assert np.all(out[2, 17:] == 0)
    else:
        wl = configs.crs_small()
        ds = wl.spec.generate(first=50, count=12)
        grid = CrsAbcGrid(wl.abc.a[::5], wl.abc.b[::5], wl.abc.v)
        cfg = ScanConfig(w=11, velocities=grid.v, kernel_variant="fast")
        r = engine.run_crs(ds, cfg, wl.apm, abc=grid)
        out = engine.nmo_correct(ds, cfg, r.best_idx, op="abc", apm=wl.apm, abc=grid)
        ref = oracle.nmo_correct(ds, "abc", grid.v, r.best_idx)
    np.testing.assert_array_equal(out.view(np.uint32), ref.view(np.uint32))


def test_nmo_correction_flattens_a_planted_event(engine):
    """A noiseless hyperbolic event at v = 2500 m/s: corrected with the picks
    the scan finds, every trace peaks at the event's zero-offset time."""
    from helpers import reference_synthetic
    ds = reference_synthetic(2, 24, 1500, 1000, [(0.6, 2500.0, 1.0), (1.1, 3000.0, 0.8)],
                             wavelet_freq=25.0, max_offset=1200.0)
    cfg = ScanConfig(w=11, velocities=velocity_grid(2000.0, 3500.0, 31), kernel_variant="fast")
    r = engine.run_cmp(ds, cfg)
    out = engine.nmo_correct(ds, cfg, r.best_idx)
    for t0 in (0.6, 1.1):
        k = int(round(t0 / 1e-3))
        win = out[:, 1:, k - 20:k + 21]  # trace 0 is zero offset already
        assert np.all(np.abs(np.argmax(win, axis=2) - 20) <= 1)
        # and the uncorrected far traces do not peak there
        assert np.argmax(ds.samples[0, -1, k - 20:k + 21]) != 20
