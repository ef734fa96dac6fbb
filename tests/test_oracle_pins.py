"""Known-answer pins of the CPU oracle, ported from the reference's own test
suite (/root/reference/proj/tests/*.cpp, Catch2 — not buildable here), plus
bitwise agreement with the reference compiled from its headers (oracle/_ref).
"""
import ctypes as C
import math

import numpy as np
import pytest

import oracle
from helpers import make_gather, random_gathers, reference_synthetic
from paper_1907_11678_b200 import velocity_grid

lib = oracle.oracle_lib()
needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def f32(x):
    return float(np.float32(x))


def one_cell(ds, t0_index, v, w, mode=0, op="nmo"):
    r = oracle.run_cells(ds, op, w, np.array([v], np.float32),
                         np.array([0], np.int32), np.array([t0_index], np.int32),
                         mode=mode, matrix=True, stack_matrix=True, threads=1)
    return float(r.matrix[0, 0]), float(r.stack_matrix[0, 0]), r.valid


# ---- test_kernel.cpp:42-46 -------------------------------------------------
def test_interpolate_is_linear():
    assert lib.vo_interpolate(1.0, 3.0, 0.5) == 2.0
    assert lib.vo_interpolate(7.0, -4.0, 0.0) == 7.0
    assert lib.vo_interpolate(2.0, 6.0, 0.25) == 3.0


# ---- test_kernel.cpp:48-84 -------------------------------------------------
def finalize(num, den, ac, m):
    num = np.asarray(num, np.float32)
    s, st = C.c_float(), C.c_float()
    lib.vo_finalize(num.ctypes.data, len(num), den, ac, m, C.byref(s), C.byref(st))
    return s.value, st.value


def test_finalize_coherence_formula():
    s, st = finalize([2, 4, 6], 2.0 * 14, 12.0, 2)        # identical traces -> M
    assert s == pytest.approx(2.0) and st == pytest.approx(2.0)
    s, _ = finalize([0, 0], 4.0, 0.0, 2)                   # anti-correlated
    assert s == 0.0
    s, _ = finalize([3, 4, 5], 26.0, 12.0, 2)              # hand-computed window
    assert s == pytest.approx(50.0 / 26.0)
    s, st = finalize([0, 0, 0], 0.0, 0.0, 0)               # dead window -> 0
    assert s == 0.0 and st == 0.0


@needs_ref
def test_finalize_matches_reference_bitwise():
    rng = np.random.default_rng(1)
    rl = oracle.ref_lib()
    for _ in range(200):
        w = int(rng.integers(1, 17))
        num = rng.normal(size=w).astype(np.float32)
        den, ac, m = float(np.float32(rng.uniform(0, 10))), float(np.float32(rng.normal())), int(rng.integers(0, 9))
        a = finalize(num, den, ac, m)
        s, st = C.c_float(), C.c_float()
        rl.vref_finalize(num.ctypes.data, w, den, ac, m, C.byref(s), C.byref(st))
        assert np.float32(a[0]).view(np.uint32) == np.float32(s.value).view(np.uint32)
        assert np.float32(a[1]).view(np.uint32) == np.float32(st.value).view(np.uint32)


# ---- test_kernel.cpp:86-105, test_oracle.cpp:14-24 --------------------------
def hand_gather():
    t1 = np.zeros(32, np.float32)
    t2 = np.zeros(32, np.float32)
    t1[7:12] = [1, 1, 2, 3, 3]
    t2[7:12] = [2, 2, 2, 2, 2]
    return make_gather([t1, t2], 244)


@pytest.mark.parametrize("mode", [0, 1])
def test_hand_case_50_over_26(mode):
    s, _, valid = one_cell(hand_gather(), 9, 2500.0, 3, mode)
    assert valid == 2
    assert s == pytest.approx(50.0 / 26.0, rel=1e-6)


# ---- test_kernel.cpp:108-131 ------------------------------------------------
def test_all_zero_gather_gives_zero():
    ds = make_gather(np.zeros((4, 64)), 244)
    s, st, valid = one_cell(ds, 32, 2500.0, 5)
    assert s == 0.0 and st == 0.0 and valid == 4


@pytest.mark.parametrize("mode", [0, 1])
def test_single_nonzero_trace_gives_one(mode):
    ds = random_gathers(np.random.default_rng(31), 1, 1, 64)
    s, _, valid = one_cell(ds, 30, 2200.0, 5, mode)
    assert valid == 1
    assert s == pytest.approx(1.0, rel=1e-6)


def test_identical_traces_saturate_at_m():
    rng = np.random.default_rng(39)
    row = (rng.integers(0, 100, 64) / 50.0 - 1.0).astype(np.float32)
    s, _, valid = one_cell(make_gather([row] * 5, 244), 30, 2500.0, 7)
    assert valid == 5
    assert s == pytest.approx(5.0, rel=1e-6)


# ---- test_kernel.cpp:311-341: bounds and scale invariance -------------------
def test_bounds_and_scale_invariance():
    rng = np.random.default_rng(39)
    for it in range(30):
        fold = int(rng.integers(2, 14))
        ds = random_gathers(rng, 1, fold, 96, 244, 20.0)
        k = int(12 + rng.integers(0, 60))
        v = float(2000 + rng.integers(0, 1000))
        s, st, m = one_cell(ds, k, v, 5)
        assert 0.0 <= s <= m * (1 + 1e-6)
        ds.samples = (ds.samples * np.float32(3.75)).astype(np.float32)
        s2, st2, _ = one_cell(ds, k, v, 5)
        assert s2 == pytest.approx(s, rel=1e-5, abs=1e-9)
        assert st2 == pytest.approx(st * 3.75, rel=1e-5, abs=1e-6)


# ---- test_traveltime.cpp:11-25 ----------------------------------------------
def test_halfpoints_follow_geometry():
    assert lib.vo_halfpoint(0, 0, 100, 0) == 2500.0
    assert lib.vo_halfpoint(0, 0, 0, 0) == 0.0
    assert lib.vo_halfpoint(0, 0, 30, 40) == 625.0


# ---- test_traveltime.cpp:27-41 ----------------------------------------------
def test_velocity_grid_spans_range():
    g = velocity_grid(2000.0, 3000.0, 101)
    assert g[0] == 2000.0 and g[100] == 3000.0
    assert g[50] == pytest.approx(2500.0)
    assert velocity_grid(1500.0, 9999.0, 1)[0] == 1500.0
    from paper_1907_11678_b200 import ParameterError
    for bad in [(0.0, 100.0, 4), (200.0, 100.0, 4), (100.0, 200.0, 0)]:
        with pytest.raises(ParameterError):
            velocity_grid(*bad)


def traveltime(op, t0, h2, dm, v, A=None, B=None):
    t0, h2, dm, v = (np.ascontiguousarray(np.atleast_1d(x), np.float32) for x in (t0, h2, dm, v))
    n = len(t0)
    A = np.zeros(n, np.float32) if A is None else np.ascontiguousarray(A, np.float32)
    B = np.zeros(n, np.float32) if B is None else np.ascontiguousarray(B, np.float32)
    out = np.zeros(n, np.float32)
    lib.vo_traveltime_batch(oracle.OP[op], t0.ctypes.data, h2.ctypes.data, dm.ctypes.data,
                            A.ctypes.data, B.ctypes.data, v.ctypes.data, n, out.ctypes.data)
    return out


# ---- test_traveltime.cpp:43-84 ----------------------------------------------
def test_nmo_traveltime_hyperbola():
    assert traveltime("nmo", 0.5, 0.0, 0, 2500.0)[0] == 0.5
    assert traveltime("nmo", 0.0, 2500.0, 0, 1000.0)[0] == pytest.approx(0.1)
    assert traveltime("nmo", 1.0, 2500.0, 0, 2000.0)[0] == pytest.approx(
        math.sqrt(1.0 + 4.0 * 2500.0 / (2000.0 * 2000.0)), rel=1e-6)


def test_crs_traveltime_extends_by_d2_and_reduces_bitwise():
    assert traveltime("d2", 0.0, 0.0, 100.0, 1000.0)[0] == pytest.approx(0.1)
    assert traveltime("d2", 1.0, 2500.0, 20.0, 2000.0)[0] == pytest.approx(
        math.sqrt(1.0 + (4.0 * 2500.0 + 400.0) / 4.0e6), rel=1e-6)
    rng = np.random.default_rng(11)
    t0 = rng.uniform(0, 2, 1000).astype(np.float32)
    h2 = rng.uniform(0, 1e6, 1000).astype(np.float32)
    v = rng.uniform(500, 6000, 1000).astype(np.float32)
    z = np.zeros(1000, np.float32)
    np.testing.assert_array_equal(traveltime("d2", t0, h2, z, v), traveltime("nmo", t0, h2, z, v))
    # the ABC operator at dm = 0 is the NMO hyperbola bit for bit
    A = rng.uniform(-2e-4, 2e-4, 1000)
    B = rng.uniform(0, 1e-7, 1000)
    np.testing.assert_array_equal(traveltime("abc", t0, h2, z, v, A, B), traveltime("nmo", t0, h2, z, v))


def test_nmo_properties():
    rng = np.random.default_rng(12)
    t0 = rng.uniform(0.01, 2, 1000).astype(np.float32)
    h2 = rng.uniform(1, 1e6, 1000).astype(np.float32)
    v1 = rng.uniform(500, 6000, 1000).astype(np.float32)
    v2 = rng.uniform(500, 6000, 1000).astype(np.float32)
    lo, hi = np.minimum(v1, v2), np.maximum(v1, v2)
    z = np.zeros(1000, np.float32)
    a, b = traveltime("nmo", t0, h2, z, lo), traveltime("nmo", t0, h2, z, hi)
    assert np.all(a >= b) and np.all(a >= t0)
    np.testing.assert_array_equal(traveltime("nmo", t0, z, z, lo), t0)


@needs_ref
def test_traveltime_matches_reference_bitwise():
    rng = np.random.default_rng(5)
    n = 20000
    t0 = rng.uniform(0, 4, n).astype(np.float32)
    h2 = rng.uniform(0, 2.5e6, n).astype(np.float32)
    dm = rng.uniform(-200, 200, n).astype(np.float32)
    v = rng.uniform(1000, 6000, n).astype(np.float32)
    d2 = (dm * dm).astype(np.float32)
    out = np.zeros(n, np.float32)
    oracle.ref_lib().vref_traveltime_batch(t0.ctypes.data, h2.ctypes.data, d2.ctypes.data,
                                           v.ctypes.data, n, out.ctypes.data)
    np.testing.assert_array_equal(traveltime("d2", t0, h2, dm, v).view(np.uint32), out.view(np.uint32))


# ---- test_traveltime.cpp:86-133 ---------------------------------------------
def hit(t, dt, ns, w):
    k1, x, v = oracle.hit_batch(np.array([t], np.float32), dt, ns, w)
    return int(k1[0]), float(x[0]), bool(v[0])


def test_hit_for_centres_the_window():
    dt = 1.0 / 4096.0
    assert hit(f32(100.0 * dt), dt, 200, 4) == (98, 0.0, True)
    k1, _, valid = hit(0.0, dt, 200, 4)
    assert k1 == -2 and not valid
    assert hit(f32(10.25 * dt), dt, 200, 3) == (9, 0.25, True)
    assert hit(f32(102.0 * dt), dt, 105, 4)[2]
    assert not hit(f32(103.0 * dt), dt, 105, 4)[2]


def test_hit_for_recovers_sample_position():
    rng = np.random.default_rng(13)
    dt, ns = 220e-6, 512
    for _ in range(2000):
        w = int(1 + rng.integers(0, 16))
        s = rng.uniform(0, 500)
        t = np.float32(s * dt)
        k1, x, valid = hit(float(t), dt, ns, w)
        assert 0.0 <= x < 1.0
        if valid:
            t_rec = (k1 + w // 2 + x) * dt
            assert abs(t_rec - float(t)) <= float(np.nextafter(t, np.float32(2 * t + 1)) - t)


@needs_ref
def test_hit_for_matches_reference_bitwise():
    rng = np.random.default_rng(14)
    for dt in (0.004, 0.002, 220e-6, 244e-6, 1.0 / 4096.0):
        ns, w = 2000, 15
        k = rng.integers(0, ns, 30000)
        t = np.concatenate([(k * dt).astype(np.float32),
                            rng.uniform(0, ns * dt, 30000).astype(np.float32),
                            np.array([0.0, 1e-30, -1.0, 1e3], np.float32)])
        # (t/dt beyond 2^31 samples hits undefined behaviour in the reference's
        # int conversion; the restatement and the GPU reject such hits)
        a = oracle.hit_batch(t, dt, ns, w)
        b = oracle.hit_batch(t, dt, ns, w, ref=True)
        np.testing.assert_array_equal(a[2], b[2])
        np.testing.assert_array_equal(a[0][a[2]], b[0][b[2]])
        np.testing.assert_array_equal(a[1].view(np.uint32), b[1].view(np.uint32))


# ---- test_cmp_pipeline.cpp:47-74: planted velocities and the tie rule -------
def test_planted_velocity_picks():
    ds = reference_synthetic(1, 16, 200, 220, [(0.0154, 2500.0, 1.0), (0.033, 2700.0, 0.8)],
                             wavelet_freq=300.0, max_offset=160.0)
    v = velocity_grid(2000.0, 3000.0, 101)
    rows, ks = oracle.all_cells(1, 200)
    r = oracle.run_cells(ds, "nmo", 4, v, rows, ks, threads=2)
    k1 = int(round(0.0154 / 220e-6))
    k2 = int(round(0.033 / 220e-6))
    assert v[r.best_idx[k1]] == 2500.0
    assert v[r.best_idx[k2]] == 2700.0
    assert r.best_semblance[k1] > 1.0


def test_all_zero_gather_picks_first_velocity():
    ds = make_gather(np.zeros((4, 128)), 220)
    v = velocity_grid(2000.0, 3000.0, 11)
    rows, ks = oracle.all_cells(1, 128)
    r = oracle.run_cells(ds, "nmo", 4, v, rows, ks, matrix=True)
    assert np.all(r.best_semblance == 0.0)
    assert np.all(r.best_idx == 0)
    assert np.all(r.matrix == 0.0)


# ---- test_oracle.cpp:43-65 / acceptance.cpp:71-134 ---------------------------
def test_kernel_order_vs_double_oracle_within_1e5():
    rng = np.random.default_rng(72)
    for it in range(10):
        fold = int(1 + rng.integers(0, 24))
        w = int(1 + rng.integers(0, 12))
        ds = random_gathers(rng, 1, fold, 128, 244, 30.0)
        v = velocity_grid(2000.0, 3000.0, 8)
        rows, ks = oracle.all_cells(1, 128)
        a = oracle.run_cells(ds, "nmo", w, v, rows, ks, mode=0, matrix=True)
        b = oracle.run_cells(ds, "nmo", w, v, rows, ks, mode=1, matrix=True)
        rep = oracle.compare(a.matrix, b.matrix)
        assert rep["max_rel_err"] <= 1e-5
        assert rep["argmax_mismatches"] == 0


@needs_ref
@pytest.mark.parametrize("seed", range(6))
def test_random_gathers_bitwise_vs_reference_kernels(seed):
    """acceptance.cpp:71-134 shapes: random fold/ns/nc/w; the C restatement
    equals velan::scan_tile_blocked (and the baseline kernel) bit for bit."""
    rng = np.random.default_rng(20260809 + seed)
    for _ in range(5):
        fold = int(1 + rng.integers(0, 64))
        ns = int(48 + rng.integers(0, 465))
        nc = int(2 + rng.integers(0, 63))
        w = int(rng.choice([1, 4, 8, 11, 16]))
        ds = random_gathers(rng, 2, fold, ns, 244, 10.0 + rng.integers(0, 40))
        v = velocity_grid(2000.0, 3000.0, nc)
        rows, ks = oracle.all_cells(2, ns)
        a = oracle.run_cells(ds, "nmo", w, v, rows, ks, matrix=True)
        for variant in (0, 1):
            b = oracle.ref_run_cells(ds, "nmo", w, v, rows, ks, variant=variant, matrix=True, workers=2)
            np.testing.assert_array_equal(a.matrix.view(np.uint32), b.matrix.view(np.uint32))
            np.testing.assert_array_equal(a.best_idx, b.best_idx)
            np.testing.assert_array_equal(a.best_stack.view(np.uint32), b.best_stack.view(np.uint32))
            assert a.valid == b.valid
        c = oracle.ref_run_cells(ds, "nmo", w, v, rows, ks, mode=1, matrix=True, workers=2)
        d = oracle.run_cells(ds, "nmo", w, v, rows, ks, mode=1, matrix=True)
        np.testing.assert_array_equal(c.matrix.view(np.uint32), d.matrix.view(np.uint32))


@needs_ref
def test_crs_d2_bitwise_vs_reference_pipeline():
    """run_crs on a 2x2 shard grid (test_oracle.cpp:67-89 shape) vs the C
    restatement's closed-ball / cdp_id-ordered sweep."""
    ds = reference_synthetic(25, 5, 160, 220, [(0.0132, 2500.0, 1.0)],
                             wavelet_freq=300.0, max_offset=100.0, cdp_spacing=12.5)
    code, msg, ref = oracle.ref_run_pipeline(ds, "crs", 2000.0, 3000.0, 11, 4,
                                             grid=(2, 2), apm=12.5, workers=2)
    assert code == 0, msg
    v = velocity_grid(2000.0, 3000.0, 11)
    rows, ks = oracle.all_cells(25, 160)
    a = oracle.run_cells(ds, "d2", 4, v, rows, ks, apm=12.5, matrix=True)
    np.testing.assert_array_equal(a.matrix.reshape(25, 160, 11).view(np.uint32), ref.matrix.view(np.uint32))
    np.testing.assert_array_equal(a.best_idx.reshape(25, 160), ref.best_idx)
    assert a.valid == ref.valid


# ---- test_oracle.cpp:91-140: compare() semantics ----------------------------
def test_compare_semantics():
    rng = np.random.default_rng(73)
    m = rng.uniform(0, 3, (96, 7)).astype(np.float32)
    rep = oracle.compare(m, m)
    assert rep["max_rel_err"] == 0.0 and rep["mean_rel_err"] == 0.0
    assert rep["argmax_mismatches"] == 0 and rep["tie_excused"] == 0
    p = m.copy()
    p[40, 3] += np.float32(1e-3)
    rep = oracle.compare(p, m)
    assert rep["max_rel_err"] == pytest.approx(1e-3 / abs(float(m[40, 3])), rel=1e-3)
    assert rep["max_rel_err"] >= rep["mean_rel_err"] >= 0.0
    assert rep["cells"] == m.size


def test_oracle_rejects_invalid_configurations():
    ds = make_gather(np.zeros((2, 8)), 244)
    rows, ks = np.zeros(1, np.int32), np.zeros(1, np.int32)
    with pytest.raises(ValueError):
        oracle.run_cells(ds, "nmo", 0, np.array([2000.0]), rows, ks)          # w < 1
    with pytest.raises(ValueError):
        oracle.run_cells(ds, "nmo", 7, np.array([2000.0]), rows, ks)          # ns <= w + 1
    with pytest.raises(ValueError):
        oracle.run_cells(ds, "nmo", 2, np.array([-1.0]), rows, ks)            # v <= 0


# ---- ragged gathers and NaN samples (types.hpp:27-39, kernel.hpp:43-50) ----
@needs_ref
@pytest.mark.parametrize("poison", [False, True])
def test_ragged_and_nan_bitwise_vs_reference(poison):
    """The C restatement on a ragged line (per-gather trace counts 1..M, NaN
    in the padding slots the reference does not have) and, with poison=True,
    NaN samples inside real traces: matrix, picks, stacks and valid counts
    bit for bit against the reference's blocked and baseline kernels, and
    the d2 CRS sweep against velan::run_crs."""
    from helpers import line_dataset, poison_samples
    ds = line_dataset(21)
    if poison:
        ds = poison_samples(ds, 6, 10)
    v = velocity_grid(1500.0, 3500.0, 9)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    a = oracle.run_cells(ds, "nmo", 11, v, rows, ks, matrix=True)
    for variant in (0, 1):
        b = oracle.ref_run_cells(ds, "nmo", 11, v, rows, ks, variant=variant, matrix=True, workers=2)
        np.testing.assert_array_equal(a.matrix.view(np.uint32), b.matrix.view(np.uint32))
        np.testing.assert_array_equal(a.best_idx, b.best_idx)
        np.testing.assert_array_equal(np.isnan(a.best_stack), np.isnan(b.best_stack))
        ok = ~np.isnan(a.best_stack)
        np.testing.assert_array_equal(a.best_stack[ok].view(np.uint32), b.best_stack[ok].view(np.uint32))
        assert a.valid == b.valid
    if poison:
        assert (a.matrix == 0).any() and np.isnan(a.best_stack).any()
    code, msg, ref = oracle.ref_run_pipeline(ds, "crs", 1500.0, 3500.0, 9, 11,
                                             grid=(1, 1), apm=75.0, workers=2)
    assert code == 0, msg
    c = oracle.run_cells(ds, "d2", 11, v, rows, ks, apm=75.0, matrix=True)
    np.testing.assert_array_equal(c.matrix.reshape(ref.matrix.shape).view(np.uint32),
                                  ref.matrix.view(np.uint32))
    np.testing.assert_array_equal(c.best_idx.reshape(ref.best_idx.shape), ref.best_idx)
    assert c.valid == ref.valid
