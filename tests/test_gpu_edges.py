"""GPU edge cases against the CPU oracle: ragged gathers (per-gather trace
counts below the padded fold, with the padding poisoned so a read of it
would show) and non-finite samples inside the traces.

The reference stores each gather's traces in a vector (types.hpp:27-39), so a
ragged line has no padding at all; the flattened layout here pads every
gather to Mmax traces and the kernels must never touch a trace at index
>= ntraces[g].  A NaN sample inside a window makes the reference's
denominator NaN, and finalize's `den > 0` test (kernel.hpp:43-50) then gives
semblance 0 while the stack stays NaN; the kernels must reproduce exactly the
cells that do so (EXACT: bitwise, NaN positions included).
"""
import numpy as np
import pytest

import oracle
from helpers import line_dataset, poison_samples
from paper_1907_11678_b200 import CrsAbcGrid, ScanConfig, velocity_grid

pytestmark = pytest.mark.gpu


def bits(a):
    return np.ascontiguousarray(a, np.float32).view(np.uint32)


def check(r, ref, ns, ncand, variant, M):
    G = r.best_idx.shape[0]
    m = r.values.reshape(G * ns, ncand)
    if variant == "exact":
        np.testing.assert_array_equal(bits(m), bits(ref.matrix))
        np.testing.assert_array_equal(r.best_idx.reshape(-1), ref.best_idx)
        np.testing.assert_array_equal(bits(r.best_semblance).reshape(-1),
                                      bits(ref.best_semblance))
        st, rs = r.stack_trace.reshape(-1), ref.best_stack
        np.testing.assert_array_equal(np.isnan(st), np.isnan(rs))
        ok = ~np.isnan(rs)
        np.testing.assert_array_equal(bits(st[ok]), bits(rs[ok]))
    else:
        ref_m = ref.matrix.astype(np.float64)
        assert not np.isnan(m).any()
        # U[-1, 1] data: relative 1e-4 plus the 2e-6 * M semblance floor
        assert np.all(np.abs(m - ref_m) <= 1e-4 * np.abs(ref_m) + 2e-6 * M)
        rep = oracle.compare(m, ref.matrix)
        assert rep["argmax_mismatches"] == 0, rep
        same = r.best_idx.reshape(-1) == ref.best_idx
        np.testing.assert_array_equal(np.isnan(r.stack_trace.reshape(-1)[same]),
                                      np.isnan(ref.best_stack[same]))
    assert r.stats.naive_fetches == ref.valid


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_ragged_cmp(engine, variant):
    """Per-gather trace counts 1..M with NaN padding (the reference's
    vector-of-traces gathers, types.hpp:27-39)."""
    ds = line_dataset(11)
    v = velocity_grid(1500.0, 3500.0, 13)
    for w in (11, 15):
        cfg = ScanConfig(w=w, velocities=v, kernel_variant=variant)
        r = engine.run_cmp(ds, cfg, emit_matrix=True)
        rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
        ref = oracle.run_cells(ds, "nmo", w, v, rows, ks, matrix=True)
        check(r, ref, ds.ns, len(v), variant, 9)
        nominal = int(ds.ntraces.sum()) * ds.ns * len(v)
        assert r.stats.nominal_intersections == nominal


@pytest.mark.parametrize("op", ["d2", "abc"])
@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_ragged_crs(engine, op, variant):
    """A CRS sweep over neighbours of different folds (TraceSweep
    concatenates each neighbour's own traces, kernel.hpp:61-113), NaN
    padding never read."""
    ds = line_dataset(12)
    w = 11
    if op == "d2":
        v = velocity_grid(1500.0, 3500.0, 9)
        cfg = ScanConfig(w=w, velocities=v, kernel_variant=variant)
        r = engine.run_crs(ds, cfg, 75.0, emit_matrix=True)
        ncand = len(v)
        rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
        ref = oracle.run_cells(ds, "d2", w, v, rows, ks, apm=75.0, matrix=True)
    else:
        grid = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 2),
                          np.linspace(1500, 3500, 5))
        cfg = ScanConfig(w=w, velocities=grid.v, kernel_variant=variant)
        r = engine.run_crs(ds, cfg, 75.0, abc=grid, emit_matrix=True)
        ncand = grid.ncand
        rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
        ref = oracle.run_cells(ds, "abc", w, None, rows, ks, apm=75.0, abc=grid,
                               matrix=True)
    check(r, ref, ds.ns, ncand, variant, 9 * 7)


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_nan_samples(engine, variant):
    """NaN samples inside traces: every cell whose window covers one gets the
    reference's semblance 0 (den is NaN, finalize's den > 0 fails) and a NaN
    stack; no other cell changes."""
    ds = poison_samples(line_dataset(13, ragged=False), 5, 12)
    v = velocity_grid(1500.0, 3500.0, 13)
    cfg = ScanConfig(w=15, velocities=v, kernel_variant=variant)
    r = engine.run_cmp(ds, cfg, emit_matrix=True)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "nmo", 15, v, rows, ks, matrix=True)
    assert np.isnan(ref.best_stack).any() or (ref.matrix == 0).any()
    check(r, ref, ds.ns, len(v), variant, 9)


def _canon(a):
    a = np.array(a, np.float32)
    a[np.isnan(a)] = np.float32("nan")
    return a.view(np.uint32)


def test_inf_samples_nan_semblance_pick_rule(engine):
    """+Inf samples make den = inf and sum_sq = inf, so the reference's
    semblance is inf/inf = NaN (kernel.hpp:43-50).  scan_sweep's pick
    (scan.hpp:167-179: best = S[0], strict '>') then keeps candidate 0 when
    S[0] is NaN, and never picks a NaN elsewhere.  The kernel's argmax runs in
    any order across warps and must follow the same rule: EXACT bitwise
    (NaNs canonicalised), picks identical, on cells of both kinds; top-k's
    entry 0 is the pick."""
    ds = line_dataset(14, ragged=False)
    rng = np.random.default_rng(21)
    for _ in range(40):
        g, m, k = int(rng.integers(0, ds.ncdps)), int(rng.integers(0, 9)), int(rng.integers(20, 230))
        ds.samples[g, m, k] = np.inf
    v = velocity_grid(1500.0, 3500.0, 37)
    cfg = ScanConfig(w=11, velocities=v, kernel_variant="exact")
    r = engine.run_cmp(ds, cfg, emit_matrix=True, topk=3)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "nmo", 11, v, rows, ks, matrix=True)
    nan0 = np.isnan(ref.matrix[:, 0])
    nan_other = np.isnan(ref.matrix[:, 1:]).any(axis=1) & ~nan0
    assert nan0.any() and nan_other.any()  # both situations occur
    m = r.values.reshape(-1, len(v))
    np.testing.assert_array_equal(_canon(m), _canon(ref.matrix))
    np.testing.assert_array_equal(r.best_idx.reshape(-1), ref.best_idx)
    np.testing.assert_array_equal(_canon(r.best_semblance.reshape(-1)), _canon(ref.best_semblance))
    assert np.all(r.best_idx.reshape(-1)[nan0] == 0)
    np.testing.assert_array_equal(r.topk_idx.reshape(-1, 3)[:, 0], ref.best_idx)
    ti = r.topk_idx.reshape(-1, 3)
    # no NaN other than at flat index 0 is ever ranked
    ts = r.topk_semblance.reshape(-1, 3)
    assert not np.isnan(ts[ti != 0]).any()
