"""Candidate-group and small-window paths of the FAST kernels (-m gpu).

* Split groups: a last candidate group that fills at most half of the
  consumer warps (1..14 candidates) is swept by two warps per candidate pair,
  half of every batch each, and merged through shared memory at finalize.
  The candidate counts below put 1, 7, 11 and 14 candidates into the last
  group (alone, after one full group, after two), with sweeps of one and of
  several batches and odd batch sizes; FAST must stay within the north-star
  tolerance of the oracle with the exact valid count, and EXACT (never split:
  it keeps the reference's summation order) bitwise.
* Windows of at most four samples interpolate every sample once with the
  reference's rounding and feed numerator and denominator from the same
  value: a one-trace sweep is S = v^2 / v^2 = 1 exactly, as in the reference
  (kernel.hpp:43-50), and short sweeps next to zero crossings keep the
  relative tolerance with a 1e-7 absolute term instead of the long
  windows' 2e-6 M floor.
"""
import numpy as np
import pytest

import oracle
from paper_1907_11678_b200 import Dataset, ScanConfig, velocity_grid

pytestmark = pytest.mark.gpu
RTOL = 1e-4


def gathers(seed, G, M, ns, dt_us=2000, ntr=None, smooth=True):
    rng = np.random.default_rng(seed)
    a = rng.standard_normal((G, M, ns)).astype(np.float32)
    if smooth:  # band-limit: the BASELINE-like regime of the long windows
        k = np.hanning(9).astype(np.float32)
        a = np.apply_along_axis(lambda t: np.convolve(t, k / k.sum(), "same"), 2, a)
        a = a.astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    h = np.linspace(25.0, 1500.0, M).astype(np.float32)
    for g in range(G):
        coords[g, :, 0] = 25.0 * g - h
        coords[g, :, 2] = 25.0 * g + h
    n = np.full(G, M, np.int32) if ntr is None else np.asarray(ntr, np.int32)
    return Dataset(a, coords, n, np.arange(G, dtype=np.uint32), dt_us)


@pytest.mark.parametrize("ncand", [1, 7, 11, 14, 15, 37, 41, 44, 71])
@pytest.mark.parametrize("M", [5, 33, 60])
def test_split_last_group_cmp(engine, ncand, M):
    ds = gathers(100 * ncand + M, 3, M, 256)
    v = velocity_grid(1400.0, 5000.0, ncand)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "nmo", 15, v, rows, ks, mode=2, matrix=True)
    ex = engine.run_cmp(ds, ScanConfig(w=15, velocities=v, kernel_variant="exact"),
                        emit_matrix=True)
    np.testing.assert_array_equal(ex.values.reshape(-1, ncand).view(np.uint32),
                                  ref.matrix.view(np.uint32))
    r = engine.run_cmp(ds, ScanConfig(w=15, velocities=v, kernel_variant="fast"),
                       emit_matrix=True)
    m = r.values.reshape(-1, ncand).astype(np.float64)
    assert r.stats.naive_fetches == ref.valid == ex.stats.naive_fetches
    assert np.all(np.abs(m - ref.matrix) <= RTOL * np.abs(ref.matrix) + 2e-6 * M)
    rep = oracle.compare(r.values.reshape(-1, ncand), ref.matrix)
    assert rep["argmax_mismatches"] == 0, rep
    st = r.stack_trace.reshape(-1).astype(np.float64)
    same = r.best_idx.reshape(-1) == ref.best_idx
    scale = float(np.abs(ds.samples).max())
    assert np.all(np.abs(st - ref.best_stack)[same]
                  <= RTOL * np.abs(ref.best_stack[same]) + 1e-6 * scale)


def test_split_last_group_crs_d2(engine):
    """The d2 operator shares the NMO kernels: a sweep of several gathers
    (one batch per leg), 11 candidates."""
    ds = gathers(7, 9, 12, 200, ntr=[12, 9, 12, 1, 12, 12, 7, 12, 12])
    v = velocity_grid(1500.0, 4000.0, 11)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "d2", 11, v, rows, ks, apm=60.0, mode=2, matrix=True)
    r = engine.run_crs(ds, ScanConfig(w=11, velocities=v, kernel_variant="fast"), 60.0,
                       emit_matrix=True)
    m = r.values.reshape(-1, 11).astype(np.float64)
    assert r.stats.naive_fetches == ref.valid
    assert np.all(np.abs(m - ref.matrix) <= RTOL * np.abs(ref.matrix) + 2e-6 * 36)
    assert oracle.compare(r.values.reshape(-1, 11), ref.matrix)["argmax_mismatches"] == 0


@pytest.mark.parametrize("w", [1, 2, 3, 4])
def test_small_windows_short_sweeps(engine, w):
    """Folds 1 and 2 on white noise (zero crossings everywhere): pure
    relative tolerance, and exactly 1 where the reference gives exactly 1."""
    ds = gathers(40 + w, 6, 2, 333, dt_us=244, ntr=[2, 1, 2, 1, 1, 2], smooth=False)
    v = velocity_grid(1200.0, 5000.0, 9)
    rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
    ref = oracle.run_cells(ds, "nmo", w, v, rows, ks, mode=2, matrix=True)
    r = engine.run_cmp(ds, ScanConfig(w=w, velocities=v, kernel_variant="fast"),
                       emit_matrix=True)
    m = r.values.reshape(-1, 9)
    assert r.stats.naive_fetches == ref.valid
    one = ref.matrix == np.float32(1.0)
    if w == 1:
        assert one.sum() > 1000            # the one-trace gathers' valid cells
        np.testing.assert_array_equal(m[one], ref.matrix[one])
    # relative 1e-4; the 1e-7 absolute term (forty times below the long
    # windows' 2e-6 M floor) covers two-trace sums that cancel to S ~ 1e-6,
    # where one ulp of the interpolation fraction shows
    err = np.abs(m.astype(np.float64) - ref.matrix)
    assert np.all(err <= RTOL * np.abs(ref.matrix) + 1e-7), float(err.max())
