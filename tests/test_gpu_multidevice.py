"""Device-count invariance of the in-process multi-device path.

The reference pins run_cmp bitwise across 1/2/4/8 workers
(/root/reference/proj/tests/test_cmp_pipeline.cpp:122-140, pool at
cmp_pipeline.hpp:34-88).  Here ``workers`` are devices: the C-ABI splits the
output rows into balanced contiguous blocks (split_rows), one host thread and
one shard (its gathers + the CRS halo, re-indexed locally) per device.  With a
single B200 the split is exercised by several contexts on device 0
(Engine([0, 0, 0, 0]): four host threads, four stream pairs, four shards),
which must equal Engine([0]) bit for bit — picks, semblance, stack, the full
matrix, top-k and the valid-intersection count.
"""
import numpy as np
import pytest

from paper_1907_11678_b200 import CrsAbcGrid, Engine, ScanConfig, configs

pytestmark = pytest.mark.gpu


def _bits(a):
    return np.asarray(a, np.float32).view(np.uint32)


def _same(a, b):
    np.testing.assert_array_equal(a.best_idx, b.best_idx)
    np.testing.assert_array_equal(_bits(a.best_semblance), _bits(b.best_semblance))
    np.testing.assert_array_equal(_bits(a.stack_trace), _bits(b.stack_trace))
    np.testing.assert_array_equal(a.row_gather, b.row_gather)
    if a.values is not None:
        np.testing.assert_array_equal(_bits(a.values), _bits(b.values))
    if a.topk_idx is not None:
        np.testing.assert_array_equal(a.topk_idx, b.topk_idx)
        np.testing.assert_array_equal(_bits(a.topk_semblance), _bits(b.topk_semblance))
    assert a.stats.naive_fetches == b.stats.naive_fetches
    assert a.stats.nominal_intersections == b.stats.nominal_intersections


@pytest.fixture(scope="module")
def engines():
    one = Engine([0])
    four = Engine([0, 0, 0, 0])
    three = Engine([0, 0, 0])
    yield one, three, four
    for e in (one, three, four):
        e.close()


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_cmp_device_count_invariant(engines, variant):
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=13)  # not a multiple of the device count
    cfg = ScanConfig(w=wl.config.w, velocities=wl.config.grid(), kernel_variant=variant)
    one, three, four = engines
    ref = one.run_cmp(ds, cfg, emit_matrix=True, topk=3)
    for eng in (three, four):
        _same(eng.run_cmp(ds, cfg, emit_matrix=True, topk=3), ref)


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_crs_d2_device_count_invariant(engines, variant):
    wl = configs.crs_small()
    ds = wl.spec.generate(count=23)
    cfg = ScanConfig(w=wl.config.w, velocities=wl.config.grid(), kernel_variant=variant)
    one, three, four = engines
    ref = one.run_crs(ds, cfg, wl.apm, emit_matrix=True, topk=2)
    for eng in (three, four):
        _same(eng.run_crs(ds, cfg, wl.apm, emit_matrix=True, topk=2), ref)


@pytest.mark.parametrize("variant", ["exact", "fast"])
def test_crs_abc_device_count_invariant(engines, variant):
    wl = configs.crs_small()
    ds = wl.spec.generate(first=100, count=30)
    grid = CrsAbcGrid(wl.abc.a[::2], wl.abc.b[::3], wl.abc.v[::2])
    cfg = ScanConfig(w=wl.config.w, velocities=grid.v, kernel_variant=variant)
    one, three, four = engines
    ref = one.run_crs(ds, cfg, wl.apm, abc=grid, emit_matrix=True, topk=4)
    for eng in (three, four):
        _same(eng.run_crs(ds, cfg, wl.apm, abc=grid, emit_matrix=True, topk=4), ref)
    # a shard's own block (rows) splits the same way
    ref = one.run_crs(ds, cfg, wl.apm, abc=grid, rows=(6, 17))
    _same(four.run_crs(ds, cfg, wl.apm, abc=grid, rows=(6, 17)), ref)


def test_reference_named_entry_points_use_the_split(engines):
    """api.run_cmp(workers=N) maps workers onto devices (min(N, visible));
    the result is independent of N."""
    from paper_1907_11678_b200 import run_cmp
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=5)
    cfg = ScanConfig(w=wl.config.w, velocities=wl.config.grid(), kernel_variant="fast")
    a = run_cmp(ds, cfg, workers=1)
    b = run_cmp(ds, cfg, workers=8)
    _same(a, b)
