"""The reference's own known answers (test_kernel.cpp, test_cmp_pipeline.cpp,
test_oracle.cpp — pinned on the CPU oracle in test_oracle_pins.py) through
the GPU path, both variants: EXACT must give the very numbers, FAST the same
picks and semblance within 1e-4 relative."""
import numpy as np
import pytest

from helpers import make_gather, random_gathers, reference_synthetic
from paper_1907_11678_b200 import ScanConfig, VelanError, velocity_grid

pytestmark = pytest.mark.gpu
VARIANTS = ["exact", "fast"]


def cell(engine, ds, k, v, w, variant):
    r = engine.run_cmp(ds, ScanConfig(w=w, velocities=np.array([v], np.float32),
                                      kernel_variant=variant), emit_matrix=True)
    return float(r.values[0, k, 0]), float(r.stack_trace[0, k])


def approx(variant, x, rel=1e-6):
    return pytest.approx(x, rel=rel if variant == "exact" else 1e-4)


@pytest.mark.parametrize("variant", VARIANTS)
def test_hand_case_50_over_26(engine, variant):
    """test_kernel.cpp:86-105: two traces, t0 = 9 dt, w = 3 -> 50/26."""
    t1 = np.zeros(32, np.float32)
    t2 = np.zeros(32, np.float32)
    t1[7:12] = [1, 1, 2, 3, 3]
    t2[7:12] = [2, 2, 2, 2, 2]
    s, _ = cell(engine, make_gather([t1, t2], 244), 9, 2500.0, 3, variant)
    assert s == approx(variant, 50.0 / 26.0)


@pytest.mark.parametrize("variant", VARIANTS)
def test_all_zero_gather(engine, variant):
    """test_kernel.cpp:108-117 / test_cmp_pipeline.cpp:64-74: zeros -> S = 0,
    stack 0, every pick the first velocity."""
    ds = make_gather(np.zeros((4, 128)), 220)
    v = velocity_grid(2000.0, 3000.0, 11)
    r = engine.run_cmp(ds, ScanConfig(w=4, velocities=v, kernel_variant=variant),
                       emit_matrix=True)
    assert np.all(r.values == 0.0)
    assert np.all(r.best_idx == 0) and np.all(r.best_semblance == 0.0)
    assert np.all(r.stack_trace == 0.0)


@pytest.mark.parametrize("variant", VARIANTS)
def test_single_trace_gives_one(engine, variant):
    """test_kernel.cpp:119-130: M = 1 -> S = 1 wherever the window is non-zero."""
    ds = random_gathers(np.random.default_rng(31), 1, 1, 64)
    s, _ = cell(engine, ds, 30, 2200.0, 5, variant)
    assert s == approx(variant, 1.0)


@pytest.mark.parametrize("variant", VARIANTS)
def test_identical_traces_saturate_at_m(engine, variant):
    """test_kernel.cpp:343-355: M identical traces at zero offset -> S = M."""
    rng = np.random.default_rng(39)
    row = (rng.integers(0, 100, 64) / 50.0 - 1.0).astype(np.float32)
    s, _ = cell(engine, make_gather([row] * 5, 244), 30, 2500.0, 7, variant)
    assert s == approx(variant, 5.0)


@pytest.mark.parametrize("variant", VARIANTS)
def test_scale_invariance(engine, variant):
    """test_kernel.cpp:311-341: S in [0, M], invariant under scaling; the stack
    scales."""
    rng = np.random.default_rng(40)
    ds = random_gathers(rng, 3, 9, 96, 244, 20.0)
    v = velocity_grid(2000.0, 3000.0, 7)
    cfg = ScanConfig(w=5, velocities=v, kernel_variant=variant)
    a = engine.run_cmp(ds, cfg, emit_matrix=True)
    assert np.all(a.values >= 0) and np.all(a.values <= 9 * (1 + 1e-5))
    ds.samples = (np.asarray(ds.samples) * np.float32(3.75)).astype(np.float32)
    b = engine.run_cmp(ds, cfg, emit_matrix=True)
    np.testing.assert_allclose(b.values, a.values, rtol=1e-5, atol=1e-7)
    np.testing.assert_allclose(b.stack_trace, a.stack_trace * 3.75, rtol=1e-4, atol=1e-5)


@pytest.mark.parametrize("variant", VARIANTS)
def test_planted_velocities(engine, variant):
    """test_cmp_pipeline.cpp:47-62: events at 2500 and 2700 m/s are picked."""
    ds = reference_synthetic(1, 16, 200, 220, [(0.0154, 2500.0, 1.0), (0.033, 2700.0, 0.8)],
                             wavelet_freq=300.0, max_offset=160.0)
    v = velocity_grid(2000.0, 3000.0, 101)
    r = engine.run_cmp(ds, ScanConfig(w=4, velocities=v, kernel_variant=variant))
    k1 = int(round(0.0154 / 220e-6))
    k2 = int(round(0.033 / 220e-6))
    assert v[r.best_idx[0, k1]] == 2500.0
    assert v[r.best_idx[0, k2]] == 2700.0
    assert r.best_semblance[0, k1] > 1.0


def test_empty_gather_fails_like_the_worker_pool(engine):
    """cmp_pipeline.hpp:77-85 + types.hpp:57-62: an empty gather is an error,
    raised before any device work."""
    ds = make_gather(np.zeros((2, 32)), 244)
    ds.ntraces[:] = 0
    with pytest.raises(VelanError):
        engine.run_cmp(ds, ScanConfig(w=3, velocities=np.array([2000.0], np.float32)))
