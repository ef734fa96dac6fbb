"""Host-side logic (no device): BASELINE workload sizes, the synthetic
generator, the sweep construction behind the C-ABI and the sharding helpers."""
import numpy as np
import pytest

import oracle
from paper_1907_11678_b200 import ScanConfig, configs, describe, neighbors_of
from paper_1907_11678_b200.sharding import block_range, line_shards, weak_shard


# nominal work of each config (exact sums, line ends truncated)
@pytest.mark.parametrize("name,evals", [
    ("cmp_small", 1_706_496_000),
    ("cmp_large", 8192 * 2000 * 401 * 60 * 15),
    ("crs_small", 2786 * 30 * 1000 * 2541 * 11),
    ("crs_large", 85906 * 60 * 2000 * 18081 * 15),
])
def test_nominal_work_matches_survey(name, evals):
    w = configs.WORKLOADS[name]()
    assert w.nominal_evals() == evals


def test_cmp_small_grid_is_slowness_linear():
    v = configs.cmp_small().config.grid()
    assert len(v) == 101
    assert v[0] == np.float32(1400.0)
    assert abs(float(v[-1]) - 4000.0) < 1e-2
    p = 1.0 / v.astype(np.float64)
    assert np.allclose(np.diff(p), np.diff(p)[0], rtol=1e-5)


def test_generator_is_deterministic_and_shardable():
    spec = configs.cmp_small().spec
    a = spec.generate(n_threads=1)
    b = spec.generate(n_threads=7)
    np.testing.assert_array_equal(a.samples, b.samples)
    np.testing.assert_array_equal(a.coords, b.coords)
    part = spec.generate(first=10, count=5, n_threads=3)
    np.testing.assert_array_equal(part.samples, a.samples[10:15])
    np.testing.assert_array_equal(part.cdp_id, np.arange(10, 15))
    # geometry: sx = mx - h, gx = mx + h, so h2 = h^2 exactly
    h = 50.0 * (np.arange(24) + 1)
    h2 = ((a.coords[0, :, 2] - a.coords[0, :, 0]) ** 2) * np.float32(0.25)
    np.testing.assert_array_equal(h2, (h * h).astype(np.float32))
    # noise sigma 0.1 plus events: roughly the right energy
    assert 0.09 < float(a.samples.std()) < 0.3


def test_crs_generator_line_and_events():
    spec = configs.crs_small().spec
    ds = spec.generate(count=32)
    mp = ds.midpoints()
    np.testing.assert_array_equal(mp[:, 0], (np.arange(32) * 25.0).astype(np.float32))
    assert np.all(mp[:, 1] == 0)
    # reflectors are global: a shard of a longer line equals the slice
    full = spec.generate()
    np.testing.assert_array_equal(spec.generate(first=100, count=8).samples, full.samples[100:108])


def test_sweeps_match_oracle_neighbourhoods():
    """The library's host sweep (velan_gpu_describe) visits the central
    gather then the closed-ball neighbours in cdp_id order, exactly like
    neighbors_of + TraceSweep::with_neighbors."""
    w = configs.crs_small()
    ds = w.spec.generate(count=40)
    # shuffle cdp ids to exercise the cdp_id ordering
    rng = np.random.default_rng(3)
    ds.cdp_id = rng.permutation(40).astype(np.uint32)
    d = describe(ds, w.config, "d2", 125.0)
    np.testing.assert_array_equal(d.row_gather, oracle.row_order(ds.cdp_id, "d2"))
    for r in range(40):
        g = d.row_gather[r]
        legs = d.leg_gather[d.leg_off[r]:d.leg_off[r + 1]]
        assert legs[0] == g
        expect = neighbors_of(ds, g, range(40), 125.0)
        np.testing.assert_array_equal(legs[1:], expect)
        assert d.sweep_traces[r] == 30 * len(legs)


def test_describe_row_block():
    w = configs.crs_small()
    ds = w.spec.generate(count=40)
    full = describe(ds, w.config, "abc", w.apm, w.abc)
    part = describe(ds, w.config, "abc", w.apm, w.abc, rows=(10, 7))
    np.testing.assert_array_equal(part.row_gather, full.row_gather[10:17])
    np.testing.assert_array_equal(part.sweep_traces, full.sweep_traces[10:17])


def test_block_and_halo_shards():
    for n in (1, 7, 64, 1000):
        for world in (1, 2, 3, 8):
            blocks = [block_range(n, world, r) for r in range(world)]
            assert blocks[0][0] == 0 and blocks[-1][1] == n
            assert all(blocks[i][1] == blocks[i + 1][0] for i in range(world - 1))
            sizes = [e - b for b, e in blocks]
            assert max(sizes) - min(sizes) <= 1
    mx = np.arange(100, dtype=np.float64) * 12.5
    sh = line_shards(mx, 4, apm=125.0)
    assert sh[0].gathers == (0, 35) and sh[0].block == (0, 25)
    assert sh[1].gathers == (15, 60) and sh[1].row_first == 10 and sh[1].row_count == 25
    assert sh[3].gathers == (65, 100)
    ws = weak_shard(8192, 2, halo=10, world=4)
    assert ws.block == (16384, 24576) and ws.gathers == (16374, 24586)


def test_exact_quotient_predicate():
    """The FAST kernels skip hit_for's near-integer fix-up when the host
    proves double(t) / dt == t * N for every float t (velan_gpu.cu, `exact_q`:
    1/dt an integer N <= 2^20 and |dt N - 1| < 2^-54).  Restated here with
    exact rationals and checked by brute force: where the predicate holds the
    double quotient of traveltime.hpp:66-80 equals the exact product on two
    million float traveltimes (so floor and fraction of the product are the
    reference's), and the inexact sample intervals of the random GPU tests
    fail it (they keep the fix-up path)."""
    from fractions import Fraction

    def exact_q(dt_us):
        dt = float(dt_us) * 1e-6          # CdpGather::dt_seconds
        inv = 1.0 / dt
        n = float(np.rint(inv))
        return (inv == n and 1.0 <= n <= 1048576.0 and
                abs(Fraction(dt) * Fraction(n) - 1) < Fraction(1, 2 ** 54)), dt, n

    rng = np.random.default_rng(5)
    t = np.concatenate([rng.uniform(0.0, 16.0, 2_000_000),
                        rng.uniform(0.0, 1e-3, 100_000)]).astype(np.float32).astype(np.float64)
    for us in (125, 250, 500, 1000, 2000, 4000, 8000):
        ok, dt, n = exact_q(us)
        assert ok, us
        assert np.array_equal(t / dt, t * n), us
    for us in (244, 1500, 3333):
        assert not exact_q(us)[0], us
