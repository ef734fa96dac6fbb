"""Test fixtures restating the reference's test helpers
(/root/reference/proj/tests/helpers.hpp, test_cmp_pipeline.cpp) in numpy."""
import math

import numpy as np

from paper_1907_11678_b200 import Dataset


def make_gather(rows, dt_us, half_offset=0.0, cdp_id=0):
    """testutil::make_gather (helpers.hpp:16-30): traces given as sample
    rows; sources at the origin, receivers at 2*half_offset along x."""
    rows = np.asarray(rows, np.float32)
    M, ns = rows.shape
    coords = np.zeros((1, M, 4), np.float32)
    coords[0, :, 2] = 2.0 * half_offset
    return Dataset(rows[None], coords, np.array([M], np.int32),
                   np.array([cdp_id], np.uint32), dt_us)


def random_gathers(rng, n, fold, ns, dt_us=244, max_offset=100.0):
    """testutil::random_gather (helpers.hpp:32-55): U[-1, 1] samples,
    offsets spread over [0, max_offset] (receiver x; source at 0)."""
    samples = rng.uniform(-1.0, 1.0, (n, fold, ns)).astype(np.float32)
    coords = np.zeros((n, fold, 4), np.float32)
    off = (np.zeros(fold) if fold == 1 else
           (max_offset * np.arange(fold, dtype=np.float32) / np.float32(fold - 1)))
    coords[:, :, 2] = np.asarray(off, np.float32)[None, :]
    return Dataset(samples, coords, np.full(n, fold, np.int32),
                   np.arange(n, dtype=np.uint32), dt_us)


def reference_synthetic(ncdps, fold, ns, dt_us, events, wavelet_freq=25.0,
                        max_offset=200.0, cdp_spacing=25.0):
    """generate_synthetic (synthetic.hpp:80-163) for snr = 0 (noiseless, so
    no RNG): midpoints on a ceil(sqrt(n)) grid, half-offsets 0..max/2,
    one Ricker per event at the fp32 NMO traveltime."""
    dt = dt_us * 1e-6
    grid_nx = int(math.ceil(math.sqrt(ncdps)))
    support = 4.0 / wavelet_freq
    samples = np.zeros((ncdps, fold, ns), np.float32)
    coords = np.zeros((ncdps, fold, 4), np.float32)
    for i in range(ncdps):
        mx = np.float32((i % grid_nx) * cdp_spacing)
        my = np.float32((i // grid_nx) * cdp_spacing)
        for m in range(fold):
            half = np.float32(0.0 if fold == 1 else 0.5 * max_offset * m / (fold - 1))
            coords[i, m] = (mx - half, my, mx + half, my)
            h2 = np.float32(half * half)
            for (t0, v, amp) in events:
                t0f, vf = np.float32(t0), np.float32(v)
                t_ev = float(np.sqrt(t0f * t0f + (np.float32(4.0) * h2) / (vf * vf)))
                lo = max(0, int(math.floor((t_ev - support) / dt)))
                hi = min(ns, int(math.ceil((t_ev + support) / dt)) + 1)
                for s in range(lo, hi):
                    tau = s * dt - t_ev
                    a = math.pi * wavelet_freq * tau
                    samples[i, m, s] += np.float32(amp * (1 - 2 * a * a) * math.exp(-a * a))
    return Dataset(samples, coords, np.full(ncdps, fold, np.int32),
                   np.arange(ncdps, dtype=np.uint32), dt_us)


def line_dataset(seed, G=10, M=9, ns=240, dt_us=4000, dx=25.0, ragged=True,
                 poison_padding=True):
    """A 2-D line of G midpoints dx apart, M half-offsets 50..50M m, U[-1, 1]
    samples; with ragged=True gather g keeps a random 1..M traces (gather 0
    keeps M) and the padding slots hold NaN."""
    rng = np.random.default_rng(seed)
    samples = rng.uniform(-1.0, 1.0, (G, M, ns)).astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    mx = (dx * np.arange(G)).astype(np.float32)
    h = (50.0 * np.arange(1, M + 1)).astype(np.float32)
    coords[:, :, 0] = mx[:, None] - h[None, :]   # sx
    coords[:, :, 2] = mx[:, None] + h[None, :]   # gx
    ntr = np.full(G, M, np.int32)
    if ragged:
        ntr = rng.integers(1, M + 1, G).astype(np.int32)
        ntr[0] = M
        ntr[G // 2] = 1
        for g in range(G):
            if poison_padding:
                samples[g, ntr[g]:] = np.nan
            # the padding's coordinates repeat the first trace's: the
            # midpoint (types.hpp:57-62) is read from trace 0 only
            coords[g, ntr[g]:] = coords[g, 0]
    return Dataset(samples, coords, ntr, np.arange(G, dtype=np.uint32), dt_us)


def poison_samples(ds, seed, count):
    """NaN at `count` seeded (gather, trace, sample) positions inside the
    gathers' real traces."""
    rng = np.random.default_rng(seed)
    for _ in range(count):
        g = int(rng.integers(0, ds.ncdps))
        m = int(rng.integers(0, ds.ntraces[g]))
        ds.samples[g, m, int(rng.integers(0, ds.ns))] = np.nan
    return ds
