"""Generate the golden fixtures in tests/golden/ from the UNMODIFIED reference.

Run in the build container (where /root/reference exists and oracle/_ref was
built by `make oracle`):

    python tests/golden/make_golden.py

Every output array comes from the reference library's own code path
(velan::scan_tile_blocked / scan_pair_baseline, velan::run_crs, velan::hit_for,
velan::crs_traveltime) through oracle/ref_shim.cpp; the inputs are seeded and
stored beside the outputs, so the fixtures pin the oracle and the GPU on any
machine without the reference.
"""
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.dirname(HERE))

import oracle  # noqa: E402
from helpers import random_gathers, reference_synthetic  # noqa: E402
from paper_1907_11678_b200 import configs, velocity_grid  # noqa: E402


def save(name, **arrays):
    path = os.path.join(HERE, name)
    np.savez_compressed(path, **arrays)
    print(f"wrote {path} ({os.path.getsize(path)} bytes)")


def ds_arrays(ds, prefix=""):
    return {prefix + "samples": ds.samples, prefix + "coords": ds.coords,
            prefix + "ntraces": ds.ntraces, prefix + "cdp_id": ds.cdp_id,
            prefix + "dt_us": np.array(ds.dt_us)}


def main():
    assert oracle.ref_available(), "build oracle/_ref first (make oracle)"

    # 1. random gathers, acceptance.cpp:71-134 shapes, w in {1,4,8,11,16}
    rng = np.random.default_rng(20260809)
    cases = {}
    for i, w in enumerate([1, 4, 8, 11, 16, 5]):
        fold = int(1 + rng.integers(0, 16))
        ns = int(48 + rng.integers(0, 150))
        nc = int(2 + rng.integers(0, 14))
        ds = random_gathers(rng, 2, fold, ns, 244, 10.0 + rng.integers(0, 40))
        v = velocity_grid(2000.0, 3000.0, nc)
        rows, ks = oracle.all_cells(2, ns)
        r = oracle.ref_run_cells(ds, "nmo", w, v, rows, ks, variant=1, matrix=True, workers=4)
        c = {**ds_arrays(ds), "w": np.array(w), "v": v, "matrix": r.matrix,
             "best_idx": r.best_idx, "best_semblance": r.best_semblance,
             "best_stack": r.best_stack, "valid": np.array(r.valid, np.uint64)}
        cases.update({f"c{i}_{k}": a for k, a in c.items()})
    save("random_gathers.npz", n_cases=np.array(6), **cases)

    # 2. two CMP-small gathers with the BASELINE slowness grid (101 C, w 11)
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=2)
    v = wl.config.grid()
    rows, ks = oracle.all_cells(2, ds.ns)
    r = oracle.ref_run_cells(ds, "nmo", 11, v, rows, ks, variant=1, matrix=True, workers=4)
    pick = np.arange(0, len(rows), 20)
    save("cmp_small_slice.npz", **ds_arrays(ds), v=v, w=np.array(11),
         best_idx=r.best_idx, best_semblance=r.best_semblance, best_stack=r.best_stack,
         matrix_cells=pick, matrix=r.matrix[pick], valid=np.array(r.valid, np.uint64))

    # 3. velan::run_crs on a 2x2 shard grid (test_oracle.cpp:67-89 shape)
    ds = reference_synthetic(25, 5, 160, 220, [(0.0132, 2500.0, 1.0)],
                             wavelet_freq=300.0, max_offset=100.0, cdp_spacing=12.5)
    code, msg, r = oracle.ref_run_pipeline(ds, "crs", 2000.0, 3000.0, 11, 4,
                                           grid=(2, 2), apm=12.5, workers=4)
    assert code == 0, msg
    save("crs_d2_run_crs.npz", **ds_arrays(ds), vmin=np.float32(2000.0),
         vmax=np.float32(3000.0), nc=np.array(11), w=np.array(4), apm=np.array(12.5),
         best_idx=r.best_idx, best_semblance=r.best_semblance, best_stack=r.best_stack,
         matrix=r.matrix, valid=np.array(r.valid, np.uint64))

    # 4. velan::run_cmp with the reference's own v-linear grid
    ds = reference_synthetic(2, 16, 200, 220, [(0.0154, 2500.0, 1.0), (0.033, 2700.0, 0.8)],
                             wavelet_freq=300.0, max_offset=160.0)
    code, msg, r = oracle.ref_run_pipeline(ds, "cmp", 2000.0, 3000.0, 101, 4, workers=2)
    assert code == 0, msg
    save("cmp_planted_run_cmp.npz", **ds_arrays(ds), vmin=np.float32(2000.0),
         vmax=np.float32(3000.0), nc=np.array(101), w=np.array(4),
         best_idx=r.best_idx, best_semblance=r.best_semblance, best_stack=r.best_stack,
         matrix=r.matrix, valid=np.array(r.valid, np.uint64))

    # 5. hit_for and crs_traveltime vectors
    rng = np.random.default_rng(99)
    out = {}
    for j, (dt, ns, w) in enumerate([(0.004, 1000, 11), (0.002, 2000, 15),
                                     (220e-6, 550, 4), (1.0 / 4096.0, 200, 3)]):
        k = rng.integers(0, ns, 4000)
        t = np.concatenate([(k * dt).astype(np.float32),
                            rng.uniform(0, ns * dt, 4000).astype(np.float32),
                            np.array([0.0, 1e-30, -1.0], np.float32)])
        k1, x, valid = oracle.hit_batch(t, dt, ns, w, ref=True)
        out.update({f"h{j}_t": t, f"h{j}_dt": np.array(dt), f"h{j}_ns": np.array(ns),
                    f"h{j}_w": np.array(w), f"h{j}_k1": k1, f"h{j}_x": x, f"h{j}_valid": valid})
    n = 5000
    t0 = rng.uniform(0, 4, n).astype(np.float32)
    h2 = rng.uniform(0, 2.5e6, n).astype(np.float32)
    d2 = rng.uniform(0, 4e4, n).astype(np.float32)
    v = rng.uniform(1000, 6000, n).astype(np.float32)
    tt = np.zeros(n, np.float32)
    oracle.ref_lib().vref_traveltime_batch(t0.ctypes.data, h2.ctypes.data, d2.ctypes.data,
                                           v.ctypes.data, n, tt.ctypes.data)
    save("hit_traveltime.npz", n_hit=np.array(4), tt_t0=t0, tt_h2=h2, tt_d2=d2, tt_v=v,
         tt_out=tt, **out)


if __name__ == "__main__":
    main()
