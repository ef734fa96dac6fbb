"""The oracle's fast and independent modes (CPU only).

* mode 2 — the blocked, trace-outer restatement (scan_tile_blocked's loop
  nest, kernel.hpp:276-316) — must be bitwise equal to mode 0
  (scan_pair_baseline order) on every operator, ragged and non-finite data;
  it is the checker of the large parity samples and the CPU port baseline.
* mode 3 — the literal BASELINE ABC formula in fp64 — pins the fp32 operator
  order shared by the restatement and the kernels: on CRS
  small, identical picks except near-ties and semblance within 1e-4 relative
  at the picks.
* The reference's dataset handle (built once, reused) and the host-only build
  of the input generator agree with the one-shot paths bitwise.
"""
import numpy as np
import pytest

import oracle
from helpers import random_gathers
from paper_1907_11678_b200 import CrsAbcGrid, Dataset, configs

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
RTOL = 1e-4


def _bits(a):
    """Bit patterns with NaNs canonicalised (the payload/sign of a NaN is the
    compiler's operand order, not arithmetic — the reference makes no promise
    about it)."""
    a = np.array(a, np.float32)
    a[np.isnan(a)] = np.float32("nan")
    return a.view(np.uint32)


def _same(a, b):
    np.testing.assert_array_equal(_bits(a.matrix), _bits(b.matrix))
    np.testing.assert_array_equal(_bits(a.stack_matrix), _bits(b.stack_matrix))
    np.testing.assert_array_equal(a.best_idx, b.best_idx)
    np.testing.assert_array_equal(_bits(a.best_semblance), _bits(b.best_semblance))
    np.testing.assert_array_equal(_bits(a.best_stack), _bits(b.best_stack))
    assert a.valid == b.valid


def _both(ds, op, w, v, rows, ks, **kw):
    a = oracle.run_cells(ds, op, w, v, rows, ks, mode=0, matrix=True, stack_matrix=True, **kw)
    b = oracle.run_cells(ds, op, w, v, rows, ks, mode=2, matrix=True, stack_matrix=True, **kw)
    return a, b


def test_blocked_equals_kernel_order_cmp():
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=6)
    rng = np.random.default_rng(3)
    rows = rng.integers(0, 6, 500).astype(np.int32)
    ks = rng.integers(0, ds.ns, 500).astype(np.int32)
    _same(*_both(ds, "nmo", wl.config.w, wl.config.grid(), rows, ks))


def test_blocked_equals_kernel_order_crs_abc_and_d2():
    wl = configs.crs_small()
    ds = wl.spec.generate(count=20)
    rng = np.random.default_rng(4)
    rows = rng.integers(0, 20, 60).astype(np.int32)
    ks = rng.integers(0, ds.ns, 60).astype(np.int32)
    abc = CrsAbcGrid(wl.abc.a[::3], wl.abc.b[::3], wl.abc.v[::2])
    _same(*_both(ds, "abc", wl.config.w, None, rows, ks, apm=wl.apm, abc=abc))
    _same(*_both(ds, "d2", wl.config.w, wl.config.grid(), rows, ks, apm=wl.apm))


@pytest.mark.parametrize("w", [1, 4, 11, 16, 32])
def test_blocked_equals_kernel_order_ragged_nonfinite(w):
    """Ragged trace counts (NaN in the padding the reference does not have),
    NaN and Inf samples inside traces, every window length class."""
    rng = np.random.default_rng(100 + w)
    ds = random_gathers(rng, 5, 9, 300, dt_us=2000, max_offset=900.0)
    ds.ntraces[:] = [9, 1, 4, 7, 9]
    for g in range(5):
        ds.samples[g, ds.ntraces[g]:] = np.nan
    ds.samples[3, 2, 40:44] = np.nan
    ds.samples[4, 5, 100] = np.inf
    v = np.linspace(1500, 4000, 23).astype(np.float32)
    rows = np.repeat(np.arange(5, dtype=np.int32), 40)
    ks = np.tile(np.arange(0, 300, 300 // 40, dtype=np.int32)[:40], 5)
    _same(*_both(ds, "nmo", w, v, rows, ks))
    ds.coords[:, :, 0] += (np.arange(5, dtype=np.float32) * 30.0)[:, None]
    ds.coords[:, :, 2] += (np.arange(5, dtype=np.float32) * 30.0)[:, None]
    abc = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 2), v[::4])
    _same(*_both(ds, "abc", w, None, rows, ks, apm=65.0, abc=abc))


def test_f64_literal_formula_pins_the_abc_order():
    """CRS small, 400 seeded cells, all 2541 candidates: the restated fp32
    operator order (t0^2 + fma(2 t0, beta, gamma), shared with the kernels)
    against the literal BASELINE formula (t0 + 2A dm)^2 + 2 t0 (B dm^2 +
    C h^2), C = 2/(t0 v^2), evaluated and summed in fp64."""
    wl = configs.crs_small()
    ds = wl.spec.generate()
    rng = np.random.default_rng(7)
    rows = rng.integers(0, 256, 400).astype(np.int32)
    ks = rng.integers(0, ds.ns, 400).astype(np.int32)
    lit = oracle.run_cells(ds, "abc", wl.config.w, None, rows, ks, apm=wl.apm, abc=wl.abc,
                           mode=3, matrix=True)
    f32 = oracle.run_cells(ds, "abc", wl.config.w, None, rows, ks, apm=wl.apm, abc=wl.abc,
                           mode=2)
    m = lit.matrix.astype(np.float64)
    top2 = -np.sort(-m, axis=1)[:, :2]
    gap = np.abs(top2[:, 0] - top2[:, 1]) / np.maximum(np.abs(top2[:, 0]), 1e-12)
    same = f32.best_idx == lit.best_idx
    assert np.all(same | (gap < RTOL)), int((~same & (gap >= RTOL)).sum())
    at = m[np.arange(len(rows)), f32.best_idx]
    rel = np.abs(f32.best_semblance - at) / np.maximum(np.abs(at), 1e-12)
    assert rel.max() <= RTOL, float(rel.max())


def test_f64_literal_formula_reduces_to_nmo():
    """dm = 0 (CMP gathers) — the literal formula is NMO in fp64: picks equal
    the reference-order NMO scan except near-ties."""
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=4)
    rows, ks = oracle.all_cells(4, ds.ns)
    lit = oracle.run_cells(ds, "nmo", wl.config.w, wl.config.grid(), rows, ks, mode=3,
                           matrix=True)
    ref = oracle.run_cells(ds, "nmo", wl.config.w, wl.config.grid(), rows, ks, mode=2)
    rep = oracle.compare(ref.best_semblance[:, None], lit.matrix[np.arange(len(rows)),
                                                                 ref.best_idx][:, None])
    assert rep["max_rel_err"] <= RTOL
    m = lit.matrix.astype(np.float64)
    top2 = -np.sort(-m, axis=1)[:, :2]
    gap = np.abs(top2[:, 0] - top2[:, 1]) / np.maximum(np.abs(top2[:, 0]), 1e-12)
    assert np.all((ref.best_idx == lit.best_idx) | (gap < RTOL))


def test_oracle_rejects_cells_outside_the_dataset():
    ds = configs.cmp_small().spec.generate(count=2)
    with pytest.raises(ValueError):
        oracle.run_cells(ds, "nmo", 11, configs.cmp_small().config.grid(), [2], [0], mode=2)
    with pytest.raises(ValueError):
        oracle.run_cells(ds, "nmo", 11, configs.cmp_small().config.grid(), [0], [ds.ns])


@needs_ref
def test_reference_dataset_handle_matches_one_shot():
    wl = configs.crs_small()
    ds = wl.spec.generate(count=16)
    v = np.linspace(1500, 3500, 40).astype(np.float32)
    rows = np.array([3, 3, 8, 12], np.int32)
    ks = np.array([100, 400, 700, 950], np.int32)
    rds = oracle.RefDataset(ds)
    a = oracle.ref_run_cells_ds(rds, "d2", 11, v, rows, ks, apm=wl.apm, matrix=True)
    b = oracle.ref_run_cells(ds, "d2", 11, v, rows, ks, apm=wl.apm, matrix=True)
    np.testing.assert_array_equal(_bits(a.matrix), _bits(b.matrix))
    assert a.valid == b.valid
    # the reference's blocked kernel on d2 == the restatement's d2 (mode 2)
    c = oracle.run_cells(ds, "d2", 11, v, rows, ks, apm=wl.apm, mode=2, matrix=True)
    np.testing.assert_array_equal(_bits(a.matrix), _bits(c.matrix))
    with pytest.raises(RuntimeError):
        oracle.ref_run_cells_ds(rds, "d2", 11, v, [16], [0], apm=wl.apm)
    rds.close()


def test_host_generator_build_matches_gpu_library_build():
    """oracle/libvelan_synth.so (synth.cpp without CUDA, for the CPU-only
    arms) generates the same bits as the GPU library's generator."""
    for f in (configs.cmp_large, configs.crs_small):
        wl = f()
        a = wl.spec.generate(first=5, count=4)
        b = wl.spec.generate(first=5, count=4, lib=oracle.synth_lib())
        np.testing.assert_array_equal(_bits(a.samples), _bits(b.samples))
        np.testing.assert_array_equal(a.coords, b.coords)
        np.testing.assert_array_equal(a.cdp_id, b.cdp_id)
