"""CPU parity checkers — TEST INFRASTRUCTURE ONLY.

Only tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / reference
legs may import this package, and only as the checker or the timed CPU
baseline.  The product path (paper_1907_11678_b200) never imports it.

Two libraries (built by oracle/Makefile):
  * libvelan_oracle.so  — semblance_oracle.c, a C restatement of the
    reference hot path (file:line citations in the source);
  * _ref/libvelan_ref.so — the UNMODIFIED reference headers
    (/root/reference/proj/include) compiled with the reference's flags and
    driven through ref_shim.cpp.  Absent on machines where it was never
    built; the GPU box receives the prebuilt copy with the repo snapshot.
"""
from __future__ import annotations

import ctypes as C
import os
from dataclasses import dataclass
from typing import Optional

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ORACLE_LIB = os.path.join(HERE, "libvelan_oracle.so")
SYNTH_LIB = os.path.join(HERE, "libvelan_synth.so")
REF_LIB = os.path.join(HERE, "_ref", "libvelan_ref.so")

OP = {"nmo": 0, "d2": 1, "abc": 2}
_P = C.c_void_p

_oracle = None
_ref = None
_synth = None


def _p(a):
    return 0 if a is None else a.ctypes.data


def oracle_lib() -> C.CDLL:
    global _oracle
    if _oracle is None:
        lib = C.CDLL(ORACLE_LIB)
        lib.vo_run_cells.restype = C.c_int
        lib.vo_run_cells.argtypes = [
            _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_int,
            C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, C.c_double, C.c_int,
            _P, _P, C.c_int, C.c_int, _P, _P, _P, _P, _P, _P]
        lib.vo_hit_batch.restype = None
        lib.vo_hit_batch.argtypes = [_P, C.c_int, C.c_double, C.c_int, C.c_int, _P, _P, _P]
        lib.vo_traveltime_batch.restype = None
        lib.vo_traveltime_batch.argtypes = [C.c_int, _P, _P, _P, _P, _P, _P, C.c_int, _P]
        lib.vo_finalize.restype = None
        lib.vo_finalize.argtypes = [_P, C.c_int, C.c_float, C.c_float, C.c_int, _P, _P]
        lib.vo_interpolate.restype = C.c_float
        lib.vo_interpolate.argtypes = [C.c_float, C.c_float, C.c_float]
        lib.vo_halfpoint.restype = C.c_float
        lib.vo_halfpoint.argtypes = [C.c_float] * 4
        lib.vo_nmo_correct.restype = None
        lib.vo_nmo_correct.argtypes = [_P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_uint32,
                                       C.c_int, _P, C.c_int, _P, _P]
        lib.vo_row_order.restype = None
        lib.vo_row_order.argtypes = [_P, C.c_int, C.c_int, _P]
        _oracle = lib
    return _oracle


def synth_lib() -> C.CDLL:
    """The seeded input generator (paper_1907_11678_b200/csrc/synth.cpp built
    without CUDA by oracle/Makefile) for the CPU-only arms: pass it to
    SynthSpec.generate(lib=...) to make inputs without loading the GPU
    library."""
    global _synth
    if _synth is None:
        from paper_1907_11678_b200 import _native as N
        lib = C.CDLL(SYNTH_LIB)
        for name in ("velan_gpu_synth_generate", "velan_gpu_synth_line_events"):
            res, args = N.SIGNATURES[name]
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _synth = lib
    return _synth


def ref_available() -> bool:
    return os.path.exists(REF_LIB)


def ref_lib() -> C.CDLL:
    global _ref
    if _ref is None:
        lib = C.CDLL(REF_LIB)
        lib.vref_last_error.restype = C.c_char_p
        lib.vref_run_cmp.restype = C.c_int
        lib.vref_run_cmp.argtypes = [
            _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_float,
            C.c_float, C.c_int, C.c_int, C.c_int, C.c_int, _P, _P, _P, _P, _P]
        lib.vref_run_crs.restype = C.c_int
        lib.vref_run_crs.argtypes = [
            _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_float,
            C.c_float, C.c_int, C.c_int, C.c_int, C.c_int, C.c_int, C.c_double,
            C.c_int, _P, _P, _P, _P, _P]
        lib.vref_run_cells.restype = C.c_int
        lib.vref_run_cells.argtypes = [
            _P, _P, _P, _P, C.c_int, C.c_int, C.c_int, C.c_uint32, C.c_int,
            C.c_int, C.c_int, _P, C.c_double, C.c_int, C.c_int, _P, _P, C.c_int,
            C.c_int, _P, _P, _P, _P, _P]
        lib.vref_dataset_create.restype = C.c_void_p
        lib.vref_dataset_create.argtypes = [_P, _P, _P, _P, C.c_int, C.c_int, C.c_int,
                                            C.c_uint32]
        lib.vref_dataset_destroy.restype = None
        lib.vref_dataset_destroy.argtypes = [_P]
        lib.vref_run_cells_ds.restype = C.c_int
        lib.vref_run_cells_ds.argtypes = [
            _P, C.c_int, C.c_int, C.c_int, _P, C.c_double, C.c_int, C.c_int, _P, _P,
            C.c_int, C.c_int, _P, _P, _P, _P, _P]
        lib.vref_hit_batch.restype = None
        lib.vref_hit_batch.argtypes = [_P, C.c_int, C.c_double, C.c_int, C.c_int, _P, _P, _P]
        lib.vref_traveltime_batch.restype = None
        lib.vref_traveltime_batch.argtypes = [_P, _P, _P, _P, C.c_int, _P]
        lib.vref_halfpoint_batch.restype = None
        lib.vref_halfpoint_batch.argtypes = [_P, C.c_int, _P]
        lib.vref_finalize.restype = None
        lib.vref_finalize.argtypes = [_P, C.c_int, C.c_float, C.c_float, C.c_int, _P, _P]
        lib.vref_interpolate.restype = C.c_float
        lib.vref_interpolate.argtypes = [C.c_float, C.c_float, C.c_float]
        lib.vref_write_dataset.restype = C.c_int
        lib.vref_write_dataset.argtypes = [C.c_char_p, _P, _P, _P, _P, C.c_int, C.c_int,
                                           C.c_int, C.c_uint32, C.c_char_p]
        lib.vref_read_dataset.restype = C.c_int
        lib.vref_read_dataset.argtypes = [C.c_char_p, _P, _P, _P, _P, _P, _P, _P]
        lib.vref_write_picks.restype = C.c_int
        lib.vref_write_picks.argtypes = [C.c_char_p, C.c_int, _P, C.c_int, C.c_int, _P, _P, _P]
        _ref = lib
    return _ref


@dataclass
class CellResult:
    best_idx: np.ndarray
    best_semblance: np.ndarray
    best_stack: np.ndarray
    matrix: Optional[np.ndarray]
    valid: int


def _flat(ds):
    return (np.ascontiguousarray(ds.samples, np.float32),
            np.ascontiguousarray(ds.coords, np.float32),
            np.ascontiguousarray(ds.ntraces, np.int32),
            np.ascontiguousarray(ds.cdp_id, np.uint32))


def all_cells(n_rows: int, ns: int):
    rows = np.repeat(np.arange(n_rows, dtype=np.int32), ns)
    ks = np.tile(np.arange(ns, dtype=np.int32), n_rows)
    return rows, ks


def run_cells(ds, op: str, w: int, v, rows, ks, apm: float = 0.0, abc=None,
              mode: int = 0, threads: int = 0, matrix: bool = False,
              stack_matrix: bool = False):
    """The C restatement over output cells (row, k).  mode 0 = kernel
    arithmetic (scan_pair_baseline order), 1 = oracle.hpp double sums,
    2 = the blocked trace-outer form (bitwise mode 0, ~25x faster on large
    sweeps: the checker for the big parity samples and the CPU port
    baseline), 3 = the literal BASELINE ABC formula in fp64 (the independent
    pin of the fp32 operator order)."""
    lib = oracle_lib()
    samples, coords, ntr, ids = _flat(ds)
    rows = np.ascontiguousarray(rows, np.int32)
    ks = np.ascontiguousarray(ks, np.int32)
    n = len(rows)
    if abc is not None:
        a, b, vv = (np.ascontiguousarray(x, np.float32) for x in (abc.a, abc.b, abc.v))
        ncand = len(a) * len(b) * len(vv)
    else:
        a = b = np.zeros(1, np.float32)
        vv = np.ascontiguousarray(v, np.float32)
        ncand = len(vv)
    bi = np.zeros(n, np.int32)
    bs = np.zeros(n, np.float32)
    bst = np.zeros(n, np.float32)
    mat = np.zeros((n, ncand), np.float32) if matrix else None
    smat = np.zeros((n, ncand), np.float32) if stack_matrix else None
    valid = C.c_uint64(0)
    if threads <= 0:
        threads = os.cpu_count() or 1
    G, M, ns = samples.shape
    code = lib.vo_run_cells(
        _p(samples), _p(coords), _p(ntr), _p(ids), G, M, ns, int(ds.dt_us),
        OP[op], int(w), len(a), len(b), len(vv), _p(a), _p(b), _p(vv),
        float(apm), int(mode), _p(rows), _p(ks), n, int(threads), _p(bi),
        _p(bs), _p(bst), _p(mat), _p(smat), C.addressof(valid))
    if code != 0:
        raise ValueError("oracle: invalid configuration")
    out = CellResult(bi, bs, bst, mat, int(valid.value))
    out.stack_matrix = smat
    return out


def nmo_correct(ds, op: str, v, picks) -> np.ndarray:
    """vo_nmo_correct: the corrected gathers [G, M, ns] of all rows."""
    lib = oracle_lib()
    samples, coords, ntr, ids = _flat(ds)
    G, M, ns = samples.shape
    vv = np.ascontiguousarray(v, np.float32)
    picks = np.ascontiguousarray(picks, np.int32)
    out = np.zeros((G, M, ns), np.float32)
    lib.vo_nmo_correct(_p(samples), _p(coords), _p(ntr), _p(ids), G, M, ns, int(ds.dt_us),
                       OP[op], _p(vv), len(vv), _p(picks), _p(out))
    return out


def ref_run_cells(ds, op: str, w: int, v, rows, ks, apm: float = 0.0,
                  variant: int = 1, mode: int = 0, workers: int = 0,
                  matrix: bool = False):
    """The reference's own kernels (variant 0 baseline / 1 blocked / 2 simd)
    or oracle::semblance_reference (mode 1) over output cells."""
    lib = ref_lib()
    samples, coords, ntr, ids = _flat(ds)
    rows = np.ascontiguousarray(rows, np.int32)
    ks = np.ascontiguousarray(ks, np.int32)
    n = len(rows)
    vv = np.ascontiguousarray(v, np.float32)
    bi = np.zeros(n, np.int32)
    bs = np.zeros(n, np.float32)
    bst = np.zeros(n, np.float32)
    mat = np.zeros((n, len(vv)), np.float32) if matrix else None
    naive = C.c_uint64(0)
    if workers <= 0:
        workers = os.cpu_count() or 1
    G, M, ns = samples.shape
    code = lib.vref_run_cells(
        _p(samples), _p(coords), _p(ntr), _p(ids), G, M, ns, int(ds.dt_us),
        OP[op], int(w), len(vv), _p(vv), float(apm), int(variant), int(mode),
        _p(rows), _p(ks), n, int(workers), _p(bi), _p(bs), _p(bst), _p(mat),
        C.addressof(naive))
    if code != 0:
        raise RuntimeError(f"reference: code {code}: {lib.vref_last_error().decode()}")
    return CellResult(bi, bs, bst, mat, int(naive.value))


class RefDataset:
    """A velan::Dataset built once from flat arrays (the reference's own
    container, types.hpp:14-54), reused across ref_run_cells calls so the
    per-trace vector copies stay out of timed regions."""

    def __init__(self, ds):
        samples, coords, ntr, ids = _flat(ds)
        G, M, ns = samples.shape
        self.G, self.ns, self.dt_us = G, ns, int(ds.dt_us)
        self.samples_abs_max = float(np.abs(samples).max()) if samples.size else 0.0
        self._h = ref_lib().vref_dataset_create(_p(samples), _p(coords), _p(ntr), _p(ids),
                                                G, M, ns, int(ds.dt_us))
        if not self._h:
            raise RuntimeError(ref_lib().vref_last_error().decode())

    def close(self):
        if getattr(self, "_h", None):
            ref_lib().vref_dataset_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ref_run_cells_ds(rds: RefDataset, op: str, w: int, v, rows, ks, apm: float = 0.0,
                     variant: int = 1, mode: int = 0, workers: int = 0,
                     matrix: bool = False):
    """ref_run_cells on a prebuilt RefDataset."""
    lib = ref_lib()
    rows = np.ascontiguousarray(rows, np.int32)
    ks = np.ascontiguousarray(ks, np.int32)
    n = len(rows)
    vv = np.ascontiguousarray(v, np.float32)
    bi = np.zeros(n, np.int32)
    bs = np.zeros(n, np.float32)
    bst = np.zeros(n, np.float32)
    mat = np.zeros((n, len(vv)), np.float32) if matrix else None
    naive = C.c_uint64(0)
    if workers <= 0:
        workers = os.cpu_count() or 1
    code = lib.vref_run_cells_ds(rds._h, OP[op], int(w), len(vv), _p(vv), float(apm),
                                 int(variant), int(mode), _p(rows), _p(ks), n, int(workers),
                                 _p(bi), _p(bs), _p(bst), _p(mat), C.addressof(naive))
    if code != 0:
        raise RuntimeError(f"reference: code {code}: {lib.vref_last_error().decode()}")
    return CellResult(bi, bs, bst, mat, int(naive.value))


def ref_run_pipeline(ds, kind: str, vmin: float, vmax: float, nc: int, w: int,
                     variant: int = 1, workers: int = 1, grid=(1, 1),
                     apm: float = 0.0, matrix: bool = True):
    """velan::run_cmp / velan::run_crs verbatim (v-linear grid).  Returns
    (code, message, CellResult-like arrays shaped [G, ns])."""
    lib = ref_lib()
    samples, coords, ntr, ids = _flat(ds)
    G = samples.shape[0]
    M = samples.shape[1] if G else 1
    ns = samples.shape[2] if G else 0
    bi = np.zeros((G, ns), np.int32)
    bs = np.zeros((G, ns), np.float32)
    bst = np.zeros((G, ns), np.float32)
    mat = np.zeros((G, ns, nc), np.float32) if matrix and nc > 0 else None
    naive = C.c_uint64(0)
    if kind == "cmp":
        code = lib.vref_run_cmp(_p(samples), _p(coords), _p(ntr), _p(ids), G, M,
                                ns, int(ds.dt_us), vmin, vmax, nc, w, variant,
                                workers, _p(bi), _p(bs), _p(bst), _p(mat),
                                C.addressof(naive))
    else:
        code = lib.vref_run_crs(_p(samples), _p(coords), _p(ntr), _p(ids), G, M,
                                ns, int(ds.dt_us), vmin, vmax, nc, w, variant,
                                grid[0], grid[1], float(apm), workers, _p(bi),
                                _p(bs), _p(bst), _p(mat), C.addressof(naive))
    msg = lib.vref_last_error().decode() if code else ""
    return code, msg, CellResult(bi, bs, bst, mat, int(naive.value))


def hit_batch(t, dt_s: float, ns: int, w: int, ref: bool = False):
    t = np.ascontiguousarray(t, np.float32)
    n = len(t)
    k1 = np.zeros(n, np.int32)
    x = np.zeros(n, np.float32)
    valid = np.zeros(n, np.uint8)
    if ref:
        ref_lib().vref_hit_batch(_p(t), n, dt_s, ns, w, _p(k1), _p(x), _p(valid))
    else:
        oracle_lib().vo_hit_batch(_p(t), n, dt_s, ns, w, _p(k1), _p(x), _p(valid))
    return k1, x, valid.astype(bool)


def row_order(cdp_id, op: str):
    ids = np.ascontiguousarray(cdp_id, np.uint32)
    out = np.zeros(len(ids), np.int32)
    oracle_lib().vo_row_order(_p(ids), len(ids), OP[op], _p(out))
    return out


def compare(run_matrix, ref_matrix):
    """oracle::compare (oracle.hpp:183-230) over [cells, ncand] matrices:
    max / mean relative error (floor 1e-12), argmax mismatches, and the
    mismatches excused because the reference's top two are within 1e-4."""
    a = np.asarray(run_matrix, np.float64)
    b = np.asarray(ref_matrix, np.float64)
    rel = np.abs(a - b) / np.maximum(np.abs(b), 1e-12)
    ra = np.argmax(np.asarray(run_matrix), axis=-1)
    rb = np.argmax(np.asarray(ref_matrix), axis=-1)
    mism = ra != rb
    excused = 0
    unexcused = 0
    if mism.any():
        bm = np.asarray(ref_matrix)[mism]
        top2 = -np.sort(-bm, axis=-1)[:, :2]
        gap = np.abs(top2[:, 0].astype(np.float64) - top2[:, 1]) / np.maximum(
            np.abs(top2[:, 0].astype(np.float64)), 1e-12)
        excused = int((gap < 1e-4).sum())
        unexcused = int((gap >= 1e-4).sum())
    return {"max_rel_err": float(rel.max()) if rel.size else 0.0,
            "mean_rel_err": float(rel.mean()) if rel.size else 0.0,
            "cells": int(rel.size), "argmax_mismatches": unexcused,
            "tie_excused": excused}


# --------------------------------------------------------------------------
# the reference's file formats (io.hpp), for byte-identity tests of the
# native SSF1/SMB1 reader and writers

def ref_write_dataset(ds, path: str, metadata: str = "") -> None:
    """velan::write_dataset (io.hpp:95-122)."""
    sm, co, nt, ids = _flat(ds)
    G, M, ns = sm.shape
    code = ref_lib().vref_write_dataset(str(path).encode(), _p(sm), _p(co), _p(nt), _p(ids),
                                        G, M, ns, int(ds.dt_us), metadata.encode())
    if code:
        raise RuntimeError(ref_lib().vref_last_error().decode())


def ref_read_dataset(path: str):
    """velan::read_dataset (io.hpp:124-166) -> (samples, coords, ntraces,
    cdp_id, dt_us, metadata); raises ValueError(format_error message)."""
    lib = ref_lib()
    dims = np.zeros(4, np.int32)
    ml = C.c_uint64(0)
    code = lib.vref_read_dataset(str(path).encode(), _p(dims), C.byref(ml), None, None, None,
                                 None, None)
    if code == 1:
        raise ValueError(lib.vref_last_error().decode())
    if code:
        raise RuntimeError(lib.vref_last_error().decode())
    G, M, ns, dt = (int(x) for x in dims)
    sm = np.zeros((G, M, ns), np.float32)
    co = np.zeros((G, M, 4), np.float32)
    nt = np.zeros(G, np.int32)
    ids = np.zeros(G, np.uint32)
    meta = C.create_string_buffer(max(ml.value, 1))
    code = lib.vref_read_dataset(str(path).encode(), _p(dims), C.byref(ml), _p(sm), _p(co),
                                 _p(nt), _p(ids), meta)
    if code:
        raise RuntimeError(lib.vref_last_error().decode())
    return sm, co, nt, ids, dt, meta.raw[:ml.value].decode()


def ref_write_picks(path: str, cdp_id, velocity, semblance, nc: int, matrix=None) -> None:
    """velan::write_picks (io.hpp:170-194)."""
    ids = np.ascontiguousarray(cdp_id, np.uint32)
    vel = np.ascontiguousarray(velocity, np.float32)
    sem = np.ascontiguousarray(semblance, np.float32)
    mat = None if matrix is None else np.ascontiguousarray(matrix, np.float32)
    n, ns = vel.shape
    code = ref_lib().vref_write_picks(str(path).encode(), n, _p(ids), ns, nc, _p(vel), _p(sem),
                                      _p(mat))
    if code:
        raise RuntimeError(ref_lib().vref_last_error().decode())
