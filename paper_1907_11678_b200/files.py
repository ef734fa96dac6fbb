"""SSF1 trace files and SMB1 pick files, over the native
reader/writer of include/velan_gpu.h.

Mirrors the reference's file API (io.hpp):

* ``read_ssf1(path)``          read_dataset  (io.hpp:124-166) -> Dataset
* ``write_ssf1(ds, path)``     write_dataset (io.hpp:95-122), byte-identical
* ``write_smb1(results, path)`` write_picks   (io.hpp:170-194), byte-identical
* ``read_smb1(path)``          read_picks    (io.hpp:196-224)

plus the streaming pieces the GPU pipeline needs: ``SSF1Reader`` (index the
file once, read gather blocks straight into the flattened — optionally
pinned — layout) and ``SMB1Writer`` (append pick records block by block).
``Engine.run_cmp_file`` (below) chains them: reading block i+1 and writing
block i-1 overlap the scan of block i.
"""
from __future__ import annotations

import ctypes as C
import json
import struct
import threading
from dataclasses import dataclass
from typing import Iterable, Optional, Sequence

import numpy as np

from . import _native as N
from .api import (ConfigError, Dataset, Engine, ParameterError, ScanConfig,
                  ScanResult, VelanError, _dataset_struct, _ptr, _raise)


class FormatError(ConfigError):
    """velan::format_error (error.hpp): malformed file, message carries the
    byte offset."""


def _check(code: int, where: str) -> None:
    if code == N.ECONFIG:
        raise FormatError(f"{where}: {N.last_error()}")
    _raise(code, where)


def _alloc(shape, dtype, pinned: bool):
    if not pinned:
        return np.zeros(shape, dtype)
    import torch
    t = torch.zeros(shape, dtype={np.float32: torch.float32}[np.dtype(dtype).type]).pin_memory()
    return t.numpy()


class SSF1Reader:
    """An indexed SSF1 file: header words of every gather, samples read on
    demand into [count, fold, ns] blocks."""

    def __init__(self, path: str):
        lib = N.load()
        h = C.c_void_p()
        info = N.SSF1Info()
        _check(lib.velan_ssf1_open(str(path).encode(), C.byref(h), C.byref(info)),
               "velan_ssf1_open")
        self._h = h
        self.path = str(path)
        self.n_gathers = int(info.n_gathers)
        self.fold = int(info.fold)
        self.ns = int(info.ns)
        self.dt_us = int(info.dt_us)
        self.uniform = bool(info.uniform)
        G = self.n_gathers
        self.cdp_id = np.zeros(G, np.uint32)
        self.ntraces = np.zeros(G, np.int32)
        self.ns_per_gather = np.zeros(G, np.uint32)
        self.dt_per_gather = np.zeros(G, np.uint32)
        _check(lib.velan_ssf1_gathers(h, _ptr(self.cdp_id), _ptr(self.ntraces),
                                      _ptr(self.ns_per_gather), _ptr(self.dt_per_gather)),
               "velan_ssf1_gathers")
        buf = C.create_string_buffer(max(int(info.metadata_bytes), 1))
        _check(lib.velan_ssf1_metadata(h, buf, int(info.metadata_bytes)), "velan_ssf1_metadata")
        self.metadata_json = buf.raw[:int(info.metadata_bytes)].decode("utf-8", "replace")

    def read(self, first: int = 0, count: Optional[int] = None, *, pinned: bool = False,
             out: Optional[tuple] = None, threads: int = 0) -> Dataset:
        """Gathers [first, first + count) as a Dataset (fold = the file's)."""
        if count is None:
            count = self.n_gathers - first
        if out is not None:
            samples, coords = out
            samples = samples[:count]
            coords = coords[:count]
        else:
            samples = _alloc((count, self.fold, self.ns), np.float32, pinned)
            coords = _alloc((count, self.fold, 4), np.float32, pinned)
        _check(N.load().velan_ssf1_read(self._h, first, count, self.fold, _ptr(samples),
                                        _ptr(coords), threads), "velan_ssf1_read")
        ds = Dataset(samples, coords, self.ntraces[first:first + count].copy(),
                     self.cdp_id[first:first + count].copy(), self.dt_us)
        if self.metadata_json:
            try:
                ds.metadata = json.loads(self.metadata_json)
            except ValueError:
                ds.metadata = {"raw": self.metadata_json}
        return ds

    def close(self):
        if getattr(self, "_h", None):
            N.load().velan_ssf1_close(self._h)
            self._h = None

    def __enter__(self):
        return self

    def __exit__(self, *a):
        self.close()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def read_ssf1(path: str, threads: int = 0) -> Dataset:
    """read_dataset (io.hpp:124-166) into the flattened layout."""
    with SSF1Reader(path) as r:
        return r.read(threads=threads)


def _metadata_bytes(ds: Dataset, metadata) -> bytes:
    if metadata is None:
        metadata = ds.metadata
    if isinstance(metadata, (bytes, bytearray)):
        return bytes(metadata)
    if isinstance(metadata, str):
        return metadata.encode()
    return json.dumps(metadata, sort_keys=True).encode() if metadata else b""


def write_ssf1(ds: Dataset, path: str, metadata=None) -> None:
    """write_dataset (io.hpp:95-122); the metadata tail is ``metadata`` (str,
    bytes or a JSON-able dict), default ds.metadata."""
    meta = _metadata_bytes(ds, metadata)
    dss = _dataset_struct(ds)
    _check(N.load().velan_ssf1_write(str(path).encode(), C.byref(dss), meta, len(meta)),
           "velan_ssf1_write")


class SMB1Writer:
    """write_picks (io.hpp:170-194) as a stream of record blocks."""

    def __init__(self, path: str, n_cdps: int, ns: int, nc: int, with_matrix: bool = False):
        h = C.c_void_p()
        _check(N.load().velan_smb1_begin(str(path).encode(), n_cdps, ns, nc,
                                         1 if with_matrix else 0, C.byref(h)),
               "velan_smb1_begin")
        self._h = h
        self.ns, self.nc, self.with_matrix = ns, nc, with_matrix

    def append(self, cdp_id, velocity, semblance, matrix=None) -> None:
        cdp = np.ascontiguousarray(cdp_id, np.uint32)
        vel = np.ascontiguousarray(velocity, np.float32)
        sem = np.ascontiguousarray(semblance, np.float32)
        mat = None if matrix is None else np.ascontiguousarray(matrix, np.float32)
        _check(N.load().velan_smb1_append(self._h, len(cdp), _ptr(cdp), _ptr(vel), _ptr(sem),
                                          _ptr(mat)), "velan_smb1_append")

    def append_result(self, res: ScanResult) -> None:
        self.append(res.cdp_id, res.best_velocity, res.best_semblance,
                    res.values if self.with_matrix else None)

    def close(self) -> None:
        if getattr(self, "_h", None):
            h, self._h = self._h, None
            _check(N.load().velan_smb1_end(h), "velan_smb1_end")

    def __enter__(self):
        return self

    def __exit__(self, exc_type, *a):
        if exc_type is None:
            self.close()
        elif getattr(self, "_h", None):  # error path: close, keep the first error
            h, self._h = self._h, None
            N.load().velan_smb1_end(h)


def write_smb1(results: Sequence[ScanResult] | ScanResult, path: str,
               include_matrix: bool = False) -> None:
    """write_picks (io.hpp:170-194) of scan results (one record per row)."""
    if isinstance(results, ScanResult):
        results = [results]
    n = sum(len(r) for r in results)
    ns = results[0].best_idx.shape[1] if results else 0
    nc = (results[0].n_candidates or len(results[0].candidates)) if results else 0
    with SMB1Writer(path, n, ns, nc, include_matrix) as w:
        for r in results:
            if include_matrix and r.values is None:
                raise ParameterError("write_smb1: include_matrix needs results with values")
            w.append_result(r)


@dataclass
class PickRecord:
    """One SMB1 record (SemblanceMatrix fields that SMB1 carries)."""
    cdp_id: int
    ns: int
    nc: int
    velocity: np.ndarray
    semblance: np.ndarray
    values: Optional[np.ndarray] = None


def read_smb1(path: str) -> list:
    """read_picks (io.hpp:196-224)."""
    data = open(path, "rb").read()
    if data[:4] != b"SMB1":
        raise FormatError("bad magic, expected SMB1 at byte 0")
    if len(data) < 16:
        raise FormatError("truncated file reading header at byte 4")
    version, ncdps, flags = struct.unpack_from("<III", data, 4)
    if version != 1:
        raise FormatError(f"unsupported version {version} at byte 4")
    off = 16
    out = []
    for _ in range(ncdps):
        if len(data) - off < 12:
            raise FormatError(f"truncated file reading record at byte {off}")
        cdp, ns, nc = struct.unpack_from("<III", data, off)
        off += 12
        need = 8 * ns + (4 * ns * nc if flags & 1 else 0)
        if len(data) - off < need:
            raise FormatError(f"truncated file reading picks at byte {off}")
        pv = np.frombuffer(data, "<f4", 2 * ns, off).reshape(ns, 2)
        off += 8 * ns
        vals = None
        if flags & 1:
            vals = np.frombuffer(data, "<f4", ns * nc, off).reshape(ns, nc).copy()
            off += 4 * ns * nc
        out.append(PickRecord(cdp, ns, nc, pv[:, 0].copy(), pv[:, 1].copy(), vals))
    if off != len(data):
        raise FormatError(f"trailing bytes at byte {off}")
    return out


# --------------------------------------------------------------------------
# streaming file -> GPU -> file pipeline (CMP)

def _blocks(n: int, block: int) -> Iterable[tuple]:
    for s in range(0, n, block):
        yield s, min(block, n - s)


def run_cmp_file(engine: Engine, ssf_path: str, config: ScanConfig,
                 smb_path: Optional[str] = None, block: int = 1024,
                 threads: int = 0, keep_results: bool = True,
                 include_matrix: bool = False, topk: int = 0):
    """run_cmp over an SSF1 file in gather blocks: a reader thread fills the
    next pinned block while the GPU scans the current one (the ctypes call
    releases the GIL), and the picks of each block are appended to the
    SMB1 file as soon as they are back.  ``include_matrix`` streams the
    full ns x n_cand panels into the SMB1 records block by block (SMB1's
    flagged matrices, io.hpp:170-194) without holding the line's matrix;
    ``topk`` keeps the k best candidates per sample in the results.
    Returns the per-block ScanResults (or only the totals when keep_results
    is False)."""
    config.validate()
    with SSF1Reader(ssf_path) as rd:
        if not rd.uniform:
            raise ConfigError("run_cmp_file: gathers differ in ns or dt_us")
        G = rd.n_gathers
        bufs = [(_alloc((block, rd.fold, rd.ns), np.float32, True),
                 _alloc((block, rd.fold, 4), np.float32, True)) for _ in range(2)]
        writer = (SMB1Writer(smb_path, G, rd.ns, len(config.grid()), include_matrix)
                  if smb_path else None)
        results = []
        valid = 0
        kernel_ms = 0.0
        blocks = list(_blocks(G, block))
        pending = {}
        err = []

        def load(i):
            try:
                s, c = blocks[i]
                pending[i] = rd.read(s, c, out=bufs[i % 2], threads=threads)
            except BaseException as e:  # surfaced in the main thread
                err.append(e)

        th = threading.Thread(target=load, args=(0,))
        th.start()
        try:
            for i in range(len(blocks)):
                th.join()
                if err:
                    raise err[0]
                ds = pending.pop(i)
                if i + 1 < len(blocks):  # prefetch into the other buffer
                    th = threading.Thread(target=load, args=(i + 1,))
                    th.start()
                r = engine.run_cmp(ds, config, emit_matrix=include_matrix, topk=topk)
                valid += r.stats.naive_fetches
                kernel_ms += r.kernel_ms
                if writer is not None:
                    writer.append_result(r)
                if keep_results:
                    if include_matrix and smb_path:
                        r.values = None  # already on disk
                    results.append(r)
            if writer is not None:
                writer.close()
        finally:
            if th.is_alive():
                th.join()
            if writer is not None and getattr(writer, "_h", None):
                N.load().velan_smb1_end(writer._h)
                writer._h = None
    return results if keep_results else {"valid_intersections": valid, "kernel_ms": kernel_ms}


# --------------------------------------------------------------------------
# streaming file -> GPU -> file pipeline (CRS, halo-aware blocks)

def check_partition(mx: np.ndarray, my: np.ndarray, dims: tuple, apm: float) -> None:
    """partition()'s configuration checks (crs_pipeline.hpp:92-158), which
    run_crs applies before any compute: grid dims >= 1, apm > 0, finite
    midpoints, and apm at most half a shard's width / height.  The results
    do not depend on the grid (run_crs matches a 1 x 1 grid run); the GPU
    path blocks the line its own way."""
    gx, gy = dims
    if gx < 1 or gy < 1:
        raise ConfigError("partition: grid dims must be >= 1")
    if not apm > 0.0:
        raise ConfigError("partition: apm must be > 0")
    if len(mx) == 0:
        raise ParameterError("partition: dataset has no CDPs")
    if not (np.isfinite(mx).all() and np.isfinite(my).all()):
        raise ParameterError("partition: non-finite midpoint")
    w = (float(mx.max()) - float(mx.min())) / (gx if gx > 1 else 1)
    h = (float(my.max()) - float(my.min())) / (gy if gy > 1 else 1)
    if gx > 1 and apm > w / 2.0:
        raise ConfigError(f"partition: apm {apm} exceeds half the shard width {w / 2.0}")
    if gy > 1 and apm > h / 2.0:
        raise ConfigError(f"partition: apm {apm} exceeds half the shard height {h / 2.0}")


def crs_blocks(mx: np.ndarray, my: np.ndarray, cdp_id: np.ndarray, apm: float,
               block: int) -> list:
    """Halo-aware blocks of a CRS line / grid: the output rows in cdp_id order
    (ties by file index, run_crs's order, crs_pipeline.hpp:449-459) cut into
    runs of ``block`` rows; each block lists the file gathers it needs — its
    own rows plus every gather within the closed apm ball of one of them
    (neighbors_of, crs_pipeline.hpp:162-180: double test of the fp32
    difference) — in file order, and the position of its first own row in
    that subset's cdp_id order.  Returns [(rows, gathers, row_first)]."""
    G = len(cdp_id)
    order = np.lexsort((np.arange(G), cdp_id.astype(np.int64)))
    by_x = np.argsort(mx, kind="stable")
    xs = mx[by_x].astype(np.float64)
    margin = apm * 1e-5 + 1e-3
    out = []
    for s in range(0, G, block):
        rows = order[s:s + block]
        need = set(int(g) for g in rows)
        for g in rows:
            lo = np.searchsorted(xs, float(mx[g]) - apm - margin, "left")
            hi = np.searchsorted(xs, float(mx[g]) + apm + margin, "right")
            cand = by_x[lo:hi]
            dx = (mx[cand] - mx[g]).astype(np.float32).astype(np.float64)
            dy = (my[cand] - my[g]).astype(np.float32).astype(np.float64)
            for o in cand[dx * dx + dy * dy <= apm * apm]:
                need.add(int(o))
        gathers = np.array(sorted(need), np.int32)
        # own rows are contiguous in the subset's (cdp_id, index) order
        key = lambda g: (int(cdp_id[g]), int(g))  # noqa: E731
        first_key = key(int(rows[0]))
        row_first = sum(1 for g in gathers if key(int(g)) < first_key)
        out.append((rows, gathers, row_first))
    return out


def run_crs_file(engine: Engine, ssf_path: str, config: ScanConfig, apm: float,
                 smb_path: Optional[str] = None, dims: tuple = (1, 1), abc=None,
                 block: int = 256, threads: int = 0, keep_results: bool = True,
                 include_matrix: bool = False):
    """``velan crs --data F --out P --grid GXxGY --apm A [--matrix]``
    (tools/velan.cpp:167-184: read_dataset, run_crs, write_picks) as a
    stream: the SSF1 file is indexed (headers and first-trace coordinates
    only), the cdp_id-ordered output rows are cut into blocks, and each
    block's gathers plus its +-apm halo are read (one pread per gather, a
    reader thread filling the next pinned block while the GPU scans the
    current one) and scanned with the outputs restricted to the block.  The
    SMB1 records are appended block by block in run_crs's order, so the file
    is byte-identical to velan::run_crs + write_picks (EXACT variant).
    ``abc`` selects BASELINE's three-parameter operator (SMB1's velocity
    column then holds the C-axis velocity of the pick)."""
    config.validate()
    lib = N.load()
    with SSF1Reader(ssf_path) as rd:
        if not rd.uniform:
            raise ConfigError("run_crs_file: gathers differ in ns or dt_us")
        G = rd.n_gathers
        if G == 0:
            if smb_path:
                with SMB1Writer(smb_path, 0, 0, 0, include_matrix):
                    pass
            return [] if keep_results else {"valid_intersections": 0, "kernel_ms": 0.0}
        mx = np.zeros(G, np.float32)
        my = np.zeros(G, np.float32)
        _check(lib.velan_ssf1_midpoints(rd._h, _ptr(mx), _ptr(my)), "velan_ssf1_midpoints")
        check_partition(mx, my, dims, apm)
        blocks = crs_blocks(mx, my, rd.cdp_id, apm, block)
        cap = max(len(b[1]) for b in blocks)
        bufs = [(_alloc((cap, rd.fold, rd.ns), np.float32, True),
                 _alloc((cap, rd.fold, 4), np.float32, True)) for _ in range(2)]
        ncand = abc.ncand if abc is not None else len(config.grid())
        writer = SMB1Writer(smb_path, G, rd.ns, ncand, include_matrix) if smb_path else None
        results, valid, kernel_ms = [], 0, 0.0
        pending, err = {}, []

        def load(i):
            try:
                gl = blocks[i][1]
                sm, co = bufs[i % 2]
                _check(lib.velan_ssf1_read_list(rd._h, _ptr(gl), len(gl), rd.fold, _ptr(sm),
                                                _ptr(co), threads), "velan_ssf1_read_list")
                n = len(gl)
                pending[i] = Dataset(sm[:n], co[:n], rd.ntraces[gl].copy(),
                                     rd.cdp_id[gl].copy(), rd.dt_us)
            except BaseException as e:  # surfaced in the main thread
                err.append(e)

        th = threading.Thread(target=load, args=(0,))
        th.start()
        try:
            for i, (rows, gl, row_first) in enumerate(blocks):
                th.join()
                if err:
                    raise err[0]
                ds = pending.pop(i)
                if i + 1 < len(blocks):
                    th = threading.Thread(target=load, args=(i + 1,))
                    th.start()
                r = engine.run_crs(ds, config, apm, abc, emit_matrix=include_matrix,
                                   rows=(row_first, len(rows)))
                r.row_gather = gl[r.row_gather]  # file gather of every row
                valid += r.stats.naive_fetches
                kernel_ms += r.kernel_ms
                if writer is not None:
                    writer.append_result(r)
                if keep_results:
                    if include_matrix and smb_path:
                        r.values = None
                    results.append(r)
            if writer is not None:
                writer.close()
        finally:
            if th.is_alive():
                th.join()
            if writer is not None and getattr(writer, "_h", None):
                lib.velan_smb1_end(writer._h)
                writer._h = None
    return results if keep_results else {"valid_intersections": valid, "kernel_ms": kernel_ms}
