"""Python mirror of the reference's pipeline interface, driving the B200 path.

Names, argument meanings and error behaviour follow the reference library
(/root/reference/proj/include/velan):

    run_cmp(dataset, config, workers, stats)      cmp_pipeline.hpp:94-106
    run_crs(dataset, config, dims, apm, ...)      crs_pipeline.hpp:283-460
    scan_cdp(gather, config)                      cmp_pipeline.hpp:17-27
    scan_central_cdp(central, neighbors, config)  crs_pipeline.hpp:184-197
    neighbors_of(central, candidates, apm)        crs_pipeline.hpp:162-180
    ScanConfig / VelocityGrid                     scan.hpp:27-79, traveltime.hpp:30-47
    error / parameter_error / config_error        error.hpp:9-40

Every scan goes through the C-ABI (include/velan_gpu.h) into the sm_100a
kernels; there is no CPU path.  ``workers`` means devices, as the reference's
worker pool becomes one host thread per GPU.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional, Sequence

import numpy as np

from . import _native as N


# --------------------------------------------------------------------------
# errors (error.hpp:9-40)

class VelanError(RuntimeError):
    """velan::error"""


class ParameterError(VelanError):
    """velan::parameter_error"""


class ConfigError(VelanError):
    """velan::config_error"""


class DeviceError(VelanError):
    """No usable sm_100 device (the GPU path has no CPU fallback)."""


def _raise(code: int, where: str) -> None:
    if code == N.OK:
        return
    msg = f"{where}: {N.last_error()}"
    if code == N.ECONFIG:
        raise ConfigError(msg)
    if code == N.EPARAM:
        raise ParameterError(msg)
    if code == N.ENODEV:
        raise DeviceError(msg)
    raise VelanError(msg)


# --------------------------------------------------------------------------
# data model (types.hpp:14-54, flattened)

@dataclass
class Dataset:
    """velan::Dataset as flat arrays.

    samples [G, M, ns] float32 (Trace::samples), coords [G, M, 4] float32
    (sx, sy, gx, gy), ntraces [G] int32, cdp_id [G] uint32, dt_us.
    ``samples`` may also be a CUDA torch tensor (device-resident input).
    """
    samples: object
    coords: np.ndarray
    ntraces: np.ndarray
    cdp_id: np.ndarray
    dt_us: int
    metadata: dict = field(default_factory=dict)

    def __post_init__(self):
        self.coords = np.ascontiguousarray(self.coords, dtype=np.float32)
        self.ntraces = np.ascontiguousarray(self.ntraces, dtype=np.int32)
        self.cdp_id = np.ascontiguousarray(self.cdp_id, dtype=np.uint32)
        if isinstance(self.samples, np.ndarray):
            self.samples = np.ascontiguousarray(self.samples, dtype=np.float32)

    @property
    def ncdps(self) -> int:
        return int(self.coords.shape[0])

    @property
    def fold(self) -> int:
        return int(self.coords.shape[1])

    @property
    def ns(self) -> int:
        return int(self.samples.shape[2])

    @property
    def dt_seconds(self) -> float:
        return float(self.dt_us) * 1e-6

    def midpoints(self) -> np.ndarray:
        """midpoint_of per gather (types.hpp:57-62), fp32."""
        c = self.coords[:, 0, :]
        mx = (c[:, 0] + c[:, 2]) * np.float32(0.5)
        my = (c[:, 1] + c[:, 3]) * np.float32(0.5)
        return np.stack([mx, my], axis=1).astype(np.float32)

    def subset(self, idx) -> "Dataset":
        idx = np.asarray(idx)
        return Dataset(np.asarray(self.samples)[idx], self.coords[idx],
                       self.ntraces[idx], self.cdp_id[idx], self.dt_us,
                       dict(self.metadata))

    @staticmethod
    def from_gathers(gathers: Sequence[dict], dt_us: int) -> "Dataset":
        """Build from reference-shaped gathers: each a dict with ``cdp_id``
        and ``traces`` = list of (sx, sy, gx, gy, samples)."""
        G = len(gathers)
        M = max([len(g["traces"]) for g in gathers] + [1])
        ns = 0
        for g in gathers:
            for t in g["traces"]:
                ns = len(t[4])
                break
            if ns:
                break
        samples = np.zeros((G, M, max(ns, 1)), np.float32)
        coords = np.zeros((G, M, 4), np.float32)
        ntr = np.zeros(G, np.int32)
        ids = np.zeros(G, np.uint32)
        for i, g in enumerate(gathers):
            ids[i] = g["cdp_id"]
            ntr[i] = len(g["traces"])
            for m, t in enumerate(g["traces"]):
                coords[i, m] = t[:4]
                samples[i, m, :] = np.asarray(t[4], np.float32)
        return Dataset(samples, coords, ntr, ids, dt_us)


# --------------------------------------------------------------------------
# scan configuration (scan.hpp:27-79, traveltime.hpp:30-47)

def velocity_grid(vmin: float, vmax: float, nc: int) -> np.ndarray:
    """VelocityGrid::value for c = 0..nc-1, in the reference's fp32 order:
    vmin + float(c) * (vmax - vmin) / float(nc - 1)."""
    f = np.float32
    if not (f(vmin) > 0) or not (f(vmax) >= f(vmin)):
        raise ParameterError("VelocityGrid: need 0 < vmin <= vmax")
    if nc < 1:
        raise ParameterError("VelocityGrid: nc must be >= 1")
    if nc == 1:
        return np.array([vmin], np.float32)
    c = np.arange(nc, dtype=np.float32)
    return (f(vmin) + (c * (f(vmax) - f(vmin))) / f(nc - 1)).astype(np.float32)


def slowness_grid(v_first: float, v_last: float, n: int) -> np.ndarray:
    """BASELINE.json's CMP grid: n velocities linear in slowness,
    p_c = 1/v_first + c (1/v_last - 1/v_first)/(n-1) (double), v_c = float(1/p_c)."""
    p0, p1 = 1.0 / v_first, 1.0 / v_last
    c = np.arange(n, dtype=np.float64)
    p = p0 + c * (p1 - p0) / max(n - 1, 1)
    return (1.0 / p).astype(np.float32)


VARIANTS = {"exact": N.VARIANT_EXACT, "fast": N.VARIANT_FAST}


@dataclass
class ScanConfig:
    """ScanConfig (scan.hpp:27-79).  The CPU tuning knobs of the reference
    (tile, lanes, size_h, scratch budget, range cap) have no GPU meaning and
    are not carried; ``kernel_variant`` selects the GPU kernel variant
    ("exact": bitwise reference arithmetic, "fast": restructured sums).
    ``velocities`` overrides the v-linear grid with an explicit candidate
    list (BASELINE's slowness-linear grid)."""
    vmin: float = 2000.0
    vmax: float = 3000.0
    nc: int = 101
    w: int = 4
    kernel_variant: str = "exact"
    velocities: Optional[np.ndarray] = None

    def grid(self) -> np.ndarray:
        if self.velocities is not None:
            return np.ascontiguousarray(self.velocities, dtype=np.float32)
        return velocity_grid(self.vmin, self.vmax, self.nc)

    def validate(self) -> None:
        if self.w < 1:
            raise ConfigError("ScanConfig: w must be >= 1")
        if self.velocities is None:
            if self.nc < 1:
                raise ConfigError("ScanConfig: nc must be >= 1")
            if not (self.vmin > 0.0) or not (self.vmax >= self.vmin):
                raise ConfigError("ScanConfig: need 0 < vmin <= vmax")
        if self.kernel_variant not in VARIANTS:
            raise ConfigError(f"ScanConfig: unknown kernel variant {self.kernel_variant!r}")


@dataclass
class CrsAbcGrid:
    """BASELINE three-parameter CRS search grid: A [s/m], B [s/m^2] and the
    C axis scanned as velocity v (C = 2/(t0 v^2)).  Flat candidate index
    (ia * nB + ib) * nC + ic."""
    a: np.ndarray
    b: np.ndarray
    v: np.ndarray

    def __post_init__(self):
        self.a = np.ascontiguousarray(self.a, dtype=np.float32)
        self.b = np.ascontiguousarray(self.b, dtype=np.float32)
        self.v = np.ascontiguousarray(self.v, dtype=np.float32)

    @property
    def ncand(self) -> int:
        return len(self.a) * len(self.b) * len(self.v)

    def decode(self, flat):
        flat = np.asarray(flat)
        ic = flat % len(self.v)
        r = flat // len(self.v)
        return r // len(self.b), r % len(self.b), ic


@dataclass
class CacheStats:
    """CacheStats (trace_cache.hpp:25-39): only naive_fetches (the valid
    curve-trace intersections, bench.hpp:126) survives on the GPU; the
    nominal count includes out-of-range hits (BASELINE's eval count / w)."""
    naive_fetches: int = 0
    nominal_intersections: int = 0


@dataclass
class ScanResult:
    """A batch of SemblanceMatrix (scan.hpp:89-103): per output row the pick
    index, its semblance (BestPick::semblance) and the stack at the pick
    (stack_trace); ``values`` is the optional [rows, ns, ncand] matrix."""
    best_idx: np.ndarray
    best_semblance: np.ndarray
    stack_trace: np.ndarray
    candidates: np.ndarray
    row_gather: np.ndarray
    cdp_id: np.ndarray
    values: Optional[np.ndarray] = None
    stats: CacheStats = field(default_factory=CacheStats)
    kernel_ms: float = 0.0
    total_ms: float = 0.0
    n_candidates: int = 0  # flat candidate count (SemblanceMatrix::nc)
    topk_idx: Optional[np.ndarray] = None        # [rows, ns, k], best first
    topk_semblance: Optional[np.ndarray] = None  # [rows, ns, k]

    @property
    def best_velocity(self) -> np.ndarray:
        """BestPick::velocity (NMO / d2 operators)."""
        return self.candidates[self.best_idx % len(self.candidates)]

    def __len__(self):
        return self.best_idx.shape[0]


# --------------------------------------------------------------------------

def _ptr(a) -> int:
    if a is None:
        return 0
    if isinstance(a, np.ndarray):
        return a.ctypes.data
    return int(a.data_ptr())  # torch tensor


def _dataset_struct(ds: Dataset) -> N.Dataset:
    s = N.Dataset()
    s.n_gathers = ds.ncdps
    s.max_traces = ds.fold if ds.ncdps else 1
    s.ns = int(ds.samples.shape[2]) if ds.ncdps else 0
    s.dt_us = int(ds.dt_us)
    s.cdp_id = _ptr(ds.cdp_id)
    s.ntraces = _ptr(ds.ntraces)
    s.coords = _ptr(ds.coords)
    s.samples = _ptr(ds.samples)
    if isinstance(ds.samples, np.ndarray):
        s.samples_mem = N.MEM_HOST
    else:
        if not ds.samples.is_cuda and not ds.samples.is_contiguous():
            raise ParameterError("samples tensor must be contiguous")
        s.samples_mem = N.MEM_DEVICE if ds.samples.is_cuda else N.MEM_HOST
        s.samples_device = ds.samples.device.index or 0 if ds.samples.is_cuda else 0
    return s


def _scan_struct(op: int, variant: str, w: int, v: np.ndarray,
                 abc: Optional[CrsAbcGrid], apm: float, keep: list,
                 rows: Optional[tuple] = None) -> N.Scan:
    sc = N.Scan()
    if rows is not None:
        sc.row_first, sc.row_count = int(rows[0]), int(rows[1])
    sc.op = op
    if variant not in VARIANTS:
        raise ConfigError(f"ScanConfig: unknown kernel variant {variant!r}")
    sc.variant = VARIANTS[variant]
    sc.w = int(w)
    if abc is not None:
        keep += [abc.a, abc.b, abc.v]
        sc.n_a, sc.n_b, sc.n_c = len(abc.a), len(abc.b), len(abc.v)
        sc.a, sc.b, sc.v = _ptr(abc.a), _ptr(abc.b), _ptr(abc.v)
    else:
        v = np.ascontiguousarray(v, dtype=np.float32)
        keep.append(v)
        sc.n_a = sc.n_b = 1
        sc.n_c = len(v)
        sc.v = _ptr(v)
    sc.apm = float(apm)
    return sc


class Engine:
    """Owns a velan_gpu context over one or more devices (the GPU analogue
    of the reference's worker pool)."""

    def __init__(self, devices: Optional[Sequence[int]] = None):
        lib = N.load()
        if devices is None:
            devices = [0]
        ids = (C.c_int32 * len(devices))(*devices)
        h = C.c_void_p()
        _raise(lib.velan_gpu_create(ids, len(devices), C.byref(h)), "velan_gpu_create")
        self._h = h
        self.devices = list(devices)

    def close(self):
        if getattr(self, "_h", None):
            N.load().velan_gpu_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def _run(self, fn, ds: Dataset, op: int, variant: str, w: int,
             v: np.ndarray, abc: Optional[CrsAbcGrid], apm: float,
             emit_matrix: bool, out=None, rows=None, topk: int = 0) -> ScanResult:
        lib = N.load()
        keep: list = []
        sc = _scan_struct(op, variant, w, v, abc, apm, keep, rows)
        dss = _dataset_struct(ds)
        G = ds.ncdps if rows is None else int(rows[1])
        ns = dss.ns
        ncand = abc.ncand if abc is not None else len(v)
        if out is not None:  # caller-provided host buffers (e.g. pinned)
            best_idx, best_s, best_st = out
        else:
            best_idx = np.zeros((G, ns), np.int32)
            best_s = np.zeros((G, ns), np.float32)
            best_st = np.zeros((G, ns), np.float32)
        rows = np.zeros(G, np.int32)
        mat = np.zeros((G, ns, ncand), np.float32) if emit_matrix else None
        tki = np.zeros((G, ns, topk), np.int32) if topk else None
        tks = np.zeros((G, ns, topk), np.float32) if topk else None
        res = N.Result()
        res.topk = topk
        res.topk_idx = _ptr(tki)
        res.topk_semblance = _ptr(tks)
        res.out_mem = N.MEM_HOST
        res.best_idx = _ptr(best_idx)
        res.best_semblance = _ptr(best_s)
        res.best_stack = _ptr(best_st)
        res.matrix = _ptr(mat)
        res.row_gather = _ptr(rows)
        code = fn(self._h, C.byref(dss), C.byref(sc), C.byref(res))
        _raise(code, fn.__name__)
        cands = abc.v if abc is not None else np.ascontiguousarray(v, np.float32)
        if G == 0:
            rows = np.zeros(0, np.int32)
        if out is not None:
            best_idx, best_s, best_st = (np.asarray(x) for x in out)
        return ScanResult(best_idx, best_s, best_st, cands, rows,
                          ds.cdp_id[rows] if G else ds.cdp_id, mat,
                          CacheStats(int(res.valid_intersections),
                                     int(res.nominal_intersections)),
                          float(res.kernel_ms), float(res.total_ms), int(ncand), tki, tks)

    def run_cmp(self, ds: Dataset, config: ScanConfig,
                emit_matrix: bool = False, out=None, rows=None,
                topk: int = 0) -> ScanResult:
        """``rows`` = (first, count) restricts the outputs to a row block;
        ``topk`` (<= 8) adds the k best candidates of every sample."""
        config.validate()
        return self._run(N.load().velan_gpu_cmp, ds, N.OP_NMO,
                         config.kernel_variant, config.w, config.grid(), None,
                         0.0, emit_matrix, out, rows, topk)

    def run_crs(self, ds: Dataset, config: ScanConfig, apm: float,
                abc: Optional[CrsAbcGrid] = None,
                emit_matrix: bool = False, out=None, rows=None,
                topk: int = 0) -> ScanResult:
        """``rows`` = (first, count): a shard's own block of the cdp_id-ordered
        rows; the remaining gathers are halo feeding the neighbourhoods."""
        config.validate()
        op = N.OP_CRS_ABC if abc is not None else N.OP_CRS_D2
        return self._run(N.load().velan_gpu_crs, ds, op, config.kernel_variant,
                         config.w, config.grid(), abc, apm, emit_matrix, out,
                         rows, topk)

    def nmo_correct(self, ds: Dataset, config: ScanConfig, picks,
                    op: str = "nmo", apm: float = 0.0,
                    abc: Optional[CrsAbcGrid] = None, rows=None) -> np.ndarray:
        """NMO-corrected output gathers [rows, max_traces, ns] of a scan's
        picks (``picks`` = ScanResult.best_idx or any [rows, ns] flat
        candidate indices): each trace interpolated (kernel.hpp:39) at the
        central traveltime of its row's pick (traveltime.hpp:53-80); the
        mean over the traces is the corrected stack."""
        lib = N.load()
        config.validate()
        opc = {"nmo": N.OP_NMO, "d2": N.OP_CRS_D2, "abc": N.OP_CRS_ABC}[op]
        keep: list = []
        sc = _scan_struct(opc, config.kernel_variant, config.w, config.grid(), abc, apm,
                          keep, rows)
        dss = _dataset_struct(ds)
        n_rows = ds.ncdps if rows is None else int(rows[1])
        picks = np.ascontiguousarray(picks, np.int32)
        if picks.shape != (n_rows, dss.ns):
            raise ParameterError(f"picks must be [{n_rows}, {dss.ns}]")
        out = np.zeros((n_rows, max(ds.fold, 1), dss.ns), np.float32)
        _raise(lib.velan_gpu_nmo_correct(self._h, C.byref(dss), C.byref(sc), _ptr(picks),
                                         _ptr(out)), "velan_gpu_nmo_correct")
        return out

    def plan(self, ds: Dataset, config: ScanConfig, op: str = "nmo",
             apm: float = 0.0, abc: Optional[CrsAbcGrid] = None,
             rows: Optional[tuple] = None) -> "Plan":
        return Plan(self, ds, config, op, apm, abc, rows)


class Plan:
    """Resident plan: tables (and samples, when given on the host) uploaded
    once; execute() only launches the scan kernels."""

    def __init__(self, engine: Engine, ds: Dataset, config: ScanConfig,
                 op: str, apm: float, abc: Optional[CrsAbcGrid],
                 rows: Optional[tuple] = None):
        lib = N.load()
        config.validate()
        opc = {"nmo": N.OP_NMO, "d2": N.OP_CRS_D2, "abc": N.OP_CRS_ABC}[op]
        self._keep: list = []
        sc = _scan_struct(opc, config.kernel_variant, config.w, config.grid(),
                          abc, apm, self._keep, rows)
        dss = _dataset_struct(ds)
        self._ds = ds  # keep device samples alive
        h = C.c_void_p()
        _raise(lib.velan_gpu_plan_create(engine._h, C.byref(dss), C.byref(sc),
                                         C.byref(h)), "velan_gpu_plan_create")
        self._h = h
        self.rows = ds.ncdps if rows is None else int(rows[1])
        self.ns = dss.ns
        self.ncand = abc.ncand if abc is not None else len(config.grid())

    def launches(self) -> int:
        return int(N.load().velan_gpu_plan_launches(self._h))

    def execute(self, best_idx, best_s, best_stack, matrix=None, stream=None,
                on_device: bool = True) -> N.Result:
        """Run the scan; output buffers are CUDA tensors (on_device) or
        numpy arrays.  ``stream`` is a torch.cuda.Stream or None."""
        res = N.Result()
        res.out_mem = N.MEM_DEVICE if on_device else N.MEM_HOST
        res.best_idx = _ptr(best_idx)
        res.best_semblance = _ptr(best_s)
        res.best_stack = _ptr(best_stack)
        res.matrix = _ptr(matrix)
        res.row_gather = 0
        st = 0 if stream is None else int(stream.cuda_stream)
        _raise(N.load().velan_gpu_plan_execute(self._h, C.byref(res), st or None),
               "velan_gpu_plan_execute")
        return res

    def close(self):
        if getattr(self, "_h", None):
            N.load().velan_gpu_plan_destroy(self._h)
            self._h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# --------------------------------------------------------------------------
# reference-named entry points

_engines: dict = {}


def _engine(workers: int) -> Engine:
    if workers < 1:
        raise ParameterError("worker count must be >= 1")
    lib = N.load()
    ndev = lib.velan_gpu_device_count()
    if ndev == 0:
        raise DeviceError("no sm_100 device visible; the scan has no CPU path")
    n = min(workers, ndev)
    if n not in _engines:
        _engines[n] = Engine(list(range(n)))
    return _engines[n]


def run_cmp(dataset: Dataset, config: ScanConfig, workers: int = 1,
            stats: Optional[CacheStats] = None,
            emit_matrix: bool = False) -> ScanResult:
    """run_cmp (cmp_pipeline.hpp:94-106).  workers = devices."""
    config.validate()
    if workers < 1:
        raise ParameterError("worker count must be >= 1")
    r = _engine(workers).run_cmp(dataset, config, emit_matrix)
    if stats is not None:
        stats.naive_fetches += r.stats.naive_fetches
        stats.nominal_intersections += r.stats.nominal_intersections
    return r


def run_crs(dataset: Dataset, config: ScanConfig, apm: float,
            workers: int = 1, stats: Optional[CacheStats] = None,
            abc: Optional[CrsAbcGrid] = None,
            emit_matrix: bool = False) -> ScanResult:
    """run_crs (crs_pipeline.hpp:283-460) on a 1-D contiguous shard layout;
    ``abc`` selects BASELINE's three-parameter operator instead of the
    reference's d2 neighbourhood operator."""
    config.validate()
    if workers < 1:
        raise ParameterError("worker count must be >= 1")
    r = _engine(workers).run_crs(dataset, config, apm, abc, emit_matrix)
    if stats is not None:
        stats.naive_fetches += r.stats.naive_fetches
        stats.nominal_intersections += r.stats.nominal_intersections
    return r


def scan_cdp(dataset: Dataset, index: int, config: ScanConfig,
             emit_matrix: bool = True) -> ScanResult:
    """scan_cdp (cmp_pipeline.hpp:17-27) for gather ``index``."""
    return run_cmp(dataset.subset([index]), config, 1, None, emit_matrix)


def neighbors_of(dataset: Dataset, central: int, candidates: Sequence[int],
                 apm: float) -> list:
    """neighbors_of (crs_pipeline.hpp:162-180): indices of the candidates in
    the closed ball |dm| <= apm (double test of the fp32 difference),
    excluding the central gather, ordered by cdp_id."""
    if not (apm > 0.0):
        raise ParameterError("neighbors_of: apm must be > 0")
    mp = dataset.midpoints()
    c = mp[central]
    out = []
    for g in candidates:
        if g == central:
            continue
        dx = float(np.float32(mp[g, 0] - c[0]))
        dy = float(np.float32(mp[g, 1] - c[1]))
        if dx * dx + dy * dy <= apm * apm:
            out.append(int(g))
    out.sort(key=lambda g: (int(dataset.cdp_id[g]), g))
    return out


def scan_central_cdp(dataset: Dataset, central: int, neighbors: Sequence[int],
                     config: ScanConfig, abc: Optional[CrsAbcGrid] = None,
                     emit_matrix: bool = True) -> ScanResult:
    """scan_central_cdp (crs_pipeline.hpp:184-197): the central gather's
    sweep extended by the given neighbours.  Implemented as a CRS run over
    the sub-dataset {central} + neighbours with an aperture that admits
    exactly those neighbours; only the central row is returned."""
    idx = [central] + [g for g in neighbors if g != central]
    sub = dataset.subset(idx)
    mp = sub.midpoints()
    d = np.sqrt(((mp[1:] - mp[0]).astype(np.float64) ** 2).sum(axis=1)) if len(idx) > 1 else np.zeros(0)
    apm = float(d.max()) * (1 + 1e-9) + 1e-9 if len(d) else 1e-9
    r = run_crs(sub, config, apm, 1, None, abc, emit_matrix)
    row = int(np.nonzero(r.row_gather == 0)[0][0])
    keep = slice(row, row + 1)
    return ScanResult(r.best_idx[keep], r.best_semblance[keep],
                      r.stack_trace[keep], r.candidates, r.row_gather[keep],
                      r.cdp_id[keep],
                      None if r.values is None else r.values[keep], r.stats,
                      r.kernel_ms, r.total_ms)


@dataclass
class SweepPlan:
    """Host-side description of the TraceSweeps a scan will run."""
    row_gather: np.ndarray    # input gather per output row
    sweep_traces: np.ndarray  # traces per sweep
    leg_off: np.ndarray       # CSR offsets [rows + 1]
    leg_gather: np.ndarray    # gathers of every sweep, central first
    nominal_intersections: int


def describe(dataset: Dataset, config: ScanConfig, op: str = "nmo",
             apm: float = 0.0, abc: Optional[CrsAbcGrid] = None,
             rows: Optional[tuple] = None) -> SweepPlan:
    """The sweeps (central gather + closed-ball neighbours in cdp_id order)
    the library builds for a scan — host only, no device needed."""
    lib = N.load()
    opc = {"nmo": N.OP_NMO, "d2": N.OP_CRS_D2, "abc": N.OP_CRS_ABC}[op]
    keep: list = []
    sc = _scan_struct(opc, config.kernel_variant, config.w, config.grid(),
                      abc, apm, keep, rows)
    dss = _dataset_struct(dataset)
    n_rows = dataset.ncdps if rows is None else int(rows[1])
    rg = np.zeros(n_rows, np.int32)
    st = np.zeros(n_rows, np.int32)
    lo = np.zeros(n_rows + 1, np.int32)
    nl, nom = C.c_int64(0), C.c_uint64(0)
    _raise(lib.velan_gpu_describe(C.byref(dss), C.byref(sc), _ptr(rg), _ptr(st),
                                  _ptr(lo), None, 0, C.byref(nl), C.byref(nom)),
           "velan_gpu_describe")
    lg = np.zeros(max(nl.value, 1), np.int32)
    _raise(lib.velan_gpu_describe(C.byref(dss), C.byref(sc), None, None, None,
                                  _ptr(lg), nl.value, C.byref(nl), C.byref(nom)),
           "velan_gpu_describe")
    return SweepPlan(rg, st, lo, lg[: nl.value], int(nom.value))


def device_count() -> int:
    return int(N.load().velan_gpu_device_count())
