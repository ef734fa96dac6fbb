"""The five BASELINE.json configurations as seeded synthetic inputs.

Shapes, sizes and value distributions follow BASELINE.json ``configs``; the
builder's choices where BASELINE is silent are recorded here and in
DESIGN.md §6 (seeds 11678 + config index; CMP-large v range 1400-5000 m/s
to cover the 4725 m/s events; CRS reflector geometry).

Generation runs in the native library (velan_gpu_synth_generate, C++ host,
multi-threaded, counter-based per-gather streams).
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field, replace
from typing import Optional

import numpy as np

from . import _native as N
from .api import CrsAbcGrid, Dataset, ParameterError, ScanConfig, slowness_grid


@dataclass
class SynthSpec:
    kind: int  # 0 CMP, 1 CRS line
    n_gathers: int
    n_traces: int
    ns: int
    dt_us: int
    spacing: float
    h0: float
    dh: float
    n_events: int
    t0_lo: float
    t0_hi: float
    v_lo: float = 1500.0
    v_hi: float = 3500.0
    v_profile: int = 0
    v_trend_0: float = 1500.0
    v_trend_slope: float = 750.0
    v_perturb: float = 0.0
    amp_lo: float = 0.5
    amp_hi: float = 1.0
    freq: float = 25.0
    sigma: float = 0.1
    a_abs: float = 2e-4
    b_max: float = 1e-7
    seed: int = 11678

    def _struct(self, first: int, count: int, n_threads: int, n_line: Optional[int]):
        s = N.Synth()
        for f, _ in N.Synth._fields_:
            if hasattr(self, f):
                setattr(s, f, getattr(self, f))
        s.n_gathers = count
        s.gather_first = first
        s.n_threads = n_threads
        s.n_line = self.n_gathers if n_line is None else n_line
        return s

    def generate_device(self, first: int = 0, count: Optional[int] = None,
                        n_line: Optional[int] = None, device: int = 0) -> Dataset:
        """Gathers [first, first + count) generated in HBM by the device
        generator (synth_gpu.cu): samples is a CUDA tensor, the geometry
        comes from the host generator (no samples)."""
        import torch
        lib = N.load()
        count = self.n_gathers if count is None else count
        s = self._struct(first, count, 0, n_line)
        samples = torch.empty((count, self.n_traces, self.ns), dtype=torch.float32,
                              device=f"cuda:{device}")
        coords = np.empty((count, self.n_traces, 4), np.float32)
        ntr = np.empty(count, np.int32)
        ids = np.empty(count, np.uint32)
        if lib.velan_gpu_synth_generate(C.byref(s), None, coords.ctypes.data,
                                        ntr.ctypes.data, ids.ctypes.data) != 0:
            raise ParameterError("velan_gpu_synth_generate: bad parameters")
        with torch.cuda.device(device):
            stream = torch.cuda.current_stream().cuda_stream
            if lib.velan_gpu_synth_generate_device(C.byref(s), samples.data_ptr(), stream) != 0:
                raise ParameterError("velan_gpu_synth_generate_device: bad parameters or "
                                     "device failure")
        return Dataset(samples, coords, ntr, ids, self.dt_us,
                       {"generator": "velan_gpu synth (device)", "spec": self.__dict__.copy(),
                        "first": first})

    def generate(self, first: int = 0, count: Optional[int] = None,
                 n_threads: int = 0, n_line: Optional[int] = None,
                 lib=None) -> Dataset:
        """Gathers [first, first + count) of the full line.  ``lib`` may name
        another build of the same host generator (oracle.synth_lib(): the
        CPU-only arms generate without loading the GPU library)."""
        lib = N.load() if lib is None else lib
        count = self.n_gathers if count is None else count
        s = self._struct(first, count, n_threads, n_line)
        samples = np.empty((count, self.n_traces, self.ns), np.float32)
        coords = np.empty((count, self.n_traces, 4), np.float32)
        ntr = np.empty(count, np.int32)
        ids = np.empty(count, np.uint32)
        code = lib.velan_gpu_synth_generate(
            C.byref(s), samples.ctypes.data, coords.ctypes.data,
            ntr.ctypes.data, ids.ctypes.data)
        if code != 0:
            raise ParameterError("velan_gpu_synth_generate: bad parameters")
        return Dataset(samples, coords, ntr, ids, self.dt_us,
                       {"generator": "velan_gpu synth", "spec": self.__dict__.copy(),
                        "first": first})


@dataclass
class Workload:
    name: str
    spec: SynthSpec
    op: str              # "nmo" | "abc"
    config: ScanConfig
    apm: float = 0.0
    abc: Optional[CrsAbcGrid] = None
    notes: str = ""

    @property
    def ncand(self) -> int:
        return self.abc.ncand if self.abc is not None else len(self.config.grid())

    def traces_per_sweep(self, row_gather_count: Optional[int] = None) -> np.ndarray:
        """Traces in aperture per output midpoint (line ends truncated)."""
        G = self.spec.n_gathers if row_gather_count is None else row_gather_count
        M = self.spec.n_traces
        if self.op == "nmo":
            return np.full(G, M, np.int64)
        ap = int(round(self.apm / self.spec.spacing))
        i = np.arange(G)
        lo = np.maximum(i - ap, 0)
        hi = np.minimum(i + ap, G - 1)
        return (hi - lo + 1).astype(np.int64) * M

    def nominal_evals(self) -> int:
        """BASELINE metric units: midpoints x t0 x candidates x traces x w."""
        return int(self.traces_per_sweep().sum()) * self.spec.ns * self.ncand * self.config.w


def cmp_small() -> Workload:
    spec = SynthSpec(kind=0, n_gathers=64, n_traces=24, ns=1000, dt_us=4000,
                     spacing=25.0, h0=50.0, dh=50.0, n_events=5, t0_lo=0.3,
                     t0_hi=3.5, v_lo=1500.0, v_hi=3500.0, freq=25.0,
                     sigma=0.1, seed=11678 + 0)
    cfg = ScanConfig(w=11, velocities=slowness_grid(1400.0, 4000.0, 101))
    return Workload("cmp_small", spec, "nmo", cfg,
                    notes="101 C linear in slowness 1400->4000 m/s, w=11")


def cmp_large() -> Workload:
    spec = SynthSpec(kind=0, n_gathers=8192, n_traces=60, ns=2000, dt_us=2000,
                     spacing=25.0, h0=25.0, dh=25.0, n_events=8, t0_lo=0.2,
                     t0_hi=3.8, v_profile=1, v_trend_0=1500.0,
                     v_trend_slope=750.0, v_perturb=0.05, freq=30.0,
                     sigma=0.2, seed=11678 + 1)
    cfg = ScanConfig(w=15, velocities=slowness_grid(1400.0, 5000.0, 401))
    return Workload("cmp_large", spec, "nmo", cfg,
                    notes="401 C linear in slowness 1400->5000 m/s "
                          "(covers the 4725 m/s events), w=15")


def _abc_grid(na: int, nb: int, nc: int) -> CrsAbcGrid:
    a = np.linspace(-2e-4, 2e-4, na).astype(np.float32)
    b = np.linspace(0.0, 1e-7, nb).astype(np.float32)
    v = np.linspace(1500.0, 3500.0, nc).astype(np.float32)
    return CrsAbcGrid(a, b, v)


def crs_small() -> Workload:
    spec = SynthSpec(kind=1, n_gathers=256, n_traces=30, ns=1000, dt_us=4000,
                     spacing=25.0, h0=50.0, dh=50.0, n_events=4, t0_lo=0.3,
                     t0_hi=3.5, v_lo=1500.0, v_hi=3500.0, freq=25.0,
                     sigma=0.1, seed=11678 + 2)
    grid = _abc_grid(11, 11, 21)
    cfg = ScanConfig(w=11, velocities=grid.v)
    return Workload("crs_small", spec, "abc", cfg, apm=125.0, abc=grid,
                    notes="aperture +-5 midpoints (apm 125 m at 25 m), "
                          "11 A x 11 B x 21 C, w=11")


def crs_large() -> Workload:
    spec = SynthSpec(kind=1, n_gathers=4096, n_traces=60, ns=2000, dt_us=2000,
                     spacing=12.5, h0=25.0, dh=25.0, n_events=10, t0_lo=0.2,
                     t0_hi=3.8, v_lo=1500.0, v_hi=3500.0, freq=25.0,
                     sigma=0.2, seed=11678 + 3)
    grid = _abc_grid(21, 21, 41)
    cfg = ScanConfig(w=15, velocities=grid.v)
    return Workload("crs_large", spec, "abc", cfg, apm=125.0, abc=grid,
                    notes="aperture +-10 midpoints (apm 125 m at 12.5 m), "
                          "21 A x 21 B x 41 C, w=15")


def scaling_cmp() -> Workload:
    w = cmp_large()
    w.name = "scaling_cmp"
    w.spec = replace(w.spec, n_gathers=65536, seed=11678 + 4)
    return w


def scaling_crs() -> Workload:
    w = crs_large()
    w.name = "scaling_crs"
    w.spec = replace(w.spec, n_gathers=32768, seed=11678 + 4)
    return w


WORKLOADS = {
    "cmp_small": cmp_small,
    "cmp_large": cmp_large,
    "crs_small": crs_small,
    "crs_large": crs_large,
    "scaling_cmp": scaling_cmp,
    "scaling_crs": scaling_crs,
}
