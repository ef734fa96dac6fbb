#!/usr/bin/env python
"""bench.py — BASELINE.json metric: semblance evals/s of the CMP/CRS parameter
search on N B200s, with the FP32 roofline fraction, the host-CPU reference and
an oracle check of a seeded sample of the gathered picks.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cmp_large|cmp_small|crs_small|crs_large|
                                scaling_cmp|scaling_crs]

A "step" is one pass of the scan over one rank's workload: the BASELINE
configuration itself (default configs[1], CMP large: 8192 gathers x 60 traces
x 2000 samples, 401 candidates, w = 15).  Multi-GPU is one process per GPU
(``--gpus N`` outside torchrun re-launches itself under
``torch.distributed.run``); the default workloads scale weakly: every rank
scans its own contiguous block of a longer line (no collective on the data
path; a barrier and the max-over-ranks timing reduction only).  The BASELINE
scaling sweep (--workload scaling_cmp: 65536 gathers, scaling_crs: 32768
midpoints) is strong scaling: the fixed line split into contiguous blocks
(CRS blocks with their replicated +-aperture halo).

After the timed region every rank's picks are gathered to rank 0 (NCCL
gather, then one D2H copy: the whole line's results on the host) and a seeded
sample of them is checked against the CPU oracle (``parity_sample``: 1 % of
the CMP cells, or a fixed 4096-cell CRS sample).

One JSON line on rank 0.  ``value`` = nominal evals (midpoints x t0 x
candidates x traces x w, BASELINE's unit) of all ranks / the max over ranks of
the device time of K steps with the input resident in HBM (3.9 GB per GPU,
larger than the 126 MB L2, so no flush is needed).  ``e2e`` = the same metric
through the one-shot C-ABI call velan_gpu_cmp/crs from pinned host buffers
(H2D of the samples and D2H of the picks inside the timed region).  The
default line also carries ``crs_small``: BASELINE configs[2] (the CRS
operator) measured the same way.
"""
from __future__ import annotations

import argparse
import json
import math
import os
import socket
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "semblance evals/sec"
UNIT = "evals/s"
RTOL = 1e-4  # north star: semblance within 1e-4 relative, picks up to near-ties


def parse():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=3)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", choices=["ours", "reference"], default="ours")
    ap.add_argument("--workload", default="cmp_large")
    ap.add_argument("--variant", default="fast", choices=["fast", "exact"])
    ap.add_argument("--cpu-seconds", type=float, default=10.0,
                    help="target CPU time of the cpu_baseline sample")
    ap.add_argument("--gathers", type=int, default=0,
                    help="override midpoints per GPU (profiling slices only)")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-parity", action="store_true")
    ap.add_argument("--no-sub", action="store_true", help="skip the crs_small sub-record")
    ap.add_argument("--parity-cells", type=int, default=0,
                    help="override the parity sample size (0 = 1%% CMP / 4096 CRS)")
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


def _free_port() -> int:
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def maybe_relaunch(args) -> None:
    """--gpus N is honoured: under torchrun WORLD_SIZE must equal N; outside
    it, N > 1 re-launches this script under torch.distributed.run with one
    process per GPU (NCCL).  Fewer visible GPUs than N is an error."""
    if "WORLD_SIZE" in os.environ:
        world = int(os.environ["WORLD_SIZE"])
        if world != args.gpus:
            print(json.dumps({"error": f"--gpus {args.gpus} but WORLD_SIZE={world}"}),
                  flush=True)
            sys.exit(2)
        return
    if args.gpus <= 1 or args.impl == "reference":
        return  # the reference arm is one CPU process (rank 0's work)
    import torch
    n = torch.cuda.device_count()
    if n < args.gpus:
        print(json.dumps({"error": f"--gpus {args.gpus} but only {n} GPU(s) visible"}),
              flush=True)
        sys.exit(2)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1",
           f"--nproc-per-node={args.gpus}", "--master-addr", "127.0.0.1",
           "--master-port", str(_free_port()), os.path.abspath(__file__)] + sys.argv[1:]
    sys.exit(subprocess.call(cmd))


# ---------------------------------------------------------------------------
# clocks during the timed region (B200_PROFILING.md clocks line)

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, gpu_index: int):
        self.gpu = gpu_index
        self.proc = None
        self.lines = []

    def start(self):
        try:
            self.proc = subprocess.Popen(
                ["nvidia-smi", f"--query-gpu={self.FIELDS}", "--format=csv,noheader,nounits",
                 "-lms", "200", "-i", str(self.gpu)],
                stdout=subprocess.PIPE, stderr=subprocess.DEVNULL, text=True)
            self.th = threading.Thread(target=self._read, daemon=True)
            self.th.start()
        except Exception:
            self.proc = None

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append(line.strip())

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        try:
            self.proc.wait(timeout=5)
        except Exception:
            self.proc.kill()
        self.th.join(timeout=2)
        sms, maxes, power, reasons = [], [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for ln in self.lines:
            f = [x.strip() for x in ln.split(",")]
            if len(f) < 9:
                continue
            try:
                sms.append(float(f[1]))
                maxes.append(float(f[2]))
                power.append(float(f[3]))
            except ValueError:
                continue
            for n, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        if not sms:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["no samples"]}
        sms.sort()
        return {"sm_mhz": sms[len(sms) // 2], "sm_max_mhz": max(maxes),
                "reasons": sorted(reasons), "samples": len(sms),
                "power_w_max": max(power) if power else None}


def physical_gpu(local: int) -> int:
    vis = os.environ.get("CUDA_VISIBLE_DEVICES")
    if vis:
        parts = [p for p in vis.split(",") if p.strip()]
        if local < len(parts) and parts[local].strip().isdigit():
            return int(parts[local])
    return local


# ---------------------------------------------------------------------------

def algorithmic_flops(valid: int, nominal: int, w: int) -> float:
    """12 + 7w flops per valid intersection, 12 per out-of-range one
    (bench.hpp:47-51)."""
    return valid * (12.0 + 7.0 * w) + (nominal - valid) * 12.0


def load_traffic(workload: str):
    """DRAM bytes (read + write) of the scan kernel per launch and per step,
    from the committed ncu launch list of the same command
    (profiles/traffic.json, tools/traffic_from_launches.py)."""
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            e = json.load(f).get(workload)
        if e is None:
            return None, None
        step = float(e["dram_bytes_per_step"])
        return step / max(int(e.get("scan_launches_per_step", 1)), 1), step
    except Exception:
        return None, None


def _proxy_velocities(wl):
    """The d2 operator's candidate list for the CRS reference proxy: as many
    velocities as the ABC search has candidates (the same per-candidate cost
    in the reference's kernel), linear over the workload's v range."""
    import numpy as np
    v = wl.config.grid()
    return np.linspace(float(v.min()), float(v.max()), wl.ncand).astype(np.float32)


def cpu_reference_sample(wl, ds, seconds: float, threads: int, kind: str = "auto",
                         rds=None):
    """Time the reference's CPU implementation on a bounded sample of output
    cells (row, t0) of the same workload, every candidate and every trace of
    each cell's sweep, on ``threads`` host threads.

    kind "reference": CMP — the UNMODIFIED reference kernels (oracle/_ref:
    velan's blocked scan_tile_blocked driven like scan_sweep,
    parallel_for_indexed over the threads), inputs in a velan::Dataset built
    once outside the timed call.  kind "reference_proxy": CRS — the ABC
    operator has no reference implementation, so the reference's blocked
    kernel runs its d2 operator through scan_central_cdp's sweep (same
    gathers, traces, window and candidate count).  kind "port": the C
    restatement of the ABC operator in the same blocked trace-outer form
    (oracle/semblance_oracle.c mode 2)."""
    import numpy as np

    import oracle
    G = ds.ncdps
    if kind == "auto":
        kind = "reference" if wl.op == "nmo" else "reference_proxy"
    if kind in ("reference", "reference_proxy") and not oracle.ref_available():
        kind = "port"
    ns = ds.ns
    rng = np.random.default_rng(5)
    tps = wl.traces_per_sweep(G) if wl.op != "nmo" else wl.traces_per_sweep()
    tps = tps[:G] if len(tps) >= G else np.full(G, tps[0])
    # CRS rows whose aperture is complete (the prefix's ends are truncated)
    halo = 0 if wl.op == "nmo" else int(round(wl.apm / wl.spec.spacing))
    r_lo, r_hi = halo, max(halo + 1, G - halo)
    # sample unit: a block of contiguous t0 at one midpoint (the blocked
    # kernels tile contiguous (t0, candidate) pairs, scan.hpp:130-165)
    blk = 64 if wl.op == "nmo" else 16
    if rds is None and kind != "port":
        rds = oracle.RefDataset(ds)
    vprox = _proxy_velocities(wl) if kind == "reference_proxy" else None

    def run(n_units):
        r0 = rng.integers(r_lo, r_hi, n_units)
        k0 = rng.integers(0, max(ns - blk, 1), n_units)
        rows = np.repeat(r0, blk).astype(np.int32)
        ks = (np.repeat(k0, blk) + np.tile(np.arange(blk), n_units)).astype(np.int32)
        order = np.lexsort((ks, rows))  # cells grouped by row (one sweep each)
        rows, ks = rows[order], ks[order]
        t = time.perf_counter()
        if kind == "reference":
            r = oracle.ref_run_cells_ds(rds, "nmo", wl.config.w, wl.config.grid(), rows, ks,
                                        variant=1, workers=threads)
        elif kind == "reference_proxy":
            r = oracle.ref_run_cells_ds(rds, "d2", wl.config.w, vprox, rows, ks,
                                        apm=wl.apm, variant=1, workers=threads)
        else:
            r = oracle.run_cells(ds, wl.op, wl.config.w, wl.config.grid(), rows, ks,
                                 apm=wl.apm, abc=wl.abc, mode=2, threads=threads)
        dt = time.perf_counter() - t
        evals = int(tps[rows].sum()) * wl.ncand * wl.config.w
        return dt, evals, r

    n0 = max(threads, 4)
    dt0, ev0, _ = run(n0)
    n = int(max(n0, 0.9 * n0 * seconds / max(dt0, 1e-3)))
    n = (n // threads) * threads or threads
    dt, evals, r = run(n)
    what = {"reference": "velan::scan_tile_blocked (oracle/_ref), NMO",
            "reference_proxy": "velan::scan_tile_blocked (oracle/_ref) on the d2 operator "
                               f"through scan_central_cdp's sweep, {wl.ncand} velocities",
            "port": "C restatement, blocked trace-outer (oracle mode 2)"}[kind]
    return {"value": evals / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n} seeded blocks of {blk} contiguous t0 (of {G} midpoints x {ns} t0), "
                      f"all {wl.ncand} candidates x traces in aperture, w={wl.config.w}: "
                      f"{dt:.2f} s; {what}",
            "valid_evals_per_s": r.valid * wl.config.w / dt}


# ---------------------------------------------------------------------------
# parity sample: the gathered picks of the whole line vs the CPU oracle

def parity_sample(wl, n_line: int, line_rows, picks, n_cells: int = 0, seed: int = 4242):
    """Check a seeded sample of the gathered picks (``picks`` = host arrays
    [rows, ns] of best index, semblance, stack for the line's output rows
    ``line_rows`` (gather indices of the line)) against the CPU oracle.

    CMP: 1 % of the cells — up to 128 seeded gathers per 8192, the same
    number of seeded t0 in each — checked with the reference's own blocked
    kernel (oracle/_ref, bitwise equal to the restatement's mode 0).  CRS: a
    fixed 4096-cell sample (64 seeded midpoints x 64 seeded t0; the 1 %
    BASELINE asks for is ~6e4 CPU-seconds at CRS scale),
    checked with the restatement (mode 2, bitwise the fp32 operator order).
    The bar (oracle.hpp:183-230 semantics): the GPU pick equals the oracle's
    except where the oracle's top two are within 1e-4 relative; semblance at
    the GPU pick within 1e-4 relative of the oracle's value of that candidate;
    stack within 1e-4 relative + 1e-6 max|sample|."""
    import numpy as np

    import oracle
    bi, bs, bst = picks
    R, ns = bi.shape
    rng = np.random.default_rng(seed)
    t_start = time.perf_counter()
    lib = oracle.synth_lib()
    if wl.op == "nmo":
        n_target = n_cells or max(1, int(round(0.01 * R * ns)))
        n_g = min(R, max(16, R // 64), n_target)
        per = min(ns, int(math.ceil(n_target / n_g)))
        rows = np.sort(rng.choice(R, n_g, replace=False))
        groups = []
        for r in rows:
            ks = np.sort(rng.choice(ns, per, replace=False)).astype(np.int32)
            groups.append((int(r), ks))
        # the sampled gathers, generated like the ranks generated them
        samples = [(r, int(line_rows[r]), ks) for r, ks in groups]
        gl = [g for _, g, _ in samples]
        parts = [wl.spec.generate(first=g, count=1, n_line=n_line, lib=lib) for g in gl]
        ds = _concat(parts)
        crow = np.concatenate([np.full(len(ks), i, np.int32) for i, (_, _, ks) in enumerate(samples)])
        ck = np.concatenate([ks for _, _, ks in samples]).astype(np.int32)
        gr = np.concatenate([np.full(len(ks), r, np.int64) for r, _, ks in samples])
        use_ref = oracle.ref_available()
        kind = "reference (oracle/_ref scan_tile_blocked)" if use_ref else "port (mode 2)"
        ref_idx = np.empty(len(ck), np.int32)
        ref_s = np.empty(len(ck), np.float32)
        ref_st = np.empty(len(ck), np.float32)
        ref_at = np.empty(len(ck), np.float64)
        gap = np.empty(len(ck), np.float64)
        rds = oracle.RefDataset(ds) if use_ref else None
        gidx_all = bi[gr, ck]
        step = 16384
        for a in range(0, len(ck), step):
            sl = slice(a, a + step)
            if use_ref:
                r = oracle.ref_run_cells_ds(rds, "nmo", wl.config.w, wl.config.grid(),
                                            crow[sl], ck[sl], variant=1, matrix=True)
            else:
                r = oracle.run_cells(ds, "nmo", wl.config.w, wl.config.grid(), crow[sl],
                                     ck[sl], mode=2, matrix=True)
            _reduce_chunk(r, gidx_all[sl], sl, ref_idx, ref_s, ref_st, ref_at, gap)
        samples_abs = float(np.abs(ds.samples).max())
        n_rows_s = len(groups)
    else:
        n_target = n_cells or 4096
        halo = int(math.ceil(wl.apm / wl.spec.spacing)) + 1
        n_r = min(R, 64)
        per = min(ns, int(math.ceil(n_target / n_r)))
        rows = np.sort(rng.choice(R, n_r, replace=False))
        kind = "port (oracle mode 2, the fp32 operator order; bitwise mode 0)"
        ref_idx, ref_s, ref_st, ref_at, gap, gr_l, ck_l = [], [], [], [], [], [], []
        samples_abs = 0.0
        for r in rows:
            g = int(line_rows[r])
            lo, hi = max(0, g - halo), min(n_line, g + halo + 1)
            ds = wl.spec.generate(first=lo, count=hi - lo, n_line=n_line, lib=lib)
            samples_abs = max(samples_abs, float(np.abs(ds.samples).max()))
            ks = np.sort(rng.choice(ns, per, replace=False)).astype(np.int32)
            crow = np.full(len(ks), g - lo, np.int32)  # cdp_id order = line order
            rr = oracle.run_cells(ds, wl.op, wl.config.w, wl.config.grid(), crow, ks,
                                  apm=wl.apm, abc=wl.abc, mode=2, matrix=True)
            n = len(ks)
            o_idx = np.empty(n, np.int32)
            o_s = np.empty(n, np.float32)
            o_st = np.empty(n, np.float32)
            o_at = np.empty(n, np.float64)
            o_gap = np.empty(n, np.float64)
            _reduce_chunk(rr, bi[r, ks], slice(0, n), o_idx, o_s, o_st, o_at, o_gap)
            ref_idx.append(o_idx), ref_s.append(o_s), ref_st.append(o_st)
            ref_at.append(o_at), gap.append(o_gap)
            gr_l.append(np.full(n, r, np.int64)), ck_l.append(ks)
        ref_idx, ref_s, ref_st = np.concatenate(ref_idx), np.concatenate(ref_s), np.concatenate(ref_st)
        ref_at, gap = np.concatenate(ref_at), np.concatenate(gap)
        gr, ck = np.concatenate(gr_l), np.concatenate(ck_l)
        n_rows_s = n_r
    g_idx = bi[gr, ck]
    g_s = bs[gr, ck].astype(np.float64)
    g_st = bst[gr, ck].astype(np.float64)
    same = g_idx == ref_idx
    unexcused = int((~same & (gap >= RTOL)).sum())
    rel = np.abs(g_s - ref_at) / np.maximum(np.abs(ref_at), 1e-12)
    floor = 1e-6 * samples_abs
    d_st = np.abs(g_st[same] - ref_st[same].astype(np.float64))
    st_bad = int((d_st > RTOL * np.abs(ref_st[same]) + floor).sum())
    st_rel = float((d_st / np.maximum(np.abs(ref_st[same]), 1e-12)).max()) if same.any() else 0.0
    return {"cells": int(len(ck)), "rows": int(n_rows_s), "line_cells": int(R * ns),
            "fraction": len(ck) / float(R * ns), "max_rel": float(rel.max()) if len(rel) else 0.0,
            "semblance_over_tol": int((rel > RTOL).sum()),
            "pick_mismatches": int((~same).sum()), "tie_excused": int((~same & (gap < RTOL)).sum()),
            "unexcused_mismatches": unexcused, "stack_over_tol": st_bad,
            "stack_max_rel": st_rel, "oracle_kind": kind,
            "seconds": time.perf_counter() - t_start,
            "pass": bool(unexcused == 0 and (rel <= RTOL).all() and st_bad == 0)}


def _reduce_chunk(r, gidx, sl, ref_idx, ref_s, ref_st, ref_at, gap):
    import numpy as np
    m = r.matrix
    n = m.shape[0]
    ref_idx[sl] = r.best_idx
    ref_s[sl] = r.best_semblance
    ref_st[sl] = r.best_stack
    ref_at[sl] = m[np.arange(n), gidx]
    part = -np.partition(-m, 1, axis=1)[:, :2]
    top = np.maximum(part[:, 0], part[:, 1]).astype(np.float64)
    sec = np.minimum(part[:, 0], part[:, 1]).astype(np.float64)
    gap[sl] = np.abs(top - sec) / np.maximum(np.abs(top), 1e-12)


def _concat(parts):
    import numpy as np

    from paper_1907_11678_b200 import Dataset
    return Dataset(np.concatenate([p.samples for p in parts]),
                   np.concatenate([p.coords for p in parts]),
                   np.concatenate([p.ntraces for p in parts]),
                   np.concatenate([p.cdp_id for p in parts]), parts[0].dt_us)


# ---------------------------------------------------------------------------

def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref)
    on the host cores, same workload/metric; rank 0 only.  Inputs come from
    the host generator built into oracle/ (no GPU library is loaded)."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    import oracle
    from paper_1907_11678_b200 import configs
    wl = configs.WORKLOADS[args.workload]()
    threads = os.cpu_count() or 1
    # a gather sample of the same workload, generated like ours (a line
    # prefix; CRS sweeps need their neighbours, so keep enough gathers)
    ds = wl.spec.generate(count=min(wl.spec.n_gathers, 256), lib=oracle.synth_lib())
    kind = "reference" if wl.op == "nmo" else "reference_proxy"
    rds = oracle.RefDataset(ds) if oracle.ref_available() else None
    per_step = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
    for _ in range(args.warmup):
        cpu_reference_sample(wl, ds, per_step, threads, kind, rds)
    vals = []
    last = None
    for _ in range(args.steps):
        last = cpu_reference_sample(wl, ds, per_step, threads, kind, rds)
        vals.append(last["value"])
    value = sorted(vals)[len(vals) // 2]
    line = {
        "metric": METRIC, "value": value, "unit": UNIT, "impl": "reference",
        "n_gpus": args.gpus, "steps": args.steps, "warmup": args.warmup,
        # the full step (the workload's nominal evals) at the sampled rate
        "ms_per_step": wl.nominal_evals() / value * 1e3 if value else None,
        "ms_per_step_basis": "extrapolated: nominal evals of one full step / sampled rate",
        "higher_is_better": True,
        "scaling": "strong" if wl.name.startswith("scaling_") else "weak",
        "vs_baseline": None, "dtype": "f32", "data": "synthetic",
        "config": {"workload": wl.name, "sample": last["sample"]},
        "cpu_baseline": {"value": value, "unit": UNIT, "cores": threads,
                         "kind": last["kind"], "sample": last["sample"]},
        "e2e": {"value": value, "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)


# ---------------------------------------------------------------------------

class Ctx:
    def __init__(self, rank, world, local, pg):
        self.rank, self.world, self.local, self.pg = rank, world, local, pg

    def barrier(self):
        import torch
        if self.pg is not None:
            self.pg.barrier()
        torch.cuda.synchronize()


def measure(ctx: Ctx, args, wl_name: str, steps: int, warmup: int, sub: bool = False):
    """Time ``steps`` scans of one workload (device-resident value + e2e),
    then gather the picks, check the parity sample, time the CPU baseline."""
    import numpy as np
    import torch

    from paper_1907_11678_b200 import Dataset, Engine, _native, configs
    from paper_1907_11678_b200.sharding import Shard, block_range, weak_shard
    rank, world, local = ctx.rank, ctx.world, ctx.local
    dev = f"cuda:{local}"
    wl = configs.WORKLOADS[wl_name]()
    wl.config.kernel_variant = args.variant
    if args.gathers > 0 and not sub:
        from dataclasses import replace
        wl.spec = replace(wl.spec, n_gathers=args.gathers)
    G = wl.spec.n_gathers
    # weak scaling: rank r owns midpoints [r*G, (r+1)*G) of a world*G line;
    # CRS ranks also hold the +-aperture halo (replicated, no exchange) and
    # restrict their outputs to the owned block.  scaling_*: strong scaling
    # of the fixed line (sharding.block_range).
    halo = 0 if wl.op == "nmo" else int(math.ceil(wl.apm / wl.spec.spacing)) + 1
    strong = wl.name.startswith("scaling_")
    if strong:
        n_line = G
        b, e = block_range(n_line, world, rank)
        shard = Shard(rank, (b, e), (max(0, b - halo), min(n_line, e + halo)))
    else:
        n_line = G * world
        shard = weak_shard(G, rank, halo, world)
    G = shard.row_count  # output rows of this rank
    lo, hi = shard.gathers
    rows = None if wl.op == "nmo" else (shard.row_first, shard.row_count)
    t_gen = time.perf_counter()
    ds = wl.spec.generate(first=lo, count=hi - lo, n_line=n_line)
    t_gen = time.perf_counter() - t_gen
    w = wl.config.w

    eng = Engine([local])
    # ---- device-resident value -------------------------------------------
    samples_dev = torch.from_numpy(ds.samples).to(dev)
    dsd = Dataset(samples_dev, ds.coords, ds.ntraces, ds.cdp_id, ds.dt_us)
    plan = eng.plan(dsd, wl.config, op=wl.op, apm=wl.apm, abc=wl.abc, rows=rows)
    ns = ds.ns
    bi = torch.empty((G, ns), dtype=torch.int32, device=dev)
    bs = torch.empty((G, ns), dtype=torch.float32, device=dev)
    bst = torch.empty((G, ns), dtype=torch.float32, device=dev)
    stream = torch.cuda.current_stream()
    for _ in range(warmup):
        res = plan.execute(bi, bs, bst, stream=stream)

    # inputs smaller than 4x L2 (126 MB): flush L2 between timed steps by
    # writing a 512 MB buffer outside the timed events; larger inputs (CMP
    # large: 3.9 GB of samples + the FAST tables per GPU) need no flush
    in_bytes = int(ds.samples.nbytes) * 5  # samples + the FAST (pair, E/G) tables
    flush = None
    if in_bytes < 4 * 126 * 2**20:
        flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=dev)
    clocks = ClockSampler(physical_gpu(local))
    ctx.barrier()
    clocks.start()
    kernel_ms = 0.0
    ms = 0.0
    for _ in range(steps):
        if flush is not None:
            flush.fill_(1.0)
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record(stream)
        res = plan.execute(bi, bs, bst, stream=stream)
        e1.record(stream)
        e1.synchronize()
        ms += e0.elapsed_time(e1)
        kernel_ms += res.kernel_ms
    # short runs (CMP small: ~0.5 ms per step) end before the 200 ms clock
    # sampler has looked: keep the same load going, untimed, for 0.6 s
    t_load = time.perf_counter()
    while ms < 600.0 and time.perf_counter() - t_load < 0.6:
        plan.execute(bi, bs, bst, stream=stream)
        torch.cuda.synchronize()
    ctx.barrier()
    clk = clocks.stop()
    launches = plan.launches() * steps
    valid, nominal = int(res.valid_intersections), int(res.nominal_intersections)

    evals_rank = nominal * w * steps
    t = torch.tensor([ms], dtype=torch.float64, device=dev)
    tot = torch.tensor([float(evals_rank), float(valid * w * steps)],
                       dtype=torch.float64, device=dev)
    if ctx.pg is not None:
        ctx.pg.all_reduce(t, op=ctx.pg.ReduceOp.MAX)
        ctx.pg.all_reduce(tot, op=ctx.pg.ReduceOp.SUM)
    ms_max = float(t.item())
    evals_all, valid_all = float(tot[0].item()), float(tot[1].item())
    value = evals_all / (ms_max * 1e-3)

    # roofline of the dominant kernel: algorithmic FP32 flops per launch /
    # average launch duration (CUDA events on the launch stream)
    flops_step = algorithmic_flops(valid, nominal, w)
    achieved_tf = flops_step * steps / (kernel_ms * 1e-3) / 1e12
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    nominal_peak = 2.0 * 128 * nsm * 1965e6 / 1e12
    import ctypes as C
    pm = C.c_double(0.0)
    _native.load().velan_gpu_measure_fp32_peak(local, C.byref(pm))
    traffic, traffic_step = load_traffic(wl.name)

    # ---- gather the picks of every rank to rank 0's host memory ----------
    t_gather = time.perf_counter()
    picks = gather_picks(ctx.pg, rank, world, (bi, bs, bst))
    t_gather = time.perf_counter() - t_gather

    # ---- e2e through the one-shot C-ABI with pinned host buffers ----------
    e2e = None
    if not args.no_e2e:
        pinned = torch.from_numpy(ds.samples).pin_memory()
        dsh = Dataset(pinned, ds.coords, ds.ntraces, ds.cdp_id, ds.dt_us)
        obi = torch.empty((G, ns), dtype=torch.int32).pin_memory()
        obs = torch.empty((G, ns), dtype=torch.float32).pin_memory()
        obst = torch.empty((G, ns), dtype=torch.float32).pin_memory()
        run = (lambda: eng.run_cmp(dsh, wl.config, out=(obi, obs, obst))) if wl.op == "nmo" \
            else (lambda: eng.run_crs(dsh, wl.config, wl.apm, wl.abc, out=(obi, obs, obst),
                                      rows=rows))
        run()  # warm-up (allocations cached in the context)
        k_e2e = max(1, min(steps, 3))
        ctx.barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            r = run()
        ctx.barrier()
        e2e_s = (time.perf_counter() - t0) / k_e2e
        te = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        if ctx.pg is not None:
            ctx.pg.all_reduce(te, op=ctx.pg.ReduceOp.MAX)
        e2e_s = float(te.item())
        h2d = ds.samples.nbytes + ds.ntraces.nbytes + (hi - lo) * ds.fold * 4 + 4 * ns
        d2h = 3 * 4 * G * ns
        e2e = {"value": (evals_all / steps) / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_s * 1e3,
               "api": f"velan_gpu_{'cmp' if wl.op == 'nmo' else 'crs'}",
               "picks_equal_resident": bool(np.array_equal(np.asarray(obi), bi.cpu().numpy()))}
    launches_per_step = plan.launches()
    plan.close()
    eng.close()

    out = None
    if rank == 0:
        # ---- parity sample of the gathered line -------------------------------
        par = None
        if not args.no_parity:
            line_rows = np.arange(n_line)  # contiguous blocks: row r = gather r
            try:
                par = parity_sample(wl, n_line, line_rows, picks, args.parity_cells)
            except Exception as ex:  # reported, not fatal
                par = {"error": f"{type(ex).__name__}: {ex}"}
        # ---- CPU baseline (rank 0, N = 1) -------------------------------------
        cpu = None
        if world == 1 and not args.no_cpu:
            try:
                import oracle
                # same procedure as --impl reference: a 256-midpoint prefix
                # of the line, one untimed warm-up sample, then the timed one
                ds_cpu = wl.spec.generate(count=min(wl.spec.n_gathers, 256),
                                          lib=oracle.synth_lib())
                threads = os.cpu_count() or 1
                rds = oracle.RefDataset(ds_cpu) if oracle.ref_available() else None
                cpu_reference_sample(wl, ds_cpu, 2.0, threads, "auto", rds)
                cpu = cpu_reference_sample(wl, ds_cpu, args.cpu_seconds, threads, "auto", rds)
                if wl.op != "nmo":  # the ABC restatement itself, same sampler
                    port = cpu_reference_sample(wl, ds_cpu, max(2.0, args.cpu_seconds / 2),
                                                threads, "port")
                    cpu["port"] = {k: port[k] for k in ("value", "kind", "sample")}
            except Exception as ex:  # reported, not fatal
                cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(),
                       "kind": "unavailable", "sample": f"error: {ex}"}
        out = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": steps, "warmup": warmup, "ms_per_step": ms_max / steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded generator, BASELINE.json shapes)",
            "config": {"workload": wl.name, "midpoints_per_gpu": G, "line_midpoints": n_line,
                       "traces": wl.spec.n_traces,
                       "ns": ns, "dt_us": wl.spec.dt_us, "candidates": wl.ncand, "w": w,
                       "operator": wl.op, "variant": args.variant,
                       "tolerance": "semblance 1e-4 rel; picks identical up to near-ties "
                                    "(top-2 within 1e-4); stack 1e-4 rel + 1e-6 max|a|"
                                    if args.variant == "fast" else "bitwise",
                       "l2": (f"L2 flushed between timed steps (512 MB write; inputs "
                              f"{in_bytes / 2**20:.0f} MB incl. tables)") if flush is not None
                       else f"inputs {in_bytes / 2**30:.1f} GB/GPU incl. tables > 126 MB L2 "
                            f"(no flush needed)",
                       "parallelism": f"dp{world} (contiguous midpoint blocks"
                                      + (")" if wl.op == "nmo" else
                                         f", +-{halo} midpoint replicated halo)")},
            "valid_evals_per_s": valid_all / (ms_max * 1e-3),
            "roofline": {"bound": "fp32", "achieved": achieved_tf, "peak": nominal_peak,
                         "unit": "TFLOP/s", "frac": achieved_tf / nominal_peak,
                         "traffic": traffic,
                         "traffic_per_step": traffic_step,
                         "traffic_source": "profiles/traffic.json (ncu launch list, "
                                           "dram__bytes_read + dram__bytes_write of the "
                                           "scan kernel, per launch)",
                         "peak_source": "nominal FP32 FMA peak 2 x 128 x SMs x 1965 MHz "
                                        "(MEASURED_PEAKS.json has no FP32 figure)",
                         "measured_fma_peak": pm.value,
                         "frac_of_measured_fma": achieved_tf / pm.value if pm.value else None,
                         "flops_per_step": flops_step,
                         "kernel_ms_per_step": kernel_ms / steps,
                         "launches_per_step": launches_per_step},
            "clocks": clk,
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "parity_sample": par,
            "gather_s": t_gather,
            "gen_s": t_gen,
        }
    return out


def gather_picks(pg, rank: int, world: int, picks):
    """Gather every rank's picks (best index int32, semblance, stack, each
    [rows_r, ns] on the rank's device) to rank 0's host memory, in rank order
    (= line order: the blocks are contiguous).  One collective (gather) after
    the timed region — the only data collective of the run.  Works for NCCL
    (CUDA tensors) and gloo (CPU tensors).  Returns numpy arrays on rank 0,
    None elsewhere."""
    import torch
    bi, bs, bst = picks
    if pg is None or world == 1:
        return (bi.cpu().numpy(), bs.cpu().numpy(), bst.cpu().numpy())
    rows, ns = bi.shape
    counts = [None] * world
    pg.all_gather_object(counts, int(rows))
    mx = max(counts)
    packed = torch.zeros((3, mx, ns), dtype=torch.float32, device=bi.device)
    packed[0, :rows] = bi.view(torch.float32)
    packed[1, :rows] = bs
    packed[2, :rows] = bst
    bufs = [torch.empty_like(packed) for _ in range(world)] if rank == 0 else None
    pg.gather(packed, bufs, dst=0)
    if rank != 0:
        return None
    host = [b.cpu() for b in bufs]
    cat = [torch.cat([h[i, :c] for h, c in zip(host, counts)]) for i in range(3)]
    return (cat[0].contiguous().view(torch.int32).numpy(), cat[1].numpy(), cat[2].numpy())


def main():
    args = parse()
    maybe_relaunch(args)
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist
    ctx = Ctx(rank, world, local, pg)
    line = measure(ctx, args, args.workload, args.steps, args.warmup)
    if args.workload == "cmp_large" and args.gathers == 0 and not args.no_sub:
        # BASELINE's CRS operator beside the CMP headline: configs[2] in full
        sub = measure(ctx, args, "crs_small", max(args.steps, 5), max(args.warmup, 3), sub=True)
        if rank == 0:
            line["crs_small"] = {k: sub[k] for k in (
                "value", "unit", "ms_per_step", "steps", "warmup", "config",
                "valid_evals_per_s", "roofline", "clocks", "gpu_launches", "e2e",
                "cpu_baseline", "parity_sample")}
            line["gpu_launches"] += sub["gpu_launches"]
    if rank == 0:
        print(json.dumps(line), flush=True)
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
