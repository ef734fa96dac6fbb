#!/usr/bin/env python
"""bench.py — BASELINE.json metric: semblance evals/s of the CMP/CRS parameter
search on N B200s, with the FP32 roofline fraction and the host-CPU reference.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
                    [--workload cmp_large|cmp_small|crs_small|crs_large|
                                scaling_cmp|scaling_crs]

A "step" is one pass of the scan over one rank's workload: the BASELINE
configuration itself (default configs[1], CMP large: 8192 gathers x 60 traces
x 2000 samples, 401 candidates, w = 15).  Multi-GPU is weak scaling: every
rank scans its own contiguous block of a longer line (no collective on the
data path; only a barrier and the max-over-ranks timing reduction).  The
BASELINE scaling sweep (--workload scaling_cmp: 65536 gathers, scaling_crs:
32768 midpoints) is strong scaling: the fixed line split into contiguous
blocks (CRS blocks with their replicated +-aperture halo).

One JSON line on rank 0.  ``value`` = nominal evals (midpoints x t0 x
candidates x traces x w, BASELINE's unit) of all ranks / the max over ranks of
the device time of K steps with the input resident in HBM (3.9 GB per GPU,
larger than the 126 MB L2, so no flush is needed).  ``e2e`` = the same metric
through the one-shot C-ABI call velan_gpu_cmp/crs from pinned host buffers
(H2D of the samples and D2H of the picks inside the timed region).
"""
from __future__ import annotations

import argparse
import json
import math
import os
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "semblance evals/sec"
UNIT = "evals/s"


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
    return ap.parse_args()


def dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


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
    p = os.path.join(ROOT, "profiles", "traffic.json")
    try:
        with open(p) as f:
            d = json.load(f)
        e = d.get(workload)
        # DRAM bytes (read + write) of the scan kernel per step, from the
        # committed ncu launch list of the same command
        return None if e is None else float(e["dram_bytes_per_step"])
    except Exception:
        return None


def cpu_reference_sample(wl, ds, seconds: float, threads: int):
    """Time the UNMODIFIED reference kernels (oracle/_ref: velan's blocked
    scan_tile_blocked driven like scan_sweep, parallel_for_indexed over all
    host threads) on a bounded sample of output cells (row, t0) of the same
    workload, every candidate and every trace of each cell's sweep.  The
    ABC operator has no reference implementation: the C restatement
    (oracle/semblance_oracle.c, kind "port") is timed instead."""
    import numpy as np

    import oracle
    G = ds.ncdps
    ref_ok = oracle.ref_available() and wl.op == "nmo"
    kind = "reference" if ref_ok else "port"
    ns = ds.ns
    rng = np.random.default_rng(5)
    tps = wl.traces_per_sweep()
    # rows of the sample come from the generated gathers (a line prefix)
    tps = tps[:G] if len(tps) >= G else np.full(G, tps[0])

    # sample unit: a block of contiguous t0 at one midpoint (the reference's
    # blocked kernel tiles contiguous (t0, candidate) pairs, scan.hpp:130-165)
    blk = 64 if wl.op == "nmo" else 1

    def run(n_units):
        r0 = rng.integers(0, G, n_units)
        k0 = rng.integers(0, max(ns - blk, 1), n_units)
        rows = np.repeat(r0, blk).astype(np.int32)
        ks = (np.repeat(k0, blk) + np.tile(np.arange(blk), n_units)).astype(np.int32)
        order = np.lexsort((ks, rows))  # cells grouped by row (one sweep each)
        rows, ks = rows[order], ks[order]
        t = time.perf_counter()
        if ref_ok:
            r = oracle.ref_run_cells(ds, "nmo", wl.config.w, wl.config.grid(), rows, ks,
                                     variant=1, workers=threads)
        else:
            r = oracle.run_cells(ds, wl.op, wl.config.w, wl.config.grid(), rows, ks,
                                 apm=wl.apm, abc=wl.abc, threads=threads)
        dt = time.perf_counter() - t
        evals = int(tps[rows].sum()) * wl.ncand * wl.config.w
        return dt, evals, r

    n0 = threads * (4 if blk > 1 else 1)
    dt0, ev0, _ = run(n0)
    n = int(max(n0, 0.9 * n0 * seconds / max(dt0, 1e-3)))
    n = (n // threads) * threads or threads
    dt, evals, r = run(n)
    return {"value": evals / dt, "unit": UNIT, "cores": threads, "kind": kind,
            "sample": f"{n} seeded blocks of {blk} contiguous t0 (of {G} midpoints x {ns} t0), "
                      f"all {wl.ncand} candidates x traces in aperture, w={wl.config.w}: "
                      f"{dt:.2f} s",
            "valid_evals_per_s": r.valid * wl.config.w / dt}


# ---------------------------------------------------------------------------

def run_reference_arm(args):
    """--impl reference: the reference's own CPU implementation (oracle/_ref)
    on the host cores, same workload/metric; rank 0 only."""
    rank, world, _ = dist_env()
    if rank != 0:
        return
    from paper_1907_11678_b200 import configs
    wl = configs.WORKLOADS[args.workload]()
    threads = os.cpu_count() or 1
    # a gather sample of the same workload, generated like ours (a line
    # prefix; CRS sweeps need their neighbours, so keep enough gathers)
    ds = wl.spec.generate(count=min(wl.spec.n_gathers, 256))
    per_step = max(2.0, 60.0 / max(args.steps + args.warmup, 1))
    for _ in range(args.warmup):
        cpu_reference_sample(wl, ds, per_step, threads)
    vals = []
    last = None
    for _ in range(args.steps):
        last = cpu_reference_sample(wl, ds, per_step, threads)
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


def main():
    args = parse()
    if args.impl == "reference":
        run_reference_arm(args)
        return
    import numpy as np
    import torch

    rank, world, local = dist_env()
    torch.cuda.set_device(local)
    pg = None
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=torch.device("cuda", local))
        pg = dist

    from paper_1907_11678_b200 import Dataset, Engine, _native, configs
    wl = configs.WORKLOADS[args.workload]()
    wl.config.kernel_variant = args.variant
    if args.gathers > 0:
        from dataclasses import replace
        wl.spec = replace(wl.spec, n_gathers=args.gathers)
    G = wl.spec.n_gathers
    # weak scaling: rank r owns midpoints [r*G, (r+1)*G) of a world*G line;
    # CRS ranks also hold the +-aperture halo (replicated, no exchange) and
    # restrict their outputs to the owned block (sharding.weak_shard).
    # The BASELINE scaling sweep (scaling_cmp / scaling_crs: a fixed 65536-
    # gather / 32768-midpoint line) is strong scaling: rank r owns the
    # contiguous block sharding.block_range gives it, plus the halo.
    from paper_1907_11678_b200.sharding import Shard, block_range, weak_shard
    halo = 0 if wl.op == "nmo" else int(math.ceil(wl.apm / wl.spec.spacing)) + 1
    strong = wl.name.startswith("scaling_")
    if strong:
        n_line = G
        b, e = block_range(n_line, world, rank)
        shard = Shard(rank, (b, e), (max(0, b - halo), min(n_line, e + halo)))
        G = e - b  # output rows of this rank
    else:
        n_line = G * world
        shard = weak_shard(G, rank, halo, world)
    lo, hi = shard.gathers
    rows = None if wl.op == "nmo" else (shard.row_first, shard.row_count)
    t_gen = time.perf_counter()
    ds = wl.spec.generate(first=lo, count=hi - lo, n_line=n_line)
    t_gen = time.perf_counter() - t_gen
    w = wl.config.w

    eng = Engine([local])
    # ---- device-resident value -------------------------------------------
    samples_dev = torch.from_numpy(ds.samples).to(f"cuda:{local}")
    dsd = Dataset(samples_dev, ds.coords, ds.ntraces, ds.cdp_id, ds.dt_us)
    plan = eng.plan(dsd, wl.config, op=wl.op, apm=wl.apm, abc=wl.abc, rows=rows)
    ns = ds.ns
    bi = torch.empty((G, ns), dtype=torch.int32, device=f"cuda:{local}")
    bs = torch.empty((G, ns), dtype=torch.float32, device=f"cuda:{local}")
    bst = torch.empty((G, ns), dtype=torch.float32, device=f"cuda:{local}")
    stream = torch.cuda.current_stream()
    for _ in range(args.warmup):
        res = plan.execute(bi, bs, bst, stream=stream)

    def barrier():
        if pg is not None:
            pg.barrier()
        torch.cuda.synchronize()

    # inputs smaller than 4x L2 (126 MB): flush L2 between timed steps by
    # writing a 512 MB buffer outside the timed events; larger inputs (CMP
    # large: 3.9 GB of samples + 15.7 GB of tables per GPU) need no flush
    in_bytes = int(ds.samples.nbytes) * 5  # samples + the FAST (pair, E/G) tables
    flush = None
    if in_bytes < 4 * 126 * 2**20:
        flush = torch.empty(512 * 2**20 // 4, dtype=torch.float32, device=f"cuda:{local}")
    clocks = ClockSampler(physical_gpu(local))
    barrier()
    clocks.start()
    kernel_ms = 0.0
    ms = 0.0
    for _ in range(args.steps):
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
    barrier()
    clk = clocks.stop()
    launches = plan.launches() * args.steps
    valid, nominal = int(res.valid_intersections), int(res.nominal_intersections)

    evals_rank = nominal * w * args.steps
    t = torch.tensor([ms], dtype=torch.float64, device=f"cuda:{local}")
    tot = torch.tensor([float(evals_rank), float(valid * w * args.steps)],
                       dtype=torch.float64, device=f"cuda:{local}")
    if pg is not None:
        pg.all_reduce(t, op=pg.ReduceOp.MAX)
        pg.all_reduce(tot, op=pg.ReduceOp.SUM)
    ms_max = float(t.item())
    evals_all, valid_all = float(tot[0].item()), float(tot[1].item())
    value = evals_all / (ms_max * 1e-3)

    # roofline of the dominant (only) kernel: algorithmic FP32 flops per
    # launch / average launch duration (CUDA events on the launch stream)
    flops_step = algorithmic_flops(valid, nominal, w)
    achieved_tf = flops_step * args.steps / (kernel_ms * 1e-3) / 1e12
    nsm = torch.cuda.get_device_properties(local).multi_processor_count
    nominal_peak = 2.0 * 128 * nsm * 1965e6 / 1e12
    import ctypes as C
    pm = C.c_double(0.0)
    _native.load().velan_gpu_measure_fp32_peak(local, C.byref(pm))
    traffic = load_traffic(wl.name)

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
        k_e2e = max(1, min(args.steps, 3))
        barrier()
        t0 = time.perf_counter()
        for _ in range(k_e2e):
            r = run()
        barrier()
        e2e_s = (time.perf_counter() - t0) / k_e2e
        te = torch.tensor([e2e_s], dtype=torch.float64, device=f"cuda:{local}")
        if pg is not None:
            pg.all_reduce(te, op=pg.ReduceOp.MAX)
        e2e_s = float(te.item())
        h2d = ds.samples.nbytes + ds.ntraces.nbytes + G * ds.fold * 4 + 4 * ns
        d2h = 3 * 4 * G * ns
        e2e = {"value": (evals_all / args.steps) / e2e_s, "unit": UNIT,
               "h2d_bytes_per_step": int(h2d), "d2h_bytes_per_step": int(d2h),
               "ms_per_step": e2e_s * 1e3, "api": f"velan_gpu_{'cmp' if wl.op == 'nmo' else 'crs'}"}

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        try:
            # same procedure as --impl reference: a 256-midpoint prefix of
            # the line, one untimed warm-up sample (pages, threads), then the
            # timed sample
            ds_cpu = wl.spec.generate(count=min(G, 256))
            cpu_reference_sample(wl, ds_cpu, 2.0, os.cpu_count() or 1)
            cpu = cpu_reference_sample(wl, ds_cpu, args.cpu_seconds, os.cpu_count() or 1)
        except Exception as ex:  # reported, not fatal
            cpu = {"value": None, "unit": UNIT, "cores": os.cpu_count(), "kind": "unavailable",
                   "sample": f"error: {ex}"}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_max / args.steps,
            "higher_is_better": True, "scaling": "strong" if strong else "weak",
            "vs_baseline": None,
            "dtype": "f32", "data": "synthetic (seeded generator, BASELINE.json shapes)",
            "config": {"workload": wl.name, "midpoints_per_gpu": G, "line_midpoints": n_line,
                       "traces": wl.spec.n_traces,
                       "ns": ns, "dt_us": wl.spec.dt_us, "candidates": wl.ncand, "w": w,
                       "operator": wl.op, "variant": args.variant,
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
                         "peak_source": "nominal FP32 FMA peak 2 x 128 x SMs x 1965 MHz "
                                        "(MEASURED_PEAKS.json has no FP32 figure)",
                         "measured_fma_peak": pm.value,
                         "frac_of_measured_fma": achieved_tf / pm.value if pm.value else None,
                         "flops_per_step": flops_step,
                         "kernel_ms_per_step": kernel_ms / args.steps,
                         "launches_per_step": plan.launches()},
            "clocks": clk,
            "gpu_launches": launches,
            "e2e": e2e,
            "cpu_baseline": cpu,
            "gen_s": t_gen,
        }
        print(json.dumps(line), flush=True)
    plan.close()
    eng.close()
    if pg is not None:
        pg.destroy_process_group()


if __name__ == "__main__":
    main()
