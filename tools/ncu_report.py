#!/usr/bin/env python
"""Summarise an ncu --set full report of the scan kernel into markdown.

    python tools/ncu_report.py gpurun_out/prof.ncu-rep "title" > profiles/x.md

Reads the report with the ncu CLI (no GPU needed): speed-of-light, pipe
utilisation, issue activity, shared-memory wavefronts/conflicts, DRAM bytes,
warp-stall breakdown and the hot-loop instruction mix (SASS executed counts).
"""
import csv
import subprocess
import sys
from collections import Counter


def raw(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"],
                         capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[0], row)) for row in r[2:]]


def source(rep):
    out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv",
                          "--print-source", "sass"], capture_output=True, text=True).stdout
    r = list(csv.reader(out.splitlines()))
    return [dict(zip(r[1], row)) for row in r[2:]]


def main():
    rep = sys.argv[1]
    title = sys.argv[2] if len(sys.argv) > 2 else rep
    print(f"# {title}\n")
    print(f"Source report: `{rep}` (ncu --set full --clock-control none --import-source on)\n")
    keys = [
        ("gpu__time_duration.sum", "duration (ms)"),
        ("launch__grid_size", "grid (CTAs)"),
        ("launch__block_size", "block"),
        ("launch__registers_per_thread", "registers/thread"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "achieved occupancy %"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue slots busy %"),
        ("smsp__inst_executed.sum", "warp instructions"),
        ("sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active", "FMA pipe %"),
        ("sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active", "FMA pipe cycles active %"),
        ("sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active", "ALU pipe %"),
        ("sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active", "LSU pipe %"),
        ("sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active", "XU (MUFU/conv) pipe %"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum", "shared-load wavefronts"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum", "shared-load bank conflicts"),
        ("dram__bytes_read.sum", "DRAM read"),
        ("dram__bytes_write.sum", "DRAM write"),
        ("dram__throughput.avg.pct_of_peak_sustained_elapsed", "DRAM throughput %"),
    ]
    for d in raw(rep):
        print(f"## `{d.get('Kernel Name')}`\n")
        print("| metric | value |\n|---|---|")
        for k, name in keys:
            if k in d:
                print(f"| {name} (`{k}`) | {d[k]} |")
        st = {k.replace("smsp__pcsamp_warps_issue_stalled_", ""): float(v)
              for k, v in d.items()
              if k.startswith("smsp__pcsamp_warps_issue_stalled_") and not k.endswith("not_issued")
              and v not in ("", "n/a")}
        tot = sum(st.values()) or 1.0
        print("\n**Warp-state samples** (share of all samples): " +
              ", ".join(f"{k} {100 * v / tot:.1f}%" for k, v in sorted(st.items(), key=lambda x: -x[1])[:10]))
    src = source(rep)
    if src:
        # the hot loop = the most executed FFMA (spin-wait loops excluded)
        top = max(int(s.get("Instructions Executed") or 0) for s in src
                  if "FFMA" in s.get("Source", ""))
        cnt = Counter()
        for s in src:
            n = int(s.get("Instructions Executed") or 0)
            if 0.7 * top <= n <= 1.3 * top:
                t = s["Source"].strip()
                op = (t.split()[1] if t.startswith("@") else t.split()[0]).split(".")[0]
                cnt[op] += n
        base = max(cnt.values()) / 37.0 if cnt else 1.0
        iters = top
        print(f"\n**Hot-loop SASS mix** (instructions executed ≥ 70 % of the hottest, per "
              f"hottest-instruction execution, i.e. per trace iteration of a warp):\n")
        print(", ".join(f"{k} {v / iters:.1f}" for k, v in cnt.most_common(30)))
        print(f"\nTotal per trace iteration: {sum(cnt.values()) / iters:.1f} warp instructions")


if __name__ == "__main__":
    main()
