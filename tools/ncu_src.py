#!/usr/bin/env python
"""Per-instruction view of an ncu report's SASS source page (no GPU needed):
    python tools/ncu_src.py rep.ncu-rep [min_exec_frac]
prints address, SASS, executions, samples, shared wavefronts (actual/ideal)
and the dominant stall reasons of every instruction executed at least
min_exec_frac x the hottest instruction."""
import csv, subprocess, sys
rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.5
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:]]
def num(v):
    try: return float(v)
    except: return 0.0
mx = max(num(d["Instructions Executed"]) for d in rows if "FFMA2" in d["Source"])
stall_cols = [c for c in h if c.startswith("stall_") or "Stall" in c and "(" not in c]
tot_s = sum(num(d["# Samples"]) for d in rows)
tot_w = sum(num(d.get("L1 Wavefronts Shared", 0)) for d in rows)
print(f"total samples {tot_s:.0f}, total shared wavefronts {tot_w:.3e}")
for d in rows:
    e = num(d["Instructions Executed"])
    if e < frac * mx: continue
    wf = num(d.get("L1 Wavefronts Shared", 0)); wi = num(d.get("L1 Wavefronts Shared Ideal", 0))
    extra = f" wf/exec {wf/e:.2f} (ideal {wi/e:.2f})" if wf else ""
    st = sorted(((num(d[c]), c[6:]) for c in h if c.startswith('stall_') and 'Not Issued' not in c), reverse=True)[:3]
    sts = ' '.join(f"{n}:{v:.0f}" for v, n in st if v > 0)
    print(f"{d['Address'][-5:]} {e/mx:5.2f} s={num(d['# Samples']):7.0f} {d['Source'].strip()[:60]:60s}{extra} | {sts}")
