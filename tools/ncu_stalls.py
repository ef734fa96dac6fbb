#!/usr/bin/env python
"""Stall-reason totals of an ncu report's SASS source page, split into the
hot loop (instructions executed >= frac x the hottest FFMA2) and the rest:
    python tools/ncu_stalls.py rep.ncu-rep [frac]"""
import csv, subprocess, sys
from collections import Counter
rep = sys.argv[1]
frac = float(sys.argv[2]) if len(sys.argv) > 2 else 0.9
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
r = list(csv.reader(out.splitlines()))
h = r[1]
rows = [dict(zip(h, x)) for x in r[2:]]
def num(v):
    try: return float(v)
    except: return 0.0
mx = max(num(d["Instructions Executed"]) for d in rows if "FFMA2" in d["Source"])
cols = [c for c in h if c.startswith("stall_") and "Not Issued" not in c]
loop, rest = Counter(), Counter()
nl = 0
ops = Counter()
for d in rows:
    e = num(d["Instructions Executed"])
    tgt = loop if e >= frac * mx else rest
    if e >= frac * mx:
        nl += 1
        ops[d["Source"].split()[0].split(".")[0] if not d["Source"].strip().startswith("@") else d["Source"].split()[1].split(".")[0]] += 1
    for c in cols:
        tgt[c[6:]] += num(d[c])
tl, tr = sum(loop.values()), sum(rest.values())
print(f"loop instructions {nl}; samples loop {tl:.0f} ({tl/(tl+tr):.1%}), rest {tr:.0f}")
print("loop:", ", ".join(f"{k} {v/tl:.1%}" for k, v in loop.most_common(10)))
print("rest:", ", ".join(f"{k} {v/tr:.1%}" for k, v in rest.most_common(8)))
print("loop ops:", dict(ops.most_common()))
