#!/usr/bin/env python
"""profiles/traffic.json from an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) of
`python bench.py --workload W --steps 1 --warmup 1 --no-e2e --no-cpu --no-parity --no-sub`
(one warm-up execute, then the measured one: each execute is a sequence of
per-wave table launches + scan launches).  The measured step = the second
half of the scan launches and the table launches among them.

    python tools/traffic_from_launches.py launches.csv workload midpoints source_note
"""
import csv
import json
import os
import sys
from collections import defaultdict

path, wl, mids, note = sys.argv[1], sys.argv[2], int(sys.argv[3]), sys.argv[4]
k = defaultdict(dict)
names = {}
hdr = None
for r in csv.reader(open(path)):
    if r and r[0] == "ID":
        hdr = {n: i for i, n in enumerate(r)}
        continue
    if hdr and len(r) > hdr["Metric Value"] and r[0].isdigit():
        k[int(r[0])][r[hdr["Metric Name"]]] = float(r[hdr["Metric Value"]].replace(",", ""))
        names[int(r[0])] = r[hdr["Kernel Name"]]
ids = sorted(k)
ours = [i for i in ids if "velan_gpu::" in names[i]]
scan = [i for i in ours if "semblance_scan_kernel" in names[i]]
half = scan[len(scan) // 2:]
first_tab = max([i for i in ours if i < half[0] and "semblance_scan" not in names[i]] or [half[0]])
step = [i for i in ours if first_tab <= i <= half[-1]]
dram = lambda i: k[i]["dram__bytes_read.sum"] + k[i]["dram__bytes_write.sum"]  # noqa: E731
t = lambda i: k[i]["gpu__time_duration.sum"]  # noqa: E731
scan_dram = sum(dram(i) for i in half)
out = {}
p = "profiles/traffic.json"
if os.path.exists(p):
    out = json.load(open(p))
out[wl] = {
    "kernel": names[half[0]].split("(")[0].replace("void ", ""),
    "scan_launches_per_step": len(half),
    "launches_per_step": len(step),
    "dram_bytes_per_step": scan_dram,
    "dram_bytes_per_midpoint": scan_dram / mids,
    "table_kernel_dram_bytes_per_step": sum(dram(i) for i in step if i not in half),
    "scan_share_of_step_time": sum(t(i) for i in half) / sum(t(i) for i in step),
    "source": note}
json.dump(out, open(p, "w"), indent=1)
print(json.dumps(out[wl], indent=1))
