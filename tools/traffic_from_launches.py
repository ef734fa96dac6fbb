#!/usr/bin/env python
"""profiles/traffic.json from an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) of `python bench.py --steps 1
--warmup 1 --no-e2e --no-cpu` (CMP large: one step = 4 wave launches of the scan
kernel over 8192 midpoints, preceded by warm-up launches).

    python tools/traffic_from_launches.py launches.csv source_note
"""
import csv, json, sys
from collections import defaultdict

path, note = sys.argv[1], sys.argv[2]
k = defaultdict(dict)
names = {}
for r in csv.reader(open(path)):
    if len(r) > 14 and r[0].isdigit():
        k[int(r[0])][r[12]] = float(r[14].replace(",", ""))
        names[int(r[0])] = r[4]
ids = sorted(k)
scan = [i for i in ids if "semblance_scan_kernel" in names[i]]
# the timed step is the last 4 scan launches (and their table launches)
step = scan[-4:]
first = step[0] - 1
step_ids = [i for i in ids if first <= i <= step[-1]]
dram = sum(k[i]["dram__bytes_read.sum"] + k[i]["dram__bytes_write.sum"] for i in step)
t_scan = sum(k[i]["gpu__time_duration.sum"] for i in step)
t_all = sum(k[i]["gpu__time_duration.sum"] for i in step_ids)
out = {"cmp_large": {
    "kernel": names[step[0]].split("(")[0].replace("void ", ""),
    "dram_bytes_per_midpoint": dram / 8192,
    "dram_bytes_per_step": dram,
    "algorithmic_table_bytes_per_midpoint": 60 * 2000 * 16,
    "scan_share_of_step_time": t_scan / t_all,
    "source": note}}
json.dump(out, open("profiles/traffic.json", "w"), indent=1)
print(json.dumps(out, indent=1))
