#!/usr/bin/env python
"""Print the hot trace loop (the backward branch whose body holds the most
FFMA2 and is shortest) of one scan-kernel instantiation from a built library:
    python tools/sass_loop.py lib.so 'ILi1ELi1ELi11ELb1ELi2ELi5120' [--dump]"""
import re, subprocess, sys
lib, key = sys.argv[1], sys.argv[2]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
f = []; on = False
for l in out.split("\n"):
    if "Function : " in l:
        on = key in l and "semblance_scan_kernel" in l
        continue
    if on: f.append(l)
ins = []
for l in f:
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if m: ins.append((int(m.group(1), 16), m.group(2).strip()))
best = None
for a, t in ins:
    if "BRA" in t:
        mm = re.findall(r"0x([0-9a-f]+)", t)
        if mm:
            tgt = int(mm[-1], 16)
            if tgt < a:
                body = [x for x in ins if tgt <= x[0] <= a]
                n2 = sum("FFMA2" in x[1] for x in body)
                if n2 >= 20 and (best is None or len(body) < len(best)):
                    best = body
from collections import Counter
c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for _, t in best)
print(len(best), "instructions:", ", ".join(f"{k} {v}" for k, v in c.most_common()))
if "--dump" in sys.argv:
    for a, t in best: print(hex(a), t)
