#!/usr/bin/env python
"""Main-path size of the hot trace loop of scan-kernel instantiations (the
loop body minus the rare near-integer fix-up block: from the loop head to the
branch that skips the fix-up after VOTE.ANY, plus the backward branch):
    python tools/loop_main.py lib.so KEY [KEY ...]"""
import re
import subprocess
import sys
from collections import Counter

lib = sys.argv[1]
out = subprocess.run(["cuobjdump", "-sass", lib], capture_output=True, text=True).stdout
funcs, cur = {}, None
for l in out.split("\n"):
    if "Function : " in l:
        cur = l.split("Function : ")[1].strip()
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", l)
    if cur and m:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
for key in sys.argv[2:]:
    name = [n for n in funcs if key in n and "semblance_scan_kernel" in n]
    if not name:
        print(key, "not found")
        continue
    ins = funcs[name[0]]
    best = None
    for a, t in ins:
        if "BRA" in t:
            mm = re.findall(r"0x([0-9a-f]+)", t)
            if mm and int(mm[-1], 16) < a:
                tgt = int(mm[-1], 16)
                body = [x for x in ins if tgt <= x[0] <= a]
                if sum("FFMA2" in x[1] for x in body) >= 20 and (best is None or len(body) < len(best)):
                    best = body
    # main path: up to the first conditional branch after VOTE.ANY
    main = []
    seen_vote = False
    for a, t in best:
        main.append(t)
        if "VOTE.ANY" in t:
            seen_vote = True
        elif seen_vote and "BRA" in t:
            break
    main.append(best[-1][1])
    c = Counter(re.sub(r"^@!?U?P\w+\s+", "", t).split()[0].split(".")[0] for t in main)
    fma = sum(v for k, v in c.items() if k in ("FFMA", "FMUL", "FADD", "IMAD"))
    fma += 2 * sum(v for k, v in c.items() if k in ("FFMA2", "FMUL2", "FADD2"))
    print(f"{key}: main {len(main)} instr, FMA-pipe cycles ~{fma}: " +
          ", ".join(f"{k} {v}" for k, v in c.most_common()))
