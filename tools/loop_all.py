#!/usr/bin/env python
"""Every trace loop (backward branch, >= 20 FFMA2) of scan-kernel
instantiations with its main-path size (up to the fix-up branch) and the
count of a few telltale instructions:
    python tools/loop_all.py lib.so KEY [KEY ...]"""
import re
import subprocess
import sys
from collections import Counter

out = subprocess.run(["cuobjdump", "-sass", sys.argv[1]], capture_output=True, text=True).stdout
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
    name = [n for n in funcs if key in n and "semblance_scan" in n][0]
    ins = funcs[name]
    seen = set()
    for a, t in ins:
        mm = re.findall(r"0x([0-9a-f]+)", t) if "BRA" in t else []
        if not mm or int(mm[-1], 16) >= a:
            continue
        tgt = int(mm[-1], 16)
        body = [x for x in ins if tgt <= x[0] <= a]
        if sum("FFMA2" in x[1] for x in body) < 20 or len(body) > 700 or tgt in seen:
            continue
        seen.add(tgt)
        main = []
        for _, t2 in body:
            main.append(t2)
            if ("VOTE.ANY" in t2 or "BSSY" in t2) and len(main) > 10:
                pass
            if re.match(r"^@!?P\d BRA", t2) and len(main) > 40:
                break
        c = Counter(re.sub(r"^@!?U?P\w+\s+", "", x).split()[0].split(".")[0] for x in main)
        fma = sum(c[k] for k in ("FFMA", "FMUL", "FADD", "IMAD")) + 2 * sum(
            c[k] for k in ("FFMA2", "FMUL2", "FADD2"))
        print(f"{key[:40]} loop@{hex(tgt)} body {len(body)} main {len(main)} fma~{fma} "
              f"FFMA2 {c['FFMA2']} LDS {c['LDS']} FSEL {c['FSEL']} IMAD {c['IMAD']} FMUL2 {c['FMUL2']}")
