#!/usr/bin/env python
"""Small scans for compute-sanitizer (one tool per GPU call):
    compute-sanitizer --tool racecheck python tools/sanitize_case.py
CMP (EXACT + FAST, TMA staging), CRS d2 and ABC (FAST) on a few gathers,
ragged gathers, a top-k scan, each checked against the oracle so a run
that the sanitizer perturbs still has to be right."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402

import oracle  # noqa: E402
from helpers import line_dataset  # noqa: E402
from paper_1907_11678_b200 import CrsAbcGrid, Engine, ScanConfig, configs  # noqa: E402

eng = Engine([0])
wl = configs.cmp_small()
ds = wl.spec.generate(count=3)
for variant in ("exact", "fast"):
    cfg = ScanConfig(w=11, velocities=wl.config.grid(), kernel_variant=variant)
    r = eng.run_cmp(ds, cfg, topk=2)
    rows, ks = oracle.all_cells(3, ds.ns)
    ref = oracle.run_cells(ds, "nmo", 11, cfg.grid(), rows, ks, mode=2)
    assert (r.best_idx.reshape(-1) == ref.best_idx).mean() > 0.999, variant
ld = line_dataset(12)
grid = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 2), np.linspace(1500, 3500, 5))
for variant in ("exact", "fast"):
    cfg = ScanConfig(w=11, velocities=grid.v, kernel_variant=variant)
    r = eng.run_crs(ld, cfg, 75.0, abc=grid)
    rows, ks = oracle.all_cells(ld.ncdps, ld.ns)
    ref = oracle.run_cells(ld, "abc", 11, None, rows, ks, apm=75.0, abc=grid, mode=2)
    assert (r.best_idx.reshape(-1) == ref.best_idx).mean() > 0.99, variant
    cfg = ScanConfig(w=15, velocities=grid.v, kernel_variant=variant)
    r = eng.run_crs(ld, cfg, 75.0)
eng.close()
print("sanitize case ok")
