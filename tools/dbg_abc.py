"""Debug: FAST ABC subset vs oracle, rep + worst cells."""
import sys
import numpy as np
sys.path.insert(0, ".")
import oracle
from paper_1907_11678_b200 import ScanConfig, CrsAbcGrid, configs, Engine
w = configs.crs_small()
ds = w.spec.generate(count=16)
grid = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 3), np.linspace(1500, 3500, 7))
eng = Engine()
cfg = ScanConfig(w=11, velocities=grid.v, kernel_variant="fast")
r = eng.run_crs(ds, cfg, 125.0, abc=grid, emit_matrix=True)
rows, ks = oracle.all_cells(ds.ncdps, ds.ns)
ref = oracle.run_cells(ds, "abc", 11, None, rows, ks, apm=125.0, abc=grid, matrix=True)
gm = r.values.reshape(-1, grid.ncand)
rep = oracle.compare(gm, ref.matrix)
print(rep, "valid", r.stats.naive_fetches, ref.valid)
rel = np.abs(gm.astype(np.float64) - ref.matrix) / np.maximum(np.abs(ref.matrix), 1e-12)
for i in np.argsort(-rel, axis=None)[:12]:
    c, j = np.unravel_index(i, rel.shape)
    print("row", c // ds.ns, "k", c % ds.ns, "cand", j, gm[c, j], ref.matrix[c, j], rel[c, j])
print("rel quantiles", np.quantile(rel, [0.5, 0.9, 0.99, 0.999]))
