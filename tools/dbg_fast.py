import sys, numpy as np
sys.path.insert(0, '.')
import oracle
from paper_1907_11678_b200 import Engine, ScanConfig, Dataset, velocity_grid
eng = Engine([0])
for ns in (131, 132):
  for w in (1, 2, 3, 4):
    rng = np.random.default_rng(100 + w)
    G, M = 3, 7
    samples = rng.uniform(-1, 1, (G, M, ns)).astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32); coords[:, :, 2] = np.linspace(0, 40, M)[None, :]
    ds = Dataset(samples, coords, np.full(G, M, np.int32), np.arange(G, dtype=np.uint32), 244)
    v = velocity_grid(2000.0, 3000.0, 9)
    r = eng.run_cmp(ds, ScanConfig(w=w, velocities=v, kernel_variant="fast"), emit_matrix=True)
    rows, ks = oracle.all_cells(G, ns)
    ref = oracle.run_cells(ds, "nmo", w, v, rows, ks, matrix=True)
    m = r.values.reshape(G*ns, -1)
    d = np.abs(m - ref.matrix)
    bad = np.argwhere(d > 1e-3)
    print(ns, w, "maxdiff", d.max(), "nbad", len(bad), "valid", r.stats.naive_fetches, ref.valid)
    for c, cand in bad[:6]:
        print("   row", c // ns, "k", c % ns, "cand", cand, m[c, cand], ref.matrix[c, cand])
