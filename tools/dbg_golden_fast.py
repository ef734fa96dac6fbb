"""Debug: FAST vs golden matrix on the cmp_small slice, worst cells."""
import numpy as np
import sys
sys.path.insert(0, "."); sys.path.insert(0, "tests")
from test_golden import load, ds_from
from paper_1907_11678_b200 import ScanConfig, Engine
z = load("cmp_small_slice.npz")
ds = ds_from(z)
eng = Engine()
r = eng.run_cmp(ds, ScanConfig(w=int(z["w"]), velocities=z["v"], kernel_variant="fast"), emit_matrix=True)
m = r.values.reshape(-1, len(z["v"]))[z["matrix_cells"]]
ref = z["matrix"]
rel = np.abs(m - ref) / np.maximum(np.abs(ref), 1e-12)
idx = np.argsort(-rel, axis=None)[:20]
for i in idx:
    c, v = np.unravel_index(i, rel.shape)
    print("cell", z["matrix_cells"][c], "cand", v, "gpu", m[c, v], "ref", ref[c, v], "rel", rel[c, v])
print("n bad", int((rel > 1e-4).sum()), "of", rel.size)
print("valid", r.stats.naive_fetches, int(z["valid"]))
# window-length case, w=11 ns=131 random
import oracle
from paper_1907_11678_b200 import Dataset, velocity_grid
for w in (1, 11):
    rng = np.random.default_rng(100 + w)
    G, M, ns = 3, 7, 132
    samples = rng.uniform(-1, 1, (G, M, ns)).astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    coords[:, :, 2] = np.linspace(0, 40, M)[None, :]
    ds = Dataset(samples, coords, np.full(G, M, np.int32), np.arange(G, dtype=np.uint32), 244)
    v = velocity_grid(2000.0, 3000.0, 9)
    r = eng.run_cmp(ds, ScanConfig(w=w, velocities=v, kernel_variant="fast"), emit_matrix=True)
    rows, ks = oracle.all_cells(G, ns)
    ref = oracle.run_cells(ds, "nmo", w, v, rows, ks, matrix=True)
    gm = r.values.reshape(-1, len(v)); rm = ref.matrix
    rel = np.abs(gm - rm) / np.maximum(np.abs(rm), 1e-6)
    bad = np.argwhere(rel > 1e-3)
    print("w", w, "bad", len(bad), "of", rel.size, "valid", r.stats.naive_fetches, ref.valid)
    for c, j in bad[:15]:
        print("  row", c // ns, "k", c % ns, "cand", j, gm[c, j], rm[c, j])
