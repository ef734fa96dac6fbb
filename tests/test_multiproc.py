"""Multi-rank host logic on CPU: world_size 2 over gloo.

The N > 1 data path has no collective: each rank generates and scans its own
contiguous block of the midpoint line (CRS: plus a replicated +-aperture
halo), and only the max-over-ranks timing and the final gather of picks go
through torch.distributed.  Here the per-rank scan is the CPU oracle standing
in for the device kernel (which is covered by the -m gpu parity tests); what
is verified is that sharding + halo replication + gathering reproduce the
single-process result exactly.
"""
import os
import socket

import numpy as np
import pytest

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _grid():
    from paper_1907_11678_b200 import CrsAbcGrid
    return CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 2),
                      np.linspace(1500, 3500, 5))


def _scan_rows(ds, rows, ks_step, abc, apm):
    import oracle
    ns = ds.ns
    ks = np.arange(0, ns, ks_step, dtype=np.int32)
    cr = np.repeat(np.asarray(rows, np.int32), len(ks))
    ck = np.tile(ks, len(rows))
    r = oracle.run_cells(ds, "abc", 11, None, cr, ck, apm=apm, abc=abc, threads=2)
    return np.stack([r.best_idx.astype(np.float64), r.best_semblance,
                     r.best_stack]).reshape(3, len(rows), len(ks))


def _worker(rank, world, port, out_q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        from paper_1907_11678_b200 import configs
        from paper_1907_11678_b200.sharding import line_shards
        spec = configs.crs_small().spec
        n = 24
        mx = np.arange(n) * spec.spacing
        shard = line_shards(mx, world, apm=125.0)[rank]
        lo, hi = shard.gathers
        ds = spec.generate(first=lo, count=hi - lo, n_line=n, n_threads=1)
        rows = list(range(shard.row_first, shard.row_first + shard.row_count))
        res = torch.from_numpy(_scan_rows(ds, rows, 50, _grid(), 125.0))
        # max-over-ranks timing reduction, as bench.py does
        t = torch.tensor([float(rank + 1)], dtype=torch.float64)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        parts = [None] * world
        dist.all_gather_object(parts, (shard.block, res.numpy()))
        if rank == 0:
            out_q.put((t.item(), parts))
    finally:
        dist.destroy_process_group()


def test_sharded_crs_line_equals_single_process():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    tmax, parts = q.get(timeout=300)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert tmax == float(world)
    from paper_1907_11678_b200 import configs
    spec = configs.crs_small().spec
    full = spec.generate(count=24, n_line=24, n_threads=1)
    ref = _scan_rows(full, list(range(24)), 50, _grid(), 125.0)
    got = np.concatenate([p[1] for p in sorted(parts, key=lambda x: x[0][0])], axis=1)
    assert [p[0] for p in sorted(parts, key=lambda x: x[0][0])] == [(0, 12), (12, 24)]
    np.testing.assert_array_equal(got, ref)


def test_weak_scaling_blocks_tile_the_line():
    """bench.py's weak scaling: rank r generates gathers [r G, (r+1) G) of a
    world*G line; the union is the single-process line."""
    from paper_1907_11678_b200 import configs
    spec = configs.cmp_small().spec
    G, world = 8, 3
    full = spec.generate(count=G * world, n_line=G * world)
    for r in range(world):
        part = spec.generate(first=r * G, count=G, n_line=G * world)
        np.testing.assert_array_equal(part.samples, full.samples[r * G:(r + 1) * G])
        np.testing.assert_array_equal(part.cdp_id, np.arange(r * G, (r + 1) * G))
