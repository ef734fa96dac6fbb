"""bench.py's host logic on CPU: the --gpus self-launch, the gather of every
rank's picks to rank 0 (world_size 2 over gloo) and the parity sample of the
gathered line against the oracle (BASELINE configs[4]: "results gathered to
host and checked against the CPU oracle on a seeded 1% sample of outputs")."""
import os
import socket
import sys
from dataclasses import replace
from types import SimpleNamespace

import numpy as np
import pytest

import oracle

torch = pytest.importorskip("torch")
import torch.distributed as dist  # noqa: E402
import torch.multiprocessing as mp  # noqa: E402

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1907_11678_b200 import CrsAbcGrid, configs  # noqa: E402


def _oracle_picks(wl, ds, abc=None):
    rr, kk = oracle.all_cells(ds.ncdps, ds.ns)
    r = oracle.run_cells(ds, wl.op, wl.config.w, wl.config.grid(), rr, kk, apm=wl.apm,
                         abc=abc, mode=2)
    G = ds.ncdps
    return (r.best_idx.reshape(G, -1), r.best_semblance.reshape(G, -1),
            r.best_stack.reshape(G, -1))


def test_parity_sample_cmp_one_percent():
    wl = configs.cmp_small()
    ds = wl.spec.generate()
    picks = _oracle_picks(wl, ds)
    rep = bench.parity_sample(wl, 64, np.arange(64), picks)
    assert rep["pass"] and rep["cells"] == 640 and rep["fraction"] == pytest.approx(0.01)
    assert rep["rows"] == 16 and rep["unexcused_mismatches"] == 0
    # a wrong pick, a wrong semblance and a wrong stack are all caught
    bi, bs, bst = (x.copy() for x in picks)
    bi[:] = (bi + 7) % 101
    assert bench.parity_sample(wl, 64, np.arange(64), (bi, bs, bst))["unexcused_mismatches"] > 600
    bi, bs, bst = (x.copy() for x in picks)
    bs *= 1.001
    rep = bench.parity_sample(wl, 64, np.arange(64), (bi, bs, bst))
    assert not rep["pass"] and rep["semblance_over_tol"] > 0
    bi, bs, bst = (x.copy() for x in picks)
    bst += 0.01
    rep = bench.parity_sample(wl, 64, np.arange(64), (bi, bs, bst))
    assert not rep["pass"] and rep["stack_over_tol"] > 0


def test_parity_sample_crs_rows_with_halo():
    wl = configs.crs_small()
    wl.spec = replace(wl.spec, n_gathers=16)
    wl.abc = CrsAbcGrid(np.linspace(-2e-4, 2e-4, 3), np.linspace(0, 1e-7, 3),
                        np.linspace(1500, 3500, 5))
    wl.config.velocities = wl.abc.v
    ds = wl.spec.generate()
    picks = _oracle_picks(wl, ds, wl.abc)
    rep = bench.parity_sample(wl, 16, np.arange(16), picks, n_cells=300)
    assert rep["pass"] and rep["rows"] == 16 and rep["cells"] >= 300
    bi = picks[0].copy()
    bi[5] = (bi[5] + 1) % wl.ncand
    rep = bench.parity_sample(wl, 16, np.arange(16), (bi, picks[1], picks[2]), n_cells=300)
    assert rep["unexcused_mismatches"] > 0


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _gather_worker(rank, world, port, q):
    sys.path.insert(0, ROOT)
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import bench as b
        rows = [3, 5][rank]  # uneven blocks (strong scaling of an odd line)
        g0 = [0, 3][rank]
        bi = torch.arange(g0 * 7, (g0 + rows) * 7, dtype=torch.int32).reshape(rows, 7)
        bs = bi.float() * 0.5
        bst = -bi.float()
        out = b.gather_picks(dist, rank, world, (bi, bs, bst))
        if rank == 0:
            q.put(out)
        else:
            assert out is None
    finally:
        dist.destroy_process_group()


def test_gather_picks_world2_gloo():
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_gather_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    bi, bs, bst = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    ref = np.arange(8 * 7, dtype=np.int32).reshape(8, 7)
    np.testing.assert_array_equal(bi, ref)
    np.testing.assert_array_equal(bs, ref * 0.5)
    np.testing.assert_array_equal(bst, -ref.astype(np.float32))


def test_gpus_flag_relaunches_under_torchrun(monkeypatch):
    args = SimpleNamespace(gpus=4, impl="ours")
    monkeypatch.delenv("WORLD_SIZE", raising=False)
    monkeypatch.setattr(sys, "argv", ["bench.py", "--gpus", "4", "--steps", "2"])
    seen = {}
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 8)
    monkeypatch.setattr(bench.subprocess, "call", lambda cmd: seen.setdefault("cmd", cmd) and 0)
    with pytest.raises(SystemExit) as ex:
        bench.maybe_relaunch(args)
    assert ex.value.code == 0
    cmd = seen["cmd"]
    assert cmd[1:3] == ["-m", "torch.distributed.run"]
    assert "--nproc-per-node=4" in cmd and "127.0.0.1" in cmd
    assert cmd[-4:] == ["--gpus", "4", "--steps", "2"]
    # too few GPUs: a clear error, no launch
    monkeypatch.setattr(torch.cuda, "device_count", lambda: 2)
    with pytest.raises(SystemExit) as ex:
        bench.maybe_relaunch(args)
    assert ex.value.code == 2
    # under torchrun: WORLD_SIZE must match --gpus
    monkeypatch.setenv("WORLD_SIZE", "2")
    with pytest.raises(SystemExit) as ex:
        bench.maybe_relaunch(args)
    assert ex.value.code == 2
    monkeypatch.setenv("WORLD_SIZE", "4")
    bench.maybe_relaunch(args)  # consistent: returns
    # N = 1 and the CPU reference arm never re-launch
    monkeypatch.delenv("WORLD_SIZE")
    bench.maybe_relaunch(SimpleNamespace(gpus=1, impl="ours"))
    bench.maybe_relaunch(SimpleNamespace(gpus=8, impl="reference"))


@pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")
def test_reference_arm_runs_without_the_gpu_library():
    """--impl reference times the reference's own kernels (oracle/_ref) on
    inputs from oracle/libvelan_synth.so: the GPU library is never loaded."""
    import json
    import subprocess
    code = ("import sys, json; sys.argv = ['bench.py', '--impl', 'reference', '--workload', "
            "'cmp_small', '--steps', '1', '--warmup', '1']; import bench; bench.main(); "
            "maps = open('/proc/self/maps').read(); "
            "print(json.dumps({'gpu_lib': 'libvelan_gpu.so' in maps, "
            "'ref_lib': 'libvelan_ref.so' in maps}))")
    out = subprocess.run([sys.executable, "-c", code], cwd=ROOT, capture_output=True,
                         text=True, timeout=600)
    assert out.returncode == 0, out.stderr
    lines = [json.loads(x) for x in out.stdout.splitlines() if x.startswith("{")]
    line, maps = lines[0], lines[1]
    assert line["impl"] == "reference" and line["value"] > 0
    assert line["cpu_baseline"]["kind"] == "reference"
    assert maps == {"gpu_lib": False, "ref_lib": True}
