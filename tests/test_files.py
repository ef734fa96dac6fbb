"""SSF1 / SMB1 files: the native reader and writers against
the reference's own io.hpp (write_dataset / read_dataset / write_picks,
compiled into oracle/_ref) — byte-identical files, identical arrays, the
same malformed inputs rejected.  CPU only, except the streaming GPU
pipeline at the end."""
import os

import numpy as np
import pytest

import oracle
from paper_1907_11678_b200 import (ConfigError, Dataset, FormatError, ParameterError,
                                   ScanConfig, SMB1Writer, SSF1Reader, configs,
                                   read_smb1, read_ssf1, run_cmp_file, write_smb1,
                                   write_ssf1)
from paper_1907_11678_b200.api import ScanResult

needs_ref = pytest.mark.skipif(not oracle.ref_available(), reason="oracle/_ref not built")


def ragged_dataset(seed=3, G=5, M=7, ns=37, dt_us=2000):
    rng = np.random.default_rng(seed)
    ntr = rng.integers(0, M + 1, G).astype(np.int32)
    ntr[0] = M
    samples = rng.standard_normal((G, M, ns)).astype(np.float32)
    coords = rng.uniform(-500, 500, (G, M, 4)).astype(np.float32)
    for g in range(G):  # the flattened layout's padding is zero
        samples[g, ntr[g]:] = 0
        coords[g, ntr[g]:] = 0
    ids = rng.permutation(1000)[:G].astype(np.uint32)
    return Dataset(samples, coords, ntr, ids, dt_us)


def same_dataset(ds, sm, co, nt, ids, dt):
    np.testing.assert_array_equal(ds.ntraces, nt)
    np.testing.assert_array_equal(ds.cdp_id, ids)
    assert ds.dt_us == dt
    for g in range(ds.ncdps):
        m = nt[g]
        np.testing.assert_array_equal(np.asarray(ds.samples)[g, :m].view(np.uint32),
                                      sm[g, :m].view(np.uint32))
        np.testing.assert_array_equal(ds.coords[g, :m].view(np.uint32),
                                      co[g, :m].view(np.uint32))


@needs_ref
def test_ssf1_reads_reference_file(tmp_path):
    ds = ragged_dataset()
    p = tmp_path / "ref.ssf"
    meta = '{"generator": "test", "seed": 3}'
    oracle.ref_write_dataset(ds, p, meta)
    got = read_ssf1(p)
    same_dataset(got, np.asarray(ds.samples), ds.coords, ds.ntraces, ds.cdp_id, ds.dt_us)
    np.testing.assert_array_equal(np.asarray(got.samples), np.asarray(ds.samples))
    assert got.metadata == {"generator": "test", "seed": 3}
    with SSF1Reader(p) as r:
        assert (r.n_gathers, r.fold, r.ns, r.dt_us, r.uniform) == (5, 7, 37, 2000, True)
        assert r.metadata_json == meta
        blk = r.read(2, 2)  # a block in the middle
        np.testing.assert_array_equal(np.asarray(blk.samples), np.asarray(ds.samples)[2:4])
        np.testing.assert_array_equal(blk.cdp_id, ds.cdp_id[2:4])


@needs_ref
@pytest.mark.parametrize("meta", ["", '{"k": [1, 2, 3]}'])
def test_ssf1_write_byte_identical(tmp_path, meta):
    ds = ragged_dataset(seed=4)
    a, b = tmp_path / "ours.ssf", tmp_path / "ref.ssf"
    write_ssf1(ds, a, metadata=meta)
    oracle.ref_write_dataset(ds, b, meta)
    assert a.read_bytes() == b.read_bytes()
    # and the reference reads ours
    sm, co, nt, ids, dt, m = oracle.ref_read_dataset(a)
    same_dataset(ds, sm, co, nt, ids, dt)
    assert m == meta


def test_ssf1_roundtrip_generated(tmp_path):
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=6)
    p = tmp_path / "g.ssf"
    write_ssf1(ds, p, metadata={"config": wl.name})
    got = read_ssf1(p, threads=3)
    np.testing.assert_array_equal(np.asarray(got.samples), np.asarray(ds.samples))
    np.testing.assert_array_equal(got.coords, ds.coords)
    assert got.metadata == {"config": wl.name}


def corrupt_cases(good: bytes):
    import struct
    cases = {
        "magic": b"SSF2" + good[4:],
        "version": good[:4] + struct.pack("<I", 2) + good[8:],
        "truncated_header": good[:10],
        "truncated_traces": good[:len(good) // 2],
        "truncated_metadata": good[:-3],
        "trailing": good + b"\x00\x01",
    }
    # gather 0 header: cdp u32, M u32, ns u32, dt u32 at byte 16
    b = bytearray(good)
    b[20:24] = struct.pack("<I", 99)  # trace count > fold
    cases["count_over_fold"] = bytes(b)
    b = bytearray(good)
    b[28:32] = struct.pack("<I", 0)  # dt 0
    cases["dt_zero"] = bytes(b)
    return cases


@needs_ref
def test_ssf1_rejects_what_the_reference_rejects(tmp_path):
    ds = ragged_dataset(seed=5)
    p = tmp_path / "good.ssf"
    oracle.ref_write_dataset(ds, p, '{"a": 1}')
    good = p.read_bytes()
    for name, blob in corrupt_cases(good).items():
        q = tmp_path / f"{name}.ssf"
        q.write_bytes(blob)
        with pytest.raises(ValueError):
            oracle.ref_read_dataset(q)
        with pytest.raises(FormatError):
            SSF1Reader(q)


def test_ssf1_missing_file(tmp_path):
    from paper_1907_11678_b200 import VelanError
    with pytest.raises(VelanError):
        SSF1Reader(tmp_path / "nope.ssf")


def test_ssf1_ragged_ns_not_flattenable(tmp_path):
    import struct
    # two gathers with different ns: a valid SSF1 file the flat layout cannot hold
    blob = b"SSF1" + struct.pack("<III", 1, 2, 1)
    for cdp, ns in ((1, 3), (2, 4)):
        blob += struct.pack("<IIII", cdp, 1, ns, 1000) + struct.pack("<4f", 0, 0, 10, 0)
        blob += struct.pack(f"<{ns}f", *range(ns))
    p = tmp_path / "ragged.ssf"
    p.write_bytes(blob)
    with SSF1Reader(p) as r:
        assert not r.uniform
        with pytest.raises(ConfigError):
            r.read()


def fake_results(seed, n, ns, nc, with_matrix):
    rng = np.random.default_rng(seed)
    cands = np.linspace(1500, 3500, nc).astype(np.float32)
    idx = rng.integers(0, nc, (n, ns)).astype(np.int32)
    sem = rng.uniform(0, 5, (n, ns)).astype(np.float32)
    st = rng.standard_normal((n, ns)).astype(np.float32)
    mat = rng.uniform(0, 5, (n, ns, nc)).astype(np.float32) if with_matrix else None
    ids = (np.arange(n) * 7 + 3).astype(np.uint32)
    return ScanResult(idx, sem, st, cands, np.arange(n, dtype=np.int32), ids, mat,
                      n_candidates=nc)


@needs_ref
@pytest.mark.parametrize("with_matrix", [False, True])
def test_smb1_byte_identical(tmp_path, with_matrix):
    r1 = fake_results(1, 3, 11, 5, with_matrix)
    r2 = fake_results(2, 2, 11, 5, with_matrix)
    a, b = tmp_path / "ours.smb", tmp_path / "ref.smb"
    write_smb1([r1, r2], a, include_matrix=with_matrix)  # two streamed blocks
    ids = np.concatenate([r1.cdp_id, r2.cdp_id])
    vel = np.concatenate([r1.best_velocity, r2.best_velocity])
    sem = np.concatenate([r1.best_semblance, r2.best_semblance])
    mat = np.concatenate([r1.values, r2.values]) if with_matrix else None
    oracle.ref_write_picks(b, ids, vel, sem, 5, mat)
    assert a.read_bytes() == b.read_bytes()
    recs = read_smb1(a)
    assert [r.cdp_id for r in recs] == list(ids)
    np.testing.assert_array_equal(np.stack([r.velocity for r in recs]), vel)
    np.testing.assert_array_equal(np.stack([r.semblance for r in recs]), sem)
    if with_matrix:
        np.testing.assert_array_equal(np.stack([r.values for r in recs]), mat)


def test_smb1_writer_counts_records(tmp_path):
    w = SMB1Writer(tmp_path / "x.smb", 2, 4, 3)
    w.append([1], np.zeros((1, 4)), np.zeros((1, 4)))
    with pytest.raises(ParameterError):
        w.close()  # one record short
    w = SMB1Writer(tmp_path / "y.smb", 1, 4, 3)
    with pytest.raises(ParameterError):
        w.append([1, 2], np.zeros((2, 4)), np.zeros((2, 4)))  # more than declared
    w.close = lambda: None


def test_smb1_reader_rejects_garbage(tmp_path):
    p = tmp_path / "bad.smb"
    p.write_bytes(b"SMB2" + b"\x00" * 12)
    with pytest.raises(FormatError):
        read_smb1(p)


# ---------------------------------------------------------------- GPU

@pytest.mark.gpu
def test_run_cmp_file_streams_like_in_memory(engine, tmp_path):
    """SSF1 file -> pinned blocks -> GPU -> SMB1 stream == run_cmp in memory
    + write_smb1 of its results (byte-identical pick file)."""
    wl = configs.cmp_small()
    ds = wl.spec.generate()
    p = tmp_path / "cmp_small.ssf"
    write_ssf1(ds, p)
    cfg = wl.config
    cfg.kernel_variant = "exact"
    out = tmp_path / "stream.smb"
    blocks = run_cmp_file(engine, p, cfg, smb_path=out, block=24)
    assert len(blocks) == 3  # 64 gathers in blocks of 24
    ref = engine.run_cmp(ds, cfg)
    np.testing.assert_array_equal(np.concatenate([b.best_idx for b in blocks]), ref.best_idx)
    np.testing.assert_array_equal(np.concatenate([b.best_semblance for b in blocks]),
                                  ref.best_semblance)
    whole = tmp_path / "whole.smb"
    write_smb1(ref, whole)
    assert out.read_bytes() == whole.read_bytes()
    assert sum(b.stats.naive_fetches for b in blocks) == ref.stats.naive_fetches


@pytest.mark.gpu
def test_run_cmp_file_streams_matrices(engine, tmp_path):
    """SMB1 with the flagged full matrices, streamed per block, equals the
    reference writer's file for the in-memory results."""
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=10)
    p = tmp_path / "c.ssf"
    write_ssf1(ds, p)
    cfg = wl.config
    cfg.kernel_variant = "exact"
    out = tmp_path / "m.smb"
    run_cmp_file(engine, p, cfg, smb_path=out, block=4, include_matrix=True)
    ref = engine.run_cmp(ds, cfg, emit_matrix=True)
    if oracle.ref_available():
        b = tmp_path / "ref.smb"
        oracle.ref_write_picks(b, ref.cdp_id, ref.best_velocity, ref.best_semblance,
                               ref.values.shape[2], ref.values)
        assert out.read_bytes() == b.read_bytes()
    recs = read_smb1(out)
    np.testing.assert_array_equal(np.stack([r.values for r in recs]), ref.values)


# ---------------------------------------------------------------- CRS file pipeline

def grid_dataset(nx=6, ny=5, M=6, ns=160, dt_us=2000, seed=8, shuffle=True):
    """A 2-D grid of midpoints 25 m apart, cdp_id row-major, written to the
    file in a shuffled order (run_crs orders its output by cdp_id)."""
    rng = np.random.default_rng(seed)
    G = nx * ny
    samples = rng.uniform(-1, 1, (G, M, ns)).astype(np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    ids = np.arange(G, dtype=np.uint32)
    h = (40.0 * np.arange(1, M + 1)).astype(np.float32)
    for g in range(G):
        mx, my = np.float32(25.0 * (g % nx)), np.float32(25.0 * (g // nx))
        coords[g, :, 0] = mx - h
        coords[g, :, 2] = mx + h
        coords[g, :, 1] = coords[g, :, 3] = my
    perm = rng.permutation(G) if shuffle else np.arange(G)
    return Dataset(samples[perm], coords[perm], np.full(G, M, np.int32), ids[perm], dt_us)


def test_ssf1_midpoints_and_gather_lists(tmp_path):
    ds = grid_dataset()
    p = tmp_path / "g.ssf"
    write_ssf1(ds, p)
    from paper_1907_11678_b200 import _native as N
    from paper_1907_11678_b200.api import _ptr
    with SSF1Reader(p) as rd:
        mx = np.zeros(rd.n_gathers, np.float32)
        my = np.zeros(rd.n_gathers, np.float32)
        assert N.load().velan_ssf1_midpoints(rd._h, _ptr(mx), _ptr(my)) == 0
        np.testing.assert_array_equal(np.stack([mx, my], 1), ds.midpoints())
        gl = np.array([7, 2, 29, 2], np.int32)
        sm = np.zeros((4, rd.fold, rd.ns), np.float32)
        co = np.zeros((4, rd.fold, 4), np.float32)
        assert N.load().velan_ssf1_read_list(rd._h, _ptr(gl), 4, rd.fold, _ptr(sm),
                                             _ptr(co), 2) == 0
        np.testing.assert_array_equal(sm, ds.samples[gl])
        np.testing.assert_array_equal(co, ds.coords[gl])


def test_crs_blocks_hold_every_sweep():
    """Each block's gather list contains the full sweep (central + closed apm
    ball, the library's own sweep builder) of every row it owns, and the
    blocks tile the cdp_id-ordered rows."""
    from paper_1907_11678_b200 import describe
    from paper_1907_11678_b200.files import crs_blocks
    ds = grid_dataset()
    cfg = ScanConfig(w=5, nc=7)
    apm = 36.0  # the 8-neighbourhood on a 25 m grid
    sw = describe(ds, cfg, op="d2", apm=apm)
    mp = ds.midpoints()
    blocks = crs_blocks(mp[:, 0], mp[:, 1], ds.cdp_id, apm, 7)
    allrows = np.concatenate([b[0] for b in blocks])
    np.testing.assert_array_equal(allrows, sw.row_gather)
    for rows, gathers, row_first in blocks:
        for g in rows:
            r = int(np.nonzero(sw.row_gather == g)[0][0])
            legs = sw.leg_gather[sw.leg_off[r]:sw.leg_off[r + 1]]
            assert set(legs.tolist()) <= set(gathers.tolist())
        sub = describe(ds.subset(gathers), cfg, op="d2", apm=apm)
        np.testing.assert_array_equal(gathers[sub.row_gather[row_first:row_first + len(rows)]],
                                      rows)


def test_crs_partition_checks_match_reference():
    from paper_1907_11678_b200.files import check_partition
    ds = grid_dataset(shuffle=False)
    mp = ds.midpoints()
    check_partition(mp[:, 0], mp[:, 1], (2, 1), 30.0)
    check_partition(mp[:, 0], mp[:, 1], (1, 1), 300.0)
    with pytest.raises(ConfigError):   # 125 m / 2 shards -> half width 31.25
        check_partition(mp[:, 0], mp[:, 1], (2, 1), 31.5)
    with pytest.raises(ConfigError):   # 100 m / 2 shards -> half height 25
        check_partition(mp[:, 0], mp[:, 1], (2, 2), 30.0)
    with pytest.raises(ConfigError):
        check_partition(mp[:, 0], mp[:, 1], (1, 1), 0.0)
    with pytest.raises(ConfigError):
        check_partition(mp[:, 0], mp[:, 1], (0, 1), 5.0)


@pytest.mark.gpu
@needs_ref
@pytest.mark.parametrize("with_matrix", [False, True])
def test_run_crs_file_byte_identical_to_reference(engine, tmp_path, with_matrix):
    """velan crs --data F --out P --grid 2x1 --apm 30 [--matrix]
    (tools/velan.cpp:167-184 = read_dataset + velan::run_crs + write_picks,
    all from oracle/_ref) against run_crs_file streaming the same SSF1 file in
    halo-aware blocks through the GPU (EXACT): the pick files are
    byte-identical."""
    from paper_1907_11678_b200 import run_crs_file
    ds = grid_dataset()
    p = tmp_path / "g.ssf"
    write_ssf1(ds, p)
    cfg = ScanConfig(vmin=1500.0, vmax=3500.0, nc=9, w=5, kernel_variant="exact")
    code, msg, ref = oracle.ref_run_pipeline(ds, "crs", 1500.0, 3500.0, 9, 5, workers=2,
                                             grid=(2, 1), apm=30.0, matrix=True)
    assert code == 0, msg
    order = np.lexsort((np.arange(ds.ncdps), ds.cdp_id))
    v = cfg.grid()
    refp = tmp_path / "ref.smb"
    oracle.ref_write_picks(refp, ds.cdp_id[order], v[ref.best_idx], ref.best_semblance, 9,
                           ref.matrix if with_matrix else None)
    out = tmp_path / "gpu.smb"
    blocks = run_crs_file(engine, p, cfg, 30.0, smb_path=out, dims=(2, 1), block=7,
                          include_matrix=with_matrix)
    assert len(blocks) == 5
    assert out.read_bytes() == refp.read_bytes()
    assert sum(b.stats.naive_fetches for b in blocks) == ref.valid
    with pytest.raises(ConfigError):
        run_crs_file(engine, p, cfg, 40.0, dims=(2, 1))
