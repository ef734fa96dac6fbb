"""The C-ABI library: it loads, exports every symbol include/velan_gpu.h
declares, and rejects invalid scans before touching a device (CPU-only; no
compute calls)."""
import ctypes as C
import os
import re

import numpy as np
import pytest

from paper_1907_11678_b200 import _native as N
from paper_1907_11678_b200 import (ConfigError, Dataset, DeviceError, Engine,
                                   ParameterError, ScanConfig, run_cmp)
from paper_1907_11678_b200.api import _dataset_struct, _scan_struct

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "velan_gpu.h")


def declared_functions():
    text = open(HEADER).read()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(velan_(?:gpu|ssf1|smb1)_[a-z0-9_]+)\s*\(", text)))


def test_header_declares_the_expected_surface():
    names = declared_functions()
    for must in ["velan_gpu_cmp", "velan_gpu_crs", "velan_gpu_create",
                 "velan_gpu_destroy", "velan_gpu_last_error",
                 "velan_gpu_plan_create", "velan_gpu_plan_execute",
                 "velan_gpu_validate", "velan_gpu_hit_batch"]:
        assert must in names


def test_library_exports_every_declared_symbol():
    lib = N.load()
    missing = [n for n in declared_functions() if not hasattr(lib, n)]
    assert not missing, missing
    # and the ctypes table covers the whole header
    assert set(declared_functions()) == set(N.SIGNATURES)


def test_library_is_sm100a_only():
    """The fatbin carries sm_100a SASS (cuobjdump lists the arch)."""
    import shutil
    import subprocess
    if not shutil.which("cuobjdump"):
        pytest.skip("cuobjdump not available")
    out = subprocess.run(["cuobjdump", "--list-elf", N.LIB_PATH],
                         capture_output=True, text=True).stdout
    assert "sm_100a" in out
    assert "sm_90" not in out and "sm_80" not in out


def test_abi_version():
    assert N.load().velan_gpu_abi_version() == 2


def test_struct_layouts_match_ctypes():
    out = np.zeros(8, np.int32)
    assert N.load().velan_gpu_abi_layout(out.ctypes.data) == 0
    expect = [C.sizeof(N.Dataset), N.Dataset.samples_device.offset,
              C.sizeof(N.Scan), N.Scan.row_count.offset,
              C.sizeof(N.Result), N.Result.topk_semblance.offset,
              C.sizeof(N.Synth), N.Synth.n_threads.offset]
    assert list(out) == expect


def make_ds(G=2, M=3, ns=64, dt=4000, ntr=None):
    samples = np.zeros((G, M, ns), np.float32)
    coords = np.zeros((G, M, 4), np.float32)
    coords[:, :, 2] = 100.0
    ntraces = np.full(G, M, np.int32) if ntr is None else np.asarray(ntr, np.int32)
    return Dataset(samples, coords, ntraces, np.arange(G, dtype=np.uint32), dt)


def validate(ds, op=N.OP_NMO, w=4, v=(2000.0, 2500.0), apm=0.0, abc=None, rows=None):
    keep = []
    sc = _scan_struct(op, "exact", w, np.asarray(v, np.float32), abc, apm, keep, rows)
    dss = _dataset_struct(ds)
    code = N.load().velan_gpu_validate(C.byref(dss), C.byref(sc))
    return code, N.last_error()


def test_validation_mirrors_scanconfig():
    ds = make_ds()
    assert validate(ds)[0] == N.OK
    code, msg = validate(ds, w=0)
    assert code == N.ECONFIG and "w must be >= 1" in msg
    code, msg = validate(ds, v=())
    assert code == N.ECONFIG and "nc must be >= 1" in msg
    code, msg = validate(ds, v=(2000.0, -1.0))
    assert code == N.ECONFIG
    code, msg = validate(ds, w=63)               # ns = 64 <= w + 1
    assert code == N.ECONFIG
    code, msg = validate(make_ds(ns=10), w=9)
    assert code == N.ECONFIG and "window does not fit" in msg
    code, msg = validate(ds, w=33)
    assert code == N.ECONFIG and "maximum" in msg


def test_validation_crs_and_shapes():
    ds = make_ds()
    code, msg = validate(ds, op=N.OP_CRS_D2, apm=0.0)
    assert code == N.ECONFIG and "apm must be > 0" in msg
    assert validate(ds, op=N.OP_CRS_D2, apm=10.0)[0] == N.OK
    # empty gathers: run_cmp's worker failure / run_crs's midpoint_of error
    bad = make_ds(ntr=[3, 0])
    code, msg = validate(bad)
    assert code == N.ERUNTIME and "worker pool failure" in msg
    code, msg = validate(bad, op=N.OP_CRS_D2, apm=10.0)
    assert code == N.EPARAM and "midpoint_of" in msg
    code, msg = validate(ds, rows=(1, 5))
    assert code == N.EPARAM
    # an empty dataset is valid (run_cmp returns {})
    empty = Dataset(np.zeros((0, 1, 64), np.float32), np.zeros((0, 1, 4), np.float32),
                    np.zeros(0, np.int32), np.zeros(0, np.uint32), 4000)
    assert validate(empty, w=0)[0] == N.ECONFIG  # config is validated first
    assert validate(empty)[0] == N.OK


def test_no_cpu_fallback_without_device():
    """Without an sm_100 device the product path fails loudly."""
    if N.load().velan_gpu_device_count() > 0:
        pytest.skip("a device is present")
    with pytest.raises(DeviceError):
        Engine([0])
    with pytest.raises(DeviceError):
        run_cmp(make_ds(), ScanConfig(w=4, nc=3))


def test_python_config_validation():
    with pytest.raises(ConfigError):
        ScanConfig(w=0).validate()
    with pytest.raises(ConfigError):
        ScanConfig(vmin=0.0).validate()
    with pytest.raises(ConfigError):
        ScanConfig(kernel_variant="simd").validate()


@pytest.mark.gpu
def test_device_samples_must_live_on_the_context_device():
    """samples_mem = DEVICE with a host pointer, or declared on another
    device, is a config error before any launch (no fault, no peer read)."""
    import torch
    from paper_1907_11678_b200 import ConfigError, Dataset, Engine, ScanConfig, configs
    wl = configs.cmp_small()
    ds = wl.spec.generate(count=2)
    eng = Engine([0])
    cfg = ScanConfig(w=11, velocities=wl.config.grid(), kernel_variant="fast")
    dev = torch.from_numpy(ds.samples).cuda()
    dd = Dataset(dev, ds.coords, ds.ntraces, ds.cdp_id, ds.dt_us)
    eng.run_cmp(dd, cfg)  # fine
    from paper_1907_11678_b200 import api
    orig = api._dataset_struct

    def lie_device(d):
        s = orig(d)
        s.samples_device = 5
        return s

    def lie_host(d):
        s = orig(d)
        s.samples_mem = 1  # MEM_DEVICE
        return s
    try:
        api._dataset_struct = lie_device
        with pytest.raises(ConfigError):
            eng.run_cmp(dd, cfg)
        with pytest.raises(ConfigError):
            eng.plan(dd, cfg)
        api._dataset_struct = lie_host
        with pytest.raises(ConfigError):
            eng.run_cmp(ds, cfg)
    finally:
        api._dataset_struct = orig
        eng.close()
