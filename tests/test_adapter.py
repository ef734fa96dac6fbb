"""The C++ drop-in (include/velan_gpu/adapter.hpp) against the reference
pipeline in one binary: oracle/_ref/test_adapter, built by oracle/Makefile
from tests/cpp/test_adapter.cpp and the unmodified reference headers."""
import os
import subprocess

import pytest

import oracle

BIN = os.path.join(oracle.HERE, "_ref", "test_adapter")


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/test_adapter not built")
def test_adapter_matches_reference_pipeline():
    r = subprocess.run([BIN], capture_output=True, text=True, timeout=600)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
    assert "FAIL" not in r.stdout


def test_adapter_binary_links_the_gpu_library():
    if not os.path.exists(BIN):
        pytest.skip("oracle/_ref/test_adapter not built")
    out = subprocess.run(["ldd", BIN], capture_output=True, text=True).stdout
    assert "libvelan_gpu.so" in out and "not found" not in out.split("libvelan_gpu.so")[1].split("\n")[0]


@pytest.mark.gpu
@pytest.mark.skipif(not os.path.exists(BIN), reason="oracle/_ref/test_adapter not built")
def test_adapter_cmp_large_without_the_matrix():
    """velan_gpu::run_cmp on CMP large (8192 x 60 x 2000, 401 C, w 15) with
    Options{fast, values = false}: the 26 GB matrix is never allocated."""
    r = subprocess.run([BIN, "large"], capture_output=True, text=True, timeout=900)
    print(r.stdout)
    assert r.returncode == 0, r.stdout + r.stderr
