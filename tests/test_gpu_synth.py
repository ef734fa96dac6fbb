"""Device synthetic generator against the host generator:
same counter-based streams and model, so the samples agree to the last bit
except where a double libm result (exp/log/sin/cos on the device vs glibc)
rounds differently into float."""
import ctypes as C

import numpy as np
import pytest

from paper_1907_11678_b200 import _native as N
from paper_1907_11678_b200 import configs


def test_geometry_only_matches_full_generation():
    wl = configs.crs_small()
    full = wl.spec.generate(first=10, count=5)
    s = wl.spec._struct(10, 5, 0, None)
    co = np.empty((5, wl.spec.n_traces, 4), np.float32)
    nt = np.empty(5, np.int32)
    ids = np.empty(5, np.uint32)
    assert N.load().velan_gpu_synth_generate(C.byref(s), None, co.ctypes.data, nt.ctypes.data,
                                             ids.ctypes.data) == 0
    np.testing.assert_array_equal(co, full.coords)
    np.testing.assert_array_equal(nt, full.ntraces)
    np.testing.assert_array_equal(ids, full.cdp_id)


def test_line_events_are_the_generators():
    wl = configs.crs_small()
    s = wl.spec._struct(0, 4, 0, None)
    ev = np.zeros((wl.spec.n_events, 6))
    assert N.load().velan_gpu_synth_line_events(C.byref(s), ev.ctypes.data) == 0
    t0, v, amp, x, A, B = ev.T
    assert np.all((t0 >= wl.spec.t0_lo) & (t0 <= wl.spec.t0_hi))
    assert np.all((v >= wl.spec.v_lo) & (v <= wl.spec.v_hi))
    assert np.all(np.abs(A) <= wl.spec.a_abs) and np.all((B >= 0) & (B <= wl.spec.b_max))


@pytest.mark.gpu
@pytest.mark.parametrize("name,first,count", [("cmp_small", 0, 16), ("cmp_large", 5000, 8),
                                              ("crs_small", 100, 16), ("crs_large", 2000, 6)])
def test_device_generator_matches_host(name, first, count):
    wl = configs.WORKLOADS[name]()
    host = wl.spec.generate(first=first, count=count)
    dev = wl.spec.generate_device(first=first, count=count)
    d = dev.samples.cpu().numpy()
    h = np.asarray(host.samples)
    np.testing.assert_array_equal(dev.coords, host.coords)
    np.testing.assert_array_equal(dev.cdp_id, host.cdp_id)
    same = (d.view(np.uint32) == h.view(np.uint32)).mean()
    assert same > 0.999, same
    scale = float(np.abs(h).max())
    assert np.abs(d - h).max() <= 4e-7 * scale
