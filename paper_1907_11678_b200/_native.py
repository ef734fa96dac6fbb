"""ctypes binding of the C-ABI in include/velan_gpu.h.

The shared library is built in-tree (``make lib``) at
``paper_1907_11678_b200/_lib/libvelan_gpu.so``.  There is no fallback: if the
library is missing, importing this module raises, and every scan fails loudly
rather than running anywhere but the CUDA kernels.
"""
from __future__ import annotations

import ctypes as C
import os

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("VELAN_GPU_LIB") or os.path.join(_HERE, "_lib", "libvelan_gpu.so")

OK, ECONFIG, EPARAM, ERUNTIME, ENODEV = 0, 1, 2, 3, 4
OP_NMO, OP_CRS_D2, OP_CRS_ABC = 0, 1, 2
VARIANT_EXACT, VARIANT_FAST = 0, 1
MEM_HOST, MEM_DEVICE = 0, 1


class Dataset(C.Structure):
    _fields_ = [
        ("n_gathers", C.c_int32),
        ("max_traces", C.c_int32),
        ("ns", C.c_int32),
        ("dt_us", C.c_uint32),
        ("cdp_id", C.c_void_p),
        ("ntraces", C.c_void_p),
        ("coords", C.c_void_p),
        ("samples", C.c_void_p),
        ("samples_mem", C.c_int32),
        ("samples_device", C.c_int32),
    ]


class Scan(C.Structure):
    _fields_ = [
        ("op", C.c_int32),
        ("variant", C.c_int32),
        ("w", C.c_int32),
        ("n_a", C.c_int32),
        ("n_b", C.c_int32),
        ("n_c", C.c_int32),
        ("a", C.c_void_p),
        ("b", C.c_void_p),
        ("v", C.c_void_p),
        ("apm", C.c_double),
        ("row_first", C.c_int32),
        ("row_count", C.c_int32),
    ]


class Result(C.Structure):
    _fields_ = [
        ("out_mem", C.c_int32),
        ("best_idx", C.c_void_p),
        ("best_semblance", C.c_void_p),
        ("best_stack", C.c_void_p),
        ("matrix", C.c_void_p),
        ("row_gather", C.c_void_p),
        ("valid_intersections", C.c_uint64),
        ("nominal_intersections", C.c_uint64),
        ("kernel_ms", C.c_double),
        ("total_ms", C.c_double),
        ("topk", C.c_int32),
        ("topk_idx", C.c_void_p),
        ("topk_semblance", C.c_void_p),
    ]


class Synth(C.Structure):
    _fields_ = [
        ("kind", C.c_int32),
        ("n_gathers", C.c_int32),
        ("n_traces", C.c_int32),
        ("ns", C.c_int32),
        ("dt_us", C.c_uint32),
        ("spacing", C.c_double),
        ("h0", C.c_double),
        ("dh", C.c_double),
        ("n_events", C.c_int32),
        ("t0_lo", C.c_double),
        ("t0_hi", C.c_double),
        ("v_lo", C.c_double),
        ("v_hi", C.c_double),
        ("v_profile", C.c_int32),
        ("v_trend_0", C.c_double),
        ("v_trend_slope", C.c_double),
        ("v_perturb", C.c_double),
        ("amp_lo", C.c_double),
        ("amp_hi", C.c_double),
        ("freq", C.c_double),
        ("sigma", C.c_double),
        ("a_abs", C.c_double),
        ("b_max", C.c_double),
        ("seed", C.c_uint64),
        ("gather_first", C.c_int32),
        ("n_line", C.c_int32),
        ("n_threads", C.c_int32),
    ]


class SSF1Info(C.Structure):
    _fields_ = [
        ("n_gathers", C.c_uint32),
        ("fold", C.c_uint32),
        ("ns", C.c_uint32),
        ("dt_us", C.c_uint32),
        ("uniform", C.c_int32),
        ("metadata_bytes", C.c_uint64),
        ("file_bytes", C.c_uint64),
    ]


# Every symbol include/velan_gpu.h declares, with its ctypes signature.
_P = C.c_void_p
SIGNATURES = {
    "velan_gpu_abi_version": (C.c_int, []),
    "velan_gpu_abi_layout": (C.c_int, [_P]),
    "velan_gpu_last_error": (C.c_char_p, []),
    "velan_gpu_device_count": (C.c_int, []),
    "velan_gpu_create": (C.c_int, [_P, C.c_int32, C.POINTER(C.c_void_p)]),
    "velan_gpu_destroy": (None, [_P]),
    "velan_gpu_validate": (C.c_int, [C.POINTER(Dataset), C.POINTER(Scan)]),
    "velan_gpu_describe": (C.c_int, [C.POINTER(Dataset), C.POINTER(Scan), _P, _P, _P, _P,
                                     C.c_int64, C.POINTER(C.c_int64), C.POINTER(C.c_uint64)]),
    "velan_gpu_cmp": (C.c_int, [_P, C.POINTER(Dataset), C.POINTER(Scan), C.POINTER(Result)]),
    "velan_gpu_crs": (C.c_int, [_P, C.POINTER(Dataset), C.POINTER(Scan), C.POINTER(Result)]),
    "velan_gpu_plan_create": (C.c_int, [_P, C.POINTER(Dataset), C.POINTER(Scan), C.POINTER(C.c_void_p)]),
    "velan_gpu_plan_execute": (C.c_int, [_P, C.POINTER(Result), _P]),
    "velan_gpu_plan_launches": (C.c_int, [_P]),
    "velan_gpu_plan_destroy": (None, [_P]),
    "velan_gpu_nmo_correct": (C.c_int, [_P, C.POINTER(Dataset), C.POINTER(Scan), _P, _P]),
    "velan_gpu_hit_batch": (C.c_int, [_P, C.c_int32, C.c_double, C.c_int32, C.c_int32, C.c_int32, _P, _P, _P]),
    "velan_gpu_synth_generate": (C.c_int, [C.POINTER(Synth), _P, _P, _P, _P]),
    "velan_gpu_synth_generate_device": (C.c_int, [C.POINTER(Synth), _P, _P]),
    "velan_gpu_synth_line_events": (C.c_int, [C.POINTER(Synth), _P]),
    "velan_gpu_measure_fp32_peak": (C.c_int, [C.c_int32, C.POINTER(C.c_double)]),
    "velan_ssf1_open": (C.c_int, [C.c_char_p, C.POINTER(C.c_void_p), C.POINTER(SSF1Info)]),
    "velan_ssf1_close": (None, [_P]),
    "velan_ssf1_gathers": (C.c_int, [_P, _P, _P, _P, _P]),
    "velan_ssf1_metadata": (C.c_int, [_P, _P, C.c_uint64]),
    "velan_ssf1_read": (C.c_int, [_P, C.c_int32, C.c_int32, C.c_int32, _P, _P, C.c_int32]),
    "velan_ssf1_read_list": (C.c_int, [_P, _P, C.c_int32, C.c_int32, _P, _P, C.c_int32]),
    "velan_ssf1_midpoints": (C.c_int, [_P, _P, _P]),
    "velan_ssf1_write": (C.c_int, [C.c_char_p, C.POINTER(Dataset), C.c_char_p, C.c_uint64]),
    "velan_smb1_begin": (C.c_int, [C.c_char_p, C.c_uint32, C.c_int32, C.c_int32, C.c_int32,
                                   C.POINTER(C.c_void_p)]),
    "velan_smb1_append": (C.c_int, [_P, C.c_int32, _P, _P, _P, _P]),
    "velan_smb1_end": (C.c_int, [_P]),
}

_lib = None


def load() -> C.CDLL:
    """Load (once) the in-tree CUDA library; raise if it was not built."""
    global _lib
    if _lib is not None:
        return _lib
    if not os.path.exists(LIB_PATH):
        raise ImportError(
            f"velan_gpu native library not built: {LIB_PATH} is missing "
            "(run `make lib` or __graft_entry__.build()); there is no CPU "
            "fallback for the scan")
    lib = C.CDLL(LIB_PATH)
    for name, (res, args) in SIGNATURES.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    _lib = lib
    return lib


def last_error() -> str:
    msg = load().velan_gpu_last_error()
    return msg.decode() if msg else ""
