"""B200-native semblance parameter search (CMP + CRS), after arXiv 1907.11678.

A drop-in for the hot path of the reference library velan
(/root/reference/proj/include/velan): traveltime -> hit/interpolation ->
windowed semblance -> argmax + stack, as hand-written sm_100a CUDA kernels
behind the C-ABI in include/velan_gpu.h.  See DESIGN.md.
"""
from .api import (  # noqa: F401
    CacheStats,
    ConfigError,
    CrsAbcGrid,
    Dataset,
    DeviceError,
    Engine,
    ParameterError,
    Plan,
    ScanConfig,
    ScanResult,
    VelanError,
    describe,
    device_count,
    neighbors_of,
    run_cmp,
    run_crs,
    scan_cdp,
    scan_central_cdp,
    slowness_grid,
    velocity_grid,
)
from . import configs  # noqa: F401
from .files import (  # noqa: F401
    FormatError,
    SMB1Writer,
    SSF1Reader,
    read_smb1,
    read_ssf1,
    run_cmp_file,
    run_crs_file,
    write_smb1,
    write_ssf1,
)

__all__ = [
    "CacheStats", "ConfigError", "CrsAbcGrid", "Dataset", "DeviceError",
    "Engine", "ParameterError", "Plan", "ScanConfig", "ScanResult",
    "VelanError", "describe", "device_count", "neighbors_of", "run_cmp", "run_crs",
    "scan_cdp", "scan_central_cdp", "slowness_grid", "velocity_grid",
    "configs", "FormatError", "SMB1Writer", "SSF1Reader", "read_smb1", "read_ssf1",
    "run_cmp_file", "run_crs_file", "write_smb1", "write_ssf1",
]
