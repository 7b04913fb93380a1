"""ctypes binding of libspmv_b200.so (the C ABI in include/spmv_b200.h).

The library is built in-tree by `_build.build()`.  There is no fallback: if
the shared library is missing or CUDA is unavailable, every entry point
raises instead of computing anything on the host.
"""

from __future__ import annotations

import ctypes
import threading
from pathlib import Path

from .errors import (
    DeviceError,
    DimensionMismatch,
    FillRatioExceeded,
    IndexOverflow,
    SparseError,
    UnsortedInput,
    UnsupportedCombination,
)

import os

# SPMV_B200_LIB overrides the library path (A/B experiments of two builds).
LIB_PATH = Path(os.environ.get("SPMV_B200_LIB") or (Path(__file__).resolve().parent / "libspmv_b200.so"))

F32, F64 = 0, 1

_STATUS = {
    1: DimensionMismatch,
    2: UnsortedInput,
    3: FillRatioExceeded,
    4: UnsupportedCombination,
    5: DeviceError,
    6: ValueError,
    7: IndexOverflow,
}

_c_i64 = ctypes.c_int64
_c_int = ctypes.c_int
_vp = ctypes.c_void_p
_pi64 = ctypes.POINTER(ctypes.c_int64)
_pint = ctypes.POINTER(ctypes.c_int)
_pu32 = ctypes.POINTER(ctypes.c_uint32)
_pvp = ctypes.POINTER(ctypes.c_void_p)

# name -> argtypes (every function returns int status unless listed in _RESTYPE)
SIGNATURES = {
    "spmv_abi_version": [],
    "spmv_last_error": [],
    "spmv_device_sm_count": [_pint],
    "spmv_csr_plan_create": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _c_int, _vp, _pvp],
    "spmv_csr_plan_destroy": [_vp],
    "spmv_plan_config_init": [_vp],
    "spmv_csr_plan_create_ex": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _pvp],
    "spmv_csr_plan_config": [_vp, _vp],
    "spmv_coo_plan_create_ex": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _pvp],
    "spmv_coo_plan_config": [_vp, _vp],
    "spmv_dia_ex": [_c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp],
    "spmv_debug_csr_phases": [ctypes.POINTER(ctypes.c_ulonglong)],
    "spmv_debug_check_counts": [ctypes.POINTER(ctypes.c_ulonglong)],
    "spmv_csr_plan_info": [_vp, _pi64, _pi64, _pi64],
    "spmv_csr": [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _vp],
    "spmv_csr_plan_tiles": [_vp, _pi64, _pi64],
    "spmv_csr_plan_groups": [_vp, _pint],
    "spmv_csr_plan_path": [_vp, _pint, _pi64],
    "spmv_csr_gapped": [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _vp],
    "spmv_coo_plan_groups": [_vp, _pint],
    "spmv_coo_plan_path": [_vp, _pint, _pi64],
    "spmv_csr_host": [_vp, _vp, _vp, _vp, _vp, _vp, _c_int, _vp],
    "spmv_host_pipe_create": [_pvp],
    "spmv_host_pipe_destroy": [_vp],
    "spmv_coo_host": [_vp, _vp, _vp, _vp, _vp, _vp, _c_int, _vp],
    "spmv_dia_host": [_vp, _c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _c_i64, _vp, _vp, _vp, _c_int, _vp, _vp],
    "spmv_csr_plan_tile_info": [_vp, _vp, _vp, _vp, _vp],
    "spmv_csr_range": [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _c_i64, _c_i64, _c_int, _vp],
    "spmv_csr_vla": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _c_int, _vp],
    "spmv_csr_vla_planned": [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _c_int, _vp],
    "spmv_coo_plan_create": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _pvp],
    "spmv_coo_plan_destroy": [_vp],
    "spmv_coo_plan_info": [_vp, _pi64, _pi64, _pi64, _pint, _pi64],
    "spmv_coo": [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _vp],
    "spmv_coo_vla": [_vp, _vp, _vp, _vp, _vp, _c_i64, _c_i64, _vp, _c_int, _pi64, _vp],
    "spmv_dia": [_c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _vp],
    "spmv_dia_gapped": [_c_int, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _c_i64, _c_i64, _c_i64, _vp, _c_i64,
                        _c_i64, _vp],
    "spmv_coo_to_csr": [_c_int, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _vp],
    "spmv_csr_to_coo": [_c_int, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _pint, _vp],
    "spmv_coo_to_dia_analyze": [_c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _pvp, _pi64],
    "spmv_coo_to_dia_offsets": [_vp, _vp, _vp],
    "spmv_coo_to_dia_fill": [_vp, _c_int, _c_i64, _vp, _vp, _vp, _vp, _vp],
    "spmv_dia_builder_destroy": [_vp],
    "spmv_dia_to_coo_count": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _pvp, _pi64],
    "spmv_dia_to_coo_fill": [_vp, _c_int, _vp, _vp, _vp, _vp, _vp, _vp],
    "spmv_dia_collect_destroy": [_vp],
    "spmv_sort_coo": [_c_int, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp, _vp, _vp, _pi64, _vp],
    "spmv_stencil27_nnz": [_c_i64, _c_i64, _c_i64, _pi64],
    "spmv_stencil27_fill": [_c_int, _c_i64, _c_i64, _c_i64, _c_i64, _c_i64, _vp, _vp, _vp, _vp],
    "spmv_csr_col_bounds": [_c_i64, _vp, _vp, _vp, _pu32, _pu32],
    "spmv_csr_halo_split": [_c_i64, _vp, _vp, _c_i64, _c_i64, _vp, _pi64, _pi64],
    "spmv_dot_workspace_entries": [],
    "spmv_dot": [_c_int, _c_i64, _vp, _vp, _vp, _vp],
    "spmv_cg_update": [_c_int, _c_i64, ctypes.c_double, _vp, _vp, _vp, _vp, _vp, _vp],
    "spmv_cg_direction": [_c_int, _c_i64, ctypes.c_double, _vp, _vp, _vp],
}
_RESTYPE = {"spmv_last_error": ctypes.c_char_p}

_lock = threading.Lock()
_handle = None


def load():
    """Load (once) and return the CDLL; raises if the library is missing."""
    global _handle
    if _handle is not None:
        return _handle
    with _lock:
        if _handle is None:
            if not LIB_PATH.exists():
                raise ImportError(
                    f"{LIB_PATH} is missing: build it with `python -m paper_2304_09511_b200._build` "
                    "(there is no CPU fallback)")
            lib = ctypes.CDLL(str(LIB_PATH))
            for name, argtypes in SIGNATURES.items():
                fn = getattr(lib, name)
                fn.argtypes = argtypes
                fn.restype = _RESTYPE.get(name, ctypes.c_int)
            _handle = lib
    return _handle


def last_error() -> str:
    msg = load().spmv_last_error()
    return msg.decode(errors="replace") if msg else ""


def check(status: int) -> None:
    """Raise the reference's exception class for a non-zero status."""
    if status == 0:
        return
    exc = _STATUS.get(status, SparseError)
    raise exc(last_error())


def call(name: str, *args) -> None:
    check(getattr(load(), name)(*args))


def dtype_code(torch_dtype) -> int:
    import torch

    if torch_dtype == torch.float64:
        return F64
    if torch_dtype == torch.float32:
        return F32
    raise TypeError(f"unsupported value dtype {torch_dtype}")
