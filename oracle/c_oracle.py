"""ctypes binding of oracle/build/libspmv_oracle.so — TEST INFRASTRUCTURE ONLY.

See spmv_oracle.c for the reference lines each kernel restates.
"""

from __future__ import annotations

import ctypes
import subprocess
from pathlib import Path

import numpy as np

HERE = Path(__file__).resolve().parent
LIB = HERE / "build" / "libspmv_oracle.so"

_lib = None


def build() -> Path:
    if not LIB.exists() or LIB.stat().st_mtime < (HERE / "spmv_oracle.c").stat().st_mtime:
        subprocess.run(["make", "-s", "-C", str(HERE)], check=True)
    return LIB


def lib():
    global _lib
    if _lib is None:
        build()
        _lib = ctypes.CDLL(str(LIB))
        _lib.oracle_max_threads.restype = ctypes.c_int
    return _lib


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def _suffix(dtype):
    return "f64" if np.dtype(dtype) == np.float64 else "f32"


def set_threads(n: int) -> None:
    lib().oracle_set_threads(ctypes.c_int(n))


def max_threads() -> int:
    return int(lib().oracle_max_threads())


def csr_plain(nrows, irp, aj, av, x):
    irp = np.ascontiguousarray(irp, dtype=np.uint32)
    aj = np.ascontiguousarray(aj, dtype=np.uint32)
    av = np.ascontiguousarray(av)
    x = np.ascontiguousarray(x, dtype=av.dtype)
    y = np.empty(nrows, dtype=av.dtype)
    getattr(lib(), "oracle_csr_plain_" + _suffix(av.dtype))(
        ctypes.c_int64(nrows), _p(irp), _p(aj), _p(av), _p(x), _p(y))
    return y


def coo_plain(nrows, ai, aj, av, x, row_sorted=True):
    ai = np.ascontiguousarray(ai, dtype=np.uint32)
    aj = np.ascontiguousarray(aj, dtype=np.uint32)
    av = np.ascontiguousarray(av)
    x = np.ascontiguousarray(x, dtype=av.dtype)
    y = np.empty(nrows, dtype=av.dtype)
    getattr(lib(), "oracle_coo_plain_" + _suffix(av.dtype))(
        ctypes.c_int64(nrows), ctypes.c_int64(av.shape[0]), _p(ai), _p(aj), _p(av), _p(x), _p(y),
        ctypes.c_int(1 if row_sorted else 0))
    return y


def dia_plain(nrows, ncols, offsets, values, x):
    offsets = np.ascontiguousarray(offsets, dtype=np.int32)
    values = np.ascontiguousarray(values)
    x = np.ascontiguousarray(x, dtype=values.dtype)
    y = np.empty(nrows, dtype=values.dtype)
    getattr(lib(), "oracle_dia_plain_" + _suffix(values.dtype))(
        ctypes.c_int64(nrows), ctypes.c_int64(ncols), ctypes.c_int64(offsets.shape[0]), _p(offsets),
        _p(values), _p(x), _p(y))
    return y


def csr_vla(nrows, irp, aj, av, x, lanes):
    irp = np.ascontiguousarray(irp, dtype=np.uint32)
    aj = np.ascontiguousarray(aj, dtype=np.uint32)
    av = np.ascontiguousarray(av)
    x = np.ascontiguousarray(x, dtype=av.dtype)
    y = np.empty(nrows, dtype=av.dtype)
    getattr(lib(), "oracle_csr_vla_" + _suffix(av.dtype))(
        ctypes.c_int64(nrows), _p(irp), _p(aj), _p(av), _p(x), _p(y), ctypes.c_int(lanes))
    return y


def stencil27_rows(nx, ny, nz, r0, r1):
    """Rows [r0, r1) of the f64 27-point operator (matrixio.py:170-210)."""
    irp = np.empty(r1 - r0 + 1, dtype=np.uint32)
    lib().oracle_stencil27_irp(ctypes.c_int64(nx), ctypes.c_int64(ny), ctypes.c_int64(nz), ctypes.c_int64(r0),
                               ctypes.c_int64(r1), _p(irp))
    nnz = int(irp[-1])
    cols = np.empty(nnz, dtype=np.uint32)
    vals = np.empty(nnz, dtype=np.float64)
    lib().oracle_stencil27_fill_f64(ctypes.c_int64(nx), ctypes.c_int64(ny), ctypes.c_int64(nz), ctypes.c_int64(r0),
                                    ctypes.c_int64(r1), _p(irp), _p(cols), _p(vals))
    return irp, cols, vals
