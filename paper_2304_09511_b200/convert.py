"""On-device conversions between COO, CSR and DIA (convert.py:1-209).

COO is the hub format, as in the reference.  Index structures are produced
by the sm_100a kernels of libspmv_b200.so and are bit-exact with the
reference; values are copied (or, for duplicate coordinates in sort_coo,
summed in np.add.reduceat order), so they are bit-exact too.
"""

from __future__ import annotations

import ctypes
from dataclasses import dataclass

import numpy as np
import torch

from . import _lib
from .errors import FillRatioExceeded, UnsortedInput
from .formats import (
    ROW_PAD,
    Container,
    CooMatrix,
    CsrMatrix,
    DiaMatrix,
    DynamicMatrix,
    Format,
    MatrixShape,
    as_container,
    as_device,
    round_up,
    scalar_tensor,
)

DEFAULT_FILL_RATIO = 10.0


@dataclass(frozen=True)
class DiaFillPolicy:
    """Budget for DIA construction (convert.py:34-44)."""

    max_fill_ratio: float = DEFAULT_FILL_RATIO
    max_ndiags: int | None = None


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr() if t.numel() else 0


def _empty_idx(n: int, dev) -> torch.Tensor:
    return torch.empty(n, dtype=torch.int32, device=dev)


def dense_to_coo(dense, dtype=None, device=None) -> CooMatrix:
    """Sorted COO from a dense 2-D array, dropping exact zeros (convert.py:47-57).

    A constructor convenience (not on the SpMV path): the nonzero scan runs
    on the host array the caller already holds."""
    arr = np.asarray(dense.cpu() if isinstance(dense, torch.Tensor) else dense)
    if arr.ndim != 2:
        raise ValueError("dense_to_coo expects a 2-D array")
    rows, cols = np.nonzero(arr)
    vals = arr[rows, cols]
    values = scalar_tensor(vals, dtype, device=device)
    shape = MatrixShape(int(arr.shape[0]), int(arr.shape[1]), int(values.shape[0]))
    return CooMatrix(shape, rows, cols, values, sorted=True)


def sort_coo(coo) -> CooMatrix:
    """(row, col)-sorted COO with duplicates summed (convert.py:60-84).

    A flagged-sorted matrix is returned unchanged.  Otherwise, on the device:
    a stable radix sort on the row (storage index as payload), each row's
    columns sorted by (column, storage index), duplicate runs added in
    np.add.reduceat order (first + numpy pairwise sum of the rest), zero sums
    kept (csrc/convert.cu spmv_sort_coo)."""
    coo = as_device(coo)
    if coo.sorted:
        return coo
    dev = coo.values.device
    nnz = coo.nnz
    ai, aj = _empty_idx(nnz, dev), _empty_idx(nnz, dev)
    av = torch.empty(nnz, dtype=coo.values.dtype, device=dev)
    n_out = ctypes.c_int64()
    _lib.call("spmv_sort_coo", _lib.dtype_code(coo.values.dtype), max(coo.nrows, 1), max(coo.ncols, 1), nnz,
              _ptr(coo.row_indices), _ptr(coo.col_indices), _ptr(coo.values), _ptr(ai), _ptr(aj), _ptr(av),
              ctypes.byref(n_out), _stream(coo.values))
    n = int(n_out.value)
    if n < nnz:  # duplicates merged: shrink to the merged count
        ai, aj, av = ai[:n].clone(), aj[:n].clone(), av[:n].clone()
    return CooMatrix(MatrixShape(coo.nrows, coo.ncols, n), ai, aj, av, sorted=True)


def coo_to_csr(coo) -> CsrMatrix:
    """Compress a sorted COO into CSR (convert.py:87-94)."""
    coo = as_device(coo)
    if not coo.sorted:
        raise UnsortedInput("coo_to_csr requires a sorted, duplicate-free COO")
    dev = coo.values.device
    irp = _empty_idx(coo.nrows + 1, dev)
    aj = _empty_idx(coo.nnz, dev)
    av = torch.empty(coo.nnz, dtype=coo.values.dtype, device=dev)
    _lib.call("spmv_coo_to_csr", _lib.dtype_code(coo.values.dtype), coo.nrows, coo.nnz, _ptr(coo.row_indices),
              _ptr(coo.col_indices), _ptr(coo.values), _ptr(irp), _ptr(aj), _ptr(av), _stream(coo.values))
    return CsrMatrix(coo.shape, irp, aj, av)


def csr_to_coo(csr) -> CooMatrix:
    """Expand CSR row pointers (convert.py:97-110); `sorted` iff columns
    strictly increase within every row."""
    csr = as_device(csr)
    dev = csr.values.device
    ai, aj = _empty_idx(csr.nnz, dev), _empty_idx(csr.nnz, dev)
    av = torch.empty(csr.nnz, dtype=csr.values.dtype, device=dev)
    flag = ctypes.c_int(1)
    _lib.call("spmv_csr_to_coo", _lib.dtype_code(csr.values.dtype), csr.nrows, csr.nnz, _ptr(csr.row_pointers),
              _ptr(csr.col_indices), _ptr(csr.values), _ptr(ai), _ptr(aj), _ptr(av), ctypes.byref(flag),
              _stream(csr.values))
    return CooMatrix(csr.shape, ai, aj, av, sorted=bool(flag.value))


def coo_to_dia(coo, policy: DiaFillPolicy | None = None, pad_to: int = ROW_PAD) -> DiaMatrix:
    """Scatter a sorted COO into diagonal storage (convert.py:113-144).

    The diagonal census runs on the device; the fill policy is applied on the
    host before the dense block is allocated (convert.py:128-139)."""
    coo = as_device(coo)
    if not coo.sorted:
        raise UnsortedInput("coo_to_dia requires a sorted, duplicate-free COO")
    policy = policy or DiaFillPolicy()
    shape = coo.shape
    dev = coo.values.device
    h = ctypes.c_void_p()
    nd = ctypes.c_int64()
    _lib.call("spmv_coo_to_dia_analyze", shape.nrows, shape.ncols, shape.nnz, _ptr(coo.row_indices),
              _ptr(coo.col_indices), _stream(coo.values), ctypes.byref(h), ctypes.byref(nd))
    try:
        ndiags = int(nd.value)
        padded_rows = round_up(shape.nrows, pad_to) if shape.nrows else 0
        max_ndiags = policy.max_ndiags
        if max_ndiags is None:
            max_ndiags = max(shape.nrows + shape.ncols - 1, 0)
        if ndiags > max_ndiags:
            raise FillRatioExceeded(f"DIA would need {ndiags} diagonals, over the cap of {max_ndiags}")
        stored = padded_rows * ndiags
        budget = policy.max_fill_ratio * max(shape.nnz, 1)
        if stored > budget:
            raise FillRatioExceeded(
                f"DIA would store {stored} cells for {shape.nnz} entries "
                f"(fill ratio cap {policy.max_fill_ratio})")
        offsets = torch.empty(ndiags, dtype=torch.int32, device=dev)
        values = torch.empty((padded_rows, ndiags), dtype=coo.values.dtype, device=dev)
        _lib.call("spmv_coo_to_dia_offsets", h, _ptr(offsets), _stream(coo.values))
        _lib.call("spmv_coo_to_dia_fill", h, _lib.dtype_code(coo.values.dtype), padded_rows, _ptr(coo.row_indices),
                  _ptr(coo.col_indices), _ptr(coo.values), _ptr(values), _stream(coo.values))
    finally:
        _lib.load().spmv_dia_builder_destroy(h)
    return DiaMatrix(shape, offsets, values)


def dia_to_coo(dia) -> CooMatrix:
    """In-bounds, nonzero diagonal cells as a sorted COO (convert.py:147-177)."""
    dia = as_device(dia)
    dev = dia.values.device
    code = _lib.dtype_code(dia.values.dtype)
    h = ctypes.c_void_p()
    n_out = ctypes.c_int64()
    _lib.call("spmv_dia_to_coo_count", code, dia.nrows, dia.ncols, dia.ndiags, _ptr(dia.offsets), _ptr(dia.values),
              _stream(dia.values), ctypes.byref(h), ctypes.byref(n_out))
    try:
        n = int(n_out.value)
        ai, aj = _empty_idx(n, dev), _empty_idx(n, dev)
        av = torch.empty(n, dtype=dia.values.dtype, device=dev)
        _lib.call("spmv_dia_to_coo_fill", h, code, _ptr(dia.offsets), _ptr(dia.values), _ptr(ai), _ptr(aj), _ptr(av),
                  _stream(dia.values))
    finally:
        _lib.load().spmv_dia_collect_destroy(h)
    return CooMatrix(MatrixShape(dia.nrows, dia.ncols, n), ai, aj, av, sorted=True)


def to_format(matrix, target: Format, policy: DiaFillPolicy | None = None, pad_to: int = ROW_PAD) -> Container:
    """Convert any container (or wrapper) to ``target`` via the COO hub
    (convert.py:180-202).  Same-format input is returned untouched, except
    that a COO result is always sorted."""
    m = as_device(as_container(matrix))
    target = Format(target)
    if m.format == target:
        return sort_coo(m) if isinstance(m, CooMatrix) else m
    if isinstance(m, CsrMatrix):
        hub = csr_to_coo(m)
    elif isinstance(m, DiaMatrix):
        hub = dia_to_coo(m)
    else:
        hub = sort_coo(m)
    hub = sort_coo(hub)
    if target == Format.COO:
        return hub
    if target == Format.CSR:
        return coo_to_csr(hub)
    return coo_to_dia(hub, policy, pad_to)


def switch_format(matrix: DynamicMatrix, target: Format, policy: DiaFillPolicy | None = None,
                  pad_to: int = ROW_PAD) -> DynamicMatrix:
    """Wrapper whose active container uses ``target`` (convert.py:205-209)."""
    return DynamicMatrix(to_format(matrix, target, policy, pad_to))
