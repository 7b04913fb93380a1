"""Device-resident sparse containers: COO, CSR, DIA and a switchable wrapper.

Mirrors the reference containers (formats.py:72-250) field for field; the
arrays live in GPU memory (HBM) as torch tensors:

* row/column indices: the reference's uint32 (formats.py:24) stored in
  int32 tensors with identical bits (torch's uint32 support is thin; every
  kernel reads them as uint32, so indices up to 2^32-1 round-trip)
* DIA offsets: int32 (formats.py:25)
* values: float32 / float64 (formats.py:27); anything else promotes to f64
* DIA values: the reference's dense row-major (padded_rows, ndiags) block,
  padded_rows a multiple of ROW_PAD (formats.py:166-207) — this row-major
  tile is what the DIA kernel stages with one TMA bulk copy per tile

Containers are immutable after construction; kernel plans are
cached on the container.  `as_device` uploads any reference-shaped host
container (duck typed on the reference attribute names) once and caches
the device copy, which is how the reference's own drivers can run on the GPU
kernels through a registry (see plugin.py / INTEGRATION.md).
"""

from __future__ import annotations

import threading
import weakref
from dataclasses import dataclass, field
from enum import Enum
from typing import Union

import numpy as np
import torch

INDEX_DTYPE = np.dtype(np.uint32)
OFFSET_DTYPE = np.dtype(np.int32)
DEFAULT_SCALAR = np.dtype(np.float64)
SCALAR_DTYPES = (np.dtype(np.float32), np.dtype(np.float64))
ROW_PAD = 8

_TORCH_SCALARS = {np.dtype(np.float32): torch.float32, np.dtype(np.float64): torch.float64}


class Format(str, Enum):
    """Identifier for the three concrete storage layouts (formats.py:33-38)."""

    COO = "coo"
    CSR = "csr"
    DIA = "dia"


def round_up(n: int, multiple: int) -> int:
    """Round ``n`` up to the next multiple of ``multiple`` (formats.py:41-45)."""
    if multiple <= 0:
        raise ValueError("multiple must be positive")
    return -(-int(n) // multiple) * multiple


def default_device() -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2304_09511_b200 needs a CUDA device (there is no CPU path)")
    return torch.device("cuda", torch.cuda.current_device())


def _target(device) -> torch.device:
    return torch.device(device) if device is not None else default_device()


def index_tensor(values, device=None) -> torch.Tensor:
    """uint32 index array -> int32 device tensor with the same bits."""
    dev = _target(device)
    if isinstance(values, torch.Tensor):
        t = values
        if t.dtype != torch.int32:
            if t.dtype == torch.uint32:
                t = t.view(torch.int32)
            else:
                t = t.to(torch.int64).to(torch.int32)  # wraps like uint32 -> int32 bits
        return t.to(dev).contiguous().reshape(-1)
    arr = np.ascontiguousarray(np.asarray(values).astype(np.int64, copy=False).astype(INDEX_DTYPE)).reshape(-1)
    return torch.from_numpy(arr.view(np.int32)).to(dev)


def offset_tensor(values, device=None) -> torch.Tensor:
    dev = _target(device)
    if isinstance(values, torch.Tensor):
        return values.to(device=dev, dtype=torch.int32).contiguous().reshape(-1)
    arr = np.ascontiguousarray(values, dtype=OFFSET_DTYPE).reshape(-1)
    return torch.from_numpy(arr).to(dev)


def scalar_tensor(values, dtype=None, device=None) -> torch.Tensor:
    """f32/f64 keep their dtype, anything else becomes f64 (formats.py:58-69)."""
    dev = _target(device)
    if isinstance(values, torch.Tensor):
        if dtype is not None:
            tgt = _TORCH_SCALARS[np.dtype(dtype)]
        elif values.dtype in (torch.float32, torch.float64):
            tgt = values.dtype
        else:
            tgt = torch.float64
        return values.to(device=dev, dtype=tgt).contiguous()
    arr = np.asarray(values)
    if dtype is not None:
        arr = np.ascontiguousarray(arr, dtype=np.dtype(dtype))
    elif arr.dtype in SCALAR_DTYPES:
        arr = np.ascontiguousarray(arr)
    else:
        arr = np.ascontiguousarray(arr, dtype=DEFAULT_SCALAR)
    return torch.from_numpy(arr).to(dev)


def host_indices(t: torch.Tensor) -> np.ndarray:
    """Device int32 index tensor -> host uint32 numpy (same bits)."""
    return t.detach().cpu().numpy().view(np.uint32)


@dataclass(frozen=True)
class MatrixShape:
    """Logical dimensions plus stored entry count (formats.py:72-78)."""

    nrows: int
    ncols: int
    nnz: int


class _Container:
    """Shared properties and the per-container plan cache."""

    shape: MatrixShape
    values: torch.Tensor

    def _init_cache(self) -> None:
        object.__setattr__(self, "_plans", {})
        object.__setattr__(self, "_plan_lock", threading.Lock())

    @property
    def nrows(self) -> int:
        return self.shape.nrows

    @property
    def ncols(self) -> int:
        return self.shape.ncols

    @property
    def nnz(self) -> int:
        return self.shape.nnz

    @property
    def device(self) -> torch.device:
        return self.values.device

    @property
    def dtype(self) -> np.dtype:
        return np.dtype(np.float64) if self.values.dtype == torch.float64 else np.dtype(np.float32)

    def plan(self, key, factory):
        """Return the cached plan for `key`, creating it once."""
        with self._plan_lock:
            p = self._plans.get(key)
            if p is None:
                p = factory()
                self._plans[key] = p
            return p


@dataclass(eq=False)
class CooMatrix(_Container):
    """Coordinate triples (formats.py:81-121); `sorted` asserts strict
    (row, col) order without duplicates."""

    shape: MatrixShape
    row_indices: torch.Tensor
    col_indices: torch.Tensor
    values: torch.Tensor
    sorted: bool = False

    def __post_init__(self) -> None:
        dev = self.values.device if isinstance(self.values, torch.Tensor) and self.values.is_cuda else None
        self.values = scalar_tensor(self.values, device=dev)
        dev = self.values.device
        self.row_indices = index_tensor(self.row_indices, dev)
        self.col_indices = index_tensor(self.col_indices, dev)
        self._init_cache()

    @classmethod
    def from_arrays(cls, nrows, ncols, rows, cols, values, sorted=False, device=None) -> "CooMatrix":
        values = scalar_tensor(values, device=device)
        shape = MatrixShape(int(nrows), int(ncols), int(values.shape[0]))
        return cls(shape, index_tensor(rows, values.device), index_tensor(cols, values.device), values, sorted)

    @property
    def format(self) -> Format:
        return Format.COO

    def to_host(self) -> dict:
        return {"shape": self.shape, "row_indices": host_indices(self.row_indices),
                "col_indices": host_indices(self.col_indices), "values": self.values.cpu().numpy(),
                "sorted": self.sorted}


@dataclass(eq=False)
class CsrMatrix(_Container):
    """Compressed sparse rows (formats.py:124-163)."""

    shape: MatrixShape
    row_pointers: torch.Tensor
    col_indices: torch.Tensor
    values: torch.Tensor

    def __post_init__(self) -> None:
        dev = self.values.device if isinstance(self.values, torch.Tensor) and self.values.is_cuda else None
        self.values = scalar_tensor(self.values, device=dev)
        dev = self.values.device
        self.row_pointers = index_tensor(self.row_pointers, dev)
        self.col_indices = index_tensor(self.col_indices, dev)
        self._init_cache()

    @classmethod
    def from_arrays(cls, nrows, ncols, row_pointers, cols, values, device=None) -> "CsrMatrix":
        values = scalar_tensor(values, device=device)
        shape = MatrixShape(int(nrows), int(ncols), int(values.shape[0]))
        return cls(shape, index_tensor(row_pointers, values.device), index_tensor(cols, values.device), values)

    @property
    def format(self) -> Format:
        return Format.CSR

    def to_host(self) -> dict:
        return {"shape": self.shape, "row_pointers": host_indices(self.row_pointers),
                "col_indices": host_indices(self.col_indices), "values": self.values.cpu().numpy()}


@dataclass(eq=False)
class DiaMatrix(_Container):
    """Diagonal storage (formats.py:166-207): strictly increasing offsets and
    a dense (padded_rows, ndiags) row-major block, out-of-matrix cells zero."""

    shape: MatrixShape
    offsets: torch.Tensor
    values: torch.Tensor

    def __post_init__(self) -> None:
        dev = self.values.device if isinstance(self.values, torch.Tensor) and self.values.is_cuda else None
        self.values = scalar_tensor(self.values, device=dev)
        self.offsets = offset_tensor(self.offsets, self.values.device)
        self._init_cache()

    @property
    def ndiags(self) -> int:
        return int(self.offsets.shape[0])

    @property
    def padded_rows(self) -> int:
        return int(self.values.shape[0]) if self.values.dim() == 2 else 0

    @property
    def format(self) -> Format:
        return Format.DIA

    def to_host(self) -> dict:
        return {"shape": self.shape, "offsets": self.offsets.cpu().numpy(), "values": self.values.cpu().numpy()}


Container = Union[CooMatrix, CsrMatrix, DiaMatrix]


@dataclass(eq=False)
class DynamicMatrix:
    """Wrapper holding one concrete container, switchable at runtime
    (formats.py:213-243)."""

    active: Container = field()

    @classmethod
    def wrap(cls, matrix) -> "DynamicMatrix":
        if isinstance(matrix, DynamicMatrix):
            return matrix
        return cls(matrix)

    @property
    def format(self) -> Format:
        return self.active.format

    @property
    def shape(self) -> MatrixShape:
        return self.active.shape

    @property
    def nrows(self) -> int:
        return self.active.nrows

    @property
    def ncols(self) -> int:
        return self.active.ncols

    @property
    def nnz(self) -> int:
        return self.active.nnz


def as_container(matrix) -> Container:
    """Unwrap a DynamicMatrix (ours or the reference's); containers pass through."""
    if isinstance(matrix, DynamicMatrix):
        return matrix.active
    if not isinstance(matrix, _Container) and hasattr(matrix, "active"):
        return matrix.active
    return matrix


# --------------------------------------------------------------- host interop --
_HOST_CACHE: dict = {}
_HOST_LOCK = threading.Lock()


def _upload(host, device) -> Container:
    shape = MatrixShape(int(host.shape.nrows), int(host.shape.ncols), int(host.shape.nnz))
    if hasattr(host, "row_pointers"):
        return CsrMatrix(shape, index_tensor(host.row_pointers, device), index_tensor(host.col_indices, device),
                         scalar_tensor(host.values, device=device))
    if hasattr(host, "offsets"):
        vals = np.asarray(host.values)
        if vals.ndim != 2:
            vals = vals.reshape(0, int(np.asarray(host.offsets).shape[0]))
        return DiaMatrix(shape, offset_tensor(host.offsets, device), scalar_tensor(vals, device=device))
    if hasattr(host, "row_indices"):
        return CooMatrix(shape, index_tensor(host.row_indices, device), index_tensor(host.col_indices, device),
                         scalar_tensor(host.values, device=device), bool(getattr(host, "sorted", False)))
    raise TypeError(f"unsupported container {type(host).__name__}")


def as_device(matrix, device=None) -> Container:
    """Return a device container for `matrix`.

    Our containers pass through.  A reference (numpy) container is uploaded
    once and cached for the lifetime of the host object (containers are
    immutable), so repeated `dispatch` calls from the reference's
    drivers do not re-upload A.
    """
    m = as_container(matrix)
    if isinstance(m, _Container):
        return m
    dev = _target(device)
    key = (id(m), str(dev))
    with _HOST_LOCK:
        hit = _HOST_CACHE.get(key)
        if hit is not None and hit[0]() is m:
            return hit[1]
    dm = _upload(m, dev)
    with _HOST_LOCK:
        try:
            ref = weakref.ref(m, lambda _r, k=key: _HOST_CACHE.pop(k, None))
        except TypeError:  # not weak-referenceable: do not cache
            return dm
        _HOST_CACHE[key] = (ref, dm)
    return dm


# ------------------------------------------------------------------ validate --
def _validate_shape(shape: MatrixShape, out: list) -> None:
    if shape.nrows < 0 or shape.ncols < 0:
        out.append("shape: negative dimension")
    if shape.nnz < 0 or shape.nnz > shape.nrows * shape.ncols:
        out.append("shape: nnz outside [0, nrows*ncols]")


def _u32(t: torch.Tensor) -> torch.Tensor:
    return t.to(torch.int64) & 0xFFFFFFFF


def _validate_coo(m: CooMatrix, out: list) -> None:
    n = m.shape.nnz
    for name, arr in (("row_indices", m.row_indices), ("col_indices", m.col_indices), ("values", m.values)):
        if arr.dim() != 1 or arr.shape[0] != n:
            out.append(f"COO: {name} length != nnz")
            return
    if n == 0:
        return
    r, c = _u32(m.row_indices), _u32(m.col_indices)
    if bool((r >= m.shape.nrows).any()):
        out.append("COO: row index out of range")
    if bool((c >= m.shape.ncols).any()):
        out.append("COO: column index out of range")
    if m.sorted and n > 1:
        ok = (r[1:] > r[:-1]) | ((r[1:] == r[:-1]) & (c[1:] > c[:-1]))
        if not bool(ok.all()):
            out.append("COO: sorted flag set but entries are not strictly (row, col) ordered")


def _validate_csr(m: CsrMatrix, out: list) -> None:
    n = m.shape.nnz
    irp = m.row_pointers
    if irp.dim() != 1 or irp.shape[0] != m.shape.nrows + 1:
        out.append("CSR: IRP length != nrows+1")
        return
    irp64 = _u32(irp)
    if irp.shape[0] and int(irp64[0]) != 0:
        out.append("CSR: IRP[0] != 0")
    if irp.shape[0] and int(irp64[-1]) != n:
        out.append("CSR: IRP[-1] != nnz")
    if irp.shape[0] > 1 and bool((irp64[1:] < irp64[:-1]).any()):
        out.append("CSR: IRP non-decreasing violated")
    for name, arr in (("col_indices", m.col_indices), ("values", m.values)):
        if arr.dim() != 1 or arr.shape[0] != n:
            out.append(f"CSR: {name} length != nnz")
            return
    if n and bool((_u32(m.col_indices) >= m.shape.ncols).any()):
        out.append("CSR: column index out of range")


def _validate_dia(m: DiaMatrix, out: list) -> None:
    offs = m.offsets.to(torch.int64)
    nd = offs.shape[0]
    if nd > 1 and bool((offs[1:] <= offs[:-1]).any()):
        out.append("DIA: offsets not strictly increasing")
    if nd and bool(((offs <= -max(m.shape.nrows, 1)) | (offs >= max(m.shape.ncols, 1))).any()):
        out.append("DIA: offset out of range")
    if m.values.dim() != 2 or m.values.shape[1] != nd:
        out.append("DIA: values is not a (padded_rows, ndiags) block")
        return
    if m.padded_rows < m.shape.nrows:
        out.append("DIA: padded_rows < nrows")
        return
    if nd == 0:
        return
    rows = torch.arange(m.padded_rows, device=m.values.device, dtype=torch.int64)[:, None]
    k = rows + offs[None, :]
    outside = (k < 0) | (k >= m.shape.ncols) | (rows >= m.shape.nrows)
    if bool((m.values[outside] != 0).any()):
        out.append("DIA: padding cells must be zero")


def validate(matrix) -> list:
    """Collect invariant violations (formats.py:327-346), same messages."""
    m = as_container(matrix)
    out: list = []
    if not isinstance(m, _Container):
        out.append(f"unknown container type: {type(m).__name__}")
        return out
    _validate_shape(m.shape, out)
    if isinstance(m, CooMatrix):
        _validate_coo(m, out)
    elif isinstance(m, CsrMatrix):
        _validate_csr(m, out)
    elif isinstance(m, DiaMatrix):
        _validate_dia(m, out)
    return out
