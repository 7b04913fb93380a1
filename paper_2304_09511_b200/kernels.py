"""SpMV entry points, kernel registry and dispatch — the drop-in boundary.

Same names, argument meaning and error behaviour as the reference's
kernels.py (kernels.py:39-297), with every product computed by the sm_100a
kernels of libspmv_b200.so:

  spmv_csr_plain  kernels.py:69-82    CSR-stream + long-row warp chunks
  spmv_coo_plain  kernels.py:56-66    fixed-tile segmented reduction
  spmv_dia_plain  kernels.py:85-101   TMA-staged row tiles
  spmv_*_vla      kernels.py:104-210  sub-warp / CTA lane kernels

Host/device behaviour: a numpy (or list) `x` gets the reference contract —
x is cast to the value dtype on the host (kernels.py:51-52) and a fresh
numpy y is returned; the upload, the product and the download are
pipelined by the C ABI (spmv_*_host, csrc/hostpipe.cuh), y lives in pinned
memory.  A CPU torch tensor x gives a (pinned) CPU tensor back.  A CUDA
tensor `x` stays on the device and a fresh CUDA tensor y is returned.
`out=` may be a CUDA tensor (reused, no allocation) or a CPU tensor that
receives y (pinned for overlapped copies).
Matrices may be our device containers or reference host containers (these
are uploaded once and cached, formats.as_device).
"""

from __future__ import annotations

import ctypes
from enum import Enum

import numpy as np
import torch

from . import _lib
from .errors import DimensionMismatch, UnsortedInput, UnsupportedCombination
from .formats import CooMatrix, CsrMatrix, DiaMatrix, Format, as_container, as_device
from .lanes import LaneConfig
from .planconfig import PlanConfig, _CPlanConfig, plan_config_of


class KernelVersion(str, Enum):
    """Identifier for the two kernel families (kernels.py:39-43)."""

    PLAIN = "plain"
    VLA = "vla"


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(device: torch.device) -> int:
    """The device's current stream handle (torch's raw query: every product
    call needs it, and torch.cuda.current_stream builds a Stream object)."""
    if _raw_stream is not None and device.index is not None:
        return _raw_stream(device.index)
    return torch.cuda.current_stream(device).cuda_stream


def _ptr(t: torch.Tensor) -> int:
    return t.data_ptr() if t.numel() else 0


def _checked_x(m, x):
    """kernels.py:46-53: 1-D of length ncols, cast to the value dtype.

    Returns (device x, origin) with origin "device", "torch_host" (a CPU
    tensor, ideally pinned: copied with non_blocking) or "numpy"."""
    if isinstance(x, torch.Tensor):
        if x.dim() != 1 or x.shape[0] != m.shape.ncols:
            raise DimensionMismatch(f"x has shape {tuple(x.shape)}, expected ({m.shape.ncols},)")
        xv = x
        if xv.dtype != m.values.dtype:
            xv = xv.to(m.values.dtype)  # cast where x lives, like the reference's astype
        if not xv.is_cuda:
            return xv.contiguous().to(m.values.device, non_blocking=xv.is_pinned()), "torch_host"
        if xv.device != m.values.device:
            xv = xv.to(m.values.device)
        return xv.contiguous(), "device"
    xh = np.asarray(x)
    if xh.ndim != 1 or xh.shape[0] != m.shape.ncols:
        raise DimensionMismatch(f"x has shape {xh.shape}, expected ({m.shape.ncols},)")
    if xh.dtype != m.dtype:
        xh = xh.astype(m.dtype)
    xv = torch.from_numpy(np.ascontiguousarray(xh)).to(m.values.device)
    return xv, "numpy"


def _new_y(m, out):
    if out is not None and out.is_cuda:
        if out.shape != (m.shape.nrows,) or out.dtype != m.values.dtype or out.device != m.values.device:
            raise DimensionMismatch("out must be a 1-D tensor of length nrows with the value dtype")
        return out
    if out is not None and (out.shape != (m.shape.nrows,) or out.dtype != m.values.dtype):
        raise DimensionMismatch("out must be a 1-D tensor of length nrows with the value dtype")
    return torch.empty(m.shape.nrows, dtype=m.values.dtype, device=m.values.device)


def _finish(y: torch.Tensor, origin: str, out=None):
    """Deliver y where the caller's x came from (or into a host `out`)."""
    if out is not None and not out.is_cuda:
        out.copy_(y, non_blocking=out.is_pinned())
        torch.cuda.current_stream(y.device).synchronize()
        return out
    if origin == "numpy":
        return y.cpu().numpy()
    if origin == "torch_host":
        return y.cpu()
    return y


# -------------------------------------------------------------------- plans --
class _Plan:
    """Owns a C plan handle; destroyed with the container's plan cache."""

    def __init__(self, kind: str, handle: ctypes.c_void_p, config: PlanConfig | None = None):
        self.kind = kind
        self.handle = handle
        self.requested = config or PlanConfig()

    def config(self) -> PlanConfig:
        """The configuration the plan resolved (what its kernels run)."""
        c = _CPlanConfig()
        _lib.call(f"spmv_{self.kind}_plan_config", self.handle, ctypes.byref(c))
        return PlanConfig.from_c(c)

    def __del__(self):
        try:
            if self.handle:
                name = "spmv_host_pipe_destroy" if self.kind == "host_pipe" else f"spmv_{self.kind}_plan_destroy"
                getattr(_lib.load(), name)(self.handle)
                self.handle = None
        except Exception:
            pass

    def info(self) -> dict:
        if self.kind == "csr":
            a, b, c = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64()
            g = ctypes.c_int()
            _lib.call("spmv_csr_plan_info", self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c))
            _lib.call("spmv_csr_plan_groups", self.handle, ctypes.byref(g))
            ws, nw = ctypes.c_int(), ctypes.c_int64()
            _lib.call("spmv_csr_plan_path", self.handle, ctypes.byref(ws), ctypes.byref(nw))
            info = {"long_rows": a.value, "tile": b.value, "launches": c.value, "groups": g.value, "kernel": "tile",
                    "config": self.config().as_dict()}
            if ws.value:  # tile/groups still serve tile-range launches
                info.update(kernel="panel" if ws.value == 2 else "warp_stream", warps=nw.value)
            return info
        a, b, c, d, e = ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int64(), ctypes.c_int(), ctypes.c_int64()
        g = ctypes.c_int()
        _lib.call("spmv_coo_plan_info", self.handle, ctypes.byref(a), ctypes.byref(b), ctypes.byref(c),
                  ctypes.byref(d), ctypes.byref(e))
        _lib.call("spmv_coo_plan_groups", self.handle, ctypes.byref(g))
        ws, nw = ctypes.c_int(), ctypes.c_int64()
        _lib.call("spmv_coo_plan_path", self.handle, ctypes.byref(ws), ctypes.byref(nw))
        info = {"runs": a.value, "long_runs": b.value, "tile": c.value, "row_sorted": bool(d.value),
                "launches": e.value, "groups": g.value, "kernel": "tile", "config": self.config().as_dict()}
        if ws.value:  # 3: whole-matrix products run the CSR tile kernel on the plan's row-pointer view
            info.update(kernel={1: "warp_stream", 2: "panel", 3: "csr_view"}[ws.value], warps=nw.value)
        return info


def _config(A, config: PlanConfig | None, exact_len: int = 0) -> PlanConfig:
    cfg = config if config is not None else plan_config_of(A)
    if exact_len:
        cfg = cfg.with_(exact_len=int(exact_len))
    return cfg


def csr_plan(A: CsrMatrix, exact_len: int = 0, config: PlanConfig | None = None) -> _Plan:
    """CSR plan: long-row work list from the row-length histogram (cached
    per configuration: the container's attached one unless `config`)."""
    cfg = _config(A, config, exact_len)

    def make():
        h = ctypes.c_void_p()
        c = cfg.to_c()
        _lib.call("spmv_csr_plan_create_ex", _lib.dtype_code(A.values.dtype), A.nrows, A.ncols, A.nnz,
                  _ptr(A.row_pointers), _ptr(A.col_indices), _ptr(A.values), ctypes.byref(c), _stream(A.device),
                  ctypes.byref(h))
        return _Plan("csr", h, cfg)

    return A.plan(("csr", cfg.key()), make)


def coo_plan(A: CooMatrix, config: PlanConfig | None = None) -> _Plan:
    """COO plan: row-order check, optional stable row sort, run table (cached
    per configuration)."""
    cfg = _config(A, config)

    def make():
        h = ctypes.c_void_p()
        c = cfg.to_c()
        _lib.call("spmv_coo_plan_create_ex", _lib.dtype_code(A.values.dtype), A.nrows, A.ncols, A.nnz,
                  _ptr(A.row_indices), _ptr(A.col_indices), _ptr(A.values), ctypes.byref(c), _stream(A.device),
                  ctypes.byref(h))
        return _Plan("coo", h, cfg)

    return A.plan(("coo", cfg.key()), make)


# --------------------------------------------------------- host pipelining --
# x and y in host memory (the reference's numpy contract): the C ABI
# pipelines the x upload, the product and the y download (csrc/hostpipe.cuh).
# y comes back as a fresh numpy array over pinned memory (torch's pinned
# caching allocator), so its download overlaps; pageable numpy x is staged
# by the library's pinned ring.
HOST_CHUNKS = int(__import__("os").environ.get("SPMV_HOST_CHUNKS", "0"))  # 0: library default


def _host_x(A, x):
    """(host x array or tensor in the value dtype, origin) when x lives on
    the host, else None (kernels.py:46-53 checks and cast)."""
    if isinstance(x, torch.Tensor):
        if x.is_cuda:
            return None
        if x.dim() != 1 or x.shape[0] != A.shape.ncols:
            raise DimensionMismatch(f"x has shape {tuple(x.shape)}, expected ({A.shape.ncols},)")
        return x.to(A.values.dtype).contiguous(), "torch_host"
    xh = np.asarray(x)
    if xh.ndim != 1 or xh.shape[0] != A.shape.ncols:
        raise DimensionMismatch(f"x has shape {xh.shape}, expected ({A.shape.ncols},)")
    return np.ascontiguousarray(xh, dtype=A.dtype), "numpy"


def _host_ptr(xh) -> int:
    return xh.data_ptr() if isinstance(xh, torch.Tensor) else xh.ctypes.data


def _host_product(A, x, out, call) -> object:
    """Run `call(x_ptr, y_ptr, stream)` (an spmv_*_host entry point) with
    host x and a pinned host y; None when x is on the device or the matrix
    is empty (the plain path handles those)."""
    hx = _host_x(A, x)
    if hx is None or A.nrows == 0 or A.ncols == 0:
        return None
    xh, origin = hx
    if out is not None:
        if out.is_cuda or out.shape != (A.nrows,) or out.dtype != A.values.dtype or not out.is_contiguous():
            return None
        yh = out
    else:
        yh = torch.empty(A.nrows, dtype=A.values.dtype, pin_memory=True)
    stream = torch.cuda.current_stream(A.device)
    call(_host_ptr(xh), yh.data_ptr(), stream.cuda_stream)
    stream.synchronize()
    if out is not None:
        return out
    return yh.numpy() if origin == "numpy" else yh


def _host_pipe(A) -> "_Plan":
    """A DIA container's own host pipe (staging, copy streams)."""
    def make():
        h = ctypes.c_void_p()
        _lib.call("spmv_host_pipe_create", ctypes.byref(h))
        return _Plan("host_pipe", h)
    return A.plan("host_pipe", make)


# ------------------------------------------------------------------ kernels --
def spmv_coo_plain(A, x, out=None, plan_config: PlanConfig | None = None):
    """``y = A @ x`` with np.add.at semantics (kernels.py:56-66).
    `plan_config` overrides the container's kernel configuration."""
    A = as_device(A)
    p = coo_plan(A, plan_config) if A.nrows else None
    if not (isinstance(x, torch.Tensor) and x.is_cuda):
        y = _host_product(A, x, out, lambda xp, yp, st: _lib.call(
            "spmv_coo_host", p.handle, _ptr(A.row_indices), _ptr(A.col_indices), _ptr(A.values), xp, yp,
            HOST_CHUNKS, st))
        if y is not None:
            return y
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if p is not None:
        _lib.call("spmv_coo", p.handle, _ptr(A.row_indices), _ptr(A.col_indices), _ptr(A.values), _ptr(xv), 0,
                  A.ncols, _ptr(y), _stream(A.device))
    return _finish(y, origin, out)


def spmv_csr_plain(A, x, out=None, plan_config: PlanConfig | None = None):
    """``y = A @ x`` with one left-to-right sum per row (kernels.py:69-82).
    `plan_config` overrides the container's kernel configuration."""
    A = as_device(A)
    p = csr_plan(A, config=plan_config) if A.nrows else None
    if A.nnz and not (isinstance(x, torch.Tensor) and x.is_cuda):
        # host x -> host y: the C ABI pipelines upload / tiles / download
        y = _host_product(A, x, out, lambda xp, yp, st: _lib.call(
            "spmv_csr_host", p.handle, _ptr(A.row_pointers), _ptr(A.col_indices), _ptr(A.values), xp, yp,
            HOST_CHUNKS, st))
        if y is not None:
            return y
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if p is not None:
        _lib.call("spmv_csr", p.handle, _ptr(A.row_pointers), _ptr(A.col_indices), _ptr(A.values), _ptr(xv), 0,
                  A.ncols, _ptr(y), _stream(A.device))
    return _finish(y, origin, out)


def spmv_dia_plain(A, x, out=None, plan_config: PlanConfig | None = None):
    """``y = A @ x`` over stored diagonals (kernels.py:85-101).
    `plan_config` (its dia_* fields) overrides the container's."""
    A = as_device(A)
    cfg = plan_config if plan_config is not None else plan_config_of(A)
    if A.ndiags > 0 and not (isinstance(x, torch.Tensor) and x.is_cuda):
        offs = A.plan("dia_offsets", lambda: A.offsets.cpu().numpy().astype(np.int64))
        pipe = _host_pipe(A)
        c = cfg.to_c()
        y = _host_product(A, x, out, lambda xp, yp, st: _lib.call(
            "spmv_dia_host", pipe.handle, _lib.dtype_code(A.values.dtype), A.nrows, A.ncols, A.ndiags,
            A.padded_rows, _ptr(A.offsets), int(offs.max()), _ptr(A.values), xp, yp, HOST_CHUNKS, ctypes.byref(c),
            st))
        if y is not None:
            return y
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if A.nrows:
        c = cfg.to_c()
        _lib.call("spmv_dia_ex", _lib.dtype_code(A.values.dtype), A.nrows, A.ncols, A.ndiags, A.padded_rows,
                  _ptr(A.offsets), _ptr(A.values), _ptr(xv), 0, 0, A.ncols, _ptr(y), ctypes.byref(c),
                  _stream(A.device))
    return _finish(y, origin, out)


def spmv_coo_vla(A, x, config: LaneConfig | None = None, stats: dict | None = None, out=None):
    """Vector-style COO product (kernels.py:104-140); requires `sorted`.

    When ``stats`` is given the reference's outer step count is recorded
    under ``"outer_steps"``."""
    cfg = config or LaneConfig()
    A = as_device(A)
    if not A.sorted:
        raise UnsortedInput("vla COO kernel requires a sorted, duplicate-free COO")
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    steps = ctypes.c_int64(0)
    if A.nrows:
        p = coo_plan(A)
        _lib.call("spmv_coo_vla", p.handle, _ptr(A.row_indices), _ptr(A.col_indices), _ptr(A.values), _ptr(xv), 0,
                  A.ncols, _ptr(y), int(cfg.lanes), ctypes.byref(steps) if stats is not None else None,
                  _stream(A.device))
    if stats is not None:
        stats["outer_steps"] = int(steps.value)
    return _finish(y, origin, out)


def spmv_csr_vla(A, x, config: LaneConfig | None = None, out=None):
    """Vector-style CSR product (kernels.py:143-171)."""
    cfg = config or LaneConfig()
    A = as_device(A)
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if A.nrows:
        _lib.call("spmv_csr_vla_planned", csr_plan(A).handle, _ptr(A.row_pointers), _ptr(A.col_indices),
                  _ptr(A.values), _ptr(xv), 0, A.ncols, _ptr(y), int(cfg.lanes), _stream(A.device))
    return _finish(y, origin, out)


def spmv_dia_vla(A, x, config: LaneConfig | None = None, out=None):
    """Vector-style DIA product (kernels.py:174-210).  Each row visits its
    diagonals in the same order for every lane count, so the GPU row kernel
    is bit-exact with it for all L."""
    _ = config or LaneConfig()
    return spmv_dia_plain(A, x, out=out)


# ----------------------------------------------------------------- registry --
class KernelRegistry:
    """Dispatch table mapping ``(format, version)`` to a kernel callable
    (kernels.py:213-244).  Callables take ``(matrix, x, config)``."""

    def __init__(self, table=None) -> None:
        self._table = dict(table or {})

    def register(self, fmt, version, fn) -> None:
        self._table[(Format(fmt), KernelVersion(version))] = fn

    def unregister(self, fmt, version) -> None:
        self._table.pop((Format(fmt), KernelVersion(version)), None)

    def supports(self, fmt, version) -> bool:
        return (Format(fmt), KernelVersion(version)) in self._table

    def lookup(self, fmt, version):
        key = (Format(fmt), KernelVersion(version))
        try:
            return self._table[key]
        except KeyError:
            raise UnsupportedCombination(
                f"no kernel registered for ({key[0].value}, {key[1].value})") from None

    def pairs(self) -> list:
        return sorted(self._table)

    def copy(self) -> "KernelRegistry":
        return KernelRegistry(self._table)


def _plain_coo(A, x, config):
    return spmv_coo_plain(A, x)


def _plain_csr(A, x, config):
    return spmv_csr_plain(A, x)


def _plain_dia(A, x, config):
    return spmv_dia_plain(A, x)


def _vla_coo(A, x, config):
    return spmv_coo_vla(A, x, config)


def _vla_csr(A, x, config):
    return spmv_csr_vla(A, x, config)


def _vla_dia(A, x, config):
    return spmv_dia_vla(A, x, config)


def default_registry() -> KernelRegistry:
    """Fresh registry holding both versions for all three formats (GPU)."""
    reg = KernelRegistry()
    reg.register(Format.COO, KernelVersion.PLAIN, _plain_coo)
    reg.register(Format.CSR, KernelVersion.PLAIN, _plain_csr)
    reg.register(Format.DIA, KernelVersion.PLAIN, _plain_dia)
    reg.register(Format.COO, KernelVersion.VLA, _vla_coo)
    reg.register(Format.CSR, KernelVersion.VLA, _vla_csr)
    reg.register(Format.DIA, KernelVersion.VLA, _vla_dia)
    return reg


_DEFAULT_REGISTRY = default_registry()


def dispatch(matrix, x, version=KernelVersion.PLAIN, config: LaneConfig | None = None,
             registry: KernelRegistry | None = None):
    """Run ``y = A @ x`` with the kernel registered for the matrix's format
    (kernels.py:286-297).  Accepts a container or a DynamicMatrix."""
    m = as_container(matrix)
    reg = registry if registry is not None else _DEFAULT_REGISTRY
    fn = reg.lookup(m.format, KernelVersion(version))
    return fn(m, x, config)
