"""SpMV entry points, kernel registry and dispatch — the drop-in boundary.

Same names, argument meaning and error behaviour as the reference's
kernels.py (kernels.py:39-297), with every product computed by the sm_100a
kernels of libspmv_b200.so:

  spmv_csr_plain  kernels.py:69-82    CSR-stream + long-row warp chunks
  spmv_coo_plain  kernels.py:56-66    fixed-tile segmented reduction
  spmv_dia_plain  kernels.py:85-101   TMA-staged row tiles
  spmv_*_vla      kernels.py:104-210  sub-warp / CTA lane kernels

Host/device behaviour: a numpy (or list) `x` gets the reference contract —
x is cast to the value dtype on the host (kernels.py:51-52), copied to the
device, and a fresh numpy y is returned.  A CPU torch tensor (pinned for
asynchronous copies) gives a CPU tensor back.  A CUDA tensor `x` stays on
the device and a fresh CUDA tensor y is returned.  `out=` may be a CUDA
tensor (reused, no allocation) or a (pinned) CPU tensor that receives y.
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


def _stream(device: torch.device) -> int:
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
                getattr(_lib.load(), f"spmv_{self.kind}_plan_destroy")(self.handle)
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
        if ws.value:
            info.update(kernel="panel" if ws.value == 2 else "warp_stream", warps=nw.value)
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
# A product whose x and y both live in host memory is PCIe-bound (x in, y
# out).  CSR and DIA products are split into row ranges so the upload of x
# (column chunks, copy stream 1), the kernels (compute stream) and the
# download of finished rows of y (copy stream 2) overlap; PCIe is full
# duplex, so the step approaches max(H2D, D2H) instead of H2D + compute + D2H.
_SIDE_STREAMS: dict = {}
PIPELINE_CHUNKS = int(__import__("os").environ.get("SPMV_PIPELINE_CHUNKS", "32"))
HOST_CHUNKS = int(__import__("os").environ.get("SPMV_HOST_CHUNKS", "0"))  # 0: library default


def _side_streams(dev):
    key = str(dev)
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = (torch.cuda.Stream(dev), torch.cuda.Stream(dev))
    return _SIDE_STREAMS[key]


def _csr_tile_info(A: CsrMatrix, p: "_Plan"):
    def make():
        nt, tile = ctypes.c_int64(), ctypes.c_int64()
        _lib.call("spmv_csr_plan_tiles", p.handle, ctypes.byref(nt), ctypes.byref(tile))
        n = int(nt.value)
        row_lo = np.empty(n + 1, dtype=np.uint32)
        maxcol = np.empty(max(n, 1), dtype=np.uint32)
        _lib.call("spmv_csr_plan_tile_info", p.handle, _ptr(A.col_indices), row_lo.ctypes.data, maxcol.ctypes.data,
                  _stream(A.device))
        return n, row_lo.astype(np.int64), np.maximum.accumulate(maxcol[:n].astype(np.int64))
    return A.plan("csr_tiles", make)


def _upload_x_chunks(xh: torch.Tensor, xd: torch.Tensor, h2d, chunks: int):
    """Column chunks of x, in order on `h2d`; returns (bounds, events)."""
    n = xh.shape[0]
    bounds = [n * j // chunks for j in range(chunks + 1)]
    events = []
    with torch.cuda.stream(h2d):
        for j in range(chunks):
            a, b = bounds[j], bounds[j + 1]
            if b > a:
                xd[a:b].copy_(xh[a:b], non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(h2d)
            events.append(ev)
    return bounds, events


def _wait_x(cur, bounds, events, col_hi: int) -> None:
    """Make `cur` wait until x[0 .. col_hi] is on the device."""
    j = 0
    while j + 1 < len(bounds) - 1 and bounds[j + 1] <= col_hi:
        j += 1
    cur.wait_event(events[j])


def _pipelined(A, xh: torch.Tensor, yh: torch.Tensor, launch_range, ranges, chunks: int, y_final_at_end: bool):
    """Generic H2D / compute / D2H overlap.  `ranges`: list of
    (col_hi, rows_done) per compute step; `launch_range(k, xd, yd, stream)`."""
    dev = A.values.device
    cur = torch.cuda.current_stream(dev)
    h2d, d2h = _side_streams(dev)
    xd = torch.empty(A.ncols, dtype=A.values.dtype, device=dev)
    yd = torch.empty(A.nrows, dtype=A.values.dtype, device=dev)
    h2d.wait_stream(cur)
    d2h.wait_stream(cur)
    bounds, events = _upload_x_chunks(xh, xd, h2d, chunks)
    done = 0
    for k, (col_hi, rows_done) in enumerate(ranges):
        _wait_x(cur, bounds, events, col_hi)
        launch_range(k, xd, yd, cur)
        if not y_final_at_end and rows_done > done:
            ev = torch.cuda.Event()
            ev.record(cur)
            d2h.wait_event(ev)
            with torch.cuda.stream(d2h):
                yh[done:rows_done].copy_(yd[done:rows_done], non_blocking=True)
            done = rows_done
    if done < A.nrows:
        ev = torch.cuda.Event()
        ev.record(cur)
        d2h.wait_event(ev)
        with torch.cuda.stream(d2h):
            yh[done:].copy_(yd[done:], non_blocking=True)
    xd.record_stream(h2d)
    yd.record_stream(d2h)
    d2h.synchronize()
    return yh


def _csr_pipelined(A: CsrMatrix, xh, yh, chunks: int = PIPELINE_CHUNKS):
    p = csr_plan(A)
    nt, row_lo, maxcol_prefix = _csr_tile_info(A, p)
    tb = [nt * k // chunks for k in range(chunks + 1)]
    steps = [(k, tb[k], tb[k + 1]) for k in range(chunks) if tb[k + 1] > tb[k]]
    ranges = [(int(maxcol_prefix[te - 1]), int(row_lo[te]) if te < nt else A.nrows) for _, _, te in steps]
    spans = p.info()["launches"] > 1  # long rows spanning tiles: y final only after the fix-up

    def launch(k, xd, yd, stream):
        _, a, b = steps[k]
        _lib.call("spmv_csr_range", p.handle, _ptr(A.row_pointers), _ptr(A.col_indices), _ptr(A.values), _ptr(xd), 0,
                  A.ncols, _ptr(yd), a, b, 1 if k == len(steps) - 1 else 0, stream.cuda_stream)

    return _pipelined(A, xh, yh, launch, ranges, chunks, spans)


def _dia_pipelined(A: DiaMatrix, xh, yh, chunks: int = PIPELINE_CHUNKS):
    offs = A.plan("dia_offsets", lambda: A.offsets.cpu().numpy().astype(np.int64))
    max_off = int(offs.max()) if offs.size else 0
    rb = [(A.nrows * k // chunks) // 8 * 8 for k in range(chunks)] + [A.nrows]
    steps = [(rb[k], rb[k + 1]) for k in range(chunks) if rb[k + 1] > rb[k]]
    ranges = [(min(A.ncols - 1, b - 1 + max_off), b) for a, b in steps]
    esz = A.values.element_size()

    def launch(k, xd, yd, stream):
        a, b = steps[k]
        _lib.call("spmv_dia", _lib.dtype_code(A.values.dtype), b - a, A.ncols, A.ndiags, A.padded_rows - a,
                  _ptr(A.offsets), A.values.data_ptr() + a * A.ndiags * esz, _ptr(xd), a, 0, A.ncols,
                  yd.data_ptr() + a * esz, stream.cuda_stream)

    return _pipelined(A, xh, yh, launch, ranges, chunks, False)


def _host_pipeline_ok(A, x, out) -> bool:
    return (isinstance(x, torch.Tensor) and not x.is_cuda and out is not None and not out.is_cuda
            and x.dtype == A.values.dtype and x.dim() == 1 and x.shape[0] == A.ncols
            and out.shape == (A.nrows,) and out.dtype == A.values.dtype and A.nnz > 0 and A.nrows > 0
            and x.is_contiguous() and out.is_contiguous())


# ------------------------------------------------------------------ kernels --
def spmv_coo_plain(A, x, out=None, plan_config: PlanConfig | None = None):
    """``y = A @ x`` with np.add.at semantics (kernels.py:56-66).
    `plan_config` overrides the container's kernel configuration."""
    A = as_device(A)
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if A.nrows:
        p = coo_plan(A, plan_config)
        _lib.call("spmv_coo", p.handle, _ptr(A.row_indices), _ptr(A.col_indices), _ptr(A.values), _ptr(xv), 0,
                  A.ncols, _ptr(y), _stream(A.device))
    return _finish(y, origin, out)


def spmv_csr_plain(A, x, out=None, plan_config: PlanConfig | None = None):
    """``y = A @ x`` with one left-to-right sum per row (kernels.py:69-82).
    `plan_config` overrides the container's kernel configuration."""
    A = as_device(A)
    if _host_pipeline_ok(A, x, out):
        # host x -> host y: the C ABI pipelines upload / tiles / download
        p = csr_plan(A, config=plan_config)
        _lib.call("spmv_csr_host", p.handle, _ptr(A.row_pointers), _ptr(A.col_indices), _ptr(A.values),
                  x.data_ptr(), out.data_ptr(), HOST_CHUNKS, _stream(A.device))
        torch.cuda.current_stream(A.device).synchronize()
        return out
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if A.nrows:
        p = csr_plan(A, config=plan_config)
        _lib.call("spmv_csr", p.handle, _ptr(A.row_pointers), _ptr(A.col_indices), _ptr(A.values), _ptr(xv), 0,
                  A.ncols, _ptr(y), _stream(A.device))
    return _finish(y, origin, out)


def spmv_dia_plain(A, x, out=None, plan_config: PlanConfig | None = None):
    """``y = A @ x`` over stored diagonals (kernels.py:85-101).
    `plan_config` (its dia_* fields) overrides the container's."""
    A = as_device(A)
    if _host_pipeline_ok(A, x, out) and A.ndiags > 0:
        return _dia_pipelined(A, x, out)
    xv, origin = _checked_x(A, x)
    y = _new_y(A, out)
    if A.nrows:
        c = (plan_config if plan_config is not None else plan_config_of(A)).to_c()
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
