"""Device conjugate gradients — the reference's HPCG vehicle (hpcg.py:211-258).

Same algorithm, stopping rule, residual history and errors as
`hpcg.cg_solve`: unpreconditioned CG from x = 0, `residual_norms` holds
||r||/||b|| after every iteration, `Diverged` on non-positive or non-finite
curvature / residual.  Every product is an SpMV kernel of this package (via
`dispatch` and its registry, so the `version` / `config` / `registry`
arguments mean what they mean in the reference); the vector work runs in
csrc/blas1.cu.

Operators (all vectors are lists of per-rank parts, like the reference):
* a device container (one GPU);
* `EmulatedRanks`: several slabs in one process, exchanged in process —
  the reference's simulated ranks on one GPU;
* a `DistributedMatrix` (one rank per GPU, NCCL halo exchange); dots are
  reduced in rank order like hpcg._global_dot (hpcg.py:192-197).
Host syncs: two scalars per iteration (p.Ap and r.r), as in the reference.
"""

from __future__ import annotations

import ctypes
import math
from dataclasses import dataclass, field

import torch

from . import _lib
from .dist import DistributedMatrix, LocalSlab, exchange_in_process
from .errors import Diverged
from .kernels import KernelVersion, dispatch
from .lanes import LaneConfig


@dataclass
class CgState:
    """Solver outcome (hpcg.py:200-208)."""

    x_parts: list
    iterations: int
    residual_norms: list
    converged: bool
    relative_residual: float


@dataclass
class EmulatedRanks:
    """Slabs of all ranks in one process (one GPU), exchanged in process."""

    slabs: list
    plans: list = field(default_factory=list)


def _stream(t: torch.Tensor) -> int:
    return torch.cuda.current_stream(t.device).cuda_stream


class _Ops:
    """Per-rank vector parts and the three operations CG needs."""

    def __init__(self, op, version, config, registry):
        self.op, self.version, self.config, self.registry = op, version, config, registry
        if isinstance(op, DistributedMatrix):
            self.kind, self.sizes = "dist", [op.slab.nloc]
            self.dev = op.slab.xw.device
            self.dtype = op.slab.xw.dtype
        elif isinstance(op, EmulatedRanks):
            self.kind, self.sizes = "emul", [s.nloc for s in op.slabs]
            self.dev = op.slabs[0].xw.device
            self.dtype = op.slabs[0].xw.dtype
        else:
            self.kind, self.sizes = "single", [op.nrows]
            self.dev = op.values.device
            self.dtype = op.values.dtype
        self.code = _lib.dtype_code(self.dtype)
        n_ws = int(_lib.load().spmv_dot_workspace_entries())
        self.ws = torch.empty(n_ws, dtype=self.dtype, device=self.dev)

    def spmv(self, p_parts):
        if self.kind == "single":
            return [dispatch(self.op, p_parts[0], self.version, self.config, self.registry)]
        if self.kind == "dist":
            return [self.op.spmv(p_parts[0])]
        slabs = self.op.slabs
        for s, p in zip(slabs, p_parts):
            s.x_local.copy_(p)
        exchange_in_process(self.op.plans, [s.xw for s in slabs])
        out = []
        for s in slabs:
            y = torch.empty(s.nloc, dtype=self.dtype, device=self.dev)
            for part in s.parts:
                s.run_part(part, y)
            out.append(y)
        return out

    def _result(self) -> float:
        return float(self.ws[-1].item())

    def _reduce(self, local: list) -> float:
        """Rank-order sum of per-rank partial dots (hpcg.py:192-197)."""
        if self.kind == "dist":
            import torch.distributed as dist
            world = dist.get_world_size(self.op.group)
            mine = torch.tensor([local[0]], dtype=torch.float64, device=self.dev)
            allp = torch.empty(world, dtype=torch.float64, device=self.dev)
            dist.all_gather_into_tensor(allp, mine, group=self.op.group)
            local = allp.cpu().tolist()
        acc = 0.0
        for v in local:
            acc += float(v)
        return acc

    def dot(self, a_parts, b_parts) -> float:
        vals = []
        for a, b in zip(a_parts, b_parts):
            _lib.call("spmv_dot", self.code, a.shape[0], a.data_ptr(), b.data_ptr(), self.ws.data_ptr(), _stream(a))
            vals.append(self._result())
        return self._reduce(vals)

    def update(self, alpha, p_parts, ap_parts, x_parts, r_parts) -> float:
        vals = []
        for p, ap, x, r in zip(p_parts, ap_parts, x_parts, r_parts):
            _lib.call("spmv_cg_update", self.code, p.shape[0], float(alpha), p.data_ptr(), ap.data_ptr(),
                      x.data_ptr(), r.data_ptr(), self.ws.data_ptr(), _stream(p))
            vals.append(self._result())
        return self._reduce(vals)

    def direction(self, beta, r_parts, p_parts) -> None:
        for r, p in zip(r_parts, p_parts):
            _lib.call("spmv_cg_direction", self.code, r.shape[0], float(beta), r.data_ptr(), p.data_ptr(), _stream(r))


def _parts(v, sizes):
    if isinstance(v, (list, tuple)):
        return [t.contiguous() for t in v]
    if len(sizes) == 1:
        return [v.contiguous()]
    return list(torch.split(v, sizes))


def cg_solve(op, b, version=KernelVersion.PLAIN, tol: float = 1e-9, max_iters: int = 500,
             config: LaneConfig | None = None, registry=None) -> CgState:
    """Unpreconditioned CG from x = 0 on the device (hpcg.py:211-258).

    `b`: a CUDA tensor (or one part per rank).  Returns the solution parts,
    the iteration count and the relative-residual history."""
    ops = _Ops(op, version, config, registry)
    b_parts = [t.to(device=ops.dev, dtype=ops.dtype) for t in _parts(b, ops.sizes)]
    bnorm = math.sqrt(ops.dot(b_parts, b_parts))
    x = [torch.zeros_like(t) for t in b_parts]
    if bnorm == 0.0:
        return CgState(x, 0, [], True, 0.0)
    r = [t.clone() for t in b_parts]
    p = [t.clone() for t in r]
    rr = ops.dot(r, r)
    norms: list = []
    converged = False
    rel = math.sqrt(rr) / bnorm
    it = 0
    if rel <= tol:
        return CgState(x, 0, [], True, rel)
    for it in range(1, max_iters + 1):
        ap = ops.spmv(p)
        pap = ops.dot(p, ap)
        if not math.isfinite(pap) or pap <= 0.0:
            raise Diverged(f"curvature p'Ap = {pap} at iteration {it}")
        alpha = rr / pap
        rr_new = ops.update(alpha, p, ap, x, r)
        if not math.isfinite(rr_new):
            raise Diverged(f"residual norm became non-finite at iteration {it}")
        rel = math.sqrt(rr_new) / bnorm
        norms.append(rel)
        if rel <= tol:
            converged = True
            break
        beta = rr_new / rr
        ops.direction(beta, r, p)
        rr = rr_new
    return CgState(x, it, norms, converged, rel)


def emulated_ranks(slabs) -> EmulatedRanks:
    """EmulatedRanks with halo plans agreed from the slabs' windows."""
    from .dist import RowPartition, build_halo_plan
    bounds = [s.rows[0] for s in slabs] + [slabs[-1].rows[1]]
    part = RowPartition(bounds[-1], tuple(bounds))
    plans = [build_halo_plan(part, [s.window for s in slabs], r) for r in range(len(slabs))]
    return EmulatedRanks(list(slabs), plans)


__all__ = ["CgState", "EmulatedRanks", "cg_solve", "emulated_ranks", "LocalSlab"]
