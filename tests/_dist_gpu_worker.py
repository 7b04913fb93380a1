"""Worker for the multi-process GPU tests of the row-partitioned path.

Every rank is one process running the product path — `DistributedMatrix`
(build, halo plan agreed over the group, `spmv` with the interior launch
overlapped or not, `gather_global`) — on cuda:0.  With backend "nccl" the
group has one rank (this box has one GPU, and NCCL refuses two ranks on one
device); with backend "gloo" several ranks share the GPU and the halo moves
through host memory (dist.halo_exchange stages device windows for gloo), so
no kernel ever waits on another rank's kernel.

The checker is the C oracle (oracle/spmv_oracle.c, test infrastructure):
the gathered y must equal the oracle's y of the whole matrix bit for bit
(rows of <= 32 entries) or within 1e-12 (longer rows).
"""

from __future__ import annotations

import os
import traceback

import numpy as np


def _case(name, sp, synthetic, c_oracle):
    """Global matrix of a test case: (host CSR arrays of A, n, dia or None,
    partition unit, reference y function of x per format)."""
    if name.startswith("stencil"):
        nx, ny, nz = {"stencil": (12, 10, 9), "stencil_wide": (20, 16, 12)}[name]
        n = nx * ny * nz
        irp, cols, vals = c_oracle.stencil27_rows(nx, ny, nz, 0, n)
        return dict(n=n, irp=irp, cols=cols, vals=vals, unit=nx * ny, rows_fn=lambda r0, r1: sp.gen_stencil27_rows(
            nx, ny, nz, r0, r1), dia=None)
    if name.startswith("banded"):
        # C4's 11 offsets (halo 4096) at 2^14 rows, or 33 diagonals: wider
        # than a 256-row DIA tile holds at f64 (the gapped launch falls back
        # to two launches)
        if name == "banded":
            n, offs = 1 << 14, synthetic.BANDED_OFFSETS
        else:
            n, offs = 3 * 2048, tuple(range(-16, 17))
        o, v, nnz = synthetic.banded_dia(n, offs, synthetic.BANDED_SEED)
        dia = sp.DiaMatrix(sp.MatrixShape(n, n, nnz), o, v)
        h = sp.to_format(dia, "csr").to_host()
        full = sp.CsrMatrix.from_arrays(n, n, h["row_pointers"], h["col_indices"], h["values"])
        from paper_2304_09511_b200.dist import _csr_rows
        return dict(n=n, irp=h["row_pointers"], cols=h["col_indices"], vals=h["values"], unit=8,
                    rows_fn=lambda r0, r1: _csr_rows(full, r0, r1), dia=(o, v))
    # random columns over all of x (all_gather), some rows over 32 entries
    rng = np.random.default_rng(9)
    n = 3000
    lens = rng.integers(0, 40, n)
    lens[::97] = 300
    irp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    cols = np.concatenate([np.sort(rng.choice(n, size=int(k), replace=False)) for k in lens]).astype(np.uint32)
    vals = rng.standard_normal(cols.shape[0])
    full = sp.CsrMatrix.from_arrays(n, n, irp, cols, vals)
    from paper_2304_09511_b200.dist import _csr_rows
    return dict(n=n, irp=irp.astype(np.uint32), cols=cols, vals=vals, unit=1,
                rows_fn=lambda r0, r1: _csr_rows(full, r0, r1), dia=None)


def run(rank, world, port, backend, case, fmts, result_q):
    try:
        import torch
        import torch.distributed as dist

        os.environ["MASTER_ADDR"] = "127.0.0.1"
        os.environ["MASTER_PORT"] = str(port)
        torch.cuda.set_device(0)
        if backend == "nccl":
            dist.init_process_group("nccl", rank=rank, world_size=world, device_id=torch.device("cuda", 0))
        else:
            dist.init_process_group("gloo", rank=rank, world_size=world)
        try:
            import paper_2304_09511_b200 as sp
            from oracle import c_oracle
            from paper_2304_09511_b200 import synthetic
            from paper_2304_09511_b200.dist import DistributedMatrix, RowPartition, gather_global

            c = _case(case, sp, synthetic, c_oracle)
            n = c["n"]
            x = np.random.default_rng(21).uniform(-1, 1, n)
            long_rows = np.diff(c["irp"].astype(np.int64)) > 32
            part = RowPartition.contiguous(n, world, unit=c["unit"])
            r0, r1 = part.rows(rank)
            out = {}
            for fmt in fmts:
                if fmt == "dia" and c["dia"] is not None:
                    o, v = c["dia"]
                    ref = c_oracle.dia_plain(n, n, o, v, x)
                else:
                    ref = c_oracle.csr_plain(n, c["irp"], c["cols"], c["vals"], x)
                for overlap in (True, False):
                    dm = DistributedMatrix.build(c["rows_fn"](r0, r1), part, rank, fmt, overlap=overlap)
                    xl = torch.from_numpy(x[r0:r1]).cuda()
                    y = dm.spmv(xl)
                    y2 = torch.full_like(y, float("nan"))
                    dm.spmv(out=y2)  # x already in the window; out= reused
                    g = gather_global(part, y).cpu().numpy()
                    same = g.view(np.uint64) == ref.view(np.uint64)
                    err = np.abs(g - ref) / np.maximum(np.abs(ref), 1.0)
                    out[(fmt, overlap)] = dict(
                        short_bit_exact=bool(same[~long_rows].all()),
                        max_rel_err=float(err.max()) if err.size else 0.0,
                        repeat_identical=bool(torch.equal(y, y2)),
                        launches=dm.launches_per_spmv(),
                        boundary=dm.slab.boundary is not None,
                        recv=dm.plan.recv_entries, allgather=dm.plan.allgather)
            result_q.put((rank, out, None))
        finally:
            dist.destroy_process_group()
    except Exception:
        result_q.put((rank, None, traceback.format_exc()))
