"""Worker for the gloo (CPU) multi-process tests of the row-partitioned path.

Each rank owns a z-slab of a small 27-point stencil, derives its x window
from its rows' column bounds, agrees on the halo plan with the other ranks
(all_gather_object), runs the real `halo_exchange` over gloo, and checks
(a) the window holds exactly the global x entries it should, and (b) the
oracle product of its rows over the window equals the global oracle product
row for row (bit-exact).  The SpMV here is the oracle (test-side checker);
the exchange and plan are the product code.
"""

import os

import numpy as np


def run(rank, world, port, dims, result_q):
    import torch
    import torch.distributed as dist

    from oracle import spmv_oracle as O
    from paper_2304_09511_b200.dist import RowPartition, build_halo_plan, halo_exchange

    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        nx, ny, nz = dims
        n = nx * ny * nz
        part = RowPartition.contiguous(n, world, unit=nx * ny)
        r0, r1 = part.rows(rank)
        irp, cols, vals = O.stencil27(nx, ny, nz, row_begin=r0, row_end=r1)
        lo = min(r0, int(cols.min())) if cols.size else r0
        hi = max(r1, int(cols.max()) + 1) if cols.size else r1
        windows = [None] * world
        dist.all_gather_object(windows, (lo, hi))
        plan = build_halo_plan(part, windows, rank)
        x = np.random.default_rng(11).uniform(-1, 1, n)
        window = torch.zeros(hi - lo, dtype=torch.float64)
        window[r0 - lo:r1 - lo] = torch.from_numpy(x[r0:r1])
        for w in halo_exchange(plan, window):
            w.wait()
        ok_window = bool(np.array_equal(window.numpy(), x[lo:hi]))
        y_local = O.csr_plain(r1 - r0, irp, cols.astype(np.int64) - lo, vals, window.numpy())
        g_irp, g_cols, g_vals = O.stencil27(nx, ny, nz)
        y_ref = O.csr_plain(n, g_irp, g_cols, g_vals, x)[r0:r1]
        ok_y = y_local.tobytes() == y_ref.tobytes()
        result_q.put((rank, ok_window, ok_y, plan.recv, plan.send))
    finally:
        dist.destroy_process_group()
