"""Per-rank step time of the row-partitioned 256^3 stencil, measured one rank
at a time on one GPU (this pool has one B200 per call).

For an N-way z-slab partition (RowPartition.contiguous, hpcg.py:109 with
procs (1,1,N)), builds rank r's slab exactly as DistributedMatrix does
(window, interior / boundary parts) and times its launches back to back
with CUDA events, in DistributedMatrix.spmv's order (CSR and DIA:
interior, then both boundary blocks in one gapped launch; COO: lower,
interior, upper).  The halo exchange is not run: on the real
path it overlaps the interior rows (512 KiB per neighbour per step over
NVLink), so the per-rank time is interior + boundary launches.  The
projection max over ranks, divided into the one-GPU time, is the scaling
the row partition allows; it is not a multi-GPU measurement.

  python tools/slab_projection.py [--fmt csr|dia|coo] [--worlds 2 4 8]
"""
import argparse
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2304_09511_b200 as sp  # noqa: E402
from paper_2304_09511_b200 import synthetic  # noqa: E402
from paper_2304_09511_b200.dist import RowPartition, build_local_slab  # noqa: E402


def time_fn(fn, steps=50, warmup=5):
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(steps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / 1e3 / steps


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--fmt", default="csr")
    ap.add_argument("--grid", type=int, default=256)
    ap.add_argument("--worlds", type=int, nargs="*", default=[2, 4, 8])
    args = ap.parse_args()
    g = args.grid
    n = g ** 3
    x = synthetic.probe_x(n, synthetic.X_SEED)
    res = {"fmt": args.fmt, "grid": g}
    def rank_time(world, rank):
        part = RowPartition.contiguous(n, world, unit=g * g)
        r0, r1 = part.rows(rank)
        rows = sp.gen_stencil27_rows(g, g, g, r0, r1)
        slab = build_local_slab(rows, r0, r1, args.fmt)
        slab.xw.copy_(torch.from_numpy(x[slab.window[0]:slab.window[1]]))
        y = torch.empty(slab.nloc, dtype=torch.float64, device="cuda")

        lower, interior, upper = slab.parts
        seq = [slab.interior_g, slab.boundary] if slab.boundary is not None else [lower, interior, upper]

        def step():  # as DistributedMatrix.spmv orders the launches
            for p in seq:
                slab.run_part(p, y)

        t = time_fn(step)
        if world == max(args.worlds) and rank == 1:
            res["parts_ms_rank1"] = [round(time_fn(lambda p=p: slab.run_part(p, y)) * 1e3, 4) for p in seq]
        del slab, rows, y
        torch.cuda.empty_cache()
        return t

    for world in [1] + args.worlds:
        # ranks 1 .. world-2 hold identical interior slabs: time one of them
        first, last = rank_time(world, 0), (rank_time(world, world - 1) if world > 1 else None)
        mid = rank_time(world, 1) if world > 2 else None
        times = [first] + ([mid] * (world - 2) if mid is not None else []) + ([last] if last is not None else [])
        res[f"n{world}"] = {"ms_per_step_max_rank": round(max(times) * 1e3, 4),
                            "per_rank_ms": [round(v * 1e3, 4) for v in times]}
    t1 = res["n1"]["ms_per_step_max_rank"]
    for world in args.worlds:
        r = res[f"n{world}"]
        r["projected_speedup"] = round(t1 / r["ms_per_step_max_rank"], 2)
    print(json.dumps(res))


if __name__ == "__main__":
    main()
