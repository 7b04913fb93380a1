"""Small products on every kernel family, for compute-sanitizer runs
(memcheck / racecheck / synccheck, one tool per gpurun call).

Each case is checked against the C oracle so a run that exits 0 also shows
the results were right under the tool.  Families: CSR tile kernel (1 and G
consumer groups, TMA rings), warp-stream CSR/COO, the column-panel path
(CSR, COO view), COO tile kernels, DIA bulk kernel presets, vla (tile path,
sub-warp, two-phase long rows), conversions and sort_coo, host-buffer
pipelines (pinned and pageable x), two streams on one plan.
"""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402
from oracle import c_oracle  # noqa: E402

rng = np.random.default_rng(0)
P = sp.PlanConfig


def check(y, ref, exact_rows=None, tol=1e-12):
    y = np.asarray(y)
    err = np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)) if y.size else 0.0
    assert err <= tol, err
    if exact_rows is not None:
        assert y[exact_rows].tobytes() == ref[exact_rows].tobytes()


def random_csr(n, ncols, lens):
    irp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(k), replace=False)) for k in lens]).astype(np.uint32)
    vals = rng.uniform(-1, 1, cols.shape[0])
    return irp.astype(np.uint32), cols, vals


# stencil: tile kernels, DIA presets, COO multi-group
A = sp.gen_stencil27(10, 9, 8)
irp, cols, vals = c_oracle.stencil27_rows(10, 9, 8, 0, A.nrows)
x = rng.uniform(-1, 1, A.ncols)
ref = c_oracle.csr_plain(A.nrows, irp, cols, vals, x)
for cfg in (P(), P(tile=1024, groups=1), P(warp_stream=1), P(tile=2048, groups=3)):
    check(sp.spmv_csr_plain(A, x, plan_config=cfg), ref, np.ones(A.nrows, bool), 0.0)
coo = sp.csr_to_coo(A)
for cfg in (P(), P(groups=1), P(warp_stream=1)):
    check(sp.spmv_coo_plain(coo, x, plan_config=cfg), ref, None, 0.0)
dia = sp.coo_to_dia(coo)
for k in range(-1, 5):
    check(sp.spmv_dia_plain(dia, x, plan_config=P(dia_kernel=k)), ref, None, 0.0)
check(sp.spmv_csr_vla(A, x, sp.LaneConfig(8)), c_oracle.csr_vla(A.nrows, irp, cols, vals, x, 8), None, 0.0)
# long rows: warp-stream, panel (CSR + COO view), tile long-row units, vla two-phase
n, nc = 3000, 70000
lens = np.where(rng.random(n) < 0.05, rng.integers(33, 2000, n), rng.integers(0, 33, n))
lirp, lcols, lvals = random_csr(n, nc, lens)
L = sp.CsrMatrix.from_arrays(n, nc, lirp, lcols, lvals)
lx = rng.uniform(-1, 1, nc)
lref = c_oracle.csr_plain(n, lirp, lcols, lvals, lx)
short = lens <= 32
for cfg in (P(panels=0, warp_stream=1, ranges_per_warp=64), P(panels=1), P(panels=0, warp_stream=0)):
    check(sp.spmv_csr_plain(L, lx, plan_config=cfg), lref, short)
lcoo = sp.csr_to_coo(L)
for cfg in (P(panels=0, warp_stream=1), P(panels=1), P(panels=0, warp_stream=0)):
    check(sp.spmv_coo_plain(lcoo, lx, plan_config=cfg), lref, short)
check(sp.spmv_csr_vla(L, lx, sp.LaneConfig(4)), c_oracle.csr_vla(n, lirp, lcols, lvals, lx, 4), None, 0.0)
# conversions and sort_coo (shuffled, with duplicates)
perm = torch.randperm(coo.nnz, device="cuda")
sh = sp.CooMatrix(coo.shape, coo.row_indices[perm], coo.col_indices[perm], coo.values[perm], sorted=False)
back = sp.coo_to_csr(sp.sort_coo(sh)).to_host()
assert np.array_equal(back["row_pointers"], irp) and np.array_equal(back["col_indices"], cols)
dup = sp.CooMatrix.from_arrays(4, 4, [0, 1, 0, 3, 1], [1, 2, 1, 0, 2], [1.0, 2.0, 3.0, 4.0, -2.0], sorted=False)
h = sp.sort_coo(dup).to_host()
assert h["values"].tolist() == [4.0, 0.0, 4.0]
# host pipelines and two streams on one plan
check(sp.spmv_csr_plain(A, x), ref, None, 0.0)
check(sp.spmv_dia_plain(dia, torch.from_numpy(x).pin_memory()).numpy(), ref, None, 0.0)
check(sp.spmv_coo_plain(coo, x), ref, None, 0.0)
xd = torch.from_numpy(lx).cuda()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
outs = []
torch.cuda.synchronize()
for s in (s1, s2, s1, s2):
    with torch.cuda.stream(s):
        outs.append(sp.spmv_csr_plain(L, xd, plan_config=P(panels=0, warp_stream=1)))
torch.cuda.synchronize()
for o in outs:
    check(o.cpu().numpy(), lref, short)
import ctypes  # noqa: E402
import os  # noqa: E402

from paper_2304_09511_b200 import _lib  # noqa: E402

if os.environ.get("SPMV_DEBUG_CHECKS") == "1":
    c = (ctypes.c_ulonglong * 4)()
    _lib.call("spmv_debug_check_counts", c)
    counts = list(c)
    print("debug check counters (stage mismatch, index range, x panel, other):", counts)
    assert counts == [0, 0, 0, 0], counts
print("sanitize cases ok")
