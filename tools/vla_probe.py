"""Device time of the vla kernels (lanes 8) on the 256^3 stencil and Zipf."""
import sys

import torch

sys.path.insert(0, __import__("os").environ.get("AB_TREE", "."))
import paper_2304_09511_b200 as sp  # noqa: E402
from paper_2304_09511_b200 import synthetic  # noqa: E402


def timeit(fn, reps=30):
    fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(reps):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / reps / 1e3


which = sys.argv[1:] or ["c5", "c3"]
for cfg in which:
    if cfg == "c5":
        A = sp.gen_stencil27(256, 256, 256)
    else:
        irp, cols, vals = synthetic.zipf_csr(2_000_000, 2_000_000, synthetic.ZIPF_SEED)
        A = sp.CsrMatrix.from_arrays(2_000_000, 2_000_000, irp, cols, vals)
    C = sp.csr_to_coo(A)
    x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
    y = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
    cfg_l = sp.LaneConfig(8)
    for name, M, fn in (("csr_vla", A, sp.spmv_csr_vla), ("coo_vla", C, sp.spmv_coo_vla)):
        t = timeit(lambda: fn(M, x, cfg_l, out=y))
        print(f"{cfg} {name} {2 * A.nnz / t / 1e9:8.1f} GFLOP/s  {t * 1e3:.3f} ms")
