"""e2e (pinned host x -> host y) timing vs pipeline chunk count, CPU vs GPU time."""
import os
import sys
import time

import torch

sys.path.insert(0, __import__("os").environ.get("AB_TREE", "."))
import paper_2304_09511_b200 as sp  # noqa: E402
from paper_2304_09511_b200 import kernels as K  # noqa: E402

A = sp.gen_stencil27(256, 256, 256)
xh = torch.rand(A.ncols, dtype=torch.float64).pin_memory()
yh = torch.empty(A.nrows, dtype=torch.float64).pin_memory()
for chunks in [int(c) for c in (__import__('sys').argv[1:] or (16, 32, 48, 64, 96, 128, 192))]:
    os.environ["X"] = "1"
    K.HOST_CHUNKS = chunks
    f = lambda: sp.spmv_csr_plain(A, xh, out=yh)  # noqa: E731
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20):
        f()
    t = (time.perf_counter() - t0) / 20
    print(f"chunks {chunks:3d}: {t * 1e3:.3f} ms/step  -> {2 * A.nnz / t / 1e9:.1f} GFLOP/s")
