"""Timeline of spmv_csr_host (SPMV_HOST_TRACE=1 lines on stderr -> summary)."""
import os
import sys

os.environ.setdefault("SPMV_HOST_TRACE", "1")
import torch  # noqa: E402

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402
from paper_2304_09511_b200 import kernels as K  # noqa: E402

A = sp.gen_stencil27(256, 256, 256)
xh = torch.rand(A.ncols, dtype=torch.float64).pin_memory()
yh = torch.empty(A.nrows, dtype=torch.float64).pin_memory()
chunks = int(sys.argv[1]) if len(sys.argv) > 1 else 48
K.HOST_CHUNKS = chunks
for _ in range(4):
    sp.spmv_csr_plain(A, xh, out=yh)
torch.cuda.synchronize()
