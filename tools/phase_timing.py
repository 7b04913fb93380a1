"""Per-phase cycle breakdown of the CSR tile kernel (needs the
-DSPMV_PHASE_TIMING build in SPMV_B200_LIB)."""
import ctypes
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402
from paper_2304_09511_b200 import _lib  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c5"
if cfg == "c5":
    A = sp.gen_stencil27(256, 256, 256)
else:
    from paper_2304_09511_b200 import synthetic
    irp, cols, vals = synthetic.zipf_csr(2_000_000, 2_000_000, 42)
    A = sp.CsrMatrix.from_arrays(2_000_000, 2_000_000, irp, cols, vals)
x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
y = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
buf = (ctypes.c_ulonglong * 8)()
for _ in range(3):
    sp.spmv_csr_plain(A, x, out=y)
torch.cuda.synchronize()
_lib.call("spmv_debug_csr_phases", buf)
for _ in range(10):
    sp.spmv_csr_plain(A, x, out=y)
_lib.call("spmv_debug_csr_phases", buf)
v = list(buf)
tiles = max(v[6], 1)
names = ["tma wait", "rows+barrier (thread 0)", "long+end barrier", "issue"]
print(cfg, "tiles", tiles, {n: round(v[i] / tiles) for i, n in enumerate(names)},
      "row-thread loop avg cycles", round(v[4] / max(v[5], 1)), "row threads/tile", round(v[5] / tiles, 1))
