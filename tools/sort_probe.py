"""One sort_coo of the shuffled 256^3 stencil COO (for an ncu launch list)."""
import sys

import torch

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402
from paper_2304_09511_b200 import convert as C  # noqa: E402

csr = sp.gen_stencil27(256, 256, 256)
coo = C.csr_to_coo(csr)
del csr
g = torch.Generator(device="cuda")
g.manual_seed(7)
perm = torch.randperm(coo.nnz, device="cuda", generator=g)
sh = sp.CooMatrix(coo.shape, coo.row_indices[perm], coo.col_indices[perm], coo.values[perm], sorted=False)
del perm, coo
for _ in range(2):
    out = C.sort_coo(sh)
    torch.cuda.synchronize()
    del out
print("ok")
