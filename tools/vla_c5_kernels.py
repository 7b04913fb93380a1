"""vla(8) CSR and COO products on the 256^3 stencil (for ncu captures)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_09511_b200 as sp
from paper_2304_09511_b200 import synthetic
A = sp.gen_stencil27(256, 256, 256)
C = sp.csr_to_coo(A)
x = torch.from_numpy(synthetic.probe_x(A.ncols, synthetic.X_SEED)).cuda()
for _ in range(3):
    sp.spmv_csr_vla(A, x, sp.LaneConfig(8))
    sp.spmv_coo_vla(C, x, sp.LaneConfig(8))
torch.cuda.synchronize()
