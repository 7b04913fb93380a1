"""One vla(8) CSR and COO product on the Zipf config (for an ncu launch list)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_09511_b200 as sp
from paper_2304_09511_b200 import synthetic
irp, cols, vals = synthetic.zipf_csr(2_000_000, 2_000_000, synthetic.ZIPF_SEED)
x = torch.from_numpy(synthetic.probe_x(2_000_000, synthetic.X_SEED)).cuda()
A = sp.CsrMatrix.from_arrays(2_000_000, 2_000_000, irp, cols, vals)
C = sp.csr_to_coo(A)
for _ in range(2):
    sp.spmv_csr_vla(A, x, sp.LaneConfig(8))
    sp.spmv_coo_vla(C, x, sp.LaneConfig(8))
torch.cuda.synchronize()
