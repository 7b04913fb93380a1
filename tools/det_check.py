import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_2304_09511_b200 as sp
from paper_2304_09511_b200 import synthetic
irp, cols, vals = synthetic.zipf_csr(2_000_000, 2_000_000, synthetic.ZIPF_SEED)
x = torch.from_numpy(synthetic.probe_x(2_000_000, synthetic.X_SEED)).cuda()
A = sp.CsrMatrix.from_arrays(2_000_000, 2_000_000, irp, cols, vals)
ys = [sp.spmv_csr_plain(A, x).cpu().numpy() for _ in range(6)]
print("csr same:", [np.array_equal(ys[0].view(np.uint64), y.view(np.uint64)) for y in ys[1:]])
d = np.nonzero(ys[0].view(np.uint64) != ys[1].view(np.uint64))[0]
print("ndiff", d.size, d[:10], np.diff(irp.astype(np.int64))[d[:10]] if d.size else None)
C = sp.csr_to_coo(A)
zs = [sp.spmv_coo_plain(C, x).cpu().numpy() for _ in range(6)]
print("coo same:", [np.array_equal(zs[0].view(np.uint64), z.view(np.uint64)) for z in zs[1:]])
