"""Host-side cost per public-API SpMV call on a tiny matrix (GPU time ~µs)."""
import os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import paper_2304_09511_b200 as sp
A = sp.gen_stencil27(16, 16, 16)
coo = sp.csr_to_coo(A)
dia = sp.coo_to_dia(coo)
x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
for name, m, f in (("csr", A, sp.spmv_csr_plain), ("coo", coo, sp.spmv_coo_plain), ("dia", dia, sp.spmv_dia_plain),
                   ("csr_vla", A, lambda m, x, out: sp.spmv_csr_vla(m, x, sp.LaneConfig(8), out=out))):
    y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
    for _ in range(20):
        f(m, x, out=y)
    torch.cuda.synchronize()
    n = 2000
    t0 = time.perf_counter()
    for _ in range(n):
        f(m, x, out=y)
    t1 = time.perf_counter()
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    print(f"{name:8s} host {1e6 * (t1 - t0) / n:7.1f} us/call, incl. drain {1e6 * (t2 - t0) / n:7.1f} us/call")
