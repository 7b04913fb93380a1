"""Host-side cost of one eager product call (device x, out=): cProfile over
20000 calls on a tiny operator, so the GPU is never the bound."""
import cProfile
import pstats
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402

A = sp.gen_stencil27(8, 8, 8)
coo = sp.csr_to_coo(A)
dia = sp.coo_to_dia(coo)
x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
y = torch.empty(A.nrows, dtype=torch.float64, device="cuda")
for name, fn, m in (("csr", sp.spmv_csr_plain, A), ("coo", sp.spmv_coo_plain, coo), ("dia", sp.spmv_dia_plain, dia)):
    for _ in range(100):
        fn(m, x, out=y)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(20000):
        fn(m, x, out=y)
    t = (time.perf_counter() - t0) / 20000
    torch.cuda.synchronize()
    print(f"{name}: {t * 1e6:.2f} us per call (host)")
pr = cProfile.Profile()
pr.enable()
for _ in range(20000):
    sp.spmv_csr_plain(A, x, out=y)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(18)
