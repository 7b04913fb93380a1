"""64^3 back-to-back products: eager launches vs one CUDA graph of 100 products
(the library calls are stream-ordered and allocation-free after the first
product, so they capture)."""
import sys
import time

import torch

sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp  # noqa: E402

A = sp.gen_stencil27(64, 64, 64)
mats = {"csr": A, "coo": sp.csr_to_coo(A), "dia": sp.coo_to_dia(sp.csr_to_coo(A))}
x = torch.rand(A.ncols, dtype=torch.float64, device="cuda")
fns = {"csr": sp.spmv_csr_plain, "coo": sp.spmv_coo_plain, "dia": sp.spmv_dia_plain}
for fmt, m in mats.items():
    y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
    fn = lambda: fns[fmt](m, x, out=y)  # noqa: E731
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    ref = y.clone()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(1000):
        fn()
    b.record()
    torch.cuda.synchronize()
    eager = a.elapsed_time(b) / 1000
    s = torch.cuda.Stream()
    s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s):
        for _ in range(3):
            fn()
    torch.cuda.current_stream().wait_stream(s)
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g):  # (torch's own capture stream: the plan's first product on it)
        for _ in range(100):
            fn()
    g.replay()
    torch.cuda.synchronize()
    a.record()
    for _ in range(10):
        g.replay()
    b.record()
    torch.cuda.synchronize()
    graph = a.elapsed_time(b) / 1000
    ok = torch.equal(y.view(torch.int64), ref.view(torch.int64))
    print(f"64^3 {fmt}: eager {eager * 1e3:.2f} us/product ({2 * m.nnz / eager / 1e6:.0f} GFLOP/s), "
          f"graph of 100 {graph * 1e3:.2f} us/product ({2 * m.nnz / graph / 1e6:.0f} GFLOP/s), bit-equal {ok}")
