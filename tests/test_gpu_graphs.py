"""CUDA graph capture of products (kernels are pure; the C ABI is
stream-ordered and allocation-free after a plan's first product on a stream,
and that first product may itself be captured: the per-stream launch scratch
is allocated under relaxed capture mode and its zero fill becomes a graph
node).  Replays must reproduce the eager y bit for bit."""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def _long_row_csr(sp):
    rng = np.random.default_rng(1)
    lens = np.array([3, 600, 0, 40, 7, 300, 1, 2000, 33, 12] * 40)
    irp = np.concatenate([[0], np.cumsum(lens)]).astype(np.uint32)
    cols = np.concatenate([np.sort(rng.choice(5000, n, replace=False)) for n in lens]).astype(np.uint32)
    vals = rng.uniform(-1.0, 1.0, int(irp[-1]))
    return sp.CsrMatrix.from_arrays(len(lens), 5000, irp, cols, vals)


@pytest.mark.parametrize("case", ["stencil", "long_rows"])
def test_graph_replay_matches_eager(sp, case):
    import torch
    if case == "stencil":
        csr = sp.gen_stencil27(12, 11, 10)
        coo = sp.csr_to_coo(csr)
        mats = [(sp.spmv_csr_plain, csr), (sp.spmv_coo_plain, coo), (sp.spmv_dia_plain, sp.coo_to_dia(coo))]
    else:
        csr = _long_row_csr(sp)
        mats = [(sp.spmv_csr_plain, csr), (sp.spmv_coo_plain, sp.csr_to_coo(csr))]
    x = torch.from_numpy(np.random.default_rng(2).uniform(-1.0, 1.0, csr.ncols)).cuda()
    for fn, m in mats:
        eager = fn(m, x).clone()
        y = torch.empty(m.nrows, dtype=torch.float64, device="cuda")
        # fresh containers: the captured product is each plan's first on the capture stream
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g):
            for _ in range(3):
                fn(m, x, out=y)
        for _ in range(2):
            y.fill_(7.0)
            g.replay()
            torch.cuda.synchronize()
            assert torch.equal(y.view(torch.int64), eager.view(torch.int64)), (case, m.format)
        # a different x through the same graph (the graph reads x's buffer)
        x2 = torch.from_numpy(np.random.default_rng(3).uniform(-1.0, 1.0, csr.ncols)).cuda()
        want = fn(m, x2).clone()
        x_keep = x.clone()
        x.copy_(x2)
        g.replay()
        torch.cuda.synchronize()
        assert torch.equal(y.view(torch.int64), want.view(torch.int64)), (case, m.format)
        x.copy_(x_keep)
