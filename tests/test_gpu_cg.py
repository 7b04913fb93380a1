"""Device CG vs the reference's hpcg.cg_solve (acceptance criterion 06,
test_acceptance.py:176-204; test_hpcg.py:108-158): same iteration counts,
residual histories within 1e-12, solution = ones within 1e-6, Diverged."""

import numpy as np
import pytest
import torch

from _util import bit_equal, load_golden

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def rhs(sp, A):
    return sp.spmv_csr_plain(A, torch.ones(A.ncols, dtype=torch.float64, device="cuda"))


@pytest.mark.parametrize("key", ["p16", "p8"])
@pytest.mark.parametrize("fmt", ["csr", "coo", "dia"])
def test_single_gpu_matches_reference(sp, key, fmt):
    from paper_2304_09511_b200.cg import cg_solve
    g = load_golden("cg")
    dims = [int(v) for v in g[f"{key}/dims"]]
    A = sp.gen_stencil27(*dims)
    b = rhs(sp, A)
    assert bit_equal(b.cpu().numpy(), g[f"{key}/b"])  # b = A @ ones, bit-exact (hpcg.py:122)
    op = sp.to_format(A, fmt)
    st = cg_solve(op, b, tol=1e-9, max_iters=200)
    assert st.converged and st.iterations == int(g[f"{key}/iterations"])
    assert np.max(np.abs(np.asarray(st.residual_norms) - g[f"{key}/norms"])) <= 1e-12
    x = st.x_parts[0].cpu().numpy()
    assert np.max(np.abs(x - 1.0)) <= 1e-6 and np.max(np.abs(x - g[f"{key}/x"])) <= 1e-9


def test_emulated_two_rank_split_replays(sp):
    from paper_2304_09511_b200.cg import cg_solve, emulated_ranks
    from paper_2304_09511_b200.dist import RowPartition, build_local_slab
    g = load_golden("cg")
    nx, ny, nz = (int(v) for v in g["p16_split/dims"])
    n = nx * ny * nz
    part = RowPartition.contiguous(n, 2, unit=nx * ny)
    slabs = [build_local_slab(sp.gen_stencil27_rows(nx, ny, nz, *part.rows(r)), *part.rows(r), "csr")
             for r in range(2)]
    b = rhs(sp, sp.gen_stencil27(nx, ny, nz))
    st = cg_solve(emulated_ranks(slabs), b, tol=1e-9, max_iters=200)
    assert st.converged and st.iterations == int(g["p16_split/iterations"]) == int(g["p16/iterations"])
    assert np.max(np.abs(np.asarray(st.residual_norms) - g["p16_split/norms"])) <= 1e-12
    x = torch.cat(st.x_parts).cpu().numpy()
    assert np.max(np.abs(x - 1.0)) <= 1e-6


def test_small_cube_zero_rhs_and_divergence(sp):
    from paper_2304_09511_b200.cg import cg_solve
    g = load_golden("cg")
    A = sp.gen_stencil27(2, 2, 2)
    b = rhs(sp, A)
    st = cg_solve(A, b, tol=1e-10, max_iters=20)
    assert st.converged and st.iterations <= 8 and st.relative_residual <= 1e-10
    assert st.iterations == int(g["p2/iterations"]) and len(st.residual_norms) == st.iterations
    z = cg_solve(A, torch.zeros_like(b))
    assert z.converged and z.iterations == 0 and z.residual_norms == []
    neg = sp.CsrMatrix(A.shape, A.row_pointers, A.col_indices, -A.values)
    with pytest.raises(sp.Diverged):
        cg_solve(neg, b)
    bad = b.clone()
    bad[0] = float("nan")
    with pytest.raises(sp.Diverged):
        cg_solve(A, bad)


def test_dot_is_deterministic(sp):
    import ctypes
    from paper_2304_09511_b200 import _lib
    n = 3_000_001
    a = torch.rand(n, dtype=torch.float64, device="cuda")
    b = torch.rand(n, dtype=torch.float64, device="cuda")
    ws = torch.empty(int(_lib.load().spmv_dot_workspace_entries()), dtype=torch.float64, device="cuda")
    vals = set()
    for _ in range(4):
        _lib.call("spmv_dot", 1, n, a.data_ptr(), b.data_ptr(), ws.data_ptr(),
                  torch.cuda.current_stream().cuda_stream)
        vals.add(float(ws[-1].item()))
    assert len(vals) == 1
    ref = float(np.dot(a.cpu().numpy(), b.cpu().numpy()))
    assert abs(vals.pop() - ref) <= 1e-12 * abs(ref)
