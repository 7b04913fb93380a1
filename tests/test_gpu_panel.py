"""The CSR column-panel path (csrc/panel.cuh) against the C oracle.

Long rows (over 32 entries) of random-column matrices are copied
panel-major by the plan and reduced per (row, panel) segment with a warp
segmented scan; rows of <= 32 entries go through the tile kernel of a
short-row sub plan.  Contract (north_star, kernels.py:69-82): rows of <= 32
entries bit-exact, every row within 1e-12 (f64) / 1e-5 of the f64-evaluated
product (f32).  Cases push every boundary of the segmented reduction:
segments spanning lanes, 256-entry steps, warp slices and CTA ranges;
one-entry segments; 50k-entry rows; many panels; empty rows; a row spanning
all panels; f32; an x window (col_base > 0).
"""

import zlib

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

PANEL = 23552  # csrc/panel.cuh kPanelCols


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def _matrix(rng, n, ncols, lens):
    irp = np.zeros(n + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(k), replace=False)) if k else np.zeros(0, np.int64)
                           for k in lens]).astype(np.uint32)
    vals = rng.uniform(-1, 1, cols.shape[0])
    return irp.astype(np.uint32), cols, vals


CASES = {
    # name: (nrows, ncols, lengths)
    "zipf_like": (30_000, 400_000, lambda r, n: np.minimum(r.zipf(1.8, n), 20_000)),
    "all_long": (3_000, 200_000, lambda r, n: r.integers(33, 600, n)),
    "huge_rows": (2_000, 300_000, lambda r, n: np.where(np.arange(n) % 500 == 7, 50_000, r.integers(0, 40, n))),
    "one_panel": (20_000, 20_000, lambda r, n: r.integers(0, 120, n)),
    "empty_gaps": (60_000, 100_000, lambda r, n: np.where((np.arange(n) // 777) % 2 == 0, 0, r.integers(0, 200, n))),
    "few_long": (50_000, 90_000, lambda r, n: np.where(r.random(n) < 0.001, 5000, r.integers(0, 33, n))),
}


def _check(y, ref, lens, tol):
    from _util import bit_equal, first_diff, rel_err
    short = lens <= 32
    assert bit_equal(y[short], ref[short]), first_diff(y[short], ref[short])
    assert rel_err(y, ref) <= tol, rel_err(y, ref)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_panel_path_matches_oracle(sp, name, dtype):
    from oracle import c_oracle
    from paper_2304_09511_b200 import kernels as K
    n, ncols, sampler = CASES[name]
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    lens = np.minimum(sampler(rng, n).astype(np.int64), ncols)
    irp, cols, vals = _matrix(rng, n, ncols, lens)
    vals = vals.astype(dtype)
    x = rng.uniform(-1, 1, ncols).astype(dtype)
    A = sp.CsrMatrix.from_arrays(n, ncols, irp, cols, vals)
    cfg = sp.PlanConfig(panels=1)
    p = K.csr_plan(A, config=cfg)
    assert p.info()["kernel"] == "panel" and p.config().panels == 1
    y = sp.spmv_csr_plain(A, x, plan_config=cfg)
    if dtype == np.float64:
        _check(y, c_oracle.csr_plain(n, irp, cols, vals, x), lens, 1e-12)
    else:
        ref64 = c_oracle.csr_plain(n, irp, cols, vals.astype(np.float64), x.astype(np.float64))
        _check(y, c_oracle.csr_plain(n, irp, cols, vals, x), lens, 1.0)  # short rows: the f32 reference order
        from _util import rel_err
        assert rel_err(y, ref64) <= 1e-5
    # deterministic, and the same as the warp-stream path within 1e-12
    assert sp.spmv_csr_plain(A, x, plan_config=cfg).tobytes() == y.tobytes()
    yw = sp.spmv_csr_plain(A, x, plan_config=sp.PlanConfig(panels=0, warp_stream=1))
    from _util import rel_err
    assert rel_err(y, yw) <= (1e-12 if dtype == np.float64 else 1e-5)


def test_panel_auto_choice_and_x_window(sp):
    """Auto picks the panel path for a Zipf-like wide matrix; a product
    through the C ABI with an x window (col_base > 0) is correct; other
    arrays than the plan's (a copy of the values) take the warp-stream
    kernel and agree."""
    import torch

    from oracle import c_oracle
    from paper_2304_09511_b200 import _lib
    from paper_2304_09511_b200 import kernels as K
    rng = np.random.default_rng(17)
    n, ncols = 40_000, 300_000
    lens = np.minimum(rng.zipf(1.6, n), 30_000)
    irp, cols, vals = _matrix(rng, n, ncols, lens)
    cols = (cols.astype(np.int64) // 2 + 150_000).astype(np.uint32)  # columns in [150000, 300000)
    cols_sorted = np.concatenate([np.sort(cols[irp[i]:irp[i + 1]]) for i in range(n)]).astype(np.uint32)
    A = sp.CsrMatrix.from_arrays(n, ncols, irp, cols_sorted, vals)
    assert K.csr_plan(A).info()["kernel"] == "panel"
    x = rng.uniform(-1, 1, ncols)
    ref = c_oracle.csr_plain(n, irp, cols_sorted, vals, x)
    _check(sp.spmv_csr_plain(A, x), ref, lens, 1e-12)
    cb = 150_000
    xw = torch.from_numpy(x[cb:]).cuda()
    y = torch.empty(n, dtype=torch.float64, device="cuda")
    p = K.csr_plan(A)
    _lib.call("spmv_csr", p.handle, A.row_pointers.data_ptr(), A.col_indices.data_ptr(), A.values.data_ptr(),
              xw.data_ptr(), cb, ncols - cb, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _check(y.cpu().numpy(), ref, lens, 1e-12)
    other = A.values.clone()
    _lib.call("spmv_csr", p.handle, A.row_pointers.data_ptr(), A.col_indices.data_ptr(), other.data_ptr(),
              xw.data_ptr(), cb, ncols - cb, y.data_ptr(), torch.cuda.current_stream().cuda_stream)
    _check(y.cpu().numpy(), ref, lens, 1e-12)


def test_panel_vla_and_host_paths_unaffected(sp):
    """vla and the host pipeline (tile ranges) of a panel plan keep their
    own kernels and contracts."""
    import torch

    from oracle import c_oracle
    rng = np.random.default_rng(3)
    n, ncols = 20_000, 200_000
    lens = np.minimum(rng.zipf(1.8, n), 5000)
    irp, cols, vals = _matrix(rng, n, ncols, lens)
    A = sp.CsrMatrix.from_arrays(n, ncols, irp, cols, vals)
    sp.set_plan_config(A, sp.PlanConfig(panels=1))
    x = rng.uniform(-1, 1, ncols)
    assert sp.spmv_csr_vla(A, x, sp.LaneConfig(8)).tobytes() == c_oracle.csr_vla(n, irp, cols, vals, x, 8).tobytes()
    xh = torch.from_numpy(x).pin_memory()
    yh = torch.empty(n, dtype=torch.float64).pin_memory()
    sp.spmv_csr_plain(A, xh, out=yh)
    _check(yh.numpy(), c_oracle.csr_plain(n, irp, cols, vals, x), lens, 1e-12)


@pytest.mark.parametrize("shuffle", [False, True])
def test_coo_panel_view(sp, shuffle):
    """COO plans with long runs take the panel path through a CSR view of
    the row-sorted triples: short rows bit-exact with np.add.at order (from
    +0.0, so a lone -0.0 product gives +0.0), long rows within 1e-12; an
    unsorted input (stable row sort, storage order kept) too."""
    from oracle import c_oracle
    from paper_2304_09511_b200 import kernels as K
    rng = np.random.default_rng(23)
    n, ncols = 30_000, 300_000
    lens = np.minimum(rng.zipf(1.7, n), 8000)
    irp, cols, vals = _matrix(rng, n, ncols, lens)
    vals[irp[5]] = -0.0  # row 5's first product is -0.0
    x = rng.uniform(-1, 1, ncols)
    rows = np.repeat(np.arange(n), lens).astype(np.uint32)
    if shuffle:
        order = rng.permutation(rows.shape[0])
        rows, cols, vals = rows[order], cols[order], vals[order]
    A = sp.CooMatrix.from_arrays(n, ncols, rows, cols, vals, sorted=not shuffle)
    p = K.coo_plan(A)
    assert p.info()["kernel"] == "panel" and p.config().panels == 1
    y = sp.spmv_coo_plain(A, x)
    ref = c_oracle.coo_plain(n, rows, cols, vals, x, row_sorted=not shuffle)
    _check(y, ref, lens, 1e-12)
    yw = sp.spmv_coo_plain(A, x, plan_config=sp.PlanConfig(panels=0))
    assert K.coo_plan(A, config=sp.PlanConfig(panels=0)).info()["kernel"] == "warp_stream"
    from _util import rel_err
    assert rel_err(y, yw) <= 1e-12
