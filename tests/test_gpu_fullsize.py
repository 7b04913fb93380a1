"""Parity at BASELINE.json's full sizes (configs 1-5), against the C oracle
(oracle/spmv_oracle.c, pinned to the reference) on the same seeded inputs,
plus size-independent properties (round trips, cross-format equality,
linearity).  Bounds per north_star: fp64 1e-12, fp32 1e-5 (vs the reference
evaluated in f64 on the f32 inputs); rows <= 32 bit-exact."""

import numpy as np
import pytest
import torch

from _util import bit_equal, rel_err
from oracle import c_oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def host_csr(m):
    h = m.to_host()
    return h["row_pointers"], h["col_indices"], h["values"]


def test_c1_c2_stencil_64_all_formats_and_conversions(sp):
    """Configs 1-2: 64^3 stencil, CSR/COO/DIA bit-exact with the reference
    order; CSR<->COO<->DIA conversions exact; 27 offsets per SURVEY.md F1."""
    from paper_2304_09511_b200.synthetic import probe_x
    A = sp.gen_stencil27(64, 64, 64)
    assert A.nnz == 6_859_000
    irp, cols, vals = host_csr(A)
    x = probe_x(A.ncols, 0)
    ref = c_oracle.csr_plain(A.nrows, irp, cols, vals, x)
    coo = sp.csr_to_coo(A)
    dia = sp.coo_to_dia(coo)
    offs = dia.offsets.cpu().tolist()
    expect = sorted({dz * 4096 + dy * 64 + dx for dz in (-1, 0, 1) for dy in (-1, 0, 1) for dx in (-1, 0, 1)})
    assert offs == expect  # ±{0,1,63,64,65,4031..4033,4095..4097,4159..4161}
    assert bit_equal(sp.spmv_csr_plain(A, x), ref)
    assert bit_equal(sp.spmv_dia_plain(dia, x), ref)
    y_coo = sp.spmv_coo_plain(coo, x)
    rows = np.repeat(np.arange(A.nrows), np.diff(irp.astype(np.int64)))
    assert bit_equal(y_coo, c_oracle.coo_plain(A.nrows, rows, cols, vals, x))
    back = sp.coo_to_csr(sp.dia_to_coo(dia))
    assert torch.equal(back.row_pointers, A.row_pointers) and torch.equal(back.col_indices, A.col_indices)
    assert torch.equal(back.values, A.values)


def test_c3_zipf_2m(sp):
    """Config 3: Zipf(1.8) 2M x 2M, CSR/COO, f64 and f32."""
    from paper_2304_09511_b200 import synthetic
    irp, cols, vals = synthetic.zipf_csr(2_000_000, 2_000_000, synthetic.ZIPF_SEED)
    n = 2_000_000
    lens = np.diff(irp.astype(np.int64))
    assert lens.min() >= 1 and lens.max() <= 50_000
    x = synthetic.probe_x(n, synthetic.X_SEED)
    ref64 = c_oracle.csr_plain(n, irp, cols, vals, x)
    A = sp.CsrMatrix.from_arrays(n, n, irp, cols, vals)
    y = sp.spmv_csr_plain(A, x)
    short = lens <= 32
    assert bit_equal(y[short], ref64[short]) and rel_err(y, ref64) <= 1e-12
    coo = sp.csr_to_coo(A)
    yc = sp.spmv_coo_plain(coo, x)
    rows = np.repeat(np.arange(n), lens)
    ref_coo = c_oracle.coo_plain(n, rows, cols, vals, x)
    assert bit_equal(yc[short], ref_coo[short]) and rel_err(yc, ref_coo) <= 1e-12
    v32, x32 = vals.astype(np.float32), x.astype(np.float32)
    A32 = sp.CsrMatrix.from_arrays(n, n, irp, cols, v32)
    y32 = sp.spmv_csr_plain(A32, x32)
    ref_f64_of_f32 = c_oracle.csr_plain(n, irp, cols, v32.astype(np.float64), x32.astype(np.float64))
    assert rel_err(y32, ref_f64_of_f32) <= 1e-5
    assert bit_equal(y32[short], c_oracle.csr_plain(n, irp, cols, v32, x32)[short])


def test_c4_banded_2p23(sp):
    """Config 4: banded 2^23 rows, 11 diagonals, N(0,1): DIA and CSR."""
    from paper_2304_09511_b200 import synthetic
    n = 1 << 23
    offs, vals, nnz = synthetic.banded_dia(n, synthetic.BANDED_OFFSETS, synthetic.BANDED_SEED)
    assert nnz == 92_263_418
    x = synthetic.probe_x(n, synthetic.X_SEED)
    ref = c_oracle.dia_plain(n, n, offs, vals, x)
    dia = sp.DiaMatrix(sp.MatrixShape(n, n, nnz), offs, vals)
    assert bit_equal(sp.spmv_dia_plain(dia, x), ref)
    csr = sp.to_format(dia, "csr")
    assert csr.nnz == nnz
    assert bit_equal(sp.spmv_csr_plain(csr, x), ref)  # rows of <= 11 entries: same order as DIA


def test_c5_stencil_256_properties(sp):
    """Config 5 (the bench workload): all formats bit-identical to each other
    and to the C oracle; linearity; exact round trip."""
    from paper_2304_09511_b200.synthetic import probe_x
    A = sp.gen_stencil27(256, 256, 256)
    assert A.nnz == 449_455_096
    x = torch.from_numpy(probe_x(A.ncols, 0)).cuda()
    y_csr = sp.spmv_csr_plain(A, x)
    coo = sp.csr_to_coo(A)
    assert coo.sorted
    assert torch.equal(sp.spmv_coo_plain(coo, x), y_csr)
    dia = sp.coo_to_dia(coo)
    del coo
    assert dia.ndiags == 27
    assert torch.equal(sp.spmv_dia_plain(dia, x), y_csr)
    del dia
    irp, cols, vals = host_csr(A)
    ref = c_oracle.csr_plain(A.nrows, irp, cols, vals, x.cpu().numpy())
    assert bit_equal(y_csr.cpu().numpy(), ref)
    x2 = torch.from_numpy(probe_x(A.ncols, 1)).cuda()
    lhs = sp.spmv_csr_plain(A, 0.5 * x - 2.0 * x2)
    rhs = 0.5 * y_csr - 2.0 * sp.spmv_csr_plain(A, x2)
    assert rel_err(lhs.cpu().numpy(), rhs.cpu().numpy()) <= 1e-12
