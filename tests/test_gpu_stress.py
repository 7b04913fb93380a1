"""Wider GPU parity: random structures the golden fixtures do not reach.

Checked against the pinned oracle (oracle/) with the exactness contract of
test_gpu_kernels.py: rows <= 32 bit-exact, everything within 1e-12 (f64) /
1e-5 of the f64-evaluated reference (f32).  Also: unaligned device pointers
(direct-load fallbacks), nnz not a multiple of 4 (tail tiles), huge rows,
runs of empty rows, rectangular shapes, wide DIA, conversions at scale.
"""

import zlib

import numpy as np
import pytest
import torch

from _util import bit_equal, first_diff, rel_err
from oracle import c_oracle
from oracle import spmv_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def random_csr(rng, nrows, ncols, lens):
    irp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    cols = np.concatenate([np.sort(rng.choice(ncols, size=int(k), replace=False)) if k else np.zeros(0, np.int64)
                           for k in lens]) if nrows else np.zeros(0, np.int64)
    vals = rng.standard_normal(cols.shape[0])
    return irp.astype(np.uint32), cols.astype(np.uint32), vals


def check(y, ref_plain, ref64, lens, tol):
    y = np.asarray(y)
    short = lens <= 32
    assert bit_equal(y[short], ref_plain[short]), first_diff(y[short], ref_plain[short])
    assert rel_err(y, ref64) <= tol


CASES = {
    # name: (nrows, ncols, length sampler)
    "mixed": (20_000, 30_000, lambda r, n: np.where(r.random(n) < 0.02, r.integers(33, 4000, n), r.integers(0, 33, n))),
    "empty_runs": (50_000, 8_000, lambda r, n: np.where((np.arange(n) // 1000) % 3 == 0, 0, r.integers(0, 6, n))),
    "huge_row": (3_000, 200_000, lambda r, n: np.where(np.arange(n) == 1500, 150_000, r.integers(0, 20, n))),
    "wide": (500, 100_000, lambda r, n: r.integers(0, 300, n)),
    "tall": (100_000, 50, lambda r, n: r.integers(0, 7, n)),
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_random_structures_csr_coo(sp, name, dtype):
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    nrows, ncols, sampler = CASES[name]
    lens = np.minimum(sampler(rng, nrows), ncols)
    irp, cols, vals = random_csr(rng, nrows, ncols, lens)
    vals = vals.astype(dtype)
    x = rng.uniform(-1, 1, ncols).astype(dtype)
    ref = c_oracle.csr_plain(nrows, irp, cols, vals, x)
    ref64 = c_oracle.csr_plain(nrows, irp, cols, vals.astype(np.float64), x.astype(np.float64))
    tol = 1e-12 if dtype == np.float64 else 1e-5
    csr = sp.CsrMatrix.from_arrays(nrows, ncols, irp, cols, vals)
    check(sp.spmv_csr_plain(csr, x), ref, ref64, lens, tol)
    coo = sp.csr_to_coo(csr)
    rows = np.repeat(np.arange(nrows), lens)
    ref_coo = c_oracle.coo_plain(nrows, rows, cols, vals, x)
    check(sp.spmv_coo_plain(coo, x), ref_coo, ref64, lens, tol)
    for lanes in (1, 8, 32, 100):
        y = sp.spmv_csr_vla(csr, x, sp.LaneConfig(lanes))
        assert bit_equal(y, c_oracle.csr_vla(nrows, irp, cols, vals, x, lanes)), lanes


@pytest.mark.parametrize("nnz_mod", [1, 2, 3])
def test_tail_tiles_and_unaligned_pointers(sp, nnz_mod):
    """nnz % 4 != 0 sends the last tiles through the cooperative loader;
    pointers off a 16-byte boundary send every tile there.  Both must give
    the same bits as the TMA path."""
    rng = np.random.default_rng(nnz_mod)
    nrows, ncols = 9000, 9000
    lens = rng.integers(1, 30, nrows)
    lens[-1] += (nnz_mod - lens.sum()) % 4
    irp, cols, vals = random_csr(rng, nrows, ncols, lens)
    assert vals.shape[0] % 4 == nnz_mod % 4
    x = torch.from_numpy(rng.uniform(-1, 1, ncols)).cuda()
    ref = c_oracle.csr_plain(nrows, irp, cols, vals, x.cpu().numpy())
    csr = sp.CsrMatrix.from_arrays(nrows, ncols, irp, cols, vals)
    y = sp.spmv_csr_plain(csr, x).cpu().numpy()
    assert bit_equal(y, ref)
    # unaligned views: one extra leading element shifts the data by 4 / 8 bytes
    aj = torch.empty(cols.shape[0] + 1, dtype=torch.int32, device="cuda")
    av = torch.empty(vals.shape[0] + 1, dtype=torch.float64, device="cuda")
    aj[1:] = csr.col_indices
    av[1:] = csr.values
    odd = sp.CsrMatrix(csr.shape, csr.row_pointers, aj[1:], av[1:])
    assert odd.col_indices.data_ptr() % 16 != 0
    assert bit_equal(sp.spmv_csr_plain(odd, x).cpu().numpy(), y)
    coo = sp.csr_to_coo(csr)
    y_coo = sp.spmv_coo_plain(coo, x).cpu().numpy()
    ai = torch.empty(coo.nnz + 1, dtype=torch.int32, device="cuda")
    ai[1:] = coo.row_indices
    odd_coo = sp.CooMatrix(coo.shape, ai[1:], aj[1:], av[1:], True)
    assert bit_equal(sp.spmv_coo_plain(odd_coo, x).cpu().numpy(), y_coo)


@pytest.mark.parametrize("nd,dtype", [(3, np.float64), (11, np.float32), (40, np.float64), (101, np.float32)])
def test_dia_widths_and_shapes(sp, nd, dtype):
    """Compile-time-unrolled widths (3, 11) and the generic loop (40, 101),
    rectangular, with out-of-range diagonals and the direct fallback."""
    rng = np.random.default_rng(nd)
    nrows, ncols = 3001, 2500
    offs = np.sort(rng.choice(np.arange(-nrows + 1, ncols), size=nd, replace=False)).astype(np.int32)
    padded = -(-nrows // 8) * 8
    vals = rng.standard_normal((padded, nd)).astype(dtype)
    r = np.arange(padded)[:, None]
    c = r + offs[None, :]
    vals[(c < 0) | (c >= ncols) | (r >= nrows)] = 0
    x = rng.uniform(-1, 1, ncols).astype(dtype)
    ref = c_oracle.dia_plain(nrows, ncols, offs, vals, x)
    dia = sp.DiaMatrix(sp.MatrixShape(nrows, ncols, int((vals != 0).sum())), offs, vals)
    y = sp.spmv_dia_plain(dia, x)
    assert bit_equal(y, ref), first_diff(y, ref)
    # unaligned block (row stride nd * size; an odd leading element breaks 16-byte alignment)
    flat = torch.empty(padded * nd + 1, dtype=dia.values.dtype, device="cuda")
    flat[1:] = dia.values.reshape(-1)
    odd = sp.DiaMatrix(dia.shape, dia.offsets, flat[1:].view(padded, nd))
    assert bit_equal(sp.spmv_dia_plain(odd, x), ref)


def test_unsorted_coo_duplicates_at_scale(sp):
    rng = np.random.default_rng(77)
    n, nnz = 40_000, 600_000
    rows = rng.integers(0, n, nnz)
    cols = rng.integers(0, n, nnz)
    rows[:5000] = 7  # one long, heavily duplicated row
    cols[:5000] = rng.integers(0, 50, 5000)
    vals = rng.standard_normal(nnz)
    x = rng.uniform(-1, 1, n)
    coo = sp.CooMatrix.from_arrays(n, n, rows, cols, vals)
    ref = O.coo_plain(n, rows, cols, vals, x)
    y = sp.spmv_coo_plain(coo, x)
    lens = np.bincount(rows, minlength=n)
    assert bit_equal(y[lens <= 32], ref[lens <= 32])
    assert rel_err(y, ref) <= 1e-12
    # sort_coo: stable lexsort + reduceat-order duplicate sums, bit-exact
    s = sp.sort_coo(coo).to_host()
    r_ref, c_ref, v_ref = O.sort_coo(rows, cols, vals)
    assert np.array_equal(s["row_indices"], r_ref) and np.array_equal(s["col_indices"], c_ref)
    assert bit_equal(s["values"], v_ref)


def test_conversion_round_trips_at_scale(sp):
    csr = sp.gen_stencil27(40, 36, 32)
    coo = sp.csr_to_coo(csr)
    assert coo.sorted
    back = sp.coo_to_csr(coo)
    for a, b in ((csr.row_pointers, back.row_pointers), (csr.col_indices, back.col_indices)):
        assert torch.equal(a, b)
    assert torch.equal(csr.values, back.values)
    dia = sp.coo_to_dia(coo)
    assert dia.ndiags == 27 and dia.padded_rows % 8 == 0
    coo2 = sp.dia_to_coo(dia)
    assert torch.equal(coo2.row_indices, coo.row_indices) and torch.equal(coo2.col_indices, coo.col_indices)
    assert torch.equal(coo2.values, coo.values)
    x = torch.rand(csr.ncols, dtype=torch.float64, device="cuda")
    ys = [sp.dispatch(m, x) for m in (csr, coo, dia)]
    assert torch.equal(ys[0], ys[2]) and torch.equal(ys[0], ys[1])


def test_stencil_slab_generator(sp):
    nx, ny, nz = 13, 11, 9
    full = sp.gen_stencil27(nx, ny, nz).to_host()
    r0, r1 = 2 * nx * ny + 5, 6 * nx * ny + 3
    slab = sp.gen_stencil27_rows(nx, ny, nz, r0, r1).to_host()
    irp = full["row_pointers"].astype(np.int64)
    assert np.array_equal(slab["row_pointers"].astype(np.int64), irp[r0:r1 + 1] - irp[r0])
    assert np.array_equal(slab["col_indices"], full["col_indices"][irp[r0]:irp[r1]])


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_vla_tile_path_all_lane_widths(sp, dtype):
    """Short-row plans run vla through the tile kernels (one thread plays all
    next_pow2(L) logical lanes; W >= 16 via the in-place product stack tree).
    Every width class, non-powers of two and L > 32 against the oracle,
    bit for bit, with signed zeros in the products."""
    rng = np.random.default_rng(7)
    nrows, ncols = 4_000, 6_000
    lens = rng.integers(0, 33, nrows)
    irp, cols, vals = random_csr(rng, nrows, ncols, lens)
    vals[rng.random(vals.shape[0]) < 0.05] = -0.0
    vals = vals.astype(dtype)
    x = rng.uniform(-1, 1, ncols).astype(dtype)
    x[rng.random(ncols) < 0.05] = 0.0
    csr = sp.CsrMatrix.from_arrays(nrows, ncols, irp, cols, vals)
    coo = sp.csr_to_coo(csr)
    rows = np.repeat(np.arange(nrows), lens).astype(np.uint32)
    for lanes in (1, 2, 3, 5, 8, 9, 16, 17, 32, 33, 100):
        y = sp.spmv_csr_vla(csr, x, sp.LaneConfig(lanes))
        assert bit_equal(y, O.csr_vla(nrows, irp, cols, vals, x, lanes)), ("csr", lanes)
        stats = {}
        ref_stats = {}
        y = sp.spmv_coo_vla(coo, x, sp.LaneConfig(lanes), stats)
        ref = O.coo_vla(nrows, rows, cols, vals, x, lanes, ref_stats)
        assert bit_equal(y, ref), ("coo", lanes, first_diff(y, ref))
        assert stats["outer_steps"] == ref_stats["outer_steps"]


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_warp_stream_threshold_lengths(sp, dtype):
    """Warp-stream plans (rows over 32 entries): row lengths on every
    threshold the kernels branch on (32 exact / 64 lane-serial / 256 chunk),
    empty rows between them, a row spanning many chunks and ranges, and a
    length total that is no multiple of the chunk."""
    rng = np.random.default_rng(11)
    base = [0, 1, 31, 32, 33, 63, 64, 65, 255, 256, 257, 511, 512, 513, 0, 0, 7]
    lens = np.array(base * 40 + [20_000] + base * 40 + [3], dtype=np.int64)
    nrows, ncols = lens.shape[0], 30_000
    irp, cols, vals = random_csr(rng, nrows, ncols, lens)
    vals = vals.astype(dtype)
    x = rng.uniform(-1, 1, ncols).astype(dtype)
    ref = c_oracle.csr_plain(nrows, irp, cols, vals, x)
    ref64 = c_oracle.csr_plain(nrows, irp, cols, vals.astype(np.float64), x.astype(np.float64))
    tol = 1e-12 if dtype == np.float64 else 1e-5
    csr = sp.CsrMatrix.from_arrays(nrows, ncols, irp, cols, vals)
    from paper_2304_09511_b200 import kernels as K
    assert K.csr_plan(csr).info()["kernel"] == "warp_stream"
    check(sp.spmv_csr_plain(csr, x), ref, ref64, lens, tol)
    coo = sp.csr_to_coo(csr)
    assert K.coo_plan(coo).info()["kernel"] == "warp_stream"
    rows = np.repeat(np.arange(nrows), lens)
    check(sp.spmv_coo_plain(coo, x), c_oracle.coo_plain(nrows, rows, cols, vals, x), ref64, lens, tol)
    # determinism: dynamic range hand-out must not change a bit
    a = sp.spmv_csr_plain(csr, x)
    b = sp.spmv_csr_plain(csr, x)
    assert bit_equal(a, b)
