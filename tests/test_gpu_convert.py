"""On-device conversions: bit-exact with the reference (convert.py), mirroring
test_convert.py and acceptance criterion 04 (test_acceptance.py:128-155)."""

import numpy as np
import pytest

from _util import bit_equal, corpus_names, load_golden, matrix_arrays
from test_gpu_kernels import dev_matrix

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def host(m):
    return m.to_host()


def assert_coo_equal(got, ref_arrs):
    h = got.to_host()
    assert h["shape"].nnz == int(ref_arrs["shape"][2])
    assert np.array_equal(h["row_indices"], ref_arrs["row_indices"])
    assert np.array_equal(h["col_indices"], ref_arrs["col_indices"])
    assert bit_equal(h["values"], ref_arrs["values"])


@pytest.mark.parametrize("name", corpus_names())
def test_corpus_conversions_bit_exact(sp, name):
    d = load_golden("corpus")
    coo_a = matrix_arrays(d, f"{name}/coo")
    csr_a = matrix_arrays(d, f"{name}/csr")
    dia_a = matrix_arrays(d, f"{name}/dia")
    orig_a = matrix_arrays(d, f"{name}/orig")
    loose = sp.DiaFillPolicy(max_fill_ratio=float("inf"))
    # the as-given container through the hub, to every format
    fmt0 = "csr" if "row_pointers" in orig_a else ("dia" if "offsets" in orig_a else "coo")
    orig = dev_matrix(sp, orig_a, fmt0)
    assert_coo_equal(sp.to_format(orig, "coo"), coo_a)
    csr = sp.to_format(orig, "csr")
    h = csr.to_host()
    assert np.array_equal(h["row_pointers"], csr_a["row_pointers"])
    assert np.array_equal(h["col_indices"], csr_a["col_indices"]) and bit_equal(h["values"], csr_a["values"])
    dia = sp.to_format(orig, "dia", loose)
    h = dia.to_host()
    assert np.array_equal(h["offsets"], dia_a["offsets"]) and bit_equal(h["values"], dia_a["values"])
    # round trips (criterion 04)
    coo = dev_matrix(sp, coo_a, "coo")
    assert_coo_equal(sp.csr_to_coo(sp.coo_to_csr(coo)), coo_a)
    try:
        dd = sp.coo_to_dia(coo)
    except sp.FillRatioExceeded:
        return
    back = sp.dia_to_coo(dd)
    keep = coo_a["values"] != 0
    ref = dict(coo_a)
    ref.update(row_indices=coo_a["row_indices"][keep], col_indices=coo_a["col_indices"][keep],
               values=coo_a["values"][keep], shape=np.array([coo_a["shape"][0], coo_a["shape"][1], keep.sum()]))
    assert_coo_equal(back, ref)


def test_sort_coo_duplicates_pairwise(sp):
    d = load_golden("convert")
    for dt in ("float64", "float32"):
        src = matrix_arrays(d, f"dups_{dt}/in")
        got = sp.sort_coo(dev_matrix(sp, src, "coo"))
        assert got.sorted
        assert_coo_equal(got, matrix_arrays(d, f"dups_{dt}/sorted"))


def test_csr_to_coo_unsorted_and_dia_specials(sp):
    d = load_golden("convert")
    coo = sp.csr_to_coo(dev_matrix(sp, matrix_arrays(d, "csr_unsorted/in"), "csr"))
    assert not coo.sorted
    assert np.array_equal(coo.to_host()["row_indices"], matrix_arrays(d, "csr_unsorted/coo")["row_indices"])
    fixed = sp.sort_coo(coo)
    assert fixed.to_host()["col_indices"].tolist()[:2] == [1, 3]
    got = sp.dia_to_coo(dev_matrix(sp, matrix_arrays(d, "dia_special/in"), "dia"))
    assert_coo_equal(got, matrix_arrays(d, "dia_special/coo"))
    rand = dev_matrix(sp, matrix_arrays(d, "rand/coo"), "coo")
    h = sp.coo_to_csr(rand).to_host()
    assert np.array_equal(h["row_pointers"], matrix_arrays(d, "rand/csr")["row_pointers"])
    h = sp.coo_to_dia(rand, sp.DiaFillPolicy(float("inf"))).to_host()
    assert np.array_equal(h["offsets"], matrix_arrays(d, "rand/dia")["offsets"])
    assert bit_equal(h["values"], matrix_arrays(d, "rand/dia")["values"])


def test_coo_to_csr_misflagged_rows(sp):
    """A COO flagged sorted whose rows are not: row pointers come from the
    per-row counts like the reference's bincount + cumsum (convert.py:92-93);
    columns and values are copied as stored."""
    d = load_golden("convert")
    want = matrix_arrays(d, "misflagged/csr")
    h = sp.coo_to_csr(dev_matrix(sp, matrix_arrays(d, "misflagged/coo"), "coo")).to_host()
    assert np.array_equal(h["row_pointers"], want["row_pointers"])
    assert np.array_equal(h["col_indices"], want["col_indices"])
    assert bit_equal(h["values"], want["values"])


def test_canonical_conversion_kats(sp):
    d = load_golden("canonical")
    can = dev_matrix(sp, matrix_arrays(d, "coo"), "coo")
    assert sp.coo_to_csr(can).to_host()["row_pointers"].tolist() == [0, 2, 4, 6, 9, 11]
    dia = sp.coo_to_dia(can)
    h = dia.to_host()
    assert h["offsets"].tolist() == [-3, -1, 0, 1, 2] and dia.padded_rows == 8
    assert h["values"][3].tolist() == [6.0, 0.0, 7.0, 8.0, 0.0] and dia.nnz == 11
    assert not h["values"][5:].any()
    assert sp.sort_coo(can) is can
    assert sp.to_format(sp.to_format(can, "csr"), "csr").format == sp.Format.CSR


def test_fill_policy(sp):
    corner = sp.CooMatrix.from_arrays(1000, 1000, [0, 999], [999, 0], [1.0, 2.0], sorted=True)
    with pytest.raises(sp.FillRatioExceeded) as exc:
        sp.coo_to_dia(corner)
    assert "fill ratio" in str(exc.value)
    n = 64
    rows = np.arange(n)
    anti = sp.CooMatrix.from_arrays(n, n, rows, n - 1 - rows, np.ones(n))
    with pytest.raises(sp.FillRatioExceeded):
        sp.coo_to_dia(sp.sort_coo(anti))
    with pytest.raises(sp.FillRatioExceeded) as exc:
        sp.coo_to_dia(sp.CooMatrix.from_arrays(3, 3, [0, 1], [1, 0], [1.0, 2.0], sorted=True),
                      sp.DiaFillPolicy(max_fill_ratio=1e9, max_ndiags=1))
    assert "cap" in str(exc.value)
    pair = sp.CooMatrix.from_arrays(16, 16, [0, 15], [15, 0], [1.0, 2.0], sorted=True)
    with pytest.raises(sp.FillRatioExceeded):
        sp.coo_to_dia(pair)
    dia = sp.coo_to_dia(pair, sp.DiaFillPolicy(max_fill_ratio=16.0))
    assert dia.to_host()["offsets"].tolist() == [-15, 15] and tuple(dia.values.shape) == (16, 2)
    with pytest.raises(sp.UnsortedInput):
        sp.coo_to_csr(sp.CooMatrix.from_arrays(2, 2, [1, 0], [0, 0], [1.0, 2.0]))
    with pytest.raises(sp.UnsortedInput):
        sp.coo_to_dia(sp.CooMatrix.from_arrays(2, 2, [1, 0], [0, 1], [1.0, 2.0]))


def test_stencil_generator_bit_exact(sp):
    d = load_golden("stencil")
    for dims in d["dims"]:
        key = "x".join(str(int(v)) for v in dims)
        ref = matrix_arrays(d, key)
        m = sp.gen_stencil27(*map(int, dims))
        h = m.to_host()
        assert np.array_equal(h["row_pointers"], ref["row_pointers"])
        assert np.array_equal(h["col_indices"], ref["col_indices"]) and bit_equal(h["values"], ref["values"])
        assert bit_equal(sp.spmv_csr_plain(m, d[f"{key}/x"]), d[f"{key}/y"])
    with pytest.raises(sp.IndexOverflow):
        sp.gen_stencil27(2048, 2048, 1024)


def test_validate_device(sp):
    d = load_golden("canonical")
    for fmt in ("coo", "csr", "dia"):
        assert sp.validate(dev_matrix(sp, matrix_arrays(d, fmt), fmt)) == []
    bad = sp.CooMatrix.from_arrays(2, 2, [1, 0], [0, 1], [1.0, 2.0], sorted=True)
    assert any("sorted flag" in v for v in sp.validate(bad))


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("nrows,ncols,offsets", [
    (1000, 1000, [-65, -1, 0, 1, 65]),                       # 8 lanes per row, 4 rows per warp step
    (5000, 5000, [-4096, -1024, -512, -2, -1, 0, 1, 2, 512, 1024, 4096]),  # 16 lanes per row
    (4097, 4097, list(range(-13, 14))),                        # 27 diagonals, a partial last tile
    (3000, 3000, list(range(-16, 16))),                        # 32 diagonals: the tile kernels' limit
    (3000, 3000, list(range(-20, 20))),                        # 40 diagonals: the per-row kernels
    (700, 2500, [-900, -3, 0, 5, 1800, 2600]),                 # wide: a diagonal with no in-bounds cell
    (2500, 300, [-2600, -2400, -7, 0, 3, 299]),                # tall
    (129, 129, [0]),                                           # one lane per row, 32 rows per warp step
])
def test_dia_to_coo_tile_kernels_match_oracle(sp, dtype, nrows, ncols, offsets):
    """dia_to_coo (per-tile count + emit kernels up to 32 diagonals, per-row
    kernels above) against the oracle's convert.py:147-177 restatement: dense
    diagonals with zeros, -0.0 (dropped) and NaN (kept) sprinkled in, several
    row tiles, every lane-group width."""
    from oracle import spmv_oracle as O
    rng = np.random.default_rng(nrows * 31 + len(offsets))
    offs = np.array(offsets, dtype=np.int32)
    padded = O.round_up(nrows, 8)
    vals = rng.uniform(-1.0, 1.0, (padded, len(offs))).astype(dtype)
    vals[rng.random(vals.shape) < 0.05] = 0.0
    vals[rng.random(vals.shape) < 0.02] = -0.0
    vals[rng.random(vals.shape) < 0.01] = np.nan
    vals[nrows:] = 0.0
    r = np.arange(padded, dtype=np.int64)[:, None] + offs[None, :].astype(np.int64)
    vals[(r < 0) | (r >= ncols)] = 0.0  # out-of-matrix cells are stored as zero (formats.py:166-207)
    wr, wc, wv = O.dia_to_coo(nrows, ncols, offs, vals)
    dia = sp.DiaMatrix(sp.MatrixShape(nrows, ncols, wr.shape[0]), offs, vals)
    got = sp.dia_to_coo(dia).to_host()
    assert got["shape"].nnz == wr.shape[0]
    assert np.array_equal(got["row_indices"], wr) and np.array_equal(got["col_indices"], wc)
    assert bit_equal(got["values"], wv)


@pytest.mark.parametrize("dtype", [np.float64, np.float32])
@pytest.mark.parametrize("nrows,ncols,offsets,pad_to,misflag", [
    (1000, 1000, [-65, -1, 0, 1, 65], 8, False),
    (4099, 4099, list(range(-13, 14)), 8, False),        # 27 diagonals
    (4099, 4099, list(range(-13, 14)), 64, False),       # padding rows past nrows
    (3000, 3500, [-2999, -40, 0, 7, 3499], 8, False),    # corner diagonals with one cell each
    (2000, 2000, list(range(-300, 300, 3)), 8, False),   # 200 diagonals
    (600, 600, list(range(-599, 600)), 8, False),        # 1199 diagonals
    (1500, 1500, [-3, 0, 4], 8, True),                    # flagged sorted, rows out of order
])
def test_coo_to_dia_structures_match_oracle(sp, dtype, nrows, ncols, offsets, pad_to, misflag):
    """coo_to_dia (diagonal census, zero fill, scatter) against the oracle's
    convert.py:113-144 restatement: empty rows, padding rows past nrows, corner
    diagonals, wide blocks, and triples flagged sorted whose rows are not."""
    from oracle import spmv_oracle as O
    rng = np.random.default_rng(nrows + 7 * len(offsets) + pad_to)
    offs = np.array(offsets, dtype=np.int64)
    rows = np.repeat(np.arange(nrows, dtype=np.int64), len(offs))
    cols = rows + np.tile(offs, nrows)
    keep = (cols >= 0) & (cols < ncols) & (rng.random(rows.shape[0]) < 0.8)
    keep &= ~np.isin(rows, rng.choice(nrows, nrows // 20, replace=False))  # some empty rows
    for o in offs:  # every diagonal keeps at least one cell
        i = int(np.flatnonzero((cols - rows == o) & (cols >= 0) & (cols < ncols))[0])
        keep[i] = True
    rows, cols = rows[keep], cols[keep]
    vals = rng.uniform(-1.0, 1.0, rows.shape[0]).astype(dtype)
    if misflag:
        perm = rng.permutation(rows.shape[0])
        rows, cols, vals = rows[perm], cols[perm], vals[perm]
    want_off, want_vals = O.coo_to_dia(nrows, ncols, rows, cols, vals, pad_to)
    coo = sp.CooMatrix.from_arrays(nrows, ncols, rows.astype(np.uint32), cols.astype(np.uint32), vals, sorted=True)
    got = sp.coo_to_dia(coo, sp.DiaFillPolicy(float("inf")), pad_to).to_host()
    assert np.array_equal(got["offsets"], want_off)
    assert got["values"].shape == want_vals.shape and bit_equal(got["values"], want_vals)
