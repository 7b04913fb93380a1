"""sort_coo paths (csrc/convert.cu) against the numpy oracle, bit for bit.

convert.py:60-84: stable lexsort((cols, rows)), duplicate runs summed in
np.add.reduceat order.  Unsorted inputs take the group path (the (column,
value) pairs ride a radix sort on the row bits above the low 8, then
256-row groups are sorted in shared memory); a group of more than 7168
entries sends the matrix to the per-row stage after one more radix pass.
Cases force each branch: rows of <= 32 and > 32 entries inside a group,
duplicates (short and long runs, -0.0, NaN), at most 256 rows (no radix
pass), a group too large (fallback), empty rows and groups, f32, rows already
in order with shuffled columns.
"""

import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def _check(sp, n, ncols, rows, cols, vals):
    from _util import bit_equal
    from oracle import spmv_oracle as O
    coo = sp.CooMatrix.from_arrays(n, ncols, rows, cols, vals)
    got = sp.sort_coo(coo)
    assert got.sorted
    h = got.to_host()
    r_ref, c_ref, v_ref = O.sort_coo(rows, cols, vals)
    assert np.array_equal(h["row_indices"], r_ref)
    assert np.array_equal(h["col_indices"], c_ref)
    assert bit_equal(h["values"], v_ref)
    assert got.nnz == r_ref.shape[0]


def _draw(rng, n, ncols, lens, dtype, dup=0.0):
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, ncols, rows.shape[0])
    if dup > 0:  # repeat some coordinates
        k = int(rows.shape[0] * dup)
        src = rng.integers(0, rows.shape[0], k)
        dst = rng.integers(0, rows.shape[0], k)
        same = rows[src] == rows[dst]
        cols[dst[same]] = cols[src[same]]
    vals = rng.standard_normal(rows.shape[0]).astype(dtype)
    order = rng.permutation(rows.shape[0])
    return rows[order], cols[order], vals[order]


CASES = {
    # name: (nrows, ncols, row lengths, duplicate fraction)
    "stencil_like": (40_000, 40_000, lambda r, n: np.full(n, 27), 0.0),
    "mixed_lengths": (20_000, 5_000, lambda r, n: r.integers(0, 60, n), 0.0),         # rows over 32 inside groups
    "dups_short": (30_000, 400, lambda r, n: r.integers(0, 20, n), 0.3),
    "dups_long_rows": (3_000, 40, lambda r, n: r.integers(20, 90, n), 0.5),           # long duplicate runs
    "few_rows": (200, 1000, lambda r, n: r.integers(0, 30, n), 0.1),                  # <= 256 rows: no radix pass
    "few_rows_big": (256, 3000, lambda r, n: r.integers(40, 120, n), 0.0),            # one group, too large: fallback
    "huge_row": (50_000, 60_000, lambda r, n: np.where(np.arange(n) == 1234, 30_000, r.integers(0, 12, n)), 0.0),
    "gaps": (300_000, 1000, lambda r, n: np.where(np.arange(n) % 997 == 0, 25, 0), 0.1),  # mostly empty groups
    "one_entry": (5, 5, lambda r, n: np.array([0, 0, 1, 0, 0]), 0.0),
    "hypersparse": (3_000_000, 50, lambda r, n: (r.random(n) < 0.001).astype(np.int64) * 3, 0.2),  # rows >> entries
}


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("dtype", [np.float64, np.float32])
def test_sort_coo_paths(sp, name, dtype):
    import zlib
    n, ncols, sampler, dup = CASES[name]
    rng = np.random.default_rng(zlib.crc32(name.encode()))
    lens = sampler(rng, n).astype(np.int64)
    rows, cols, vals = _draw(rng, n, ncols, lens, dtype, dup)
    _check(sp, n, ncols, rows, cols, vals)


def test_sort_coo_signed_zero_and_nan_duplicates(sp):
    """Duplicate sums keep numpy's reduceat arithmetic: -0.0 + -0.0 = -0.0,
    NaN propagates, cancelling pairs leave a stored zero."""
    rng = np.random.default_rng(11)
    n = 3000
    rows = rng.integers(0, n, 40_000)
    cols = rng.integers(0, 8, 40_000)
    vals = rng.standard_normal(40_000)
    vals[rng.integers(0, 40_000, 4000)] = -0.0
    vals[rng.integers(0, 40_000, 50)] = np.nan
    vals[1::2][:5000] = -vals[0::2][:5000]
    _check(sp, n, 8, rows, cols, vals)


def test_sort_coo_rows_in_order_columns_shuffled(sp):
    """Rows already non-decreasing (flag unset): no radix sort at all."""
    rng = np.random.default_rng(12)
    n = 30_000
    lens = rng.integers(0, 50, n)
    rows = np.repeat(np.arange(n), lens)
    cols = rng.integers(0, 500, rows.shape[0])
    vals = rng.standard_normal(rows.shape[0])
    _check(sp, n, 500, rows, cols, vals)
