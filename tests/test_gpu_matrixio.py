"""Matrix Market ingest (host parse, device sort_coo) vs the reference's
read_matrix_market outputs (tests/golden/mm.npz), plus write/read round trip."""

import io

import numpy as np
import pytest

from _util import bit_equal, load_golden, matrix_arrays


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


@pytest.mark.gpu
def test_read_matches_reference(sp):
    from paper_2304_09511_b200.matrixio import read_matrix_market
    d = load_golden("mm")
    for name in d["names"]:
        name = str(name)
        got = read_matrix_market(str(d[f"{name}/text"]).encode())
        ref = matrix_arrays(d, f"{name}/coo")
        h = got.to_host()
        assert got.sorted and h["shape"].nnz == int(ref["shape"][2]), name
        assert np.array_equal(h["row_indices"], ref["row_indices"]), name
        assert np.array_equal(h["col_indices"], ref["col_indices"]), name
        assert bit_equal(h["values"], ref["values"]), name


@pytest.mark.gpu
def test_write_read_round_trip(sp):
    from paper_2304_09511_b200.matrixio import read_matrix_market, write_matrix_market
    A = sp.gen_stencil27(5, 4, 3)
    rng = np.random.default_rng(0)
    A = sp.CsrMatrix(A.shape, A.row_pointers, A.col_indices, A.values * 0 + sp.formats.scalar_tensor(
        rng.standard_normal(A.nnz), device=A.values.device))
    buf = io.StringIO()
    write_matrix_market(A, buf, comment="round trip")
    back = read_matrix_market(buf.getvalue().encode())
    h, ref = back.to_host(), sp.csr_to_coo(A).to_host()
    assert np.array_equal(h["row_indices"], ref["row_indices"]) and bit_equal(h["values"], ref["values"])


def test_parse_errors():
    import paper_2304_09511_b200.errors as E
    from paper_2304_09511_b200.matrixio import read_matrix_market
    bad = {
        b"hello": E.ParseError,
        b"%%MatrixMarket matrix array real general\n2 2\n1\n2\n3\n4\n": E.UnsupportedField,
        b"%%MatrixMarket matrix coordinate complex general\n1 1 1\n1 1 1 0\n": E.UnsupportedField,
        b"%%MatrixMarket matrix coordinate real hermitian\n1 1 1\n1 1 1\n": E.UnsupportedField,
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n3 1 1.0\n": E.ParseError,
        b"%%MatrixMarket matrix coordinate real general\n2 2 2\n1 1 1.0\n": E.ParseError,
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 1.0\n2 2 2.0\n": E.ParseError,
        b"%%MatrixMarket matrix coordinate real general\n2 2 1\n1 1 x\n": E.ParseError,
    }
    for text, exc in bad.items():
        with pytest.raises(exc):
            read_matrix_market(text)


def test_bulk_parse_equals_line_walk():
    """The numpy text-reader pass and the reference-style line walk give the
    same (row, column, value) arrays, bit for bit, on well-formed entry lines
    (tabs, exponents, signed zeros, subnormals, inf / nan), and the bulk pass
    declines (None) what only the line walk may judge."""
    from paper_2304_09511_b200 import matrixio as M
    rng = np.random.default_rng(5)
    n = 20000
    i, j = rng.integers(1, 5001, n), rng.integers(1, 5001, n)
    v = rng.standard_normal(n) * 10.0 ** rng.integers(-300, 300, n)
    data = ["%d %d %.17g" % t for t in zip(i.tolist(), j.tolist(), v.tolist())]
    data += ["1\t2   3e-2", "3 4 -1E5", "5 6 nan", "7 8 -inf", "9 10 +.5", "11 12 1e-320", "13 14 -0.0", "+15 16 1."]
    bulk, walk = M._mm_entries_bulk(data, 3), M._mm_entries_by_line(data, 3, 5000, 5000)
    assert bulk is not None and all(a.tobytes() == b.tobytes() for a, b in zip(bulk, walk))
    pat = ["%d %d" % t for t in zip(i.tolist(), j.tolist())]
    bulk, walk = M._mm_entries_bulk(pat, 2), M._mm_entries_by_line(pat, 2, 5000, 5000)
    assert all(a.tobytes() == b.tobytes() for a, b in zip(bulk, walk))
    for odd in (["1 2 3", "1.0 2 3"], ["1 2 3 4", "1 2"], ["1 2 x"], ["1_0 2 3"], ["99999999999999999999 1 3"]):
        assert M._mm_entries_bulk(odd, 3) is None
