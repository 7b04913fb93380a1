"""Pin the CPU oracle to the reference: every oracle function must reproduce
the golden vectors (made by running spmvkit itself, tests/golden/
make_golden.py) bit for bit.  CPU only."""

import numpy as np
import pytest

from _util import bit_equal, corpus_names, first_diff, load_golden, matrix_arrays
from oracle import c_oracle
from oracle import spmv_oracle as O

LANES = (1, 2, 3, 4, 8, 16, 32, 64)


@pytest.fixture(scope="module", params=corpus_names())
def case(request):
    d = load_golden("corpus")
    name = request.param
    return name, d


def test_corpus_size():
    assert len(corpus_names()) >= 30


def test_corpus_plain_numpy(case):
    name, d = case
    x = d[f"{name}/x"]
    csr = matrix_arrays(d, f"{name}/csr")
    nrows, ncols, _ = csr["shape"]
    y = O.csr_plain(nrows, csr["row_pointers"], csr["col_indices"], csr["values"], x)
    assert bit_equal(y, d[f"{name}/csr/y_plain"]), first_diff(y, d[f"{name}/csr/y_plain"])
    coo = matrix_arrays(d, f"{name}/coo")
    y = O.coo_plain(nrows, coo["row_indices"], coo["col_indices"], coo["values"], x)
    assert bit_equal(y, d[f"{name}/coo/y_plain"])
    dia = matrix_arrays(d, f"{name}/dia")
    y = O.dia_plain(nrows, ncols, dia["offsets"], dia["values"], x)
    assert bit_equal(y, d[f"{name}/dia/y_plain"])


def test_corpus_vla_numpy(case):
    name, d = case
    x = d[f"{name}/x"]
    csr = matrix_arrays(d, f"{name}/csr")
    coo = matrix_arrays(d, f"{name}/coo")
    dia = matrix_arrays(d, f"{name}/dia")
    nrows, ncols, _ = csr["shape"]
    for lanes in LANES:
        y = O.csr_vla(nrows, csr["row_pointers"], csr["col_indices"], csr["values"], x, lanes)
        assert bit_equal(y, d[f"{name}/csr/y_vla{lanes}"]), (lanes, first_diff(y, d[f"{name}/csr/y_vla{lanes}"]))
        stats = {}
        y = O.coo_vla(nrows, coo["row_indices"], coo["col_indices"], coo["values"], x, lanes, stats)
        assert bit_equal(y, d[f"{name}/coo/y_vla{lanes}"]), lanes
        assert stats["outer_steps"] == int(d[f"{name}/coo/steps_vla{lanes}"])
        y = O.dia_vla(nrows, ncols, dia["offsets"], dia["values"], x, lanes)
        assert bit_equal(y, d[f"{name}/dia/y_vla{lanes}"]), lanes


def test_corpus_c_oracle(case):
    name, d = case
    x = d[f"{name}/x"]
    csr = matrix_arrays(d, f"{name}/csr")
    coo = matrix_arrays(d, f"{name}/coo")
    dia = matrix_arrays(d, f"{name}/dia")
    nrows, ncols, _ = csr["shape"]
    assert bit_equal(c_oracle.csr_plain(nrows, csr["row_pointers"], csr["col_indices"], csr["values"], x),
                     d[f"{name}/csr/y_plain"])
    assert bit_equal(c_oracle.coo_plain(nrows, coo["row_indices"], coo["col_indices"], coo["values"], x),
                     d[f"{name}/coo/y_plain"])
    assert bit_equal(c_oracle.dia_plain(nrows, ncols, dia["offsets"], dia["values"], x), d[f"{name}/dia/y_plain"])
    for lanes in LANES:
        y = c_oracle.csr_vla(nrows, csr["row_pointers"], csr["col_indices"], csr["values"], x, lanes)
        assert bit_equal(y, d[f"{name}/csr/y_vla{lanes}"]), lanes


def test_corpus_conversions(case):
    name, d = case
    coo = matrix_arrays(d, f"{name}/coo")
    csr = matrix_arrays(d, f"{name}/csr")
    dia = matrix_arrays(d, f"{name}/dia")
    nrows, ncols, nnz = coo["shape"]
    assert np.array_equal(O.coo_to_csr(nrows, coo["row_indices"]), csr["row_pointers"])
    rows, ok = O.csr_to_coo(nrows, csr["row_pointers"], csr["col_indices"])
    assert ok and np.array_equal(rows, coo["row_indices"])
    offs, vals = O.coo_to_dia(nrows, ncols, coo["row_indices"], coo["col_indices"], coo["values"])
    assert np.array_equal(offs, dia["offsets"]) and bit_equal(vals, dia["values"])
    r, c, v = O.dia_to_coo(nrows, ncols, dia["offsets"], dia["values"])
    ref_r, ref_c, ref_v = coo["row_indices"], coo["col_indices"], coo["values"]
    keep = ref_v != 0  # dia_to_coo drops stored zeros (convert.py:164)
    assert np.array_equal(r, ref_r[keep]) and np.array_equal(c, ref_c[keep]) and bit_equal(v, ref_v[keep])
    orig = matrix_arrays(d, f"{name}/orig")
    if "row_indices" in orig and not bool(orig["sorted"]):
        r, c, v = O.sort_coo(orig["row_indices"], orig["col_indices"], orig["values"])
        assert np.array_equal(r, ref_r) and np.array_equal(c, ref_c) and bit_equal(v, ref_v)


def test_canonical_kats():
    d = load_golden("canonical")
    assert d["csr/ones/y_plain"].tolist() == [3.0, 14.0, 9.0, 21.0, 19.0]
    assert d["csr/ramp/y_plain"].tolist() == [7.0, 17.0, 32.0, 74.0, 68.0]
    assert d["csr/row_pointers"].tolist() == [0, 2, 4, 6, 9, 11]
    assert d["dia/offsets"].tolist() == [-3, -1, 0, 1, 2]
    assert d["dia/values"][3].tolist() == [6.0, 0.0, 7.0, 8.0, 0.0]
    # COO vla step counts (test_kernels.py:95-120)
    assert int(d["row20/ones/steps_vla4"]) == 5
    assert int(d["coo/ones/steps_vla4"]) == 5
    assert int(d["coo/ones/steps_vla1"]) == 11
    assert int(d["row20/arange/steps_vla8"]) == 3
    coo = matrix_arrays(d, "coo")
    for xn, x in (("ones", np.ones(5)), ("ramp", np.arange(1.0, 6.0))):
        assert bit_equal(O.coo_plain(5, coo["row_indices"], coo["col_indices"], coo["values"], x),
                         d[f"coo/{xn}/y_plain"])


def test_long_rows_oracle():
    d = load_golden("long_rows")
    for name in d["names"]:
        name = str(name)
        x = d[f"{name}/x"]
        csr = matrix_arrays(d, f"{name}/csr")
        coo = matrix_arrays(d, f"{name}/coo")
        n = int(csr["shape"][0])
        assert bit_equal(O.csr_plain(n, csr["row_pointers"], csr["col_indices"], csr["values"], x),
                         d[f"{name}/csr/y_plain"])
        assert bit_equal(c_oracle.csr_plain(n, csr["row_pointers"], csr["col_indices"], csr["values"], x),
                         d[f"{name}/csr/y_plain"])
        assert bit_equal(O.coo_plain(n, coo["row_indices"], coo["col_indices"], coo["values"], x),
                         d[f"{name}/coo/y_plain"])
        for lanes in (1, 4, 32):
            assert bit_equal(c_oracle.csr_vla(n, csr["row_pointers"], csr["col_indices"], csr["values"], x, lanes),
                             d[f"{name}/csr/y_vla{lanes}"])


def test_reduceat_model():
    d = load_golden("reduceat")
    for dt in ("float64", "float32"):
        a, idx = d[f"{dt}/a"], d[f"{dt}/idx"]
        ends = list(idx[1:]) + [a.shape[0]]
        got = np.array([O.reduceat_sum(a[s:e]) for s, e in zip(idx, ends)], dtype=a.dtype)
        assert bit_equal(got, d[f"{dt}/out"])


def test_convert_edge_cases():
    d = load_golden("convert")
    for dt in ("float64", "float32"):
        src = matrix_arrays(d, f"dups_{dt}/in")
        ref = matrix_arrays(d, f"dups_{dt}/sorted")
        r, c, v = O.sort_coo(src["row_indices"], src["col_indices"], src["values"])
        assert np.array_equal(r, ref["row_indices"]) and np.array_equal(c, ref["col_indices"])
        assert bit_equal(v, ref["values"]), first_diff(v, ref["values"])
    src = matrix_arrays(d, "csr_unsorted/in")
    ref = matrix_arrays(d, "csr_unsorted/coo")
    rows, ok = O.csr_to_coo(3, src["row_pointers"], src["col_indices"])
    assert np.array_equal(rows, ref["row_indices"]) and ok == bool(ref["sorted"]) and not ok
    src = matrix_arrays(d, "dia_special/in")
    ref = matrix_arrays(d, "dia_special/coo")
    r, c, v = O.dia_to_coo(6, 7, src["offsets"], src["values"])
    assert np.array_equal(r, ref["row_indices"]) and np.array_equal(c, ref["col_indices"]) and bit_equal(v, ref["values"])
    coo = matrix_arrays(d, "rand/coo")
    assert np.array_equal(O.coo_to_csr(40, coo["row_indices"]), matrix_arrays(d, "rand/csr")["row_pointers"])
    offs, vals = O.coo_to_dia(40, 50, coo["row_indices"], coo["col_indices"], coo["values"])
    dia = matrix_arrays(d, "rand/dia")
    assert np.array_equal(offs, dia["offsets"]) and bit_equal(vals, dia["values"])


def test_stencil_generator():
    d = load_golden("stencil")
    for dims in d["dims"]:
        key = "x".join(str(int(v)) for v in dims)
        ref = matrix_arrays(d, key)
        irp, cols, vals = O.stencil27(*map(int, dims))
        assert np.array_equal(irp, ref["row_pointers"]) and np.array_equal(cols, ref["col_indices"])
        assert bit_equal(vals, ref["values"])
        n = int(ref["shape"][0])
        assert bit_equal(O.csr_plain(n, irp, cols, vals, d[f"{key}/x"]), d[f"{key}/y"])


def test_stencil_row_slab_and_closed_form():
    from paper_2304_09511_b200.matrixio import stencil_row_pointer
    nx, ny, nz = 7, 5, 4
    irp, cols, vals = O.stencil27(nx, ny, nz)
    for p in range(nx * ny * nz + 1):
        assert stencil_row_pointer(nx, ny, nz, p) == int(irp[p])
    s_irp, s_cols, s_vals = O.stencil27(nx, ny, nz, row_begin=35, row_end=105)
    assert np.array_equal(s_irp.astype(np.int64), irp[35:106].astype(np.int64) - int(irp[35]))
    assert np.array_equal(s_cols, cols[irp[35]:irp[105]])
