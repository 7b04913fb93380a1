"""GPU parity of the SpMV kernels against the reference's golden vectors and
the pinned oracle.  Mirrors the reference's test_kernels.py / acceptance
criteria 01-03 (test_acceptance.py:75-118).

Exactness contract checked here:
  * DIA plain/vla                     bit-exact, every row
  * CSR plain, rows <= 32 entries     bit-exact with spmv_csr_plain
  * COO plain, rows <= 32 entries     bit-exact with spmv_coo_plain
  * rows of 33..256 entries inside    bit-exact with spmv_csr_vla(lanes=32)
    one tile (entries [T t, T t + T), T = the plan's tile, 1024 or 2048)
  * all other rows                    rel_err <= 1e-12 (f64) / 1e-5 (f32)
  * CSR/COO vla, any lane count       bit-exact with the reference vla
"""

import numpy as np
import pytest
import torch

from _util import bit_equal, corpus_names, first_diff, load_golden, matrix_arrays, rel_err

pytestmark = pytest.mark.gpu

LANES = (1, 2, 3, 4, 8, 16, 32, 64)


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


def dev_matrix(sp, arrs: dict, fmt: str):
    nrows, ncols, nnz = (int(v) for v in arrs["shape"])
    shape = sp.MatrixShape(nrows, ncols, nnz)
    if fmt == "csr":
        return sp.CsrMatrix(shape, arrs["row_pointers"], arrs["col_indices"], arrs["values"])
    if fmt == "coo":
        return sp.CooMatrix(shape, arrs["row_indices"], arrs["col_indices"], arrs["values"], bool(arrs["sorted"]))
    return sp.DiaMatrix(shape, arrs["offsets"], arrs["values"])


def row_lengths(arrs: dict) -> np.ndarray:
    return np.diff(arrs["row_pointers"].astype(np.int64))


def plan_tile(m) -> dict:
    """The plan's kernel choice: {"tile": entries per tile, "kernel": ...}."""
    from paper_2304_09511_b200 import kernels as K
    return K.csr_plan(m).info() if m.format.value == "csr" else K.coo_plan(m).info()


def check_rowwise(y, y_plain, y_vla32, lens, tol, plan):
    """Apply the exactness contract row by row.  Tile kernels: rows <= 32
    bit-exact, rows of 33..256 inside one tile bit-exact with vla(32), the
    rest within tol.  Warp-stream and panel kernels (csrc/wstream.cuh,
    csrc/panel.cuh): rows <= 32 bit-exact, the rest within tol."""
    y = np.asarray(y)
    short = lens <= 32
    assert bit_equal(y[short], y_plain[short]), first_diff(y[short], y_plain[short])
    if plan.get("kernel") in ("warp_stream", "panel"):
        if (~short).any():
            assert rel_err(y[~short], y_plain[~short]) <= tol
        return
    TILE = plan["tile"]
    ends = np.cumsum(lens)
    starts = ends - lens
    one_tile = (lens > 32) & (lens <= 256) & (starts // TILE == (ends - 1) // TILE)
    assert bit_equal(y[one_tile], y_vla32[one_tile]), first_diff(y[one_tile], y_vla32[one_tile])
    spanning = (lens > 32) & ~one_tile
    if spanning.any():
        assert rel_err(y[spanning], y_plain[spanning]) <= tol


@pytest.mark.parametrize("name", corpus_names())
def test_corpus_all_kernels(sp, name):
    d = load_golden("corpus")
    x = d[f"{name}/x"]
    lens = row_lengths(matrix_arrays(d, f"{name}/csr"))
    for fmt in ("csr", "coo", "dia"):
        m = dev_matrix(sp, matrix_arrays(d, f"{name}/{fmt}"), fmt)
        y = sp.dispatch(m, x, "plain")
        assert isinstance(y, np.ndarray) and y.dtype == m.dtype
        ref = d[f"{name}/{fmt}/y_plain"]
        if fmt == "dia":
            assert bit_equal(y, ref), (fmt, first_diff(y, ref))
        else:
            check_rowwise(y, ref, d[f"{name}/csr/y_vla32"], lens, 1e-12, plan_tile(m))
        for lanes in LANES:
            stats = {}
            if fmt == "coo":
                y = sp.spmv_coo_vla(m, x, sp.LaneConfig(lanes), stats)
                assert stats["outer_steps"] == int(d[f"{name}/coo/steps_vla{lanes}"])
            else:
                y = sp.dispatch(m, x, "vla", sp.LaneConfig(lanes))
            ref = d[f"{name}/{fmt}/y_vla{lanes}"]
            assert bit_equal(y, ref), (fmt, lanes, first_diff(y, ref))


def test_canonical_kats_all_formats(sp):
    d = load_golden("canonical")
    for fmt in ("coo", "csr", "dia"):
        m = dev_matrix(sp, matrix_arrays(d, fmt), fmt)
        assert sp.dispatch(m, np.ones(5)).tolist() == [3.0, 14.0, 9.0, 21.0, 19.0]
        assert sp.dispatch(m, np.arange(1.0, 6.0)).tolist() == [7.0, 17.0, 32.0, 74.0, 68.0]
        for lanes in (1, 2, 4, 8, 16):
            y = sp.dispatch(m, np.arange(1.0, 6.0), "vla", sp.LaneConfig(lanes))
            assert bit_equal(y, d[f"{fmt}/ramp/y_vla{lanes}"])
        m32 = dev_matrix(sp, matrix_arrays(d, f"f32/{fmt}"), fmt)
        y = sp.dispatch(m32, np.arange(1.0, 6.0).astype(np.float32))
        assert y.dtype == np.float32 and bit_equal(y, d[f"f32/{fmt}/ramp/y_plain"])


def test_coo_vla_step_counts(sp):
    d = load_golden("canonical")
    row = dev_matrix(sp, matrix_arrays(d, "row20"), "coo")
    stats = {}
    y = sp.spmv_coo_vla(row, np.ones(20), sp.LaneConfig(4), stats)
    assert y.tolist() == [210.0] and stats["outer_steps"] == 5
    can = dev_matrix(sp, matrix_arrays(d, "coo"), "coo")
    for lanes, steps in ((4, 5), (1, 11), (8, 5)):
        stats = {}
        sp.spmv_coo_vla(can, np.ones(5), sp.LaneConfig(lanes), stats)
        assert stats["outer_steps"] == steps
    stats = {}
    sp.spmv_coo_vla(row, np.arange(20.0), sp.LaneConfig(8), stats)
    assert stats["outer_steps"] == 3


@pytest.mark.parametrize("name", ["pl64", "pl32", "plempty", "edges"])
def test_long_rows(sp, name):
    d = load_golden("long_rows")
    x = d[f"{name}/x"]
    csr_a = matrix_arrays(d, f"{name}/csr")
    lens = row_lengths(csr_a)
    tol = 1e-12 if csr_a["values"].dtype == np.float64 else 1e-5
    csr = dev_matrix(sp, csr_a, "csr")
    coo = dev_matrix(sp, matrix_arrays(d, f"{name}/coo"), "coo")
    for m, fmt in ((csr, "csr"), (coo, "coo")):
        y = sp.dispatch(m, x)
        ref = d[f"{name}/{fmt}/y_plain"]
        if tol == 1e-12:
            check_rowwise(y, ref, d[f"{name}/csr/y_vla32"], lens, tol, plan_tile(m))
        else:
            # fp32: against the reference evaluated in f64 on the f32 inputs
            from oracle import spmv_oracle as O
            r64 = O.csr_plain(len(lens), csr_a["row_pointers"], csr_a["col_indices"],
                              csr_a["values"].astype(np.float64), x.astype(np.float64))
            assert rel_err(y, r64) <= tol
            short = lens <= 32
            assert bit_equal(y[short], ref[short])
    for lanes in (1, 4, 32):
        y = sp.dispatch(csr, x, "vla", sp.LaneConfig(lanes))
        assert bit_equal(y, d[f"{name}/csr/y_vla{lanes}"]), lanes
    for lanes in (4, 32):
        stats = {}
        y = sp.spmv_coo_vla(coo, x, sp.LaneConfig(lanes), stats)
        assert bit_equal(y, d[f"{name}/coo/y_vla{lanes}"]) and stats["outer_steps"] == int(
            d[f"{name}/coo/steps_vla{lanes}"])


def test_repeat_is_deterministic(sp):
    d = load_golden("long_rows")
    csr = dev_matrix(sp, matrix_arrays(d, "edges/csr"), "csr")
    x = torch.from_numpy(d["edges/x"]).cuda()
    y0 = sp.spmv_csr_plain(csr, x)
    for _ in range(5):
        assert torch.equal(sp.spmv_csr_plain(csr, x), y0)


def test_unsorted_coo_storage_order(sp):
    """np.add.at sums in storage order; the plan's stable row sort keeps it."""
    from oracle import spmv_oracle as O
    rng = np.random.default_rng(3)
    n, nnz = 500, 6000
    rows = rng.integers(0, n, nnz)
    cols = rng.integers(0, n, nnz)  # duplicates allowed: plain COO does not care
    vals = rng.standard_normal(nnz)
    x = rng.uniform(-1, 1, n)
    m = sp.CooMatrix.from_arrays(n, n, rows, cols, vals)
    ref = O.coo_plain(n, rows, cols, vals, x)
    y = sp.spmv_coo_plain(m, x)
    lens = np.bincount(rows, minlength=n)
    short = lens <= 32
    assert bit_equal(y[short], ref[short])
    assert rel_err(y, ref) <= 1e-12


def test_empty_and_errors(sp):
    for fmt in ("coo", "csr", "dia"):
        empty = sp.to_format(sp.CooMatrix.from_arrays(6, 6, [], [], [], sorted=True), fmt)
        for version in ("plain", "vla"):
            assert sp.dispatch(empty, np.ones(6), version).tolist() == [0.0] * 6
    d = load_golden("canonical")
    for fmt in ("coo", "csr", "dia"):
        m = dev_matrix(sp, matrix_arrays(d, fmt), fmt)
        for version in ("plain", "vla"):
            with pytest.raises(sp.DimensionMismatch):
                sp.dispatch(m, np.ones(4), version)
            with pytest.raises(sp.DimensionMismatch):
                sp.dispatch(m, np.ones((5, 1)), version)
    unsorted = sp.CooMatrix.from_arrays(2, 2, [1, 0], [0, 1], [1.0, 2.0])
    with pytest.raises(sp.UnsortedInput):
        sp.spmv_coo_vla(unsorted, np.ones(2))
    assert sp.spmv_coo_plain(unsorted, np.ones(2)).tolist() == [2.0, 1.0]
    dia = sp.DiaMatrix(sp.MatrixShape(5, 5, 0), [5], np.zeros((8, 1)))
    assert sp.spmv_dia_plain(dia, np.arange(1.0, 6.0)).tolist() == [0.0] * 5


def test_large_empty_row_gaps(sp):
    """Rows with long empty stretches before, between and after them (the
    COO kernel pre-zeroes y instead of filling gaps per thread)."""
    n = 3_000_000
    rows = np.array([5, 5, 1_000_000, 1_000_000, 1_000_001, 2_000_000])
    cols = np.array([0, 7, 3, 4, 4, 9])
    vals = np.array([1.5, -2.0, 3.0, 0.25, -1.0, 4.0])
    x = np.arange(1.0, 11.0)
    want = np.zeros(n)
    np.add.at(want, rows, vals * x[cols])
    coo = sp.CooMatrix.from_arrays(n, 10, rows, cols, vals, sorted=True)
    for fmt in ("coo", "csr"):
        m = sp.to_format(coo, fmt)
        for version in ("plain", "vla"):
            y = sp.dispatch(m, x, version)
            assert bit_equal(y, want), (fmt, version)


def test_device_io_and_out(sp):
    d = load_golden("corpus")
    name = "stencil-8"
    m = dev_matrix(sp, matrix_arrays(d, f"{name}/csr"), "csr")
    x = torch.from_numpy(d[f"{name}/x"]).cuda()
    y = sp.spmv_csr_plain(m, x)
    assert y.is_cuda and y.dtype == torch.float64
    out = torch.empty_like(y)
    y2 = sp.spmv_csr_plain(m, x, out=out)
    assert y2 is out and torch.equal(out, y)
    # x cast to the value dtype (kernels.py:51-52)
    y3 = sp.spmv_csr_plain(m, x.float())
    assert bit_equal(y3.cpu().numpy(), sp.spmv_csr_plain(m, x.float().double()).cpu().numpy())


def test_registry_and_dispatch(sp):
    reg = sp.default_registry()
    assert len(reg.pairs()) == 6
    d = load_golden("canonical")
    can = dev_matrix(sp, matrix_arrays(d, "coo"), "coo")
    reg.unregister("coo", "vla")
    with pytest.raises(sp.UnsupportedCombination):
        sp.dispatch(can, np.ones(5), "vla", registry=reg)
    y = sp.dispatch(sp.DynamicMatrix.wrap(can), np.ones(5), sp.KernelVersion.VLA, sp.LaneConfig(8))
    assert y.tolist() == [3.0, 14.0, 9.0, 21.0, 19.0]


def test_linearity(sp):
    d = load_golden("corpus")
    name = "random-3"
    x1 = np.linspace(0.0, 1.0, 60)
    x2 = np.linspace(-2.0, 2.0, 60)
    for fmt in ("coo", "csr", "dia"):
        m = dev_matrix(sp, matrix_arrays(d, f"{name}/{fmt}"), fmt)
        for version in ("plain", "vla"):
            lhs = sp.dispatch(m, 0.6 * x1 - 1.2 * x2, version)
            rhs = 0.6 * sp.dispatch(m, x1, version) - 1.2 * sp.dispatch(m, x2, version)
            assert rel_err(lhs, rhs) <= 1e-10


def test_host_pipelined_products_match(sp):
    """Host x -> host y products are pipelined (x uploaded in column chunks,
    tile ranges launched as their x arrives, finished rows downloaded while
    later tiles run); the result must equal the device product bit for bit,
    also with long rows spanning tiles (y downloaded after the fix-up)."""
    from paper_2304_09511_b200 import kernels as K
    A = sp.gen_stencil27(48, 40, 36)
    xh = torch.rand(A.ncols, dtype=torch.float64).pin_memory()
    yh = torch.empty(A.nrows, dtype=torch.float64).pin_memory()
    ref = sp.spmv_csr_plain(A, xh.cuda()).cpu()
    assert torch.equal(sp.spmv_csr_plain(A, xh, out=yh), ref)
    dia = sp.to_format(A, "dia")
    yh2 = torch.empty_like(yh)
    assert torch.equal(sp.spmv_dia_plain(dia, xh, out=yh2), sp.spmv_dia_plain(dia, xh.cuda()).cpu())
    d = load_golden("long_rows")
    csr = dev_matrix(sp, matrix_arrays(d, "edges/csr"), "csr")
    x = torch.from_numpy(d["edges/x"])
    y_dev = sp.spmv_csr_plain(csr, x.cuda()).cpu()
    y3 = torch.empty(csr.nrows, dtype=torch.float64)
    assert torch.equal(sp.spmv_csr_plain(csr, x, out=y3), y_dev)


@pytest.mark.parametrize("fmt", ["csr", "coo", "dia"])
def test_numpy_host_products(sp, fmt):
    """The reference contract through the host pipeline (csrc/hostpipe.cuh):
    numpy x (pageable, and over pinned memory), list x, CPU tensor x, and a
    wrong-length x; y is a fresh numpy array equal bit for bit to the device
    product."""
    from paper_2304_09511_b200.plugin import gpu_kernel
    A = sp.gen_stencil27(40, 36, 30)
    m = {"csr": A, "coo": sp.csr_to_coo(A), "dia": sp.coo_to_dia(sp.csr_to_coo(A))}[fmt]
    x = np.random.default_rng(4).uniform(-1, 1, A.ncols)
    ref = sp.dispatch(m, torch.from_numpy(x).cuda()).cpu().numpy()
    fn = gpu_kernel(fmt, "plain")
    pinned = torch.from_numpy(x).pin_memory()
    for xh in (x, pinned.numpy(), x.tolist(), x.astype(np.float32)):
        y = fn(m, xh, None)
        assert isinstance(y, np.ndarray) and y.dtype == np.float64
        want = ref if np.asarray(xh).dtype == np.float64 else \
            sp.dispatch(m, torch.from_numpy(x.astype(np.float32).astype(np.float64)).cuda()).cpu().numpy()
        assert y.tobytes() == want.tobytes()
    yt = sp.dispatch(m, pinned)
    assert isinstance(yt, torch.Tensor) and not yt.is_cuda and torch.equal(yt, torch.from_numpy(ref))
    with pytest.raises(sp.DimensionMismatch):
        fn(m, x[:-1], None)
    # repeated calls reuse the pinned y blocks and the plan's pipe
    for _ in range(3):
        assert fn(m, x, None).tobytes() == ref.tobytes()
