"""Generate golden vectors by running the reference package itself.

Run in the build container (where /root/reference exists):
    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

It imports `spmvkit` from /root/reference/pkg/src (read-only) plus the
reference test helpers (/root/reference/pkg/tests/helpers.py, for the
fixture corpus and its Matrix Market files), evaluates the reference's own
kernels and conversions, and writes small .npz fixtures next to this file.
Those fixtures travel to the GPU box; /root/reference does not.

Files written:
  corpus.npz      the reference test corpus (>= 30 matrices) in all three
                  formats + plain/vla outputs on probe vectors
  canonical.npz   the 5x5 canonical matrix, KAT vectors, vla step counts
  long_rows.npz   power-law rows up to 3000 entries (long-row paths)
  convert.npz     sort_coo / coo_to_csr / csr_to_coo / coo_to_dia / dia_to_coo
                  edge cases (duplicates, signed zeros, NaN, unsorted cols)
  reduceat.npz    np.add.reduceat segments (pins the pairwise-sum model)
  stencil.npz     gen_stencil27 on small grids
  cg.npz          hpcg.cg_solve: iterations, residual histories, solutions
  mm.npz          read_matrix_market on small hand-written files
  sweep.npz       bench.py CSV records and reports, corpus manifest parsing,
                  gen_banded / gen_random_sparse generator specs
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF_SRC = Path("/root/reference/pkg/src")
REF_TESTS = Path("/root/reference/pkg/tests")
OUT = Path(__file__).resolve().parent

sys.dont_write_bytecode = True
sys.path.insert(0, str(REF_SRC))
sys.path.insert(0, str(REF_TESTS))

from spmvkit.convert import (  # noqa: E402
    DiaFillPolicy, coo_to_csr, coo_to_dia, csr_to_coo, dia_to_coo, sort_coo, to_format)
from spmvkit.formats import CooMatrix, CsrMatrix, DiaMatrix, Format, MatrixShape  # noqa: E402
from spmvkit.kernels import (  # noqa: E402
    spmv_coo_plain, spmv_coo_vla, spmv_csr_plain, spmv_csr_vla, spmv_dia_plain, spmv_dia_vla)
from spmvkit.lanes import LaneConfig  # noqa: E402
from spmvkit.matrixio import gen_stencil27  # noqa: E402

import helpers  # noqa: E402  (reference test helpers: corpus + canonical)

LOOSE = DiaFillPolicy(max_fill_ratio=float("inf"))
VLA_LANES = (1, 2, 3, 4, 8, 16, 32, 64)


def put_matrix(d: dict, key: str, m) -> None:
    d[f"{key}/shape"] = np.array([m.shape.nrows, m.shape.ncols, m.shape.nnz], dtype=np.int64)
    if isinstance(m, CooMatrix):
        d[f"{key}/row_indices"] = m.row_indices
        d[f"{key}/col_indices"] = m.col_indices
        d[f"{key}/values"] = m.values
        d[f"{key}/sorted"] = np.array(bool(m.sorted))
    elif isinstance(m, CsrMatrix):
        d[f"{key}/row_pointers"] = m.row_pointers
        d[f"{key}/col_indices"] = m.col_indices
        d[f"{key}/values"] = m.values
    else:
        d[f"{key}/offsets"] = m.offsets
        d[f"{key}/values"] = m.values


def kernel_outputs(d: dict, key: str, fmt: Format, m, x) -> None:
    plain = {Format.COO: spmv_coo_plain, Format.CSR: spmv_csr_plain, Format.DIA: spmv_dia_plain}[fmt]
    vla = {Format.COO: spmv_coo_vla, Format.CSR: spmv_csr_vla, Format.DIA: spmv_dia_vla}[fmt]
    d[f"{key}/y_plain"] = plain(m, x)
    for lanes in VLA_LANES:
        if fmt == Format.COO:
            stats = {}
            d[f"{key}/y_vla{lanes}"] = vla(m, x, LaneConfig(lanes), stats)
            d[f"{key}/steps_vla{lanes}"] = np.array(stats["outer_steps"], dtype=np.int64)
        else:
            d[f"{key}/y_vla{lanes}"] = vla(m, x, LaneConfig(lanes))


def make_corpus() -> None:
    d: dict = {}
    names = []
    for salt, (name, matrix) in enumerate(helpers.build_corpus()):
        names.append(name)
        # probe_x of test_acceptance.py:66-68
        x = np.random.default_rng(salt).uniform(-1.0, 1.0, size=matrix.shape.ncols)
        d[f"{name}/x"] = x
        for fmt in Format:
            m = to_format(matrix, fmt, LOOSE)
            put_matrix(d, f"{name}/{fmt.value}", m)
            kernel_outputs(d, f"{name}/{fmt.value}", fmt, m, x)
        # the as-given container too (some corpus COOs are unsorted/duplicated)
        put_matrix(d, f"{name}/orig", matrix)
    d["names"] = np.array(names)
    np.savez_compressed(OUT / "corpus.npz", **d)


def make_canonical() -> None:
    d: dict = {}
    can = helpers.canonical_coo()
    for fmt in Format:
        m = to_format(can, fmt)
        put_matrix(d, fmt.value, m)
        for xname, x in (("ones", np.ones(5)), ("ramp", np.arange(1.0, 6.0))):
            kernel_outputs(d, f"{fmt.value}/{xname}", fmt, m, x)
    can32 = helpers.canonical_coo(dtype=np.float32)
    for fmt in Format:
        m = to_format(can32, fmt)
        put_matrix(d, f"f32/{fmt.value}", m)
        kernel_outputs(d, f"f32/{fmt.value}/ramp", fmt, m, np.arange(1.0, 6.0).astype(np.float32))
    # single-row step-count fixture (test_kernels.py:95-120)
    row = CooMatrix.from_arrays(1, 20, [0] * 20, range(20), np.arange(1.0, 21.0), sorted=True)
    put_matrix(d, "row20", row)
    kernel_outputs(d, "row20/ones", Format.COO, row, np.ones(20))
    kernel_outputs(d, "row20/arange", Format.COO, row, np.arange(20.0))
    np.savez_compressed(OUT / "canonical.npz", **d)


def power_law_csr(nrows, ncols, seed, max_len, dtype=np.float64, empty_every=0):
    rng = np.random.default_rng(seed)
    lens = np.minimum(rng.zipf(1.6, size=nrows), max_len)
    if empty_every:
        lens[::empty_every] = 0
    cols = []
    for ln in lens:
        c = np.sort(rng.choice(ncols, size=int(ln), replace=False))
        cols.append(c)
    irp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    aj = np.concatenate(cols) if cols else np.zeros(0, dtype=np.int64)
    av = rng.uniform(-1.0, 1.0, size=aj.shape[0]).astype(dtype)
    return CsrMatrix.from_arrays(nrows, ncols, irp, aj, av)


def make_long_rows() -> None:
    d: dict = {}
    cases = {
        "pl64": power_law_csr(600, 5000, 11, 3000),
        "pl32": power_law_csr(600, 5000, 12, 3000, dtype=np.float32),
        "plempty": power_law_csr(300, 4000, 13, 2500, empty_every=7),
    }
    # rows straddling the 32-entry exact threshold and chunk boundaries
    lens = np.array([31, 32, 33, 0, 1, 64, 2047, 2048, 2049, 4096, 4097, 5, 32, 33, 0, 6000])
    rng = np.random.default_rng(99)
    cols = [np.sort(rng.choice(7000, size=int(n), replace=False)) for n in lens]
    irp = np.zeros(lens.shape[0] + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    aj = np.concatenate(cols)
    cases["edges"] = CsrMatrix.from_arrays(lens.shape[0], 7000, irp, aj, rng.uniform(-1, 1, aj.shape[0]))
    names = []
    for name, csr in cases.items():
        names.append(name)
        x = np.random.default_rng(5).uniform(-1.0, 1.0, csr.shape.ncols).astype(csr.values.dtype)
        d[f"{name}/x"] = x
        put_matrix(d, f"{name}/csr", csr)
        d[f"{name}/csr/y_plain"] = spmv_csr_plain(csr, x)
        for lanes in (1, 4, 32):
            d[f"{name}/csr/y_vla{lanes}"] = spmv_csr_vla(csr, x, LaneConfig(lanes))
        coo = csr_to_coo(csr)
        put_matrix(d, f"{name}/coo", coo)
        d[f"{name}/coo/y_plain"] = spmv_coo_plain(coo, x)
        for lanes in (4, 32):
            stats = {}
            d[f"{name}/coo/y_vla{lanes}"] = spmv_coo_vla(coo, x, LaneConfig(lanes), stats)
            d[f"{name}/coo/steps_vla{lanes}"] = np.array(stats["outer_steps"])
    d["names"] = np.array(names)
    np.savez_compressed(OUT / "long_rows.npz", **d)


def make_convert() -> None:
    d: dict = {}
    rng = np.random.default_rng(2024)
    # unsorted COO with duplicate runs of many lengths (pairwise paths: <8,
    # <=128, >128), signed zeros and exact cancellations
    n = 64
    rows, cols, vals = [], [], []
    for run in (1, 2, 3, 7, 8, 9, 15, 16, 17, 100, 128, 129, 200, 300, 1000):
        r, c = rng.integers(0, n), rng.integers(0, n)
        rows += [r] * run
        cols += [c] * run
        vals += list(rng.standard_normal(run) * 10.0 ** rng.integers(-4, 12, run))
    for _ in range(40):
        rows.append(rng.integers(0, n))
        cols.append(rng.integers(0, n))
        vals.append(rng.standard_normal())
    rows += [3, 3, 5, 5, 5]
    cols += [60, 60, 61, 61, 61]
    vals += [-0.0, -0.0, 2.0, -2.0, -0.0]
    perm = rng.permutation(len(rows))
    for dt in (np.float64, np.float32):
        coo = CooMatrix.from_arrays(n, n, np.array(rows)[perm], np.array(cols)[perm],
                                    np.array(vals, dtype=dt)[perm])
        key = f"dups_{np.dtype(dt).name}"
        put_matrix(d, f"{key}/in", coo)
        put_matrix(d, f"{key}/sorted", sort_coo(coo))
    # csr with an unsorted row
    csr = CsrMatrix.from_arrays(3, 4, [0, 2, 2, 5], [1, 3, 0, 2, 1], [1.0, 2.0, 3.0, 4.0, 5.0])
    put_matrix(d, "csr_unsorted/in", csr)
    put_matrix(d, "csr_unsorted/coo", csr_to_coo(csr))
    # dia with stored zeros, -0.0, NaN and out-of-bounds padding
    vals = np.zeros((8, 3))
    vals[0, 0] = 1.0
    vals[1, 1] = -0.0
    vals[2, 1] = np.nan
    vals[3, 2] = 4.0
    vals[4, 0] = -5.0
    dia = DiaMatrix(MatrixShape(6, 7, 4), [-1, 0, 2], vals)
    put_matrix(d, "dia_special/in", dia)
    put_matrix(d, "dia_special/coo", dia_to_coo(dia))
    # random sorted COO -> CSR / DIA
    coo = sort_coo(CooMatrix.from_arrays(
        40, 50, rng.integers(0, 40, 300), rng.integers(0, 50, 300), rng.standard_normal(300)))
    put_matrix(d, "rand/coo", coo)
    put_matrix(d, "rand/csr", coo_to_csr(coo))
    put_matrix(d, "rand/dia", coo_to_dia(coo, LOOSE))
    # COO flagged sorted whose rows are not: coo_to_csr trusts the flag and
    # builds row pointers from counts (bincount + cumsum, convert.py:92-93)
    flat = np.random.default_rng(1).choice(3600, 180, replace=False)
    mis = CooMatrix.from_arrays(60, 60, flat // 60, flat % 60, np.linspace(-1.0, 1.0, 180), sorted=True)
    put_matrix(d, "misflagged/coo", mis)
    put_matrix(d, "misflagged/csr", coo_to_csr(mis))
    np.savez_compressed(OUT / "convert.npz", **d)


def make_reduceat() -> None:
    d: dict = {}
    rng = np.random.default_rng(7)
    for dt in (np.float64, np.float32):
        lens = rng.integers(1, 700, size=60)
        a = (rng.standard_normal(lens.sum()) * 10.0 ** rng.integers(-3, 13, lens.sum())).astype(dt)
        idx = np.zeros(lens.shape[0], dtype=np.int64)
        np.cumsum(lens[:-1], out=idx[1:])
        name = np.dtype(dt).name
        d[f"{name}/a"] = a
        d[f"{name}/idx"] = idx
        d[f"{name}/out"] = np.add.reduceat(a, idx)
    np.savez_compressed(OUT / "reduceat.npz", **d)


def make_stencil() -> None:
    d: dict = {}
    dims = [(1, 1, 1), (2, 2, 2), (2, 3, 4), (4, 4, 4), (5, 3, 1), (8, 8, 8), (16, 16, 4)]
    for dims_ in dims:
        key = "x".join(map(str, dims_))
        m = gen_stencil27(*dims_)
        put_matrix(d, key, m)
        x = np.random.default_rng(1).uniform(-1, 1, m.shape.ncols)
        d[f"{key}/x"] = x
        d[f"{key}/y"] = spmv_csr_plain(m, x)
    d["dims"] = np.array(dims, dtype=np.int64)
    np.savez_compressed(OUT / "stencil.npz", **d)


MM_TEXTS = {
    "general_dups": "%%MatrixMarket matrix coordinate real general\n% comment\n4 5 7\n1 1 1.5\n3 2 -2.25\n"
                    "1 1 0.125\n4 5 1e-3\n2 3 7\n3 2 2.25\n1 4 -0.0\n",
    "symmetric": "%%MatrixMarket matrix coordinate real symmetric\n5 5 6\n1 1 4\n2 1 -1\n3 2 -1.5\n"
                 "5 3 0.5\n4 4 3.25\n5 5 2\n",
    "skew": "%%MatrixMarket matrix coordinate real skew-symmetric\n4 4 3\n2 1 1.5\n3 1 -2\n4 3 0.75\n",
    "pattern": "%%MatrixMarket matrix coordinate pattern general\n3 6 4\n1 6\n3 1\n2 2\n1 1\n",
    "integer_sym": "%%MatrixMarket matrix coordinate integer symmetric\n% x\n\n3 3 4\n1 1 2\n2 1 -3\n"
                   "3 1 5\n3 3 -7\n",
    "empty": "%%MatrixMarket matrix coordinate real general\n3 4 0\n",
}


def make_mm() -> None:
    """matrixio.read_matrix_market on small hand-written files."""
    from spmvkit.matrixio import read_matrix_market
    d: dict = {}
    for name, text in MM_TEXTS.items():
        d[f"{name}/text"] = np.array(text)
        put_matrix(d, f"{name}/coo", read_matrix_market(text.encode()))
    d["names"] = np.array(list(MM_TEXTS))
    np.savez_compressed(OUT / "mm.npz", **d)


def make_cg() -> None:
    """hpcg.cg_solve runs (acceptance criterion 06, test_hpcg.py:108-158)."""
    from spmvkit.hpcg import ProblemSpec, build_problem, cg_solve, gather_global
    d: dict = {}
    for key, spec, tol, iters in (("p16", ProblemSpec(16, 16, 16), 1e-9, 200),
                                  ("p16_split", ProblemSpec(8, 16, 16, 2, 1, 1), 1e-9, 200),
                                  ("p8", ProblemSpec(8, 8, 8), 1e-9, 200),
                                  ("p2", ProblemSpec(2, 2, 2), 1e-10, 20)):
        ranks = build_problem(spec)
        st = cg_solve(ranks, tol=tol, max_iters=iters)
        d[f"{key}/dims"] = np.array(spec.global_dims, dtype=np.int64)
        d[f"{key}/iterations"] = np.array(st.iterations)
        d[f"{key}/norms"] = np.asarray(st.residual_norms, dtype=np.float64)
        d[f"{key}/converged"] = np.array(st.converged)
        d[f"{key}/x"] = gather_global(ranks, st.x_parts)
        d[f"{key}/b"] = gather_global(ranks, [rs.b_local for rs in ranks])
    np.savez_compressed(OUT / "cg.npz", **d)


SWEEP_MANIFEST = ("# corpus\n"
                  "canon\tgeneral.mtx\n"
                  "cube  stencil27:2,2,3\n"
                  "\n"
                  "band\tbanded:12,-2,0,1\n"
                  "rnd\trandom:20,0.1,5\n")


def _sweep_records():
    from spmvkit.bench import BenchRecord
    from spmvkit.kernels import KernelVersion as V
    C, O, D = Format.CSR, Format.COO, Format.DIA
    P, L = V.PLAIN, V.VLA

    def rec(mid, fmt, ver, median, nnz=10, status="ok"):
        return BenchRecord(mid, 4, 4, nnz, fmt, ver, 100, 10, median if status == "ok" else None,
                           (2.0 * nnz * 100 / median / 1e9) if status == "ok" else None, None, status)

    return {
        "basic": [rec("m1", C, P, 2e-3), rec("m1", O, P, 1e-3), rec("m2", C, P, 2e-3), rec("m2", O, P, 4e-3),
                  rec("m2", D, P, None, status="fill_exceeded")],
        "mixed": [rec("a", C, P, 3.25e-4, nnz=27), rec("a", O, P, 2.5e-4, nnz=27), rec("a", D, P, 1.5e-4, nnz=27),
                  rec("a", C, L, 9e-4, nnz=27), rec("a", O, L, 8e-4, nnz=27), rec("a", D, L, 7e-4, nnz=27),
                  rec("b", C, P, 1e-3, nnz=5), rec("b", O, P, 1e-3, nnz=5),
                  rec("b", D, P, None, nnz=5, status="unsupported"),
                  rec("b", C, L, 2e-3, nnz=5), rec("gone", None, None, None, status="error")],
        "missing_pair": [rec("m1", C, P, 2e-3), rec("m1", O, P, 1e-3), rec("m2", C, P, 2e-3)],
    }


def make_sweep() -> None:
    """bench.py records, CSV text and reports; matrixio manifest and
    generator specs."""
    import io

    from spmvkit.bench import make_report, render_report, write_records
    from spmvkit.kernels import KernelVersion as V
    from spmvkit.matrixio import gen_banded, gen_random_sparse, load_manifest
    d: dict = {}
    for name, records in _sweep_records().items():
        buf = io.StringIO()
        write_records(records, buf)
        d[f"records/{name}/csv"] = np.array(buf.getvalue())
        for bname, base in (("csr_plain", (Format.CSR, V.PLAIN)), ("coo_vla", (Format.COO, V.VLA))):
            try:
                d[f"records/{name}/report_{bname}"] = np.array(render_report(make_report(records, base)))
            except Exception as exc:  # MissingBaseline / EmptyInput
                d[f"records/{name}/report_{bname}"] = np.array(f"raises {type(exc).__name__}")
    d["records/names"] = np.array(list(_sweep_records()))
    import tempfile
    with tempfile.TemporaryDirectory() as tmp:
        mf = Path(tmp) / "m.txt"
        mf.write_text(SWEEP_MANIFEST)
        ents = load_manifest(mf)
    d["manifest/text"] = np.array(SWEEP_MANIFEST)
    d["manifest/ids"] = np.array([e.id for e in ents])
    d["manifest/sources"] = np.array([e.source for e in ents])
    for key, (n, offs) in {"b12": (12, (-2, 0, 1)), "b9": (9, (3, -4, 0, 3)), "b1": (1, (0,))}.items():
        put_matrix(d, f"banded/{key}", gen_banded(n, offs))
        d[f"banded/{key}/spec"] = np.array([n, *offs], dtype=np.int64)
    for key, (nr, nc, dens, seed) in {"r20": (20, 20, 0.1, 5), "r7x13": (7, 13, 0.3, 11),
                                      "r0": (6, 6, 0.0, 1)}.items():
        put_matrix(d, f"random/{key}", gen_random_sparse(nr, nc, dens, seed))
        d[f"random/{key}/spec"] = np.array([nr, nc, dens, seed], dtype=np.float64)
    np.savez_compressed(OUT / "sweep.npz", **d)


if __name__ == "__main__":
    os.environ.setdefault("PYTHONDONTWRITEBYTECODE", "1")
    make_sweep()
    make_mm()
    make_cg()
    make_canonical()
    make_convert()
    make_reduceat()
    make_stencil()
    make_long_rows()
    make_corpus()
    for f in sorted(OUT.glob("*.npz")):
        print(f.name, f.stat().st_size)
