"""Sweep records and corpus inputs.

CPU tests pin the CSV text byte for byte against the reference's own output
(tests/golden/sweep.npz, made by tests/golden/make_golden.py), so GPU rows
load in the reference's report tooling.  GPU tests check the corpus
generators against the reference's arrays and run device sweeps."""

from __future__ import annotations

import io
import itertools

import numpy as np
import pytest

from _util import GOLDEN, bit_equal

import paper_2304_09511_b200 as sp
from paper_2304_09511_b200 import sweep as S
from paper_2304_09511_b200.formats import Format
from paper_2304_09511_b200.kernels import KernelVersion as V

G = np.load(GOLDEN / "sweep.npz")
NAMES = [str(n) for n in G["records/names"]]


def rec(mid, fmt, ver, median, nnz=10, status="ok"):
    return S.BenchRecord(mid, 4, 4, nnz, fmt, ver, 100, 10, median if status == "ok" else None,
                         0.5 if status == "ok" else None, None, status)


# ------------------------------------------------------------------ CPU --
@pytest.mark.parametrize("name", NAMES)
def test_csv_text_matches_reference(name):
    text = str(G[f"records/{name}/csv"])
    records = S.read_records(io.StringIO(text))
    buf = io.StringIO()
    S.write_records(records, buf)
    assert buf.getvalue() == text


def test_records_file_round_trip(tmp_path):
    records = [rec("m1", Format.CSR, V.PLAIN, 2e-3), rec("x", None, None, None, status="error")]
    S.write_records(records, tmp_path / "r.csv")
    assert S.read_records(tmp_path / "r.csv") == records


def test_compare_records():
    cpu = [rec("a", Format.CSR, V.PLAIN, 1.0), rec("a", Format.COO, V.PLAIN, 2.0),
           rec("b", Format.CSR, V.PLAIN, 4.0), rec("c", Format.CSR, V.PLAIN, 1.0)]
    gpu = [rec("a", Format.CSR, V.PLAIN, 0.01), rec("a", Format.COO, V.PLAIN, 0.01),
           rec("b", Format.CSR, V.PLAIN, 0.01), rec("b", Format.DIA, V.PLAIN, None, status="fill_exceeded")]
    c = S.compare_records(cpu, gpu)
    assert c.speedups[("a", Format.CSR, V.PLAIN)] == pytest.approx(100.0)
    assert c.geomeans[(Format.CSR, V.PLAIN)] == pytest.approx(200.0)
    assert c.unmatched == [("c", Format.CSR, V.PLAIN)]
    assert "geomean GPU speedup over CPU" in S.render_comparison(c)
    with pytest.raises(sp.EmptyInput):
        S.compare_records([], gpu)


def test_manifest_matches_reference(tmp_path):
    f = tmp_path / "m.txt"
    f.write_text(str(G["manifest/text"]))
    ents = sp.load_manifest(f)
    assert [e.id for e in ents] == [str(v) for v in G["manifest/ids"]]
    assert [e.source for e in ents] == [str(v) for v in G["manifest/sources"]]


@pytest.mark.parametrize("text", ["a\tb\na\tc\n", "lonely\n", "x\t\n"])
def test_manifest_errors(tmp_path, text):
    f = tmp_path / "m.txt"
    f.write_text(text)
    with pytest.raises(sp.ParseError):
        sp.load_manifest(f)


@pytest.mark.parametrize("src", ["stencil27:2,2", "stencil27:a,b,c", "banded:5", "random:5,0.1",
                                 "random:5,x,1", "banded:4,9"])
def test_load_entry_bad_specs(src):
    with pytest.raises(sp.ParseError):
        sp.load_entry(sp.CorpusEntry("e", src))


# ------------------------------------------------------------------ GPU --
@pytest.mark.gpu
@pytest.mark.parametrize("key", ["b12", "b9", "b1"])
def test_gen_banded_matches_reference(key):
    spec = G[f"banded/{key}/spec"].tolist()
    m = sp.gen_banded(spec[0], spec[1:])
    h = m.to_host()
    assert tuple(np.asarray(G[f"banded/{key}/shape"]).tolist()) == (m.nrows, m.ncols, m.nnz)
    assert np.array_equal(h["offsets"], G[f"banded/{key}/offsets"])
    assert bit_equal(h["values"], G[f"banded/{key}/values"])


@pytest.mark.gpu
@pytest.mark.parametrize("key", ["r20", "r7x13", "r0"])
def test_gen_random_matches_reference(key):
    nr, nc, dens, seed = G[f"random/{key}/spec"].tolist()
    m = sp.gen_random_sparse(int(nr), int(nc), dens, int(seed))
    h = m.to_host()
    assert m.nnz == int(G[f"random/{key}/shape"][2])
    assert np.array_equal(h["row_indices"], G[f"random/{key}/row_indices"])
    assert np.array_equal(h["col_indices"], G[f"random/{key}/col_indices"])
    assert bit_equal(h["values"], G[f"random/{key}/values"])


MM = "%%MatrixMarket matrix coordinate real general\n4 4 6\n1 1 2\n2 2 3\n3 1 -1\n3 3 4\n4 2 0.5\n4 4 5\n"


@pytest.mark.gpu
def test_run_corpus_on_gpu(tmp_path):
    (tmp_path / "small.mtx").write_text(MM)
    entries = [sp.CorpusEntry("mm", "small.mtx"), sp.CorpusEntry("cube", "stencil27:3,3,3"),
               sp.CorpusEntry("band", "banded:12,-2,0,1"), sp.CorpusEntry("rnd", "random:20,0.1,5"),
               sp.CorpusEntry("missing", "nope.mtx")]
    recs = S.run_corpus(entries, iterations=3, reps=2, base_dir=tmp_path)
    assert [r.matrix_id for r in recs[:6]] == ["mm"] * 6
    assert len(recs) == 4 * 6 + 1 and recs[-1].status == S.STATUS_ERROR
    ok = [r for r in recs if r.status == S.STATUS_OK]
    assert ok and all(r.gflops > 0 and r.median_seconds > 0 for r in ok)
    assert {r.status for r in recs} <= {S.STATUS_OK, S.STATUS_FILL, S.STATUS_ERROR}
    assert any(r.matrix_id == "rnd" and r.format == Format.DIA and r.status == S.STATUS_FILL for r in recs)
    par = S.run_corpus(entries, iterations=3, reps=2, base_dir=tmp_path, jobs=3)
    assert [(r.matrix_id, r.format, r.version, r.status) for r in par] == \
        [(r.matrix_id, r.format, r.version, r.status) for r in recs]
    buf, buf2 = io.StringIO(), io.StringIO()
    S.write_records(recs, buf)
    S.write_records(S.read_records(io.StringIO(buf.getvalue())), buf2)  # CSV rounds like the reference
    assert buf2.getvalue() == buf.getvalue()
    # the GPU rows set against themselves: every measured row matches
    c = S.compare_records(recs, recs)
    assert len(c.speedups) == len(ok) and all(v == 1.0 for v in c.speedups.values())


@pytest.mark.gpu
def test_run_corpus_tuned_plans(tmp_path):
    """tune_plans=True: each matrix/format gets its kernel configuration
    tuned first; the rows still cover every pair."""
    entries = [sp.CorpusEntry("cube", "stencil27:6,6,6"), sp.CorpusEntry("rnd", "random:300,0.05,5")]
    recs = S.run_corpus(entries, iterations=3, reps=2, tune_plans=True)
    assert len(recs) == 12 and all(r.status in (S.STATUS_OK, S.STATUS_FILL) for r in recs)


@pytest.mark.gpu
def test_run_corpus_injected_timer(tmp_path):
    """The reference's deterministic clock injection (helpers.CountingClock:
    each read advances 1 s), honoured like autotune.measure does."""
    class CountingClock:
        def __init__(self):
            self.t = 0.0

        def __call__(self):
            self.t += 1.0
            return self.t

    recs = S.run_corpus([sp.CorpusEntry("cube", "stencil27:2,2,2")], formats=[Format.CSR],
                        versions=[V.PLAIN], iterations=1, reps=3, timer=CountingClock())
    assert len(recs) == 1 and recs[0].median_seconds == 1.0
