"""The reference's own drivers running the GPU kernels.

The plugin exists so that the reference's drivers run unchanged with
`registry=register_gpu_kernels(spmvkit.kernels.KernelRegistry())`:
`dispatch` (kernels.py:286-297), `autotune.measure` / `tune`
(autotune.py:60-64, :110-114), `hpcg.distributed_spmv` / `cg_solve`
(hpcg.py:167-169, :211-213) and `bench.run_corpus` (bench.py:149-154).
These tests drive them with the reference's real containers (built by its
own generators and conversions) from the installed reference package
(`baseline/_ref`, `pip install --target baseline/_ref` of /root/reference,
git-ignored, shipped to the GPU box with the repo snapshot) and compare
with the same drivers on the reference's CPU kernels.  Skipped only when
that install is absent.
"""

import sys
from pathlib import Path

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

REF = Path(__file__).resolve().parents[1] / "baseline" / "_ref"


@pytest.fixture(scope="module")
def ref():
    if not (REF / "spmvkit" / "__init__.py").exists():
        pytest.skip("reference package not installed in baseline/_ref")
    sys.path.insert(0, str(REF))
    import spmvkit
    return spmvkit


@pytest.fixture(scope="module")
def reg(ref, lib_built):
    from paper_2304_09511_b200.plugin import register_gpu_kernels
    from spmvkit.kernels import KernelRegistry
    return register_gpu_kernels(KernelRegistry())


def _rel(a, b):
    a, b = np.asarray(a, dtype=np.float64), np.asarray(b, dtype=np.float64)
    return float(np.max(np.abs(a - b) / np.maximum(np.abs(b), 1.0))) if a.size else 0.0


def test_dispatch_all_formats_and_versions(ref, reg):
    from spmvkit.convert import to_format
    from spmvkit.kernels import dispatch
    from spmvkit.lanes import LaneConfig
    from spmvkit.matrixio import gen_stencil27
    csr = gen_stencil27(9, 7, 8)
    x = np.random.default_rng(3).uniform(-1, 1, csr.shape.ncols)
    for fmt in ("csr", "coo", "dia"):
        m = to_format(csr, fmt)
        for version, cfg in (("plain", None), ("vla", LaneConfig(8)), ("vla", LaneConfig(3))):
            y_gpu = dispatch(m, x, version, cfg, registry=reg)
            y_cpu = dispatch(m, x, version, cfg)
            assert isinstance(y_gpu, np.ndarray) and y_gpu.dtype == y_cpu.dtype
            assert y_gpu.tobytes() == y_cpu.tobytes(), (fmt, version)


def test_autotune_measure_and_tune(ref, reg):
    from spmvkit.autotune import measure, tune
    from spmvkit.matrixio import gen_stencil27
    csr = gen_stencil27(12, 12, 12)
    m = measure(csr, "csr", "plain", iterations=3, reps=2, registry=reg, matrix_id="s12")
    assert m.gflops > 0 and len(m.samples) == 2 and m.matrix_id == "s12"
    choice = tune(csr, iterations=2, reps=2, registry=reg)
    assert len(choice.candidates) == 6 and not choice.skipped
    assert choice.median_seconds == min(c.median_seconds for c in choice.candidates)


def test_hpcg_distributed_spmv_and_cg(ref, reg):
    from spmvkit.hpcg import ProblemSpec, build_problem, cg_solve, distributed_spmv, gather_global, halo_exchange
    spec = ProblemSpec(6, 5, 4, 1, 1, 3)
    ranks = build_problem(spec)
    rng = np.random.default_rng(8)
    for r in ranks:
        r.x_local = rng.uniform(-1, 1, r.x_local.shape[0])
    halo_exchange(ranks)
    y_gpu = gather_global(ranks, distributed_spmv(ranks, registry=reg))
    y_cpu = gather_global(ranks, distributed_spmv(ranks))
    assert _rel(y_gpu, y_cpu) == 0.0
    s_gpu = cg_solve(build_problem(spec), tol=1e-9, registry=reg)
    s_cpu = cg_solve(build_problem(spec), tol=1e-9)
    assert s_gpu.iterations == s_cpu.iterations
    assert _rel(s_gpu.residual_norms, s_cpu.residual_norms) <= 1e-12


def test_bench_run_corpus(ref, reg, tmp_path):
    from spmvkit.bench import make_report, render_report, run_corpus
    from spmvkit.matrixio import CorpusEntry
    entries = [CorpusEntry("cube", "stencil27:5,5,5"), CorpusEntry("band", "banded:40,-2,0,1"),
               CorpusEntry("rnd", "random:30,0.1,7")]
    recs = run_corpus(entries, iterations=2, reps=2, registry=reg, base_dir=tmp_path)
    assert len(recs) == 18
    ok = [r for r in recs if r.status == "ok"]
    assert ok and all(r.gflops > 0 for r in ok)
    text = render_report(make_report(recs))
    assert "baseline: csr/plain" in text
