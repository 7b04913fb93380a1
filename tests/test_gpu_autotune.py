"""Device-timed tuner: the reference's protocol and tie-breaks
(test_autotune.py), run on the GPU kernels."""

from types import SimpleNamespace

import numpy as np
import pytest

from _util import load_golden, matrix_arrays

pytestmark = pytest.mark.gpu


class CountingClock:  # tests/helpers.py:80-93
    def __init__(self):
        self.calls = 0

    def __call__(self):
        self.calls += 1
        return float(self.calls)


class ScriptedClock:  # tests/helpers.py:96-109
    def __init__(self, increments=(), default=1.0):
        self.pending, self.default, self.now, self.calls = list(increments), default, 0.0, 0

    def __call__(self):
        self.now += self.pending.pop(0) if self.pending else self.default
        self.calls += 1
        return self.now


def sample_schedule(durations, reps):
    out = []
    for d in durations:
        out.extend([0.0, d] * reps)
    return out


@pytest.fixture(scope="module")
def sp(lib_built):
    import paper_2304_09511_b200 as sp
    return sp


@pytest.fixture()
def canonical(sp):
    from test_gpu_kernels import dev_matrix
    return dev_matrix(sp, matrix_arrays(load_golden("canonical"), "coo"), "coo")


def test_protocol_and_ties(sp, canonical):
    from paper_2304_09511_b200.autotune import DEFAULT_CANDIDATES, measure, tune
    assert DEFAULT_CANDIDATES[0] == (sp.Format.CSR, sp.KernelVersion.PLAIN) and len(DEFAULT_CANDIDATES) == 6
    clock = CountingClock()
    m = measure(canonical, "coo", "plain", iterations=3, reps=4, timer=clock)
    assert clock.calls == 8 and m.samples == [1.0] * 4
    clock = ScriptedClock(sample_schedule([1e-3], 1) + sample_schedule([2e-3], 1) + sample_schedule([3e-3], 1))
    m = measure(canonical, "csr", "plain", iterations=1, reps=3, timer=clock, matrix_id="canon")
    assert m.median_seconds == pytest.approx(2e-3) and m.matrix_id == "canon"
    durations = [5.0, 3.0, 4.0, 6.0, 2.0, 7.0]
    choice = tune(canonical, iterations=1, reps=1, timer=ScriptedClock(sample_schedule(durations, 1)))
    assert (choice.format, choice.version) == (sp.Format.COO, sp.KernelVersion.VLA)
    tie = tune(canonical, iterations=1, reps=1, timer=CountingClock())
    assert (tie.format, tie.version) == (sp.Format.CSR, sp.KernelVersion.PLAIN)
    with pytest.raises(ValueError):
        measure(canonical, "csr", "plain", iterations=0)


def test_skips_and_failures(sp):
    from paper_2304_09511_b200.autotune import distribution_report, tune
    rng = np.random.default_rng(1)
    flat = rng.choice(3600, 180, replace=False)
    m = sp.CooMatrix.from_arrays(60, 60, flat // 60, flat % 60, rng.uniform(-1, 1, 180), sorted=True)
    choice = tune(m, iterations=1, reps=1, timer=CountingClock())
    assert choice.format == sp.Format.CSR and len(choice.candidates) == 4
    assert all("fill" in reason for _, _, reason in choice.skipped)
    with pytest.raises(sp.SparseError):
        tune(m, [("dia", "plain")], iterations=1, reps=1, timer=CountingClock())
    rep = distribution_report([SimpleNamespace(version="plain", format="csr"),
                               SimpleNamespace(version="plain", format="dia")])
    assert rep[sp.KernelVersion.PLAIN][sp.Format.CSR] == 50.0


def test_device_timing_picks_dia_on_stencil(sp):
    """With real device timings the stencil's DIA beats CSR and COO
    (fewer bytes per SpMV: SURVEY.md §8(d))."""
    from paper_2304_09511_b200.autotune import tune
    A = sp.gen_stencil27(96, 96, 96)
    choice = tune(A, [("csr", "plain"), ("coo", "plain"), ("dia", "plain")], iterations=20, reps=3)
    assert choice.format == sp.Format.DIA
    assert all(m.gflops > 0 for m in choice.candidates)
