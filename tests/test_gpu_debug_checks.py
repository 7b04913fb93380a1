"""Device-side consistency checks in place of compute-sanitizer (closed on
this pool: profiles/r2_compute_sanitizer_closed.log).

libspmv_b200_debug.so (`_build.build(debug=True)`, -DSPMV_DEBUG_CHECKS)
compares every TMA-staged tile (CSR, COO, DIA rings, with G consumer groups
sharing G + 1 stages), every panel-path warp stage and x panel with global
memory after its barrier completes — a ring race or stale stage shows up as
a mismatch — and bounds-checks the panel path's columns.  These tests run
parity suites in child processes on that library and require every counter
to be zero (the children also check their results against the oracle).
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]


@pytest.fixture(scope="module")
def debug_env():
    from paper_2304_09511_b200 import _build
    lib = _build.build(debug=True)  # incremental: a no-op when up to date
    return dict(os.environ, SPMV_B200_LIB=str(lib), SPMV_DEBUG_CHECKS="1")


def test_sanitize_cases_under_debug_checks(debug_env):
    r = subprocess.run([sys.executable, "tools/sanitize_cases.py"], cwd=ROOT, env=debug_env, capture_output=True,
                       text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert "debug check counters" in r.stdout and "[0, 0, 0, 0]" in r.stdout


@pytest.mark.parametrize("suite", [
    "tests/test_gpu_kernels.py::test_corpus_all_kernels",
    "tests/test_gpu_stress.py",
    "tests/test_gpu_panel.py",
    "tests/test_dist.py",
])
def test_parity_suites_under_debug_checks(debug_env, suite):
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", "-s", suite],
                       cwd=ROOT, env=debug_env, capture_output=True, text=True, timeout=1800)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
    assert "debug check counters (stage mismatch, index range, x panel, other): [0, 0, 0, 0]" in r.stdout
