"""A short fixed-seed run of the randomised parity sweep (tools/fuzz_parity.py):
random shapes and row-length mixes through CSR/COO plain and vla and DIA
(conversions + product) against the oracle."""

import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu
ROOT = Path(__file__).resolve().parents[1]


@pytest.mark.parametrize("seed", [101, 102])
def test_fuzz_parity(lib_built, seed):
    r = subprocess.run([sys.executable, str(ROOT / "tools" / "fuzz_parity.py"), "60", str(seed)], cwd=ROOT,
                       capture_output=True, text=True, timeout=600)
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-2000:]
