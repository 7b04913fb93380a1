"""Both whole-matrix CSR/COO kernels on every parity case.

Plans pick the warp-stream kernel (csrc/wstream.cuh) for matrices with rows
or runs over 32 entries and the tile kernel otherwise.  The knobs are read
once per process, so the corpus, stress and tail-tile parity tests re-run in
child processes with the choice forced each way (SPMV_CSR_WS / SPMV_COO_WS),
the warp-stream runs with 64 ranges per warp so that long rows split across
many ranges and the fix-up path carries most of them.
"""

import os
import subprocess
import sys
from pathlib import Path

import pytest

pytestmark = pytest.mark.gpu

ROOT = Path(__file__).resolve().parents[1]
TESTS = [
    "tests/test_gpu_kernels.py::test_corpus_all_kernels",
    "tests/test_gpu_kernels.py::test_canonical_kats_all_formats",
    "tests/test_gpu_kernels.py::test_long_rows",
    "tests/test_gpu_stress.py::test_random_structures_csr_coo",
    "tests/test_gpu_stress.py::test_tail_tiles_and_unaligned_pointers",
    "tests/test_gpu_stress.py::test_unsorted_coo_duplicates_at_scale",
    "tests/test_dist.py::test_emulated_ranks_bit_identical",          # x windows (col_base > 0)
    "tests/test_dist.py::test_emulated_ranks_random_matrix_allgather",
]


@pytest.mark.parametrize("env", [
    {"SPMV_CSR_WS": "1", "SPMV_COO_WS": "1", "SPMV_WS_RANGES": "64"},
    {"SPMV_CSR_WS": "1", "SPMV_COO_WS": "1", "SPMV_WS_RANGES": "1"},
    {"SPMV_CSR_WS": "0", "SPMV_COO_WS": "0"},
], ids=["ws_r64", "ws_r1", "tiles"])
def test_forced_kernel_choice(lib_built, env):
    e = dict(os.environ, **env)
    r = subprocess.run([sys.executable, "-m", "pytest", "-x", "-q", "-p", "no:cacheprovider", *TESTS],
                       cwd=ROOT, env=e, capture_output=True, text=True, timeout=900)
    assert r.returncode == 0, r.stdout[-4000:] + r.stderr[-2000:]
