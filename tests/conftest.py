import sys
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
sys.path.insert(0, str(ROOT))
sys.path.insert(0, str(Path(__file__).resolve().parent))


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (B200, sm_100a)")
    config.addinivalue_line("markers", "slow: large (BASELINE.json full-size) configurations")


def pytest_collection_modifyitems(config, items):
    # GPU tests are skipped (not failed) when collected on a CPU-only box
    # without an explicit -m gpu; with -m gpu and no device they fail loudly.
    try:
        import torch
        has_gpu = torch.cuda.is_available()
    except Exception:  # pragma: no cover
        has_gpu = False
    if has_gpu:
        return
    markexpr = config.getoption("-m") or ""
    if "gpu" in markexpr and "not gpu" not in markexpr:
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for item in items:
        if "gpu" in item.keywords:
            item.add_marker(skip)


@pytest.fixture(scope="session")
def golden():
    from _util import load_golden
    return load_golden


@pytest.fixture(scope="session")
def lib_built():
    """Build libspmv_b200.so in-tree (cheap when up to date)."""
    from paper_2304_09511_b200 import _build
    return _build.build()


def pytest_sessionfinish(session, exitstatus):
    """Debug-library runs (SPMV_DEBUG_CHECKS=1 with SPMV_B200_LIB pointing at
    libspmv_b200_debug.so): the device-side check counters must be zero."""
    import os
    if os.environ.get("SPMV_DEBUG_CHECKS") != "1":
        return
    import ctypes

    from paper_2304_09511_b200 import _lib
    c = (ctypes.c_ulonglong * 4)()
    _lib.call("spmv_debug_check_counts", c)
    counts = list(c)
    print(f"\ndebug check counters (stage mismatch, index range, x panel, other): {counts}")
    if any(counts):
        session.exitstatus = 1
