"""The C-ABI library: builds for sm_100a, loads without a GPU, exports every
symbol include/spmv_b200.h declares, maps status codes onto the reference's
exception classes.  CPU only: no call here reaches a CUDA kernel."""

import ctypes
import re
import subprocess
from pathlib import Path

import pytest

ROOT = Path(__file__).resolve().parent.parent
HEADER = ROOT / "include" / "spmv_b200.h"


def declared_functions() -> list:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(spmv_[a-z0-9_]+)\s*\(", text)))


def test_header_lists_entry_points():
    names = declared_functions()
    for must in ("spmv_csr", "spmv_coo", "spmv_dia", "spmv_csr_vla", "spmv_coo_vla", "spmv_coo_to_csr",
                 "spmv_csr_to_coo", "spmv_coo_to_dia_analyze", "spmv_dia_to_coo_count", "spmv_sort_coo",
                 "spmv_stencil27_fill", "spmv_last_error"):
        assert must in names


def test_library_exports_every_declared_symbol(lib_built):
    lib = ctypes.CDLL(str(lib_built))
    for name in declared_functions():
        assert hasattr(lib, name), name
    out = subprocess.run(["nm", "-D", "--defined-only", str(lib_built)], capture_output=True, text=True).stdout
    exported = {line.split()[-1] for line in out.splitlines() if line.strip()}
    assert set(declared_functions()) == {s for s in exported if s.startswith("spmv_")}


def test_sm100a_cubin_inside(lib_built):
    out = subprocess.run(["/usr/local/cuda/bin/cuobjdump", "--list-elf", str(lib_built)], capture_output=True,
                         text=True).stdout
    assert "sm_100a" in out


def test_python_binding_matches_header(lib_built):
    from paper_2304_09511_b200 import _lib
    assert set(_lib.SIGNATURES) == set(declared_functions())
    lib = _lib.load()
    assert lib.spmv_abi_version() == 2


def test_status_codes_map_to_reference_errors(lib_built):
    from paper_2304_09511_b200 import _lib
    from paper_2304_09511_b200.errors import IndexOverflow
    out = ctypes.c_int64()
    with pytest.raises(IndexOverflow):
        _lib.call("spmv_stencil27_nnz", 2048, 2048, 1024, ctypes.byref(out))
    with pytest.raises(ValueError):
        _lib.call("spmv_stencil27_nnz", 0, 1, 1, ctypes.byref(out))
    assert "grid dimensions" in _lib.last_error()
    _lib.call("spmv_stencil27_nnz", 64, 64, 64, ctypes.byref(out))
    assert out.value == 6_859_000
    _lib.call("spmv_stencil27_nnz", 256, 256, 256, ctypes.byref(out))
    assert out.value == 449_455_096
    with pytest.raises(ValueError):  # lanes < 1 rejected before any device work
        _lib.call("spmv_csr_vla", 1, 4, 4, 0, None, None, None, None, 0, 4, None, 0, None)
    from paper_2304_09511_b200.errors import UnsupportedCombination
    with pytest.raises(UnsupportedCombination):
        _lib.call("spmv_csr_vla", 1, 4, 4, 0, None, None, None, None, 0, 4, None, 2048, None)


def test_plan_config_struct_matches_header(lib_built):
    """ctypes layout of spmv_plan_config == the C struct (16 int32 fields),
    and spmv_plan_config_init fills the auto values PlanConfig() holds."""
    import ctypes

    from paper_2304_09511_b200 import _lib
    from paper_2304_09511_b200.planconfig import VERSION, PlanConfig, _CPlanConfig
    assert ctypes.sizeof(_CPlanConfig) == 16 * 4
    text = (Path(__file__).resolve().parent.parent / "include" / "spmv_b200.h").read_text()
    assert f"#define SPMV_PLAN_CONFIG_VERSION {VERSION}" in text
    c = _CPlanConfig()
    _lib.call("spmv_plan_config_init", ctypes.byref(c))
    assert c.version == VERSION and PlanConfig.from_c(c) == PlanConfig()
    assert PlanConfig(tile=1024, warp_stream=0).to_c().tile == 1024
