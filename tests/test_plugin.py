"""Reference-facing plugin: the GPU kernels registered into a registry with
the reference's interface, driven with reference-shaped host containers."""

import sys
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import pytest

from _util import bit_equal, load_golden, matrix_arrays

REF_SRC = Path("/root/reference/pkg/src")


@dataclass(frozen=True)
class Shape:
    nrows: int
    ncols: int
    nnz: int


@dataclass(eq=False)
class HostCsr:  # the reference's CsrMatrix attribute names (formats.py:124-163)
    shape: Shape
    row_pointers: np.ndarray
    col_indices: np.ndarray
    values: np.ndarray

    @property
    def format(self):
        return "csr"


def test_registers_six_pairs_into_our_registry():
    from paper_2304_09511_b200.kernels import KernelRegistry
    from paper_2304_09511_b200.plugin import gpu_kernel, register_gpu_kernels
    reg = register_gpu_kernels(KernelRegistry())
    assert len(reg.pairs()) == 6
    assert reg.lookup("csr", "plain") is gpu_kernel("csr", "plain")


@pytest.mark.skipif(not REF_SRC.exists(), reason="reference package not present (GPU box)")
def test_registers_into_the_reference_registry():
    sys.path.insert(0, str(REF_SRC))
    try:
        from spmvkit.kernels import KernelRegistry, KernelVersion
        from spmvkit.formats import Format
        from paper_2304_09511_b200.plugin import register_gpu_kernels
        reg = register_gpu_kernels(KernelRegistry())
        for fmt in Format:
            for version in KernelVersion:
                assert reg.supports(fmt, version)
    finally:
        sys.path.remove(str(REF_SRC))


@pytest.mark.gpu
def test_host_container_round_trip_and_cache(lib_built):
    from paper_2304_09511_b200.formats import as_device
    from paper_2304_09511_b200.kernels import KernelRegistry, dispatch
    from paper_2304_09511_b200.plugin import register_gpu_kernels
    d = load_golden("corpus")
    a = matrix_arrays(d, "stencil-6/csr")
    host = HostCsr(Shape(*map(int, a["shape"])), a["row_pointers"], a["col_indices"], a["values"])
    reg = register_gpu_kernels(KernelRegistry())
    x = d["stencil-6/x"]
    y = dispatch(host, x, "plain", registry=reg)
    assert isinstance(y, np.ndarray) and bit_equal(y, d["stencil-6/csr/y_plain"])
    assert as_device(host) is as_device(host)  # uploaded once
