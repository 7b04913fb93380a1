"""Reference-facing plugin: run the reference's own drivers on the GPU kernels.

The reference threads one `KernelRegistry` through every driver that runs a
product: `dispatch` (kernels.py:286-297), `autotune.measure` / `tune`
(autotune.py:60-64, :110-114), `bench.run_corpus` (bench.py:149-154),
`hpcg.distributed_spmv` / `cg_solve` / `run_phases` (hpcg.py:167-169,
:211-213, :360-366) and `cli.main` (cli.py:259-266).  A registered callable
takes ``(matrix, x, config)`` and returns a numpy y (kernels.py:216-217).

`register_gpu_kernels(registry)` puts the sm_100a kernels under the six
``(format, version)`` keys of any registry with that interface — the
reference's or ours.  The callables accept the reference's numpy containers
(uploaded once per container and cached, formats.as_device) and numpy x, and
return numpy y, so the reference's drivers run unchanged:

    from spmvkit.kernels import KernelRegistry          # the reference
    from paper_2304_09511_b200.plugin import register_gpu_kernels
    reg = register_gpu_kernels(KernelRegistry())
    measure(matrix, "csr", "plain", registry=reg)       # timed on the B200
"""

from __future__ import annotations

from . import kernels as K

FORMATS = ("coo", "csr", "dia")
VERSIONS = ("plain", "vla")

_CALLABLES = {
    ("coo", "plain"): K._plain_coo,
    ("csr", "plain"): K._plain_csr,
    ("dia", "plain"): K._plain_dia,
    ("coo", "vla"): K._vla_coo,
    ("csr", "vla"): K._vla_csr,
    ("dia", "vla"): K._vla_dia,
}


def gpu_kernel(fmt: str, version: str):
    """The GPU callable for one (format, version) pair."""
    return _CALLABLES[(str(getattr(fmt, "value", fmt)), str(getattr(version, "value", version)))]


def register_gpu_kernels(registry, formats=FORMATS, versions=VERSIONS):
    """Register the GPU kernels into `registry` (anything with the
    reference's ``register(fmt, version, fn)``) and return it."""
    for fmt in formats:
        for version in versions:
            registry.register(fmt, version, gpu_kernel(fmt, version))
    return registry
