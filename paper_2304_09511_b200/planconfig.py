"""Per-plan kernel configuration (include/spmv_b200.h `spmv_plan_config`).

The reference tunes the storage format per matrix by running every
candidate (autotune.py:60-139) and, in its HPCG study, the kernel variant
(hpcg.py:270-304).  On the GPU the same choice extends to the kernel
"bins": tile size, consumer groups, the row-length threshold for the
one-thread-per-row path, the whole-matrix warp-stream kernel, its range
count, the TMA L2 hint and the DIA kernel shape.  A `PlanConfig` holds
those choices; every field left at its auto value keeps the plan's
measured default (which depends on the row-length histogram).

A configuration belongs to a plan, not to the process: two plans of one
matrix with different configurations coexist (the plan cache is keyed by
it), so a tuner can time candidates side by side
(`autotune.tune_plan`).  Attach the winner to a container with
`set_plan_config(A, cfg)`; every product of A then runs it.
"""

from __future__ import annotations

import ctypes
import os
import threading
from contextlib import contextmanager
from dataclasses import asdict, dataclass, fields, replace

VERSION = 1


class _CPlanConfig(ctypes.Structure):
    _fields_ = [("version", ctypes.c_int32), ("tile", ctypes.c_int32), ("groups", ctypes.c_int32),
                ("exact_len", ctypes.c_int32), ("warp_stream", ctypes.c_int32),
                ("ranges_per_warp", ctypes.c_int32), ("tma_hint", ctypes.c_int32), ("ctas_per_sm", ctypes.c_int32),
                ("dia_kernel", ctypes.c_int32), ("dia_rows", ctypes.c_int32), ("flags", ctypes.c_int32),
                ("panels", ctypes.c_int32), ("reserved", ctypes.c_int32 * 4)]


@dataclass(frozen=True)
class PlanConfig:
    """Kernel choices of one plan; 0 / -1 = the plan's own choice.

    tile            entries per TMA tile (CSR 1024/1664/2048/2304/4096,
                    COO 1024/1536/2048)
    groups          consumer groups per tile CTA (CSR 1/3/4, COO 1/6/7)
    exact_len       CSR warp-stream kernel: rows of <= exact_len entries stay
                    whole in one warp range, summed left to right (bit-exact
                    with kernels.py:69-82), 1..32; tile kernels always use 32
    warp_stream     whole-matrix kernel: -1 auto, 0 tile kernel, 1 warp-stream
    ranges_per_warp warp-stream entry ranges per resident warp, 1..64
    tma_hint        L2 evict_first on the TMA matrix stream: -1 auto, 0, 1
    ctas_per_sm     cap on resident CTAs per SM (0 = occupancy)
    dia_kernel      DIA (groups, stages, threads) preset 0..4, -1 auto
    dia_rows        DIA rows per tile (multiple of 8), 0 auto
    flags           experiments (bit0 products mode, bit1 warp per long segment)
    panels          CSR column-panel path for long rows (csrc/panel.cuh): -1 auto,
                    0 off, 1 on
    """

    tile: int = 0
    groups: int = 0
    exact_len: int = 0
    warp_stream: int = -1
    ranges_per_warp: int = 0
    tma_hint: int = -1
    ctas_per_sm: int = 0
    dia_kernel: int = -1
    dia_rows: int = 0
    flags: int = 0
    panels: int = -1

    def to_c(self) -> _CPlanConfig:
        """The C struct (built once per instance; the callee only reads it)."""
        c = self.__dict__.get("_c")
        if c is None:
            c = _CPlanConfig()
            c.version = VERSION
            for f in fields(self):
                setattr(c, f.name, int(getattr(self, f.name)))
            object.__setattr__(self, "_c", c)
        return c

    @classmethod
    def from_c(cls, c: _CPlanConfig) -> "PlanConfig":
        return cls(**{f.name: int(getattr(c, f.name)) for f in fields(cls)})

    def key(self) -> tuple:
        """Plan-cache key (every product looks its plan up by it: computed
        once per instance, the dataclass is frozen)."""
        k = self.__dict__.get("_key")
        if k is None:
            k = tuple(getattr(self, f.name) for f in fields(self))
            object.__setattr__(self, "_key", k)
        return k

    def with_(self, **kw) -> "PlanConfig":
        return replace(self, **kw)

    def as_dict(self) -> dict:
        return asdict(self)

    @classmethod
    def from_env(cls) -> "PlanConfig":
        """Experiment scripts (tools/): the round-1 SPMV_* switches as a
        configuration.  Never read implicitly by the library."""
        env = {"tile": "SPMV_TILE", "flags": "SPMV_TILE_MODE", "tma_hint": "SPMV_TMA_HINT",
               "ranges_per_warp": "SPMV_WS_RANGES", "ctas_per_sm": "SPMV_CTAS_PER_SM", "dia_rows": "SPMV_DIA_ROWS",
               "dia_kernel": "SPMV_DIA_CFG", "panels": "SPMV_PANELS"}
        kw = {k: int(os.environ[v]) for k, v in env.items() if os.environ.get(v)}
        for k, v in (("groups", "SPMV_CSR_GROUPS"), ("groups", "SPMV_COO_GROUPS")):
            if os.environ.get(v):
                kw[k] = int(os.environ[v])
        for v in ("SPMV_CSR_WS", "SPMV_COO_WS"):
            if os.environ.get(v):
                kw["warp_stream"] = int(os.environ[v])
        return cls(**kw)


AUTO = PlanConfig()


def set_plan_config(matrix, cfg: PlanConfig | None) -> None:
    """Attach a configuration to a device container: its products (plain,
    vla, host pipeline) use plans built with `cfg` (None detaches it)."""
    object.__setattr__(matrix, "_plan_config", cfg)


_DEFAULT = threading.local()


def plan_config_of(matrix) -> PlanConfig:
    """The container's attached configuration, else this thread's scoped
    default (`using_plan_config`), else AUTO."""
    cfg = getattr(matrix, "_plan_config", None)
    if cfg is not None:
        return cfg
    return getattr(_DEFAULT, "cfg", None) or AUTO


@contextmanager
def using_plan_config(cfg: PlanConfig):
    """Scoped default for containers without an attached configuration, in
    this thread only (tests force each kernel path in-process with it)."""
    prev = getattr(_DEFAULT, "cfg", None)
    _DEFAULT.cfg = cfg
    try:
        yield cfg
    finally:
        _DEFAULT.cfg = prev
