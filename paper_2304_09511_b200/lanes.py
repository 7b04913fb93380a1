"""Lane configuration for the vector-style (vla) kernels (lanes.py:19-43).

On the GPU a "lane" is a thread of a sub-warp (L <= 32) or of a CTA
(32 < L <= 1024): lane l accumulates entries s+l, s+l+L, ... and the lanes
are folded with the reference's pairwise-halving tree (lanes.py:107-128),
realised with __shfl_down_sync, so results are bit-identical to the
reference's vla kernels for every lane count.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

LANES_ENV_VAR = "SPMV_LANES"
DEFAULT_LANES = 8
MAX_GPU_LANES = 1024


@dataclass(frozen=True)
class LaneConfig:
    """Lane count for the vector-style kernels.  Must be at least 1."""

    lanes: int = DEFAULT_LANES

    def __post_init__(self) -> None:
        if self.lanes < 1:
            raise ValueError("lane count must be >= 1")

    @classmethod
    def from_env(cls, default: int = DEFAULT_LANES) -> "LaneConfig":
        """Read the lane count from ``SPMV_LANES``; bad values raise ValueError."""
        raw = os.environ.get(LANES_ENV_VAR)
        if raw is None or not raw.strip():
            return cls(default)
        try:
            lanes = int(raw)
        except ValueError as exc:
            raise ValueError(f"{LANES_ENV_VAR} must be an integer, got {raw!r}") from exc
        return cls(lanes)
