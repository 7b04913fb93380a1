"""Shared test helpers: golden fixtures, bitwise comparison, rel_err."""

from __future__ import annotations

from functools import lru_cache
from pathlib import Path

import numpy as np

GOLDEN = Path(__file__).resolve().parent / "golden"


@lru_cache(maxsize=None)
def load_golden(name: str) -> dict:
    with np.load(GOLDEN / f"{name}.npz", allow_pickle=False) as z:
        return {k: z[k] for k in z.files}


def bit_equal(a, b) -> bool:
    """Same shape and dtype; NaN positions agree; all other bits identical
    (so +0.0 vs -0.0 counts as a difference)."""
    a = np.asarray(a)
    b = np.asarray(b)
    if a.shape != b.shape or a.dtype != b.dtype:
        return False
    if a.size == 0:
        return True
    na, nb = np.isnan(a), np.isnan(b)
    if not np.array_equal(na, nb):
        return False
    ui = np.uint64 if a.dtype.itemsize == 8 else np.uint32
    return bool(np.array_equal(a[~na].view(ui), b[~nb].view(ui)))


def first_diff(a, b) -> str:
    a = np.asarray(a)
    b = np.asarray(b)
    ne = ~((a == b) | (np.isnan(a) & np.isnan(b))) | (np.signbit(a) != np.signbit(b))
    idx = np.flatnonzero(ne)
    if idx.size == 0:
        return "no difference"
    i = idx[0]
    return f"{idx.size} differ; first at {i}: {a[i]!r} vs {b[i]!r}"


def rel_err(y, ref) -> float:
    """Reference test helper semantics (tests/helpers.py:71-77)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.size == 0:
        return 0.0
    return float(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)))


def matrix_arrays(d: dict, key: str) -> dict:
    """Collect the arrays stored under `key/` by make_golden.put_matrix."""
    out = {}
    pre = key + "/"
    for k, v in d.items():
        if k.startswith(pre) and "/" not in k[len(pre):]:
            out[k[len(pre):]] = v
    return out


def corpus_names() -> list:
    return [str(n) for n in load_golden("corpus")["names"]]
