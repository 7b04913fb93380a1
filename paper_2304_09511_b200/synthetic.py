"""Seeded synthetic inputs for the BASELINE.json configurations.

The reference has no generator for configs 3 and 4:
`gen_random_sparse` draws uniform positions and `gen_banded` writes
deterministic values.  These host-side (numpy) generators define them, fully
seeded, and return host arrays that the caller uploads into device
containers.  They are input generators, not part of the SpMV path.

* zipf_csr     config 3: row lengths ~ Zipf(a) rejected to [1, max_len],
               columns uniform without duplicates inside a row (sorted),
               values U[-1, 1]
* banded_dia   config 4: square DIA, given offsets, in-bounds cells N(0, 1),
               out-of-matrix and padding cells 0
* probe_x      x = default_rng(seed).uniform(-1, 1, n) (test_acceptance.py:66-68)
"""

from __future__ import annotations

import numpy as np

ROW_PAD = 8


def probe_x(n: int, seed: int, dtype=np.float64) -> np.ndarray:
    return np.random.default_rng(seed).uniform(-1.0, 1.0, size=n).astype(dtype)


def zipf_csr(nrows: int, ncols: int, seed: int, exponent: float = 1.8, max_len: int = 50_000,
             dtype=np.float64):
    """Returns (irp uint32[nrows+1], cols uint32[nnz], vals dtype[nnz])."""
    rng = np.random.default_rng(seed)
    lens = rng.zipf(exponent, size=nrows)
    bad = lens > max_len
    while bad.any():
        lens[bad] = rng.zipf(exponent, size=int(bad.sum()))
        bad = lens > max_len
    lens = np.minimum(lens, ncols)
    nnz = int(lens.sum())
    rows = np.repeat(np.arange(nrows, dtype=np.int64), lens)
    cols = rng.integers(0, ncols, size=nnz, dtype=np.int64)
    while True:
        key = rows * ncols + cols
        order = np.argsort(key, kind="stable")
        key = key[order]
        rows, cols = rows[order], cols[order]
        dup = np.zeros(nnz, dtype=bool)
        dup[1:] = key[1:] == key[:-1]
        if not dup.any():
            break
        cols[dup] = rng.integers(0, ncols, size=int(dup.sum()), dtype=np.int64)
    irp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(lens, out=irp[1:])
    vals = rng.uniform(-1.0, 1.0, size=nnz).astype(dtype)
    return irp.astype(np.uint32), cols.astype(np.uint32), vals


def banded_dia(n: int, offsets, seed: int, dtype=np.float64, pad_to: int = ROW_PAD):
    """Returns (offsets int32[nd] ascending, values dtype[(padded, nd)], nnz)."""
    offs = np.unique(np.asarray(list(offsets), dtype=np.int64))
    padded = -(-n // pad_to) * pad_to
    rng = np.random.default_rng(seed)
    vals = rng.standard_normal((padded, offs.shape[0])).astype(dtype)
    rows = np.arange(padded, dtype=np.int64)[:, None]
    cols = rows + offs[None, :]
    outside = (cols < 0) | (cols >= n) | (rows >= n)
    vals[outside] = 0
    nnz = int(np.count_nonzero(vals))
    return offs.astype(np.int32), vals, nnz


# BASELINE.json configs 1-5
BANDED_OFFSETS = (0, -1, 1, -2, 2, -512, 512, -1024, 1024, -4096, 4096)
ZIPF_SEED = 42
BANDED_SEED = 4
X_SEED = 0
