"""CPU oracle for the SpMV hot path — TEST INFRASTRUCTURE ONLY.

This module restates, in numpy, the reference package `spmvkit` 0.1.0
(/root/reference/pkg/src/spmvkit, pure Python + numpy 2.3) for the functions
on the hot path.  Only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import it,
and only as the checker or the timed CPU baseline.  The product package
(``paper_2304_09511_b200``) never imports it and has no CPU fallback.

Parity pin: every function below is checked bit-for-bit against golden
vectors produced by the reference itself (tests/golden/make_golden.py,
fixtures in tests/golden/*.npz; test: tests/test_oracle_golden.py).

Order semantics that matter for bit-exactness:
  * kernels.py:65   np.add.at — sequential per row in storage order, from +0.0
  * kernels.py:75-81 products rounded first, then cumsum (left to right,
                    starting from the first product, so a lone -0.0 stays -0.0)
  * kernels.py:95-100 per-diagonal += in ascending offset order, from +0.0
  * lanes.py:101-128 lane accumulators then pairwise-halving tree
  * convert.py:80   np.add.reduceat — first element + numpy pairwise_sum of
                    the rest (numpy 2.3.5 loops_utils.h; modelled below)
No FMA anywhere (numpy rounds each product).
"""

from __future__ import annotations

import numpy as np

ROW_PAD = 8  # formats.py:30
INDEX_DTYPE = np.dtype(np.uint32)  # formats.py:24
OFFSET_DTYPE = np.dtype(np.int32)  # formats.py:25


def round_up(n: int, multiple: int) -> int:
    """formats.py:41-45."""
    return -(-int(n) // multiple) * multiple


def _cast_x(x, dtype):
    """kernels.py:46-53 (_checked_x) minus the error raise."""
    x = np.asarray(x)
    return x if x.dtype == dtype else x.astype(dtype)


# ----------------------------------------------------------------- kernels --
def csr_plain(nrows, irp, aj, av, x):
    """kernels.py:69-82.  y[r] = left-to-right sum of the rounded products.

    np.add.at is sequential in index order; seeding y with -0.0 (the IEEE
    additive identity) reproduces cumsum's "start from the first product",
    and empty rows are reset to +0.0 as the reference's zeros() leaves them.
    """
    x = _cast_x(x, av.dtype)
    irp = np.asarray(irp, dtype=np.int64)
    y = np.full(nrows, -0.0, dtype=av.dtype)
    if av.shape[0]:
        rows = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(irp))
        np.add.at(y, rows, av * x[np.asarray(aj, dtype=np.int64)])
    y[np.diff(irp) == 0] = 0.0
    return y


def coo_plain(nrows, ai, aj, av, x):
    """kernels.py:56-66.  zeros() then np.add.at in storage order."""
    x = _cast_x(x, av.dtype)
    y = np.zeros(nrows, dtype=av.dtype)
    if av.shape[0]:
        np.add.at(y, np.asarray(ai, dtype=np.int64), av * x[np.asarray(aj, dtype=np.int64)])
    return y


def dia_plain(nrows, ncols, offsets, values, x):
    """kernels.py:85-101.  Ascending diagonals, in-bounds rows only."""
    x = _cast_x(x, values.dtype)
    y = np.zeros(nrows, dtype=values.dtype)
    for d, off in enumerate(np.asarray(offsets, dtype=np.int64).tolist()):
        lo, hi = max(0, -off), min(nrows, ncols - off)
        if hi > lo:
            y[lo:hi] += values[lo:hi, d] * x[lo + off:hi + off]
    return y


def tree_reduce(vec: np.ndarray):
    """lanes.py:107-128 with an all-active mask: pad to 2^k, halve."""
    n = vec.shape[0]
    if n == 1:
        return vec[0]
    width = 1 << (n - 1).bit_length()
    vals = np.zeros(width, dtype=vec.dtype)
    vals[:n] = vec
    while width > 1:
        width //= 2
        vals = vals[:width] + vals[width:2 * width]
    return vals[0]


def csr_vla(nrows, irp, aj, av, x, lanes: int):
    """kernels.py:143-171: lane l sums entries s+l, s+l+L, ...; tree per row.

    Vectorised across rows: the lane accumulators of every row are built
    column by column (step k adds entry s + k*L + l), which is the same
    per-lane sequence as the reference's while loop.
    """
    x = _cast_x(x, av.dtype)
    irp = np.asarray(irp, dtype=np.int64)
    aj = np.asarray(aj, dtype=np.int64)
    lens = np.diff(irp)
    y = np.zeros(nrows, dtype=av.dtype)
    if av.shape[0] == 0:
        return y
    acc = np.zeros((nrows, lanes), dtype=av.dtype)
    steps = -(-lens // lanes)
    for k in range(int(steps.max())):
        for lane in range(lanes):
            j = irp[:-1] + k * lanes + lane
            m = j < irp[1:]
            jj = j[m]
            acc[m, lane] = acc[m, lane] + av[jj] * x[aj[jj]]
    width = 1 << (lanes - 1).bit_length() if lanes > 1 else 1
    if width != lanes:
        acc = np.concatenate([acc, np.zeros((nrows, width - lanes), dtype=av.dtype)], axis=1)
    while width > 1:
        width //= 2
        acc = acc[:, :width] + acc[:, width:2 * width]
    out = acc[:, 0]
    y[lens > 0] = out[lens > 0]
    return y


def coo_vla(nrows, ai, aj, av, x, lanes: int, stats: dict | None = None):
    """kernels.py:104-140 on a sorted COO: L-entry steps that never cross a
    row, each tree-reduced (zero-padded lanes) and added once into y[row]."""
    x = _cast_x(x, av.dtype)
    ai = np.asarray(ai, dtype=np.int64)
    aj = np.asarray(aj, dtype=np.int64)
    y = np.zeros(nrows, dtype=av.dtype)
    nnz = av.shape[0]
    steps = 0
    i = 0
    prod = av * x[aj] if nnz else av
    while i < nnz:
        r = ai[i]
        end = i
        lim = min(nnz, i + lanes)
        while end < lim and ai[end] == r:
            end += 1
        vec = np.zeros(lanes, dtype=av.dtype)
        vec[:end - i] = prod[i:end]
        y[r] += tree_reduce(vec)
        i = end
        steps += 1
    if stats is not None:
        stats["outer_steps"] = steps
    return y


def dia_vla(nrows, ncols, offsets, values, x, lanes: int = 8):
    """kernels.py:174-210.  Per row the diagonal order equals dia_plain's."""
    return dia_plain(nrows, ncols, offsets, values, x)


# ------------------------------------------------------------- conversions --
def coo_to_csr(nrows, ai):
    """convert.py:87-94 (IRP part): [0, cumsum(bincount(rows))]."""
    irp = np.zeros(nrows + 1, dtype=np.int64)
    np.cumsum(np.bincount(np.asarray(ai, dtype=np.int64), minlength=nrows), out=irp[1:])
    return irp.astype(INDEX_DTYPE)


def csr_to_coo(nrows, irp, aj):
    """convert.py:97-110: repeat rows; sorted iff cols strictly rise per row."""
    irp = np.asarray(irp, dtype=np.int64)
    rows = np.repeat(np.arange(nrows, dtype=np.int64), np.diff(irp))
    aj = np.asarray(aj)
    ok = True
    if aj.shape[0] > 1:
        same = rows[1:] == rows[:-1]
        ok = bool((aj[1:][same] > aj[:-1][same]).all())
    return rows.astype(INDEX_DTYPE), ok


def dia_fill_check(nrows, ncols, nnz, ndiags, max_fill_ratio=10.0, max_ndiags=None, pad_to=ROW_PAD):
    """convert.py:127-139: returns None or the FillRatioExceeded message kind."""
    padded = round_up(nrows, pad_to) if nrows else 0
    cap = max_ndiags if max_ndiags is not None else max(nrows + ncols - 1, 0)
    if ndiags > cap:
        return "cap"
    if padded * ndiags > max_fill_ratio * max(nnz, 1):
        return "fill ratio"
    return None


def coo_to_dia(nrows, ncols, ai, aj, av, pad_to=ROW_PAD):
    """convert.py:113-144 (after the fill check): unique offsets, scatter."""
    r = np.asarray(ai, dtype=np.int64)
    c = np.asarray(aj, dtype=np.int64)
    offsets = np.unique(c - r)
    padded = round_up(nrows, pad_to) if nrows else 0
    values = np.zeros((padded, offsets.shape[0]), dtype=av.dtype)
    if av.shape[0]:
        values[r, np.searchsorted(offsets, c - r)] = av
    return offsets.astype(OFFSET_DTYPE), values


def dia_to_coo(nrows, ncols, offsets, values):
    """convert.py:147-177: in-bounds cells != 0 (NaN kept, -0.0 dropped).

    Row-major traversal over (row, ascending diagonal) already yields the
    (row, col) order the reference obtains with lexsort.
    """
    offs = np.asarray(offsets, dtype=np.int64)
    if nrows == 0 or offs.shape[0] == 0:
        return (np.zeros(0, INDEX_DTYPE), np.zeros(0, INDEX_DTYPE), np.zeros(0, values.dtype))
    rows = np.arange(nrows, dtype=np.int64)[:, None]
    cols = rows + offs[None, :]
    block = values[:nrows]
    keep = (cols >= 0) & (cols < ncols) & (block != 0)
    rr = np.broadcast_to(rows, keep.shape)[keep]
    return rr.astype(INDEX_DTYPE), cols[keep].astype(INDEX_DTYPE), block[keep]


def np_pairwise_sum(a: np.ndarray):
    """numpy 2.3.5 pairwise_sum (numpy/_core/src/umath/loops_utils.h.src):
    < 8 terms: sequential from -0.0; <= 128: eight interleaved accumulators
    combined ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail; else split
    at n/2 rounded down to a multiple of 8.  Pinned against np.add.reduceat
    by tests/test_oracle_golden.py::test_reduceat_model."""
    t = a.dtype.type
    n = a.shape[0]
    if n < 8:
        res = t(-0.0)
        for v in a:
            res = t(res + v)
        return res
    if n <= 128:
        r = [a[j] for j in range(8)]
        i = 8
        while i < n - (n % 8):
            for j in range(8):
                r[j] = t(r[j] + a[i + j])
            i += 8
        res = t(t(t(r[0] + r[1]) + t(r[2] + r[3])) + t(t(r[4] + r[5]) + t(r[6] + r[7])))
        while i < n:
            res = t(res + a[i])
            i += 1
        return res
    n2 = n // 2
    n2 -= n2 % 8
    return t(np_pairwise_sum(a[:n2]) + np_pairwise_sum(a[n2:]))


def reduceat_sum(a: np.ndarray):
    """One segment of np.add.reduceat: a[0] + pairwise_sum(a[1:])."""
    if a.shape[0] == 1:
        return a[0]
    return a.dtype.type(a[0] + np_pairwise_sum(a[1:]))


def sort_coo(ai, aj, av):
    """convert.py:60-84 for an unsorted COO: stable lexsort by (row, col);
    duplicate runs summed like np.add.reduceat; zero sums kept."""
    ai = np.asarray(ai, dtype=np.int64)
    aj = np.asarray(aj, dtype=np.int64)
    order = np.lexsort((aj, ai))
    r, c, v = ai[order], aj[order], av[order]
    if r.shape[0] > 1:
        new = np.empty(r.shape[0], dtype=bool)
        new[0] = True
        new[1:] = (r[1:] != r[:-1]) | (c[1:] != c[:-1])
        if not new.all():
            starts = np.flatnonzero(new)
            ends = list(starts[1:]) + [r.shape[0]]
            v = np.array([reduceat_sum(v[s:e]) for s, e in zip(starts, ends)], dtype=v.dtype)
            r, c = r[starts], c[starts]
    return r.astype(INDEX_DTYPE), c.astype(INDEX_DTYPE), v


# -------------------------------------------------------------- generators --
def stencil27(nx, ny, nz, dtype=np.float64, row_begin=0, row_end=None):
    """matrixio.py:170-210, optionally restricted to rows [row_begin, row_end).

    Row p = (z*ny + y)*nx + x; neighbours in (dz, dy, dx) lexicographic order
    give ascending columns; 26.0 on the diagonal, -1.0 elsewhere.
    Returns (irp rebased to 0, cols, vals) as uint32/uint32/dtype.
    """
    n = nx * ny * nz
    row_end = n if row_end is None else row_end
    p = np.arange(row_begin, row_end, dtype=np.int64)
    x, y, z = p % nx, (p // nx) % ny, p // (nx * ny)
    cols = np.full((p.shape[0], 27), -1, dtype=np.int64)
    vals = np.zeros((p.shape[0], 27), dtype=dtype)
    k = 0
    for dz in (-1, 0, 1):
        for dy in (-1, 0, 1):
            for dx in (-1, 0, 1):
                qx, qy, qz = x + dx, y + dy, z + dz
                ok = (qx >= 0) & (qx < nx) & (qy >= 0) & (qy < ny) & (qz >= 0) & (qz < nz)
                cols[ok, k] = ((qz * ny + qy) * nx + qx)[ok]
                vals[ok, k] = 26.0 if (dx, dy, dz) == (0, 0, 0) else -1.0
                k += 1
    keep = cols >= 0
    irp = np.zeros(p.shape[0] + 1, dtype=np.int64)
    np.cumsum(keep.sum(axis=1), out=irp[1:])
    return irp.astype(INDEX_DTYPE), cols[keep].astype(INDEX_DTYPE), vals[keep]


def rel_err(y, ref) -> float:
    """tests/helpers.py:71-77: max |y - ref| / max(|ref|, 1)."""
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.size == 0:
        return 0.0
    return float(np.max(np.abs(y - ref) / np.maximum(np.abs(ref), 1.0)))
