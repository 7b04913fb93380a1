"""Randomised parity sweep of the product kernels against the C oracle.

Random shapes and row-length mixes (empty rows, short rows, rows on the
32 / 64 / 256 thresholds, long rows), f64 and f32, CSR / COO plain and vla
at random lane counts, on whichever kernel each plan picks, plus sort_coo of
the shuffled triples (with repeated coordinates) and the unsorted COO product.  Contract as in
tests/test_gpu_kernels.py: rows <= 32 bit-exact, everything within 1e-12
(f64) / 1e-5 of the f64-evaluated product (f32); vla bit-exact.  Prints
one line per failure and a summary; exit code 1 on any failure.

  python tools/fuzz_parity.py [cases=200] [seed=0] [scale=1]
"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

import paper_2304_09511_b200 as sp  # noqa: E402
from oracle import c_oracle  # noqa: E402
from oracle import spmv_oracle as O  # noqa: E402


def rel_err(y, ref):
    y = np.asarray(y, dtype=np.float64)
    ref = np.asarray(ref, dtype=np.float64)
    if y.size == 0:
        return 0.0
    return float(np.max(np.abs(y - ref)) / max(np.max(np.abs(ref)), 1.0))


def bit_equal(a, b):
    return np.asarray(a).tobytes() == np.asarray(b).tobytes()


def random_lens(rng, nrows, ncols):
    kind = rng.integers(0, 5)
    if kind == 0:  # short rows with empties
        lens = rng.integers(0, 33, nrows)
    elif kind == 1:  # thresholds
        lens = rng.choice([0, 1, 31, 32, 33, 63, 64, 65, 255, 256, 257, 600], nrows)
    elif kind == 2:  # power law
        lens = np.minimum(rng.zipf(1.6, nrows), 5000)
    elif kind == 3:  # a few huge rows
        lens = rng.integers(0, 8, nrows)
        lens[rng.integers(0, nrows, 3)] = rng.integers(1000, 20000, 3)
    else:  # mixed
        lens = np.where(rng.random(nrows) < 0.05, rng.integers(33, 3000, nrows), rng.integers(0, 20, nrows))
    return np.minimum(lens, ncols).astype(np.int64)


def main():
    cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
    seed = int(sys.argv[2]) if len(sys.argv) > 2 else 0
    scale = int(sys.argv[3]) if len(sys.argv) > 3 else 1  # > 1: bigger matrices (many warp-stream ranges)
    rng = np.random.default_rng(seed)
    fails = 0
    refused = 0
    for case in range(cases):
        nrows = int(rng.integers(1, 6000 * scale))
        ncols = int(rng.integers(1, 40000 * scale))
        lens = random_lens(rng, nrows, ncols)
        irp = np.zeros(nrows + 1, dtype=np.int64)
        np.cumsum(lens, out=irp[1:])
        cols = np.concatenate([np.sort(rng.choice(ncols, size=int(k), replace=False)) if k else np.zeros(0, np.int64)
                               for k in lens]).astype(np.uint32)
        dtype = np.float64 if rng.random() < 0.7 else np.float32
        vals = rng.standard_normal(cols.shape[0]).astype(dtype)
        if rng.random() < 0.2:
            vals[rng.random(vals.shape[0]) < 0.1] = -0.0
        x = rng.uniform(-1, 1, ncols).astype(dtype)
        irp32 = irp.astype(np.uint32)
        ref = c_oracle.csr_plain(nrows, irp32, cols, vals, x)
        ref64 = c_oracle.csr_plain(nrows, irp32, cols, vals.astype(np.float64), x.astype(np.float64))
        tol = 1e-12 if dtype == np.float64 else 1e-5
        short = lens <= 32
        try:
            A = sp.CsrMatrix.from_arrays(nrows, ncols, irp32, cols, vals)
            y = sp.spmv_csr_plain(A, x)
            ok = bit_equal(y[short], ref[short]) and rel_err(y, ref64) <= tol
            C = sp.csr_to_coo(A)
            rows = np.repeat(np.arange(nrows), lens).astype(np.uint32)
            ref_c = c_oracle.coo_plain(nrows, rows, cols, vals, x)
            yc = sp.spmv_coo_plain(C, x)
            ok_c = bit_equal(yc[short], ref_c[short]) and rel_err(yc, ref64) <= tol
            lanes = int(rng.choice([1, 2, 3, 4, 5, 8, 9, 16, 17, 32, 33, 64]))
            ok_v = bit_equal(sp.spmv_csr_vla(A, x, sp.LaneConfig(lanes)),
                             c_oracle.csr_vla(nrows, irp32, cols, vals, x, lanes))
            small = cols.shape[0] <= 60000  # the python COO-vla oracle is a loop
            ok_cv = True
            if small:
                st, rst = {}, {}
                yv = sp.spmv_coo_vla(C, x, sp.LaneConfig(lanes), st)
                ok_cv = bit_equal(yv, O.coo_vla(nrows, rows, cols, vals, x, lanes, rst)) and \
                    st["outer_steps"] == rst["outer_steps"]
            # sort_coo of the shuffled triples, some coordinates repeated
            # (stable lexsort + reduceat-order duplicate sums, bit-exact) and
            # the product of the unsorted COO (stable row sort in the plan)
            ok_s = ok_u = True
            if cols.shape[0] and cols.shape[0] <= 400000:
                perm = rng.permutation(cols.shape[0])
                sr, sc, sv = rows[perm].copy(), cols[perm].copy(), vals[perm].copy()
                U = sp.CooMatrix.from_arrays(nrows, ncols, sr, sc, sv, False)
                yu = sp.spmv_coo_plain(U, x)
                ref_u = c_oracle.coo_plain(nrows, sr, sc, sv, x, row_sorted=False)
                ok_u = bit_equal(yu[short], ref_u[short]) and rel_err(yu, ref64) <= tol
                if rng.random() < 0.5:
                    k = max(1, cols.shape[0] // 5)
                    src, dst = rng.integers(0, cols.shape[0], k), rng.integers(0, cols.shape[0], k)
                    sr[dst], sc[dst] = sr[src], sc[src]
                got = sp.sort_coo(sp.CooMatrix.from_arrays(nrows, ncols, sr, sc, sv, False)).to_host()
                r_ref, c_ref, v_ref = O.sort_coo(sr, sc, sv)
                ok_s = np.array_equal(got["row_indices"], r_ref) and np.array_equal(got["col_indices"], c_ref) and \
                    bit_equal(got["values"], v_ref)
        except Exception as e:  # noqa: BLE001
            print(f"case {case}: exception {type(e).__name__}: {e}")
            fails += 1
            continue
        if not (ok and ok_c and ok_v and ok_cv and ok_s and ok_u):
            fails += 1
            print(f"case {case}: nrows={nrows} ncols={ncols} nnz={cols.shape[0]} {np.dtype(dtype).name} "
                  f"lanes={lanes} csr={ok} coo={ok_c} csr_vla={ok_v} coo_vla={ok_cv} sort_coo={ok_s} "
                  f"coo_unsorted={ok_u} max_len={lens.max()}")
    # DIA: random diagonal sets (conversions on the device, product and
    # round trip bit-exact against the oracle)
    for case in range(cases // 2):
        n = int(rng.integers(8, 5000))
        m = int(rng.integers(8, 5000))
        nd = int(rng.integers(1, 12))
        if rng.random() < 0.7:  # banded (the fill policy admits it)
            offs = np.unique(rng.integers(-min(n - 1, 64), min(m, 65), nd))
        else:
            offs = np.unique(rng.integers(-(n - 1), m, nd))
        rr, cc = [], []
        for o in offs:
            r = np.arange(max(0, -o), min(n, m - o))
            keep = r[rng.random(r.shape[0]) < 0.8]
            rr.append(keep)
            cc.append(keep + o)
        rows = np.concatenate(rr).astype(np.int64)
        cols_ = np.concatenate(cc).astype(np.int64)
        order = np.lexsort((cols_, rows))
        rows, cols_ = rows[order].astype(np.uint32), cols_[order].astype(np.uint32)
        dtype = np.float64 if rng.random() < 0.7 else np.float32
        vals = rng.standard_normal(rows.shape[0]).astype(dtype)
        x = rng.uniform(-1, 1, m).astype(dtype)
        try:
            coo = sp.CooMatrix.from_arrays(n, m, rows, cols_, vals, True)
            if O.dia_fill_check(n, m, rows.shape[0], offs.shape[0]) is not None:
                # the reference refuses this fill (convert.py:128-139): so must we
                try:
                    sp.coo_to_dia(coo)
                    print(f"dia case {case}: fill policy not enforced")
                    fails += 1
                except sp.FillRatioExceeded:
                    refused += 1
                continue
            dia = sp.coo_to_dia(coo)
            h = dia.to_host()
            ref_off, ref_vals = O.coo_to_dia(n, m, rows, cols_, vals)
            ok_conv = np.array_equal(h["offsets"], ref_off) and bit_equal(h["values"], ref_vals)
            y = sp.spmv_dia_plain(dia, x)
            ok_y = bit_equal(y, O.dia_plain(n, m, ref_off, ref_vals, x))
            back = sp.dia_to_coo(dia).to_host()
            b_r, b_c, b_v = O.dia_to_coo(n, m, ref_off, ref_vals)
            ok_back = np.array_equal(back["row_indices"], b_r) and np.array_equal(back["col_indices"], b_c) and \
                bit_equal(back["values"], b_v)
        except Exception as e:  # noqa: BLE001
            print(f"dia case {case}: exception {type(e).__name__}: {e}")
            fails += 1
            continue
        if not (ok_conv and ok_y and ok_back):
            fails += 1
            print(f"dia case {case}: n={n} m={m} nd={offs.shape[0]} {np.dtype(dtype).name} conv={ok_conv} "
                  f"y={ok_y} back={ok_back}")
    print(f"fuzz: {cases} CSR/COO cases + {cases // 2} DIA cases ({refused} refused by the fill policy, as the "
          f"reference refuses them), {fails} failures (seed {seed})")
    sys.exit(1 if fails else 0)


if __name__ == "__main__":
    main()
