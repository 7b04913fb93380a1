"""sort_coo: first mismatch against the numpy oracle on a small case (debugging aid)."""
import sys
import numpy as np
sys.path.insert(0, ".")
import paper_2304_09511_b200 as sp
from oracle import spmv_oracle as O

rng = np.random.default_rng(1)
n, ncols = int(sys.argv[1]) if len(sys.argv) > 1 else 20000, 5000
lens = rng.integers(0, 60, n)
rows = np.repeat(np.arange(n), lens)
cols = rng.integers(0, ncols, rows.shape[0])
vals = rng.standard_normal(rows.shape[0])
o = rng.permutation(rows.shape[0])
rows, cols, vals = rows[o], cols[o], vals[o]
h = sp.sort_coo(sp.CooMatrix.from_arrays(n, ncols, rows, cols, vals)).to_host()
r, c, v = O.sort_coo(rows, cols, vals)
bad = np.flatnonzero(h["row_indices"] != r)
print("nnz", r.shape[0], "row mismatches", bad.shape[0])
if bad.shape[0]:
    i = bad[0]
    print("first at", i, "got", h["row_indices"][i - 2:i + 6], "want", r[i - 2:i + 6])
    print("last at", bad[-1], "got", h["row_indices"][bad[-1]], "want", r[bad[-1]])
    g = r[bad] >> 8
    print("groups of the mismatches:", np.unique(g)[:20], "rows&255:", np.unique(r[bad] & 255)[:40])
badc = np.flatnonzero(h["col_indices"] != c)
print("col mismatches", badc.shape[0], badc[:5])
