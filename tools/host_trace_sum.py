"""Summarise SPMV_HOST_TRACE lines: per-stream end times and chunk periods."""
import sys

for f in sys.argv[1:]:
    lines = [ln for ln in open(f) if ln.startswith("host-trace")]
    if not lines:
        print(f, "no trace")
        continue
    ev = [(t[0], float(t[1:])) for t in lines[-1].split()[1:]]
    h = [t for k, t in ev if k == "h"]
    d = [t for k, t in ev if k == "d"]
    e = [t for k, t in ev if k == "e"]
    d2h = f"D2H first {d[0]:.3f} last {d[-1]:.3f}" if d else "no D2H"
    print(f"{f}: chunks {len(h)}  H2D last {h[-1]:.3f}  {d2h}  end {e[-1]:.3f} ms")
