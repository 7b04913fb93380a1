# C3 CSR: one bench line per environment setting given as arguments ("VAR=val VAR2=val" each).
mkdir -p gpurun_out
for setting in "$@"; do
  env $setting python bench.py --config c3 --no-extras --steps 100 --warmup 5 --cpu-budget 1 > gpurun_out/c3_s.json 2> gpurun_out/c3_s.err || { tail -3 gpurun_out/c3_s.err; continue; }
  python - "$setting" <<'PY'
import json, sys
d = json.load(open("gpurun_out/c3_s.json"))
v = d["per_format"]["csr"]
print(f"{sys.argv[1]:50s} {v['gflops']:8.1f} GFLOP/s {v['ms_per_spmv']*1000:7.1f} us frac {v['roofline_frac']:.3f}")
PY
done
