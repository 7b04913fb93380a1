mkdir -p gpurun_out
( time python bench.py > gpurun_out/r2d_bench_default.json 2> gpurun_out/r2d_bench_default.err ) 2> gpurun_out/r2d_bench_default.time || { tail -5 gpurun_out/r2d_bench_default.err; exit 1; }
cat gpurun_out/r2d_bench_default.time
( time python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2d_bench_reference.json 2> gpurun_out/r2d_bench_reference.err ) 2>&1 | tail -4
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2d_bench_default.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"])
for c, v in d["per_config"].items():
    print(c, {k: (x["gflops"], x["roofline_frac"], x.get("l2_resident", {}).get("gflops")) for k, x in v.items() if isinstance(x, dict)})
r = json.loads(open("gpurun_out/r2d_bench_reference.json").read().strip().splitlines()[-1])
print(r["value"], r["reference_numpy"])
PY
