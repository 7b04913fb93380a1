mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/r2i_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2i_gputests.log
tail -4 gpurun_out/r2i_gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2i_smoke.log 2>&1; tail -2 gpurun_out/r2i_smoke.log
python bench.py > gpurun_out/r2i_bench_default.json 2> gpurun_out/r2i_bench_default.err || { tail -5 gpurun_out/r2i_bench_default.err; exit 1; }
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2i_bench_reference.json 2> gpurun_out/r2i_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2i_launches_c5.csv python bench.py --steps 20 --warmup 3 --cpu-budget 1 --no-per-config > gpurun_out/ncu_launch_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2i_launches_conversions.csv python bench.py --conversions > gpurun_out/ncu_launch_conv.log 2>&1
python - <<'PY'
import json
d = json.loads(open("gpurun_out/r2i_bench_default.json").read().strip().splitlines()[-1])
print(d["value"], d["e2e"]["value"], d["roofline"]["frac"], {k: v["ms"] for k, v in d["conversions"].items() if isinstance(v, dict)})
PY
echo final_ok
