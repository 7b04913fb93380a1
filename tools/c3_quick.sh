# C3 quick look on one B200: bench line, launch list (cold, serialised), optional full captures.
mkdir -p gpurun_out
python bench.py --config c3 --no-extras --steps 100 --warmup 5 > gpurun_out/c3_q.json 2> gpurun_out/c3_q.err || { tail -5 gpurun_out/c3_q.err; exit 1; }
python - <<'PY'
import json
d = json.load(open("gpurun_out/c3_q.json"))
for k, v in d["per_format"].items():
    print(k, v["gflops"], v["ms_per_spmv"], v["roofline_frac"])
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c3_q_launches.csv python bench.py --config c3 --no-extras --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/c3_q_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/c3_q_launches.csv")) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4][:60]].append(float(r[-1]))
for k, v in agg.items():
    v = sorted(v)
    print(f"{k:62s} n={len(v):3d} median={v[len(v)//2]/1000:8.1f} us")
PY
if [ -n "$FULL" ]; then
for k in $FULL; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -f -o gpurun_out/c3_q_$k python bench.py --config c3 --no-extras --steps 3 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_$k.log 2>&1
done
fi
