# Launch list (cold, serialised) of the conversions bench: per-kernel medians.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/conv_launches.csv python bench.py --conversions > gpurun_out/ncu_launch_conv.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/conv_launches.csv")) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4][:70]].append(float(r[-1]))
for k, v in agg.items():
    v = sorted(v)
    print(f"{k:72s} n={len(v):3d} median={v[len(v)//2]/1000:9.1f} us")
PY
