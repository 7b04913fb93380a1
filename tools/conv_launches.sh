# Conversions at 256^3: bench numbers, then the launch list of the last sort_coo call (cold, serialised).
mkdir -p gpurun_out
python bench.py --conversions > gpurun_out/conv.json 2> gpurun_out/conv.err || tail -3 gpurun_out/conv.err
python - <<'PY'
import json
d = json.load(open("gpurun_out/conv.json"))["conversions"]
for k, v in d.items():
    if isinstance(v, dict):
        print(f"{k:26s} {v['ms']:8.3f} ms  frac {v['roofline_frac']:.3f}")
PY
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/conv_launches.csv python bench.py --conversions > /dev/null 2>&1
python - <<'PY'
import csv
rows = [r for r in csv.reader(open("gpurun_out/conv_launches.csv")) if len(r) > 10 and r[0].isdigit()]
idx = [i for i, r in enumerate(rows) if "sort_pack_kernel" in r[4]]
if idx:
    for r in rows[idx[-1] - 1: idx[-1] + 12]:
        print(f"{r[4][:90]:92s} {float(r[-1])/1000:9.1f} us")
PY
