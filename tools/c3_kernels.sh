# C3 CSR per-kernel times (ncu launch list, cold) for each environment setting given as an argument.
mkdir -p gpurun_out
for setting in "$@"; do
  env $setting ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/c3_k.csv python bench.py --config c3 --no-extras --steps 5 --warmup 3 --cpu-budget 1 > gpurun_out/c3_k.log 2>&1
  python - "$setting" <<'PY'
import csv, collections, sys
rows = [r for r in csv.reader(open("gpurun_out/c3_k.csv")) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4].split("(")[0][-40:]].append(float(r[-1]))
out = []
for k, v in agg.items():
    if len(v) >= 8:
        v = sorted(v)
        out.append(f"{k.split('::')[-1]} {v[len(v)//2]/1000:.1f}")
print(sys.argv[1], "|", " | ".join(out))
PY
done
