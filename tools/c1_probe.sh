# C1 (64^3): launch list (cold, serialised) and full captures of the CSR tile and DIA kernels.
mkdir -p gpurun_out
ncu --metrics gpu__time_duration.sum --clock-control none -c 300 --csv --log-file gpurun_out/c1_launches.csv python bench.py --config c1 --no-extras --steps 10 --warmup 3 --cpu-budget 1 > gpurun_out/c1_ncu.log 2>&1
python - <<'PY'
import csv, collections
rows = [r for r in csv.reader(open("gpurun_out/c1_launches.csv")) if len(r) > 10 and r[0].isdigit()]
agg = collections.defaultdict(list)
for r in rows:
    agg[r[4][:70]].append(float(r[-1]))
for k, v in agg.items():
    v = sorted(v)
    print(f"{k:72s} n={len(v):3d} median={v[len(v)//2]/1000:8.1f} us min={v[0]/1000:8.1f}")
PY
for k in csr_tile_kernel dia_bulk_kernel; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -f -o gpurun_out/c1_$k python bench.py --config c1 --format ${k:0:3} --no-extras --steps 3 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_c1_$k.log 2>&1
  tail -2 gpurun_out/ncu_c1_$k.log
done
ls -la gpurun_out/c1_*.ncu-rep
