# Round-1 evidence: launch list of the default bench and full captures of the top kernels.
set -e
python bench.py --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/plain_default.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 120 --csv --log-file gpurun_out/r1_launches_c5.csv python bench.py --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch.log 2>&1
for f in csr dia coo; do
  python bench.py --no-extras --format $f --steps 3 --warmup 3 > gpurun_out/plain_$f.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"csr_tile|dia_bulk|coo_tile" -s 2 -c 1 -o gpurun_out/r1_c5_$f python bench.py --no-extras --format $f --steps 3 --warmup 3 > gpurun_out/ncu_$f.log 2>&1
done
python bench.py --config c3 --no-extras --steps 3 --warmup 3 > gpurun_out/plain_c3.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:"csr_tile|csr_span" -s 2 -c 2 -o gpurun_out/r1_c3_csr python bench.py --config c3 --no-extras --steps 3 --warmup 3 > gpurun_out/ncu_c3.log 2>&1
for f in csr dia; do
  python bench.py --config c4 --no-extras --format $f --steps 3 --warmup 3 > gpurun_out/plain_c4_$f.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"csr_tile|dia_bulk" -s 2 -c 1 -o gpurun_out/r1_c4_$f python bench.py --config c4 --no-extras --format $f --steps 3 --warmup 3 > gpurun_out/ncu_c4_$f.log 2>&1
done
echo profile_ok
