# Warp-stream kernels on the Zipf config: bench line + ncu full captures (CSR, COO).
set -e
python bench.py --config c3 --steps 50 > gpurun_out/r1_bench_c3.json 2> gpurun_out/r1_bench_c3.err
for f in csr coo; do
  python bench.py --config c3 --format $f --no-extras --steps 3 --warmup 3 > gpurun_out/plain_c3_$f.log 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"wstream|span_fixup" -s 2 -c 2 -o gpurun_out/r1_c3_ws_$f python bench.py --config c3 --format $f --no-extras --steps 3 --warmup 3 > gpurun_out/ncu_c3_$f.log 2>&1
done
ncu --metrics gpu__time_duration.sum --clock-control none -c 60 --csv --log-file gpurun_out/r1_launches_c3.csv python bench.py --config c3 --steps 10 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch_c3.log 2>&1
echo profile_ok
