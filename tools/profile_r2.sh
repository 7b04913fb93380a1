# Round-2 evidence on one B200: GPU suite, default bench line, launch lists, full captures of the C3 panel-path kernels.
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/r2_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2_gputests.log
python bench.py > gpurun_out/r2_bench_default.json 2> gpurun_out/r2_bench_default.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2_launches_c5.csv python bench.py --steps 20 --warmup 3 --cpu-budget 1 --no-per-config > gpurun_out/ncu_launch_c5.log 2>&1
python bench.py --config c3 --no-extras --steps 20 --warmup 3 > gpurun_out/r2_c3_plain.json 2> gpurun_out/r2_c3_plain.err || exit 1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2_launches_c3.csv python bench.py --config c3 --no-extras --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch_c3.log 2>&1
for k in short_ell csr_panel_kernel csr_panel_finish; do
  ncu --set full --clock-control none --import-source on -k regex:"$k" -s 3 -c 1 -f -o gpurun_out/r2_c3_$k python bench.py --config c3 --no-extras --steps 3 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_$k.log 2>&1
done
echo profile_ok
