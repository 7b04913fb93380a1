# Round-2 closing evidence after the COO row-pointer view: default bench line, launch lists (c5, c3).
mkdir -p gpurun_out
python bench.py > gpurun_out/r2c_bench_default.json 2> gpurun_out/r2c_bench_default.err || { tail -5 gpurun_out/r2c_bench_default.err; exit 1; }
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2c_launches_c5.csv python bench.py --steps 20 --warmup 3 --cpu-budget 1 --no-per-config > gpurun_out/ncu_launch_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2c_launches_c3.csv python bench.py --config c3 --no-extras --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch_c3.log 2>&1
python bench.py --config c1 > gpurun_out/r2c_bench_c1.json 2> gpurun_out/r2c_bench_c1.err
python bench.py --config c4 > gpurun_out/r2c_bench_c4.json 2> gpurun_out/r2c_bench_c4.err
echo profile_ok
