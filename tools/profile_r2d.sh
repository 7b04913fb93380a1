# Round-2 closing evidence (session 5): GPU suite, smoke, default bench line, reference arm, launch lists (c5, c3),
# full captures of the headline kernels (traffic per launch), c1 / c3 / c4 lines, conversions launch list.
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/r2d_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2d_gputests.log
tail -4 gpurun_out/r2d_gputests.log
python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" > gpurun_out/r2d_smoke.log 2>&1; tail -2 gpurun_out/r2d_smoke.log
python bench.py > gpurun_out/r2d_bench_default.json 2> gpurun_out/r2d_bench_default.err || { tail -5 gpurun_out/r2d_bench_default.err; exit 1; }
python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/r2d_bench_reference.json 2> gpurun_out/r2d_bench_reference.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 600 --csv --log-file gpurun_out/r2d_launches_c5.csv python bench.py --steps 20 --warmup 3 --cpu-budget 1 --no-per-config > gpurun_out/ncu_launch_c5.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2d_launches_c3.csv python bench.py --config c3 --no-extras --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch_c3.log 2>&1
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2d_launches_conversions.csv python bench.py --conversions > gpurun_out/ncu_launch_conv.log 2>&1
for f in csr dia coo; do
  ncu --set full --clock-control none --import-source on -k regex:"csr_tile_kernel|dia_bulk_kernel" -s 3 -c 1 -f -o gpurun_out/r2d_c5_$f python bench.py --format $f --no-extras --steps 3 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_c5_$f.log 2>&1
done
python bench.py --config c1 > gpurun_out/r2d_bench_c1.json 2> gpurun_out/r2d_bench_c1.err
python bench.py --config c4 > gpurun_out/r2d_bench_c4.json 2> gpurun_out/r2d_bench_c4.err
python bench.py --config c3 > gpurun_out/r2d_bench_c3.json 2> gpurun_out/r2d_bench_c3.err
ls -la gpurun_out/r2d_* | head -40
echo profile_ok
