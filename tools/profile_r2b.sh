# Round-2 final evidence on one B200: GPU suite, default bench line, reference arm, launch lists, group-sort capture.
mkdir -p gpurun_out
( time timeout 2400 python -m pytest tests -m gpu -x -q ) > gpurun_out/r2b_gputests.log 2>&1
echo "pytest exit $?" >> gpurun_out/r2b_gputests.log
tail -3 gpurun_out/r2b_gputests.log
python bench.py > gpurun_out/r2b_bench_default.json 2> gpurun_out/r2b_bench_default.err || { tail -5 gpurun_out/r2b_bench_default.err; exit 1; }
python bench.py --impl reference --steps 5 --warmup 1 > gpurun_out/r2b_bench_reference.json 2> gpurun_out/r2b_bench_reference.err
python bench.py --conversions > gpurun_out/r2b_conversions.json 2> gpurun_out/r2b_conversions.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r2b_launches_conversions.csv python bench.py --conversions > gpurun_out/ncu_conv.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:group_sort_kernel -c 1 -f -o gpurun_out/r2b_group_sort python bench.py --conversions > gpurun_out/ncu_gs.log 2>&1
echo profile_ok
