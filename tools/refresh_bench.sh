# Refresh the committed bench lines (profiles/r1_bench_*.json) on one B200.
set -e
for c in c5 c3 c4 c1; do
  python bench.py --config $c --steps 100 > gpurun_out/r1_bench_$c.json 2> gpurun_out/r1_bench_$c.err
done
python bench.py --conversions > gpurun_out/r1_conversions_c5.json 2> gpurun_out/r1_conversions_c5.err
echo refresh_ok
