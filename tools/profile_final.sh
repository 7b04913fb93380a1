# Final round-1 evidence for the default bench (c5): plain run, launch list, full capture of the headline kernel.
set -e
python bench.py --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/plain_default.json 2> gpurun_out/plain_default.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/r1_launches_c5.csv python bench.py --steps 20 --warmup 3 --cpu-budget 1 > gpurun_out/ncu_launch.log 2>&1
python bench.py --no-extras --steps 3 --warmup 3 > gpurun_out/plain_csr.json 2>&1
ncu --set full --clock-control none --import-source on -k regex:"csr_tile" -s 3 -c 1 -o gpurun_out/r1_c5_csr python bench.py --no-extras --steps 3 --warmup 3 > gpurun_out/ncu_csr.log 2>&1
echo profile_ok
