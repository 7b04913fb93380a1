# Refresh the ncu full captures of the current kernels (one launch each, after a plain run).
set -e
for spec in "c5 dia dia_bulk" "c5 coo coo_tile" "c4 csr csr_tile" "c4 dia dia_bulk"; do
  set -- $spec
  python bench.py --config $1 --format $2 --no-extras --steps 3 --warmup 3 > gpurun_out/plain_$1_$2.json 2>&1
  ncu --set full --clock-control none --import-source on -k regex:"$3" -s 3 -c 1 -o gpurun_out/r1_$1_$2 python bench.py --config $1 --format $2 --no-extras --steps 3 --warmup 3 > gpurun_out/ncu_$1_$2.log 2>&1
done
echo refresh_ok
