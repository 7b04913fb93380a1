# C1: L2 prefetch of x / row pointers at kernel start (default) vs none (SPMV_NO_PF=1), alternating.
for rep in 1 2; do for pf in 1 0; do
  if [ $pf = 0 ]; then export SPMV_NO_PF=1; else unset SPMV_NO_PF; fi
  python bench.py --config c1 --no-extras --steps 200 --cpu-budget 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read())
print('c1 prefetch=$pf', {k:(v['gflops'], round(v['ms_per_spmv']*1000,2)) for k,v in d['per_format'].items()})"
done; done
unset SPMV_NO_PF
timeout 900 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_stress.py -m gpu -x -q 2>&1 | tail -3
