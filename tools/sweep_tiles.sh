set -x
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo pytest_rc=$?; tail -3 gpurun_out/pytest_gpu.log
SPMV_TILE=1024 timeout 600 python -m pytest tests/test_gpu_kernels.py -m gpu -x -q > gpurun_out/pytest_gpu_t1024.log 2>&1; echo pytest1024_rc=$?; tail -3 gpurun_out/pytest_gpu_t1024.log
for t in 1024 2048; do for f in csr coo; do SPMV_TILE=$t python bench.py --no-extras --format $f --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('TILE $t $f', d['per_format']['$f'])"; done; done
for r in 128 256 512; do for s in 2 3; do SPMV_DIA_ROWS=$r SPMV_DIA_STAGES=$s python bench.py --no-extras --format dia --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('DIA rows $r stages $s', d['per_format']['dia'])"; done; done
