for m in 0 1; do for f in csr coo; do for c in c3 c5; do
SPMV_TILE_MODE=$m python bench.py --config $c --format $f --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$f']; print('mode $m $c $f', v['gflops'], v['roofline_frac'])"
done; done; done
for t in 1024; do for f in csr coo; do SPMV_TILE=$t SPMV_TILE_MODE=1 python bench.py --config c3 --format $f --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$f']; print('tile $t mode 1 c3 $f', v['gflops'], v['roofline_frac'])"; done; done
