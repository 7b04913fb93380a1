for rep in 1 2; do for m in 0 1; do
SPMV_TILE_MODE=$m python bench.py --config c4 --format csr --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['csr']; print('c4 csr mode=$m', v['gflops'], v['roofline_frac'], v['plan'])"
done; done
