for rep in 1 2; do for g in 0 6; do
SPMV_TILE=1536 SPMV_COO_GROUPS=$g python bench.py --format coo --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['coo']; print('c5 coo g=$g', v['gflops'], v['plan'])"
done; done
