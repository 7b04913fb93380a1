for rep in 1 2; do for cfg in -1 2 4 1; do
SPMV_DIA_CFG=$cfg python bench.py --config c1 --format dia --no-extras --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['dia']; print('c1 dia cfg=$cfg', v['gflops'], v['roofline_frac'])"
done; done
