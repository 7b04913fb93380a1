for rep in 1 2; do for cfg in -1 3 4; do for rows in 0 256; do
SPMV_DIA_CFG=$cfg SPMV_DIA_ROWS=$rows python bench.py --config c4 --format dia --no-extras --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['dia']; print('c4 dia cfg=$cfg rows=$rows', v['gflops'], v['roofline_frac'])"
done; done; done
