for rep in 1 2; do for ws in 0 1; do for f in csr coo; do
SPMV_CSR_WS=$ws SPMV_COO_WS=$ws python bench.py --config c1 --format $f --no-extras --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$f']; print('c1 $f ws=$ws', v['gflops'], v['roofline_frac'])"
done; done; done
