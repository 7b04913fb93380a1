# Warp-stream vs tile kernels on the short-row configs (env overrides).
for cfg in "c5 coo" "c5 csr" "c4 csr"; do set -- $cfg
  for ws in 0 1; do
    SPMV_CSR_WS=$ws SPMV_COO_WS=$ws python bench.py --config $1 --format $2 --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$2']; print('$1 $2 ws=$ws', v['gflops'], v['roofline_frac'])"
  done
done
