for cfg in "2048 0" "2048 3" "2048 2" "4096 0" "4096 1"; do set -- $cfg
SPMV_TILE=$1 SPMV_CTAS_PER_SM=$2 python bench.py --config c5 --format csr --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['csr']; print('tile $1 ctas $2', v['gflops'], v['roofline_frac'])"
done
