# C1 (64^3, L2 flushed between steps): CSR / COO tile x groups and the DIA presets, one line each.
run() {  # format, settings...
  f=$1; shift
  env "$@" python bench.py --config c1 --format $f --no-extras --steps 100 --cpu-budget 1 2>/dev/null | python -c "
import json,sys
d=json.loads(sys.stdin.read()); v=d['per_format']['$f']
print('c1 %-4s %-40s %8.1f GFLOP/s %7.2f us frac %.3f plan %s' % ('$f', '$*', v['gflops'], v['ms_per_spmv']*1000, v['roofline_frac'], v.get('plan')))"
}
run csr X=0
for t in 1024 1664 2048 2304; do for g in 1 3 4; do run csr SPMV_TILE=$t SPMV_CSR_GROUPS=$g; done; done
run csr SPMV_CTAS_PER_SM=1
run coo X=0
for t in 1024 1536 2048; do for g in 1 6 7; do run coo SPMV_TILE=$t SPMV_COO_GROUPS=$g; done; done
run dia X=0
for c in 0 1 2 3 4; do run dia SPMV_DIA_CFG=$c; done
for r in 64 128 256; do run dia SPMV_DIA_ROWS=$r; done
