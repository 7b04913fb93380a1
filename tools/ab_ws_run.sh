#!/bin/bash
# Alternate _ab/ libraries on one config/format (GPU box): NAMES="a b" CFG=c3 FMT=csr
for rep in 1 2; do
  for n in $NAMES; do
    L=paper_2304_09511_b200/_ab/libspmv_b200_$n.so
    SPMV_B200_LIB=$PWD/$L python bench.py --config ${CFG:-c3} --format ${FMT:-csr} --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['${FMT:-csr}']; print('$n', v['gflops'], v['roofline_frac'])"
  done
done
