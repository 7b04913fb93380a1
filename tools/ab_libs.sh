#!/bin/bash
# A/B several library builds (_ab/libspmv_b200_<name>.so) over workloads, alternating rounds.
# usage: LIBS="base tma x both" COMBOS="c5:csr c5:dia" ROUNDS=2 tools/ab_libs.sh
LIBS=${LIBS:-"base"}; COMBOS=${COMBOS:-"c5:csr"}; ROUNDS=${ROUNDS:-2}; STEPS=${STEPS:-50}
for r in $(seq $ROUNDS); do for c in $COMBOS; do cfg=${c%%:*}; fmt=${c#*:}; for n in $LIBS; do
  SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config $cfg --format $fmt --no-extras --steps $STEPS 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$fmt']; print('$n $cfg $fmt', v['gflops'], v['roofline_frac'])"
done; done; done
