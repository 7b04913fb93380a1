#!/bin/bash
# A/B environment settings on one library: ENVS="SPMV_TILE=2048 SPMV_TILE=1664" COMBOS="c5:csr" tools/ab_env.sh
ENVS=${ENVS:-"X=1"}; COMBOS=${COMBOS:-"c5:csr"}; ROUNDS=${ROUNDS:-2}; STEPS=${STEPS:-50}
for r in $(seq $ROUNDS); do for c in $COMBOS; do cfg=${c%%:*}; fmt=${c#*:}; for e in $ENVS; do
  env ${e//,/ } python bench.py --config $cfg --format $fmt --no-extras --steps $STEPS 2>/dev/null \
   | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$fmt']; print('$e $cfg $fmt', v['gflops'], v['roofline_frac'])"
done; done; done
