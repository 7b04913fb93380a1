# A/B: bench the same workload with two library builds, alternating.
A=${A:-paper_2304_09511_b200/libspmv_b200.so}; B=${B:-paper_2304_09511_b200/_ab/libspmv_b200_HEAD.so}
CFG=${CFG:-c5}; FMT=${FMT:-csr}
for i in 1 2; do for L in $A $B; do
  SPMV_B200_LIB=$PWD/$L python bench.py --config $CFG --format $FMT --no-extras --steps 50 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('$L', {k:(v['gflops'],v['roofline_frac']) for k,v in d['per_format'].items()})"
done; done
