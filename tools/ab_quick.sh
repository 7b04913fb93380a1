# A vs B on a few combos, 2 rounds
A=${A:-paper_2304_09511_b200/libspmv_b200.so}; B=${B:-paper_2304_09511_b200/_ab/libspmv_b200_HEAD.so}
for combo in ${COMBOS:-"c5 csr" "c5 coo" "c3 csr" "c4 csr"}; do
  set -- $combo
  for L in $A $B $A $B; do
    SPMV_B200_LIB=$PWD/$L python bench.py --config $1 --format $2 --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$2']; print('$1 $2 $(basename $L)', v['gflops'], v['roofline_frac'])"
  done
done
