# Run A/B for several (config, format, tile) combos; one line each.
A=${A:-paper_2304_09511_b200/libspmv_b200.so}; B=${B:-paper_2304_09511_b200/_ab/libspmv_b200_HEAD.so}
for combo in "c5 csr 2048" "c5 coo 2048" "c5 dia 2048" "c3 csr 2048" "c3 coo 2048" "c3 csr 1024" "c3 coo 1024" "c4 csr 2048" "c4 dia 2048"; do
  set -- $combo
  for L in $A $B; do
    SPMV_TILE=$3 SPMV_B200_LIB=$PWD/$L python bench.py --config $1 --format $2 --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$2']; print('$1 $2 tile=$3 $(basename $L)', v['gflops'], v['roofline_frac'])"
  done
done
