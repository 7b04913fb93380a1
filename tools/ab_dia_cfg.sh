for r in 1 2; do
 for c in c5 c4; do
  SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_HEAD.so python bench.py --config $c --format dia --no-extras --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['dia']; print('HEAD $c', v['gflops'], v['roofline_frac'])"
  for cfg in 0 1 2 3 4; do
   SPMV_DIA_CFG=$cfg python bench.py --config $c --format dia --no-extras --steps 50 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['dia']; print('cfg$cfg $c', v['gflops'], v['roofline_frac'])"
  done
 done
done
