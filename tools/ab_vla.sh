# A/B of _ab libraries on the vla(8) products: NAMES="a b" [CONFIGS="c5 c4"]
for rep in 1 2; do for c in ${CONFIGS:-c5 c4}; do for n in $NAMES; do
  SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config $c --steps 40 --cpu-budget 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format_vla']; print('$c $n', {k:(x['gflops'],x['roofline_frac']) for k,x in v.items() if k != 'dia'})"
done; done; done
