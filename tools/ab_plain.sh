# A/B of _ab libraries on plain products: NAMES="a b" [CONFIGS="c5:csr c4:csr"]
for rep in 1 2; do for combo in ${CONFIGS:-c5:csr c5:coo c4:csr c1:csr}; do c=${combo%%:*}; f=${combo##*:}; for n in $NAMES; do
  SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config $c --format $f --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$f']; print('$c $f $n', v['gflops'], v['roofline_frac'])"
done; done; done
