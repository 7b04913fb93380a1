# A/B of _ab libraries on DIA: NAMES="a b"
for rep in 1 2; do for n in $NAMES; do for c in c5 c4 c1; do
SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config $c --format dia --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['dia']; print('$c $n', v['gflops'], v['roofline_frac'])"
done; done; done
