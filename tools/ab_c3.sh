# A/B of _ab libraries on the Zipf config: NAMES="a b"
for rep in 1 2; do for f in csr coo; do for n in $NAMES; do
SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config c3 --format $f --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$f']; print('c3 $f $n', v['gflops'], v['roofline_frac'])"
done; done; done
