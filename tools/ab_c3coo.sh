for rep in 1 2 3; do for n in $NAMES; do
SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config c3 --format coo --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['coo']; print('c3 coo $n', v['gflops'], v['roofline_frac'])"
done; done
