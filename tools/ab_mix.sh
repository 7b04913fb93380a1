for rep in 1 2; do for n in $NAMES; do
for combo in c5:csr c5:coo c4:csr; do c=${combo%%:*}; f=${combo##*:};
  SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config $c --format $f --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$f']; print('$c $f $n', v['gflops'])"
done
SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config c3 --steps 30 --cpu-budget 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c3 vla $n', {k:x['gflops'] for k,x in d['per_format_vla'].items()})"
SPMV_B200_LIB=$PWD/paper_2304_09511_b200/_ab/libspmv_b200_$n.so python bench.py --config c5 --steps 30 --cpu-budget 1 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('c5 vla $n', {k:x['gflops'] for k,x in d['per_format_vla'].items() if k!='dia'})"
done; done
