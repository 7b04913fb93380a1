for L in paper_2304_09511_b200/libspmv_b200.so paper_2304_09511_b200/_ab/libspmv_b200_b16_m3.so paper_2304_09511_b200/_ab/libspmv_b200_b32_m3.so paper_2304_09511_b200/_ab/libspmv_b200_b16_m4.so; do
 for combo in "c5 csr" "c4 csr" "c3 csr" "c5 coo"; do set -- $combo
  SPMV_B200_LIB=$PWD/$L python bench.py --config $1 --format $2 --no-extras --steps 40 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); v=d['per_format']['$2']; print('$(basename $L) $1 $2', v['gflops'], v['roofline_frac'])"
 done
done
