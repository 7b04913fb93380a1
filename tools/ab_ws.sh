#!/bin/bash
# Build warp-stream variants (SPMV_NVCC_EXTRA macro sets) into _ab/: name=flags
set -e
out=/root/repo/paper_2304_09511_b200/_ab
mkdir -p $out
for spec in "$@"; do
  name=${spec%%=*}; flags=${spec#*=}
  tmp=$(mktemp -d)
  cp -r /root/repo/paper_2304_09511_b200 /root/repo/include $tmp/
  rm -rf $tmp/paper_2304_09511_b200/_ab $tmp/paper_2304_09511_b200/_objs
  SPMV_NVCC_EXTRA="$flags" python $tmp/paper_2304_09511_b200/_build.py > /dev/null
  cp $tmp/paper_2304_09511_b200/libspmv_b200.so $out/libspmv_b200_$name.so
  rm -rf $tmp
  echo $out/libspmv_b200_$name.so
done
