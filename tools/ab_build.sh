#!/bin/bash
# Build libspmv_b200.so from git revision $1 into paper_2304_09511_b200/_ab/libspmv_b200_$1.so
set -e
rev=$1
out=/root/repo/paper_2304_09511_b200/_ab
mkdir -p $out
tmp=$(mktemp -d)
git -C /root/repo archive $rev | tar -x -C $tmp
python $tmp/paper_2304_09511_b200/_build.py > /dev/null
cp $tmp/paper_2304_09511_b200/libspmv_b200.so $out/libspmv_b200_$rev.so
rm -rf $tmp
echo $out/libspmv_b200_$rev.so
