#!/bin/bash
# device-timed A/B of two library builds on C2, C4 (bit-identity checked) and C5
cd "$(dirname "$0")/.."
A=$1; B=$2
for w in c2 c4; do
  for v in $A $B $A $B; do
    tag=b; [ "$v" = "$A" ] && tag=a
    CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so timeout 300 python tools/filter_ab.py $w $tag 2>&1 | grep -E "ms/step|same|differ" | cut -c1-120 | sed "s/^/$v /"
  done
done
for v in $A $B; do
  CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so C5_ITERS=3 timeout 300 python tools/c5_diag.py 2>&1 | grep "iter [12]" | cut -c1-200 | sed "s/^/$v /"
done
