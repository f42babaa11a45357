#!/bin/bash
# filter trace per variant at C5 (one front end each)
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  CTD_FILTER_TRACE=1 CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so C5_ITERS=1 python tools/c5_diag.py > gpurun_out/tr_$v.log 2>&1
  grep -E "iter 0|cycles/candidate" gpurun_out/tr_$v.log | cut -c1-250
  grep -E "cand (1476|2952)" gpurun_out/tr_$v.log | grep -oE "P2 chain.*"
done
