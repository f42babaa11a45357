#!/bin/bash
# A/B of filter variants (make variant VAR=...): C5 front end and C2 front end per variant.
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so C5_ITERS=2 python tools/c5_diag.py 2>&1 | grep "iter 1" | cut -c1-200
  CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so python tools/c2_trace.py 4 2>&1 | tail -1
done
