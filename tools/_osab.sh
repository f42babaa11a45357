#!/bin/bash
# A/B of onesweep builds: bit-exact bucketing tests on the default build, then
# device-timed matricize at C2 and C5 for the default and each named variant
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_capi.py -m gpu -x -q 2>&1 | tail -5
for v in "" "$@"; do
  lib=""; [ -n "$v" ] && lib=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so
  for w in c2 c5; do
    CTD_GPU_LIB=$lib timeout 600 python tools/matricize_prof.py $w 4 2>&1 | tail -3 | sed "s/^/[${v:-default}] /"
  done
done
