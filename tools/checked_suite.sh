#!/bin/bash
# The GPU parity suite against the checked build (device asserts on the hot
# kernels' indices and invariants, CTD_CHECK in csrc/common.cuh): the stand-in
# for compute-sanitizer, which is closed on the GPU pool.  Log: gpurun_out/checked_suite.log
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
export CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_checked.so
{
  echo "checked build: $CTD_GPU_LIB"
  timeout 600 python tools/sanitize_smoke.py 2>&1 | tail -3
  timeout 1500 python -m pytest tests -m gpu -q -x -p no:cacheprovider \
    --deselect tests/test_datagen_gpu.py 2>&1 | tail -5
} > gpurun_out/checked_suite.log 2>&1
cat gpurun_out/checked_suite.log
