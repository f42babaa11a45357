#!/bin/bash
# C3 CTD-D step latency (lazy core, 500 bootstrap slices + 500 steps) per library build
cd "$(dirname "$0")/.."
for v in "$@"; do
  echo "== $v"
  CORE=lazy SPIKE_MS=25 CTD_ARENA_TRACE=1 CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so \
    timeout 600 python tools/ctdd_phases.py 500 500 2>&1 | grep -E "p50|arena|step [2-9][0-9]\.|step [0-9]{3}" | cut -c1-220 | tail -30
done
