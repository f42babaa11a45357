#!/bin/bash
# C5 front-end timing + filter trace, C2 timing, then the bit-exact full-size and parity suites.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C5_ITERS=2 timeout 300 python tools/c5_diag.py > gpurun_out/c5_diag.log 2>&1; tail -2 gpurun_out/c5_diag.log
CTD_FILTER_TRACE=1 C5_ITERS=1 timeout 300 python tools/c5_diag.py > gpurun_out/c5_trace.log 2>&1; grep -E "cycles/candidate|cand (1476|2952)" gpurun_out/c5_trace.log | grep -oE "cycles/candidate.*|P2 ring.*|cand [0-9]+: [0-9 ]+"
timeout 300 python tools/c2_trace.py 4 2>&1 | grep "front end"
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_stream_c3.py -x -q -m gpu 2>&1 | tail -3
