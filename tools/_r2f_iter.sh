#!/bin/bash
# Round-2 (session f): chunk-major k_gram_sym. Parity suites, C5/C2 phase times, onesweep all-poll A/B.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_fullsize.py tests/test_gpu_parity.py tests/test_gpu_stream_c3.py -x -q -m gpu 2>&1 | tail -3
C5_ITERS=2 timeout 300 python tools/c5_diag.py > gpurun_out/c5_diag_r2f.log 2>&1; tail -2 gpurun_out/c5_diag_r2f.log
timeout 300 python tools/c2_trace.py 4 2>&1 | grep "front end"
W=c5 bash tools/_oslist.sh allpoll 2>&1 | tee gpurun_out/oslist_r2f.log
