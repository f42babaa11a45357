#!/bin/bash
# Round-2 (session e) baseline under gpurun: the GPU suite and the default bench line.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2e.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r2e.log
tail -3 gpurun_out/gputest_r2e.log
timeout 1200 python bench.py > gpurun_out/bench_r2e.json 2> gpurun_out/bench_r2e.err || { echo "bench failed"; tail gpurun_out/bench_r2e.err; }
tail -c 400 gpurun_out/bench_r2e.json
