#!/bin/bash
# Round-2 final check under gpurun: smoke(), the GPU suite, the default bench line, the reference arm.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
timeout 300 python -c "import __graft_entry__ as g; g.smoke(); print('smoke ok')" 2>&1 | tail -2
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/gputest_r2f.log 2>&1; echo "pytest rc=$?" >> gpurun_out/gputest_r2f.log
tail -3 gpurun_out/gputest_r2f.log
timeout 1200 python bench.py > gpurun_out/bench_r2f.json 2> gpurun_out/bench_r2f.err || { echo "bench failed"; tail gpurun_out/bench_r2f.err; }
tail -c 200 gpurun_out/bench_r2f.json
timeout 600 python bench.py --impl reference --steps 1 --warmup 0 > gpurun_out/bench_r2f_ref.json 2> gpurun_out/bench_r2f_ref.err; echo "ref rc=$?"; tail -c 600 gpurun_out/bench_r2f_ref.json
