#!/bin/bash
# Round-2 profiles (run under gpurun): launch lists + ncu --set full captures.
cd "$(dirname "$0")/.."
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ctdd --no-c4 --no-c5"
$B > gpurun_out/b_r2.log 2>&1 || { echo "bench failed"; tail gpurun_out/b_r2.log; exit 1; }
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r2.csv $B > /dev/null 2>&1
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-ctdd --no-c4 --no-c5"
for k in k_filter k_os_pass k_cdw k_gemm k_seq_local k_spec_y; do
  ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -o gpurun_out/r2_$k $B1 > /dev/null 2>&1
done
# C4 (speculative rejection batches)
ncu --set full --import-source on --clock-control none -k regex:"k_spec_y|k_spec_res" -c 2 -o gpurun_out/r2_spec \
    python tools/filter_ab.py c4 a > /dev/null 2>&1
C5_ITERS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^k_" --csv --log-file gpurun_out/launches_c5_r2.csv python tools/c5_diag.py > /dev/null 2>&1
ls -la gpurun_out/*r2*
