#!/bin/bash
# Round-2 (session e) measurements under gpurun: the default bench line, the C2
# step's launch list, --set full captures of the top kernels, the C5 launch list.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
B="python bench.py --steps 1 --warmup 3 --no-e2e --no-cpu --no-ctdd --no-c4 --no-c5"
timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
    --log-file gpurun_out/launches_r2e.csv $B > /dev/null 2>&1
B1="python bench.py --steps 1 --warmup 0 --no-e2e --no-cpu --no-ctdd --no-c4 --no-c5"
for k in k_filter k_os_pass k_cdw; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:"$k" -c 1 -f -o gpurun_out/r2e_$k $B1 > /dev/null 2>&1
done
C5_ITERS=1 timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^k_" --csv --log-file gpurun_out/launches_c5_r2e.csv python tools/c5_diag.py > /dev/null 2>&1
ls -la gpurun_out/*r2e*
