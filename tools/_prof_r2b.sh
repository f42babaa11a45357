#!/bin/bash
# Round-2 (second pass) profiles under gpurun: C5 launch list with the current build, a C3
# lazy-core launch list (steps t = 900..909 of the stream) and full captures of the new kernels.
cd "$(dirname "$0")/.."
C5_ITERS=1 python tools/c5_diag.py > gpurun_out/c5_ok.log 2>&1 || { echo "c5 failed"; exit 1; }
C5_ITERS=1 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^k_" --csv --log-file gpurun_out/launches_c5_r2b.csv python tools/c5_diag.py > /dev/null 2>&1
C5_ITERS=1 ncu --set full --import-source on --clock-control none -k regex:"k_gram_sym|k_os_pass" -c 2 \
    -o gpurun_out/r2b_c5 python tools/c5_diag.py > /dev/null 2>&1
CORE=lazy python tools/ctdd_phases.py 900 10 > gpurun_out/ctdd_ok.log 2>&1 || { echo "ctdd failed"; exit 1; }
CORE=lazy ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"^k_" --csv --log-file gpurun_out/launches_c3_r2b.csv python tools/ctdd_phases.py 900 10 > /dev/null 2>&1
CORE=lazy ncu --set full --import-source on --clock-control none -k regex:"k_core|k_gram_cols|k_left_nz" \
    --launch-skip 6 -c 4 -o gpurun_out/r2b_c3core python tools/ctdd_phases.py 900 10 > /dev/null 2>&1
ls -la gpurun_out/*r2b*
