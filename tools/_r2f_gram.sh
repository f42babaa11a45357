#!/bin/bash
# k_gram_sym at C5: launch-list time/DRAM bytes and one --set full capture.
cd "$(dirname "$0")/.."
mkdir -p gpurun_out
C5_ITERS=1 timeout 600 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
    -k regex:"k_gram|k_dense" --csv --log-file gpurun_out/gram_c5_r2f.csv python tools/c5_diag.py > /dev/null 2>&1
python tools/ncu_list.py gpurun_out/gram_c5_r2f.csv
C5_ITERS=1 timeout 900 ncu --set full --import-source on --clock-control none -k regex:k_gram_sym -c 1 -f -o gpurun_out/r2f_k_gram_sym python tools/c5_diag.py > /dev/null 2>&1
ls -la gpurun_out/r2f_k_gram_sym.ncu-rep
