#!/bin/bash
# per-kernel times (ncu launch list, k_os_* only) of C5 matricize for the default build and each named variant
cd "$(dirname "$0")/.."
W=${W:-c5}
for rep in 1 2; do
for v in "" "$@"; do
  lib=""; [ -n "$v" ] && lib=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so
  CTD_GPU_LIB=$lib ncu --metrics gpu__time_duration.sum --clock-control none -k regex:k_os --csv \
     --log-file gpurun_out/_osl.csv python tools/matricize_prof.py $W 1 > /dev/null 2>&1
  echo "[${v:-default}] $(python tools/ncu_list.py gpurun_out/_osl.csv | awk '/k_os/{printf "%s=%.0f ", substr($2,index($2,"k_os")+5), $3} /total/{print "total", $2}')"
done
done
