# ncu --set full of one k_filter launch (C2 front end), variant lib in $1
export CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$1.so
python tools/c2_trace.py 1 > gpurun_out/ncu_pre.log 2>&1 || exit 1
ncu --set full --import-source on --clock-control none -k regex:k_filter -c 1 -o gpurun_out/filt_$1 -f python tools/c2_trace.py 1 > gpurun_out/ncu_$1.log 2>&1
tail -3 gpurun_out/ncu_$1.log
