for v in "$@"; do
  echo "== $v"
  CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so python tools/c2_trace.py 2 2>&1 | tail -2
  CTD_FILTER_TRACE=1 CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so python tools/c2_trace.py 1 2>&1 | grep -E "cycles/cand|cand 632|cand 1264" | cut -c1-420
done
