for i in 1 2; do
for v in old new; do
  echo "== $v"; CTD_GPU_LIB=paper_1710_03608_b200/csrc/build/libctd_gpu_$v.so python tools/c2_trace.py 4 2>&1 | tail -2
done; done
