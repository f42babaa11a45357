import sys, time, numpy as np, torch
sys.path.insert(0, '.')
import bench
from paper_1710_03608_b200 import ctd as api
x = bench.load_c3()
ctx = api.Context(0, torch.cuda.current_stream().cuda_stream)
H = int(sys.argv[1]) if len(sys.argv) > 1 else 900
hist = x.time_slab(0, H)
st = api.init_stream(api.SparseTensor.from_datagen(hist), 0, int(sys.argv[2]) if len(sys.argv) > 2 else 500, 1e-6, 42, ctx=ctx)
slabs = bench.time_slices(x, H, H + 4)
print("K after init:", len(st.factors().kept_flat), flush=True)
for i, v in slabs:
    d = api.DeviceTensor(api.SparseTensor([5000, 5000, 1], i, v), ctx)
    torch.cuda.synchronize(); t0 = time.perf_counter()
    api.ctd_d_step(st, d, 500)
    torch.cuda.synchronize(); print("step ms", (time.perf_counter() - t0) * 1e3, flush=True)
