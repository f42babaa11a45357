"""C2 front end with the filter's clock64 trace (run with CTD_FILTER_TRACE=1)."""
import sys, time
sys.path.insert(0, '.')
import bench
from paper_1710_03608_b200 import ctd as api
x = bench.load_c2()
ctx = api.Context(0)
t = api.DeviceTensor(api.SparseTensor.from_datagen(x), ctx)
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 2):
    t0 = time.perf_counter()
    f = api.ctd_s(t, 0, 2000, 1e-6, 42, ctx=ctx)
    print("front end ms", (time.perf_counter() - t0) * 1e3, "kept", f.kept_count(), flush=True)
