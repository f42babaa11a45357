"""Time the relative-error pass on a BASELINE config: python tools/relerr_time.py c2|c5."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1710_03608_b200 as ctd  # noqa: E402
from paper_1710_03608_b200 import ctd as api  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
ctx = ctd.Context(0, torch.cuda.current_stream().cuda_stream)
dev = torch.device("cuda", 0)
if which == "c5":
    from paper_1710_03608_b200 import datagen_gpu
    idx, val, meta = datagen_gpu.traffic(bench.C5["shape"], bench.C5["nnz"], bench.C5["gen_seed"])
    shape, nnz, cfg = bench.C5["shape"], meta["nnz"], bench.C5
    ptrs = [idx[k].data_ptr() for k in range(3)]
else:
    x = bench.load_c2(0)
    cfg = bench.C2
    idx_t = torch.from_numpy(np.ascontiguousarray(x.idx.T.astype(np.int32))).to(dev)
    val = torch.from_numpy(x.val).to(dev)
    shape, nnz = x.shape, x.nnz
    ptrs = [idx_t[k].data_ptr() for k in range(3)]
torch.cuda.empty_cache()
dt = api.DeviceTensor.from_device_ptrs(shape, nnz, ptrs, val.data_ptr(), ctx)
h, info = api.ctd_s_raw(dt, cfg["mode"], cfg["c"], cfg["eps"], cfg["seed"], ctx=ctx, keep_panel=True)
for it in range(3):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    rel = api.relative_error_raw(dt, h, ctx)
    torch.cuda.synchronize()
    print(f"{which} relative_error call {it}: {1e3 * (time.perf_counter() - t0):.1f} ms  value {rel!r}", flush=True)
