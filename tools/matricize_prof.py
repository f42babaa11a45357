"""Matricize alone (bucketing + norms) on a BASELINE config, for launch lists:
    python tools/matricize_prof.py c2|c5 [iters]
Prints the device time per call (CUDA events)."""
import os
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
import paper_1710_03608_b200 as ctd  # noqa: E402
from paper_1710_03608_b200 import ctd as api  # noqa: E402

which = sys.argv[1] if len(sys.argv) > 1 else "c2"
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 3
ctx = ctd.Context(0, torch.cuda.current_stream().cuda_stream)
dev = torch.device("cuda", 0)
if which == "c5":
    from paper_1710_03608_b200 import datagen_gpu
    idx, val, meta = datagen_gpu.traffic(bench.C5["shape"], bench.C5["nnz"], bench.C5["gen_seed"])
    shape, nnz = bench.C5["shape"], meta["nnz"]
    ptrs = [idx[k].data_ptr() for k in range(3)]
else:
    x = bench.load_c2(0) if which == "c2" else bench.load_c4()
    idx_t = torch.from_numpy(np.ascontiguousarray(x.idx.T.astype(np.int32))).to(dev)
    val = torch.from_numpy(x.val).to(dev)
    shape, nnz = x.shape, x.nnz
    ptrs = [idx_t[k].data_ptr() for k in range(3)]
torch.cuda.empty_cache()
dt = api.DeviceTensor.from_device_ptrs(shape, nnz, ptrs, val.data_ptr(), ctx)
F = C_int = None
import ctypes as C  # noqa: E402
for it in range(iters):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    nf = C.c_int64()
    e0.record()
    api._check(ctx.L.ctd_gpu_matricize(ctx.h, dt.h, 0, C.byref(nf), None, None, None, None, None))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{which} matricize: {ms:.3f} ms  F={nf.value}  {(32 * nnz + 24 * nf.value) / ms / 1e6:.1f} GB/s "
          f"(32 nnz + 24 F)", flush=True)
