"""C5 (1e9 nnz) diagnostics: generate on the device, run one CTD-S front end with
the host/seq-sum traces on (CTD_HOST_TRACE, CTD_SEQ_TRACE), print phase times."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_1710_03608_b200 as ctd  # noqa: E402
from paper_1710_03608_b200 import ctd as api  # noqa: E402
from paper_1710_03608_b200 import datagen_gpu  # noqa: E402

scale = float(os.environ.get("C5_SCALE", "1"))
t0 = time.perf_counter()
idx, val, meta = datagen_gpu.c5(scale=scale)
torch.cuda.synchronize()
print("gen", round(time.perf_counter() - t0, 2), meta, flush=True)
torch.cuda.empty_cache()
shape = [100000, 100000, max(1, int(round(1000 * scale)))]
ctx = ctd.Context(0, torch.cuda.current_stream().cuda_stream)
dt = api.DeviceTensor.from_device_ptrs(shape, meta["nnz"], [idx[k].data_ptr() for k in range(3)],
                                       val.data_ptr(), ctx)
for it in range(int(os.environ.get("C5_ITERS", "2"))):
    ctx.set_timing(True)
    ctx.phase_times(reset=True)
    t0 = time.perf_counter()
    h, info = api.ctd_s_raw(dt, 0, 10000, 1e-6, 42, ctx=ctx)
    torch.cuda.synchronize()
    print("iter", it, round(time.perf_counter() - t0, 3), "s; F", info.n_fibers, "unique", info.n_unique,
          "kept", info.kept, {k: round(v[0] / max(1, v[1]), 2) for k, v in ctx.phase_times(reset=True).items()
                              if v[1]}, flush=True)
    api.free_factors(ctx, h)
