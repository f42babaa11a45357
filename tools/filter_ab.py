"""A/B the filter on BASELINE configs (device time of the ctd_s front end and
its filter phase), e.g. with and without CTD_NO_SPEC=1, and check the outcome
is bit-identical between the two runs (written to/compared with a .npz)."""
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

which = sys.argv[1] if len(sys.argv) > 1 else "c4"
tag = sys.argv[2] if len(sys.argv) > 2 else "a"
ctx = ctd.Context(0, torch.cuda.current_stream().cuda_stream)
if which == "c4":
    x, cfg = bench.load_c4(), bench.C4
elif which == "c2":
    x, cfg = bench.load_c2(0), bench.C2
dev = torch.device("cuda", 0)
idx_t = torch.from_numpy(np.ascontiguousarray(x.idx.T.astype(np.int32))).to(dev)
val_t = torch.from_numpy(x.val).to(dev)
dt = api.DeviceTensor.from_device_ptrs(x.shape, x.nnz, [idx_t[k].data_ptr() for k in range(3)], val_t.data_ptr(), ctx)
ms, info, phases, launches = bench._time_frontend(ctx, dt, cfg, 3, 1, torch)
h, info = api.ctd_s_raw(dt, cfg["mode"], cfg["c"], cfg["eps"], cfg["seed"], ctx=ctx)
kept, u = api.factors_result(ctx, h, info)
tr = api.factors_trace(ctx, h, info)
delta = np.zeros(max(info.n_unique, 1))
ctx.L.ctd_gpu_factors_trace(h, None, None, None, None, api._p(delta))
api.free_factors(ctx, h)
print(f"{which} {tag}: {ms:.3f} ms/step phases={phases} launches={launches} kept={info.kept} "
      f"unique={info.n_unique}", flush=True)
out = os.path.join(ROOT, "gpurun_out", f"ab_{which}.npz")
if os.path.exists(out) and tag != "a":
    z = np.load(out)
    same = (np.array_equal(z["kept"], kept) and np.array_equal(z["u"].view(np.int64), u.view(np.int64))
            and np.array_equal(z["acc"], tr["accepted"]) and np.array_equal(z["delta"].view(np.int64), delta.view(np.int64)))
    print(f"{which}: identical to run a: {same}", flush=True)
    assert same
else:
    np.savez(out, kept=kept, u=u, acc=tr["accepted"], delta=delta)
