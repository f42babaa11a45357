"""C3 CTD-D steps with per-phase device times: init_stream on the first H slices,
then N ctd_d_steps; prints per-step ms and the phase split (every 50th step)."""
import os
import sys
import time

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import bench  # noqa: E402
from paper_1710_03608_b200 import ctd as api  # noqa: E402

H = int(sys.argv[1]) if len(sys.argv) > 1 else 500
N = int(sys.argv[2]) if len(sys.argv) > 2 else 500
x = bench.load_c3()
ctx = api.Context(0, torch.cuda.current_stream().cuda_stream)
hist = x.time_slab(0, H)
LAZY = os.environ.get("CORE", "") == "lazy"
st = api.init_stream(api.SparseTensor.from_datagen(hist), 0, 500, 1e-6, 42, lazy_core=LAZY, ctx=ctx)
slabs = bench.time_slices(x, H, H + N)
dev = [api.DeviceTensor(api.SparseTensor([5000, 5000, 1], i, v), ctx) for i, v in slabs]
lat, agg = [], {}
ctx.set_timing(True)
for k, d in enumerate(dev):
    ctx.phase_times(reset=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    api.ctd_d_step(st, d, 500)
    torch.cuda.synchronize()
    ms = (time.perf_counter() - t0) * 1e3
    lat.append(ms)
    ph = {kk: v[0] for kk, v in ctx.phase_times(reset=True).items() if v[1]}
    for kk, v in ph.items():
        agg[kk] = agg.get(kk, 0.0) + v
    if k % 50 == 0 or ms > float(os.environ.get("SPIKE_MS", "60")):
        print(f"t={H + k} step {ms:.2f} ms  phases {({kk: round(v, 2) for kk, v in ph.items()})}", flush=True)
lat = np.array(lat)
print(f"p50 {np.percentile(lat, 50):.2f} p99 {np.percentile(lat, 99):.2f} mean {lat.mean():.2f} ms; "
      f"phase totals per step {({k: round(v / len(lat), 2) for k, v in agg.items()})}", flush=True)
if LAZY:
    print("core records", st.core_pending(), "kept", st.n_kept(), flush=True)
