"""A small end-to-end pass over every kernel family for compute-sanitizer:
CTD-S with the error pass and the core (C1), a rejection-heavy CP case, a
heavy-fiber (oversize bucket) case, a short CTD-D stream with the core and
history, and the sharded building blocks.  Checks the results against the
oracle so a silent corruption under the tool also fails."""
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import paper_1710_03608_b200 as ctd  # noqa: E402
from oracle.bindings import Port  # noqa: E402
from paper_1710_03608_b200 import datagen as g  # noqa: E402

P = Port()
ctx = ctd.Context(0)


def check_frontend(x, s, mode=0):
    f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), mode, s, 1e-6, 42, with_error=True, with_core=True, ctx=ctx)
    o = P.frontend(x.shape, x.flat_idx(), x.val, mode, s, 1e-6, 42)
    assert np.array_equal(f.kept_flat, o.kept_flat)
    assert np.array_equal(f.U, o.U)
    return f


check_frontend(g.c1(), 200)
check_frontend(g.c4(seed=4, scale_j=60, scale_k=10), 300)
from test_gpu_parity import _heavy_fibers  # noqa: E402
check_frontend(_heavy_fibers(), 100)
# CTD-D with the core and the history
x = g.c3_stream(seed=3, n_steps=2, slices_per_step=3, n=300)
h = x.time_slab(0, 3)
st = ctd.init_stream(ctd.SparseTensor.from_datagen(h), 0, 60, 1e-6, 42, keep_history=True, ctx=ctx)
for t in range(3, 6):
    sl = x.time_slab(t, t + 1)
    ctd.ctd_d_step(st, ctd.SparseTensor.from_datagen(sl), 60)
print("drift", ctd.core_drift(st))
ps = P.stream(h.shape, h.flat_idx(), h.val, 0, 60, 1e-6, 42)
for t in range(3, 6):
    sl = x.time_slab(t, t + 1)
    ps.step(sl.shape, sl.flat_idx(), sl.val, 60)
assert np.array_equal(st.factors().kept_flat, ps.kept_flat())
print("sanitize smoke ok, launches", ctx.launches)
