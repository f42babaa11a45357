"""CTD-D at BASELINE.json configs[2] (C3) scale: init_stream on the first 500
slices of the 5000 x 5000 stream (50 steps x 10 slices), then one
ctd_d_step per slice (d = 500, seed ^ t) against the C restatement's stream
(front end only: the reference's Eq. 13 core of a 500-slice history does not
fit a CPU run), comparing the kept fiber ids after every checkpoint and U bit
for bit at the end.  CTD_C3_STEPS sets the streamed slices (default 150:
K grows from ~380 to ~3400)."""
import os

import numpy as np
import pytest

import paper_1710_03608_b200 as ctd
from paper_1710_03608_b200 import ctd as api

pytestmark = pytest.mark.gpu


def test_c3_stream_front_end_bitexact(ctx, port):
    import bench
    x = bench.load_c3()
    H = bench.C3["hist_steps"] * bench.C3["slices"]
    n_steps = int(os.environ.get("CTD_C3_STEPS", "150"))
    d, eps, seed = bench.C3["d"], bench.C3["eps"], bench.C3["seed"]
    h = x.time_slab(0, H)
    gs = api.init_stream(api.SparseTensor.from_datagen(h), 0, d, eps, seed, ctx=ctx)
    ps = port.stream(h.shape, h.flat_idx(), h.val, 0, d, eps, seed, core=False)
    assert np.array_equal(gs.factors().kept_flat, ps.kept_flat())
    for k, t in enumerate(range(H, H + n_steps)):
        sl = x.time_slab(t, t + 1)
        api.ctd_d_step(gs, api.SparseTensor.from_datagen(sl), d)
        ps.step(sl.shape, sl.flat_idx(), sl.val, d)
        if (k + 1) % 25 == 0 or k + 1 == n_steps:
            f = gs.factors()
            assert np.array_equal(f.kept_flat, ps.kept_flat()), t
    f = gs.factors()
    assert f.kept_count() > 1000
    assert np.array_equal(f.U.view(np.int64), ps.U().view(np.int64))
    gs.close()
