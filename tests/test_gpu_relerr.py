"""The relative-error pass (relerr.cu + ortho.cu) against the double-double
oracle (oracle/relerr_dd.c, itself pinned to the reference's relative_error by
tests/test_relerr_oracle.py) at small sizes and at BASELINE.json's full C2 and
C4 (tests/golden/relerr_golden.json).  Bar: |d| <= 1e-9 max(1, |ref|)
(north_star); the observed gap is ~1e-15, so a tighter diagnostic bound is
asserted too.  Both ways of building the orthonormal panel are covered: from
the filter's residual panel (ctd_s with the error pass or keep_panel) and from
R alone (factors computed without it)."""
import json
import os

import numpy as np
import pytest

import paper_1710_03608_b200 as ctd
from paper_1710_03608_b200 import ctd as api
from paper_1710_03608_b200 import datagen as g

pytestmark = pytest.mark.gpu
HERE = os.path.dirname(os.path.abspath(__file__))

SMALL = {
    "c1": (lambda: g.c1(), 200),
    "traffic_1k": (lambda: g.traffic([1000, 1000, 40], 150000, 21), 400),
    "traffic_2k": (lambda: g.traffic([2000, 2000, 50], 400000, 22), 800),
    "cp": (lambda: g.c4(seed=4, scale_j=300, scale_k=30), 300),
    "lowrank": (lambda: g.low_rank([40, 12, 10], 3, 0.7, 9), 200),
    "rand_fp": (lambda: g.random_sparse([30, 40, 50], 0.05, 7), 200),
}


def _both_paths(ctx, x, s, eps=1e-6, seed=42):
    d = ctd.DeviceTensor(ctd.SparseTensor.from_datagen(x), ctx)
    out = []
    for keep in (True, False):
        h, info = api.ctd_s_raw(d, 0, s, eps, seed, ctx=ctx, keep_panel=keep)
        try:
            out.append(api.relative_error_raw(d, h, ctx))
            out.append(api.relative_error_raw(d, h, ctx))  # cached panel: same bits
        finally:
            api.free_factors(ctx, h)
    d.close()
    assert out[0] == out[1] and out[2] == out[3]
    return out[0], out[2]


@pytest.mark.parametrize("name", list(SMALL))
def test_relerr_vs_dd_oracle(ctx, port, name):
    make, s = SMALL[name]
    x = make()
    fe = port.frontend(x.shape, x.flat_idx(), x.val, 0, s, 1e-6, 42)
    xm = port.matricize(x.shape, x.flat_idx(), x.val, 0)
    want = port.relerr_dd_full(xm, fe.R, fe.U)
    for v in _both_paths(ctx, x, s):
        assert abs(v - want) <= 1e-9 * max(1.0, abs(want)), (v, want)
        assert abs(v - want) <= 1e-13 * max(1.0, abs(want)), (v, want)


@pytest.mark.parametrize("name", ["c2", "c4"])
def test_relerr_baseline_configs(ctx, name):
    """C2 (configs[1]) and C4 (configs[3]) at full size against the committed
    double-double values; the kept ids and U are first checked to be the ones
    the golden value was computed from."""
    import hashlib
    gold = json.load(open(os.path.join(HERE, "golden", "relerr_golden.json")))[name]
    x = g.traffic(gold["shape"], gold["nnz"], 2) if name == "c2" else g.c4(seed=4)
    f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), 0, gold["c"], gold["eps"], gold["seed"], with_error=True,
                  ctx=ctx)
    assert f.kept_count() == gold["kept"]
    assert hashlib.sha256(np.ascontiguousarray(f.kept_flat.astype(np.int64)).tobytes()).hexdigest() == gold["kept_sha"]
    assert hashlib.sha256(np.ascontiguousarray(f.U).tobytes()).hexdigest() == gold["U_sha"]
    want = gold["relative_error"]
    v_panel = f.relative_error
    v_w, v_r = _both_paths(ctx, x, gold["c"])
    assert v_w == v_panel
    for v in (v_w, v_r):
        assert abs(v - want) <= 1e-9 * max(1.0, abs(want)), (v, want)
        assert abs(v - want) <= 1e-12 * max(1.0, abs(want)), (v, want)
