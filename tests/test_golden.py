"""Golden fixtures produced by the unmodified reference (tests/golden/
make_golden.py).  CPU: the C restatement reproduces them bit for bit.  GPU:
the CUDA path reproduces them bit for bit (kept fibers, draws, delta, U hash)
and the relative error within 1e-9*max(1,|ref|)."""
import glob
import hashlib
import os

import numpy as np
import pytest

from paper_1710_03608_b200 import datagen as g

HERE = os.path.dirname(os.path.abspath(__file__))
GOLD = os.path.join(HERE, "golden")

MAKERS = {
    "c1": lambda: g.c1(),
    "cp_small": lambda: g.c4(seed=4, scale_j=40, scale_k=8),
    "traffic_small": lambda: g.traffic([300, 300, 20], 8000, 11),
    "lowrank": lambda: g.low_rank([40, 12, 10], 3, 0.7, 9),
}


def sha(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def load(name):
    z = np.load(os.path.join(GOLD, f"golden_{name}.npz"))
    x = MAKERS[name]()
    assert str(z["input_sha"]) == sha(x.flat_idx()) + sha(x.val), "generator drifted"
    return z, x


def test_fixture_inventory():
    found = sorted(os.path.basename(p) for p in glob.glob(os.path.join(GOLD, "golden_*.npz")))
    assert found == sorted([f"golden_{k}.npz" for k in MAKERS] + ["golden_stream.npz"])


@pytest.mark.parametrize("name", list(MAKERS))
def test_port_reproduces_golden(port, name):
    z, x = load(name)
    fe = port.frontend(x.shape, x.flat_idx(), x.val, 0, int(z["s"]), float(z["eps"]), int(z["seed"]))
    assert np.array_equal(fe.drawn, z["drawn"])
    assert np.array_equal(fe.unique, z["unique"])
    assert np.array_equal(fe.accepted, z["accepted"])
    assert np.array_equal(fe.delta, z["delta"])
    assert np.array_equal(fe.kept_flat, z["kept_flat"])
    assert sha(fe.U) == str(z["u_sha"])
    assert fe.total == float(z["total"])
    _, core, err = port.ctd_s_error(x.shape, x.flat_idx(), x.val, 0, int(z["s"]), float(z["eps"]),
                                    int(z["seed"]))
    assert err == float(z["rel_error"]) and core.nnz == int(z["c_nnz"])


def test_port_reproduces_golden_stream(port):
    z = np.load(os.path.join(GOLD, "golden_stream.npz"))
    x = g.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2000, n=300,
                    planted_step=2, block=20)
    assert str(z["input_sha"]) == sha(x.flat_idx()) + sha(x.val)
    hist = x.time_slab(0, 3)
    st = port.stream(hist.shape, hist.flat_idx(), hist.val, 0, 120, 1e-6, 7)
    kept = []
    for t in range(3, x.shape[2]):
        slab = x.time_slab(t, t + 1)
        st.step(slab.shape, slab.flat_idx(), slab.val, 40)
        kept.append(len(st.kept_flat()))
    assert kept == list(z["kept_per_step"])
    assert np.array_equal(st.kept_flat(), z["kept_flat"])
    assert sha(st.U()) == str(z["u_sha"])


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(MAKERS))
def test_gpu_reproduces_golden(ctx, name):
    import paper_1710_03608_b200 as ctd
    z, x = load(name)
    f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), 0, int(z["s"]), float(z["eps"]), int(z["seed"]),
                  with_error=True, ctx=ctx)
    assert np.array_equal(f.drawn, z["drawn"])
    assert np.array_equal(f.unique, z["unique"])
    assert np.array_equal(f.accepted.astype(bool), z["accepted"].astype(bool))
    assert np.array_equal(f.delta, z["delta"])
    assert np.array_equal(f.kept_flat, z["kept_flat"])
    assert sha(f.U) == str(z["u_sha"])
    assert f.total_sq_norm == float(z["total"])
    e = float(z["rel_error"])
    assert abs(f.relative_error - e) <= 1e-9 * max(1.0, abs(e))


@pytest.mark.gpu
def test_gpu_reproduces_golden_stream(ctx):
    import paper_1710_03608_b200 as ctd
    z = np.load(os.path.join(GOLD, "golden_stream.npz"))
    x = g.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2000, n=300,
                    planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    st = ctd.init_stream(ctd.SparseTensor.from_datagen(hist), 0, 120, 1e-6, 7, ctx=ctx)
    kept = []
    for t in range(3, x.shape[2]):
        ctd.ctd_d_step(st, ctd.SparseTensor.from_datagen(x.time_slab(t, t + 1)), 40)
        kept.append(len(st.factors().kept_flat))
    f = st.factors()
    assert kept == list(z["kept_per_step"])
    assert np.array_equal(f.kept_flat, z["kept_flat"])
    assert sha(f.U) == str(z["u_sha"])
