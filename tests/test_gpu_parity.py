"""GPU parity: every stage of the hot path through the C-ABI (libctd_gpu.so)
against the CPU oracle on identical seeded inputs.  Integer/index results and
U must be bit-identical; the relative error within 1e-9*max(1,|ref|)."""
import numpy as np
import pytest

import paper_1710_03608_b200 as ctd
from paper_1710_03608_b200 import ctd as api
from paper_1710_03608_b200 import datagen as g

pytestmark = pytest.mark.gpu

CASES = {
    "c1": lambda: g.c1(),
    "rand_fp": lambda: g.random_sparse([30, 40, 50], 0.05, 7),
    "rand_int": lambda: g.random_sparse([25, 30, 20], 0.1, 8, integer=True),
    "lowrank": lambda: g.low_rank([40, 12, 10], 3, 0.7, 9),
    "traffic": lambda: g.traffic([500, 500, 20], 20000, 11),
    "cp_small": lambda: g.c4(seed=4, scale_j=60, scale_k=10),
    "order4": lambda: g.random_sparse([8, 9, 10, 11], 0.05, 12),
    "heavy_fibers": lambda: _heavy_fibers(),
}


def _heavy_fibers():
    """Mode-0 fibers longer than one CTA's shared-memory bucket (8192 entries):
    the device-wide radix-sort path of the bucketing (bucket.cu, oversize)."""
    I = 40000
    base = g.random_sparse([I, 6, 5], 0.002, 13)
    extra = []
    for j, (a, b, n) in enumerate([(0, 0, 15000), (3, 2, 9000), (5, 4, 30000), (1, 1, 8193)]):
        rows = np.nonzero(g.uniform(50 + j, 0, 0, I) < n / I)[0]
        extra.append(np.stack([rows, np.full_like(rows, a), np.full_like(rows, b)], axis=1))
    idx = np.concatenate([base.idx] + extra)
    val = np.concatenate([base.val] + [np.floor(g.uniform(60 + j, 0, 0, e.shape[0]) * 7) + 1
                                       for j, e in enumerate(extra)])
    return g.coalesce([I, 6, 5], idx, val)


def _st(x):
    return ctd.SparseTensor.from_datagen(x)


@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("mode", [0, 1])
def test_matricize_bitexact(ctx, port, name, mode):
    x = CASES[name]()
    m = ctd.matricize(_st(x), mode, ctx)
    o = port.matricize(x.shape, x.flat_idx(), x.val, mode)
    assert np.array_equal(m.dense_col_ptr(), o.col_ptr)
    assert np.array_equal(m.row.astype(np.int64), o.row)
    assert np.array_equal(m.val, o.val)
    assert np.array_equal(m.dense_norms(), port.column_sq_norms(o))


@pytest.mark.parametrize("mode", [0, 1, 2])
def test_matricize_wide_columns(ctx, port, mode):
    """>= 2^17 columns in every mode: 9-bit digits, so the first onesweep pass takes
    its order-3 path (index columns by bulk copy, j = i_a + i_b * shape_a), on
    full tiles and a ragged tail."""
    x = g.random_sparse([300, 400, 500], 5e-4, 21, integer=(mode == 1))
    assert x.nnz > 3 * 4096 and x.nnz % 4096 != 0
    m = ctd.matricize(_st(x), mode, ctx)
    o = port.matricize(x.shape, x.flat_idx(), x.val, mode)
    assert np.array_equal(m.dense_col_ptr(), o.col_ptr)
    assert np.array_equal(m.row.astype(np.int64), o.row)
    assert np.array_equal(m.val, o.val)
    assert np.array_equal(m.dense_norms(), port.column_sq_norms(o))


def test_norms_integer_exact_parallel(ctx, port):
    """Integer-valued tensor with mid (33..1024) and long (> 1024) fibers: the
    norms kernels reduce in parallel (any order is exact below 2^52) and must
    still equal the reference's sequential sums bit for bit."""
    x = _heavy_fibers()
    x.val = np.floor(np.abs(x.val) * 5.0) + 1.0
    m = ctd.matricize(_st(x), 0, ctx)
    o = port.matricize(x.shape, x.flat_idx(), x.val, 0)
    lens = np.diff(o.col_ptr)
    assert (lens > 1024).any() and ((lens > 32) & (lens <= 1024)).any()
    assert np.array_equal(m.val, o.val)
    assert np.array_equal(m.dense_norms(), port.column_sq_norms(o))


def test_norms_integer_large_take_sequential_path(ctx, port):
    """Integer values near 2^26: a fiber's sum of squares passes 2^52 after two
    entries, so partial sums round and only the reference's order gives its
    bits; the parallel reduction must detect that per fiber and fall back."""
    x = _heavy_fibers()
    x.val = 67108864.0 - np.floor(np.abs(x.val) * 1000.0) % 4096.0
    assert (x.val == np.rint(x.val)).all() and x.val.max() <= 67108864.0 and x.val.min() >= 1.0
    m = ctd.matricize(_st(x), 0, ctx)
    o = port.matricize(x.shape, x.flat_idx(), x.val, 0)
    ref = port.column_sq_norms(o)
    assert (ref >= 2.0 ** 52).any()
    assert np.array_equal(m.val, o.val)
    assert np.array_equal(m.dense_norms(), ref)


def test_matricize_unaligned_device_pointers(ctx, port):
    """Borrowed device arrays that are only element-aligned (not 16 bytes): the
    onesweep pass must take its non-bulk staging path and give the same result."""
    import torch
    x = CASES["c1"]()
    dev = torch.device("cuda", 0)
    idx = np.ascontiguousarray(x.idx.T.astype(np.int32))
    hold = []
    ptrs = []
    for k in range(3):
        t = torch.zeros(x.nnz + 1, dtype=torch.int32, device=dev)
        t[1:] = torch.from_numpy(idx[k]).to(dev)
        hold.append(t)
        ptrs.append(t.data_ptr() + 4)
    v = torch.zeros(x.nnz + 1, dtype=torch.float64, device=dev)
    v[1:] = torch.from_numpy(x.val).to(dev)
    torch.cuda.synchronize()
    assert (v.data_ptr() + 8) % 16 != 0
    d = api.DeviceTensor.from_device_ptrs(x.shape, x.nnz, ptrs, v.data_ptr() + 8, ctx)
    for mode in (0, 1):
        m = ctd.matricize(d, mode, ctx)
        o = port.matricize(x.shape, x.flat_idx(), x.val, mode)
        assert np.array_equal(m.dense_col_ptr(), o.col_ptr)
        assert np.array_equal(m.row.astype(np.int64), o.row)
        assert np.array_equal(m.val, o.val)
        assert np.array_equal(m.dense_norms(), port.column_sq_norms(o))


@pytest.mark.parametrize("name", list(CASES))
def test_distribution_and_cdf_bitexact(ctx, port, name):
    x = CASES[name]()
    d = ctd.column_distribution(_st(x), 0, ctx)
    o = port.matricize(x.shape, x.flat_idx(), x.val, 0)
    p, tot = port.column_distribution(o)
    assert d.total_sq_norm == tot
    assert np.array_equal(d.dense(), p)
    # the reference's clamped cumulative array restricted to nonempty fibers
    cum = np.cumsum(p)  # placeholder shape; exact values compared below
    acc = 0.0
    last = int(np.nonzero(p > 0)[0][-1])
    for i in range(len(p)):
        acc += p[i]
        cum[i] = acc
    cum[last:] = 1.0
    assert np.array_equal(d.cumulative, cum[d.fiber_col])


def test_sampling_and_dedup(ctx, port):
    rng = np.random.default_rng(3)
    p = rng.random(5000) ** 4
    p[rng.random(5000) < 0.3] = 0.0
    p /= p.sum()
    for seed in (0, 1, 42, 2**63 + 5):
        a = ctd.sample_with_replacement(p, 3000, seed, ctx)
        b = port.sample_with_replacement(p, 3000, seed)
        assert np.array_equal(a, b)
        assert np.array_equal(ctd.unique_first_occurrence(a, ctx), port.unique_first_occurrence(b))
    assert list(ctd.unique_first_occurrence([3, 1, 3, 2, 1], ctx)) == [3, 1, 2]
    assert len(ctd.sample_with_replacement(p, 0, 1, ctx)) == 0
    with pytest.raises(ctd.ArgumentError):
        ctd.sample_with_replacement(p, -1, 1, ctx)
    with pytest.raises(ctd.EmptyInputError):
        ctd.sample_with_replacement(np.zeros(10), 5, 1, ctx)


def test_fiber_basis_known_answers(ctx):
    # test_fiber_basis.cpp:30-68,115-131 restated
    b = ctd.FiberBasis(4, ctx)
    r = b.try_append_fiber([1, 3], [3.0, 4.0], 1e-6)
    assert r.accepted and r.delta == 25.0 and b.inverse_gram()[0, 0] == 1.0 / 25.0
    b = ctd.FiberBasis(4, ctx)
    assert b.try_append_fiber([0, 2], [1.0, -2.0], 1e-6).accepted
    r = b.try_append_fiber([0, 2], [1.0, -2.0], 1e-6)
    assert not r.accepted and not r.degenerate and b.size() == 1
    assert not b.try_append_fiber([], [], 1e-6).accepted
    b = ctd.FiberBasis(6, ctx)
    assert b.try_append_fiber([0, 1], [1.0, 2.0], 1e-6).accepted
    r = b.try_append_fiber([3, 5], [2.0, 1.0], 1e-6)
    assert r.accepted and r.delta == 5.0 and list(r.y) == [0.0]
    b = ctd.FiberBasis(4, ctx)
    assert b.try_append_fiber([0], [1.0], 1e-6).accepted
    r = b.try_append_fiber([2], [1e-160], 1e-6)
    assert not r.accepted and r.degenerate and b.size() == 1
    with pytest.raises(ctd.ShapeError):
        b.try_append_fiber([0], [1.0], 1e-6, dim=5)


def test_fiber_basis_random_vs_port(ctx, port):
    for seed in range(6):
        x = g.random_sparse([12, 20, 1], 0.4, 100 + seed)
        m = port.matricize(x.shape, x.flat_idx(), x.val, 0)
        gb, pb = ctd.FiberBasis(12, ctx), port.basis(12)
        for j in range(m.cols):
            i0, i1 = m.col_ptr[j], m.col_ptr[j + 1]
            r1 = gb.try_append_fiber(m.row[i0:i1], m.val[i0:i1], 1e-6)
            a, d, dl, y = pb.try_append(m.row[i0:i1], m.val[i0:i1], 1e-6)
            assert (r1.accepted, r1.degenerate, r1.delta) == (a, d, dl)
            assert np.array_equal(r1.y, y)
        assert np.array_equal(gb.inverse_gram(), pb.U())


@pytest.mark.parametrize("name", list(CASES))
def test_ctd_s_frontend_bitexact(ctx, port, name):
    x = CASES[name]()
    s = 300
    f = ctd.ctd_s(_st(x), 0, s, 1e-6, 42, ctx=ctx)
    o = port.frontend(x.shape, x.flat_idx(), x.val, 0, s, 1e-6, 42)
    assert np.array_equal(f.drawn, o.drawn)
    assert np.array_equal(f.unique, o.unique)
    assert np.array_equal(f.accepted.astype(bool), o.accepted.astype(bool))
    assert np.array_equal(f.degenerate.astype(bool), o.degenerate.astype(bool))
    assert np.array_equal(f.delta, o.delta)
    assert np.array_equal(f.kept_flat, o.kept_flat)
    assert np.array_equal(f.U, o.U)
    assert np.array_equal(f.R_col_ptr, o.R.col_ptr)
    assert np.array_equal(f.R_row, o.R.row)
    assert np.array_equal(f.R_val, o.R.val)


@pytest.mark.parametrize("name", ["c1", "rand_fp", "lowrank", "traffic", "cp_small"])
def test_relative_error(ctx, ref, name):
    x = CASES[name]()
    f = ctd.ctd_s(_st(x), 0, 200, 1e-6, 42, with_error=True, ctx=ctx)
    t = ref.tensor(x.shape, x.flat_idx(), x.val)
    r = ref.ctd_s(t, 0, 200, 1e-6, 42)
    e = r.extra["relative_error"]
    assert abs(f.relative_error - e) <= 1e-9 * max(1.0, abs(e)), (f.relative_error, e)


@pytest.mark.parametrize("name", ["c1", "rand_fp", "lowrank", "traffic", "cp_small"])
def test_relative_error_panel_and_two_panel_paths(ctx, ref, name):
    """The orthonormal-panel pass (factors kept with the panel) and the
    two-panel fallback (without it) both match the reference."""
    x = CASES[name]()
    t = ref.tensor(x.shape, x.flat_idx(), x.val)
    e = ref.ctd_s(t, 0, 200, 1e-6, 42).extra["relative_error"]
    d = ctd.DeviceTensor(_st(x), ctx)
    vals = []
    for keep in (True, False):
        h, _ = api.ctd_s_raw(d, 0, 200, 1e-6, 42, ctx=ctx, keep_panel=keep)
        try:
            vals.append(api.relative_error_raw(d, h, ctx))
        finally:
            api.free_factors(ctx, h)
    for v in vals:
        assert abs(v - e) <= 1e-9 * max(1.0, abs(e)), (vals, e)


@pytest.mark.parametrize("heavy_rows", [None, "1", "6"])
@pytest.mark.parametrize("name,mode", [("c1", 0), ("c1", 2), ("rand_fp", 1), ("rand_int", 0), ("lowrank", 0),
                                       ("traffic", 0), ("order4", 3), ("cp_small", 0)])
def test_core_bitexact(ctx, port, name, mode, heavy_rows, monkeypatch):
    """compute_core (ctd_static.cpp:12-17): C_(mode) = R^T X_(mode) entry for entry,
    including the 1e-14 drop rule, against the oracle's multiply_columns.
    ``heavy_rows`` moves the split between the row-merge CTAs and the
    transposed walk over R's columns (k_core_heavy) so both paths are covered."""
    if heavy_rows is not None:
        monkeypatch.setenv("CTD_CORE_HEAVY_ROWS", heavy_rows)
    x = CASES[name]()
    f = ctd.ctd_s(_st(x), mode, 150, 1e-6, 42, with_core=True, ctx=ctx)
    xm = port.matricize(x.shape, x.idx.reshape(-1), x.val, mode)
    o = port.frontend(x.shape, x.idx.reshape(-1), x.val, mode, 150, 1e-6, 42)
    c = port.core_matricized(xm, o.R)
    nonempty = np.nonzero(np.diff(c.col_ptr) > 0)[0]
    assert np.array_equal(f.C_col, nonempty)
    assert np.array_equal(f.C_ptr, np.concatenate([[0], np.cumsum(np.diff(c.col_ptr)[nonempty])]))
    assert np.array_equal(f.C_row, c.row)
    assert np.array_equal(f.C_val.view(np.int64), c.val.view(np.int64))


@pytest.mark.parametrize("name", ["c1", "rand_fp", "lowrank"])
def test_memory_usage(ctx, ref, name):
    x = CASES[name]()
    st = _st(x)
    f = ctd.ctd_s(st, 0, 200, 1e-6, 42, with_core=True, ctx=ctx)
    r = ref.ctd_s(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 200, 1e-6, 42)
    assert int(f.info.c_nnz) == r.extra["c_nnz"]
    assert ctd.memory_usage(st, f, ctx=ctx) == r.extra["memory_usage"]


def test_stream_vs_port(ctx, port):
    x = g.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=3000, n=400,
                    planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    st = ctd.init_stream(_st(hist), 0, 150, 1e-6, 7, ctx=ctx)
    ps = port.stream(hist.shape, hist.flat_idx(), hist.val, 0, 150, 1e-6, 7)
    for t in range(3, x.shape[2]):
        slab = x.time_slab(t, t + 1)
        ctd.ctd_d_step(st, _st(slab), 60)
        ps.step(slab.shape, slab.flat_idx(), slab.val, 60)
        f = st.factors()
        assert np.array_equal(f.kept_flat, ps.kept_flat()), t
        assert np.array_equal(f.U, ps.U()), t
    assert st.t == ps.t


def _dense_cols(ncols, C_col, C_ptr):
    cp = np.zeros(ncols + 1, np.int64)
    cnt = np.zeros(ncols, np.int64)
    cnt[C_col] = np.diff(C_ptr)
    cp[1:] = np.cumsum(cnt)
    return cp


@pytest.mark.parametrize("seed,d,lazy,read_every,legacy", [(5, 60, False, 1, False), (6, 25, False, 1, False),
                                                          (5, 60, True, 1, False), (6, 25, True, 3, False),
                                                          (6, 25, False, 1, True)])
def test_stream_core_vs_port(ctx, port, seed, d, lazy, read_every, legacy, monkeypatch):
    """CTD-D with the core maintained (Eq. 13: top-right R^T dX, chain-product
    bottom-left, bottom-right dR^T dX, assemble_blocks) bit for bit; with
    ``lazy`` the steps only record their blocks and the core is assembled when
    it is read (every ``read_every`` steps, so several records are pending);
    ``legacy`` runs the row-merge gram / per-(a, c) chain-product kernels."""
    if legacy:
        monkeypatch.setenv("CTD_CORE_LEGACY", "1")
    x = g.c3_stream(seed=seed, n_steps=3, slices_per_step=3, draws_per_slice=2500, n=300,
                    planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    st = ctd.init_stream(_st(hist), 0, 120, 1e-6, 7, with_core=True, lazy_core=lazy, ctx=ctx)
    ps = port.stream(hist.shape, hist.flat_idx(), hist.val, 0, 120, 1e-6, 7)
    grew = 0
    for t in range(3, x.shape[2]):
        slab = x.time_slab(t, t + 1)
        k0 = len(ps.kept_flat())
        ctd.ctd_d_step(st, _st(slab), d)
        ps.step(slab.shape, slab.flat_idx(), slab.val, d)
        grew += len(ps.kept_flat()) > k0
        if (t - 2) % read_every and t + 1 < x.shape[2]:
            continue
        f = st.factors()
        c = ps.core()
        assert np.array_equal(f.kept_flat, ps.kept_flat()), t
        assert c.cols == x.shape[1] * (t + 1)
        assert np.array_equal(_dense_cols(c.cols, f.C_col, f.C_ptr), c.col_ptr), t
        assert np.array_equal(f.C_row, c.row), t
        assert np.array_equal(f.C_val.view(np.int64), c.val.view(np.int64)), t
    assert grew >= 2  # the chain-product (bottom-left) block was exercised


def _stream_history_case(ctx, ref, x, h, s, seed, d, keep_history, exact_core, lazy=False):
    """init_stream(keep_history, exact_core) + ctd_d_step per slab against the
    compiled reference: kept ids, the whole core and core_drift, bit for bit."""
    hist = x.time_slab(0, h)
    st = ctd.init_stream(_st(hist), 0, s, 1e-6, seed, keep_history=keep_history, exact_core=exact_core,
                         lazy_core=lazy, ctx=ctx)
    rs = ref.stream(ref.tensor(hist.shape, hist.flat_idx(), hist.val), 0, s, 1e-6, seed,
                    keep_history=keep_history, exact_core=exact_core)
    drifts = []
    for t in range(h, x.shape[2]):
        slab = x.time_slab(t, t + 1)
        ctd.ctd_d_step(st, _st(slab), d)
        rs.step(ref.tensor(slab.shape, slab.flat_idx(), slab.val), d)
        f = st.factors()
        c = rs.core()
        assert np.array_equal(f.kept_flat, rs.factors().kept_flat), t
        assert np.array_equal(_dense_cols(c.cols, f.C_col, f.C_ptr), c.col_ptr), t
        assert np.array_equal(f.C_row, c.row), t
        assert np.array_equal(f.C_val.view(np.int64), c.val.view(np.int64)), t
        dr = ctd.core_drift(st)
        assert dr == rs.core_drift(), t
        scale = max(1.0, float(np.sqrt(np.sum(c.val * c.val))))
        drifts.append(dr / scale)
    return drifts


def test_stream_exact_core_vs_reference(ctx, ref):
    """test_ctd_dynamic.cpp:61-70: exact_core keeps the core equal to R^T X_hist."""
    x = g.random_sparse([9, 7, 8], 0.08, 501)
    drifts = _stream_history_case(ctx, ref, x, 3, 25, 17, 10, True, True)
    assert max(drifts) <= 1e-12


def test_stream_keep_history_drift_vs_reference(ctx, ref):
    """test_ctd_dynamic.cpp:44-59: on exactly low-rank data the substituted
    (chain-product) bottom-left block keeps the drift at roundoff."""
    x = g.low_rank([10, 5, 6], 2, 0.95, 29)
    drifts = _stream_history_case(ctx, ref, x, 2, 200, 7, 40, True, False)
    assert max(drifts) <= 1e-10
    assert _stream_history_case(ctx, ref, x, 2, 200, 7, 40, True, False, lazy=True) == drifts
    # larger stream with appends every step, exact_core, against the reference
    y = g.c3_stream(seed=6, n_steps=2, slices_per_step=4, draws_per_slice=1500, n=200,
                    planted_step=1, block=15)
    _stream_history_case(ctx, ref, y, 3, 80, 9, 30, False, True)


def test_core_drift_requires_history(ctx):
    x = g.random_sparse([9, 7, 8], 0.08, 501)
    st = ctd.init_stream(_st(x.time_slab(0, 3)), 0, 25, 1e-6, 17, with_core=True, ctx=ctx)
    with pytest.raises(ctd.ArgumentError):
        ctd.core_drift(st)


def test_errors(ctx):
    x = g.c1()
    t = _st(x)
    with pytest.raises(ctd.ArgumentError):
        ctd.ctd_s(t, 3, 10, ctx=ctx)
    with pytest.raises(ctd.ArgumentError):
        ctd.ctd_s(t, 0, 0, ctx=ctx)
    with pytest.raises(ctd.ArgumentError):
        ctd.ctd_s(t, 0, 10, epsilon=0.0, ctx=ctx)
    with pytest.raises(ctd.EmptyInputError):
        ctd.ctd_s(ctd.SparseTensor([3, 3, 3], np.zeros((0, 3), np.int64), np.zeros(0)), 0, 5, ctx=ctx)
    bad = ctd.SparseTensor([3, 3, 3], np.array([[0, 0, 5]], np.int64), np.array([1.0]))
    with pytest.raises(ctd.ShapeError):
        ctd.ctd_s(bad, 0, 5, ctx=ctx)


_KVEC_SCRIPT = r"""
import sys, numpy as np
sys.path.insert(0, {root!r})
import paper_1710_03608_b200 as ctd
from paper_1710_03608_b200 import ctd as api
from paper_1710_03608_b200 import datagen as g
from oracle.bindings import Port
port = Port()
cases = [g.c1(), g.traffic([500, 500, 20], 20000, 11), g.low_rank([40, 12, 10], 3, 0.7, 9)]
assert ctd.ctd_s(ctd.SparseTensor.from_datagen(cases[0]), 0, 300, 1e-6, 42).kept_count() > 64
for x in cases:
    f = ctd.ctd_s(ctd.SparseTensor.from_datagen(x), 0, 300, 1e-6, 42)
    o = port.frontend(x.shape, x.idx.reshape(-1), x.val, 0, 300, 1e-6, 42)
    assert np.array_equal(f.kept_flat, o.kept_flat)
    assert np.array_equal(f.accepted, o.accepted)
    assert np.array_equal(f.delta.view(np.int64), o.delta.view(np.int64))
    assert np.array_equal(f.U.view(np.int64), o.U.view(np.int64))
print("OK")
"""


def test_filter_global_operand_path():
    """K beyond the shared-memory staging limit: g and y come from global
    memory (CTD_FILTER_KVEC lowers the limit to 64 in a fresh process)."""
    import os
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    env = dict(os.environ, CTD_FILTER_KVEC="64")
    r = subprocess.run([sys.executable, "-c", _KVEC_SCRIPT.format(root=root)], env=env, capture_output=True,
                       text=True, timeout=600)
    assert r.returncode == 0 and "OK" in r.stdout, r.stdout + r.stderr

