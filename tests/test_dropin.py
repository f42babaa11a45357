"""The compiled C++ drop-in (paper_1710_03608_b200/shim): the reference's own
library relinked with `ld --wrap` so ctd::ctd_s / ctd::init_stream /
ctd::ctd_d_step run on the B200 through libctd_gpu.so.  The reference's own
driver code (oracle/ref_driver.cpp, through the `Ref` binding) is called on
both builds: the unmodified CPU library and the drop-in; everything the
caller sees (kept fibers, R, U, the folded core C, relative_error and
memory_usage computed by the reference's own evaluation code on the returned
factors, the stream's matricized core) must be identical."""
import ctypes as C
import os

import numpy as np
import pytest

from paper_1710_03608_b200 import datagen as g

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
DROPIN = os.path.join(ROOT, "paper_1710_03608_b200", "shim", "libctd_dropin.so")
WRAPPED = ("_ZN3ctd5ctd_sERKNS_12SparseTensorEildm",
           "_ZN3ctd11init_streamERKNS_12SparseTensorEildmbb",
           "_ZN3ctd10ctd_d_stepENS_11StreamStateERKNS_12SparseTensorEl",
           "_ZNK3ctd11StreamState7factorsEv",
           "_ZN3ctd10core_driftERKNS_11StreamStateE",
           "_ZN3ctd14relative_errorERKNS_12SparseTensorERKNS_9LRFactorsE",
           "_ZN3ctd9matricizeERKNS_12SparseTensorEi",
           "_ZN3ctd15column_sq_normsERKNS_12SparseMatrixE",
           "_ZN3ctd19column_distributionERKNS_12SparseMatrixE",
           "_ZN3ctd23sample_with_replacementERKNS_18ColumnDistributionElm",
           "_ZN3ctd23unique_first_occurrenceESt4spanIKlLm18446744073709551615EE",
           "_ZN3ctd12compute_coreERKNS_12SparseTensorERKNS_12SparseMatrixEi",
           "_ZN3ctd13chain_productERKNS_12SparseMatrixES2_RKNS_11DenseMatrixES2_")

needs_dropin = pytest.mark.skipif(not os.path.exists(DROPIN),
                                  reason="drop-in not built (make -C paper_1710_03608_b200/shim)")


@needs_dropin
def test_dropin_exports_wrappers():
    """Loads on a GPU-less host; the wrapped entry points and the reference
    driver's symbols are present."""
    lib = C.CDLL(DROPIN)
    for s in WRAPPED:
        assert hasattr(lib, "__wrap_" + s), s
    for s in ("ref_ctd_s", "ref_init_stream", "ref_stream_step", "ref_relative_error"):
        assert hasattr(lib, s), s


def _fold_c(R, h):
    L = R.L
    n = int(L.ref_factors_c_nnz(h))
    order = int(L.ref_factors_c_order(h))
    shape = np.zeros(order, np.int64)
    L.ref_factors_c_shape(h, shape.ctypes.data)
    idx = np.zeros(n * order, np.int64)
    val = np.zeros(n)
    L.ref_factors_c(h, idx.ctypes.data, val.ctypes.data)
    return shape, idx, val


def _ctd_s_full(R, x, mode, s, eps, seed):
    t = R.tensor(x.shape, x.flat_idx(), x.val)
    h = C.c_void_p()
    R._chk(R.L.ref_ctd_s(t.h, mode, s, eps, C.c_uint64(seed), C.byref(h)), "ctd_s")
    try:
        fe = R._factors(h, False)
        shape, idx, val = _fold_c(R, h)
        e, m = C.c_double(), C.c_double()
        R._chk(R.L.ref_relative_error(t.h, h, C.byref(e)), "relative_error")
        R._chk(R.L.ref_memory_usage(t.h, h, C.byref(m)), "memory_usage")
        return fe, shape, idx, val, e.value, m.value
    finally:
        R.L.ref_factors_free(h)


CASES = {
    "c1": (lambda: g.c1(), 0, 200),
    "rand_fp_m1": (lambda: g.random_sparse([30, 40, 50], 0.05, 7), 1, 300),
    "traffic": (lambda: g.traffic([500, 500, 20], 20000, 11), 0, 400),
    "order4": (lambda: g.random_sparse([8, 9, 10, 11], 0.05, 12), 2, 150),
}


@pytest.fixture(scope="module")
def dropin():
    from oracle.bindings import Ref
    return Ref(DROPIN)


@pytest.mark.gpu
@needs_dropin
@pytest.mark.parametrize("name", list(CASES))
def test_dropin_ctd_s(ref, dropin, name):
    make, mode, s = CASES[name]
    x = make()
    a = _ctd_s_full(ref, x, mode, s, 1e-6, 42)
    b = _ctd_s_full(dropin, x, mode, s, 1e-6, 42)
    fa, fb = a[0], b[0]
    assert np.array_equal(fa.kept_flat, fb.kept_flat)
    assert np.array_equal(fa.U.view(np.int64), fb.U.view(np.int64))
    assert np.array_equal(fa.R.col_ptr, fb.R.col_ptr)
    assert np.array_equal(fa.R.row, fb.R.row)
    assert np.array_equal(fa.R.val.view(np.int64), fb.R.val.view(np.int64))
    assert np.array_equal(a[1], b[1])  # folded core shape
    assert np.array_equal(a[2], b[2])  # core coordinates (reference fold order)
    assert np.array_equal(a[3].view(np.int64), b[3].view(np.int64))  # core values, bit for bit
    # the reference's own evaluation on identical factors: identical results
    assert a[4] == b[4] or abs(a[4] - b[4]) <= 1e-9 * max(1.0, abs(a[4]))
    assert a[5] == b[5]


@pytest.mark.gpu
@needs_dropin
def test_dropin_errors(ref, dropin):
    from oracle.bindings import OracleError
    x = g.c1()
    for mode, s, eps in ((3, 10, 1e-6), (0, 0, 1e-6), (0, 10, 0.0)):
        codes = []
        for R in (ref, dropin):
            t = R.tensor(x.shape, x.flat_idx(), x.val)
            h = C.c_void_p()
            with pytest.raises(OracleError) as ei:
                R._chk(R.L.ref_ctd_s(t.h, mode, s, eps, C.c_uint64(42), C.byref(h)), "ctd_s")
            codes.append(ei.value.code)
        assert codes[0] == codes[1], (mode, s, eps, codes)


@pytest.mark.gpu
@needs_dropin
@pytest.mark.parametrize("keep_history,exact_core", [(False, False), (True, False), (True, True)])
def test_dropin_stream(ref, dropin, keep_history, exact_core):
    x = g.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2500, n=300,
                    planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    sa = ref.stream(ref.tensor(hist.shape, hist.flat_idx(), hist.val), 0, 120, 1e-6, 7,
                    keep_history=keep_history, exact_core=exact_core)
    sb = dropin.stream(dropin.tensor(hist.shape, hist.flat_idx(), hist.val), 0, 120, 1e-6, 7,
                       keep_history=keep_history, exact_core=exact_core)
    grew = 0
    for t in range(3, x.shape[2]):
        slab = x.time_slab(t, t + 1)
        k0 = len(sa.factors().kept_flat)
        sa.step(ref.tensor(slab.shape, slab.flat_idx(), slab.val), 40)
        sb.step(dropin.tensor(slab.shape, slab.flat_idx(), slab.val), 40)
        fa, fb = sa.factors(), sb.factors()
        grew += len(fa.kept_flat) > k0
        assert sa.t == sb.t == t + 1
        assert np.array_equal(fa.kept_flat, fb.kept_flat), t
        assert np.array_equal(fa.U.view(np.int64), fb.U.view(np.int64)), t
        assert np.array_equal(fa.R.row, fb.R.row) and np.array_equal(fa.R.val, fb.R.val), t
        ca, cb = sa.core(), sb.core()
        assert (ca.rows, ca.cols) == (cb.rows, cb.cols), t
        assert np.array_equal(ca.col_ptr, cb.col_ptr), t
        assert np.array_equal(ca.row, cb.row), t
        assert np.array_equal(ca.val.view(np.int64), cb.val.view(np.int64)), t
        if keep_history:  # core_drift reads the retained history (concatenated by the shim)
            da, db = sa.core_drift(), sb.core_drift()
            assert da == db or abs(da - db) <= 1e-9 * max(1.0, abs(da)), t
    assert grew >= 1


@pytest.mark.gpu
@needs_dropin
@pytest.mark.parametrize("name", list(CASES))
def test_dropin_tensor_ops_and_sampling(ref, dropin, name):
    """matricize, column_sq_norms, column_distribution, sample_with_replacement
    and unique_first_occurrence through the drop-in: bit-identical."""
    make, mode, s = CASES[name]
    x = make()
    ta, tb = ref.tensor(x.shape, x.flat_idx(), x.val), dropin.tensor(x.shape, x.flat_idx(), x.val)
    (ma, na), (mb, nb) = ref.matricize(ta, mode), dropin.matricize(tb, mode)
    assert np.array_equal(ma.col_ptr, mb.col_ptr) and np.array_equal(ma.row, mb.row)
    assert np.array_equal(ma.val.view(np.int64), mb.val.view(np.int64))
    assert np.array_equal(na.view(np.int64), nb.view(np.int64))
    (pa, ta_), (pb, tb_) = ref.column_distribution(ta, mode), dropin.column_distribution(tb, mode)
    assert ta_ == tb_ and np.array_equal(pa.view(np.int64), pb.view(np.int64))
    for seed in (1, 42, 2**63 + 5):
        da, db = ref.sample_with_replacement(pa, s, seed), dropin.sample_with_replacement(pb, s, seed)
        assert np.array_equal(da, db)
        assert np.array_equal(ref.unique_first_occurrence(da), dropin.unique_first_occurrence(db))


@pytest.mark.gpu
@needs_dropin
def test_dropin_run_stream(ref, dropin):
    """The reference's own run_stream (stream_harness.cpp:48-107) through the
    drop-in: every ctd_d_step, StreamState::factors and relative_error on the
    GPU, per-step kept counts and memory usage equal, errors within 1e-9."""
    x = g.c3_stream(seed=6, n_steps=4, slices_per_step=3, draws_per_slice=2500, n=300, planted_step=3, block=20)
    a = ref.run_stream(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 120, 40, 0.5, 1e-6, 7)
    b = dropin.run_stream(dropin.tensor(x.shape, x.flat_idx(), x.val), 0, 120, 40, 0.5, 1e-6, 7)
    assert np.array_equal(a["step"], b["step"])
    assert np.array_equal(a["kept_fibers"], b["kept_fibers"])
    assert np.array_equal(a["memory_usage"], b["memory_usage"])
    for ea, eb in zip(a["relative_error"], b["relative_error"]):
        assert abs(ea - eb) <= 1e-9 * max(1.0, abs(ea)), (ea, eb)


def _cols(m, lo, hi):
    """Columns [lo, hi) of a Csc."""
    from oracle.bindings import Csc
    a, b = m.col_ptr[lo], m.col_ptr[hi]
    return Csc(m.rows, hi - lo, (m.col_ptr[lo:hi + 1] - a).astype(np.int64), m.row[a:b].copy(), m.val[a:b].copy())


@pytest.mark.gpu
@needs_dropin
@pytest.mark.parametrize("name", list(CASES))
def test_dropin_compute_core_and_chain_product(ref, dropin, name):
    """compute_core (ctd_static.hpp:28) and chain_product (ctd_dynamic.hpp:61-62)
    called by the reference's own driver code: bit-identical results through the
    drop-in, and the reference's ShapeError on mismatched operands."""
    from oracle.bindings import Csc, OracleError
    make, mode, s = CASES[name]
    x = make()
    ta, tb = ref.tensor(x.shape, x.flat_idx(), x.val), dropin.tensor(x.shape, x.flat_idx(), x.val)
    fe = ref.frontend(ta, mode, s)
    ca, cb = ref.compute_core(ta, fe.R, mode), dropin.compute_core(tb, fe.R, mode)
    (ia, va), (ib, vb) = ca.data(), cb.data()
    assert ca.shape == cb.shape and np.array_equal(ia, ib)
    assert np.array_equal(va.view(np.int64), vb.view(np.int64))
    # chain_product((dR, R_old, U_old, C_old)): the last A kept fibers against the others
    K = fe.R.cols
    A = max(1, min(6, K // 3))
    r_old, d_r = _cols(fe.R, 0, K - A), _cols(fe.R, K - A, K)
    u_old = np.ascontiguousarray(fe.U[:K - A, :K - A])
    core_t = ref.compute_core(ta, r_old, mode)
    core_m, _ = ref.matricize(core_t, mode)
    pa, pb = ref.chain_product(d_r, r_old, u_old, core_m), dropin.chain_product(d_r, r_old, u_old, core_m)
    assert (pa.rows, pa.cols) == (pb.rows, pb.cols) == (A, core_m.cols)
    assert pa.col_ptr[-1] > 0
    assert np.array_equal(pa.col_ptr, pb.col_ptr) and np.array_equal(pa.row, pb.row)
    assert np.array_equal(pa.val.view(np.int64), pb.val.view(np.int64))
    for lib in (ref, dropin):
        with pytest.raises(OracleError) as e:  # U's size differs from R's column count
            lib.chain_product(d_r, r_old, np.ascontiguousarray(u_old[:-1, :-1]), core_m)
        assert e.value.code == 2  # ShapeError
        with pytest.raises(OracleError) as e:  # dR and R over different fiber lengths
            lib.chain_product(Csc(d_r.rows + 1, d_r.cols, d_r.col_ptr, d_r.row, d_r.val), r_old, u_old, core_m)
        assert e.value.code == 2
        bad = Csc(fe.R.rows + 1, fe.R.cols, fe.R.col_ptr, fe.R.row, fe.R.val)  # rows != the tensor extent
        with pytest.raises(OracleError) as e:
            lib.compute_core(ta if lib is ref else tb, bad, mode)
        assert e.value.code == 2


@pytest.mark.gpu
def test_python_compute_core_and_chain_product(ref):
    """The Python mirror's compute_core / chain_product on the device against
    the compiled reference."""
    from paper_1710_03608_b200 import ctd
    x = g.traffic([300, 300, 20], 12000, 3)
    ta = ref.tensor(x.shape, x.flat_idx(), x.val)
    fe = ref.frontend(ta, 0, 200)
    got = ctd.compute_core(ctd.SparseTensor.from_datagen(x), fe.R.col_ptr, fe.R.row, fe.R.val, fe.R.cols, 0)
    want, _ = ref.matricize(ref.compute_core(ta, fe.R, 0), 0)
    cols = np.nonzero(np.diff(want.col_ptr))[0]
    assert np.array_equal(got.col_id, cols)
    assert np.array_equal(got.row, want.row) and np.array_equal(got.val.view(np.int64), want.val.view(np.int64))
    K = fe.R.cols
    r_old, d_r = _cols(fe.R, 0, K - 4), _cols(fe.R, K - 4, K)
    core_m, _ = ref.matricize(ref.compute_core(ta, r_old, 0), 0)
    u = np.ascontiguousarray(fe.U[:K - 4, :K - 4])
    pa = ref.chain_product(d_r, r_old, u, core_m)
    pb = ctd.chain_product(fe.R.rows, (d_r.col_ptr, d_r.row, d_r.val), (r_old.col_ptr, r_old.row, r_old.val), u,
                           (core_m.col_ptr, core_m.row, core_m.val), core_m.cols)
    assert np.array_equal(pb.col_id, np.nonzero(np.diff(pa.col_ptr))[0])
    assert np.array_equal(pb.row, pa.row) and np.array_equal(pb.val.view(np.int64), pa.val.view(np.int64))
