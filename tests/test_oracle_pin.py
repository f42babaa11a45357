"""Pin the C restatement (oracle/ctd_oracle.c) to the unmodified reference
(oracle/_ref/libctdref.so) and to the known-answer vectors of the
reference's own unit tests (proj/tests/*.cpp, restated here as data).
CPU only."""
import math

import numpy as np
import pytest

from paper_1710_03608_b200 import datagen as g

CASES = {
    "c1": lambda: g.c1(),
    "rand_fp": lambda: g.random_sparse([30, 40, 50], 0.05, 7),
    "rand_int": lambda: g.random_sparse([25, 30, 20], 0.1, 8, integer=True),
    "lowrank": lambda: g.low_rank([40, 12, 10], 3, 0.7, 9),
    "traffic": lambda: g.traffic([300, 300, 20], 8000, 11),
    "cp_small": lambda: g.c4(seed=4, scale_j=40, scale_k=8),
    "order4": lambda: g.random_sparse([8, 9, 10, 11], 0.05, 12),
}


# ---------------------------------------------------------------------------
# known answers from the reference test-suite

def test_matricize_index_mapping(port):
    # test_tensor_core.cpp:42-50: (1,0,1) in a 2x2x2 tensor -> column 2 at mode 0
    m = port.matricize([2, 2, 2], [1, 0, 1], [5.0], 0)
    assert m.cols == 4 and list(np.diff(m.col_ptr)) == [0, 0, 1, 0]
    assert m.row[0] == 1 and m.val[0] == 5.0


def test_column_sq_norms_known(port):
    # test_tensor_core.cpp:155-162: columns (3,4) and (0,5) -> 25, 25
    m = port.matricize([2, 2], [0, 0, 1, 0, 1, 1], [3.0, 4.0, 5.0], 0)
    assert list(port.column_sq_norms(m)) == [25.0, 25.0]


def test_distribution_known(port):
    # test_sampling.cpp:24-30: total 50, P = (0.5, 0.5)
    m = port.matricize([2, 2], [0, 0, 1, 0, 1, 1], [3.0, 4.0, 5.0], 0)
    p, tot = port.column_distribution(m)
    assert tot == 50.0 and list(p) == [0.5, 0.5]


def test_sampling_properties(port):
    # point mass (test_sampling.cpp:55-60), zero prob never drawn (:82-90),
    # determinism (:62-69), empty sample, tail clamp reachability (:92-102)
    assert list(port.sample_with_replacement([0.0, 1.0, 0.0], 5, 3)) == [1] * 5
    d = port.sample_with_replacement([0.2, 0.0, 0.8], 2000, 9)
    assert 1 not in set(d)
    assert np.array_equal(d, port.sample_with_replacement([0.2, 0.0, 0.8], 2000, 9))
    assert len(port.sample_with_replacement([0.5, 0.5], 0, 1)) == 0
    p = np.full(3, (1.0 - 1e-12) / 3)  # cumulative residue below 1: clamp keeps last reachable
    assert set(port.sample_with_replacement(p, 10000, 4)) <= {0, 1, 2}


def test_frequency_three_standard_errors(port):
    # test_sampling.cpp:71-80: P=(0.5,0.5), n=1e5 -> within 3 SE
    d = port.sample_with_replacement([0.5, 0.5], 100000, 42)
    f = (d == 0).mean()
    assert abs(f - 0.5) <= 3 * math.sqrt(0.25 / 100000)


def test_unique_known(port):
    # test_sampling.cpp:113-116 and SPEC examples
    assert list(port.unique_first_occurrence([3, 1, 3, 2, 1])) == [3, 1, 2]
    assert list(port.unique_first_occurrence([7, 7, 7])) == [7]
    assert list(port.unique_first_occurrence([])) == []


def test_mt19937_64_known_value(port):
    # The C++ standard pins the 10000th output of default-seeded mt19937_64.
    assert int(port.mt19937_64(5489, 10000)[-1]) == 9981545732273789042


def test_fiber_basis_known(port):
    # test_fiber_basis.cpp:30-68,115-126
    b = port.basis(4)
    a, d, dl, _ = b.try_append([1, 3], [3.0, 4.0])
    assert a and dl == 25.0 and b.U()[0, 0] == 1.0 / 25.0
    b = port.basis(4)
    assert b.try_append([0, 2], [1.0, -2.0])[0]
    a, d, _, _ = b.try_append([0, 2], [1.0, -2.0])
    assert not a and not d and b.size() == 1
    assert not b.try_append([], [])[0]
    b = port.basis(6)
    assert b.try_append([0, 1], [1.0, 2.0])[0]
    a, d, dl, y = b.try_append([3, 5], [2.0, 1.0])
    assert a and dl == 5.0 and list(y) == [0.0]
    b = port.basis(4)
    assert b.try_append([0], [1.0])[0]
    a, d, _, _ = b.try_append([2], [1e-160])
    assert not a and d and b.size() == 1


def test_fiber_basis_inverse_gram_invariant(port):
    # test_fiber_basis.cpp:90-102: |(R^T R) U - I| <= 1e-8
    for seed in range(4):
        x = g.random_sparse([12, 20, 1], 0.4, 500 + seed)
        m = port.matricize(x.shape, x.flat_idx(), x.val, 0)
        b = port.basis(12)
        for j in range(m.cols):
            b.try_append(m.row[m.col_ptr[j]:m.col_ptr[j + 1]], m.val[m.col_ptr[j]:m.col_ptr[j + 1]])
        k = b.size()
        if k == 0:
            continue
        R = np.zeros((12, k))
        fe = port.frontend(x.shape, x.flat_idx(), x.val, 0, 1, 1e-6, 1)  # for the R layout check
        del fe
        # rebuild R from the accepted columns (order) via a second pass
        b2 = port.basis(12)
        col = 0
        for j in range(m.cols):
            i0, i1 = m.col_ptr[j], m.col_ptr[j + 1]
            if b2.try_append(m.row[i0:i1], m.val[i0:i1])[0]:
                R[m.row[i0:i1], col] = m.val[i0:i1]
                col += 1
        G = R.T @ R
        assert np.abs(G @ b.U() - np.eye(k)).max() <= 1e-8
        assert np.array_equal(b.U(), b.U().T)  # symmetric by construction


def test_default_step_samples():
    # test_stream_harness.cpp:31-38
    from paper_1710_03608_b200.ctd import default_step_samples
    assert default_step_samples(1000) == 10
    assert default_step_samples(249) == 2
    assert default_step_samples(250) == 3
    assert default_step_samples(10) == 1


# ---------------------------------------------------------------------------
# restatement == reference, bit for bit

@pytest.mark.parametrize("name", list(CASES))
@pytest.mark.parametrize("mode", [0, 1])
def test_port_matches_reference_matricize(port, ref, name, mode):
    x = CASES[name]()
    t = ref.tensor(x.shape, x.flat_idx(), x.val)
    mr, nr = ref.matricize(t, mode)
    mp = port.matricize(x.shape, x.flat_idx(), x.val, mode)
    assert np.array_equal(mr.col_ptr, mp.col_ptr)
    assert np.array_equal(mr.row, mp.row)
    assert np.array_equal(mr.val, mp.val)
    assert np.array_equal(nr, port.column_sq_norms(mp))
    pr, tr = ref.column_distribution(t, mode)
    pp, tp = port.column_distribution(mp)
    assert tr == tp and np.array_equal(pr, pp)


@pytest.mark.parametrize("name", list(CASES))
def test_port_matches_reference_frontend(port, ref, name):
    x = CASES[name]()
    t = ref.tensor(x.shape, x.flat_idx(), x.val)
    for s, eps, seed in [(200, 1e-6, 42), (50, 0.15, 7)]:
        a = ref.frontend(t, 0, s, eps, seed)
        b = port.frontend(x.shape, x.flat_idx(), x.val, 0, s, eps, seed)
        assert np.array_equal(a.drawn, b.drawn)
        assert np.array_equal(a.unique, b.unique)
        assert np.array_equal(a.accepted, b.accepted)
        assert np.array_equal(a.degenerate, b.degenerate)
        assert np.array_equal(a.delta, b.delta)
        assert np.array_equal(a.kept_flat, b.kept_flat)
        assert np.array_equal(a.U, b.U)
        assert np.array_equal(a.R.col_ptr, b.R.col_ptr)
        assert np.array_equal(a.R.row, b.R.row) and np.array_equal(a.R.val, b.R.val)
        assert a.total == b.total


@pytest.mark.parametrize("name", ["c1", "rand_fp", "lowrank", "cp_small"])
def test_port_matches_reference_error(port, ref, name):
    x = CASES[name]()
    t = ref.tensor(x.shape, x.flat_idx(), x.val)
    r = ref.ctd_s(t, 0, 120, 1e-6, 42)
    fe, core, err = port.ctd_s_error(x.shape, x.flat_idx(), x.val, 0, 120, 1e-6, 42)
    assert core.nnz == r.extra["c_nnz"]
    assert err == r.extra["relative_error"]  # same operation order: bit-exact


def test_port_matches_reference_stream(port, ref):
    x = g.c3_stream(seed=5, n_steps=3, slices_per_step=3, draws_per_slice=2000, n=300,
                    planted_step=2, block=20)
    hist = x.time_slab(0, 3)
    rs = ref.stream(ref.tensor(hist.shape, hist.flat_idx(), hist.val), 0, 120, 1e-6, 7)
    ps = port.stream(hist.shape, hist.flat_idx(), hist.val, 0, 120, 1e-6, 7)
    for t in range(3, x.shape[2]):
        slab = x.time_slab(t, t + 1)
        rs.step(ref.tensor(slab.shape, slab.flat_idx(), slab.val), 40)
        ps.step(slab.shape, slab.flat_idx(), slab.val, 40)
        fr = rs.factors()
        assert np.array_equal(fr.kept_flat, ps.kept_flat())
        assert np.array_equal(fr.U, ps.U())
        cr, cp = rs.core(), ps.core()
        assert np.array_equal(cr.col_ptr, cp.col_ptr)
        assert np.array_equal(cr.row, cp.row) and np.array_equal(cr.val, cp.val)
    assert rs.t == ps.t


def test_lemma2_projection_optimality(port):
    """test_ctd_static.cpp:88-120 with a numpy lstsq witness for the Eigen
    oracle: the CTD-S error equals the projection error onto ALL sampled
    fibers (Lemma 2), 1e-8 relative."""
    x = g.random_sparse([30, 12, 10], 0.08, 21)
    s = 60
    fe, core, err = port.ctd_s_error(x.shape, x.flat_idx(), x.val, 0, s, 1e-6, 42)
    m = port.matricize(x.shape, x.flat_idx(), x.val, 0)
    X = np.zeros((m.rows, m.cols))
    for j in range(m.cols):
        X[m.row[m.col_ptr[j]:m.col_ptr[j + 1]], j] = m.val[m.col_ptr[j]:m.col_ptr[j + 1]]
    R0 = X[:, fe.drawn]
    coef, *_ = np.linalg.lstsq(R0, X, rcond=1e-10)
    proj = np.linalg.norm(X - R0 @ coef) ** 2 / np.linalg.norm(X) ** 2
    assert abs(err - proj) <= 1e-8 * max(1.0, proj)


def test_errors(port):
    from oracle.bindings import OracleError
    with pytest.raises(OracleError) as e:
        port.frontend([3, 3, 3], np.zeros(0, np.int64), np.zeros(0), 0, 5)
    assert e.value.code == 3  # EmptyInputError
    x = g.c1()
    with pytest.raises(OracleError) as e:
        port.frontend(x.shape, x.flat_idx(), x.val, 3, 5)
    assert e.value.code == 1
    with pytest.raises(OracleError) as e:
        port.frontend(x.shape, x.flat_idx(), x.val, 0, 0)
    assert e.value.code == 1
