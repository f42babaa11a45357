"""The multi-threaded filter replay (oracle/filter_par.c) the C5 parity test
uses is bit-identical to the sequential restatement (and so to the
reference) on every decision, delta and U."""
import numpy as np
import pytest

from paper_1710_03608_b200 import datagen as g

CASES = {
    "c1": (lambda: g.c1(), 200),
    "traffic": (lambda: g.traffic([500, 500, 20], 20000, 11), 300),
    "traffic_1k": (lambda: g.traffic([1000, 1000, 40], 150000, 21), 400),
    "cp": (lambda: g.c4(seed=4, scale_j=100, scale_k=10), 400),
    "lowrank": (lambda: g.low_rank([40, 12, 10], 3, 0.7, 9), 200),
}


@pytest.mark.parametrize("name", list(CASES))
def test_filter_par_bitexact(port, name):
    make, s = CASES[name]
    x = make()
    fe = port.frontend(x.shape, x.flat_idx(), x.val, 0, s, 1e-6, 42)
    m = port.matricize(x.shape, x.flat_idx(), x.val, 0)
    cols = fe.unique
    lens = m.col_ptr[cols + 1] - m.col_ptr[cols]
    cp = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
    rows = np.concatenate([m.row[m.col_ptr[c]:m.col_ptr[c + 1]] for c in cols])
    vals = np.concatenate([m.val[m.col_ptr[c]:m.col_ptr[c + 1]] for c in cols])
    acc, deg, dl, U = port.filter_par(x.shape[0], cp, rows, vals, 1e-6)
    assert np.array_equal(acc.astype(bool), fe.accepted.astype(bool))
    assert np.array_equal(deg.astype(bool), fe.degenerate.astype(bool))
    assert np.array_equal(dl.view(np.int64), fe.delta.view(np.int64))
    assert np.array_equal(U.view(np.int64), fe.U.view(np.int64))
