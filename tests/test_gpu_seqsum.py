"""The exact sequential running sum (seqsum.cuh) against numpy's sequential
np.add.accumulate on adversarial inputs: binade crossings, exact half-ulp ties,
zero prefixes, subnormals, huge dynamic range.  Bit-exact."""
import numpy as np
import pytest

import paper_1710_03608_b200 as ctd
from paper_1710_03608_b200 import ctd as api

pytestmark = pytest.mark.gpu


def _cases():
    r = np.random.default_rng(11)
    yield "tiny", np.array([0.5])
    yield "uniform_2049", r.random(2049)
    yield "uniform_1e5", r.random(100_000)
    yield "uniform_3e6", r.random(3_000_000)
    yield "ints", np.floor(r.random(200_000) * 100)
    yield "zero_prefix", np.concatenate([np.zeros(5000), r.random(5000), np.zeros(10), r.random(10)])
    # exact ties: 1 + 2^-53 rounds to even; alternate parities
    t = np.full(300_000, 2.0 ** -53)
    t[::7] = 1.0
    t[::13] = 2.0 ** -52 * 3
    yield "ties", t
    yield "wide", np.exp(r.uniform(-700, 700, 50_000))
    yield "subnormal", np.concatenate([np.full(1000, 5e-324), r.random(1000) * 1e-310, r.random(1000)])
    p = r.random(1_000_000) ** 8
    yield "cdf_like", p / p.sum()
    # a CDF creeping up to 1.0 in tiny steps (C5's law: 8e7 fibers): every term of
    # the tail lies inside the binade-edge margin, so whole blocks are walked
    tail = r.random(600_000) * 2e-13
    yield "edge_creep", np.concatenate([[1.0 - tail.sum() * 0.7], tail, r.random(5000) * 1e-3])
    yield "edge_creep_mid", np.concatenate([r.random(3000) * 1e-4, [0.5 - 0.3 - 1e-9],
                                            np.full(300_000, 1e-14), r.random(9000)])
    # growing terms (many crossings)
    yield "geometric", 1.0001 ** np.arange(200_000)


@pytest.mark.parametrize("name,x", list(_cases()))
def test_seq_cumsum_bitexact(ctx, name, x):
    got = api.seq_cumsum(x, ctx)
    want = np.add.accumulate(x)
    bad = np.nonzero(got != want)[0]
    assert bad.size == 0, f"{name}: first mismatch at {bad[:5]} got {got[bad[:3]]} want {want[bad[:3]]}"


def test_block_exact_sum_long_fibers(ctx, port):
    """|x|^2 and the residual of long fibers go through the block-level sum."""
    r = np.random.default_rng(5)
    dim = 9000
    gb, pb = ctd.FiberBasis(dim, ctx), port.basis(dim)
    for k in range(12):
        n = int(r.integers(2000, 8000))
        idx = np.sort(r.choice(dim, n, replace=False))
        mag = np.exp(r.uniform(-30, 30, n)) if k % 2 else np.floor(r.random(n) * 7) + 1
        val = mag * np.where(r.random(n) < 0.5, -1, 1)
        a = gb.try_append_fiber(idx, val, 1e-6)
        b = pb.try_append(idx, val, 1e-6)
        assert (a.accepted, a.degenerate, a.delta) == b[:3]
        assert np.array_equal(a.y, b[3])
    assert np.array_equal(gb.inverse_gram(), pb.U())
