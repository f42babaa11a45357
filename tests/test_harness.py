"""The stream harness (run_stream, stream_harness.cpp:48-107) and its TSV
records (evaluation.cpp:47-62): host formatting and validation against the
compiled reference on CPU; the whole protocol on the GPU against the
reference's own run_stream (kept fibers and memory usage exact, relative
error within 1e-9 * max(1, |ref|))."""
import numpy as np
import pytest

from paper_1710_03608_b200 import ctd as api
from paper_1710_03608_b200 import datagen as g
from paper_1710_03608_b200 import harness as H


def test_tsv_matches_reference(ref):
    if not hasattr(ref.L, "ref_tsv_line"):
        pytest.skip("reference driver predates ref_tsv_line")
    assert H.tsv_header() == ref.tsv_line(-1)
    for args in [(3, 0.25, 0.125, 0.5, 7), (0, 1.0 / 3.0, 1e-7, 12.75, 0), (17, 0.1, 2.5e-3, 1.0 + 2**-52, 123)]:
        step, err, secs, mem, kept = args
        rep = H.EvalReport(relative_error=err, memory_usage=mem, wall_time_seconds=secs, kept_fibers=kept)
        assert H.tsv_line(step, rep) == ref.tsv_line(step, err, secs, mem, kept)
    # test_evaluation.cpp:202-206
    assert H.tsv_line(3, H.EvalReport(0.25, 0.5, 0.125, 7)) == "3\t0.25\t0.125\t0.5\t7"


def test_time_slab_and_defaults():
    x = api.SparseTensor.from_datagen(g.random_sparse([6, 5, 9], 0.2, 3))
    s = H.time_slab(x, 2, 5)
    ref = g.Tensor(x.shape, x.indices, x.values).time_slab(2, 5)
    assert s.shape == [6, 5, 3]
    assert np.array_equal(s.indices, ref.idx) and np.array_equal(s.values, ref.val)
    with pytest.raises(api.ArgumentError):
        H.time_slab(x, 5, 2)
    with pytest.raises(api.ArgumentError):
        H.time_slab(x, 0, 10)
    assert [H.default_step_samples(v) for v in (1000, 249, 250, 10)] == [10, 2, 3, 1]


def test_run_stream_validation():
    x = api.SparseTensor.from_datagen(g.random_sparse([6, 5, 9], 0.2, 3))
    for bad in (0.0, 1.0, -0.5, float("nan")):
        with pytest.raises(api.ArgumentError):
            H.run_stream(x, H.HarnessOptions(split=bad))
    with pytest.raises(api.ArgumentError):
        H.run_stream(api.SparseTensor.from_datagen(g.random_sparse([6, 5, 4], 0.3, 3)))


CASES = {
    "traffic_stream": (lambda: g.c3_stream(seed=8, n_steps=2, slices_per_step=4, draws_per_slice=1200, n=150,
                                           planted_step=1, block=12),
                       dict(sample_size=120, step_samples=30, seed=11)),
    "random_exact_core": (lambda: g.random_sparse([9, 7, 8], 0.08, 501),
                          dict(sample_size=25, step_samples=10, seed=17, split=0.375, exact_core=True)),
    "low_rank": (lambda: g.low_rank([10, 5, 6], 2, 0.95, 29),
                 dict(sample_size=200, seed=7, split=0.34)),
}


@pytest.mark.gpu
@pytest.mark.parametrize("name", list(CASES))
def test_run_stream_vs_reference(ctx, ref, name):
    make, opts = CASES[name]
    x = make()
    o = H.HarnessOptions(**opts)
    got = H.run_stream(x, o, ctx)
    want = ref.run_stream(ref.tensor(x.shape, x.flat_idx(), x.val), o.mode, o.sample_size, o.step_samples,
                          o.split, o.epsilon, o.seed, o.exact_core)
    assert [s.step for s in got.steps] == list(want["step"])
    assert [s.eval.kept_fibers for s in got.steps] == list(want["kept_fibers"])
    assert [s.eval.memory_usage for s in got.steps] == list(want["memory_usage"])
    for s, e in zip(got.steps, want["relative_error"]):
        assert abs(s.eval.relative_error - e) <= 1e-9 * max(1.0, abs(e)), (s.step, s.eval.relative_error, e)
    assert abs(got.mean.relative_error - want["mean"][0]) <= 1e-9 * max(1.0, abs(want["mean"][0]))
    assert got.mean.memory_usage == want["mean"][1]
    assert got.mean.kept_fibers == int(want["mean"][3])
    assert all(s.eval.wall_time_seconds > 0 for s in got.steps)
