"""Factor bundles (factor_io.cpp) and DDoS post-processing (ddos.cpp):
bundles written by this package are byte-identical to the reference's, the
loader round-trips the reference's bundles, and the detector flags the same
candidates; the GPU cases write bundles of GPU-computed factors."""
import os

import numpy as np
import pytest

from paper_1710_03608_b200 import ctd as api
from paper_1710_03608_b200 import datagen as g
from paper_1710_03608_b200 import ddos
from paper_1710_03608_b200 import factor_io as fio

FILES = ("manifest.txt", "R.tsv", "C.tsv", "U.tsv")


def _same_bundle(a, b):
    for n in FILES:
        with open(os.path.join(a, n), "rb") as fa, open(os.path.join(b, n), "rb") as fb:
            assert fa.read() == fb.read(), n


def _need(ref):
    if not hasattr(ref.L, "ref_save_factors"):
        pytest.skip("reference driver predates ref_save_factors")


def _traffic():
    # small src x dst x time traffic with a planted block (a DDoS-like burst)
    return g.c3_stream(seed=4, n_steps=2, slices_per_step=4, draws_per_slice=900, n=120, planted_step=1,
                       block=10)


@pytest.mark.parametrize("name", ["c1", "traffic"])
def test_bundle_roundtrip_matches_reference(ref, tmp_path, name):
    _need(ref)
    x = g.c1() if name == "c1" else _traffic()
    a, b, c = (str(tmp_path / n) for n in "abc")
    ref.ctd_s_bundle(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 150, 1e-6, 42, save_dir=a)
    f = fio.load_factors(a)
    fio.save_factors(f, b)
    _same_bundle(a, b)
    ref.resave(b, c)
    _same_bundle(b, c)


def test_detect_on_reference_factors(ref, tmp_path):
    _need(ref)
    x = _traffic()
    a = str(tmp_path / "a")
    want = ref.ctd_s_bundle(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 200, 1e-6, 42, save_dir=a,
                            detect=True)["detect"]
    got = ddos.detect_ddos(fio.load_factors(a))
    assert [(c.dst, c.bin, c.norm) for c in got] == want
    assert want  # something was flagged


def test_bundle_errors(ref, tmp_path):
    _need(ref)
    x = g.c1()
    a = str(tmp_path / "a")
    ref.ctd_s_bundle(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 50, 1e-6, 42, save_dir=a)
    with pytest.raises(fio.IoError):
        fio.load_factors(str(tmp_path / "missing"))
    m = os.path.join(a, "manifest.txt")
    txt = open(m).read()
    for bad in (txt.replace("ctd-factors", "not-factors"), txt.replace("ctd-factors 1", "ctd-factors 2"),
                txt.replace("kept ", "kept 1")):
        open(m, "w").write(bad)
        with pytest.raises(fio.IoError):
            fio.load_factors(a)
    open(m, "w").write(txt)
    u = os.path.join(a, "U.tsv")
    open(u, "a").write("1\n")
    with pytest.raises(fio.IoError):
        fio.load_factors(a)


def test_score_detection():
    cands = [ddos.Candidate(3, 1, 5.0), ddos.Candidate(7, 2, 4.0), ddos.Candidate(9, 0, 1.0)]
    attacks = [ddos.AttackSpec(3, 1), ddos.AttackSpec(7, 5), ddos.AttackSpec(11, 0)]
    r = ddos.score_detection(cands, attacks)
    assert (r.precision, r.recall, r.time_matches) == (2 / 3, 2 / 3, 1)
    assert abs(r.f1 - 2 / 3) < 1e-15
    assert ddos.score_detection([], []).f1 == 0.0


@pytest.mark.gpu
def test_gpu_bundle_matches_reference(ctx, ref, tmp_path):
    _need(ref)
    x = g.c1()
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    ref.ctd_s_bundle(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 200, 1e-6, 42, save_dir=a)
    f = api.ctd_s(api.SparseTensor.from_datagen(x), 0, 200, 1e-6, 42, with_core=True, ctx=ctx)
    fio.save_factors(f, b)
    _same_bundle(a, b)


@pytest.mark.gpu
def test_gpu_decompose_online_and_detect(ctx, ref, tmp_path):
    _need(ref)
    x = _traffic()
    a, b = str(tmp_path / "a"), str(tmp_path / "b")
    want = ref.decompose_online(ref.tensor(x.shape, x.flat_idx(), x.val), 0, 60, 1e-6, 42, save_dir=a,
                                detect=True)["detect"]
    f = ddos.decompose_online(x, 0, 60, 1e-6, 42, ctx=ctx)
    fio.save_factors(f, b)
    _same_bundle(a, b)
    assert [(c.dst, c.bin, c.norm) for c in ddos.detect_ddos(f)] == want
