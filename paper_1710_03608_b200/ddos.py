"""DDoS post-processing over the decomposition (ddos.hpp, ddos.cpp:99-184):
detect_ddos groups the kept fibers of a source-mode decomposition by
destination and flags representatives with an above-mean R column norm;
score_detection scores candidates against injected attacks;
decompose_online runs the slab-by-slab CTD-D pass (on the GPU) the detector
reads.  Host code over the factors, in the reference's arithmetic order."""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import ctd as api
from . import harness


@dataclass
class AttackSpec:
    victim: int = 0
    bin: int = 0
    sources: list = field(default_factory=list)
    intensity: float = 0.0


@dataclass
class Candidate:
    dst: int = 0
    bin: int = 0
    norm: float = 0.0


@dataclass
class DetectionReport:
    candidates: list = field(default_factory=list)
    recall: float = 0.0
    precision: float = 0.0
    f1: float = 0.0
    time_matches: int = 0


def detect_ddos(f: api.LRFactors) -> list:
    """detect_ddos (ddos.cpp:99-129)."""
    order = len(f.shape)
    if order < 2:
        raise api.ArgumentError("factors carry no decodable fibers")
    if f.mode == order - 1:
        raise api.ArgumentError("detection needs a non-time decomposition mode")
    reps = []
    seen = set()
    cp = np.asarray(f.R_col_ptr, np.int64)
    for k, j in enumerate(f.kept_flat):
        c = api.make_fiber_id(f.shape, f.mode, int(j)).coords
        dst, b = c[0], c[-1]
        if dst in seen:
            continue
        seen.add(dst)
        s = 0.0
        for v in f.R_val[cp[k]:cp[k + 1]]:
            s += float(v) * float(v)
        reps.append(Candidate(dst, b, math.sqrt(s)))
    if not reps:
        return []
    mean = 0.0
    for r in reps:
        mean += r.norm
    mean /= float(len(reps))
    return [r for r in reps if r.norm > mean]


def score_detection(candidates: list, attacks: list) -> DetectionReport:
    """score_detection (ddos.cpp:131-164)."""
    rep = DetectionReport(candidates=list(candidates))
    if not rep.candidates and not attacks:
        return rep
    tp = 0
    for c in rep.candidates:
        hit = next((a for a in attacks if a.victim == c.dst), None)
        if hit is not None:
            tp += 1
            if hit.bin == c.bin:
                rep.time_matches += 1
    recalled = sum(1 for a in attacks if any(c.dst == a.victim for c in rep.candidates))
    rep.precision = 0.0 if not rep.candidates else tp / len(rep.candidates)
    rep.recall = 0.0 if not attacks else recalled / len(attacks)
    pr = rep.precision + rep.recall
    rep.f1 = 0.0 if pr == 0.0 else 2.0 * rep.precision * rep.recall / pr
    return rep


def decompose_online(x, mode: int, d: int, epsilon: float = 1e-6, seed: int = 42, ctx=None) -> api.LRFactors:
    """decompose_online (ddos.cpp:166-184): init_stream on the shortest prefix
    holding traffic, then one ctd_d_step per remaining slab; the stream's
    factors (with its core)."""
    if not isinstance(x, api.SparseTensor):
        x = api.SparseTensor.from_datagen(x)
    if x.order < 2:
        raise api.ArgumentError("online decomposition needs a time mode")
    if x.nnz == 0:
        raise api.EmptyInputError("cannot decompose an empty traffic tensor")
    ctx = ctx or api.default_context()
    horizon = int(x.shape[-1])
    first = 0
    while harness.time_slab(x, first, first + 1).nnz == 0:
        first += 1
    st = api.init_stream(api.DeviceTensor(harness.time_slab(x, 0, first + 1), ctx), mode, d, epsilon, seed,
                         with_core=True, ctx=ctx)
    for t in range(first + 1, horizon):
        api.ctd_d_step(st, api.DeviceTensor(harness.time_slab(x, t, t + 1), ctx), d)
    return st.factors()
