"""Stream harness: the historical/incoming split protocol with per-step
evaluation (stream_harness.hpp / stream_harness.cpp:48-107), and the
evaluation record with its TSV form (evaluation.hpp:11-21, evaluation.cpp:47-62).

The decomposition steps and every evaluation run on the GPU through the
package API (``init_stream`` / ``ctd_d_step`` / ``relative_error`` /
``memory_usage``); this module is the host orchestration the reference's
``run_stream`` performs, with the same options, validation, step numbering,
timing scope (the step only) and averages.
"""
from __future__ import annotations

import math
import time
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import ctd as api

__all__ = ["HarnessOptions", "EvalReport", "StepReport", "StreamRunResult", "time_slab",
           "run_stream", "tsv_header", "tsv_line", "default_step_samples"]

default_step_samples = api.default_step_samples


@dataclass
class HarnessOptions:
    """HarnessOptions (stream_harness.hpp:16-24)."""
    mode: int = 0
    sample_size: int = 100
    step_samples: Optional[int] = None   # d; default max(1, round(0.01 * s))
    split: float = 0.8
    epsilon: float = 1e-6
    seed: int = 42
    exact_core: bool = False


@dataclass
class EvalReport:
    """EvalReport (evaluation.hpp:11-18)."""
    relative_error: float = 0.0
    memory_usage: float = 0.0
    wall_time_seconds: float = 0.0
    kept_fibers: int = 0


@dataclass
class StepReport:
    step: int = 0        # 0 = static bootstrap, then one per incoming slab
    eval: EvalReport = field(default_factory=EvalReport)


@dataclass
class StreamRunResult:
    steps: list = field(default_factory=list)
    mean: EvalReport = field(default_factory=EvalReport)   # dynamic steps only
    factors: Optional[api.LRFactors] = None


def _fmt(v: float) -> str:
    """format_double (evaluation.cpp:13-17): printf %.17g."""
    return "%.17g" % v


def tsv_header() -> str:
    return "step\terror\tseconds\tmemory_usage\tkept_fibers"


def tsv_line(step: int, r: EvalReport) -> str:
    return f"{int(step)}\t{_fmt(r.relative_error)}\t{_fmt(r.wall_time_seconds)}\t{_fmt(r.memory_usage)}\t" \
           f"{int(r.kept_fibers)}"


def time_slab(x: api.SparseTensor, t0: int, t1: int) -> api.SparseTensor:
    """time_slab (stream_harness.cpp:26-46): entries with t0 <= t < t1, re-based."""
    tm = x.order - 1
    if tm < 0:
        raise api.ArgumentError("tensor has no modes")
    if t0 < 0 or t1 < t0 or t1 > x.shape[tm]:
        raise api.ArgumentError("time window out of range")
    idx = np.asarray(x.indices, dtype=np.int64).reshape(-1, x.order)
    sel = (idx[:, tm] >= t0) & (idx[:, tm] < t1)
    out = idx[sel].copy()
    out[:, tm] -= t0
    shape = list(x.shape)
    shape[tm] = t1 - t0
    return api.SparseTensor(shape, out, np.asarray(x.values, dtype=np.float64)[sel].copy())


def run_stream(x, options: HarnessOptions = HarnessOptions(),
               ctx: Optional[api.Context] = None) -> StreamRunResult:
    """run_stream (stream_harness.cpp:48-107): floor(split*T) historical slabs
    decomposed by init_stream, the rest fed one by one; every step evaluated
    against the tensor grown so far (relative error, memory usage, the step's
    wall time, kept fibers)."""
    if not isinstance(x, api.SparseTensor):
        x = api.SparseTensor.from_datagen(x)
    if not (options.split > 0.0) or not (options.split < 1.0):
        raise api.ArgumentError("split must lie strictly inside (0, 1)")
    if x.order < 2:
        raise api.ArgumentError("a stream needs a time mode")
    horizon = int(x.shape[-1])
    if horizon < 5:
        raise api.ArgumentError("stream needs a time extent of at least 5")
    historical = int(math.floor(options.split * float(horizon)))
    historical = min(max(historical, 1), horizon - 1)
    d = options.step_samples if options.step_samples is not None else default_step_samples(options.sample_size)
    ctx = ctx or api.default_context()

    res = StreamRunResult()
    hist = api.DeviceTensor(time_slab(x, 0, historical), ctx)
    ctx.synchronize()
    t0 = time.perf_counter()
    state = api.init_stream(hist, options.mode, options.sample_size, options.epsilon, options.seed,
                            keep_history=False, exact_core=options.exact_core, with_core=True, ctx=ctx)
    ctx.synchronize()
    elapsed = time.perf_counter() - t0

    def evaluate(upto: int, step_seconds: float) -> EvalReport:
        prefix = api.DeviceTensor(time_slab(x, 0, upto), ctx)
        f = state.factors()
        rep = EvalReport(relative_error=api.relative_error(prefix, f, ctx),
                         memory_usage=api.memory_usage(prefix, f, ctx),
                         wall_time_seconds=step_seconds, kept_fibers=f.kept_count())
        prefix.close()
        return rep

    res.steps.append(StepReport(0, evaluate(historical, elapsed)))
    mean = EvalReport()
    dynamic = horizon - historical
    for k in range(dynamic):
        t = historical + k
        slab = api.DeviceTensor(time_slab(x, t, t + 1), ctx)
        ctx.synchronize()
        t0 = time.perf_counter()
        api.ctd_d_step(state, slab, d)
        ctx.synchronize()
        elapsed = time.perf_counter() - t0
        slab.close()
        rep = evaluate(t + 1, elapsed)
        res.steps.append(StepReport(k + 1, rep))
        mean.relative_error += rep.relative_error
        mean.memory_usage += rep.memory_usage
        mean.wall_time_seconds += rep.wall_time_seconds
        mean.kept_fibers += rep.kept_fibers
    mean.relative_error /= dynamic
    mean.memory_usage /= dynamic
    mean.wall_time_seconds /= dynamic
    mean.kept_fibers = res.steps[-1].eval.kept_fibers
    res.mean = mean
    res.factors = state.factors()
    return res
