#!/usr/bin/env python
"""CTD-S throughput on BASELINE.json configs[1] (C2) on N B200s.

One step = one CTD-S front end over the resident C2 tensor (10^4 x 10^4 x 10^3
synthetic traffic, 1e7 coalesced nnz, c = 2000, eps = 1e-6, seed 42, mode 0):
bucketing + exact squared norms, sampling law and CDF, mt19937_64 draws and
dedup, the bit-exact independence filter + U -- the scope of the reference's
ctd_s minus compute_core (C is not materialized: ~4e9 entries at C2, SURVEY
H3), which is also what `--impl reference` times.  `value` = nnz / device-timed
step (inputs already in HBM); `e2e` = the same through the public C-ABI from
pinned host COO (H2D + D2H inside the region).  The relative-error pass
(evaluation.cpp:88-122) is reported as a second metric (`error_pass`,
`ctd_s_with_error`), since the reference evaluates it outside ctd_s
(stream_harness.cpp:72-81).  Secondary objects: C3 (CTD-D latency), C4, C5.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]

--gpus N > 1 without a torchrun environment re-launches itself under
torch.distributed.run with N ranks (fails if fewer than N GPUs are visible).
"""
from __future__ import annotations

import argparse
import ctypes as C
import json
import math
import os
import subprocess
import sys
import tempfile
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

METRIC = "ctd_s_nnz_per_s"
UNIT = "nnz/s"
C2 = dict(shape=[10000, 10000, 1000], nnz=10_000_000, c=2000, eps=1e-6, seed=42, mode=0, gen_seed=2)
WORKLOAD = ("C2: CTD-S on synthetic traffic 1e4x1e4x1e3 (Zipf(1.2) src/dst, uniform time, "
            "log-uniform counts 1..100), 1e7 coalesced nnz, c=2000, eps=1e-6, mode 0")
STEP_SCOPE = ("ctd_s front end: matricize+norms, column_distribution/CDF, mt19937_64 draws, dedup, "
              "FiberBasis filter + U (compute_core excluded: C not materialized)")


def bench_config(world: int = 1) -> dict:
    """The `config` object both arms print, identical so the driver can match them."""
    cfg = {"workload": WORKLOAD, "shape": C2["shape"], "nnz": C2["nnz"], "c": C2["c"], "eps": C2["eps"],
           "seed": C2["seed"], "mode": C2["mode"], "generator_seed": C2["gen_seed"], "step": STEP_SCOPE,
           "l2": "inputs larger than L2 (200 MB COO + 120 MB bucketed per step)"}
    if world > 1:
        cfg["workload"] = WORKLOAD + f"; weak-scaled: {world} time-concatenated C2 shards"
        cfg["parallelism"] = f"fiber-range shards x{world} (NCCL)"
    return cfg


def _np_default(o):
    if hasattr(o, "item"):
        return o.item()
    return str(o)


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    if os.path.exists(p):
        with open(p) as f:
            d = json.load(f)
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# data (cached per box in /tmp; regenerated when absent — identical bytes)

def load_c2(rank: int = 0):
    from paper_1710_03608_b200 import datagen
    seed = C2["gen_seed"] + 1000 * rank
    cache = os.path.join(tempfile.gettempdir(), f"ctd_c2_seed{seed}.npz")
    if os.path.exists(cache):
        try:
            z = np.load(cache)
            return datagen.Tensor(list(z["shape"]), z["idx"], z["val"], {"draws": int(z["draws"]),
                                                                         "seed": seed})
        except Exception:
            pass
    x = datagen.traffic(C2["shape"], C2["nnz"], seed)
    try:
        np.savez(cache, shape=np.array(x.shape), idx=x.idx, val=x.val, draws=x.meta["draws"])
    except Exception:
        pass
    return x


C3 = dict(n=5000, steps=100, slices=10, d=500, eps=1e-6, seed=42, mode=0, hist_steps=50, gen_seed=3)


def load_c3():
    from paper_1710_03608_b200 import datagen
    seed = C3["gen_seed"]
    cache = os.path.join(tempfile.gettempdir(), f"ctd_c3_seed{seed}.npz")
    if os.path.exists(cache):
        try:
            z = np.load(cache)
            return datagen.Tensor(list(z["shape"]), z["idx"], z["val"], {"seed": seed})
        except Exception:
            pass
    x = datagen.c3_stream(seed=seed, n_steps=C3["steps"], slices_per_step=C3["slices"], n=C3["n"])
    try:
        np.savez(cache, shape=np.array(x.shape), idx=x.idx, val=x.val)
    except Exception:
        pass
    return x


def time_slices(x, t0, t1):
    """Per-slice slabs [I1, I2, 1] for t0 <= t < t1 (sorted, coalesced), host arrays."""
    tm = x.order - 1
    order = np.argsort(x.idx[:, tm], kind="stable")  # keeps (src, dst) order within a slice
    ts = x.idx[order, tm]
    bounds = np.searchsorted(ts, np.arange(t0, t1 + 1))
    out = []
    for k in range(t1 - t0):
        sel = order[bounds[k]:bounds[k + 1]]
        idx = x.idx[sel].copy()
        idx[:, tm] = 0
        out.append((idx, x.val[sel].copy()))
    return out


def run_ctd_d(args, ctx, torch):
    """C3 (BASELINE configs[2]): CTD-D per-step latency.  init_stream on the first
    hist_steps x 10 slices, then one ctd_d_step per incoming slice (time extent 1,
    d = 500 samples, seed ^ t), each timed alone like stream_harness.cpp:90-92 (step
    only; slabs already resident on the device).  Scope: the whole ctd_d_step
    (slab bucketing + norms, law/CDF, draws, dedup, bit-exact filter against R(t),
    kept-id append) with the Eq. 13 core maintained as block records
    (lazy_core: each step computes the slab's columns R^T dX and the chain
    product's left factor (dR^T R) U; the bottom-left expansion over the old
    columns, dense over every historical column, is applied when the core is
    read).  `same_scope` times the step with the eagerly assembled
    core on both sides at t = 10..14, where the reference still runs."""
    from paper_1710_03608_b200 import ctd as api
    x = load_c3()
    H = C3["hist_steps"] * C3["slices"]
    T = C3["steps"] * C3["slices"]
    hist = x.time_slab(0, H)
    slabs_h = time_slices(x, H, T)
    shape1 = [C3["n"], C3["n"], 1]
    dev = [api.DeviceTensor(api.SparseTensor(shape1, i, v), ctx) if v.shape[0] else None for i, v in slabs_h]
    ht = api.DeviceTensor(api.SparseTensor.from_datagen(hist), ctx)
    t0 = time.perf_counter()
    st = api.init_stream(ht, C3["mode"], C3["d"], C3["eps"], C3["seed"], lazy_core=True, ctx=ctx)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    lat = []
    nnz_steps = 0
    bd_total = 0
    written = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for k, dt in enumerate(dev):
        if dt is None:
            continue
        i, _ = slabs_h[k]
        dF = int(np.unique(np.delete(i, C3["mode"], axis=1), axis=0).shape[0])
        before = st.core_pending()[1]
        torch.cuda.synchronize()
        e0.record()
        api.ctd_d_step(st, dt, C3["d"])
        e1.record()
        torch.cuda.synchronize()
        lat.append(e0.elapsed_time(e1) / 1e3)
        nnz_steps += dt.nnz
        w = st.core_pending()[1] - before
        written += w
        bd_total += 44 * dt.nnz + 24 * dF + 12 * w  # SURVEY 8d B_D; no C(t) tiles are read (lazy)
    n_rec, n_entries, rec_bytes = st.core_pending()
    kept_final = st.n_kept()  # factors() would assemble the core (dense bottom-left over 5e6 columns)
    lat_ms = np.array(lat) * 1e3
    for d in dev:
        if d is not None:
            d.close()
    ht.close()
    st.close()
    out = {"workload": "C3: CTD-D on 5000x5000 src x dst, 10 slices/step x 100 steps, Zipf(1.2), "
                       "counts 1..50, planted 50x50x10 block (+100) at step 60; d=500, eps=1e-6",
           "history_slices": H, "streamed_slices": len(lat), "history_nnz": hist.nnz,
           "init_stream_ms": round(init_s * 1e3, 2),
           "step_ms_p50": round(float(np.percentile(lat_ms, 50)), 3),
           "step_ms_p99": round(float(np.percentile(lat_ms, 99)), 3),
           "step_ms_mean": round(float(lat_ms.mean()), 3),
           "step_ms_max": round(float(lat_ms.max()), 3),
           "slices_per_s": round(len(lat) / (lat_ms.sum() / 1e3), 1),
           "nnz_per_s": round(nnz_steps / (lat_ms.sum() / 1e3), 1),
           "kept_final": kept_final,
           "core_records": n_rec, "core_entries_written": n_entries,
           "core_record_mb": round(rec_bytes / 2**20, 1),
           "roofline": {"bound": "hbm", "what": "B_D = 44 nnz(dX) + 24 dF + 12 nnz(core tiles written) per step "
                                                "(no C(t) tiles read: the bottom-left is applied on read), summed "
                                                "over the streamed steps / their summed device time",
                        "bytes_per_step_mean": round(bd_total / max(1, len(lat))),
                        "achieved": round(bd_total / lat_ms.sum() * 1e3 / 1e9, 2),
                        "peak": peaks()[0], "unit": "GB/s",
                        "frac": round(bd_total / lat_ms.sum() * 1e3 / 1e9 / peaks()[0], 5)},
           "scope": "whole ctd_d_step: bucketing, law, seed^t draws, dedup, bit-exact filter vs R(t), kept-id "
                    "append, and the Eq. 13 core maintained as per-step block records (slab columns R^T dX + "
                    "left factor (dR^T R) U); the bottom-left expansion is applied on read (lazy_core)"}
    out["same_scope"] = ctd_d_same_scope(args, ctx, torch, x)
    return out


def ctd_d_same_scope(args, ctx, torch, x=None):
    """ctd_d_step WITH the Eq. 13 core update (transpose_times, chain_product,
    assemble_blocks; ctd_dynamic.cpp:149-229) on both sides, same inputs, same t:
    init_stream on C3's first 10 slices, then 5 timed steps (t = 10..14)."""
    from paper_1710_03608_b200 import ctd as api
    from paper_1710_03608_b200 import datagen
    x = x if x is not None else load_c3()
    h = x.time_slab(0, 10)
    slabs = time_slices(x, 10, 15)
    shape1 = [C3["n"], C3["n"], 1]
    nnz = sum(int(v.shape[0]) for _, v in slabs)
    st = api.init_stream(api.SparseTensor.from_datagen(h), C3["mode"], C3["d"], C3["eps"], C3["seed"],
                         with_core=True, ctx=ctx)
    dev = [api.DeviceTensor(api.SparseTensor(shape1, i, v), ctx) for i, v in slabs]
    torch.cuda.synchronize()
    lat = []
    for dt in dev:
        t0 = time.perf_counter()
        api.ctd_d_step(st, dt, C3["d"])
        torch.cuda.synchronize()
        lat.append(time.perf_counter() - t0)
    f = st.factors()
    gpu_core = int(f.C_val.shape[0]) if getattr(f, "C_val", None) is not None else None
    for d in dev:
        d.close()
    st.close()
    out = {"what": "ctd_d_step incl. the Eq. 13 core (bit-exact with the reference's), t = 10..14 after "
                   "init_stream on 10 slices of C3", "slab_nnz": nnz,
           "gpu_step_ms": [round(v * 1e3, 3) for v in lat], "gpu_step_ms_mean": round(float(np.mean(lat)) * 1e3, 3),
           "core_nnz_after": gpu_core}
    if not args.no_cpu:
        try:
            from oracle.bindings import Ref, ref_available
            if ref_available():
                R = Ref()
                rs = R.stream(R.tensor(h.shape, h.flat_idx(), h.val), C3["mode"], C3["d"], C3["eps"], C3["seed"])
                secs = []
                for idx, val in slabs:
                    sl = datagen.Tensor(shape1, idx, val)
                    secs.append(rs.step(R.tensor(sl.shape, sl.flat_idx(), sl.val), C3["d"]))
                out["reference_step_ms"] = [round(v * 1e3, 3) for v in secs]
                out["reference_step_ms_mean"] = round(float(np.mean(secs)) * 1e3, 3)
                out["reference"] = {"kind": "reference", "cores": 1, "cpu": _cpu_model(),
                                    "sample": "the reference ctd_d_step (oracle/_ref) on the same slabs, single-threaded"}
                out["speedup_mean"] = round(float(np.mean(secs)) / float(np.mean(lat)), 1)
        except Exception as e:  # pragma: no cover
            out["reference"] = {"sample": f"failed: {e}"}
    return out


C4 = dict(c=5000, eps=1e-6, seed=42, mode=0, gen_seed=4)
C5 = dict(shape=[100000, 100000, 1000], nnz=1_000_000_000, c=10000, eps=1e-6, seed=42, mode=0,
          gen_seed=5)


def load_c4():
    from paper_1710_03608_b200 import datagen
    seed = C4["gen_seed"]
    cache = os.path.join(tempfile.gettempdir(), f"ctd_c4_seed{seed}.npz")
    if os.path.exists(cache):
        try:
            z = np.load(cache)
            return datagen.Tensor(list(z["shape"]), z["idx"], z["val"], {"seed": seed})
        except Exception:
            pass
    x = datagen.c4(seed=seed)
    try:
        np.savez(cache, shape=np.array(x.shape), idx=x.idx, val=x.val)
    except Exception:
        pass
    return x


def _time_frontend(ctx, dt, cfg, steps, warmup, torch):
    """Device time of `steps` CTD-S front ends on a resident tensor (CUDA events on
    the launch stream), plus the per-phase split of the last run."""
    from paper_1710_03608_b200 import ctd as api
    for _ in range(warmup):
        h, info = api.ctd_s_raw(dt, cfg["mode"], cfg["c"], cfg["eps"], cfg["seed"], ctx=ctx)
        api.free_factors(ctx, h)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.phase_times(reset=True)
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    hs = []
    e0.record()
    for _ in range(steps):
        hs.append(api.ctd_s_raw(dt, cfg["mode"], cfg["c"], cfg["eps"], cfg["seed"], ctx=ctx))
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / steps
    launches = (ctx.launches - l0) // steps
    ph = ctx.phase_times(reset=True)
    ctx.set_timing(False)
    info = hs[-1][1]
    for h, _ in hs:
        api.free_factors(ctx, h)
    phases = {k: round(v[0] / max(1, v[1]), 3) for k, v in ph.items() if v[1]}
    return ms, info, phases, launches


def run_c4(args, ctx, torch):
    """BASELINE configs[3] (C4): 1000x1000x100 at 10% density, planted rank-20 CP +
    N(0, 0.01^2), non-integer fp64; c = 5000 (the filter saturates at 1000 kept and
    rejects the rest).  Same step scope as the headline (the ctd_s front end)."""
    from paper_1710_03608_b200 import ctd as api
    x = load_c4()
    dev = torch.device("cuda", torch.cuda.current_device())
    idx_t = torch.from_numpy(np.ascontiguousarray(x.idx.T.astype(np.int32))).to(dev)
    val_t = torch.from_numpy(x.val).to(dev)
    dt = api.DeviceTensor.from_device_ptrs(x.shape, x.nnz, [idx_t[k].data_ptr() for k in range(3)],
                                           val_t.data_ptr(), ctx)
    ms, info, phases, launches = _time_frontend(ctx, dt, C4, max(1, min(args.steps, 3)), 3, torch)
    out = {"workload": "C4: CTD-S on 1000x1000x100 at 10% density, planted rank-20 CP + N(0,0.01^2) "
                       "(non-integer fp64), c=5000, eps=1e-6, mode 0",
           "nnz": x.nnz, "ms_per_step": round(ms, 3), "nnz_per_s": round(x.nnz / (ms / 1e3), 1),
           "unique_sampled": info.n_unique, "kept": info.kept, "phases_ms": phases,
           "gpu_launches_per_step": launches}
    dt.close()
    if not args.no_cpu:
        try:
            from oracle.bindings import Ref, ref_available
            if ref_available():
                R = Ref()
                fe = R.frontend(R.tensor(x.shape, x.flat_idx(), x.val), C4["mode"], C4["c"], C4["eps"],
                                C4["seed"])
                out["cpu_reference"] = {"value": round(x.nnz / fe.seconds, 1), "unit": UNIT,
                                        "seconds": round(fe.seconds, 3), "cores": 1, "kind": "reference",
                                        "sample": "full C4 tensor, reference ctd_s front end, "
                                                  "single-threaded"}
        except Exception as e:  # pragma: no cover
            out["cpu_reference"] = {"sample": f"failed: {e}"}
    return out


def run_full_ctd_s(args, ctx, torch):
    """The reference's whole ctd_s (ctd_static.cpp:19-50), compute_core
    (C = X x_mode R^T, tensor_ops.cpp:27-59) included, on the configs where the
    reference finishes: C1 (configs[0]) against the reference, and C4
    (configs[3], C fully dense: ~1e8 entries) where the reference's
    compute_core alone takes ~3 min (SURVEY probe: DNF in this budget)."""
    from paper_1710_03608_b200 import ctd as api
    from paper_1710_03608_b200 import datagen
    out = {}
    for name, x, s in (("c1", datagen.c1(), 200), ("c4", load_c4(), C4["c"])):
        d = api.DeviceTensor(api.SparseTensor.from_datagen(x), ctx)
        times = []
        for it in range(4):
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            h, info = api.ctd_s_raw(d, 0, s, 1e-6, 42, ctx=ctx, with_core=True)
            e1.record()
            torch.cuda.synchronize()
            if it:
                times.append(e0.elapsed_time(e1))
            api.free_factors(ctx, h)
        d.close()
        o = {"gpu_ms": round(float(np.median(times)), 3), "nnz": x.nnz, "kept": info.kept, "c_nnz": info.c_nnz}
        if not args.no_cpu and name == "c1":
            try:
                from oracle.bindings import Ref, ref_available
                if ref_available():
                    R = Ref()
                    t = R.tensor(x.shape, x.flat_idx(), x.val)
                    secs = []
                    for _ in range(3):
                        h2 = C.c_void_p()
                        R._chk(R.L.ref_ctd_s(t.h, 0, s, 1e-6, C.c_uint64(42), C.byref(h2)), "ctd_s")
                        fe = R._factors(h2, False)
                        R.L.ref_factors_free(h2)
                        secs.append(fe.seconds)
                    o["reference_ms"] = round(float(np.median(secs)) * 1e3, 3)
                    o["speedup"] = round(o["reference_ms"] / o["gpu_ms"], 1)
            except Exception as e:  # pragma: no cover
                o["reference"] = f"failed: {e}"
        elif name == "c4":
            o["reference"] = "DNF: the reference's compute_core alone takes ~176 s at C4 (BASELINE.md section 4)"
        out[name] = o
    return out


def run_c5(args, ctx, torch):
    """BASELINE configs[4] (C5) on one GPU: 1e5x1e5x1e3 traffic with 1e9 coalesced nnz
    (Zipf(1.2) src/dst, uniform time, log-uniform counts 1..100; int32 indices),
    c = 10000.  Generated on the device (datagen_gpu, same law as the host generator);
    the front end is timed on the resident tensor (20 GB of COO, far above L2), then
    end to end from pinned host COO (32 GB in the reference's int64 layout), and the
    reference front end on a 1/100 time-scaled C5 (full C5 does not finish: ~1e9 nnz
    std::sort + a filter over fibers of ~1e4-1e5 entries)."""
    from paper_1710_03608_b200 import ctd as api
    from paper_1710_03608_b200 import datagen_gpu
    free, _ = torch.cuda.mem_get_info()
    if free < 120e9:
        return {"skipped": f"needs ~120 GB free device memory, have {free / 1e9:.0f} GB"}
    t0 = time.perf_counter()
    idx, val, meta = datagen_gpu.traffic(C5["shape"], C5["nnz"], C5["gen_seed"])
    torch.cuda.synchronize()
    gen_s = time.perf_counter() - t0
    torch.cuda.empty_cache()
    nnz = meta["nnz"]
    dt = api.DeviceTensor.from_device_ptrs(C5["shape"], nnz, [idx[k].data_ptr() for k in range(3)],
                                           val.data_ptr(), ctx)
    ms, info, phases, launches = _time_frontend(ctx, dt, C5, max(1, min(args.steps, 2)), 2, torch)
    pk, pk_kind = peaks()
    bs = 44 * nnz + 24 * info.n_fibers
    mat_ms = phases.get("matricize")
    out = {"workload": "C5: CTD-S on 1e5x1e5x1e3 traffic, 1e9 coalesced nnz (Zipf(1.2), uniform time, "
                       "log-uniform counts 1..100, int32 indices), c=10000, eps=1e-6, mode 0; 1 GPU",
           "nnz": nnz, "draws": meta["draws"], "fibers": info.n_fibers, "generate_s": round(gen_s, 2),
           "ms_per_step": round(ms, 3), "nnz_per_s": round(nnz / (ms / 1e3), 1),
           "unique_sampled": info.n_unique, "kept": info.kept, "phases_ms": phases,
           "gpu_launches_per_step": launches,
           "step_bytes_44nnz_24F": bs, "step_frac_of_peak": round(bs / (ms / 1e3) / 1e9 / pk, 4)}
    if mat_ms:
        mb = 32 * nnz + 24 * info.n_fibers
        out["roofline"] = {"bound": "hbm", "kernel": "matricize (bucketing + norms)", "achieved": round(mb / (mat_ms / 1e3) / 1e9, 1),
                           "peak": pk, "unit": "GB/s", "frac": round(mb / (mat_ms / 1e3) / 1e9 / pk, 4),
                           "bytes": mb, "peak_kind": pk_kind,
                           "note": "the HBM-bound phase at C5; the filter (latency-bound) is in phases_ms"}
    # error pass at C5 (the second metric)
    try:
        h, _ = api.ctd_s_raw(dt, C5["mode"], C5["c"], C5["eps"], C5["seed"], ctx=ctx, keep_panel=True)
        torch.cuda.synchronize()
        t1 = time.perf_counter()
        rel = api.relative_error_raw(dt, h, ctx)
        torch.cuda.synchronize()
        out["error_pass"] = {"ms_first": round((time.perf_counter() - t1) * 1e3, 2), "relative_error": rel}
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        rel = api.relative_error_raw(dt, h, ctx)
        e1.record()
        torch.cuda.synchronize()
        out["error_pass"]["ms_cached_panel"] = round(e0.elapsed_time(e1), 2)
        api.free_factors(ctx, h)
    except Exception as e:  # pragma: no cover
        out["error_pass"] = {"failed": str(e)}
    dt.close()
    # e2e: the reference's host layout (int64 AoS + fp64) from pinned memory
    if not args.no_e2e:
        try:
            out["e2e"] = c5_e2e(ctx, idx, val, nnz, torch)
        except Exception as e:  # pragma: no cover
            out["e2e"] = {"failed": str(e)}
    del idx, val
    torch.cuda.empty_cache()
    if not args.no_cpu:
        out["cpu_baseline"] = c5_cpu_baseline()
    return out


def c5_e2e(ctx, idx, val, nnz, torch):
    from paper_1710_03608_b200 import ctd as api
    ih = torch.empty((nnz, 3), dtype=torch.int64, pin_memory=True)
    vh = torch.empty(nnz, dtype=torch.float64, pin_memory=True)
    step = 1 << 27
    for a in range(0, nnz, step):
        b = min(nnz, a + step)
        ih[a:b].copy_(torch.stack([idx[0][a:b], idx[1][a:b], idx[2][a:b]], 1).to(torch.int64))
    vh.copy_(val)
    torch.cuda.synchronize()
    del idx, val
    torch.cuda.empty_cache()
    t0 = time.perf_counter()
    t = api.DeviceTensor.from_host_ptrs(C5["shape"], nnz, ih.data_ptr(), vh.data_ptr(), ctx)
    h, info = api.ctd_s_raw(t, C5["mode"], C5["c"], C5["eps"], C5["seed"], ctx=ctx)
    kept, u = api.factors_result(ctx, h, info)
    api.free_factors(ctx, h)
    t.close()
    torch.cuda.synchronize()
    sec = time.perf_counter() - t0
    return {"value": round(nnz / sec, 1), "unit": UNIT, "ms_per_step": round(sec * 1e3, 1),
            "h2d_bytes_per_step": nnz * (3 * 8 + 8), "d2h_bytes_per_step": int(kept.nbytes + u.nbytes),
            "path": "ctd_gpu_tensor_from_host (pinned int64 AoS + fp64, 32 GB) -> ctd_gpu_ctd_s -> kept ids + U"}


def c5_cpu_baseline():
    """The reference front end on C5 scaled 1/100 in time (1e5 x 1e5 x 10, 1e7 nnz,
    c = 10000): the full C5 does not fit the reference's budget (DNF)."""
    try:
        from oracle.bindings import Ref, ref_available
        from paper_1710_03608_b200 import datagen
        if not ref_available():
            return {"value": None, "sample": "unavailable: oracle/_ref/libctdref.so not built"}
        x = datagen.traffic([100000, 100000, 10], 10_000_000, C5["gen_seed"])
        R = Ref()
        t = R.tensor(x.shape, x.flat_idx(), x.val)
        fe = R.frontend(t, C5["mode"], C5["c"], C5["eps"], C5["seed"])
        return {"value": round(x.nnz / fe.seconds, 1), "unit": UNIT, "cores": 1, "kind": "reference",
                "seconds": round(fe.seconds, 3), "cpu": _cpu_model(),
                "sample": "reference ctd_s front end on C5 scaled 1/100 in time (1e5x1e5x10, 1e7 nnz, same "
                          "generator law, c=10000), single-threaded; full C5: DNF (1e9 nnz)"}
    except Exception as e:  # pragma: no cover
        return {"value": None, "sample": f"failed: {e}"}


# ---------------------------------------------------------------------------
# clocks during the timed region

class Clocks:
    Q = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
         "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
         "clocks_event_reasons.sw_power_cap")

    def __init__(self, device: int):
        self.device = device
        self.f = tempfile.NamedTemporaryFile("w+", suffix=".csv", delete=False)
        self.p = None

    def __enter__(self):
        try:
            self.p = subprocess.Popen(["nvidia-smi", "-i", str(self.device), f"--query-gpu={self.Q}",
                                       "--format=csv,noheader,nounits", "-lms", "100"],
                                      stdout=self.f, stderr=subprocess.DEVNULL)
        except Exception:
            self.p = None
        time.sleep(0.3)
        return self

    def __exit__(self, *a):
        if self.p:
            self.p.terminate()
            try:
                self.p.wait(timeout=5)
            except Exception:
                self.p.kill()

    def summary(self):
        self.f.flush()
        rows = []
        try:
            with open(self.f.name) as fh:
                for line in fh:
                    parts = [s.strip() for s in line.split(",")]
                    if len(parts) >= 8 and parts[1].replace(".", "").isdigit():
                        rows.append(parts)
        except Exception:
            pass
        if not rows:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unsampled"]}
        sm = sorted(float(r[1]) for r in rows)
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        reasons = sorted({names[i] for r in rows for i in range(4) if r[4 + i].lower() == "active"})
        return {"sm_mhz": sm[len(sm) // 2], "sm_max_mhz": float(rows[0][2]), "reasons": reasons,
                "samples": len(rows)}


# ---------------------------------------------------------------------------
# algorithmic bytes (frozen before measuring)

def phase_bytes(nnz, F, kept_seq, r_lens):
    """Algorithmic HBM bytes per phase for one CTD-S step.  Filter:
    per candidate one read of U (y = U g, the update fused into the same pass)
    and of R's row index (z = R y, 12 B/entry); per accept one write of the
    (K+1)^2 U."""
    filt = 0
    K = 0
    rn = 0
    for j, acc in enumerate(kept_seq):
        filt += 8 * K * K + 12 * rn          # y = U g reads U; z reads R's row index
        if acc:
            filt += 8 * (K + 1) * (K + 1)   # U update written once
            rn += r_lens[K]
            K += 1
    return {
        "matricize": 32 * nnz + 24 * F,      # read COO (3x4+8), write (row,val), fiber col/ptr/norm
        "law": 24 * F,                        # read norms, write probs and cumulative
        "sample": 0,
        "filter_prep": 0,
        "filter": filt,
    }


def chain_floor_cycles(kept_seq, r_ptr, r_rows, dim):
    """The filter's dependency floor: per candidate, the two sequential fp64 add
    chains the reference's summation order imposes - y = U g (K adds per row,
    dense_matrix.cpp:42-47) and z = R y (the longest R row's multiplicity,
    fiber_basis.cpp:56-65) - at the measured DADD latency (8.2 cycles,
    profiles/r1_ubench.md).  The exact residual sum and the cross-SM exchanges
    are not counted, so the floor is optimistic."""
    mult = np.zeros(dim + 1, np.int64)
    mx = 0
    K = 0
    steps = 0
    for acc in kept_seq:
        steps += K + mx
        if acc:
            rows = r_rows[r_ptr[K]:r_ptr[K + 1]]
            mult[rows] += 1
            if rows.size:
                mx = max(mx, int(mult[rows].max()))
            K += 1
    return 8.2 * steps


# ---------------------------------------------------------------------------

# phase -> its dominant kernel in the committed ncu captures (profiles/)
PHASE_KERNEL = {"filter": "k_filter", "matricize": "k_bucket_sort", "law": "k_seq_local",
                "error": "k_cd"}


def ncu_traffic(phase):
    """DRAM bytes per launch (dram__bytes_read.sum + dram__bytes_write.sum) of the phase's
    kernel from the latest committed `ncu --set full` capture (profiles/r*_kernels.json),
    or None when that kernel was not captured."""
    import glob
    kern = PHASE_KERNEL.get(phase)
    files = sorted(glob.glob(os.path.join(ROOT, "profiles", "r*_kernels.json")))
    if not kern or not files:
        return None
    for f in reversed(files):  # the newest capture that has this kernel
        rows = [d for d in json.load(open(f)) if d.get("kernel") == kern
                and d.get("dram_read") is not None and d.get("dram_write") is not None]
        if rows:
            return int(sum(d["dram_read"] + d["dram_write"] for d in rows) / len(rows))
    return None


def run_sharded(args, rank, world, local_rank):
    """N > 1: one process per GPU, sharded CTD-S (paper_1710_03608_b200.dist).
    Weak scaling: the global tensor is the time-concatenation of N C2-sized traffic
    shards (rank r generates its own, times shifted by 1000 r), so at mode 0 rank r
    owns the contiguous fiber range [r, r+1) x 1e7.  Collectives (NCCL): all-gather of
    the fibers' ids and exact norms and of the owned candidates, all-reduce of the
    error partials; law/draws/filter replicated.  value = global nnz / max-rank time."""
    import torch

    import paper_1710_03608_b200 as ctd
    from paper_1710_03608_b200 import ctd as api
    from paper_1710_03608_b200 import dist

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    ctx = ctd.Context(local_rank, torch.cuda.current_stream().cuda_stream)
    comm = dist.Comm()
    kern = dist.GpuKernels(ctx)
    x = load_c2(rank)
    T0 = C2["shape"][2]
    gshape = [C2["shape"][0], C2["shape"][1], T0 * world]
    idx = x.idx.copy()
    idx[:, 2] += T0 * rank
    nnz_local = x.nnz
    nnz = int(comm.allreduce_sum(np.array([nnz_local], dtype=np.int64))[0])
    idx_t = torch.from_numpy(np.ascontiguousarray(idx.T.astype(np.int32))).to(dev)
    val_t = torch.from_numpy(x.val).to(dev)
    dt = api.DeviceTensor.from_device_ptrs(gshape, nnz_local, [idx_t[k].data_ptr() for k in range(3)],
                                           val_t.data_ptr(), ctx)
    c, eps, seed, mode = C2["c"], C2["eps"], C2["seed"], C2["mode"]
    # default: the orchestration inside the library (ctd_gpu_ctd_s_sharded, C++;
    # NCCL communicator of its own, or host callbacks when the ranks share a GPU
    # over gloo); CTD_BENCH_DIST=py: the Python orchestrator (dist.ctd_s_sharded)
    native = os.environ.get("CTD_BENCH_DIST", "native") != "py"
    if native:
        ncomm = dist.NativeComm(ctx, "nccl" if torch.distributed.get_backend() == "nccl" else "host")

    def step(src=dt, err=False):
        if native:
            local = src if isinstance(src, api.DeviceTensor) else api.DeviceTensor(
                api.SparseTensor(gshape, src[0], src[1]), ctx)
            return dist.ctd_s_sharded_native(local, mode, c, eps, seed, comm=ncomm, with_error=err)
        return dist.ctd_s_sharded(gshape, src, mode, c, eps, seed, comm=comm, kernels=kern, with_error=err)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.phase_times(reset=True)
    l0 = ctx.launches
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(local_rank) as clk:
        e0.record()
        for _ in range(args.steps):
            r = step()
        e1.record()
        torch.cuda.synchronize()
        sec = e0.elapsed_time(e1) / 1e3 / args.steps
    torch.distributed.barrier()
    launches = ctx.launches - l0
    phases = ctx.phase_times(reset=True)
    ctx.set_timing(False)
    t = torch.tensor([sec], device=dev, dtype=torch.float64)
    torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
    sec = float(t.item())
    value = nnz / sec
    rel = step(err=True).relative_error
    # e2e: the local shard from pinned host memory each step
    e2e = None
    if not args.no_e2e:
        ih = torch.from_numpy(np.ascontiguousarray(idx)).pin_memory().numpy()
        vh = torch.from_numpy(np.ascontiguousarray(x.val)).pin_memory().numpy()
        step((ih, vh))
        torch.distributed.barrier()
        t0 = time.perf_counter()
        k = max(1, min(args.steps, 3))
        for _ in range(k):
            rr = step((ih, vh))
        torch.cuda.synchronize()
        es = torch.tensor([(time.perf_counter() - t0) / k], device=dev, dtype=torch.float64)
        torch.distributed.all_reduce(es, op=torch.distributed.ReduceOp.MAX)
        e2e = {"value": round(nnz / float(es.item()), 1), "unit": UNIT,
               "h2d_bytes_per_step": nnz_local * (3 * 8 + 8) * world,
               "d2h_bytes_per_step": int(rr.kept_flat.nbytes + rr.U.nbytes) * world,
               "path": "per rank: host shard -> ctd_gpu_tensor_from_host -> sharded CTD-S (NCCL)"}
    pk, pk_kind = peaks()
    per_phase = {k: {"ms": round(v[0] / max(1, v[1]), 4)} for k, v in phases.items() if v[1]}
    dom = max(per_phase, key=lambda k: per_phase[k]["ms"]) if per_phase else "filter"
    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(sec * 1e3, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 generator, SURVEY §8d)",
        "config": bench_config(world),
        "orchestration": ("C++ in libctd_gpu (ctd_gpu_ctd_s_sharded), "
                          + ("NCCL all-reduces on device buffers" if torch.distributed.get_backend() == "nccl"
                             else "host-callback all-reduces (gloo)")) if native else "Python (dist.ctd_s_sharded)",
        "result": {"nnz_global": nnz, "global_shape": gshape,
                   "kept": int(r.kept_flat.shape[0]), "unique_sampled": int(r.unique.shape[0]),
                   "relative_error": rel, "fibers_global": r.n_fibers},
        "roofline": {"bound": "hbm", "kernel": dom, "achieved": None, "peak": pk, "unit": "GB/s",
                     "frac": None, "traffic": ncu_traffic(dom), "peak_kind": pk_kind,
                     "note": "multi-rank step includes host collectives; per-kernel roofline in the N=1 line"},
        "phases": per_phase, "gpu_launches": launches, "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if rank == 0:
        print(json.dumps(line, default=_np_default), flush=True)


def run_ours(args, rank, world, local_rank):
    import torch

    import paper_1710_03608_b200 as ctd
    from paper_1710_03608_b200 import ctd as api

    torch.cuda.set_device(local_rank)
    dev = torch.device("cuda", local_rank)
    stream = torch.cuda.current_stream().cuda_stream
    ctx = ctd.Context(local_rank, stream)
    x = load_c2(rank)
    nnz = x.nnz
    # resident in HBM: SoA int32 coordinates + fp64 values
    idx_t = torch.from_numpy(np.ascontiguousarray(x.idx.T.astype(np.int32))).to(dev)
    val_t = torch.from_numpy(x.val).to(dev)
    dt = api.DeviceTensor.from_device_ptrs(x.shape, nnz, [idx_t[k].data_ptr() for k in range(3)],
                                           val_t.data_ptr(), ctx)
    c, eps, seed, mode = C2["c"], C2["eps"], C2["seed"], C2["mode"]

    def step():
        h, info = api.ctd_s_raw(dt, mode, c, eps, seed, with_error=False, ctx=ctx)
        return h, info

    for _ in range(args.warmup):
        h, info = step()
        api.free_factors(ctx, h)
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.phase_times(reset=True)
    if world > 1:
        torch.distributed.barrier()
    torch.cuda.synchronize()
    l0 = ctx.launches
    start, end = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    infos = []
    with Clocks(local_rank) as clk:
        start.record()
        for _ in range(args.steps):
            h, info = step()
            infos.append((h, info))
        end.record()
        torch.cuda.synchronize()
    if world > 1:
        torch.distributed.barrier()
    launches = ctx.launches - l0
    ms = start.elapsed_time(end) / args.steps
    phases = ctx.phase_times(reset=True)
    ctx.set_timing(False)
    info = infos[-1][1]
    tr = api.factors_trace(ctx, infos[-1][0], info)
    # ---- the relative-error pass (evaluation.cpp:88-122), timed on its own:
    # the reference evaluates it outside ctd_s (stream_harness.cpp:72-81).
    for h, _ in infos:
        api.free_factors(ctx, h)
    # the factors for the error pass keep the orthonormal panel W (built by the
    # filter on request, CTD_GPU_KEEP_PANEL: ~2% of the front end, not in the
    # timed steps above, which match the reference's ctd_s)
    # (one untimed pair first: the panel kernels' module load and first allocations
    # are process start-up cost, not part of a factors' first error call)
    hw, _ = api.ctd_s_raw(dt, mode, c, eps, seed, with_error=False, ctx=ctx, keep_panel=True)
    api.relative_error_raw(dt, hw, ctx)
    api.free_factors(ctx, hw)
    torch.cuda.synchronize()
    p0 = time.perf_counter()
    q0, q1, q2 = (torch.cuda.Event(enable_timing=True) for _ in range(3))
    q0.record()
    hlast, _ = api.ctd_s_raw(dt, mode, c, eps, seed, with_error=False, ctx=ctx, keep_panel=True)
    q1.record()
    torch.cuda.synchronize()
    panel_front_ms = (time.perf_counter() - p0) * 1e3
    rel = api.relative_error_raw(dt, hlast, ctx)
    q2.record()
    torch.cuda.synchronize()
    panel_front_ms_dev = q0.elapsed_time(q1)
    err_first_ms = q1.elapsed_time(q2)
    ctx.set_timing(True)
    ctx.phase_times(reset=True)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    ne = max(1, min(args.steps, 3))
    e0.record()
    for _ in range(ne):
        rel = api.relative_error_raw(dt, hlast, ctx)
    e1.record()
    torch.cuda.synchronize()
    err_phases = ctx.phase_times(reset=True)
    ctx.set_timing(False)
    api.free_factors(ctx, hlast)
    err_ms = e0.elapsed_time(e1) / ne
    err_kernel_ms = err_phases["error"][0] / max(1, err_phases["error"][1])
    if world > 1:
        t = torch.tensor([ms], device=dev)
        torch.distributed.all_reduce(t, op=torch.distributed.ReduceOp.MAX)
        ms = float(t.item())
    value = world * nnz / (ms / 1e3)

    # ---- roofline of the dominant phase (CUDA events on the launch stream)
    pk, pk_kind = peaks()
    pb = phase_bytes(nnz, info.n_fibers, tr["accepted"], tr["r_lens"])
    per_phase = {}
    for name, (tot_ms, n) in phases.items():
        if n == 0:
            continue
        avg = tot_ms / n
        b = pb.get(name, 0)
        per_phase[name] = {"ms": round(avg, 4), "bytes": b,
                           "gbs": round(b / (avg / 1e3) / 1e9, 1) if b and avg > 0 else None}
    dom = max(per_phase, key=lambda k: per_phase[k]["ms"])
    dbytes = pb.get(dom, 0)
    dms = per_phase[dom]["ms"]
    achieved = dbytes / (dms / 1e3) / 1e9 if dms > 0 else 0.0
    roof = {"bound": "hbm", "kernel": dom, "achieved": round(achieved, 1), "peak": pk,
            "unit": "GB/s", "frac": round(achieved / pk, 4), "traffic": ncu_traffic(dom),
            "peak_kind": pk_kind}
    if dom == "filter":
        fc = chain_floor_cycles(tr["accepted"], tr["r_ptr"], tr["r_rows"], int(x.shape[C2["mode"]]))
        clk_hz = 1.965e9
        roof["latency_floor"] = {
            "what": "dependent fp64 add chains in the reference's order (y = U g: K adds; z = R y: longest "
                    "R row), 8.2-cycle DADD latency at 1965 MHz; exchanges and the exact residual sum excluded",
            "floor_ms": round(fc / clk_hz * 1e3, 3), "frac": round(fc / clk_hz * 1e3 / dms, 4)}
    # SURVEY §8d byte formula for the front-end step (the 12 B/nnz error-pass
    # re-read of 44 nnz + 24 F belongs to error_pass)
    bs = 32 * nnz + 24 * info.n_fibers

    # ---- e2e through the public C-ABI from pinned host COO
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, x, torch)

    # ---- CPU baseline: the compiled reference on this host (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(x)

    # The C3 stream runs last: its record arena (tens of GB, chunks allocated on a
    # helper thread) going back to the driver stalls whatever allocates next
    # (measured: C4 filter prep 1.4 -> 7 ms, C5 step + 300 ms when they followed it)
    c4 = c5 = full = None
    if rank == 0 and world == 1 and not args.no_c4:
        c4 = run_c4(args, ctx, torch)
        try:
            full = run_full_ctd_s(args, ctx, torch)
        except Exception as e:  # pragma: no cover
            full = {"failed": str(e)}
    if rank == 0 and world == 1 and not args.no_c5:
        del idx_t, val_t
        dt.close()
        ctx.trim()  # the library's cached blocks back to the driver for the C5 generator
        torch.cuda.empty_cache()
        c5 = run_c5(args, ctx, torch)
        ctx.trim()
        torch.cuda.empty_cache()
    ctdd = None
    if rank == 0 and world == 1 and not args.no_ctdd:
        ctdd = run_ctd_d(args, ctx, torch)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 generator, SURVEY §8d)",
        "config": bench_config(1),
        "result": {"nnz": nnz, "fibers": info.n_fibers, "unique_sampled": info.n_unique, "kept": info.kept,
                   "relative_error": rel,
                   "step_bytes_32nnz_24F": bs, "step_frac_of_peak": round(bs / (ms / 1e3) / 1e9 / pk, 4),
                   "step_bytes_note": "front end: read COO (20 B) + write bucketed row/val (12 B) per nnz, "
                                      "fiber col/ptr/norm (24 B) per fiber; the error pass's 12 B/nnz "
                                      "re-read is charged to error_pass"},
        "roofline": roof, "phases": per_phase, "gpu_launches": launches,
        "error_pass": {"ms": round(err_ms, 3), "kernel_ms": round(err_kernel_ms, 3),
                       "nnz_per_s": round(nnz / (err_ms / 1e3), 1),
                       "bytes": 32 * nnz + 24 * info.n_fibers + 12 * nnz,
                       "gbs": round((44 * nnz + 24 * info.n_fibers) / (err_ms / 1e3) / 1e9, 1),
                       "first_call_ms": round(err_first_ms, 3),
                       "what": "relative_error(X, factors): matricize + |X|^2 - sum_j |Q^T x_j|^2 over all nnz, "
                               "Q orthonormal with span(Q) = span(R) (ortho.cu: DMMA polar iteration from the "
                               "filter's residual panel, cached on the factors after the first call)",
                       "front_end_with_panel_ms": round(panel_front_ms, 3)},
        "ctd_s_with_error": {"ms_per_step": round(panel_front_ms_dev + err_first_ms, 3),
                             "nnz_per_s": round(nnz / ((panel_front_ms_dev + err_first_ms) / 1e3), 1),
                             "what": "front end (keeping the panel) + the first relative_error call (panel "
                                     "orthonormalization + sweep), device-timed"},
        "clocks": clk.summary(),
    }
    if e2e:
        line["e2e"] = e2e
    if cpu:
        line["cpu_baseline"] = cpu
    if ctdd is not None:
        line["ctd_d"] = ctdd
    if c4 is not None:
        line["c4"] = c4
    if full is not None:
        line["ctd_s_with_core"] = full
    if c5 is not None:
        line["c5"] = c5
    if rank == 0:
        print(json.dumps(line, default=_np_default), flush=True)


def run_e2e(args, ctx, x, torch):
    from paper_1710_03608_b200 import ctd as api
    nnz = x.nnz
    idx_h = torch.from_numpy(np.ascontiguousarray(x.idx, dtype=np.int64).reshape(-1)).pin_memory()
    val_h = torch.from_numpy(np.ascontiguousarray(x.val)).pin_memory()
    c, eps, seed, mode = C2["c"], C2["eps"], C2["seed"], C2["mode"]
    shape = np.asarray(x.shape, dtype=np.int64)

    u_h = torch.empty(c * c, dtype=torch.float64).pin_memory().numpy()   # the caller's result buffer

    def step():
        t = api.DeviceTensor.from_host_ptrs(x.shape, nnz, idx_h.data_ptr(), val_h.data_ptr(), ctx)
        h, info = api.ctd_s_raw(t, mode, c, eps, seed, with_error=False, ctx=ctx)
        kept, u = api.factors_result(ctx, h, info, u_out=u_h)   # D2H: kept ids + U
        api.free_factors(ctx, h)
        t.close()
        return info, kept, u

    for _ in range(max(1, min(args.warmup, 2))):
        step()
    torch.cuda.synchronize()
    k = max(1, min(args.steps, 3))
    t0 = time.perf_counter()
    for _ in range(k):
        info, kept, u = step()
    torch.cuda.synchronize()
    sec = (time.perf_counter() - t0) / k
    return {"value": round(nnz / sec, 1), "unit": UNIT, "h2d_bytes_per_step": nnz * (3 * 8 + 8),
            "d2h_bytes_per_step": int(kept.nbytes + u.nbytes), "ms_per_step": round(sec * 1e3, 3),
            "path": "ctd_gpu_tensor_from_host (pinned int64 AoS + fp64) -> ctd_gpu_ctd_s -> "
                    "kept ids + U to host"}


def cpu_baseline(x):
    """The unmodified reference (oracle/_ref) on this host's cores: the ctd_s
    front end (matricize -> column_distribution -> sample -> dedup -> FiberBasis
    loop) on the full C2 tensor.  compute_core / relative_error are excluded
    (they do not finish at this size: SURVEY §8d, H8)."""
    try:
        from oracle.bindings import Ref, ref_available
        if not ref_available():
            return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference",
                    "sample": "unavailable: oracle/_ref/libctdref.so not built"}
        R = Ref()
        t = R.tensor(x.shape, x.flat_idx(), x.val)
        fe = R.frontend(t, C2["mode"], C2["c"], C2["eps"], C2["seed"])
        sec = fe.seconds
        return {"value": round(x.nnz / sec, 1), "unit": UNIT, "cores": 1, "kind": "reference",
                "seconds": round(sec, 3),
                "sample": "full C2 tensor, reference ctd_s front end (matricize..FiberBasis loop), "
                          "single-threaded like the reference; compute_core/relative_error excluded (DNF)",
                "cpu": _cpu_model()}
    except Exception as e:  # pragma: no cover
        return {"value": None, "unit": UNIT, "cores": 1, "kind": "reference", "sample": f"failed: {e}"}


def _cpu_model():
    try:
        with open("/proc/cpuinfo") as f:
            for line in f:
                if line.startswith("model name"):
                    return line.split(":", 1)[1].strip() + f" ({os.cpu_count()} threads)"
    except Exception:
        pass
    return None


def run_reference(args, rank, world):
    """--impl reference: the reference's own CPU implementation (oracle/_ref, the
    unmodified proj/core compiled from /root/reference), rank 0 only, every step the
    full C2 front end -- the same config and step scope as our arm (the
    reference has no threading, so one host core)."""
    if rank != 0:
        return
    from oracle.bindings import Ref, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libctdref.so not built"}))
        return
    x = load_c2(0)
    R = Ref()
    t = R.tensor(x.shape, x.flat_idx(), x.val)
    secs = []
    for i in range(args.steps + args.warmup):
        fe = R.frontend(t, C2["mode"], C2["c"], C2["eps"], C2["seed"])
        if i >= args.warmup:
            secs.append(fe.seconds)
    sec = float(np.mean(secs))
    value = x.nnz / sec
    sample = ("the full C2 tensor every step: reference ctd_s front end (matricize -> column_distribution "
              "-> sample_with_replacement -> unique_first_occurrence -> FiberBasis loop); single-threaded "
              "(the reference has no threading); input SparseTensor built once outside the timer")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic (seeded splitmix64 generator, SURVEY §8d)",
        "config": bench_config(1),
        "result": {"nnz": x.nnz, "kept": int(len(fe.kept_flat)), "unique_sampled": int(len(fe.unique)),
                   "step_seconds": [round(v, 3) for v in secs]},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": sample, "cpu": _cpu_model()},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


def _relaunch(args) -> int:
    """--gpus N > 1 outside torchrun: re-launch under torch.distributed.run with N
    ranks on this node, or fail loudly when fewer than N GPUs are visible."""
    import torch
    have = torch.cuda.device_count()
    if args.impl == "ours" and have < args.gpus:
        print(f"bench.py: --gpus {args.gpus} requested but only {have} GPU(s) visible", file=sys.stderr)
        return 2
    port = 29500 + (os.getpid() % 1000)
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", os.path.abspath(__file__)] + sys.argv[1:]
    return subprocess.call(cmd)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=5)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-ctdd", action="store_true", help="skip the C3 CTD-D per-step latency run")
    ap.add_argument("--no-c4", action="store_true", help="skip the C4 (planted CP, c=5000) line")
    ap.add_argument("--no-c5", action="store_true", help="skip the C5 (1e9 nnz) line")
    args = ap.parse_args()
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(_relaunch(args))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}", file=sys.stderr)
        sys.exit(2)
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    if world > 1:
        import torch
        if os.environ.get("CTD_BENCH_SAME_GPU") == "1":
            # test hook: every rank on GPU 0 with host-side gloo collectives (one-GPU boxes)
            local_rank = 0
            backend = "gloo"
        else:
            backend = "nccl"
            if torch.cuda.device_count() < world:
                print(f"bench.py: {world} ranks but only {torch.cuda.device_count()} GPU(s) visible",
                      file=sys.stderr)
                sys.exit(2)
        torch.cuda.set_device(local_rank)
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        torch.distributed.init_process_group(backend)
    if world > 1:
        run_sharded(args, rank, world, local_rank)
    else:
        run_ours(args, rank, world, local_rank)
    if world > 1:
        import torch
        torch.distributed.destroy_process_group()


if __name__ == "__main__":
    main()
