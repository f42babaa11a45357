#!/usr/bin/env python
"""CTD-S throughput on BASELINE.json configs[1] (C2) on N B200s.

One step = one CTD-S pass over the resident C2 tensor (10^4 x 10^4 x 10^3
synthetic traffic, 1e7 coalesced nnz, c = 2000, eps = 1e-6, seed 42, mode 0):
bucketing + exact squared norms, sampling law and CDF, mt19937_64 draws and
dedup, the bit-exact independence filter + U, and the relative-error pass.
`value` = nnz / device-timed step (inputs already in HBM); `e2e` = the same
through the public C-ABI from pinned host COO (H2D + D2H inside the region).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference]
"""
from __future__ import annotations

import argparse
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
    only; slabs already resident on the device).  Scope: the step's front end
    (slab bucketing + norms, law/CDF, draws, dedup, bit-exact filter against R(t),
    kept-id append); the Eq. 13 core blocks are not maintained."""
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
    st = api.init_stream(ht, C3["mode"], C3["d"], C3["eps"], C3["seed"], ctx=ctx)
    torch.cuda.synchronize()
    init_s = time.perf_counter() - t0
    lat = []
    nnz_steps = 0
    for k, dt in enumerate(dev):
        if dt is None:
            continue
        t0 = time.perf_counter()
        api.ctd_d_step(st, dt, C3["d"])
        torch.cuda.synchronize()
        lat.append(time.perf_counter() - t0)
        nnz_steps += dt.nnz
    kept = st.factors()
    lat_ms = np.array(lat) * 1e3
    for d in dev:
        if d is not None:
            d.close()
    ht.close()
    return {"workload": "C3: CTD-D on 5000x5000 src x dst, 10 slices/step x 100 steps, Zipf(1.2), "
                        "counts 1..50, planted 50x50x10 block (+100) at step 60; d=500, eps=1e-6",
            "history_slices": H, "streamed_slices": len(lat), "history_nnz": hist.nnz,
            "init_stream_ms": round(init_s * 1e3, 2),
            "step_ms_p50": round(float(np.percentile(lat_ms, 50)), 3),
            "step_ms_p99": round(float(np.percentile(lat_ms, 99)), 3),
            "step_ms_mean": round(float(lat_ms.mean()), 3),
            "slices_per_s": round(len(lat) / (lat_ms.sum() / 1e3), 1),
            "nnz_per_s": round(nnz_steps / (lat_ms.sum() / 1e3), 1),
            "kept_final": len(kept.kept_flat) if hasattr(kept, "kept_flat") else None,
            "scope": "step front end (bucketing, law, seed^t draws, dedup, bit-exact filter vs R(t), "
                     "kept-id append); Eq. 13 core blocks not maintained (SURVEY 8f #2)"}


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
    ms, info, phases, launches = _time_frontend(ctx, dt, C4, max(1, min(args.steps, 3)), 1, torch)
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


def run_c5(args, ctx, torch):
    """BASELINE configs[4] (C5) on one GPU: 1e5x1e5x1e3 traffic with 1e9 coalesced nnz
    (Zipf(1.2) src/dst, uniform time, log-uniform counts 1..100; int32 indices),
    c = 10000.  Generated on the device (datagen_gpu, same law as the host generator);
    the front end is timed on the resident tensor (20 GB of COO, far above L2)."""
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
    ms, info, phases, launches = _time_frontend(ctx, dt, C5, max(1, min(args.steps, 2)), 1, torch)
    pk, _ = peaks()
    bs = 44 * nnz + 24 * info.n_fibers
    mat_ms = phases.get("matricize")
    out = {"workload": "C5: CTD-S on 1e5x1e5x1e3 traffic, 1e9 coalesced nnz (Zipf(1.2), uniform time, "
                       "log-uniform counts 1..100, int32 indices), c=10000, eps=1e-6, mode 0; 1 GPU",
           "nnz": nnz, "draws": meta["draws"], "fibers": info.n_fibers, "generate_s": round(gen_s, 2),
           "ms_per_step": round(ms, 3), "nnz_per_s": round(nnz / (ms / 1e3), 1),
           "unique_sampled": info.n_unique, "kept": info.kept, "phases_ms": phases,
           "gpu_launches_per_step": launches,
           "step_bytes_44nnz_24F": bs, "step_frac_of_peak": round(bs / (ms / 1e3) / 1e9 / pk, 4),
           "matricize_gbs": round((32 * nnz + 24 * info.n_fibers) / (mat_ms / 1e3) / 1e9, 1)
           if mat_ms else None}
    dt.close()
    del idx, val
    torch.cuda.empty_cache()
    return out


def ctd_d_reference_sample():
    """The reference ctd_d_step (oracle/_ref, which also updates the Eq. 13 core) on C3:
    init_stream on the first 10 slices, then 5 timed steps (a bounded sample)."""
    try:
        from oracle.bindings import Ref, ref_available
        if not ref_available():
            return None
        x = load_c3()
        R = Ref()
        h = x.time_slab(0, 10)
        st = R.stream(R.tensor(h.shape, h.flat_idx(), h.val), C3["mode"], C3["d"], C3["eps"], C3["seed"])
        secs = []
        for i, (idx, val) in enumerate(time_slices(x, 10, 15)):
            from paper_1710_03608_b200 import datagen
            sl = datagen.Tensor([C3["n"], C3["n"], 1], idx, val)
            secs.append(st.step(R.tensor(sl.shape, sl.flat_idx(), sl.val), C3["d"]))
        return {"step_ms_mean": round(float(np.mean(secs)) * 1e3, 2), "cores": 1, "kind": "reference",
                "sample": "reference ctd_d_step (includes its Eq. 13 core update) at t = 10..14 "
                          "after init_stream on 10 slices; single-threaded"}
    except Exception as e:  # pragma: no cover
        return {"sample": f"failed: {e}"}


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
    """Algorithmic HBM bytes per phase for one CTD-S step."""
    filt = 0
    K = 0
    rn = 0
    for j, acc in enumerate(kept_seq):
        filt += 8 * K * K + 12 * rn          # y = U g reads U; z reads R's row index
        if acc:
            filt += 16 * (K + 1) * (K + 1)  # U update read + write
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
    rows = [d for d in json.load(open(files[-1])) if d.get("kernel") == kern
            and d.get("dram_read") is not None and d.get("dram_write") is not None]
    if not rows:
        return None
    return int(sum(d["dram_read"] + d["dram_write"] for d in rows) / len(rows))


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

    def step(src=dt, err=False):
        return dist.ctd_s_sharded(gshape, src, mode, c, eps, seed, comm=comm, kernels=kern, with_error=err)

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    torch.distributed.barrier()
    torch.cuda.synchronize()
    ctx.set_timing(True)
    ctx.phase_times(reset=True)
    l0 = ctx.launches
    with Clocks(local_rank) as clk:
        t0 = time.perf_counter()
        for _ in range(args.steps):
            r = step()
        torch.cuda.synchronize()
        sec = (time.perf_counter() - t0) / args.steps
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
        "config": {"workload": WORKLOAD + f"; weak-scaled: {world} time-concatenated C2 shards",
                   "nnz": nnz, "global_shape": gshape, "parallelism": f"fiber-range shards x{world} (NCCL)",
                   "kept": int(r.kept_flat.shape[0]), "unique_sampled": int(r.unique.shape[0]),
                   "relative_error": rel, "fibers_global": r.n_fibers,
                   "l2": "inputs larger than L2 (200 MB COO per rank)"},
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
    torch.cuda.synchronize()
    p0 = time.perf_counter()
    hlast, _ = api.ctd_s_raw(dt, mode, c, eps, seed, with_error=False, ctx=ctx, keep_panel=True)
    torch.cuda.synchronize()
    panel_front_ms = (time.perf_counter() - p0) * 1e3
    rel = api.relative_error_raw(dt, hlast, ctx)
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
    # SURVEY §8d end-to-end byte formula for the step
    bs = 44 * nnz + 24 * info.n_fibers

    # ---- e2e through the public C-ABI from pinned host COO
    e2e = None
    if not args.no_e2e:
        e2e = run_e2e(args, ctx, x, torch)

    # ---- CPU baseline: the compiled reference on this host (rank 0, N=1)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:
        cpu = cpu_baseline(x)

    ctdd = None
    if rank == 0 and world == 1 and not args.no_ctdd:
        ctdd = run_ctd_d(args, ctx, torch)
        if not args.no_cpu:
            ctdd["cpu_reference"] = ctd_d_reference_sample()

    c4 = c5 = None
    if rank == 0 and world == 1 and not args.no_c4:
        c4 = run_c4(args, ctx, torch)
    if rank == 0 and world == 1 and not args.no_c5:
        del idx_t, val_t
        dt.close()
        torch.cuda.empty_cache()
        c5 = run_c5(args, ctx, torch)

    line = {
        "metric": METRIC, "value": round(value, 1), "unit": UNIT, "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 4),
        "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": "f64",
        "data": "synthetic (seeded splitmix64 generator, SURVEY §8d)",
        "config": {"workload": WORKLOAD, "nnz": nnz, "fibers": info.n_fibers,
                   "step": "ctd_s front end: matricize+norms, law/CDF, mt19937_64 draws, dedup, "
                           "bit-exact filter + U (C not materialized, as the CPU baseline)",
                   "unique_sampled": info.n_unique, "kept": info.kept,
                   "relative_error": rel,
                   "l2": "inputs larger than L2 (200 MB COO + 120 MB bucketed per step)",
                   "parallelism": f"fiber-range shards x{world}" if world > 1 else "1 GPU",
                   "step_bytes_44nnz_24F": bs,
                   "step_frac_of_peak": round(bs / (ms / 1e3) / 1e9 / pk, 4)},
        "roofline": roof, "phases": per_phase, "gpu_launches": launches,
        "error_pass": {"ms": round(err_ms, 3), "kernel_ms": round(err_kernel_ms, 3),
                       "nnz_per_s": round(nnz / (err_ms / 1e3), 1),
                       "what": "relative_error(X, factors): matricize + one pass over all nnz against the orthonormal panel W = R T (U = T T^T)",
                       "panel": "W kept by the filter on request (CTD_GPU_KEEP_PANEL)",
                       "front_end_with_panel_ms": round(panel_front_ms, 3)},
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

    def step():
        t = api.DeviceTensor.from_host_ptrs(x.shape, nnz, idx_h.data_ptr(), val_h.data_ptr(), ctx)
        h, info = api.ctd_s_raw(t, mode, c, eps, seed, with_error=False, ctx=ctx)
        kept, u = api.factors_result(ctx, h, info)   # D2H: kept ids + U
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
    """--impl reference: the reference's own CPU implementation (oracle/_ref),
    rank 0 only, each step a bounded sample of C2 (the first T' time slices)."""
    if rank != 0:
        return
    from oracle.bindings import Ref, ref_available
    if not ref_available():
        print(json.dumps({"impl": "reference", "unavailable": "oracle/_ref/libctdref.so not built"}))
        return
    x = load_c2(0)
    n_steps = args.steps + args.warmup
    frac = 1.0 if n_steps <= 6 else max(0.05, 6.0 / n_steps)
    T1 = max(1, int(round(C2["shape"][2] * frac)))
    xs = x if T1 >= C2["shape"][2] else x.time_slab(0, T1)
    R = Ref()
    t = R.tensor(xs.shape, xs.flat_idx(), xs.val)
    secs = []
    for i in range(n_steps):
        fe = R.frontend(t, C2["mode"], C2["c"], C2["eps"], C2["seed"])
        if i >= args.warmup:
            secs.append(fe.seconds)
    sec = float(np.mean(secs))
    value = xs.nnz / sec
    sample = (f"reference ctd_s front end on the first {T1} of 1000 time slices of C2 "
              f"({xs.nnz} nnz); single-threaded (the reference has no threading)")
    print(json.dumps({
        "impl": "reference", "metric": METRIC, "value": round(value, 1), "unit": UNIT,
        "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": round(sec * 1e3, 3), "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "f64", "data": "synthetic",
        "config": {"workload": WORKLOAD, "sample_nnz": xs.nnz},
        "cpu_baseline": {"value": round(value, 1), "unit": UNIT, "cores": 1, "kind": "reference",
                         "sample": sample, "cpu": _cpu_model()},
        "e2e": {"value": round(value, 1), "unit": UNIT, "h2d_bytes_per_step": 0,
                "d2h_bytes_per_step": 0}}), flush=True)


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
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local_rank = int(os.environ.get("LOCAL_RANK", "0"))
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
