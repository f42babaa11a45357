"""Sharded CTD-S across ranks: one process per GPU, nonzeros
partitioned by contiguous fiber-id range.

Per rank (reference functions in parentheses):
  1. bucket the local shard and compute its fibers' exact squared norms
     (matricize + column_sq_norms, tensor_ops.cpp:118-135,194-202);
  2. the sampling law's two sequential sums (the normalizer and the CDF,
     sampling.cpp:26-27,42-49) run over the columns in order, and the shards are
     ascending column ranges, so each sum is CHAINED across the ranks: rank r
     resumes it from the running value rank r-1 passes on (one double per hop)
     over its own fibers only, bit-exact.  Every rank then generates the same
     mt19937_64 uniforms and resolves the draws that fall in its CDF segment;
     an all-gather of the (draw, fiber) pairs and a replicated dedup give the
     unique list (sample_with_replacement / unique_first_occurrence,
     sampling.cpp:33-78).  Law work per rank is its shard, whatever N is;
  3. the owner of each unique candidate contributes its fiber; an all-gather
     assembles every candidate in draw order on every rank;
  4. the filter and U recurrence run replicated (deterministic: identical
     decisions and bits on every rank, FiberBasis::try_append_fiber,
     fiber_basis.cpp:43-109);
  5. the relative error's two sums are computed on each shard and all-reduced
     (relative_error, evaluation.cpp:88-122; the scalar is only checked to
     1e-9, so the reduction order does not matter).

Collectives go through torch.distributed (NCCL over NVLink on GPUs, gloo on
CPU tests).  The per-rank compute is a `kernels` object: `GpuKernels` (the
C-ABI library, the only product implementation) by default.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import ctd as api


# ---------------------------------------------------------------------------
# fiber ids and range partitions

def fiber_strides(shape, mode):
    """fiber_strides (tensor_ops.cpp:106-116): the non-mode extents, first fastest."""
    strides = []
    s = 1
    for k, n in enumerate(shape):
        if k == mode:
            strides.append(0)
        else:
            strides.append(s)
            s *= int(n)
    return np.asarray(strides, dtype=np.int64), s


def fiber_ids(shape, mode, idx: np.ndarray) -> np.ndarray:
    st, _ = fiber_strides(shape, mode)
    return (np.asarray(idx, dtype=np.int64) * st[None, :]).sum(axis=1)


def fiber_range_bounds(shape, mode, idx: np.ndarray, world: int) -> np.ndarray:
    """Contiguous fiber-id ranges [b[r], b[r+1]) balanced by nnz (world+1 bounds)."""
    _, n_cols = fiber_strides(shape, mode)
    j = np.sort(fiber_ids(shape, mode, idx))
    b = [0]
    for r in range(1, world):
        q = j[min(len(j) - 1, (len(j) * r) // world)] if len(j) else 0
        b.append(max(b[-1], int(q)))
    b.append(n_cols)
    return np.asarray(b, dtype=np.int64)


def shard(x_shape, idx: np.ndarray, val: np.ndarray, mode: int, bounds: np.ndarray, rank: int):
    """The entries of the global tensor whose fiber id lies in rank's range
    (still in the global index space, so fiber ids stay global)."""
    j = fiber_ids(x_shape, mode, idx)
    sel = (j >= bounds[rank]) & (j < bounds[rank + 1])
    return idx[sel], val[sel]


# ---------------------------------------------------------------------------
# collectives (torch.distributed)

class Comm:
    def __init__(self, group=None):
        import torch
        import torch.distributed as dist
        self.torch, self.dist, self.group = torch, dist, group
        self.rank = dist.get_rank(group)
        self.world = dist.get_world_size(group)
        backend = dist.get_backend(group)
        self.device = (torch.device("cuda", torch.cuda.current_device())
                       if backend == "nccl" else torch.device("cpu"))

    def _t(self, a: np.ndarray):
        return self.torch.from_numpy(np.ascontiguousarray(a)).to(self.device)

    def allgather(self, a: np.ndarray) -> list:
        """Variable-length all-gather of a 1-D array; returns every rank's array."""
        n = self._t(np.array([a.shape[0]], dtype=np.int64))
        ns = [self.torch.zeros_like(n) for _ in range(self.world)]
        self.dist.all_gather(ns, n, group=self.group)
        ns = [int(t.item()) for t in ns]
        m = max(ns) if ns else 0
        buf = np.zeros(max(m, 1), dtype=a.dtype)
        buf[:a.shape[0]] = a
        t = self._t(buf)
        outs = [self.torch.zeros_like(t) for _ in range(self.world)]
        self.dist.all_gather(outs, t, group=self.group)
        return [o.cpu().numpy()[:k] for o, k in zip(outs, ns)]

    def allreduce_sum(self, a: np.ndarray) -> np.ndarray:
        t = self._t(a)
        self.dist.all_reduce(t, op=self.dist.ReduceOp.SUM, group=self.group)
        return t.cpu().numpy()

    def allgather_dev(self, t, counts):
        """Variable-length all-gather of a 1-D DEVICE tensor whose length on rank
        r is counts[r] (known everywhere); the concatenation in rank order on
        t's device.  NCCL gathers in place on the device (all_gather_into_tensor);
        gloo (CPU tests) stages through the host."""
        torch = self.torch
        m = max(max(counts), 1)
        buf = torch.zeros(m, dtype=t.dtype, device=t.device)
        buf[:t.shape[0]] = t
        if self.device.type == "cuda":
            out = torch.empty(self.world * m, dtype=t.dtype, device=t.device)
            self.dist.all_gather_into_tensor(out, buf, group=self.group)
            parts = [out[r * m: r * m + counts[r]] for r in range(self.world)]
        else:
            cb = buf.cpu()
            outs = [torch.empty_like(cb) for _ in range(self.world)]
            self.dist.all_gather(outs, cb, group=self.group)
            parts = [o[:counts[r]].to(t.device) for r, o in enumerate(outs)]
        return torch.cat(parts)

    def chain(self, fn, start: float = 0.0):
        """Sequential hand-off in rank order: rank r receives the value rank r-1
        produced (rank 0 starts from `start`), applies fn, passes the result on.
        Returns (value received, value produced)."""
        v = self.torch.tensor([start], dtype=self.torch.float64, device=self.device)
        if self.rank > 0:
            self.dist.recv(v, src=self.global_rank(self.rank - 1), group=self.group)
        c_in = float(v.item())
        c_out = fn(c_in)
        if self.rank < self.world - 1:
            v = self.torch.tensor([c_out], dtype=self.torch.float64, device=self.device)
            self.dist.send(v, dst=self.global_rank(self.rank + 1), group=self.group)
        return c_in, c_out

    def bcast(self, value: float, src: int) -> float:
        v = self.torch.tensor([value], dtype=self.torch.float64, device=self.device)
        self.dist.broadcast(v, src=self.global_rank(src), group=self.group)
        return float(v.item())

    def global_rank(self, r: int) -> int:
        return r if self.group is None else self.dist.get_global_rank(self.group, r)


# ---------------------------------------------------------------------------
# per-rank kernels (the C-ABI library)

@dataclass
class LocalFibers:
    """Compressed CSC of the local shard's nonempty fibers (global column ids)."""
    col: np.ndarray
    ptr: np.ndarray
    row: np.ndarray
    val: np.ndarray
    norm: np.ndarray


class GpuKernels:
    """Per-rank compute through libctd_gpu (no CPU fallback).  `device_plane`:
    candidate payloads stay in device memory (owner gather -> device all-gather
    -> draw-order assembly -> filter), no host round trip."""

    device_plane = True

    def __init__(self, ctx: Optional[api.Context] = None):
        self.ctx = ctx or api.default_context()
        self.L = self.ctx.L

    def shard(self, x, mode):
        """Bucket this rank's entries once (x: DeviceTensor, or (shape, idx, val) host
        arrays in the global index space); the fibers stay resident in HBM."""
        if not isinstance(x, api.DeviceTensor):
            shape, idx, val = x
            x = api.DeviceTensor(api.SparseTensor(list(shape), idx, val), self.ctx)
        return _GpuShard(self, x, mode)

    def unique(self, drawn):
        drawn = np.ascontiguousarray(drawn, np.int64)
        out = np.zeros(max(drawn.shape[0], 1), np.int64)
        n = C.c_int64()
        api._check(self.L.ctd_gpu_unique_first_occurrence(self.ctx.h, api._p(drawn), drawn.shape[0], api._p(out),
                                                          C.byref(n)))
        return out[:n.value].copy()

    def sample_fibers(self, col, norm, s, seed):
        col = np.ascontiguousarray(col, dtype=np.int64)
        norm = np.ascontiguousarray(norm, dtype=np.float64)
        out = np.zeros(s, dtype=np.int64)
        nu = C.c_int64()
        tot = C.c_double()
        api._check(self.L.ctd_gpu_sample_fibers(self.ctx.h, col.shape[0], api._p(col), api._p(norm), s,
                                                C.c_uint64(seed), C.byref(tot), api._p(out), C.byref(nu)))
        return tot.value, out[:nu.value].copy()

    def basis(self, dim):
        return _GpuBasis(self, dim)

    def core_shard(self, hist_shard, basis):
        return _GpuCoreShard(self, hist_shard, basis)


class _GpuCoreShard:
    """This rank's columns of a sharded stream's Eq. 13 core (ctd_gpu_core_shard)."""

    def __init__(self, k, hist_shard, basis):
        self.k = k
        h = C.c_void_p()
        api._check(k.L.ctd_gpu_core_shard_create(hist_shard.h, basis.h, C.byref(h)))
        self.h = h

    def begin(self, basis):
        api._check(self.k.L.ctd_gpu_core_shard_begin(self.h, basis.h))

    def step(self, slab_shard, basis, col_offset: int):
        api._check(self.k.L.ctd_gpu_core_shard_step(self.h, slab_shard.h, basis.h, int(col_offset)))

    def columns(self):
        nc, nz = C.c_int64(), C.c_int64()
        api._check(self.k.L.ctd_gpu_core_shard_copy(self.h, C.byref(nc), C.byref(nz), None, None, None, None))
        col = np.zeros(max(nc.value, 1), np.int64)
        ptr = np.zeros(nc.value + 1, np.int64)
        rows = np.zeros(max(nz.value, 1), np.int64)
        vals = np.zeros(max(nz.value, 1))
        api._check(self.k.L.ctd_gpu_core_shard_copy(self.h, C.byref(nc), C.byref(nz), api._p(col), api._p(ptr),
                                                    api._p(rows), api._p(vals)))
        return col[:nc.value], ptr, rows[:nz.value], vals[:nz.value]

    def close(self):
        if getattr(self, "h", None):
            self.k.L.ctd_gpu_core_shard_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _GpuShard:
    def __init__(self, k: GpuKernels, x: "api.DeviceTensor", mode: int):
        self.k, self.x = k, x
        h = C.c_void_p()
        api._check(k.L.ctd_gpu_shard_create(k.ctx.h, x.h, mode, C.byref(h)))
        self.h = h
        F = int(k.L.ctd_gpu_shard_n_fibers(h))
        self.col = np.zeros(max(F, 1), np.int64)
        self.norm = np.zeros(max(F, 1))
        api._check(k.L.ctd_gpu_shard_fibers(h, api._p(self.col), api._p(self.norm)))
        self.col, self.norm = self.col[:F], self.norm[:F]

    def gather(self, cols):
        cols = np.ascontiguousarray(cols, np.int64)
        n = cols.shape[0]
        ptr = np.zeros(n + 1, np.int64)
        api._check(self.k.L.ctd_gpu_shard_gather(self.h, n, api._p(cols), api._p(ptr), None, None))
        rows = np.zeros(max(int(ptr[-1]), 1), np.int64)
        vals = np.zeros(max(int(ptr[-1]), 1))
        api._check(self.k.L.ctd_gpu_shard_gather(self.h, n, api._p(cols), api._p(ptr), api._p(rows), api._p(vals)))
        return ptr, rows[:ptr[-1]], vals[:ptr[-1]]

    def gather_device(self, cols):
        """(cand_ptr on the host, rows int32 and vals on the device) of the given
        local fibers, in the given order."""
        import torch
        cols = np.ascontiguousarray(cols, np.int64)
        n = cols.shape[0]
        ptr = np.zeros(n + 1, np.int64)
        api._check(self.k.L.ctd_gpu_shard_gather(self.h, n, api._p(cols), api._p(ptr), None, None))
        dev = torch.device("cuda", torch.cuda.current_device())
        rows = torch.empty(max(int(ptr[-1]), 1), dtype=torch.int32, device=dev)
        vals = torch.empty(max(int(ptr[-1]), 1), dtype=torch.float64, device=dev)
        api._check(self.k.L.ctd_gpu_shard_gather_device(self.h, n, api._p(cols), api._p(ptr), rows.data_ptr(),
                                                        vals.data_ptr()))
        return ptr, rows[:int(ptr[-1])], vals[:int(ptr[-1])]

    def error_partials(self, basis):
        xs, cr = C.c_double(), C.c_double()
        api._check(self.k.L.ctd_gpu_shard_error_partials(self.h, basis.h, C.byref(xs), C.byref(cr)))
        return xs.value, cr.value

    def nnz_local(self):
        return int(self.x.nnz)

    def core(self, basis):
        """This shard's core columns C_p = R^T X_p from the replicated basis
        (compute_core, ctd_static.cpp:12-17): (col_id, col_ptr, rows, vals)."""
        nc, nz = C.c_int64(), C.c_int64()
        api._check(self.k.L.ctd_gpu_shard_core(self.h, basis.h, C.byref(nc), C.byref(nz)))
        col = np.zeros(max(nc.value, 1), np.int64)
        ptr = np.zeros(nc.value + 1, np.int64)
        rows = np.zeros(max(nz.value, 1), np.int64)
        vals = np.zeros(max(nz.value, 1))
        api._check(self.k.L.ctd_gpu_shard_core_copy(self.h, api._p(col), api._p(ptr), api._p(rows), api._p(vals)))
        return col[:nc.value], ptr, rows[:nz.value], vals[:nz.value]

    # the chained sampling law (ctd_gpu_shard_seq_total / _cdf / _clamp / _draw)
    def seq_total(self, start):
        out = C.c_double()
        api._check(self.k.L.ctd_gpu_shard_seq_total(self.h, C.c_double(start), C.byref(out)))
        return out.value

    def cdf(self, total, start):
        end, pos = C.c_double(), C.c_int()
        api._check(self.k.L.ctd_gpu_shard_cdf(self.h, C.c_double(total), C.c_double(start), C.byref(end),
                                              C.byref(pos)))
        return end.value, bool(pos.value)

    def clamp(self):
        api._check(self.k.L.ctd_gpu_shard_clamp(self.h))

    def draw(self, count, seed):
        out = np.zeros(max(count, 1), np.int64)
        api._check(self.k.L.ctd_gpu_shard_draw(self.h, count, C.c_uint64(seed), api._p(out)))
        return out[:count]

    def close(self):
        if getattr(self, "h", None):
            self.k.L.ctd_gpu_shard_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


class _GpuBasis:
    def __init__(self, k: GpuKernels, dim: int):
        self.k, self.dim = k, dim
        h = C.c_void_p()
        api._check(k.L.ctd_gpu_basis_create(k.ctx.h, dim, C.byref(h)))
        self.h = h

    def append_batch(self, ptr, rows, vals, eps):
        n = ptr.shape[0] - 1
        acc = np.zeros(max(n, 1), np.int32)
        deg = np.zeros(max(n, 1), np.int32)
        dl = np.zeros(max(n, 1))
        ptr = np.ascontiguousarray(ptr, np.int64)
        rows = np.ascontiguousarray(rows, np.int64)
        vals = np.ascontiguousarray(vals, np.float64)
        api._check(self.k.L.ctd_gpu_basis_append_batch(self.h, n, api._p(ptr), api._p(rows), api._p(vals), eps,
                                                       api._p(acc), api._p(deg), api._p(dl)))
        return acc[:n], deg[:n], dl[:n]

    def append_batch_device(self, ptr, rows, vals, eps):
        """Candidates in device memory (rows int32, vals fp64 torch tensors)."""
        import torch
        n = ptr.shape[0] - 1
        acc = np.zeros(max(n, 1), np.int32)
        deg = np.zeros(max(n, 1), np.int32)
        dl = np.zeros(max(n, 1))
        ptr = np.ascontiguousarray(ptr, np.int64)
        rows = rows.to(torch.int32).contiguous()
        vals = vals.to(torch.float64).contiguous()
        torch.cuda.current_stream().synchronize()  # the assembly ran on torch's stream
        api._check(self.k.L.ctd_gpu_basis_append_batch_device(self.h, n, api._p(ptr), rows.data_ptr(),
                                                              vals.data_ptr(), eps, api._p(acc), api._p(deg),
                                                              api._p(dl)))
        return acc[:n], deg[:n], dl[:n]

    def size(self):
        return int(self.k.L.ctd_gpu_basis_size(self.h))

    def u(self):
        K = self.size()
        u = np.zeros(K * K)
        if K:
            api._check(self.k.L.ctd_gpu_basis_u(self.h, api._p(u)))
        return u.reshape(K, K)

    def r(self):
        K = self.size()
        nnz = int(self.k.L.ctd_gpu_basis_r_nnz(self.h))
        cp = np.zeros(K + 1, np.int64)
        rows = np.zeros(max(nnz, 1), np.int64)
        vals = np.zeros(max(nnz, 1))
        api._check(self.k.L.ctd_gpu_basis_r(self.h, api._p(cp), api._p(rows), api._p(vals)))
        return cp, rows[:nnz], vals[:nnz]

    def close(self):
        if getattr(self, "h", None):
            self.k.L.ctd_gpu_basis_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# the sharded front end

@dataclass
class ShardedResult:
    kept_flat: np.ndarray
    U: np.ndarray
    R_col_ptr: np.ndarray
    R_row: np.ndarray
    R_val: np.ndarray
    unique: np.ndarray
    accepted: np.ndarray
    degenerate: np.ndarray
    delta: np.ndarray
    total_sq_norm: float
    relative_error: Optional[float] = None
    n_fibers: int = 0
    stats: dict = field(default_factory=dict)
    # with_core: this rank's core columns (col_id, col_ptr, rows, vals) -- C is
    # column-sharded like X -- and the global nnz(C) / memory_usage
    core: Optional[tuple] = None
    core_nnz: int = 0
    memory_usage: Optional[float] = None


def _check_ranges(sh, comm) -> int:
    """Shards must be disjoint ascending fiber ranges in rank order (checked on
    every rank's first/last column); returns the global fiber count."""
    ends = np.array([sh.col[0], sh.col[-1]] if sh.col.shape[0] else [-1, -1], dtype=np.int64)
    last = -1
    for e in comm.allgather(ends):
        if e[0] < 0:
            continue
        if e[0] <= last:
            raise api.ArgumentError("shards must hold disjoint ascending fiber ranges in rank order")
        last = e[1]
    return int(comm.allreduce_sum(np.array([sh.col.shape[0]], dtype=np.int64))[0])


def _sample_sharded(sh, comm, k, count: int, seed: int):
    """column_distribution + sample_with_replacement + unique_first_occurrence
    (sampling.cpp:21-78) over the ranks' fiber ranges: the normalizer and the
    CDF are sequential sums over the columns in order, so each is chained rank
    to rank (one double per hop, every rank summing only its own fibers); the
    rank whose CDF segment holds a uniform resolves that draw."""
    _, t_last = comm.chain(sh.seq_total, 0.0)
    total = comm.bcast(t_last, comm.world - 1)
    if not (total > 0.0):
        raise api.EmptyInputError("column distribution of a tensor without nonzero entries")
    flag = {}

    def cdf(start):
        end, has = sh.cdf(total, start)
        flag["has"] = has
        return end

    comm.chain(cdf, 0.0)
    flags = comm.allgather(np.array([1 if flag["has"] else 0], dtype=np.int64))
    if comm.rank == max(r for r, f in enumerate(flags) if f[0]):
        sh.clamp()  # the tail clamp on the rank holding the last positive column (:54)
    mine = sh.draw(count, seed)
    got = comm.allgather(np.stack([np.nonzero(mine >= 0)[0], mine[mine >= 0]], 1).reshape(-1).astype(np.int64))
    drawn = np.full(count, -1, np.int64)
    for g in got:
        g = g.reshape(-1, 2)
        drawn[g[:, 0]] = g[:, 1]
    if (drawn < 0).any():
        raise api.CtdError("a draw fell in no shard's CDF segment")
    return total, k.unique(drawn)


def _gather_candidates(sh, comm, unique):
    """The unique candidates' fibers from their owners, all-gathered and laid
    out in draw order (CSC: ptr, rows, vals) on every rank."""
    pos = np.searchsorted(sh.col, unique)
    ok = pos < sh.col.shape[0]
    mine = np.zeros(unique.shape[0], bool)
    mine[ok] = sh.col[pos[ok]] == unique[ok]
    which = np.nonzero(mine)[0].astype(np.int64)
    lptr, lrows, lvals = sh.gather(unique[which])
    g_which = comm.allgather(which)
    g_lens = comm.allgather(np.diff(lptr).astype(np.int64))
    g_rows = comm.allgather(lrows.astype(np.int64))
    g_vals = comm.allgather(lvals.astype(np.float64))
    n_u = unique.shape[0]
    owner = np.full(n_u, -1, np.int64)
    cand_len = np.zeros(n_u, np.int64)
    for r, (w, ln) in enumerate(zip(g_which, g_lens)):
        owner[w] = r
        cand_len[w] = ln
    if n_u and owner.min() < 0:
        raise api.CtdError("a drawn fiber has no owner (shards do not cover the fiber space)")
    cptr = np.concatenate([[0], np.cumsum(cand_len)]).astype(np.int64)
    crow = np.zeros(int(cptr[-1]), np.int64)
    cval = np.zeros(int(cptr[-1]))
    for w, ln, rr, vv in zip(g_which, g_lens, g_rows, g_vals):
        if w.size == 0:
            continue
        n_e = int(ln.sum())
        src0 = np.concatenate([[0], np.cumsum(ln)[:-1]])
        dst_idx = np.repeat(cptr[w] - src0, ln) + np.arange(n_e)
        crow[dst_idx] = rr[:n_e]
        cval[dst_idx] = vv[:n_e]
    return cptr, crow, cval


def _gather_candidates_device(sh, comm, unique):
    """_gather_candidates with the payload on the device: each owner gathers
    its candidates into device memory, one variable-length device all-gather
    per array (NCCL), and the draw-order layout is a device gather.  Only the
    per-candidate lengths and owners (O(candidates)) cross the host."""
    import torch
    pos = np.searchsorted(sh.col, unique)
    ok = pos < sh.col.shape[0]
    mine = np.zeros(unique.shape[0], bool)
    mine[ok] = sh.col[pos[ok]] == unique[ok]
    which = np.nonzero(mine)[0].astype(np.int64)
    lptr, lrows, lvals = sh.gather_device(unique[which])
    g_which = comm.allgather(which)
    g_lens = comm.allgather(np.diff(lptr).astype(np.int64))
    counts = [int(ln.sum()) for ln in g_lens]
    rows_all = comm.allgather_dev(lrows, counts)
    vals_all = comm.allgather_dev(lvals, counts)
    n_u = unique.shape[0]
    owner = np.full(n_u, -1, np.int64)
    cand_len = np.zeros(n_u, np.int64)
    src = np.zeros(n_u, np.int64)
    base = 0
    for r, (w, ln) in enumerate(zip(g_which, g_lens)):
        owner[w] = r
        cand_len[w] = ln
        if w.size:
            src[w] = base + np.concatenate([[0], np.cumsum(ln)[:-1]]).astype(np.int64)
        base += counts[r]
    if n_u and owner.min() < 0:
        raise api.CtdError("a drawn fiber has no owner (shards do not cover the fiber space)")
    cptr = np.concatenate([[0], np.cumsum(cand_len)]).astype(np.int64)
    total = int(cptr[-1])
    dev = rows_all.device
    if total:
        shift = torch.from_numpy(src - cptr[:-1]).to(dev)
        idx = torch.repeat_interleave(shift, torch.from_numpy(cand_len).to(dev)) + torch.arange(total, device=dev)
        crow, cval = rows_all[idx], vals_all[idx]
    else:
        crow = torch.zeros(0, dtype=torch.int32, device=dev)
        cval = torch.zeros(0, dtype=torch.float64, device=dev)
    return cptr, crow, cval


def _candidates_and_filter(sh, comm, k, B, unique, epsilon):
    """Assemble the candidates (device plane when the kernels have one) and
    run the replicated filter; (accepted, degenerate, delta, candidate nnz)."""
    if getattr(k, "device_plane", False):
        cptr, crow, cval = _gather_candidates_device(sh, comm, unique)
        acc, deg, dl = B.append_batch_device(cptr, crow, cval, epsilon)
    else:
        cptr, crow, cval = _gather_candidates(sh, comm, unique)
        acc, deg, dl = B.append_batch(cptr, crow, cval, epsilon)
    return acc, deg, dl, int(cptr[-1])


def ctd_s_sharded(shape, local, mode: int, sample_size: int, epsilon: float = 1e-6, seed: int = 42,
                  comm: Optional[Comm] = None, kernels=None, with_error: bool = False,
                  with_core: bool = False) -> ShardedResult:
    """CTD-S front end over fiber-range shards; every rank returns the same
    (replicated) kept ids, U and R.  `local` is this rank's part of X in the
    GLOBAL index space (see `shard`): a DeviceTensor or (idx, val) host arrays.
    Mirrors ctd_s (ctd_static.cpp:19-50); with_core adds compute_core
    (ctd_static.cpp:12-17, :47) as this rank's columns of C (no exchange: a
    core column is the same fiber's) and the global nnz(C) for memory_usage
    (evaluation.cpp:124-129, one all-reduce)."""
    comm = comm or Comm()
    k = kernels or GpuKernels()
    if sample_size < 1:
        raise api.ArgumentError("sample size must be at least 1")
    if not (epsilon > 0.0):
        raise api.ArgumentError("epsilon must be positive")
    import os
    import time
    trace = os.environ.get("CTD_DIST_TRACE") == "1"
    tm = [time.perf_counter()]

    def mark():
        if trace:
            try:
                import torch
                torch.cuda.synchronize()
            except Exception:
                pass
            tm.append(time.perf_counter())

    # 1. local bucketing + exact norms (resident)
    sh = k.shard(local if isinstance(local, api.DeviceTensor) else (shape, local[0], local[1]), mode)
    mark()
    n_fibers = _check_ranges(sh, comm)
    mark()
    # 2. the law, chained across the ranks; draws and dedup
    total, unique = _sample_sharded(sh, comm, k, sample_size, seed)
    mark()
    # 3-4. candidate payloads from their owners, assembled in draw order;
    # replicated filter + U recurrence
    dim = int(shape[mode])
    B = k.basis(dim)
    acc, deg, dl, cand_nnz = _candidates_and_filter(sh, comm, k, B, unique, epsilon)
    mark()
    kept = unique[np.nonzero(acc)[0]]
    U = B.u()
    rp, rr, rv = B.r()
    mark()
    if trace:
        names = ["shard", "range check", "law+draws", "candidates+filter", "U/R"]
        print("[dist trace] rank %d: " % comm.rank + " ".join(
            f"{n}={1e3 * (b - a):.1f}ms" for n, a, b in zip(names, tm[:-1], tm[1:])), flush=True)
    res = ShardedResult(kept, U, rp, rr, rv, unique, acc, deg, dl, float(total), None, n_fibers,
                        {"local_fibers": int(sh.col.shape[0]), "candidate_nnz": cand_nnz})
    # 5. the core, column-sharded like X
    if with_core:
        res.core = sh.core(B)
        nl = np.array([res.core[2].shape[0], sh.nnz_local()], dtype=np.int64)
        tot = comm.allreduce_sum(nl)
        res.core_nnz = int(tot[0])
        # memory_usage: (nnz(C) + nnz(U) + nnz(R)) / nnz(X), U's exact non-zeros
        # (dense_matrix.cpp:24-29)
        res.memory_usage = float(res.core_nnz + int(np.count_nonzero(U)) + int(rr.shape[0])) / float(tot[1])
    # 6. error partials, all-reduced
    if with_error:
        xs, cr = sh.error_partials(B)
        s = comm.allreduce_sum(np.array([xs, cr], dtype=np.float64))
        if s[0] == 0.0:
            raise api.MetricError("relative error undefined for a zero tensor")
        res.relative_error = 1.0 if U.shape[0] == 0 else float((s[0] - s[1]) / s[0])
    B.close()
    sh.close()
    return res


# ---------------------------------------------------------------------------
# the same front end with the orchestration inside the library (C++, dist.cu)

class NativeComm:
    """A `ctd_gpu_comm` for `ctd_s_sharded_native`: the library's own NCCL
    communicator (rank 0's 128-byte id is broadcast over torch.distributed,
    then every exchange is an ncclAllReduce on the library's stream), or,
    with backend="host", the host-callback communicator over torch.distributed
    (gloo: CPU tests and several ranks sharing one GPU)."""

    def __init__(self, ctx: "api.Context", backend: str = "nccl", group=None):
        import torch
        import torch.distributed as tdist
        from . import _lib
        self.L, self.ctx = ctx.L, ctx
        self.rank, self.world = tdist.get_rank(group), tdist.get_world_size(group)
        h = C.c_void_p()
        if backend == "nccl":
            idb = (C.c_ubyte * 128)()
            if self.rank == 0:
                api._check(self.L.ctd_gpu_comm_nccl_unique_id(idb))
            box = [bytes(idb)]
            src = 0 if group is None else tdist.get_global_rank(group, 0)
            tdist.broadcast_object_list(box, src=src, group=group)
            idb = (C.c_ubyte * 128).from_buffer_copy(box[0])
            api._check(self.L.ctd_gpu_comm_nccl_create(ctx.h, self.world, self.rank, idb, C.byref(h)))
        elif backend == "host":
            def allreduce(user, buf, n, dtype):
                try:
                    ct = C.c_int64 if dtype else C.c_int32
                    a = np.ctypeslib.as_array((ct * n).from_address(buf))
                    t = torch.from_numpy(a.copy())
                    tdist.all_reduce(t, op=tdist.ReduceOp.SUM, group=group)
                    a[:] = t.numpy()
                    return 0
                except Exception:  # reported by the library as a device error
                    return 1
            self._cb = _lib.ALLREDUCE_FN(allreduce)  # kept alive with the communicator
            api._check(self.L.ctd_gpu_comm_host_create(ctx.h, self.world, self.rank, self._cb, None, C.byref(h)))
        else:
            raise api.ArgumentError(f"unknown communicator backend {backend!r}")
        self.h = h

    def close(self):
        if getattr(self, "h", None):
            self.L.ctd_gpu_comm_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def ctd_s_sharded_native(local: "api.DeviceTensor", mode: int, sample_size: int, epsilon: float = 1e-6,
                         seed: int = 42, comm: Optional[NativeComm] = None, with_error: bool = False,
                         with_core: bool = False) -> ShardedResult:
    """ctd_s over fiber-range shards through `ctd_gpu_ctd_s_sharded`: the
    whole host orchestration (range check, chained law, draws, candidate
    exchange, replicated filter, error partials) runs in the library, with
    every exchange an all-reduce of a device buffer.  Same contract and
    results as `ctd_s_sharded` (`local` is this rank's part of X in the
    global index space, on the context's device)."""
    if comm is None:
        raise api.ArgumentError("ctd_s_sharded_native needs a NativeComm")
    L = comm.L
    flags = (1 if with_error else 0) | (2 if with_core else 0)
    h = C.c_void_p()
    api._check(L.ctd_gpu_ctd_s_sharded(comm.ctx.h, comm.h, local.h, mode, sample_size, C.c_double(epsilon),
                                       C.c_uint64(seed), flags, C.byref(h)))
    try:
        from . import _lib
        info = _lib.ShardedInfo()
        api._check(L.ctd_gpu_sharded_info_get(h, C.byref(info)))
        nk, nu = int(info.n_kept), int(info.n_unique)
        kept = np.zeros(max(nk, 1), np.int64)
        api._check(L.ctd_gpu_sharded_kept(h, api._p(kept)))
        uniq = np.zeros(max(nu, 1), np.int64)
        acc = np.zeros(max(nu, 1), np.int32)
        deg = np.zeros(max(nu, 1), np.int32)
        dl = np.zeros(max(nu, 1))
        api._check(L.ctd_gpu_sharded_trace(h, api._p(uniq), api._p(acc), api._p(deg), api._p(dl)))
        b = L.ctd_gpu_sharded_basis(h)
        K = int(L.ctd_gpu_basis_size(b))
        U = np.zeros((K, K))
        if K:
            api._check(L.ctd_gpu_basis_u(b, api._p(U)))
        rp = np.zeros(K + 1, np.int64)
        rr = np.zeros(max(int(info.r_nnz), 1), np.int64)
        rv = np.zeros(max(int(info.r_nnz), 1))
        api._check(L.ctd_gpu_basis_r(b, api._p(rp), api._p(rr), api._p(rv)))
        res = ShardedResult(kept[:nk], U, rp, rr[:info.r_nnz], rv[:info.r_nnz], uniq[:nu], acc[:nu], deg[:nu],
                            dl[:nu], float(info.total_sq_norm),
                            float(info.relative_error) if with_error else None, int(info.n_fibers),
                            {"local_fibers": int(info.local_fibers), "candidate_nnz": int(info.cand_nnz),
                             "native": True})
        if with_core:
            nc, nz = int(info.core_cols), int(info.core_nnz)
            col = np.zeros(max(nc, 1), np.int64)
            ptr = np.zeros(nc + 1, np.int64)
            rows = np.zeros(max(nz, 1), np.int64)
            vals = np.zeros(max(nz, 1))
            api._check(L.ctd_gpu_shard_core_copy(L.ctd_gpu_sharded_shard(h), api._p(col), api._p(ptr),
                                                 api._p(rows), api._p(vals)))
            res.core = (col[:nc], ptr, rows[:nz], vals[:nz])
        return res
    finally:
        L.ctd_gpu_sharded_destroy(h)


# ---------------------------------------------------------------------------
# CTD-D over fiber-range shards

class ShardedStream:
    """init_stream / ctd_d_step (ctd_dynamic.cpp:129-229) with every slab split
    by fiber range across the ranks: each step buckets the rank's part of the
    slab, runs the chained law with seed ^ t (:177), gathers the candidates and
    filters them against the replicated basis (:178-187).  Every rank holds the
    same kept ids (flat ids j + t * slab_columns on the grown shape, :184-185),
    R and U.  with_core: every rank also maintains ITS columns of the Eq. 13
    core (ctd_dynamic.cpp:188-222) -- the columns of its history shard and of
    its part of every slab -- from its own data and the replicated basis, so
    the core stays column-sharded with no exchange."""

    def __init__(self, hist_shape, local, mode: int, sample_size: int, epsilon: float = 1e-6, seed: int = 42,
                 comm: Optional[Comm] = None, kernels=None, with_core: bool = False):
        self.comm = comm or Comm()
        self.k = kernels or GpuKernels()
        if len(hist_shape) < 2 or not (0 <= mode < len(hist_shape) - 1):
            raise api.ArgumentError("mode must precede the time mode")
        self.mode, self.eps, self.seed = mode, epsilon, seed
        self.slab_shape = list(hist_shape[:-1])
        self.slab_cols = int(np.prod([n for i, n in enumerate(self.slab_shape) if i != mode], dtype=np.int64))
        self.t = int(hist_shape[-1])
        sh = self.k.shard((list(hist_shape), local[0], local[1]), mode)
        _check_ranges(sh, self.comm)
        _, unique = _sample_sharded(sh, self.comm, self.k, sample_size, seed)
        self.B = self.k.basis(int(hist_shape[mode]))
        acc, _, _, _ = _candidates_and_filter(sh, self.comm, self.k, self.B, unique, epsilon)
        self.core = self.k.core_shard(sh, self.B) if with_core else None  # init_stream's core (:129-147)
        sh.close()
        self.kept_flat = list(unique[np.nonzero(acc)[0]])

    def step(self, local, sample_size: int):
        """One slab of time extent 1; `local` = this rank's (idx, val) of it (slab
        index space, time coordinate 0) in its fiber range."""
        idx, val = local
        nnz = int(self.comm.allreduce_sum(np.array([len(val)], dtype=np.int64))[0])
        if nnz > 0:
            sh = self.k.shard((self.slab_shape + [1], idx, val), self.mode)
            _check_ranges(sh, self.comm)
            _, unique = _sample_sharded(sh, self.comm, self.k, sample_size, self.seed ^ self.t)
            if self.core is not None:
                self.core.begin(self.B)  # U^(t), R^(t) before this step's appends (:165-167)
            acc, _, _, _ = _candidates_and_filter(sh, self.comm, self.k, self.B, unique, self.eps)
            if self.core is not None:
                self.core.step(sh, self.B, self.t * self.slab_cols)
            sh.close()
            self.kept_flat += [int(j) + self.t * self.slab_cols for j in unique[np.nonzero(acc)[0]]]
        self.t += 1
        return self

    def U(self):
        return self.B.u()

    def core_columns(self):
        """This rank's columns of the core: (col ids ascending, col_ptr, rows, vals)."""
        if self.core is None:
            raise api.ArgumentError("the stream was created without with_core")
        return self.core.columns()

    def close(self):
        if self.core is not None:
            self.core.close()
        self.B.close()
