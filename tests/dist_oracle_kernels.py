"""Test-only per-rank kernels for paper_1710_03608_b200.dist built on the CPU
oracle (oracle/ctd_oracle.c via oracle.bindings.Port), so the sharded host
logic and its collectives can run in gloo world_size>1 tests without a GPU.
Never used by the product path (GpuKernels is the only product backend).
"""
import numpy as np

from paper_1710_03608_b200.dist import LocalFibers


class OracleKernels:
    def __init__(self, port):
        self.P = port

    def shard(self, x, mode):
        shape, idx, val = x
        return _OracleShard(self.P, shape, idx, val, mode)

    def sample_fibers(self, col, norm, s, seed):
        # column_distribution (sampling.cpp:21-31): sequential total, p = n / T
        total = 0.0
        for v in norm:
            total += float(v)
        probs = np.asarray(norm, dtype=np.float64) / total
        drawn = self.P.sample_with_replacement(probs, s, seed)
        uniq = self.P.unique_first_occurrence(drawn)
        return total, np.asarray(col, dtype=np.int64)[uniq]

    def unique(self, drawn):
        return self.P.unique_first_occurrence(drawn)

    def basis(self, dim):
        return _OracleBasis(self.P.basis(dim))

    def core_shard(self, hist_shard, basis):
        return _OracleCoreShard(self.P, hist_shard, basis)


class _OracleShard:
    def __init__(self, P, shape, idx, val, mode):
        self.P = P
        m = P.matricize(shape, np.asarray(idx).reshape(-1), val, mode)
        self.m = m
        counts = np.diff(m.col_ptr)
        cols = np.nonzero(counts > 0)[0].astype(np.int64)
        sel = np.concatenate([np.arange(m.col_ptr[c], m.col_ptr[c + 1]) for c in cols]) if cols.size else \
            np.zeros(0, np.int64)
        self.lf = LocalFibers(cols, np.concatenate([[0], np.cumsum(counts[cols])]).astype(np.int64),
                              m.row[sel].astype(np.int64), m.val[sel], P.column_sq_norms(m)[cols])
        self.col, self.norm = self.lf.col, self.lf.norm

    # the chained law (sampling.cpp:26-27,42-54): sequential sums resumed from
    # the running value of the earlier shards
    def seq_total(self, start):
        t = float(start)
        for v in self.norm:
            t += float(v)
        return t

    def cdf(self, total, start):
        self.probs = np.asarray(self.norm, dtype=np.float64) / total
        c = float(start)
        self.cum = np.zeros(self.probs.shape[0])
        for i, p in enumerate(self.probs):
            c += float(p)
            self.cum[i] = c
        self.lo, self.hi = float(start), c
        pos = np.nonzero(self.probs > 0)[0]
        self.last_pos = int(pos[-1]) if pos.size else -1
        return c, self.last_pos >= 0

    def clamp(self):
        self.cum[self.last_pos:] = 1.0
        self.hi = 1.0

    def draw(self, count, seed):
        raw = self.P.mt19937_64(seed, count)
        u = (raw >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)
        out = np.full(count, -1, np.int64)
        sel = (u >= self.lo) & (u < self.hi)
        out[sel] = self.col[np.searchsorted(self.cum, u[sel], side="right")]
        return out

    def gather(self, cols):
        lf = self.lf
        f = np.searchsorted(lf.col, cols)
        ptr = np.concatenate([[0], np.cumsum(lf.ptr[f + 1] - lf.ptr[f])]).astype(np.int64)
        rows = np.concatenate([lf.row[lf.ptr[a]:lf.ptr[a + 1]] for a in f]) if f.size else np.zeros(0, np.int64)
        vals = np.concatenate([lf.val[lf.ptr[a]:lf.ptr[a + 1]] for a in f]) if f.size else np.zeros(0)
        return ptr, rows, vals

    def error_partials(self, basis):
        lf = self.lf
        xs = float(np.sum(lf.val * lf.val))
        K = basis.size()
        if K == 0:
            return xs, 0.0
        cp, rr, rv = basis.r()
        Rd = np.zeros((basis.b.dim, K))
        for k in range(K):
            Rd[rr[cp[k]:cp[k + 1]], k] = rv[cp[k]:cp[k + 1]]
        U = basis.u()
        cross = 0.0
        for f in range(lf.col.shape[0]):
            g = Rd[lf.row[lf.ptr[f]:lf.ptr[f + 1]]].T @ lf.val[lf.ptr[f]:lf.ptr[f + 1]]
            cross += float(g @ (U @ g))
        return xs, cross

    def nnz_local(self):
        return int(self.m.nnz)

    def core(self, basis):
        # compute_core on this shard's columns (ctd_static.cpp:12-17) by the oracle
        from oracle.bindings import Csc
        cp, rr, rv = basis.r()
        R = Csc(self.m.rows, basis.size(), np.asarray(cp, np.int64), np.asarray(rr, np.int64), np.asarray(rv))
        c = self.P.core_matricized(self.m, R)
        counts = np.diff(c.col_ptr)
        cols = np.nonzero(counts > 0)[0].astype(np.int64)
        sel = np.concatenate([np.arange(c.col_ptr[j], c.col_ptr[j + 1]) for j in cols]) if cols.size else \
            np.zeros(0, np.int64)
        ptr = np.concatenate([[0], np.cumsum(counts[cols])]).astype(np.int64)
        return cols, ptr, np.asarray(c.row, np.int64)[sel], np.asarray(c.val)[sel]

    def close(self):
        pass


class _OracleBasis:
    def __init__(self, b):
        self.b = b
        self.cols = []

    def append_batch(self, ptr, rows, vals, eps):
        n = ptr.shape[0] - 1
        acc = np.zeros(n, np.int32)
        deg = np.zeros(n, np.int32)
        dl = np.zeros(n)
        for k in range(n):
            r, v = rows[ptr[k]:ptr[k + 1]], vals[ptr[k]:ptr[k + 1]]
            a, d, delta, _ = self.b.try_append(r, v, eps)
            acc[k], deg[k], dl[k] = a, d, delta
            if a:
                self.cols.append((r.copy(), v.copy()))
        return acc, deg, dl

    def size(self):
        return self.b.size()

    def u(self):
        return self.b.U()

    def r(self):
        cp = np.concatenate([[0], np.cumsum([c[0].shape[0] for c in self.cols])]).astype(np.int64)
        rows = np.concatenate([c[0] for c in self.cols]) if self.cols else np.zeros(0, np.int64)
        vals = np.concatenate([c[1] for c in self.cols]) if self.cols else np.zeros(0)
        return cp, rows, vals

    def close(self):
        pass


class _OracleCoreShard:
    """A rank's columns of the stream core (ctd_dynamic.cpp:188-222) restated
    in numpy in the reference's operation order: transpose_times merges
    (:53-85), chain_product (:231-269), compute_core for the slab columns."""

    def __init__(self, P, hist_shard, basis):
        self.P = P
        self.cols = {}  # global column id -> (rows, vals)
        self._add(hist_shard.core(basis), 0)

    def _add(self, core, offset):
        cols, ptr, rows, vals = core
        for q, j in enumerate(cols):
            self.cols[int(j) + offset] = (rows[ptr[q]:ptr[q + 1]].copy(), vals[ptr[q]:ptr[q + 1]].copy())

    def begin(self, basis):
        self.Kold = basis.size()
        self.Rold = basis.r()
        self.Uold = basis.u() if self.Kold else np.zeros((0, 0))

    def step(self, slab_shard, basis, col_offset):
        K, Kold = basis.size(), self.Kold
        cp, rr, rv = basis.r()
        A = K - Kold
        if A > 0 and Kold > 0:
            ocp, orr, orv = self.Rold
            gram = np.zeros((A, Kold))
            for a in range(A):
                ar, av = rr[cp[Kold + a]:cp[Kold + a + 1]], rv[cp[Kold + a]:cp[Kold + a + 1]]
                for j in range(Kold):
                    br, bv = orr[ocp[j]:ocp[j + 1]], orv[ocp[j]:ocp[j + 1]]
                    _, ia, ib = np.intersect1d(ar, br, assume_unique=True, return_indices=True)
                    acc = 0.0
                    for x, y in zip(av[ia], bv[ib]):  # ascending common rows, sequential
                        acc += float(x) * float(y)
                    if abs(acc) >= 1e-14:
                        gram[a, j] = acc
            left = np.zeros((A, Kold))
            for j in range(Kold):
                for i in np.nonzero(gram[:, j])[0]:
                    left[i, :] += gram[i, j] * self.Uold[j, :]
            for c, (crow, cval) in list(self.cols.items()):
                acc = np.zeros(A)
                for r, v in zip(crow, cval):
                    acc += left[:, r] * v
                keep = np.nonzero(np.abs(acc) >= 1e-14)[0]
                if keep.size:
                    self.cols[c] = (np.concatenate([crow, Kold + keep]), np.concatenate([cval, acc[keep]]))
        self._add(slab_shard.core(basis), int(col_offset))
        self.Kold = -1

    def columns(self):
        ids = np.array(sorted(self.cols), dtype=np.int64)
        ptr = np.concatenate([[0], np.cumsum([self.cols[int(j)][0].shape[0] for j in ids])]).astype(np.int64)
        rows = np.concatenate([self.cols[int(j)][0] for j in ids]) if ids.size else np.zeros(0, np.int64)
        vals = np.concatenate([self.cols[int(j)][1] for j in ids]) if ids.size else np.zeros(0)
        return ids, ptr, rows.astype(np.int64), vals

    def close(self):
        pass
