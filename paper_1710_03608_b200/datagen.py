"""Seeded synthetic inputs for BASELINE.json's configs C1-C5.

The paper's KONECT/CAIDA datasets are not available; these generators stand in
for them with the shapes, sizes and value laws BASELINE.json names.  Every
random number is a counter-based splitmix64 draw (``uniform(stream, i)``), so a
tensor is a pure function of (config, seed) — identical bytes for the GPU path,
the C restatement and the compiled reference, on any host and any numpy
version.  Tensors are returned exactly as the reference's ``SparseTensor``
stores them (sparse_tensor.cpp:62-102): entries sorted lexicographically,
duplicates summed, no stored zeros, int64 indices row-concatenated.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

_M64 = np.uint64(0xFFFFFFFFFFFFFFFF)


def _splitmix64(x: np.ndarray) -> np.ndarray:
    with np.errstate(over="ignore"):
        z = x + np.uint64(0x9E3779B97F4A7C15)
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
        return z ^ (z >> np.uint64(31))


def uniform(seed: int, stream: int, start: int, count: int) -> np.ndarray:
    """count uniforms in [0,1) from counters start..start+count of (seed, stream)."""
    key = _splitmix64(np.array([(seed * 0x100000001B3 + stream * 0x9E37) & 0xFFFFFFFFFFFFFFFF],
                               dtype=np.uint64))[0]
    ctr = np.arange(start, start + count, dtype=np.uint64)
    with np.errstate(over="ignore"):
        bits = _splitmix64(ctr * np.uint64(0xD1B54A32D192ED03) + key)
    return (bits >> np.uint64(11)).astype(np.float64) * (1.0 / 9007199254740992.0)


@dataclass
class Tensor:
    """Host COO in SparseTensor layout plus provenance."""
    shape: list
    idx: np.ndarray   # int64 [nnz, order], lexicographically sorted, unique
    val: np.ndarray   # float64 [nnz], no zeros
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.val.shape[0])

    @property
    def order(self) -> int:
        return len(self.shape)

    def flat_idx(self) -> np.ndarray:
        return np.ascontiguousarray(self.idx, dtype=np.int64).reshape(-1)

    def time_slab(self, t0: int, t1: int) -> "Tensor":
        """time_slab (stream_harness.cpp:26-46): entries with t0 <= t < t1."""
        tm = self.order - 1
        sel = (self.idx[:, tm] >= t0) & (self.idx[:, tm] < t1)
        idx = self.idx[sel].copy()
        idx[:, tm] -= t0
        shape = list(self.shape)
        shape[tm] = t1 - t0
        return Tensor(shape, idx, self.val[sel].copy(), {"slab": (t0, t1)})


def _sorted_runs(k: np.ndarray):
    """Distinct values of k (sorted) and the index of each one's first occurrence."""
    n = k.shape[0]
    sh = max(1, int(n - 1).bit_length())
    if k.shape[0] and int(k.max()) < (1 << (62 - sh)):
        s = np.sort((k << sh) | np.arange(n, dtype=np.int64))  # radix-friendly composite
        ks, ix = s >> sh, s & ((1 << sh) - 1)
    else:
        ix = np.argsort(k, kind="stable")
        ks = k[ix]
    head = np.ones(n, dtype=bool)
    head[1:] = ks[1:] != ks[:-1]
    return ks[head], ix[head]


def _coalesce_sorted(k: np.ndarray, v: np.ndarray):
    """(distinct sorted keys, values summed in input order)."""
    n = k.shape[0]
    if n == 0:
        return k, v
    sh = max(1, int(n - 1).bit_length())
    if int(k.max()) < (1 << (62 - sh)):
        s = np.sort((k << sh) | np.arange(n, dtype=np.int64))
        ks, ix = s >> sh, s & ((1 << sh) - 1)
    else:
        ix = np.argsort(k, kind="stable")
        ks = k[ix]
    head = np.ones(n, dtype=bool)
    head[1:] = ks[1:] != ks[:-1]
    starts = np.nonzero(head)[0]
    return ks[starts], np.add.reduceat(v[ix], starts)


def coalesce(shape, idx: np.ndarray, val: np.ndarray) -> Tensor:
    """Sort lexicographically, sum duplicates in input order, drop zeros."""
    shape = [int(s) for s in shape]
    key = np.zeros(idx.shape[0], dtype=np.int64)
    for k, s in enumerate(shape):
        key = key * s + idx[:, k].astype(np.int64)
    uk, summed = _coalesce_sorted(key, np.asarray(val, dtype=np.float64))
    keep = summed != 0.0
    uk, summed = uk[keep], summed[keep]
    out = np.zeros((uk.shape[0], len(shape)), dtype=np.int64)
    rem = uk.copy()
    for k in range(len(shape) - 1, -1, -1):
        out[:, k] = rem % shape[k]
        rem //= shape[k]
    return Tensor(shape, out, summed)


def _zipf_sampler(n: int, s: float, seed: int, stream: int):
    """Inverse-CDF Zipf(s) over n ids with a seeded rank->id shuffle
    (the role traffic.cpp:35-62 gives SkewedLaw)."""
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm = np.argsort(uniform(seed, stream, 0, n), kind="stable")

    def draw(u: np.ndarray) -> np.ndarray:
        r = np.searchsorted(cdf, u, side="right")
        return perm[np.minimum(r, n - 1)]
    return draw


def c1(seed: int = 1) -> Tensor:
    """C1: 200x200x50, 20,000 uniform coordinate draws, values Poisson(3)+1."""
    shape = [200, 200, 50]
    n = 20000
    u = [uniform(seed, s, 0, n) for s in range(4)]
    idx = np.stack([(u[k] * shape[k]).astype(np.int64) for k in range(3)], axis=1)
    # Poisson(3) by inverse CDF.
    lam = 3.0
    pk = np.exp(-lam) * np.cumprod(np.r_[1.0, lam / np.arange(1, 40)])
    cdf = np.cumsum(pk)
    pois = np.searchsorted(cdf, u[3], side="right")
    t = coalesce(shape, idx, (pois + 1).astype(np.float64))
    t.meta = {"config": "C1", "seed": seed, "draws": n}
    return t


def traffic(shape, target_nnz: int, seed: int, max_count: int = 100, log_counts=True,
            zipf_s: float = 1.2, batch: int = 1 << 22, t_offset: int = 0,
            t_total: int | None = None) -> Tensor:
    """Traffic tensor (src x dst x time): src/dst Zipf(s) with shuffled ids, time
    uniform, integer counts (log-uniform in [1,max] or uniform 1..max) as fp64.
    Draws continue until the coalesced nnz reaches target_nnz (H9b); the draw
    count is recorded in meta.  ``t_offset``/``t_total`` carve one rank's time
    range out of a larger stream (fiber-range sharding)."""
    I, J, T = (int(s) for s in shape)
    zs = _zipf_sampler(I, zipf_s, seed, 100)
    zd = _zipf_sampler(J, zipf_s, seed, 101)
    keys = []
    vals = []
    drawn = 0
    seen = np.zeros(0, dtype=np.int64)  # sorted distinct keys so far
    hi = None
    while hi is None:
        n = batch
        src = zs(uniform(seed, 1, drawn, n))
        dst = zd(uniform(seed, 2, drawn, n))
        tt = (uniform(seed, 3, drawn, n) * T).astype(np.int64)
        uc = uniform(seed, 4, drawn, n)
        if log_counts:
            cnt = np.clip(np.floor(np.exp(uc * np.log(max_count + 1.0))), 1, max_count)
        else:
            cnt = np.floor(uc * max_count) + 1
        k = (src.astype(np.int64) * J + dst) * T + tt
        # novelty of each draw: first occurrence in this batch and not seen before
        uk, first = _sorted_runs(k)
        pos = np.searchsorted(seen, uk)
        novel = (pos >= seen.shape[0]) | (seen[np.minimum(pos, max(seen.shape[0] - 1, 0))] != uk) \
            if seen.shape[0] else np.ones(uk.shape[0], dtype=bool)
        is_new = np.zeros(n, dtype=bool)
        is_new[first[novel]] = True
        run = seen.shape[0] + np.cumsum(is_new)
        keys.append(k)
        vals.append(cnt)
        if run[-1] >= target_nnz:
            # shortest prefix of all draws whose coalesced nnz reaches the target
            hi = drawn + int(np.argmax(run >= target_nnz)) + 1
        else:
            seen = np.sort(np.concatenate([seen, uk[novel]]))
        drawn += n
    k = np.concatenate(keys)[:hi]
    v = np.concatenate(vals)[:hi]
    uk, summed = _coalesce_sorted(k, v)
    idx = np.stack([uk // (J * T), (uk // T) % J, uk % T], axis=1)
    t = Tensor([I, J, T], idx.astype(np.int64), summed)
    t.meta = {"seed": seed, "draws": int(hi), "zipf": zipf_s}
    return t


def c2(seed: int = 2, scale: float = 1.0) -> Tensor:
    """C2: 10^4 x 10^4 x 10^3 traffic, 1e7 coalesced nnz (scale shrinks time/nnz)."""
    T = max(1, int(round(1000 * scale)))
    t = traffic([10000, 10000, T], int(round(1e7 * scale)), seed)
    t.meta["config"] = "C2" if scale == 1.0 else f"C2x{scale:g}"
    return t


def c4(seed: int = 4, scale_j: int = 1000, scale_k: int = 100, rank: int = 20,
       density: float = 0.1, sigma: float = 0.01) -> Tensor:
    """C4: 1000 x 1000 x 100 at 10 % density, planted rank-20 CP (U(0,1) factors)
    plus N(0, sigma^2) noise, non-integer fp64."""
    I, J, K = 1000, scale_j, scale_k
    A = uniform(seed, 10, 0, I * rank).reshape(I, rank)
    B = uniform(seed, 11, 0, J * rank).reshape(J, rank)
    Cm = uniform(seed, 12, 0, K * rank).reshape(K, rank)
    cells = I * J * K
    chunks = []
    step = 1 << 24
    for s0 in range(0, cells, step):
        n = min(step, cells - s0)
        sel = np.nonzero(uniform(seed, 13, s0, n) < density)[0] + s0
        chunks.append(sel)
    flat = np.concatenate(chunks).astype(np.int64)
    i, rem = flat // (J * K), flat % (J * K)
    j, k = rem // K, rem % K
    val = np.einsum("nr,nr,nr->n", A[i], B[j], Cm[k])
    u1 = uniform(seed, 14, 0, flat.shape[0])
    u2 = uniform(seed, 15, 0, flat.shape[0])
    gauss = np.sqrt(-2.0 * np.log1p(-u1)) * np.cos(2 * np.pi * u2)
    val = val + sigma * gauss
    t = Tensor([I, J, K], np.stack([i, j, k], axis=1), val)
    t.meta = {"config": "C4" if (J, K) == (1000, 100) else f"C4[{I}x{J}x{K}]", "seed": seed}
    return t


def c3_stream(seed: int = 3, n_steps: int = 100, slices_per_step: int = 10,
              draws_per_slice: int = 20000, n: int = 5000, planted_step: int = 60,
              block: int = 50, bump: float = 100.0) -> Tensor:
    """C3: 5000 x 5000 x (steps*slices) stream; per slice ~2e4 Zipf(1.2) draws with
    counts U{1..50}; at ``planted_step`` every cell of a 50x50 src x dst block gets
    +100 in all the step's slices (H9c: added)."""
    T = n_steps * slices_per_step
    zs = _zipf_sampler(n, 1.2, seed, 100)
    zd = _zipf_sampler(n, 1.2, seed, 101)
    total = T * draws_per_slice
    src = zs(uniform(seed, 1, 0, total))
    dst = zd(uniform(seed, 2, 0, total))
    tt = np.repeat(np.arange(T, dtype=np.int64), draws_per_slice)
    cnt = np.floor(uniform(seed, 4, 0, total) * 50) + 1
    idx = [np.stack([src, dst, tt], axis=1)]
    val = [cnt]
    if 0 <= planted_step < n_steps:
        b0 = int(uniform(seed, 20, 0, 1)[0] * (n - block))
        bs, bd = np.meshgrid(np.arange(b0, b0 + block), np.arange(b0, b0 + block), indexing="ij")
        for s in range(slices_per_step):
            t = planted_step * slices_per_step + s
            idx.append(np.stack([bs.ravel(), bd.ravel(), np.full(block * block, t)], axis=1))
            val.append(np.full(block * block, bump))
    out = coalesce([n, n, T], np.concatenate(idx).astype(np.int64), np.concatenate(val))
    out.meta = {"config": "C3", "seed": seed, "steps": n_steps, "slices_per_step": slices_per_step}
    return out


def random_sparse(shape, density: float, seed: int, integer: bool = False) -> Tensor:
    """Small seeded random tensor (tests): Bernoulli(density) cells, values in
    +-[0.1, 1] (the reference test generator's law, oracles.cpp:19-22) or small ints."""
    cells = int(np.prod(shape))
    sel = np.nonzero(uniform(seed, 30, 0, cells) < density)[0]
    idx = np.stack(np.unravel_index(sel, shape), axis=1).astype(np.int64)
    u = uniform(seed, 31, 0, sel.shape[0])
    if integer:
        val = np.floor(u * 9) + 1
    else:
        s = np.where(uniform(seed, 32, 0, sel.shape[0]) < 0.5, -1.0, 1.0)
        val = s * (0.1 + 0.9 * u)
    return Tensor(list(shape), idx, val)


def low_rank(shape, rank: int, density: float, seed: int, mode: int = 0) -> Tensor:
    """Exactly low-rank along `mode` (every mode-`mode` fiber is a combination of
    `rank` fixed vectors) with small integer values, masked at fiber granularity
    so the rank survives sparsification (the idea of oracles.cpp:193-238)."""
    I = shape[mode]
    others = [s for k, s in enumerate(shape) if k != mode]
    ncols = int(np.prod(others))
    basis = np.floor(uniform(seed, 40, 0, I * rank) * 5).reshape(I, rank) - 2
    coef = np.floor(uniform(seed, 41, 0, ncols * rank) * 5).reshape(ncols, rank) - 2
    keep = uniform(seed, 42, 0, ncols) < density
    dense = (basis @ coef.T)  # I x ncols
    dense[:, ~keep] = 0.0
    r, c = np.nonzero(dense)
    # column c decodes over the other modes in increasing mode order (stride 1 first)
    coords = []
    rem = c.copy()
    for s in others:
        coords.append(rem % s)
        rem //= s
    full = []
    oi = 0
    for k in range(len(shape)):
        if k == mode:
            full.append(r)
        else:
            full.append(coords[oi])
            oi += 1
    idx = np.stack(full, axis=1).astype(np.int64)
    return coalesce(shape, idx, dense[r, c])
