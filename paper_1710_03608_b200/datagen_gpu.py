"""Device-side form of ``datagen.traffic`` for inputs too large for the host
generator (BASELINE.json configs[4], C5: 1e5 x 1e5 x 1e3 with 1e9 coalesced nnz).

Same law and same definition as ``datagen.traffic``: counter-based splitmix64
uniforms (stream 1 src, 2 dst, 3 time, 4 count), Zipf(s) src/dst through the
seeded rank->id shuffle, uniform time, log-uniform integer counts, and the
tensor is the SHORTEST PREFIX of the draw sequence whose coalesced nnz reaches
the target, duplicates summed.  ``tests/test_datagen_gpu.py`` checks that both
generators produce identical bytes on shared sizes (torch CPU here, CUDA on
the box).

Output stays on the device in the layout ``ctd_gpu_tensor_from_device`` takes:
int32 coordinates per mode (SoA) and fp64 values, lexicographically sorted.
This is benchmark/test input generation, not part of the CTD path.
"""
from __future__ import annotations

import numpy as np
import torch

from . import datagen

_C_INC = 0x9E3779B97F4A7C15
_C_M1 = 0xBF58476D1CE4E5B9
_C_M2 = 0x94D049BB133111EB
_C_CTR = 0xD1B54A32D192ED03


def _s64(x: int) -> int:
    """uint64 constant as the int64 with the same bits."""
    x &= 0xFFFFFFFFFFFFFFFF
    return x - (1 << 64) if x >= (1 << 63) else x


def _srl(z: torch.Tensor, s: int) -> torch.Tensor:
    """logical right shift of int64 bits."""
    return (z >> s) & ((1 << (64 - s)) - 1)


def _splitmix64(x: torch.Tensor) -> torch.Tensor:
    z = x + _s64(_C_INC)
    z = (z ^ _srl(z, 30)) * _s64(_C_M1)
    z = (z ^ _srl(z, 27)) * _s64(_C_M2)
    return z ^ _srl(z, 31)


def uniform(seed: int, stream: int, start: int, count: int, device) -> torch.Tensor:
    """``datagen.uniform`` on the device (bit-identical)."""
    key = int(datagen._splitmix64(np.array([(seed * 0x100000001B3 + stream * 0x9E37)
                                            & 0xFFFFFFFFFFFFFFFF], dtype=np.uint64))[0])
    ctr = torch.arange(start, start + count, dtype=torch.int64, device=device)
    bits = _splitmix64(ctr * _s64(_C_CTR) + _s64(key))
    return _srl(bits, 11).to(torch.float64) * (1.0 / 9007199254740992.0)


def _zipf_tables(n: int, s: float, seed: int, stream: int, device):
    w = np.arange(1, n + 1, dtype=np.float64) ** (-s)
    cdf = np.cumsum(w)
    cdf /= cdf[-1]
    perm = np.argsort(datagen.uniform(seed, stream, 0, n), kind="stable")
    return (torch.from_numpy(cdf).to(device), torch.from_numpy(perm.astype(np.int64)).to(device))


def _draw_batch(shape, seed, start, n, tabs, max_count, log_counts, device):
    I, J, T = shape
    (cs, ps), (cd, pd) = tabs
    src = ps[torch.searchsorted(cs, uniform(seed, 1, start, n, device), right=True).clamp_(max=I - 1)]
    dst = pd[torch.searchsorted(cd, uniform(seed, 2, start, n, device), right=True).clamp_(max=J - 1)]
    tt = (uniform(seed, 3, start, n, device) * T).to(torch.int64)
    uc = uniform(seed, 4, start, n, device)
    if log_counts:
        cnt = torch.floor(torch.exp(uc * float(np.log(max_count + 1.0)))).clamp_(1, max_count)
    else:
        cnt = torch.floor(uc * max_count) + 1
    key = (src * J + dst) * T + tt
    return key, cnt.to(torch.uint8 if max_count < 256 else torch.int32)


def _partitions(key: torch.Tensor, parts: int):
    """Key-range boundaries splitting the draws into ~equal parts (from a strided sample)."""
    step = max(1, key.shape[0] // (parts * 4096))
    smp = torch.sort(key[::step]).values
    q = torch.linspace(0, smp.shape[0] - 1, parts + 1, device=key.device).round().to(torch.int64)
    b = smp[q[1:-1]].tolist()
    lo = [None] + b
    hi = b + [None]
    return list(zip(lo, hi))


def _select(key, lo, hi):
    if lo is None and hi is None:
        return torch.arange(key.shape[0], device=key.device)
    m = torch.ones_like(key, dtype=torch.bool)
    if lo is not None:
        m &= key >= lo
    if hi is not None:
        m &= key < hi
    return torch.nonzero(m).squeeze(1)


def _first_occurrences(key, parts):
    """Per key-range part: (sorted distinct keys, first draw index of each)."""
    out = []
    for lo, hi in parts:
        sel = _select(key, lo, hi)                    # ascending draw indices
        ks, perm = torch.sort(key[sel], stable=True)
        head = torch.ones_like(ks, dtype=torch.bool)
        head[1:] = ks[1:] != ks[:-1]
        out.append((ks[head], sel[perm[head]]))
        del sel, ks, perm, head
    return out


def traffic(shape, target_nnz: int, seed: int, max_count: int = 100, log_counts: bool = True,
            zipf_s: float = 1.2, device="cuda", batch: int = 1 << 26, parts: int = 16):
    """Returns (idx int32 [order, nnz] on device, val fp64 [nnz] on device, meta)."""
    I, J, T = (int(s) for s in shape)
    dev = torch.device(device)
    tabs = (_zipf_tables(I, zipf_s, seed, 100, dev), _zipf_tables(J, zipf_s, seed, 101, dev))
    keys, cnts = [], []
    drawn = 0
    want = int(target_nnz * 1.6) + batch
    while True:
        while drawn < want:
            n = min(batch, want - drawn)
            k, c = _draw_batch((I, J, T), seed, drawn, n, tabs, max_count, log_counts, dev)
            keys.append(k)
            cnts.append(c)
            drawn += n
        key = torch.cat(keys) if len(keys) > 1 else keys[0]
        keys = [key]
        cnt = torch.cat(cnts) if len(cnts) > 1 else cnts[0]
        cnts = [cnt]
        pts = _partitions(key, parts) if key.shape[0] > (1 << 24) else [(None, None)]
        fo = _first_occurrences(key, pts)
        total = sum(int(f[0].shape[0]) for f in fo)
        if total >= target_nnz:
            break
        want = int(drawn * max(1.2, 1.05 * target_nnz / max(total, 1)))
    # hi = shortest prefix of draws with target_nnz distinct keys
    firsts = torch.cat([f[1] for f in fo])
    hi = int(torch.sort(firsts).values[target_nnz - 1]) + 1
    del firsts
    # coalesce draws < hi per part (integer counts: the sum is exact in any order)
    nnz = sum(int((f[1] < hi).sum()) for f in fo)
    idx = torch.empty((3, nnz), dtype=torch.int32, device=dev)
    val = torch.empty(nnz, dtype=torch.float64, device=dev)
    pos = 0
    for (lo, hi_k), (uk, first) in zip(pts, fo):
        sel = _select(key, lo, hi_k)
        sel = sel[sel < hi]
        ks, perm = torch.sort(key[sel])
        gid = torch.searchsorted(uk, ks)
        live = uk[first < hi]
        sums = torch.zeros(uk.shape[0], dtype=torch.float64, device=dev)
        sums.index_add_(0, gid, cnt[sel[perm]].to(torch.float64))
        sums = sums[first < hi]
        m = live.shape[0]
        idx[0, pos:pos + m] = (live // (J * T)).to(torch.int32)
        idx[1, pos:pos + m] = ((live // T) % J).to(torch.int32)
        idx[2, pos:pos + m] = (live % T).to(torch.int32)
        val[pos:pos + m] = sums
        pos += m
        del sel, ks, perm, gid, sums
    assert pos == nnz
    return idx, val, {"seed": seed, "draws": hi, "zipf": zipf_s, "nnz": nnz}


def c5(seed: int = 5, device="cuda", scale: float = 1.0):
    """C5: 1e5 x 1e5 x 1e3 traffic, 1e9 coalesced nnz (``scale`` shrinks nnz and time)."""
    T = max(1, int(round(1000 * scale)))
    return traffic([100000, 100000, T], int(round(1e9 * scale)), seed, device=device)
