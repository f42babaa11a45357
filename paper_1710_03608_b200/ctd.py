"""Python mirror of the reference ``ctd::`` hot-path API, backed by the B200
CUDA library through its C-ABI (include/ctd_gpu.h).

Names, argument meaning and error behaviour follow proj/core/include/ctd:
``ctd_s`` (ctd_static.hpp:22-24), ``init_stream`` / ``ctd_d_step``
(ctd_dynamic.hpp:42-58), ``column_distribution`` / ``sample_with_replacement``
/ ``unique_first_occurrence`` (sampling.hpp:20-31), ``matricize`` /
``column_sq_norms`` (tensor_ops.hpp:21,39), ``FiberBasis`` (fiber_basis.hpp),
``relative_error`` (evaluation.hpp:39).  Errors raise the reference's error
classes (error.hpp:11-73) with the same ``error_class`` values.
"""
from __future__ import annotations

import ctypes as C
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib

# ---------------------------------------------------------------------------
# Error taxonomy (error.hpp:11-73) + device failures.


class CtdError(RuntimeError):
    error_class = 0


class ArgumentError(CtdError):
    error_class = 1


class ShapeError(CtdError):
    error_class = 2


class EmptyInputError(CtdError):
    error_class = 3


class MetricError(CtdError):
    error_class = 5


class DeviceError(CtdError):
    error_class = 8


class NumericError(CtdError):
    error_class = 9


_ERRORS = {1: ArgumentError, 2: ShapeError, 3: EmptyInputError, 5: MetricError,
           8: DeviceError, 9: NumericError}

WITH_ERROR = 0x1
WITH_CORE = 0x2
KEEP_PANEL = 0x4  # keep the orthonormal panel for a later relative_error (implied by WITH_ERROR)
KEEP_HISTORY = 0x8  # init_stream(keep_history=True): retain the raw history (core_drift)
EXACT_CORE = 0x10   # init_stream(exact_core=True): bottom-left block from the history
LAZY_CORE = 0x20    # init_stream(lazy_core=True): core updates recorded per step, applied on read


def _check(st: int):
    if st:
        msg = _lib.load().ctd_gpu_last_error().decode()
        raise _ERRORS.get(st, CtdError)(msg)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


# ---------------------------------------------------------------------------
# Context: device + stream + launch counter.

class Context:
    """Device context.  ``stream`` is a cudaStream_t integer (torch's
    ``torch.cuda.current_stream().cuda_stream``) or None for the default."""

    def __init__(self, device: int = 0, stream: Optional[int] = None):
        self.L = _lib.load()
        h = C.c_void_p()
        _check(self.L.ctd_gpu_ctx_create(device, C.c_void_p(stream or 0), C.byref(h)))
        self.h = h

    def set_stream(self, stream: Optional[int]):
        _check(self.L.ctd_gpu_ctx_set_stream(self.h, C.c_void_p(stream or 0)))

    def synchronize(self):
        _check(self.L.ctd_gpu_ctx_synchronize(self.h))

    @property
    def launches(self) -> int:
        return int(self.L.ctd_gpu_ctx_launches(self.h))

    def set_timing(self, enable: bool):
        _check(self.L.ctd_gpu_ctx_set_timing(self.h, int(enable)))

    def phase_times(self, reset: bool = True) -> dict:
        """{phase: (total_ms, count)} from CUDA events on the context stream."""
        ms = np.zeros(8)
        n = np.zeros(8, dtype=np.int64)
        _check(self.L.ctd_gpu_ctx_phase_times(self.h, _p(ms), _p(n), int(reset)))
        return {self.L.ctd_gpu_phase_name(i).decode(): (float(ms[i]), int(n[i])) for i in range(8)}

    def trim(self):
        """Returns cached device memory to the driver (torch.cuda.empty_cache's
        counterpart for this context)."""
        _check(self.L.ctd_gpu_ctx_trim(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.L.ctd_gpu_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


_default_ctx: Optional[Context] = None


def default_context() -> Context:
    global _default_ctx
    if _default_ctx is None:
        stream = None
        try:
            import torch
            if torch.cuda.is_available():
                stream = torch.cuda.current_stream().cuda_stream
        except Exception:
            stream = None
        _default_ctx = Context(0, stream)
    return _default_ctx


# ---------------------------------------------------------------------------
# SparseTensor (sparse_tensor.hpp:17-60): host COO, normalized.

@dataclass
class SparseTensor:
    shape: list
    indices: np.ndarray          # int64 [nnz, order] (row-concatenated like the reference)
    values: np.ndarray           # float64 [nnz]

    @property
    def order(self) -> int:
        return len(self.shape)

    @property
    def nnz(self) -> int:
        return int(self.values.shape[0])

    @classmethod
    def from_datagen(cls, t) -> "SparseTensor":
        return cls(list(t.shape), np.ascontiguousarray(t.idx, dtype=np.int64),
                   np.ascontiguousarray(t.val, dtype=np.float64))


class DeviceTensor:
    """A SparseTensor resident in HBM (ctd_gpu_tensor)."""

    def __init__(self, x: SparseTensor, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.shape = [int(s) for s in x.shape]
        shape = np.asarray(self.shape, dtype=np.int64)
        idx = np.ascontiguousarray(x.indices, dtype=np.int64).reshape(-1)
        val = np.ascontiguousarray(x.values, dtype=np.float64)
        h = C.c_void_p()
        _check(self.ctx.L.ctd_gpu_tensor_from_host(self.ctx.h, len(shape), _p(shape), x.nnz,
                                                   _p(idx), _p(val), C.byref(h)))
        self.h = h
        self.nnz = x.nnz
        self.order = len(shape)

    @classmethod
    def from_host_ptrs(cls, shape, nnz: int, idx_ptr: int, val_ptr: int,
                       ctx: Optional[Context] = None) -> "DeviceTensor":
        """Copy a host SparseTensor given raw (e.g. pinned) pointers: int64
        row-concatenated coordinates and fp64 values."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.shape = [int(s) for s in shape]
        shp = np.asarray(self.shape, dtype=np.int64)
        h = C.c_void_p()
        _check(self.ctx.L.ctd_gpu_tensor_from_host(self.ctx.h, len(shp), _p(shp), nnz,
                                                   C.c_void_p(int(idx_ptr)),
                                                   C.c_void_p(int(val_ptr)), C.byref(h)))
        self.h = h
        self.nnz = nnz
        self.order = len(shp)
        return self

    @classmethod
    def from_device_ptrs(cls, shape, nnz: int, mode_ptrs, val_ptr: int,
                         ctx: Optional[Context] = None) -> "DeviceTensor":
        """Borrow device SoA int32 coordinate arrays + fp64 values (e.g. torch tensors'
        data_ptr()); the caller keeps them alive."""
        self = cls.__new__(cls)
        self.ctx = ctx or default_context()
        self.shape = [int(s) for s in shape]
        shp = np.asarray(self.shape, dtype=np.int64)
        ptrs = (C.c_void_p * len(shape))(*[C.c_void_p(int(p)) for p in mode_ptrs])
        h = C.c_void_p()
        _check(self.ctx.L.ctd_gpu_tensor_from_device(self.ctx.h, len(shape), _p(shp), nnz,
                                                     C.cast(ptrs, C.c_void_p),
                                                     C.c_void_p(int(val_ptr)), C.byref(h)))
        self.h = h
        self.nnz = nnz
        self.order = len(shape)
        return self

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.ctd_gpu_tensor_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def _dev(x, ctx) -> DeviceTensor:
    if isinstance(x, DeviceTensor):
        return x
    return DeviceTensor(x, ctx)


# ---------------------------------------------------------------------------
# tensor_ops / sampling pieces

@dataclass
class Matricized:
    """Compressed CSC of X_(mode): only the F nonempty fibers."""
    rows: int
    cols: int
    fiber_col: np.ndarray
    fiber_ptr: np.ndarray
    row: np.ndarray
    val: np.ndarray
    sq_norms: np.ndarray

    def dense_col_ptr(self) -> np.ndarray:
        """col_ptr over all N_alpha columns (the reference's layout)."""
        counts = np.zeros(self.cols, dtype=np.int64)
        counts[self.fiber_col] = np.diff(self.fiber_ptr)
        return np.concatenate([[0], np.cumsum(counts)])

    def dense_norms(self) -> np.ndarray:
        out = np.zeros(self.cols)
        out[self.fiber_col] = self.sq_norms
        return out


def matricize(x, mode: int, ctx: Optional[Context] = None) -> Matricized:
    """matricize + column_sq_norms (tensor_ops.cpp:118-135, 194-202)."""
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    nnz = d.nnz
    F = C.c_int64()
    col = np.zeros(max(nnz, 1), dtype=np.int64)
    ptr = np.zeros(nnz + 1, dtype=np.int64)
    row = np.zeros(max(nnz, 1), dtype=np.int32)
    val = np.zeros(max(nnz, 1))
    nrm = np.zeros(max(nnz, 1))
    _check(ctx.L.ctd_gpu_matricize(ctx.h, d.h, mode, C.byref(F), _p(col), _p(ptr), _p(row),
                                   _p(val), _p(nrm)))
    f = F.value
    cols = int(np.prod([s for k, s in enumerate(d.shape) if k != mode], dtype=np.int64))
    return Matricized(d.shape[mode], cols, col[:f].copy(), ptr[:f + 1].copy(), row[:nnz].copy(),
                      val[:nnz].copy(), nrm[:f].copy())


def column_sq_norms(x, mode: int, ctx: Optional[Context] = None) -> np.ndarray:
    """Dense per-column squared norms, length N_alpha (tensor_ops.hpp:39)."""
    return matricize(x, mode, ctx).dense_norms()


@dataclass
class ColumnDistribution:
    """column_distribution over the nonempty fibers (every other column has
    probability exactly 0); ``cumulative`` is sample_with_replacement's
    clamped array restricted to the same fibers."""
    fiber_col: np.ndarray
    probabilities: np.ndarray
    cumulative: np.ndarray
    total_sq_norm: float
    cols: int

    def dense(self) -> np.ndarray:
        out = np.zeros(self.cols)
        out[self.fiber_col] = self.probabilities
        return out


def column_distribution(x, mode: int, ctx: Optional[Context] = None) -> ColumnDistribution:
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    m = matricize(d, mode, ctx)
    F = len(m.fiber_col)
    tot = C.c_double()
    p = np.zeros(max(F, 1))
    cum = np.zeros(max(F, 1))
    _check(ctx.L.ctd_gpu_column_distribution(ctx.h, d.h, mode, C.byref(tot), _p(p), _p(cum)))
    return ColumnDistribution(m.fiber_col, p[:F].copy(), cum[:F].copy(), tot.value, m.cols)


def sample_with_replacement(probabilities, count: int, seed: int,
                            ctx: Optional[Context] = None) -> np.ndarray:
    """sample_with_replacement (sampling.hpp:27-28) over a dense probability vector."""
    ctx = ctx or default_context()
    p = np.ascontiguousarray(probabilities, dtype=np.float64)
    out = np.zeros(max(count, 1), dtype=np.int64)
    _check(ctx.L.ctd_gpu_sample_with_replacement(ctx.h, _p(p), len(p), count, C.c_uint64(seed),
                                                 _p(out)))
    return out[:max(count, 0)].copy()


def seq_cumsum(x, ctx: Optional[Context] = None) -> np.ndarray:
    """Bit-exact sequential running sum of non-negative doubles on the GPU."""
    ctx = ctx or default_context()
    a = np.ascontiguousarray(x, dtype=np.float64)
    out = np.zeros(max(len(a), 1))
    _check(ctx.L.ctd_gpu_seq_cumsum(ctx.h, _p(a), len(a), _p(out)))
    return out[:len(a)].copy()


def unique_first_occurrence(drawn, ctx: Optional[Context] = None) -> np.ndarray:
    ctx = ctx or default_context()
    d = np.ascontiguousarray(drawn, dtype=np.int64)
    out = np.zeros(max(len(d), 1), dtype=np.int64)
    n = C.c_int64()
    _check(ctx.L.ctd_gpu_unique_first_occurrence(ctx.h, _p(d), len(d), _p(out), C.byref(n)))
    return out[:n.value].copy()


# ---------------------------------------------------------------------------
# FiberBasis (fiber_basis.hpp:21-61)

@dataclass
class AppendResult:
    accepted: bool
    degenerate: bool
    delta: float
    y: np.ndarray


class FiberBasis:
    def __init__(self, dim: int, ctx: Optional[Context] = None):
        self.ctx = ctx or default_context()
        self.dim = dim
        h = C.c_void_p()
        _check(self.ctx.L.ctd_gpu_basis_create(self.ctx.h, dim, C.byref(h)))
        self.h = h

    def size(self) -> int:
        return int(self.ctx.L.ctd_gpu_basis_size(self.h))

    def inverse_gram(self) -> np.ndarray:
        k = self.size()
        u = np.zeros(max(k * k, 1))
        _check(self.ctx.L.ctd_gpu_basis_u(self.h, _p(u)))
        return u[:k * k].reshape(k, k)

    def try_append_fiber(self, idx, val, epsilon: float, dim: Optional[int] = None) -> AppendResult:
        idx = np.ascontiguousarray(idx, dtype=np.int64)
        val = np.ascontiguousarray(val, dtype=np.float64)
        k = self.size()
        y = np.zeros(max(k, 1))
        a, dg, dl = C.c_int32(), C.c_int32(), C.c_double()
        _check(self.ctx.L.ctd_gpu_basis_try_append(self.h, self.dim if dim is None else dim,
                                                   len(val), _p(idx), _p(val), epsilon,
                                                   C.byref(a), C.byref(dg), C.byref(dl), _p(y)))
        return AppendResult(bool(a.value), bool(dg.value), dl.value, y[:k].copy())

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.ctd_gpu_basis_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


# ---------------------------------------------------------------------------
# LRFactors (factors.hpp:32-47)

@dataclass
class FiberId:
    flat: int
    coords: tuple


def make_fiber_id(shape, mode: int, flat: int) -> FiberId:
    """make_fiber_id (factors.cpp:8-29)."""
    others = [s for k, s in enumerate(shape) if k != mode]
    total = int(np.prod(others, dtype=np.int64)) if others else 1
    if flat < 0 or flat >= total:
        raise ArgumentError("fiber index out of range")
    coords = []
    rem = flat
    for s in others:
        coords.append(rem % s)
        rem //= s
    return FiberId(int(flat), tuple(int(c) for c in coords))


@dataclass
class LRFactors:
    mode: int
    shape: list
    epsilon: float
    seed: int
    kept_flat: np.ndarray
    U: np.ndarray
    R_col_ptr: np.ndarray
    R_row: np.ndarray
    R_val: np.ndarray
    drawn: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    unique: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int64))
    accepted: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    degenerate: np.ndarray = field(default_factory=lambda: np.zeros(0, np.int32))
    delta: np.ndarray = field(default_factory=lambda: np.zeros(0))
    total_sq_norm: float = 0.0
    relative_error: float = float("nan")
    min_margin: float = float("inf")
    info: Optional[_lib.FactorsInfo] = None
    handle: object = None
    # C_(mode) = R^T X_(mode) (compute_core) when requested: CSC over the columns
    # that keep an entry (C_col: their column ids), rows = kept-fiber index
    C_col: Optional[np.ndarray] = None
    C_ptr: Optional[np.ndarray] = None
    C_row: Optional[np.ndarray] = None
    C_val: Optional[np.ndarray] = None

    @property
    def kept_fibers(self):
        return [make_fiber_id(self.shape, self.mode, int(f)) for f in self.kept_flat]

    def kept_count(self) -> int:
        return int(len(self.kept_flat))


class _FactorsHandle:
    def __init__(self, ctx, h):
        self.ctx, self.h = ctx, h

    def __del__(self):
        try:
            self.ctx.L.ctd_gpu_factors_destroy(self.h)
        except Exception:
            pass


def _read_factors(ctx: Context, h, shape, mode, trace=True) -> LRFactors:
    L = ctx.L
    info = _lib.FactorsInfo()
    _check(L.ctd_gpu_factors_info_get(h, C.byref(info)))
    k = info.kept
    kept = np.zeros(max(k, 1), dtype=np.int64)
    _check(L.ctd_gpu_factors_kept_flat(h, _p(kept)))
    u = np.zeros(max(k * k, 1))
    _check(L.ctd_gpu_factors_u(h, _p(u)))
    cp = np.zeros(k + 1, dtype=np.int64)
    rr = np.zeros(max(info.r_nnz, 1), dtype=np.int64)
    rv = np.zeros(max(info.r_nnz, 1))
    _check(L.ctd_gpu_factors_r(h, _p(cp), _p(rr), _p(rv)))
    f = LRFactors(mode, list(shape), info.epsilon, info.seed, kept[:k].copy(),
                  u[:k * k].reshape(k, k), cp, rr[:info.r_nnz].copy(), rv[:info.r_nnz].copy(),
                  total_sq_norm=info.total_sq_norm, relative_error=info.relative_error,
                  min_margin=info.min_margin, info=info, handle=_FactorsHandle(ctx, h))
    if info.c_nnz or (with_core_flag(h, ctx)):
        cc = C.c_int64()
        _check(L.ctd_gpu_factors_core(h, C.byref(cc), None, None, None, None))
        nc, nz = cc.value, info.c_nnz
        f.C_col = np.zeros(max(nc, 1), np.int64)
        f.C_ptr = np.zeros(nc + 1, np.int64)
        f.C_row = np.zeros(max(nz, 1), np.int64)
        f.C_val = np.zeros(max(nz, 1))
        _check(L.ctd_gpu_factors_core(h, C.byref(cc), _p(f.C_col), _p(f.C_ptr), _p(f.C_row), _p(f.C_val)))
        f.C_col, f.C_row, f.C_val = f.C_col[:nc], f.C_row[:nz], f.C_val[:nz]
    if trace and info.n_drawn:
        nd, nu = info.n_drawn, info.n_unique
        f.drawn = np.zeros(nd, np.int64)
        f.unique = np.zeros(max(nu, 1), np.int64)
        f.accepted = np.zeros(max(nu, 1), np.int32)
        f.degenerate = np.zeros(max(nu, 1), np.int32)
        f.delta = np.zeros(max(nu, 1))
        _check(L.ctd_gpu_factors_trace(h, _p(f.drawn), _p(f.unique), _p(f.accepted),
                                       _p(f.degenerate), _p(f.delta)))
        f.unique, f.accepted, f.degenerate, f.delta = (f.unique[:nu], f.accepted[:nu],
                                                       f.degenerate[:nu], f.delta[:nu])
    return f


def with_core_flag(h, ctx) -> bool:
    """Whether the factors carry C (a zero-entry core still has columns info)."""
    cc = C.c_int64()
    return ctx.L.ctd_gpu_factors_core(h, C.byref(cc), None, None, None, None) == 0


def ctd_s(x, mode: int, sample_size: int, epsilon: float = 1e-6, seed: int = 42,
          with_error: bool = False, with_core: bool = False, ctx: Optional[Context] = None) -> LRFactors:
    """Algorithm 1 (ctd_static.hpp:22-24).  ``with_core`` materializes
    C = X x_mode R^T (compute_core, ctd_static.cpp:12-17) as its matricization;
    ``with_error`` runs the relative-error pass (evaluation.cpp:88-122)."""
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    h = C.c_void_p()
    flags = (WITH_ERROR if with_error else 0) | (WITH_CORE if with_core else 0)
    _check(ctx.L.ctd_gpu_ctd_s(ctx.h, d.h, mode, sample_size, epsilon, C.c_uint64(seed), flags,
                               C.byref(h)))
    return _read_factors(ctx, h, d.shape, mode)


@dataclass
class Csc:
    """A compressed sparse matrix: only the columns that keep an entry (col_id)."""
    rows: int
    col_id: np.ndarray
    col_ptr: np.ndarray
    row: np.ndarray
    val: np.ndarray


def _read_csc(ctx: Context, h) -> Csc:
    try:
        r, nc, nz = C.c_int64(), C.c_int64(), C.c_int64()
        _check(ctx.L.ctd_gpu_csc_info(h, C.byref(r), C.byref(nc), C.byref(nz)))
        col = np.zeros(max(nc.value, 1), np.int64)
        ptr = np.zeros(nc.value + 1, np.int64)
        row = np.zeros(max(nz.value, 1), np.int64)
        val = np.zeros(max(nz.value, 1))
        _check(ctx.L.ctd_gpu_csc_copy(h, _p(col), _p(ptr), _p(row), _p(val)))
        return Csc(r.value, col[:nc.value], ptr, row[:nz.value], val[:nz.value])
    finally:
        ctx.L.ctd_gpu_csc_destroy(h)


def compute_core(x, r_col_ptr, r_row, r_val, r_cols: int, mode: int, ctx: Optional[Context] = None) -> Csc:
    """compute_core (ctd_static.hpp:28): C_(mode) = R^T X_(mode) for a given R
    (CSC over x's extent in `mode`), on the device."""
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    cp = np.ascontiguousarray(r_col_ptr, np.int64)
    rr = np.ascontiguousarray(r_row, np.int64)
    rv = np.ascontiguousarray(r_val, np.float64)
    h = C.c_void_p()
    _check(ctx.L.ctd_gpu_compute_core(ctx.h, d.h, mode, int(d.shape[mode]), int(r_cols), _p(cp), _p(rr), _p(rv),
                                      C.byref(h)))
    return _read_csc(ctx, h)


def chain_product(dim: int, dr, r, u, c, c_cols: int, ctx: Optional[Context] = None) -> Csc:
    """chain_product (ctd_dynamic.hpp:61-62): ((dR^T R) U) C on the device.
    dr, r, c: (col_ptr, rows, vals) CSC triples (dr, r over `dim` rows; c with
    one row per column of r), u: k x k."""
    ctx = ctx or default_context()
    a = [np.ascontiguousarray(v) for v in dr]
    b = [np.ascontiguousarray(v) for v in r]
    cc = [np.ascontiguousarray(v) for v in c]
    a[0], a[1], b[0], b[1], cc[0], cc[1] = (np.asarray(v, np.int64) for v in (a[0], a[1], b[0], b[1], cc[0], cc[1]))
    uu = np.ascontiguousarray(u, np.float64)
    k = b[0].shape[0] - 1
    h = C.c_void_p()
    _check(ctx.L.ctd_gpu_chain_product(ctx.h, int(dim), a[0].shape[0] - 1, _p(a[0]), _p(a[1]), _p(a[2]), k, _p(b[0]),
                                       _p(b[1]), _p(b[2]), _p(uu), int(c_cols), _p(cc[0]), _p(cc[1]), _p(cc[2]),
                                       C.byref(h)))
    return _read_csc(ctx, h)


def memory_usage(x, f: LRFactors, ctx: Optional[Context] = None) -> float:
    """memory_usage (evaluation.cpp:124-129): (nnz(C) + nnz(U) + nnz(R)) / nnz(X);
    the factors must carry C (``ctd_s(..., with_core=True)``)."""
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    out = C.c_double()
    _check(ctx.L.ctd_gpu_memory_usage(d.h, f.handle.h, C.byref(out)))
    return out.value


def ctd_s_raw(x, mode: int, sample_size: int, epsilon: float = 1e-6, seed: int = 42,
              with_error: bool = False, ctx: Optional[Context] = None, keep_panel: bool = False,
              with_core: bool = False):
    """ctd_s without copying R/U to the host: returns (handle, FactorsInfo).
    Free the handle with ``free_factors``.  keep_panel: maintain the
    orthonormal panel so a later ``relative_error_raw`` takes one pass."""
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    h = C.c_void_p()
    flags = (WITH_ERROR if with_error else 0) | (KEEP_PANEL if keep_panel else 0) | (WITH_CORE if with_core else 0)
    _check(ctx.L.ctd_gpu_ctd_s(ctx.h, d.h, mode, sample_size, epsilon, C.c_uint64(seed), flags, C.byref(h)))
    info = _lib.FactorsInfo()
    _check(ctx.L.ctd_gpu_factors_info_get(h, C.byref(info)))
    return h, info


def relative_error_raw(x, h, ctx: Optional[Context] = None) -> float:
    """relative_error(X, factors) for a raw factors handle from ctd_s_raw."""
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    out = C.c_double()
    _check(ctx.L.ctd_gpu_relative_error(ctx.h, d.h, h, C.byref(out)))
    return out.value


def free_factors(ctx: Context, h) -> None:
    _check(ctx.L.ctd_gpu_factors_destroy(h))


def factors_trace(ctx: Context, h, info) -> dict:
    """Per-candidate decisions and R's column lengths (for byte accounting)."""
    nu, k = info.n_unique, info.kept
    acc = np.zeros(max(nu, 1), np.int32)
    _check(ctx.L.ctd_gpu_factors_trace(h, None, None, _p(acc), None, None))
    cp = np.zeros(k + 1, np.int64)
    _check(ctx.L.ctd_gpu_factors_r(h, _p(cp), None, None))
    rows = np.zeros(max(int(cp[-1]), 1), np.int64)
    vals = np.zeros(max(int(cp[-1]), 1))
    _check(ctx.L.ctd_gpu_factors_r(h, _p(cp), _p(rows), _p(vals)))
    return {"accepted": acc[:nu].astype(bool), "r_lens": np.diff(cp), "r_ptr": cp,
            "r_rows": rows[:int(cp[-1])]}


def factors_result(ctx: Context, h, info, u_out=None):
    """The decomposition's result on the host: kept fiber ids and U.  `u_out`: a
    caller-owned float64 array of at least kept^2 elements to receive U (e.g. a
    view of pinned memory, which the copy then reaches directly)."""
    k = info.kept
    kept = np.zeros(max(k, 1), dtype=np.int64)
    _check(ctx.L.ctd_gpu_factors_kept_flat(h, _p(kept)))
    if u_out is None:
        u = np.empty(max(k * k, 1))
    else:
        u = u_out
        if u.dtype != np.float64 or not u.flags.c_contiguous or u.size < max(k * k, 1):
            raise ValueError("u_out must be a contiguous float64 array of at least kept^2 elements")
        u = u.reshape(-1)
    _check(ctx.L.ctd_gpu_factors_u(h, _p(u)))
    return kept[:k], u[:k * k].reshape(k, k)


def relative_error(x, factors: LRFactors, ctx: Optional[Context] = None) -> float:
    ctx = ctx or default_context()
    d = _dev(x, ctx)
    out = C.c_double()
    _check(ctx.L.ctd_gpu_relative_error(ctx.h, d.h, factors.handle.h, C.byref(out)))
    return out.value


# ---------------------------------------------------------------------------
# CTD-D (ctd_dynamic.hpp:18-66)

class StreamState:
    def __init__(self, ctx: Context, h, mode: int, slab_shape):
        self.ctx, self.h, self.mode = ctx, h, mode
        self.slab_shape = list(slab_shape)

    @property
    def t(self) -> int:
        return int(self.ctx.L.ctd_gpu_stream_t(self.h))

    def factors(self) -> LRFactors:
        h = C.c_void_p()
        _check(self.ctx.L.ctd_gpu_stream_factors(self.h, C.byref(h)))
        return _read_factors(self.ctx, h, self.slab_shape + [self.t], self.mode, trace=False)

    def n_kept(self) -> int:
        return int(self.ctx.L.ctd_gpu_stream_n_kept(self.h))

    def core_pending(self):
        """(records, slab-column entries, bytes) of the lazily kept core updates
        (lazy_core)."""
        r, e, b = C.c_int64(), C.c_int64(), C.c_int64()
        _check(self.ctx.L.ctd_gpu_stream_core_pending(self.h, C.byref(r), C.byref(e), C.byref(b)))
        return r.value, e.value, b.value

    def core_sync(self):
        """Applies the lazily kept core updates (factors() and core_drift do this)."""
        _check(self.ctx.L.ctd_gpu_stream_core_sync(self.h))

    def close(self):
        if getattr(self, "h", None):
            self.ctx.L.ctd_gpu_stream_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass


def init_stream(historical, mode: int, sample_size: int, epsilon: float = 1e-6,
                seed: int = 42, keep_history: bool = False, exact_core: bool = False,
                with_core: bool = False, lazy_core: bool = False,
                ctx: Optional[Context] = None) -> StreamState:
    """init_stream (ctd_dynamic.hpp:42-45, ctd_dynamic.cpp:129-147).  ``with_core``
    maintains the core C(t) through every step (Eq. 13 blocks); ``factors()`` then
    carries it.  ``keep_history`` retains the raw history on the device (for
    ``core_drift``); ``exact_core`` computes the bottom-left block from it
    (ctd_dynamic.cpp:207-211).  Either implies ``with_core``.  ``lazy_core``
    maintains the same core as per-step records (the slab's columns and the
    chain product's left factor) applied when the core is read; it implies
    ``with_core`` and is ignored with ``exact_core``."""
    ctx = ctx or default_context()
    d = _dev(historical, ctx)
    h = C.c_void_p()
    flags = ((WITH_CORE if with_core else 0) | (KEEP_HISTORY if keep_history else 0)
             | (EXACT_CORE if exact_core else 0) | (LAZY_CORE if lazy_core else 0))
    _check(ctx.L.ctd_gpu_stream_init(ctx.h, d.h, mode, sample_size, epsilon, C.c_uint64(seed),
                                     flags, C.byref(h)))
    return StreamState(ctx, h, mode, d.shape[:-1])


def core_drift(state: StreamState) -> float:
    """core_drift (ctd_dynamic.hpp:64-66): |C - R^T X_hist|_F against the retained
    history; ArgumentError without it (ctd_dynamic.cpp:272-273)."""
    out = C.c_double()
    _check(state.ctx.L.ctd_gpu_stream_core_drift(state.h, C.byref(out)))
    return out.value


def ctd_d_step(state: StreamState, slab, sample_size: int) -> StreamState:
    """One Algorithm 2 step on a slab of time extent 1 (state updated in place
    and returned, like the reference's move-in/return-out)."""
    d = _dev(slab, state.ctx)
    _check(state.ctx.L.ctd_gpu_stream_step(state.h, d.h, sample_size))
    return state


def default_step_samples(sample_size: int) -> int:
    """default_step_samples (stream_harness.cpp:21-24): max(1, llround(0.01 s))."""
    import math
    v = 0.01 * float(sample_size)
    r = math.floor(v + 0.5) if v >= 0 else -math.floor(-v + 0.5)
    return max(1, int(r))
