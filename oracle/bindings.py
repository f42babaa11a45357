"""TEST INFRASTRUCTURE ONLY — ctypes bindings of the two CPU oracles.

``Port`` wraps our C restatement (oracle/ctd_oracle.c); ``Ref`` wraps the
unmodified reference library built by ``make -C oracle ref``.  Both expose the
same Python surface so parity tests can run against either.
"""
from __future__ import annotations

import ctypes as C
import os
import subprocess
from dataclasses import dataclass, field

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
PORT_SO = os.path.join(HERE, "libctd_oracle.so")
REF_SO = os.path.join(HERE, "_ref", "libctdref.so")
REF_SRC = "/root/reference/proj/core"

ERROR_NAMES = {1: "argument", 2: "shape", 3: "empty_input", 4: "parse",
               5: "metric", 6: "oracle", 7: "io", 99: "other"}


class OracleError(RuntimeError):
    def __init__(self, code: int, msg: str = ""):
        super().__init__(f"{ERROR_NAMES.get(code, code)}: {msg}")
        self.code = code


def build(ref: bool = True) -> None:
    """Compile the port, and the reference when its sources are present."""
    subprocess.run(["make", "-s", "-C", HERE, "port"], check=True)
    if ref and os.path.isdir(REF_SRC):
        subprocess.run(["make", "-s", "-C", HERE, "ref", f"-j{os.cpu_count() or 4}"],
                       check=True)


def ref_available() -> bool:
    return os.path.exists(REF_SO)


def _p(a: np.ndarray):
    return a.ctypes.data_as(C.c_void_p)


def _i64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.int64)


def _f64(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float64)


@dataclass
class Csc:
    rows: int
    cols: int
    col_ptr: np.ndarray
    row: np.ndarray
    val: np.ndarray

    @property
    def nnz(self) -> int:
        return int(self.col_ptr[-1])


@dataclass
class FrontEnd:
    """Outcome of the Algorithm 1 front end (drawn, unique, decisions, R, U)."""
    drawn: np.ndarray
    unique: np.ndarray
    accepted: np.ndarray
    degenerate: np.ndarray
    delta: np.ndarray
    kept_flat: np.ndarray
    U: np.ndarray
    R: Csc
    total: float = 0.0
    seconds: float = 0.0
    extra: dict = field(default_factory=dict)


class _CscStruct(C.Structure):
    _fields_ = [("rows", C.c_int64), ("cols", C.c_int64), ("nnz", C.c_int64),
                ("col_ptr", C.POINTER(C.c_int64)), ("row", C.POINTER(C.c_int64)),
                ("val", C.POINTER(C.c_double))]


class _FrontStruct(C.Structure):
    _fields_ = [("n_drawn", C.c_int64), ("n_unique", C.c_int64), ("kept", C.c_int64),
                ("drawn", C.POINTER(C.c_int64)), ("unique", C.POINTER(C.c_int64)),
                ("kept_flat", C.POINTER(C.c_int64)),
                ("accepted", C.POINTER(C.c_int)), ("degenerate", C.POINTER(C.c_int)),
                ("delta", C.POINTER(C.c_double)), ("total", C.c_double),
                ("basis", C.c_void_p)]


def _arr(ptr, n, dtype):
    if n == 0:
        return np.zeros(0, dtype=dtype)
    return np.ctypeslib.as_array(ptr, shape=(n,)).astype(dtype, copy=True)


def _csc_from_struct(s: _CscStruct) -> Csc:
    return Csc(int(s.rows), int(s.cols), _arr(s.col_ptr, s.cols + 1, np.int64),
               _arr(s.row, s.nnz, np.int64), _arr(s.val, s.nnz, np.float64))


class Port:
    """Our C restatement (oracle/ctd_oracle.c)."""

    def __init__(self, path: str = PORT_SO):
        if not os.path.exists(path):
            build(ref=False)
        L = self.L = C.CDLL(path)
        v, i64, f64, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.cto_matricize.argtypes = [i32, v, i64, v, v, i32, C.POINTER(_CscStruct)]
        L.cto_csc_free.argtypes = [C.POINTER(_CscStruct)]
        L.cto_column_sq_norms.argtypes = [C.POINTER(_CscStruct), v]
        L.cto_column_distribution.argtypes = [C.POINTER(_CscStruct), v, C.POINTER(f64)]
        L.cto_sample_with_replacement.argtypes = [v, i64, i64, C.c_uint64, v]
        L.cto_unique_first_occurrence.argtypes = [v, i64, v]
        L.cto_unique_first_occurrence.restype = i64
        L.cto_mt19937_64.argtypes = [C.c_uint64, i64, v]
        L.cto_basis_new.argtypes = [i64]
        L.cto_basis_new.restype = v
        L.cto_basis_free.argtypes = [v]
        L.cto_basis_size.argtypes = [v]
        L.cto_basis_size.restype = i64
        L.cto_basis_u.argtypes = [v]
        L.cto_basis_u.restype = C.POINTER(f64)
        L.cto_basis_try_append.argtypes = [v, i64, i64, v, v, f64, C.POINTER(i32),
                                           C.POINTER(i32), C.POINTER(f64), v]
        L.cto_basis_r.argtypes = [v, C.POINTER(_CscStruct)]
        L.cto_ctd_s_frontend.argtypes = [i32, v, i64, v, v, i32, i64, f64, C.c_uint64,
                                         C.POINTER(_FrontStruct)]
        L.cto_frontend_free.argtypes = [C.POINTER(_FrontStruct)]
        L.cto_core_matricized.argtypes = [C.POINTER(_CscStruct)] * 3
        L.cto_relative_error.argtypes = [C.POINTER(_CscStruct), f64, C.POINTER(_CscStruct),
                                         v, C.POINTER(_CscStruct), C.POINTER(f64)]
        L.cto_relerr_dd_direct.argtypes = [C.POINTER(_CscStruct), C.POINTER(_CscStruct), v] + \
            [C.POINTER(f64)] * 4
        L.cto_relerr_dd_full.argtypes = [C.POINTER(_CscStruct), C.POINTER(_CscStruct), v] + \
            [C.POINTER(f64)] * 3
        L.cto_filter_par.argtypes = [i64, i64, v, v, v, f64, v, v, v, C.POINTER(i64), v]
        L.cto_stream_init2.argtypes = [i32, v, i64, v, v, i32, i64, f64, C.c_uint64, i32, C.POINTER(v)]
        L.cto_stream_init.argtypes = [i32, v, i64, v, v, i32, i64, f64, C.c_uint64,
                                      C.POINTER(v)]
        L.cto_stream_step.argtypes = [v, i32, v, i64, v, v, i64]
        L.cto_stream_free.argtypes = [v]
        for n in ("cto_stream_t", "cto_stream_kept"):
            getattr(L, n).argtypes = [v]
            getattr(L, n).restype = i64
        L.cto_stream_kept_flat.argtypes = [v]
        L.cto_stream_kept_flat.restype = C.POINTER(i64)
        L.cto_stream_basis.argtypes = [v]
        L.cto_stream_basis.restype = v
        L.cto_stream_core.argtypes = [v]
        L.cto_stream_core.restype = C.POINTER(_CscStruct)

    def _chk(self, st, what=""):
        if st:
            raise OracleError(st, what)

    # -- tensor_ops -----------------------------------------------------------
    def matricize(self, shape, idx, val, mode) -> Csc:
        shape, idx, val = _i64(shape), _i64(idx), _f64(val)
        s = _CscStruct()
        self._chk(self.L.cto_matricize(len(shape), _p(shape), len(val), _p(idx), _p(val),
                                       mode, C.byref(s)), "matricize")
        out = _csc_from_struct(s)
        self.L.cto_csc_free(C.byref(s))
        return out

    @staticmethod
    def _struct(m: Csc, keep: list) -> _CscStruct:
        cp, r, v = _i64(m.col_ptr), _i64(m.row), _f64(m.val)
        keep += [cp, r, v]
        return _CscStruct(m.rows, m.cols, m.nnz, cp.ctypes.data_as(C.POINTER(C.c_int64)),
                          r.ctypes.data_as(C.POINTER(C.c_int64)),
                          v.ctypes.data_as(C.POINTER(C.c_double)))

    def column_sq_norms(self, m: Csc) -> np.ndarray:
        keep: list = []
        s = self._struct(m, keep)
        out = np.zeros(m.cols)
        self.L.cto_column_sq_norms(C.byref(s), _p(out))
        return out

    def column_distribution(self, m: Csc):
        keep: list = []
        s = self._struct(m, keep)
        out = np.zeros(m.cols)
        tot = C.c_double()
        self._chk(self.L.cto_column_distribution(C.byref(s), _p(out), C.byref(tot)),
                  "column_distribution")
        return out, tot.value

    def sample_with_replacement(self, probs, count, seed) -> np.ndarray:
        probs = _f64(probs)
        out = np.zeros(max(count, 0), dtype=np.int64)
        self._chk(self.L.cto_sample_with_replacement(_p(probs), len(probs), count,
                                                     C.c_uint64(seed), _p(out)), "sample")
        return out

    def unique_first_occurrence(self, drawn) -> np.ndarray:
        drawn = _i64(drawn)
        out = np.zeros(len(drawn), dtype=np.int64)
        n = self.L.cto_unique_first_occurrence(_p(drawn), len(drawn), _p(out))
        return out[:n].copy()

    def mt19937_64(self, seed, count) -> np.ndarray:
        out = np.zeros(count, dtype=np.uint64)
        self.L.cto_mt19937_64(C.c_uint64(seed), count, _p(out))
        return out

    # -- FiberBasis -------------------------------------------------------------
    def basis(self, dim):
        return _PortBasis(self, dim)

    # -- ctd_s front end --------------------------------------------------------
    def frontend(self, shape, idx, val, mode, s, eps=1e-6, seed=42) -> FrontEnd:
        shape, idx, val = _i64(shape), _i64(idx), _f64(val)
        f = _FrontStruct()
        st = self.L.cto_ctd_s_frontend(len(shape), _p(shape), len(val), _p(idx), _p(val),
                                       mode, s, eps, C.c_uint64(seed), C.byref(f))
        if st:
            self.L.cto_frontend_free(C.byref(f))
            raise OracleError(st, "ctd_s")
        k = int(f.kept)
        u = np.ctypeslib.as_array(self.L.cto_basis_u(f.basis), shape=(k * k,)).reshape(k, k).copy() if k else np.zeros((0, 0))
        rs = _CscStruct()
        self.L.cto_basis_r(f.basis, C.byref(rs))
        R = _csc_from_struct(rs)
        self.L.cto_csc_free(C.byref(rs))
        nu = int(f.n_unique)
        out = FrontEnd(_arr(f.drawn, f.n_drawn, np.int64), _arr(f.unique, nu, np.int64),
                       _arr(f.accepted, nu, np.int32), _arr(f.degenerate, nu, np.int32),
                       _arr(f.delta, nu, np.float64), _arr(f.kept_flat, k, np.int64), u, R,
                       total=float(f.total))
        self.L.cto_frontend_free(C.byref(f))
        return out

    def core_matricized(self, x: Csc, r: Csc) -> Csc:
        keep: list = []
        a, b = self._struct(x, keep), self._struct(r, keep)
        o = _CscStruct()
        self._chk(self.L.cto_core_matricized(C.byref(a), C.byref(b), C.byref(o)), "core")
        out = _csc_from_struct(o)
        self.L.cto_csc_free(C.byref(o))
        return out

    def relative_error(self, x: Csc, x_sq: float, r: Csc, u: np.ndarray, core: Csc) -> float:
        keep: list = []
        a, b, c = self._struct(x, keep), self._struct(r, keep), self._struct(core, keep)
        u = _f64(u).reshape(-1)
        out = C.c_double()
        self._chk(self.L.cto_relative_error(C.byref(a), x_sq, C.byref(b), _p(u), C.byref(c),
                                            C.byref(out)), "relative_error")
        return out.value

    def relerr_dd_direct(self, x: Csc, r: Csc, u: np.ndarray):
        """Double-double |x_j - R U R^T x_j|^2 summed over the columns of x, and |x|^2,
        each as (hi, lo) (relerr_dd.c, evaluation.cpp:100-121)."""
        keep: list = []
        a, b = self._struct(x, keep), self._struct(r, keep)
        u = _f64(u).reshape(-1)
        o = [C.c_double() for _ in range(4)]
        self._chk(self.L.cto_relerr_dd_direct(C.byref(a), C.byref(b), _p(u), *[C.byref(t) for t in o]),
                  "relerr_dd_direct")
        return (o[0].value, o[1].value), (o[2].value, o[3].value)

    def relerr_dd_full(self, x: Csc, r: Csc, u: np.ndarray):
        """Double-double relative error of the whole matricized tensor x (relerr_dd.c)."""
        keep: list = []
        a, b = self._struct(x, keep), self._struct(r, keep)
        u = _f64(u).reshape(-1)
        o = [C.c_double() for _ in range(3)]
        self._chk(self.L.cto_relerr_dd_full(C.byref(a), C.byref(b), _p(u), *[C.byref(t) for t in o]),
                  "relerr_dd_full")
        return o[0].value

    def filter_par(self, dim, cand_ptr, rows, vals, eps=1e-6):
        """The filter loop over candidate fibers (CSC) from an empty basis,
        multi-threaded, bit-identical to FiberBasis (filter_par.c).  Returns
        (accepted, degenerate, delta, U)."""
        cand_ptr, rows, vals = _i64(cand_ptr), _i64(rows), _f64(vals)
        n = cand_ptr.shape[0] - 1
        acc = np.zeros(max(n, 1), np.int32)
        deg = np.zeros(max(n, 1), np.int32)
        dl = np.zeros(max(n, 1))
        u = np.zeros(max(n * n, 1))
        k = C.c_int64()
        self._chk(self.L.cto_filter_par(dim, n, _p(cand_ptr), _p(rows), _p(vals), eps, _p(acc), _p(deg), _p(dl),
                                        C.byref(k), _p(u)), "filter_par")
        K = k.value
        return acc[:n], deg[:n], dl[:n], u[:K * K].reshape(K, K).copy()

    def ctd_s_error(self, shape, idx, val, mode, s, eps=1e-6, seed=42):
        """Front end + compute_core + relative_error (the reference composition)."""
        fe = self.frontend(shape, idx, val, mode, s, eps, seed)
        xm = self.matricize(shape, idx, val, mode)
        core = self.core_matricized(xm, fe.R)
        x_sq = 0.0
        for v in _f64(val):  # evaluation.cpp:91-92, sequential in tensor order
            x_sq += v * v
        return fe, core, self.relative_error(xm, x_sq, fe.R, fe.U, core)

    # -- CTD-D ------------------------------------------------------------------
    def stream(self, shape, idx, val, mode, s, eps=1e-6, seed=42, core=True):
        """init_stream; core=False keeps only the front end (kept ids, basis)."""
        return _PortStream(self, shape, idx, val, mode, s, eps, seed, core)


class _PortBasis:
    def __init__(self, port: Port, dim: int):
        self.P, self.dim = port, dim
        self.h = port.L.cto_basis_new(dim)

    def __del__(self):
        if getattr(self, "h", None):
            self.P.L.cto_basis_free(self.h)
            self.h = None

    def size(self) -> int:
        return int(self.P.L.cto_basis_size(self.h))

    def U(self) -> np.ndarray:
        k = self.size()
        if k == 0:
            return np.zeros((0, 0))
        return np.ctypeslib.as_array(self.P.L.cto_basis_u(self.h), shape=(k * k,)).reshape(k, k).copy()

    def try_append(self, idx, val, eps=1e-6, dim=None):
        idx, val = _i64(idx), _f64(val)
        k = self.size()
        y = np.zeros(max(k, 1))
        a, d, dl = C.c_int(), C.c_int(), C.c_double()
        self.P._chk(self.P.L.cto_basis_try_append(self.h, self.dim if dim is None else dim,
                                                  len(val), _p(idx), _p(val), eps,
                                                  C.byref(a), C.byref(d), C.byref(dl), _p(y)),
                    "try_append")
        return bool(a.value), bool(d.value), dl.value, y[:k].copy()


class _PortStream:
    def __init__(self, port, shape, idx, val, mode, s, eps, seed, core=True):
        self.P = port
        shape, idx, val = _i64(shape), _i64(idx), _f64(val)
        h = C.c_void_p()
        port._chk(port.L.cto_stream_init2(len(shape), _p(shape), len(val), _p(idx), _p(val),
                                          mode, s, eps, C.c_uint64(seed), 0 if core else 1, C.byref(h)),
                  "init_stream")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.P.L.cto_stream_free(self.h)
            self.h = None

    def step(self, shape, idx, val, d):
        shape, idx, val = _i64(shape), _i64(idx), _f64(val)
        self.P._chk(self.P.L.cto_stream_step(self.h, len(shape), _p(shape), len(val), _p(idx),
                                             _p(val), d), "ctd_d_step")

    @property
    def t(self) -> int:
        return int(self.P.L.cto_stream_t(self.h))

    def kept_flat(self) -> np.ndarray:
        k = int(self.P.L.cto_stream_kept(self.h))
        return _arr(self.P.L.cto_stream_kept_flat(self.h), k, np.int64)

    def U(self) -> np.ndarray:
        b = self.P.L.cto_stream_basis(self.h)
        k = int(self.P.L.cto_basis_size(b))
        if k == 0:
            return np.zeros((0, 0))
        return np.ctypeslib.as_array(self.P.L.cto_basis_u(b), shape=(k * k,)).reshape(k, k).copy()

    def core(self) -> Csc:
        return _csc_from_struct(self.P.L.cto_stream_core(self.h).contents)


class Ref:
    """The unmodified reference (oracle/_ref/libctdref.so)."""

    def __init__(self, path: str = REF_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle ref` where "
                                    f"/root/reference is present")
        L = self.L = C.CDLL(path)
        v, i64, f64, i32 = C.c_void_p, C.c_int64, C.c_double, C.c_int
        L.ref_last_error.restype = C.c_char_p
        L.ref_tensor_new.argtypes = [i32, v, i64, v, v, C.POINTER(v)]
        L.ref_tensor_free.argtypes = [v]
        L.ref_tensor_nnz.argtypes = [v]
        L.ref_tensor_nnz.restype = i64
        L.ref_tensor_data.argtypes = [v, v, v]
        L.ref_matricize.argtypes = [v, i32, v, v, v, v]
        L.ref_column_distribution.argtypes = [v, i32, v, C.POINTER(f64)]
        L.ref_sample_with_replacement.argtypes = [v, i64, f64, i64, C.c_uint64, v]
        L.ref_unique_first_occurrence.argtypes = [v, i64, v, C.POINTER(i64)]
        L.ref_basis_new.argtypes = [i64, C.POINTER(v)]
        L.ref_basis_free.argtypes = [v]
        L.ref_basis_size.argtypes = [v]
        L.ref_basis_size.restype = i64
        L.ref_basis_u.argtypes = [v, v]
        L.ref_basis_try_append.argtypes = [v, i64, i64, v, v, f64, C.POINTER(i32),
                                           C.POINTER(i32), C.POINTER(f64), v]
        L.ref_ctd_s.argtypes = [v, i32, i64, f64, C.c_uint64, C.POINTER(v)]
        L.ref_frontend.argtypes = [v, i32, i64, f64, C.c_uint64, C.POINTER(v)]
        L.ref_factors_free.argtypes = [v]
        for n in ("ref_factors_kept", "ref_factors_r_rows", "ref_factors_r_nnz",
                  "ref_factors_c_nnz"):
            getattr(L, n).argtypes = [v]
            getattr(L, n).restype = i64
        L.ref_factors_seconds.argtypes = [v]
        L.ref_factors_seconds.restype = f64
        L.ref_factors_c_order.argtypes = [v]
        L.ref_factors_c_shape.argtypes = [v, v]
        L.ref_factors_kept_flat.argtypes = [v, v]
        L.ref_factors_kept_coords.argtypes = [v, v]
        L.ref_factors_r.argtypes = [v, v, v, v]
        L.ref_factors_u.argtypes = [v, v]
        L.ref_factors_c.argtypes = [v, v, v]
        L.ref_trace_len.argtypes = [v, i32]
        L.ref_trace_len.restype = i64
        L.ref_trace.argtypes = [v, v, v, v, v, v]
        L.ref_trace_total.argtypes = [v]
        L.ref_trace_total.restype = f64
        L.ref_relative_error.argtypes = [v, v, C.POINTER(f64)]
        L.ref_memory_usage.argtypes = [v, v, C.POINTER(f64)]
        L.ref_init_stream.argtypes = [v, i32, i64, f64, C.c_uint64, i32, i32, C.POINTER(v)]
        L.ref_stream_free.argtypes = [v]
        L.ref_stream_step.argtypes = [v, v, i64, C.POINTER(f64)]
        L.ref_stream_t.argtypes = [v]
        L.ref_stream_t.restype = i64
        L.ref_stream_factors.argtypes = [v, C.POINTER(v)]
        for n in ("ref_stream_core_nnz", "ref_stream_core_rows", "ref_stream_core_cols"):
            getattr(L, n).argtypes = [v]
            getattr(L, n).restype = i64
        L.ref_stream_core.argtypes = [v, v, v, v]
        L.ref_core_drift.argtypes = [v, C.POINTER(f64)]
        if hasattr(L, "ref_run_stream"):
            L.ref_run_stream.argtypes = [v, i32, i64, i64, f64, f64, C.c_uint64, i32, C.POINTER(i64), v, v, v,
                                         v, v, v]
            L.ref_tsv_line.argtypes = [i64, f64, f64, f64, i64, C.c_char_p, i64]
        if hasattr(L, "ref_compute_core"):
            L.ref_compute_core.argtypes = [v, i32, i64, i64, v, v, v, C.POINTER(v)]
            L.ref_chain_product.argtypes = [i64, i64, v, v, v, i64, i64, v, v, v, i64, i64, v, i64, i64, v, v, v,
                                            C.POINTER(v)]
            L.ref_matrix_free.argtypes = [v]
            L.ref_matrix_shape.argtypes = [v, v, v, v]
            L.ref_matrix_data.argtypes = [v, v, v, v]
        if hasattr(L, "ref_save_factors"):
            L.ref_save_factors.argtypes = [v, C.c_char_p]
            L.ref_load_factors.argtypes = [C.c_char_p, C.POINTER(v)]
            L.ref_detect_ddos.argtypes = [v, C.POINTER(i64), v, v, v]
            L.ref_decompose_online.argtypes = [v, i32, i64, f64, C.c_uint64, C.POINTER(v)]

    def _chk(self, st, what=""):
        if st:
            raise OracleError(st, f"{what}: {self.L.ref_last_error().decode()}")

    def tensor(self, shape, idx, val):
        return _RefTensor(self, shape, idx, val)

    def compute_core(self, t: "_RefTensor", r: Csc, mode: int):
        """ctd::compute_core (ctd_static.hpp:28) -> (shape, flat indices, values) of C."""
        h = C.c_void_p()
        cp, rr, rv = _i64(r.col_ptr), _i64(r.row), _f64(r.val)  # held across the call
        self._chk(self.L.ref_compute_core(t.h, mode, r.rows, r.cols, _p(cp), _p(rr), _p(rv), C.byref(h)),
                  "compute_core")
        out = _RefTensor.__new__(_RefTensor)
        out.R, out.h = self, h
        out.nnz = int(self.L.ref_tensor_nnz(h))
        shape = list(t.shape)
        shape[mode] = r.cols
        out.shape = shape
        return out

    def chain_product(self, dr: Csc, r: Csc, u: np.ndarray, core: Csc) -> Csc:
        """ctd::chain_product (ctd_dynamic.hpp:61-62)."""
        h = C.c_void_p()
        uu = np.ascontiguousarray(u, np.float64)
        a = (_i64(dr.col_ptr), _i64(dr.row), _f64(dr.val))  # held across the call
        b = (_i64(r.col_ptr), _i64(r.row), _f64(r.val))
        c = (_i64(core.col_ptr), _i64(core.row), _f64(core.val))
        self._chk(self.L.ref_chain_product(dr.rows, dr.cols, _p(a[0]), _p(a[1]), _p(a[2]), r.rows, r.cols,
                                           _p(b[0]), _p(b[1]), _p(b[2]), uu.shape[0], uu.shape[1], _p(uu), core.rows,
                                           core.cols, _p(c[0]), _p(c[1]), _p(c[2]), C.byref(h)), "chain_product")
        try:
            rows, cols, nnz = C.c_int64(), C.c_int64(), C.c_int64()
            self.L.ref_matrix_shape(h, C.byref(rows), C.byref(cols), C.byref(nnz))
            cp = np.zeros(cols.value + 1, np.int64)
            rr = np.zeros(max(nnz.value, 1), np.int64)
            vv = np.zeros(max(nnz.value, 1))
            self.L.ref_matrix_data(h, _p(cp), _p(rr), _p(vv))
            return Csc(rows.value, cols.value, cp, rr[:nnz.value], vv[:nnz.value])
        finally:
            self.L.ref_matrix_free(h)

    def matricize(self, t: "_RefTensor", mode: int):
        shape = t.shape
        cols = int(np.prod([s for k, s in enumerate(shape) if k != mode], dtype=np.int64))
        cp = np.zeros(cols + 1, dtype=np.int64)
        rows = np.zeros(t.nnz, dtype=np.int64)
        vals = np.zeros(t.nnz)
        norms = np.zeros(cols)
        self._chk(self.L.ref_matricize(t.h, mode, _p(cp), _p(rows), _p(vals), _p(norms)),
                  "matricize")
        return Csc(int(shape[mode]), cols, cp, rows, vals), norms

    def column_distribution(self, t, mode):
        cols = int(np.prod([s for k, s in enumerate(t.shape) if k != mode], dtype=np.int64))
        p = np.zeros(cols)
        tot = C.c_double()
        self._chk(self.L.ref_column_distribution(t.h, mode, _p(p), C.byref(tot)),
                  "column_distribution")
        return p, tot.value

    def sample_with_replacement(self, probs, count, seed, total=1.0):
        probs = _f64(probs)
        out = np.zeros(max(count, 0), dtype=np.int64)
        self._chk(self.L.ref_sample_with_replacement(_p(probs), len(probs), total, count,
                                                     C.c_uint64(seed), _p(out)), "sample")
        return out

    def unique_first_occurrence(self, drawn):
        drawn = _i64(drawn)
        out = np.zeros(len(drawn), dtype=np.int64)
        n = C.c_int64()
        self._chk(self.L.ref_unique_first_occurrence(_p(drawn), len(drawn), _p(out),
                                                     C.byref(n)), "unique")
        return out[:n.value].copy()

    def basis(self, dim):
        return _RefBasis(self, dim)

    def _factors(self, h, trace: bool) -> FrontEnd:
        L = self.L
        k = int(L.ref_factors_kept(h))
        rows = int(L.ref_factors_r_rows(h))
        rnnz = int(L.ref_factors_r_nnz(h))
        cp = np.zeros(k + 1, dtype=np.int64)
        rr = np.zeros(rnnz, dtype=np.int64)
        rv = np.zeros(rnnz)
        L.ref_factors_r(h, _p(cp), _p(rr), _p(rv))
        u = np.zeros(k * k)
        L.ref_factors_u(h, _p(u))
        kf = np.zeros(k, dtype=np.int64)
        L.ref_factors_kept_flat(h, _p(kf))
        fe = FrontEnd(np.zeros(0, np.int64), np.zeros(0, np.int64), np.zeros(0, np.int32),
                      np.zeros(0, np.int32), np.zeros(0), kf, u.reshape(k, k),
                      Csc(rows, k, cp, rr, rv), seconds=float(L.ref_factors_seconds(h)))
        if trace:
            nd, nu = int(L.ref_trace_len(h, 0)), int(L.ref_trace_len(h, 1))
            fe.drawn = np.zeros(nd, np.int64)
            fe.unique = np.zeros(nu, np.int64)
            fe.accepted = np.zeros(nu, np.int32)
            fe.degenerate = np.zeros(nu, np.int32)
            fe.delta = np.zeros(nu)
            L.ref_trace(h, _p(fe.drawn), _p(fe.unique), _p(fe.accepted), _p(fe.degenerate),
                        _p(fe.delta))
            fe.total = float(L.ref_trace_total(h))
        return fe

    def frontend(self, t, mode, s, eps=1e-6, seed=42) -> FrontEnd:
        h = C.c_void_p()
        self._chk(self.L.ref_frontend(t.h, mode, s, eps, C.c_uint64(seed), C.byref(h)), "frontend")
        try:
            return self._factors(h, True)
        finally:
            self.L.ref_factors_free(h)

    def ctd_s(self, t, mode, s, eps=1e-6, seed=42, error=True):
        """Full reference ctd_s; returns (FrontEnd-like factors, core CSC..., rel err)."""
        h = C.c_void_p()
        self._chk(self.L.ref_ctd_s(t.h, mode, s, eps, C.c_uint64(seed), C.byref(h)), "ctd_s")
        try:
            fe = self._factors(h, False)
            fe.extra["c_nnz"] = int(self.L.ref_factors_c_nnz(h))
            if error:
                e = C.c_double()
                self._chk(self.L.ref_relative_error(t.h, h, C.byref(e)), "relative_error")
                fe.extra["relative_error"] = e.value
                m = C.c_double()
                self._chk(self.L.ref_memory_usage(t.h, h, C.byref(m)), "memory_usage")
                fe.extra["memory_usage"] = m.value
            return fe
        finally:
            self.L.ref_factors_free(h)

    def _with_factors(self, h, save_dir=None, detect=False):
        try:
            out = {}
            if save_dir is not None:
                self._chk(self.L.ref_save_factors(h, save_dir.encode()), "save_factors")
            if detect:
                k = int(self.L.ref_factors_kept(h))
                n = C.c_int64()
                dst, b = np.zeros(max(k, 1), np.int64), np.zeros(max(k, 1), np.int64)
                nrm = np.zeros(max(k, 1))
                self._chk(self.L.ref_detect_ddos(h, C.byref(n), _p(dst), _p(b), _p(nrm)), "detect_ddos")
                out["detect"] = [(int(dst[i]), int(b[i]), float(nrm[i])) for i in range(n.value)]
            return out
        finally:
            self.L.ref_factors_free(h)

    def ctd_s_bundle(self, t, mode, s, eps, seed, save_dir=None, detect=False) -> dict:
        """Reference ctd_s, then save_factors / detect_ddos on its factors."""
        h = C.c_void_p()
        self._chk(self.L.ref_ctd_s(t.h, mode, s, eps, C.c_uint64(seed), C.byref(h)), "ctd_s")
        return self._with_factors(h, save_dir, detect)

    def decompose_online(self, t, mode, d, eps, seed, save_dir=None, detect=False) -> dict:
        h = C.c_void_p()
        self._chk(self.L.ref_decompose_online(t.h, mode, d, eps, C.c_uint64(seed), C.byref(h)),
                  "decompose_online")
        return self._with_factors(h, save_dir, detect)

    def resave(self, src_dir, dst_dir) -> None:
        """load_factors(src) then save_factors(dst) with the reference."""
        h = C.c_void_p()
        self._chk(self.L.ref_load_factors(src_dir.encode(), C.byref(h)), "load_factors")
        self._with_factors(h, dst_dir)

    def run_stream(self, x, mode=0, sample_size=100, step_samples=None, split=0.8, eps=1e-6, seed=42,
                   exact_core=False) -> dict:
        """run_stream (stream_harness.cpp:48-107) on a _RefTensor: per-step reports + mean."""
        T = int(x.shape[-1])
        n = C.c_int64()
        step = np.zeros(T + 1, np.int64)
        err, mem, secs = np.zeros(T + 1), np.zeros(T + 1), np.zeros(T + 1)
        kept = np.zeros(T + 1, np.int64)
        mean = np.zeros(4)
        self._chk(self.L.ref_run_stream(x.h, mode, sample_size, step_samples or 0, split, eps,
                                        C.c_uint64(seed), int(exact_core), C.byref(n), _p(step), _p(err),
                                        _p(mem), _p(secs), _p(kept), _p(mean)), "run_stream")
        k = n.value
        return {"step": step[:k], "relative_error": err[:k], "memory_usage": mem[:k],
                "seconds": secs[:k], "kept_fibers": kept[:k], "mean": mean}

    def tsv_line(self, step, err=0.0, secs=0.0, mem=0.0, kept=0) -> str:
        """tsv_line (evaluation.cpp:51-62); step < 0 gives tsv_header()."""
        buf = C.create_string_buffer(256)
        self._chk(self.L.ref_tsv_line(step, err, secs, mem, kept, buf, 256), "tsv_line")
        return buf.value.decode()

    def stream(self, hist, mode, s, eps=1e-6, seed=42, keep_history=False, exact_core=False):
        return _RefStream(self, hist, mode, s, eps, seed, keep_history, exact_core)


class _RefTensor:
    def __init__(self, R: Ref, shape, idx, val):
        self.R = R
        self.shape = [int(s) for s in shape]
        shape, idx, val = _i64(shape), _i64(idx), _f64(val)
        h = C.c_void_p()
        R._chk(R.L.ref_tensor_new(len(shape), _p(shape), len(val), _p(idx), _p(val),
                                  C.byref(h)), "SparseTensor")
        self.h = h
        self.nnz = int(R.L.ref_tensor_nnz(h))

    def __del__(self):
        if getattr(self, "h", None):
            self.R.L.ref_tensor_free(self.h)
            self.h = None

    def data(self):
        idx = np.zeros(self.nnz * len(self.shape), dtype=np.int64)
        val = np.zeros(self.nnz)
        self.R.L.ref_tensor_data(self.h, _p(idx), _p(val))
        return idx, val


class _RefBasis:
    def __init__(self, R: Ref, dim: int):
        self.R, self.dim = R, dim
        h = C.c_void_p()
        R._chk(R.L.ref_basis_new(dim, C.byref(h)), "FiberBasis")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.R.L.ref_basis_free(self.h)
            self.h = None

    def size(self):
        return int(self.R.L.ref_basis_size(self.h))

    def U(self):
        k = self.size()
        u = np.zeros(k * k)
        self.R.L.ref_basis_u(self.h, _p(u))
        return u.reshape(k, k)

    def try_append(self, idx, val, eps=1e-6, dim=None):
        idx, val = _i64(idx), _f64(val)
        k = self.size()
        y = np.zeros(max(k, 1))
        a, d, dl = C.c_int(), C.c_int(), C.c_double()
        self.R._chk(self.R.L.ref_basis_try_append(self.h, self.dim if dim is None else dim,
                                                  len(val), _p(idx), _p(val), eps, C.byref(a),
                                                  C.byref(d), C.byref(dl), _p(y)), "try_append")
        return bool(a.value), bool(d.value), dl.value, y[:k].copy()


class _RefStream:
    def __init__(self, R, hist, mode, s, eps, seed, keep_history, exact_core):
        self.R = R
        h = C.c_void_p()
        R._chk(R.L.ref_init_stream(hist.h, mode, s, eps, C.c_uint64(seed), int(keep_history),
                                   int(exact_core), C.byref(h)), "init_stream")
        self.h = h

    def __del__(self):
        if getattr(self, "h", None):
            self.R.L.ref_stream_free(self.h)
            self.h = None

    def step(self, slab, d) -> float:
        sec = C.c_double()
        self.R._chk(self.R.L.ref_stream_step(self.h, slab.h, d, C.byref(sec)), "ctd_d_step")
        return sec.value

    @property
    def t(self):
        return int(self.R.L.ref_stream_t(self.h))

    def factors(self) -> FrontEnd:
        h = C.c_void_p()
        self.R._chk(self.R.L.ref_stream_factors(self.h, C.byref(h)), "factors")
        try:
            return self.R._factors(h, False)
        finally:
            self.R.L.ref_factors_free(h)

    def core(self) -> Csc:
        L = self.R.L
        n, r, c = (int(L.ref_stream_core_nnz(self.h)), int(L.ref_stream_core_rows(self.h)),
                   int(L.ref_stream_core_cols(self.h)))
        cp = np.zeros(c + 1, np.int64)
        rows = np.zeros(n, np.int64)
        vals = np.zeros(n)
        L.ref_stream_core(self.h, _p(cp), _p(rows), _p(vals))
        return Csc(r, c, cp, rows, vals)

    def core_drift(self) -> float:
        out = C.c_double()
        self.R._chk(self.R.L.ref_core_drift(self.h, C.byref(out)), "core_drift")
        return out.value
