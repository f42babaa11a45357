"""ctypes loader for libctd_gpu.so (the C-ABI in include/ctd_gpu.h).

There is no CPU fallback: if the CUDA library is not built, importing the
product API raises immediately.
"""
from __future__ import annotations

import ctypes as C
import os

HERE = os.path.dirname(os.path.abspath(__file__))
# CTD_GPU_LIB: an alternative build of the same library (kernel-variant experiments)
LIB_PATH = os.environ.get("CTD_GPU_LIB") or os.path.join(HERE, "libctd_gpu.so")

_lib = None


class ShardedInfo(C.Structure):
    _fields_ = [("n_fibers", C.c_int64), ("n_unique", C.c_int64), ("n_kept", C.c_int64),
                ("r_nnz", C.c_int64), ("cand_nnz", C.c_int64), ("local_fibers", C.c_int64),
                ("core_cols", C.c_int64), ("core_nnz", C.c_int64),
                ("total_sq_norm", C.c_double), ("relative_error", C.c_double)]


# int (*)(void *user, void *buf, int64_t n, int dtype): the host all-reduce callback
ALLREDUCE_FN = C.CFUNCTYPE(C.c_int, C.c_void_p, C.c_void_p, C.c_int64, C.c_int)


class FactorsInfo(C.Structure):
    _fields_ = [("kept", C.c_int64), ("r_rows", C.c_int64), ("r_nnz", C.c_int64),
                ("c_nnz", C.c_int64), ("n_drawn", C.c_int64), ("n_unique", C.c_int64),
                ("n_fibers", C.c_int64), ("n_cols", C.c_int64), ("u_nnz", C.c_int64),
                ("mode", C.c_int), ("order", C.c_int), ("epsilon", C.c_double),
                ("seed", C.c_uint64), ("total_sq_norm", C.c_double),
                ("relative_error", C.c_double), ("min_margin", C.c_double),
                ("integer_exact", C.c_int)]


# (name, restype, argtypes) for every symbol declared in include/ctd_gpu.h.
_V, _I, _I64, _D, _U64, _P = C.c_void_p, C.c_int, C.c_int64, C.c_double, C.c_uint64, C.c_void_p
_PV = C.POINTER(C.c_void_p)
SIGNATURES = [
    ("ctd_gpu_last_error", C.c_char_p, []),
    ("ctd_gpu_version", C.c_char_p, []),
    ("ctd_gpu_ctx_create", _I, [_I, _V, _PV]),
    ("ctd_gpu_ctx_set_stream", _I, [_V, _V]),
    ("ctd_gpu_ctx_trim", _I, [_V]),
    ("ctd_gpu_ctx_synchronize", _I, [_V]),
    ("ctd_gpu_ctx_destroy", _I, [_V]),
    ("ctd_gpu_ctx_launches", _I64, [_V]),
    ("ctd_gpu_ctx_set_timing", _I, [_V, _I]),
    ("ctd_gpu_ctx_phase_times", _I, [_V, _P, _P, _I]),
    ("ctd_gpu_phase_name", C.c_char_p, [_I]),
    ("ctd_gpu_tensor_from_host", _I, [_V, _I, _P, _I64, _P, _P, _PV]),
    ("ctd_gpu_tensor_from_device", _I, [_V, _I, _P, _I64, _P, _P, _PV]),
    ("ctd_gpu_tensor_nnz", _I64, [_V]),
    ("ctd_gpu_tensor_destroy", _I, [_V]),
    ("ctd_gpu_matricize", _I, [_V, _V, _I, _P, _P, _P, _P, _P, _P]),
    ("ctd_gpu_column_distribution", _I, [_V, _V, _I, _P, _P, _P]),
    ("ctd_gpu_column_sq_norms_csc", _I, [_V, _I64, _I64, _P, _P, _P, _P]),
    ("ctd_gpu_column_distribution_csc", _I, [_V, _I64, _I64, _P, _P, _P, _P, _P]),
    ("ctd_gpu_sample_with_replacement", _I, [_V, _P, _I64, _I64, _U64, _P]),
    ("ctd_gpu_seq_cumsum", _I, [_V, _P, _I64, _P]),
    ("ctd_gpu_unique_first_occurrence", _I, [_V, _P, _I64, _P, _P]),
    ("ctd_gpu_ctd_s", _I, [_V, _V, _I, _I64, _D, _U64, C.c_uint, _PV]),
    ("ctd_gpu_factors_info_get", _I, [_V, C.POINTER(FactorsInfo)]),
    ("ctd_gpu_factors_kept_flat", _I, [_V, _P]),
    ("ctd_gpu_factors_r", _I, [_V, _P, _P, _P]),
    ("ctd_gpu_factors_u", _I, [_V, _P]),
    ("ctd_gpu_factors_core", _I, [_V, _P, _P, _P, _P, _P]),
    ("ctd_gpu_factors_trace", _I, [_V, _P, _P, _P, _P, _P]),
    ("ctd_gpu_factors_destroy", _I, [_V]),
    ("ctd_gpu_relative_error", _I, [_V, _V, _V, _P]),
    ("ctd_gpu_memory_usage", _I, [_V, _V, _P]),
    ("ctd_gpu_basis_create", _I, [_V, _I64, _PV]),
    ("ctd_gpu_basis_destroy", _I, [_V]),
    ("ctd_gpu_basis_size", _I64, [_V]),
    ("ctd_gpu_basis_try_append", _I, [_V, _I64, _I64, _P, _P, _D, _P, _P, _P, _P]),
    ("ctd_gpu_basis_u", _I, [_V, _P]),
    ("ctd_gpu_sample_fibers", _I, [_V, _I64, _P, _P, _I64, _U64, _P, _P, _P]),
    ("ctd_gpu_basis_append_batch", _I, [_V, _I64, _P, _P, _P, _D, _P, _P, _P]),
    ("ctd_gpu_basis_append_batch_device", _I, [_V, _I64, _P, _P, _P, _D, _P, _P, _P]),
    ("ctd_gpu_basis_r_nnz", _I64, [_V]),
    ("ctd_gpu_basis_r", _I, [_V, _P, _P, _P]),
    ("ctd_gpu_basis_error_partials", _I, [_V, _V, _V, _I, _P, _P]),
    ("ctd_gpu_shard_create", _I, [_V, _V, _I, _PV]),
    ("ctd_gpu_shard_n_fibers", _I64, [_V]),
    ("ctd_gpu_shard_fibers", _I, [_V, _P, _P]),
    ("ctd_gpu_shard_gather", _I, [_V, _I64, _P, _P, _P, _P]),
    ("ctd_gpu_shard_gather_device", _I, [_V, _I64, _P, _P, _P, _P]),
    ("ctd_gpu_shard_error_partials", _I, [_V, _V, _P, _P]),
    ("ctd_gpu_shard_core", _I, [_V, _V, _P, _P]),
    ("ctd_gpu_shard_core_copy", _I, [_V, _P, _P, _P, _P]),
    ("ctd_gpu_compute_core", _I, [_V, _V, _I, _I64, _I64, _P, _P, _P, _PV]),
    ("ctd_gpu_chain_product", _I, [_V, _I64, _I64, _P, _P, _P, _I64, _P, _P, _P, _P, _I64, _P, _P, _P, _PV]),
    ("ctd_gpu_csc_info", _I, [_V, _P, _P, _P]),
    ("ctd_gpu_csc_copy", _I, [_V, _P, _P, _P, _P]),
    ("ctd_gpu_csc_destroy", _I, [_V]),
    ("ctd_gpu_core_shard_create", _I, [_V, _V, _PV]),
    ("ctd_gpu_core_shard_begin", _I, [_V, _V]),
    ("ctd_gpu_core_shard_step", _I, [_V, _V, _V, _I64]),
    ("ctd_gpu_core_shard_copy", _I, [_V, _P, _P, _P, _P, _P, _P]),
    ("ctd_gpu_core_shard_destroy", _I, [_V]),
    ("ctd_gpu_shard_destroy", _I, [_V]),
    ("ctd_gpu_shard_seq_total", _I, [_V, _D, _P]),
    ("ctd_gpu_shard_cdf", _I, [_V, _D, _D, _P, _P]),
    ("ctd_gpu_shard_clamp", _I, [_V]),
    ("ctd_gpu_shard_draw", _I, [_V, _I64, _U64, _P]),
    ("ctd_gpu_shard_find", _I, [_V, _I64, _P, _P]),
    ("ctd_gpu_shard_gather_into", _I, [_V, _I64, _P, _P, _P, _P]),
    ("ctd_gpu_comm_nccl_unique_id", _I, [_P]),
    ("ctd_gpu_comm_nccl_create", _I, [_V, _I, _I, _P, _PV]),
    ("ctd_gpu_comm_host_create", _I, [_V, _I, _I, ALLREDUCE_FN, _V, _PV]),
    ("ctd_gpu_comm_world", _I, [_V, C.POINTER(C.c_int), C.POINTER(C.c_int)]),
    ("ctd_gpu_comm_destroy", _I, [_V]),
    ("ctd_gpu_ctd_s_sharded", _I, [_V, _V, _V, _I, _I64, _D, _U64, C.c_uint, _PV]),
    ("ctd_gpu_sharded_info_get", _I, [_V, C.POINTER(ShardedInfo)]),
    ("ctd_gpu_sharded_kept", _I, [_V, _P]),
    ("ctd_gpu_sharded_trace", _I, [_V, _P, _P, _P, _P]),
    ("ctd_gpu_sharded_basis", _V, [_V]),
    ("ctd_gpu_sharded_shard", _V, [_V]),
    ("ctd_gpu_sharded_destroy", _I, [_V]),
    ("ctd_gpu_stream_init", _I, [_V, _V, _I, _I64, _D, _U64, C.c_uint, _PV]),
    ("ctd_gpu_stream_step", _I, [_V, _V, _I64]),
    ("ctd_gpu_stream_t", _I64, [_V]),
    ("ctd_gpu_stream_n_kept", _I64, [_V]),
    ("ctd_gpu_stream_factors", _I, [_V, _PV]),
    ("ctd_gpu_stream_core_drift", _I, [_V, C.POINTER(C.c_double)]),
    ("ctd_gpu_stream_core_pending", _I, [_V, C.POINTER(C.c_int64), C.POINTER(C.c_int64), C.POINTER(C.c_int64)]),
    ("ctd_gpu_stream_core_sync", _I, [_V]),
    ("ctd_gpu_stream_destroy", _I, [_V]),
]


def load(path: str = LIB_PATH):
    """Load libctd_gpu.so and bind every C-ABI symbol (raises if absent)."""
    global _lib
    if _lib is not None and path == LIB_PATH:
        return _lib
    if not os.path.exists(path):
        raise ImportError(f"{path} is not built; run `python -c 'import __graft_entry__ as g; "
                          f"g.build()'` (there is no CPU fallback)")
    lib = C.CDLL(path)
    for name, res, args in SIGNATURES:
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    if path == LIB_PATH:
        _lib = lib
    return lib
