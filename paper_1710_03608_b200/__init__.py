"""B200-native CTD-S / CTD-D hot path (arXiv 1710.03608) behind the reference's
proj/core entry points.  The compute lives in libctd_gpu.so (hand-written
sm_100a CUDA, C-ABI in include/ctd_gpu.h); this package is the host-side
mirror of the reference's ``ctd::`` interface.
"""
from .ctd import (ArgumentError, ColumnDistribution, Context, CtdError, DeviceError,  # noqa: F401
                  DeviceTensor, EmptyInputError, FiberBasis, LRFactors, Matricized,
                  MetricError, NumericError, ShapeError, SparseTensor, StreamState,
                  column_distribution, column_sq_norms, ctd_d_step, ctd_s,
                  core_drift, default_step_samples, init_stream, make_fiber_id, matricize,
                  memory_usage, relative_error, sample_with_replacement, unique_first_occurrence)

__version__ = "0.1.0"
