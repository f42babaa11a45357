#pragma once
#include "ctx.cuh"

namespace ctdgpu {

// cum[i] = fl(cum[i-1] + x[i]) (sequential order, bit-exact), x[i] >= 0.
// cum may be null (total only).  *d_total (device) receives the last value.
void seq_cumsum(Ctx* ctx, const double* x, int64_t n, double* cum, double* d_total);

// column_distribution + the clamped cumulative array of
// sample_with_replacement over F nonempty fibers with squared norms `norms`.
void sampling_law(Ctx* ctx, const double* norms, int64_t F, double* d_total, double* probs,
                  double* cum, unsigned* d_flags);

// Cumulative array of an arbitrary probability vector with the
// last-positive tail clamp (sampling.cpp:42-54).  FLAG_EMPTY if all zero.
void clamped_cdf(Ctx* ctx, const double* probs, int64_t n, double* cum, unsigned* d_flags);

}  // namespace ctdgpu
