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

// probs[i] = fl(norms[i] / total) (sampling.cpp:29); *d_last_pos = the last
// i with probs[i] > 0, or -1.
void probs_from_norms(Ctx* ctx, const double* norms, int64_t F, const double* d_total, double* probs,
                      int* d_last_pos);
// cum[i] = 1.0 for i >= *d_last_pos (the tail clamp, sampling.cpp:54).
void clamp_from(Ctx* ctx, double* cum, int64_t n, const int* d_last_pos);

// Cumulative array of an arbitrary probability vector with the
// last-positive tail clamp (sampling.cpp:42-54).  FLAG_EMPTY if all zero.
void clamped_cdf(Ctx* ctx, const double* probs, int64_t n, double* cum, unsigned* d_flags);

}  // namespace ctdgpu
