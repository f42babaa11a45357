#pragma once
#include "ctx.cuh"

namespace ctdgpu {

// Raw outputs of std::mt19937_64(seed) (device).
void mt19937_64(Ctx* ctx, uint64_t seed, int64_t count, uint64_t* d_out);
// count draws: fiber index = upper_bound(cum[0..F), u_k).
void draw_fibers(Ctx* ctx, const double* cum, int64_t F, int64_t count, uint64_t seed,
                 int32_t* d_fibers);
// First-occurrence dedup of count ids; *d_n_unique (device) receives s'.
void dedup_first(Ctx* ctx, const int32_t* d_drawn, int64_t count, int32_t* d_unique,
                 int* d_n_unique);

// Same over an arbitrary cumulative array of n columns (int64 column ids).
void draw_columns(Ctx* ctx, const double* cum, int64_t n, int64_t count, uint64_t seed, int64_t* d_out);
// First-occurrence dedup of arbitrary int64 ids.
void dedup_first64(Ctx* ctx, const int64_t* d_in, int64_t count, int64_t* d_out, int* d_n_unique);

}  // namespace ctdgpu
