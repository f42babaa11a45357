#pragma once
#include "bucket.cuh"
#include "core.cuh"
#include "filter.cuh"

namespace ctdgpu {

// relative_error (evaluation.cpp:88-122) of the matricized tensor against the
// factors (R, U) with C = R^T X implied.
double relative_error(Ctx* ctx, const Fibers& fb, const Basis& B);

// relative_error against an explicit core (the CTD-D stream's C(t), which is
// not R^T X after chain-product substitutions): |X - (R U) C|^2 / |X|^2 column
// by column over the core's columns, the rest |x_j|^2 (evaluation.cpp:100-121).
double relative_error_core(Ctx* ctx, const Fibers& fb, const Basis& B, const Core& core);

// The two sums relative_error combines, over the fibers of fb (one shard of
// X in the sharded path): |X|^2 and sum_j |Q^T x_j|^2 (Q an orthonormal basis
// of span(R), ortho_panel), so rel = (|X|^2 - cross) / |X|^2 after summing
// the shards' partials.
void error_partials(Ctx* ctx, const Fibers& fb, const Basis& B, double* x_sq, double* cross);

// Q = (dim x K, leading dimension *ldq) orthonormal with span(Q) = span(R),
// built once per basis size (ortho.cu) and cached on the basis.
const double* ortho_panel(Ctx* ctx, const Basis& B, int64_t* ldq);

}  // namespace ctdgpu
