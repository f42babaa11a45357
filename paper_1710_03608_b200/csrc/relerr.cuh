#pragma once
#include "bucket.cuh"
#include "filter.cuh"

namespace ctdgpu {

// relative_error (evaluation.cpp:88-122) of the matricized tensor against the
// factors (R, U) with C = R^T X implied.
double relative_error(Ctx* ctx, const Fibers& fb, const Basis& B);

}  // namespace ctdgpu
