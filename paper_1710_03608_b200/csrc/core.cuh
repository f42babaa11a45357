#pragma once
#include <vector>

#include "bucket.cuh"
#include "filter.cuh"

namespace ctdgpu {

// C_(alpha) = R^T X_(alpha) (compute_core, ctd_static.cpp:12-17) as CSC over
// the columns of X_(alpha) that keep at least one entry: col_id[cols] their
// column ids j, ptr[cols+1] offsets (host); row[nnz] kept-column index k
// ascending within a column and val[nnz] (device).
struct Core {
  int64_t rows = 0, cols = 0, nnz = 0;
  std::vector<int64_t> col_id, ptr;
  Buf<int32_t> row;
  Buf<double> val;
};

void compute_core(Ctx* ctx, const Fibers& fb, const Basis& B, Core& out);

}  // namespace ctdgpu
