#pragma once
#include <vector>

#include "core.cuh"

namespace ctdgpu {

// The CTD-D stream's matricized core (StreamState::core, ctd_dynamic.hpp:18-39)
// as compressed CSC on the device: col[cols] global column ids ascending,
// ptr[cols+1], row[nnz] kept-fiber index ascending within a column, val[nnz].
struct DevCore {
  int64_t cols = 0, nnz = 0;
  Buf<int64_t> col, ptr;
  Buf<int32_t> row;
  Buf<double> val;
};

void core_from_static(Ctx* ctx, const Core& c, DevCore& out);

// One ctd_d_step core update (Eq. 13).  B is the basis after this step's
// appends, Kold its size before them and uold (Kold x Kold, row-major) U
// before them; appended_fib the appended candidates' fiber indices into fb in
// acceptance order; col_offset = t * slab_columns.
void core_step(Ctx* ctx, DevCore& core, const Fibers& fb, const Basis& B, int64_t Kold, const double* uold,
               const std::vector<int32_t>& appended_fib, int64_t col_offset);

}  // namespace ctdgpu
