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

// exact_core variant (ctd_dynamic.cpp:207-211): the bottom-left block is
// dR^T X_hist (transpose_times over the retained history's matricization hf,
// columns in the core's time-extended space) instead of the chain product;
// it may add entries to columns that are empty in the old core.
void core_step_exact(Ctx* ctx, DevCore& core, const Fibers& fb, const Fibers& hf, const Basis& B, int64_t Kold,
                     int64_t col_offset);

// core_drift (ctd_dynamic.cpp:271-301): sqrt of the sequential sum, over the
// columns ascending and each column's merged rows, of (c - e)^2 / c^2 / e^2
// between the maintained core and R^T X_hist.
double core_drift(Ctx* ctx, const DevCore& core, const Fibers& hf, const Basis& B);

}  // namespace ctdgpu
