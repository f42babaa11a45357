#pragma once
#include "ctx.cuh"

namespace ctdgpu {

// Mode-`mode` matricization of a SparseTensor in compressed CSC form (only
// the F nonempty fibers), entries ordered by (column, row) exactly as the
// reference's SparseMatrix stores them (sparse_matrix.cpp:38-66), with the
// squared norm of every fiber summed in ascending-row order
// (tensor_ops.cpp:194-202).
struct Fibers {
  int64_t rows = 0;  // I_alpha
  int64_t cols = 0;  // N_alpha
  int64_t nnz = 0;
  int64_t F = 0;
  int mode = 0;
  Buf<int64_t> col;   // [F] column id j of each nonempty fiber
  Buf<int64_t> ptr;   // [F+1] offsets
  Buf<int32_t> row;   // [nnz]
  Buf<double> val;    // [nnz]
  Buf<double> norm;   // [F]
  bool integer_exact = false;  // all values integral, |v| <= 2^26, sum v^2 < 2^52
  double sum_sq = 0.0;         // sum of v^2 (any order; exact when integer_exact)
};

// Dispatches to matricize_onesweep (the stable LSD partition, for inputs
// whose rows ascend inside every column, i.e. any normalized SparseTensor)
// and falls back to the general bucket sort otherwise.
void matricize(Ctx* ctx, const Tensor& x, int mode, Fibers& out);
// Returns false (nothing usable in out) when the input's rows do not ascend
// inside a column; raises the usual input errors otherwise.
bool matricize_onesweep(Ctx* ctx, const Tensor& x, int mode, Fibers& out);
// column_sq_norms (tensor_ops.cpp:194-202) of fb's fibers into fb.norm, each
// summed in stored (ascending-row) order.
void fiber_norms(Ctx* ctx, Fibers& fb);

}  // namespace ctdgpu
