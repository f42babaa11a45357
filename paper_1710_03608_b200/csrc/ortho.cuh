#pragma once
#include "ctx.cuh"

namespace ctdgpu {

// FP64 GEMM on the tensor cores (mma.sync m8n8k4 .f64 -> DMMA on sm_100a):
//   C[M x N] = alpha * op(A) B + beta * C + gamma * I
// B is row-major [Kr x N] (ldb).  trans_a: A is stored [Kr x M] (lda) and
// op(A) = A^T (the Gram / SYRK shape, reduction over the long dimension);
// otherwise A is row-major [M x Kr].  C is row-major (ldc).  Deterministic:
// split-K partials are reduced in a fixed order.  abs_operands: |op(A)| |B|
// (the magnitudes rounding-error bounds are built from).
void gemm_f64(Ctx* ctx, bool trans_a, int64_t M, int64_t N, int64_t Kr, const double* A, int64_t lda,
              const double* B, int64_t ldb, double* C, int64_t ldc, double alpha, double beta, double gamma,
              bool abs_operands = false);

// |H - I|_F and |H|_F of a K x K matrix.
double frob_defect(Ctx* ctx, const double* H, int64_t K);
double frob_norm(Ctx* ctx, const double* H, int64_t K);

// Orthonormalizes the columns of A (n x K, row-major, lda) in place: A <- A
// (A^T A)^(-1/2), the polar factor, by the Newton-Schulz iteration with the
// third-order term, A <- A (I - E/2 + 3/8 E^2), E = A^T A - I (all products
// on DMMA).  The span is unchanged.  Returns the number of iterations and the
// final |A^T A - I|_F (before the last update) in *defect.  A is first scaled
// so that |A|_2 <= 1 when far from orthonormal, which makes the iteration
// converge for any full-rank A; fails with CTD_ERR_NUMERIC after max_iter.
int orthonormalize(Ctx* ctx, double* A, int64_t n, int64_t K, int64_t lda, double* defect, int max_iter = 80);

}  // namespace ctdgpu
