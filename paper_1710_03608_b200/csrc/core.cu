// compute_core (ctd_static.cpp:12-17): C = X x_alpha R^T through
// n_mode_product_impl -> multiply_columns(SparseMatrix, SparseMatrix)
// (tensor_ops.cpp:27-59, 90-102), kept in matricized CSC form
// C_(alpha) = R^T X_(alpha) over the nonempty columns of X_(alpha).
//
// Per column j of X_(alpha) the reference accumulates, for the column's rows r
// in ascending order and for every kept column k containing r (R^T's column
// r, ascending k), acc[k] += R[r,k] * x_rj, then emits the touched k with
// |acc[k]| >= 1e-14 (tensor_ops.hpp:13); the SparseMatrix constructor sorts
// the entries by (column, row).  One CTA per column: the rows are processed
// in order (a CTA barrier between rows), the k of one row in parallel, acc[k]
// in shared memory; so every C entry is the same sequence of fp64 operations
// as the reference's.  Two passes: count per column, then fill at the scanned
// offsets.
#include "core.cuh"

namespace ctdgpu {

namespace {

constexpr double kDropTolerance = 1e-14;  // tensor_ops.hpp:13
constexpr int kCoreThreads = 256;

__global__ void __launch_bounds__(kCoreThreads) k_core(int pass, const int64_t* fptr, const int32_t* frow,
                                                       const double* fval, long long F, const int64_t* rowbase,
                                                       const int32_t* rowlen, const int32_t* rek,
                                                       const double* rev, int K, long long* count,
                                                       const long long* off, int32_t* orow, double* oval) {
  extern __shared__ double acc[];  // [K]
  __shared__ int s_warp[kCoreThreads / 32];
  for (int k = threadIdx.x; k < K; k += blockDim.x) acc[k] = 0.0;
  __syncthreads();
  for (long long f = blockIdx.x; f < F; f += gridDim.x) {
    for (int64_t t = fptr[f]; t < fptr[f + 1]; ++t) {
      const int r = frow[t];
      const double x = fval[t];
      const int L = rowlen[r];
      const int64_t b = rowbase[r];
      for (int u = threadIdx.x; u < L; u += blockDim.x) {
        const int k = rek[b + u];
        acc[k] = dadd(acc[k], dmul(rev[b + u], x));  // mv[u] * xv[t] (tensor_ops.cpp:45)
      }
      __syncthreads();
    }
    // emit |acc[k]| >= tol in ascending k: block-wide running offset over K
    long long base = (pass == 1) ? off[f] : 0;
    long long total = 0;
    for (int k0 = 0; k0 < K; k0 += blockDim.x) {
      const int k = k0 + threadIdx.x;
      const double v = k < K ? acc[k] : 0.0;
      const bool keep = k < K && fabs(v) >= kDropTolerance;
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = __popc(bal);
      __syncthreads();
      int before = 0, all = 0;
      for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
        if (w < (int)(threadIdx.x >> 5)) before += s_warp[w];
        all += s_warp[w];
      }
      before += __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
      if (pass == 1 && keep) {
        orow[base + total + before] = k;
        oval[base + total + before] = v;
      }
      total += all;
      if (k < K) acc[k] = 0.0;
      __syncthreads();
    }
    if (pass == 0 && threadIdx.x == 0) count[f] = total;
  }
}

}  // namespace

void compute_core(Ctx* ctx, const Fibers& fb, const Basis& B, Core& out) {
  const long long F = fb.F;
  const int K = (int)B.K;
  out = Core{};
  out.rows = K;
  if (F == 0 || K == 0) return;
  const size_t smem = (size_t)K * sizeof(double);
  if (smem > 200 * 1024) fail(CTD_ERR_ARGUMENT, "core materialization supports at most 25600 kept fibers");
  CUDA_OK(cudaFuncSetAttribute(k_core, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const unsigned grid = (unsigned)std::min<long long>(F, (long long)ctx->sm_count * 4);
  Buf<long long> cnt(ctx, F), off(ctx, F + 1);
  LAUNCH(ctx, k_core, grid, kCoreThreads, smem, 0, fb.ptr.p, fb.row.p, fb.val.p, F, B.rowbase.p, B.rowlen.p,
         B.rek.p, B.rev.p, K, cnt.p, (const long long*)nullptr, (int32_t*)nullptr, (double*)nullptr);
  std::vector<long long> hc(F);
  std::vector<int64_t> hcol(F);
  ctx->to_host(hc.data(), cnt.p, F);
  ctx->to_host(hcol.data(), fb.col.p, F);
  ctx->sync();
  std::vector<long long> ho(F + 1, 0);
  for (long long f = 0; f < F; ++f) ho[f + 1] = ho[f] + hc[f];
  const long long nnz = ho[F];
  out.nnz = nnz;
  for (long long f = 0; f < F; ++f)
    if (hc[f] > 0) {
      out.col_id.push_back(hcol[f]);
      out.ptr.push_back(ho[f]);
    }
  out.ptr.push_back(nnz);
  out.cols = (int64_t)out.col_id.size();
  if (nnz == 0) return;
  out.row.alloc(ctx, nnz);
  out.val.alloc(ctx, nnz);
  ctx->to_dev(off.p, ho.data(), F + 1);
  LAUNCH(ctx, k_core, grid, kCoreThreads, smem, 1, fb.ptr.p, fb.row.p, fb.val.p, F, B.rowbase.p, B.rowlen.p,
         B.rek.p, B.rev.p, K, (long long*)nullptr, (const long long*)off.p, out.row.p, out.val.p);
  ctx->sync();
}

}  // namespace ctdgpu
