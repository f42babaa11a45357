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
//
// A column with many rows makes that CTA a chain of dependent global loads
// per row (the long tail of a step).  Columns with more than kHeavyRows rows
// take the transposed walk instead (k_core_heavy): the column is scattered
// densely into shared memory and one thread per k sums, over R_k's rows
// ascending, x[r] * R[r,k] -- the same rows in the same order as the merge,
// since a row contributes to acc[k] exactly when it is in both R_k and the
// column (rows of R_k absent from the column hold 0 and are skipped).
#include <algorithm>
#include <cstdio>
#include <cstdlib>

#include "core.cuh"

namespace ctdgpu {

namespace {

constexpr double kDropTolerance = 1e-14;  // tensor_ops.hpp:13
constexpr int kCoreThreads = 256;
constexpr int kHeavyRows = 48;
constexpr int kMaxHeavy = 256;

__global__ void __launch_bounds__(kCoreThreads) k_core(int pass, const int64_t* fptr, const int32_t* frow,
                                                       const double* fval, long long F, const int64_t* rowbase,
                                                       const int32_t* rowlen, const int32_t* rek,
                                                       const double* rev, int K, long long* count,
                                                       const long long* off, int32_t* orow, double* oval,
                                                       int heavy_rows) {
  extern __shared__ double acc[];  // [K]
  __shared__ int s_warp[kCoreThreads / 32];
  for (int k = threadIdx.x; k < K; k += blockDim.x) acc[k] = 0.0;
  __syncthreads();
  for (long long f = blockIdx.x; f < F; f += gridDim.x) {
    if (heavy_rows > 0 && fptr[f + 1] - fptr[f] > heavy_rows) continue;  // k_core_heavy
    for (int64_t t = fptr[f]; t < fptr[f + 1]; ++t) {
      const int r = frow[t];
      const double x = fval[t];
      const int L = rowlen[r];
      const int64_t b = rowbase[r];
      for (int u = threadIdx.x; u < L; u += blockDim.x) {
        const int k = rek[b + u];
        CTD_CHECK(k >= 0 && k < K);
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

// Heavy columns: grid (ceil(K/256), n_heavy).  pass 0 stores the kept count
// of each (column, k-block); pass 1 writes at hoff[h][kb] (scanned).
__global__ void __launch_bounds__(kCoreThreads) k_core_heavy(int pass, const int64_t* hcols, int nkb,
                                                             const int64_t* fptr, const int32_t* frow,
                                                             const double* fval, int dim, const int64_t* rptr,
                                                             const int32_t* rrow, const double* rval, int K,
                                                             int* hcnt, const long long* hoff, int32_t* orow,
                                                             double* oval) {
  extern __shared__ double xs[];  // [dim]
  __shared__ int s_warp[kCoreThreads / 32];
  const int h = blockIdx.y;
  const long long f = hcols[h];
  for (int r = threadIdx.x; r < dim; r += blockDim.x) xs[r] = 0.0;
  __syncthreads();
  for (int64_t t = fptr[f] + threadIdx.x; t < fptr[f + 1]; t += blockDim.x) xs[frow[t]] = fval[t];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (k < K)
    for (int64_t e = rptr[k]; e < rptr[k + 1]; ++e) {
      const double x = xs[rrow[e]];
      if (x != 0.0) acc = dadd(acc, dmul(rval[e], x));  // mv[u] * xv[t]
    }
  const bool keep = k < K && fabs(acc) >= kDropTolerance;
  const unsigned bal = __ballot_sync(0xffffffffu, keep);
  if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = __popc(bal);
  __syncthreads();
  int before = 0, all = 0;
  for (int w = 0; w < (int)(blockDim.x >> 5); ++w) {
    if (w < (int)(threadIdx.x >> 5)) before += s_warp[w];
    all += s_warp[w];
  }
  before += __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
  if (pass == 0) {
    if (threadIdx.x == 0) hcnt[(long long)h * nkb + blockIdx.x] = all;
  } else if (keep) {
    const long long o = hoff[(long long)h * nkb + blockIdx.x] + before;
    orow[o] = k;
    oval[o] = acc;
  }
}

__global__ void k_heavy_list(const int64_t* fptr, long long F, int heavy_rows, int64_t* hcols, int* nh) {
  const long long f = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (f < F && fptr[f + 1] - fptr[f] > heavy_rows) hcols[atomicAdd(nh, 1)] = f;
}

// per heavy column: its total into count[f] (pass 0 follow-up), or the
// per-k-block write offsets from off[f] (pass 1)
__global__ void k_heavy_scan(int pass, const int64_t* hcols, int nh, int nkb, const int* hcnt, long long* count,
                             const long long* off, long long* hoff) {
  const int h = blockIdx.x * blockDim.x + threadIdx.x;
  if (h >= nh) return;
  const long long f = hcols[h];
  long long run = pass == 0 ? 0 : off[f];
  for (int b = 0; b < nkb; ++b) {
    if (pass == 1) hoff[(long long)h * nkb + b] = run;
    run += hcnt[(long long)h * nkb + b];
  }
  if (pass == 0) count[f] = run;
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
  // heavy columns (transposed walk) when the column fits in shared memory
  const size_t xsmem = (size_t)B.dim * sizeof(double);
  const bool heavy = xsmem <= 96 * 1024 && B.rptr.p && !getenv("CTD_CORE_LEGACY");
  const char* hr_env = getenv("CTD_CORE_HEAVY_ROWS");  // tests: move the path split
  int heavy_rows = heavy ? (hr_env ? std::max(1, atoi(hr_env)) : kHeavyRows) : 0;
  const int nkb = (int)ceil_div((uint64_t)K, kCoreThreads);
  int nh = 0;
  Buf<int64_t> hcols;
  Buf<int> hcnt;
  if (heavy) {
    // the transposed walk costs nnz(R) per column: keep it to the longest few
    Buf<int> d_nh(ctx, 1);
    hcols.alloc(ctx, F);
    for (;;) {
      d_nh.zero();
      LAUNCH(ctx, k_heavy_list, ceil_div((uint64_t)F, 256), 256, 0, fb.ptr.p, F, heavy_rows, hcols.p, d_nh.p);
      ctx->to_host(&nh, d_nh.p, 1);
      ctx->sync();
      if (nh <= kMaxHeavy) break;
      heavy_rows *= 2;
    }
    if (getenv("CTD_CORE_TRACE")) fprintf(stderr, "[compute_core] F=%lld K=%d heavy: %d columns > %d rows\n", F, K, nh, heavy_rows);
    if (nh) {
      if (xsmem > 48 * 1024)
        CUDA_OK(cudaFuncSetAttribute(k_core_heavy, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem));
      hcnt.alloc(ctx, (size_t)nh * nkb);
      LAUNCH(ctx, k_core_heavy, dim3(nkb, nh), kCoreThreads, xsmem, 0, hcols.p, nkb, fb.ptr.p, fb.row.p, fb.val.p,
             (int)B.dim, B.rptr.p, B.rrow.p, B.rval.p, K, hcnt.p, (const long long*)nullptr, (int32_t*)nullptr,
             (double*)nullptr);
    }
  }
  LAUNCH(ctx, k_core, grid, kCoreThreads, smem, 0, fb.ptr.p, fb.row.p, fb.val.p, F, B.rowbase.p, B.rowlen.p,
         B.rek.p, B.rev.p, K, cnt.p, (const long long*)nullptr, (int32_t*)nullptr, (double*)nullptr, heavy_rows);
  if (nh)
    LAUNCH(ctx, k_heavy_scan, ceil_div((uint64_t)nh, 128), 128, 0, 0, hcols.p, nh, nkb, hcnt.p, cnt.p,
           (const long long*)nullptr, (long long*)nullptr);
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
         B.rek.p, B.rev.p, K, (long long*)nullptr, (const long long*)off.p, out.row.p, out.val.p, heavy_rows);
  if (nh) {
    Buf<long long> hoff(ctx, (size_t)nh * nkb);
    LAUNCH(ctx, k_heavy_scan, ceil_div((uint64_t)nh, 128), 128, 0, 1, hcols.p, nh, nkb, hcnt.p, (long long*)nullptr,
           (const long long*)off.p, hoff.p);
    LAUNCH(ctx, k_core_heavy, dim3(nkb, nh), kCoreThreads, xsmem, 1, hcols.p, nkb, fb.ptr.p, fb.row.p, fb.val.p,
           (int)B.dim, B.rptr.p, B.rrow.p, B.rval.p, K, (int*)nullptr, (const long long*)hoff.p, out.row.p,
           out.val.p);
  }
  ctx->sync();
}

}  // namespace ctdgpu
