// The CTD-D core update of ctd_d_step (ctd_dynamic.cpp:190-223), Eq. 13:
//
//   core(t+1) = [[ core(t),      R_old^T dX   ],      top-left / top-right
//                [ BL,           dR^T dX      ]]      bottom-left / bottom-right
//   BL = ((dR^T R_old) U_old) core(t)                 chain_product (:231-269)
//
// kept as a growing compressed CSC over the time-extended column space
// (column j of the slab at step t is global column j + t * slab_columns):
// old columns gain the bottom-left rows at their end (rows K_old.. ascending,
// the assembled SparseMatrix order of assemble_blocks, :18-50), the slab's
// columns are appended.  Every entry is the reference's sequence of fp64
// operations:
//   * top-right + bottom-right = R_new^T dX: compute_core's kernel on the slab
//     with the basis after the appends (transpose_times merges in ascending
//     row order with the product a*b, :58-83; the same as multiply_columns);
//   * dR^T R_old (the chain product's sparse Gram, drop rule applied) with the
//     same kernel on the appended fibers, restricted to k < K_old;
//   * left = gram U_old: per (a, c) the sum over gram's stored entries in
//     ascending j of gram[a,j] * U_old[j,c] (:244-249);
//   * BL[a, col] = sum over the column's entries (k ascending) of
//     left[a,k] * core[k,col] (:256-258), entries with |v| >= 1e-14 kept.
#include "stream_core.cuh"

namespace ctdgpu {

namespace {

constexpr double kDropTol = 1e-14;  // tensor_ops.hpp:13

// gram[a][k] (k < K_old) = dR_a^T R_k over the appended fibers; dropped
// entries are stored as 0 (they then contribute nothing to `left`).
__global__ void k_gram_old(const int32_t* fib, int A, const int64_t* fptr, const int32_t* frow, const double* fval,
                           const int64_t* rowbase, const int32_t* rowlen, const int32_t* rek, const double* rev,
                           int Kold, double* gram) {
  extern __shared__ double acc[];  // [Kold]
  for (int a = blockIdx.x; a < A; a += gridDim.x) {
    for (int k = threadIdx.x; k < Kold; k += blockDim.x) acc[k] = 0.0;
    __syncthreads();
    const int f = fib[a];
    for (int64_t t = fptr[f]; t < fptr[f + 1]; ++t) {
      const int r = frow[t];
      const double x = fval[t];
      const int L = rowlen[r];
      const int64_t b = rowbase[r];
      for (int u = threadIdx.x; u < L; u += blockDim.x) {
        const int k = rek[b + u];
        if (k < Kold) acc[k] = dadd(acc[k], dmul(x, rev[b + u]));  // av[p] * bv[q], a = dR
      }
      __syncthreads();
    }
    for (int k = threadIdx.x; k < Kold; k += blockDim.x) {
      const double v = acc[k];
      gram[(long long)a * Kold + k] = fabs(v) >= kDropTol ? v : 0.0;
    }
    __syncthreads();
  }
}

// left[a][c] = sum_{j: gram[a][j] != 0, ascending} gram[a][j] * U_old[j][c]
__global__ void k_left(const double* gram, int A, int Kold, const double* uold, double* left) {
  const long long id = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (id >= (long long)A * Kold) return;
  const int a = (int)(id / Kold), c = (int)(id - (long long)a * Kold);
  double acc = 0.0;
  for (int j = 0; j < Kold; ++j) {
    const double g = gram[(long long)a * Kold + j];
    if (g != 0.0) acc = dadd(acc, dmul(g, uold[(long long)j * Kold + c]));
  }
  left[id] = acc;
}

// Bottom-left block over the old core's columns: warp per column, lane a
// (chunks of 32 appended rows).  pass 0 counts kept entries per column; pass
// 1 writes them after the column's old entries in the assembled core.
__global__ void k_bottom_left(int pass, const int64_t* optr, const int32_t* orow, const double* oval, long long cols,
                              const double* left, int A, int Kold, long long* cnt, const int64_t* nptr,
                              int32_t* nrow, double* nval) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= cols) return;
  const int64_t b0 = optr[w], b1 = optr[w + 1];
  long long kept = 0;
  for (int a0 = 0; a0 < A; a0 += 32) {
    const int a = a0 + lane;
    double acc = 0.0;
    if (a < A)
      for (int64_t t = b0; t < b1; ++t) acc = dadd(acc, dmul(left[(long long)a * Kold + orow[t]], oval[t]));
    const bool keep = a < A && fabs(acc) >= kDropTol;
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    if (pass == 1 && keep) {
      const int64_t pos = nptr[w] + (b1 - b0) + kept + __popc(bal & ((1u << lane) - 1u));
      nrow[pos] = Kold + a;
      nval[pos] = acc;
    }
    kept += __popc(bal);
  }
  if (pass == 0 && lane == 0) cnt[w] = kept;
}

// copy each old column's entries to its new position
__global__ void k_copy_cols(const int64_t* optr, const int32_t* orow, const double* oval, long long cols,
                            const int64_t* nptr, int32_t* nrow, double* nval) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= cols) return;
  const int64_t b0 = optr[w], n = optr[w + 1] - b0, d = nptr[w];
  for (int64_t i = lane; i < n; i += 32) {
    nrow[d + i] = orow[b0 + i];
    nval[d + i] = oval[b0 + i];
  }
}

}  // namespace

void core_from_static(Ctx* ctx, const Core& c, DevCore& out) {
  out.cols = c.cols;
  out.nnz = c.nnz;
  out.col.alloc(ctx, c.cols + 1);
  out.ptr.alloc(ctx, c.cols + 1);
  if (c.cols) ctx->to_dev(out.col.p, c.col_id.data(), c.cols);
  ctx->to_dev(out.ptr.p, c.ptr.data(), c.cols + 1);
  out.row.alloc(ctx, c.nnz + 1);
  out.val.alloc(ctx, c.nnz + 1);
  if (c.nnz) {
    CUDA_OK(cudaMemcpyAsync(out.row.p, c.row.p, c.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_OK(cudaMemcpyAsync(out.val.p, c.val.p, c.nnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
}

void core_step(Ctx* ctx, DevCore& core, const Fibers& fb, const Basis& B, int64_t Kold, const double* uold,
               const std::vector<int32_t>& appended_fib, int64_t col_offset) {
  const int A = (int)appended_fib.size();
  const long long oc = core.cols;
  // slab columns: R_new^T dX (top-right rows < K_old, bottom-right rows >= K_old)
  Core sc;
  compute_core(ctx, fb, B, sc);
  // bottom-left counts over the old columns
  Buf<double> left(ctx, (size_t)A * Kold + 1);
  Buf<long long> blc(ctx, oc + 1);
  const unsigned wgrid = ceil_div((uint64_t)oc * 32, 256);
  if (A > 0 && Kold > 0 && oc > 0) {
    Buf<int32_t> fib(ctx, A);
    ctx->to_dev(fib.p, appended_fib.data(), A);
    Buf<double> gram(ctx, (size_t)A * Kold);
    const size_t smem = (size_t)Kold * sizeof(double);
    if (smem > 200 * 1024) fail(CTD_ERR_ARGUMENT, "core update supports at most 25600 kept fibers");
    CUDA_OK(cudaFuncSetAttribute(k_gram_old, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    LAUNCH(ctx, k_gram_old, (unsigned)std::min(A, ctx->sm_count * 4), 256, smem, fib.p, A, fb.ptr.p, fb.row.p,
           fb.val.p, B.rowbase.p, B.rowlen.p, B.rek.p, B.rev.p, (int)Kold, gram.p);
    LAUNCH(ctx, k_left, ceil_div((uint64_t)A * Kold, 256), 256, 0, gram.p, A, (int)Kold, uold, left.p);
    LAUNCH(ctx, k_bottom_left, wgrid, 256, 0, 0, core.ptr.p, core.row.p, core.val.p, oc, left.p, A, (int)Kold,
           blc.p, (const int64_t*)nullptr, (int32_t*)nullptr, (double*)nullptr);
  } else if (oc > 0) {
    CUDA_OK(cudaMemsetAsync(blc.p, 0, (oc + 1) * sizeof(long long), ctx->stream));
  }
  // new column pointers: old columns (old entries + bottom-left), then the slab's
  std::vector<int64_t> optr(oc + 1);
  std::vector<long long> hb(oc + 1, 0);
  if (oc) {
    ctx->to_host(optr.data(), core.ptr.p, oc + 1);
    ctx->to_host(hb.data(), blc.p, oc);
  } else {
    optr[0] = 0;
  }
  ctx->sync();
  const long long nc = oc + sc.cols;
  std::vector<int64_t> nptr(nc + 1, 0), ncol(nc);
  for (long long c = 0; c < oc; ++c) nptr[c + 1] = nptr[c] + (optr[c + 1] - optr[c]) + hb[c];
  for (long long s = 0; s < sc.cols; ++s) nptr[oc + s + 1] = nptr[oc + s] + (sc.ptr[s + 1] - sc.ptr[s]);
  if (oc) ctx->to_host(ncol.data(), core.col.p, oc);
  ctx->sync();
  for (long long s = 0; s < sc.cols; ++s) ncol[oc + s] = sc.col_id[s] + col_offset;
  DevCore nw;
  nw.cols = nc;
  nw.nnz = nptr[nc];
  nw.col.alloc(ctx, nc + 1);
  nw.ptr.alloc(ctx, nc + 1);
  nw.row.alloc(ctx, nw.nnz + 1);
  nw.val.alloc(ctx, nw.nnz + 1);
  if (nc) ctx->to_dev(nw.col.p, ncol.data(), nc);
  ctx->to_dev(nw.ptr.p, nptr.data(), nc + 1);
  if (oc) {
    LAUNCH(ctx, k_copy_cols, wgrid, 256, 0, core.ptr.p, core.row.p, core.val.p, oc, nw.ptr.p, nw.row.p, nw.val.p);
    if (A > 0 && Kold > 0)
      LAUNCH(ctx, k_bottom_left, wgrid, 256, 0, 1, core.ptr.p, core.row.p, core.val.p, oc, left.p, A, (int)Kold,
             (long long*)nullptr, nw.ptr.p, nw.row.p, nw.val.p);
  }
  if (sc.nnz) {
    const int64_t d = nptr[oc];
    CUDA_OK(cudaMemcpyAsync(nw.row.p + d, sc.row.p, sc.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_OK(cudaMemcpyAsync(nw.val.p + d, sc.val.p, sc.nnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ctx->sync();
  core = std::move(nw);
}

}  // namespace ctdgpu
