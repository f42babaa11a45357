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
#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "cdf.cuh"
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

// The same gram by columns of R: gram[a][k] = the sum over R_k's rows r
// ascending (the rows of the merge in transpose_times) of x_a[r] * R[r,k],
// with fiber a scattered densely into shared memory.  Rows of R_k absent from
// fiber a hold 0 there and are skipped (adding the product 0 * R[r,k] would
// not change the sum either).  A thread per (a, k): A x K_old independent
// sums instead of one CTA per appended fiber with a barrier per row.
__global__ void __launch_bounds__(256) k_gram_cols(const int32_t* fib, const int64_t* fptr, const int32_t* frow,
                                                   const double* fval, int dim, const int64_t* rptr,
                                                   const int32_t* rrow, const double* rval, int Kold,
                                                   double* gram) {
  extern __shared__ double xs[];  // [dim]
  const int a = blockIdx.y;
  const int f = fib[a];
  for (int r = threadIdx.x; r < dim; r += blockDim.x) xs[r] = 0.0;
  __syncthreads();
  for (int64_t t = fptr[f] + threadIdx.x; t < fptr[f + 1]; t += blockDim.x) xs[frow[t]] = fval[t];
  __syncthreads();
  const int k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= Kold) return;
  double acc = 0.0;
  for (int64_t e = rptr[k]; e < rptr[k + 1]; ++e) {
    const double x = xs[rrow[e]];
    if (x != 0.0) acc = dadd(acc, dmul(x, rval[e]));  // av[p] * bv[q], a = dR
  }
  gram[(long long)a * Kold + k] = fabs(acc) >= kDropTol ? acc : 0.0;
}

// Ordered compaction of each gram row's stored entries (j ascending): the
// chain product's inner loop visits only them.
__global__ void __launch_bounds__(256) k_gram_compact(const double* gram, int Kold, int32_t* nzj, double* nzg,
                                                      int* nzn) {
  __shared__ int s_warp[8];
  const int a = blockIdx.x;
  const double* g = gram + (long long)a * Kold;
  int base = 0;
  for (int j0 = 0; j0 < Kold; j0 += 256) {
    const int j = j0 + threadIdx.x;
    const double v = j < Kold ? g[j] : 0.0;
    const bool nz = v != 0.0;
    const unsigned bal = __ballot_sync(0xffffffffu, nz);
    if ((threadIdx.x & 31) == 0) s_warp[threadIdx.x >> 5] = __popc(bal);
    __syncthreads();
    int before = 0, all = 0;
    for (int w = 0; w < 8; ++w) {
      if (w < (int)(threadIdx.x >> 5)) before += s_warp[w];
      all += s_warp[w];
    }
    before += __popc(bal & ((1u << (threadIdx.x & 31)) - 1u));
    if (nz) {
      nzj[(long long)a * Kold + base + before] = j;
      nzg[(long long)a * Kold + base + before] = v;
    }
    base += all;
    __syncthreads();
  }
  if (threadIdx.x == 0) nzn[a] = base;
}

// left[a][c] over the compacted entries; blockIdx.x = a varies fastest so the
// CTAs of all appended rows stream through the same rows of U_old together
// (one HBM read of U_old, the other A-1 from L2).
__global__ void __launch_bounds__(256) k_left_nz(const int32_t* nzj, const double* nzg, const int* nzn, int Kold,
                                                 const double* uold, double* left) {
  const int a = blockIdx.x;
  const int c = blockIdx.y * blockDim.x + threadIdx.x;
  if (c >= Kold) return;
  const int n = nzn[a];
  const int32_t* jj = nzj + (long long)a * Kold;
  const double* gg = nzg + (long long)a * Kold;
  double acc = 0.0;
  int i = 0;
  for (; i + 4 <= n; i += 4) {
    const double u0 = uold[(long long)jj[i] * Kold + c], u1 = uold[(long long)jj[i + 1] * Kold + c];
    const double u2 = uold[(long long)jj[i + 2] * Kold + c], u3 = uold[(long long)jj[i + 3] * Kold + c];
    acc = dadd(acc, dmul(gg[i], u0));
    acc = dadd(acc, dmul(gg[i + 1], u1));
    acc = dadd(acc, dmul(gg[i + 2], u2));
    acc = dadd(acc, dmul(gg[i + 3], u3));
  }
  for (; i < n; ++i) acc = dadd(acc, dmul(gg[i], uold[(long long)jj[i] * Kold + c]));
  left[(long long)a * Kold + c] = acc;
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


// copy segment i (cnt[i] entries from sbeg[i]) to dbeg[i]; warp per segment
__global__ void k_copy_segs(const int64_t* sbeg, const int64_t* cnt, const int64_t* dbeg, long long nseg,
                            const int32_t* srow, const double* sval, int32_t* drow, double* dval) {
  const long long w = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (w >= nseg) return;
  const int64_t b = sbeg[w], n = cnt[w], d = dbeg[w];
  for (int64_t i = lane; i < n; i += 32) {
    drow[d + i] = srow[b + i];
    dval[d + i] = sval[b + i];
  }
}

// per column of a Core: the first entry with row >= K0 (rows ascend)
__global__ void k_split_rows(const int64_t* ptr, long long cols, const int32_t* row, int K0, int64_t* split) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= cols) return;
  int64_t lo = ptr[c], hi = ptr[c + 1];
  while (lo < hi) {
    const int64_t mid = (lo + hi) >> 1;
    if (row[mid] < K0) lo = mid + 1;
    else hi = mid;
  }
  split[c] = lo;
}

// core_drift terms of one column pair in the reference's merge order
// (ctd_dynamic.cpp:282-297); slots past the merged count hold 0 (adding 0 to
// a non-negative running sum changes nothing)
__global__ void k_drift_terms(const int64_t* ca, const int64_t* cb, long long n, const int64_t* aptr,
                              const int32_t* arow, const double* aval, const int64_t* bptr,
                              const int32_t* brow, const double* bval, const int64_t* toff, double* terms) {
  const long long u = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (u >= n) return;
  const int64_t ia = ca[u], ib = cb[u];
  int64_t p = ia >= 0 ? aptr[ia] : 0, pe = ia >= 0 ? aptr[ia + 1] : 0;
  int64_t q = ib >= 0 ? bptr[ib] : 0, qe = ib >= 0 ? bptr[ib + 1] : 0;
  int64_t o = toff[u];
  const int64_t oe = toff[u + 1];
  while (p < pe || q < qe) {
    double t;
    if (q == qe || (p < pe && arow[p] < brow[q])) {
      t = dmul(aval[p], aval[p]);
      ++p;
    } else if (p == pe || brow[q] < arow[p]) {
      t = dmul(bval[q], bval[q]);
      ++q;
    } else {
      const double d = dsub(aval[p], bval[q]);
      t = dmul(d, d);
      ++p;
      ++q;
    }
    terms[o++] = t;
  }
  while (o < oe) terms[o++] = 0.0;
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

void* CoreArena::take(Ctx* ctx, size_t bytes) {
  bytes = (bytes + 255) & ~size_t(255);
  static const bool trace = getenv("CTD_ARENA_TRACE") != nullptr;
  if (chunks.empty() || used + bytes > chunks.back().second) {
    // geometric growth: O(log) allocations over a long stream
    const size_t n = std::max({bytes, chunk_bytes, this->bytes() / 2});
    std::pair<char*, size_t> c{nullptr, 0};
    const auto t0 = std::chrono::steady_clock::now();
    if (next.valid()) {
      c = next.get();
      if (c.first && c.second < bytes) {
        cudaFree(c.first);
        c = {nullptr, 0};
      }
    }
    const bool pre = c.first != nullptr;
    if (!pre) {
      void* p = nullptr;
      CUDA_OK(cudaMalloc(&p, n));
      c = {static_cast<char*>(p), n};
    }
    if (trace)
      fprintf(stderr, "[arena] chunk %zu MB (%s) waited %.2f ms (%zu chunks)\n", c.second >> 20,
              pre ? "prefetched" : "inline",
              std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t0).count(),
              chunks.size() + 1);
    chunks.push_back(c);
    used = 0;
  }
  void* p = chunks.back().first + used;
  used += bytes;
  if (!next.valid() && used * 2 > chunks.back().second) {
    const size_t n2 = std::max(chunk_bytes, (this->bytes() + chunks.back().second) / 2);
    const int dev = ctx->device;
    next = std::async(std::launch::async, [n2, dev]() -> std::pair<char*, size_t> {
      cudaSetDevice(dev);
      void* q = nullptr;
      if (cudaMalloc(&q, n2) != cudaSuccess) {
        cudaGetLastError();  // this thread's error state only; take() allocates inline instead
        return {nullptr, 0};
      }
      return {static_cast<char*>(q), n2};
    });
  }
  return p;
}

void CoreArena::clear() {
  if (next.valid()) {
    auto c = next.get();
    if (c.first) cudaFree(c.first);
  }
  for (auto& c : chunks) cudaFree(c.first);
  chunks.clear();
  used = 0;
}

size_t CoreArena::bytes() const {
  size_t b = 0;
  for (const auto& c : chunks) b += c.second;
  return b;
}

// left = (dR^T R_old) U_old (A x Kold, row-major): the chain product's dense
// left factor (ctd_dynamic.cpp:234-246), dR = columns fib[0..A) of (fptr,
// frow, fval), R_old = B's first Kold columns.
void chain_left(Ctx* ctx, const int32_t* fib, int A, const int64_t* dptr, const int32_t* drow, const double* dval,
                const Basis& B, int64_t Kold, const double* uold, double* left) {
    Buf<double> gram(ctx, (size_t)A * Kold);
    const size_t xsmem = (size_t)B.dim * sizeof(double);
    if (xsmem <= 96 * 1024 && !getenv("CTD_CORE_LEGACY")) {
      if (xsmem > 48 * 1024)
        CUDA_OK(cudaFuncSetAttribute(k_gram_cols, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)xsmem));
      const dim3 grid(ceil_div((uint64_t)Kold, 256), A);
      LAUNCH(ctx, k_gram_cols, grid, 256, xsmem, fib, dptr, drow, dval, (int)B.dim, B.rptr.p, B.rrow.p,
             B.rval.p, (int)Kold, gram.p);
    } else {
      const size_t smem = (size_t)Kold * sizeof(double);
      if (smem > 200 * 1024) fail(CTD_ERR_ARGUMENT, "core update supports at most 25600 kept fibers");
      CUDA_OK(cudaFuncSetAttribute(k_gram_old, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      LAUNCH(ctx, k_gram_old, (unsigned)std::min(A, ctx->sm_count * 4), 256, smem, fib, A, dptr, drow, dval,
             B.rowbase.p, B.rowlen.p, B.rek.p, B.rev.p, (int)Kold, gram.p);
    }
    if (!getenv("CTD_CORE_LEGACY")) {
      Buf<int32_t> nzj(ctx, (size_t)A * Kold);
      Buf<double> nzg(ctx, (size_t)A * Kold);
      Buf<int> nzn(ctx, A);
      LAUNCH(ctx, k_gram_compact, A, 256, 0, gram.p, (int)Kold, nzj.p, nzg.p, nzn.p);
      const dim3 grid(A, ceil_div((uint64_t)Kold, 256));
      LAUNCH(ctx, k_left_nz, grid, 256, 0, nzj.p, nzg.p, nzn.p, (int)Kold, uold, left);
    } else {
      LAUNCH(ctx, k_left, ceil_div((uint64_t)A * Kold, 256), 256, 0, gram.p, A, (int)Kold, uold, left);
    }
}

void core_record(Ctx* ctx, const Fibers& fb, const Basis& B, int64_t Kold, const double* uold,
                 const std::vector<int32_t>& appended_fib, int64_t col_offset, CoreArena* arena,
                 CoreRecord& rec, bool dr_from_basis) {
  const int A = dr_from_basis ? (int)(B.K - Kold) : (int)appended_fib.size();
  rec.A = A;
  rec.Kold = Kold;
  rec.col_offset = col_offset;
  static const bool trace = getenv("CTD_CORE_TRACE") != nullptr;
  double tm[4] = {0, 0, 0, 0};
  auto lap = [&](int i) {
    if (!trace) return;
    static std::chrono::steady_clock::time_point t0;
    ctx->sync();
    const auto now = std::chrono::steady_clock::now();
    if (i >= 0) tm[i] = std::chrono::duration<double, std::milli>(now - t0).count();
    t0 = now;
  };
  lap(-1);
  // slab columns: R_new^T dX (top-right rows < K_old, bottom-right rows >= K_old)
  {
    Core sc;
    compute_core(ctx, fb, B, sc);
    lap(0);
    rec.cols = sc.cols;
    rec.nnz = sc.nnz;
    rec.col_id = std::move(sc.col_id);
    rec.ptr = std::move(sc.ptr);
    if (sc.nnz && arena) {
      int32_t* r = static_cast<int32_t*>(arena->take(ctx, sc.nnz * sizeof(int32_t)));
      double* v = static_cast<double*>(arena->take(ctx, sc.nnz * sizeof(double)));
      CUDA_OK(cudaMemcpyAsync(r, sc.row.p, sc.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
      CUDA_OK(cudaMemcpyAsync(v, sc.val.p, sc.nnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
      rec.row = r;
      rec.val = v;
    } else if (sc.nnz) {
      rec.own_sc = std::move(sc);
      rec.row = rec.own_sc.row.p;
      rec.val = rec.own_sc.val.p;
    }
    lap(1);
  }
  if (A > 0 && Kold > 0) {
    double* left;
    if (arena) {
      left = static_cast<double*>(arena->take(ctx, (size_t)A * Kold * sizeof(double)));
    } else {
      rec.own_left.alloc(ctx, (size_t)A * Kold);
      left = rec.own_left.p;
    }
    rec.left = left;
    Buf<int32_t> fib(ctx, A);
    // dR's columns: fibers of fb, or the basis's own columns Kold..K-1
    std::vector<int32_t> bcols;
    if (dr_from_basis)
      for (int a = 0; a < A; ++a) bcols.push_back((int32_t)(Kold + a));
    ctx->to_dev(fib.p, dr_from_basis ? bcols.data() : appended_fib.data(), A);
    const int64_t* dptr = dr_from_basis ? B.rptr.p : fb.ptr.p;
    const int32_t* drow = dr_from_basis ? B.rrow.p : fb.row.p;
    const double* dval = dr_from_basis ? B.rval.p : fb.val.p;
    chain_left(ctx, fib.p, A, dptr, drow, dval, B, Kold, uold, left);
    lap(2);
  }
  if (trace && tm[0] + tm[1] + tm[2] > 10.0)
    fprintf(stderr, "[core_record] K=%lld A=%d F=%lld nnz=%lld: compute_core %.2f copy %.2f gram+left %.2f ms\n",
            (long long)B.K, A, (long long)fb.F, (long long)rec.nnz, tm[0], tm[1], tm[2]);
}

void core_apply(Ctx* ctx, DevCore& core, const CoreRecord& rec) {
  const int A = rec.A;
  const int64_t Kold = rec.Kold;
  const long long oc = core.cols;
  // bottom-left counts over the old columns
  Buf<long long> blc(ctx, oc + 1);
  const unsigned wgrid = ceil_div((uint64_t)oc * 32, 256);
  if (A > 0 && Kold > 0 && oc > 0) {
    LAUNCH(ctx, k_bottom_left, wgrid, 256, 0, 0, core.ptr.p, core.row.p, core.val.p, oc, rec.left, A, (int)Kold,
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
  const long long nc = oc + rec.cols;
  std::vector<int64_t> nptr(nc + 1, 0), ncol(nc);
  for (long long c = 0; c < oc; ++c) nptr[c + 1] = nptr[c] + (optr[c + 1] - optr[c]) + hb[c];
  for (long long s = 0; s < rec.cols; ++s) nptr[oc + s + 1] = nptr[oc + s] + (rec.ptr[s + 1] - rec.ptr[s]);
  if (oc) ctx->to_host(ncol.data(), core.col.p, oc);
  ctx->sync();
  for (long long s = 0; s < rec.cols; ++s) ncol[oc + s] = rec.col_id[s] + rec.col_offset;
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
      LAUNCH(ctx, k_bottom_left, wgrid, 256, 0, 1, core.ptr.p, core.row.p, core.val.p, oc, rec.left, A, (int)Kold,
             (long long*)nullptr, nw.ptr.p, nw.row.p, nw.val.p);
  }
  if (rec.nnz) {
    const int64_t d = nptr[oc];
    CUDA_OK(cudaMemcpyAsync(nw.row.p + d, rec.row, rec.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_OK(cudaMemcpyAsync(nw.val.p + d, rec.val, rec.nnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ctx->sync();
  core = std::move(nw);
}

void core_step(Ctx* ctx, DevCore& core, const Fibers& fb, const Basis& B, int64_t Kold, const double* uold,
               const std::vector<int32_t>& appended_fib, int64_t col_offset, bool dr_from_basis) {
  CoreRecord rec;
  core_record(ctx, fb, B, Kold, uold, appended_fib, col_offset, nullptr, rec, dr_from_basis);
  core_apply(ctx, core, rec);
}

void core_step_exact(Ctx* ctx, DevCore& core, const Fibers& fb, const Fibers& hf, const Basis& B, int64_t Kold,
                     int64_t col_offset) {
  const long long oc = core.cols;
  Core sc;  // slab columns: R_new^T dX
  compute_core(ctx, fb, B, sc);
  // bottom-left: rows >= Kold of R_new^T X_hist (transpose_times(dR, X_hist)
  // entry by entry: the same merges and the same per-entry drop rule)
  Core full;
  std::vector<int64_t> split;
  if (B.K > Kold) {
    compute_core(ctx, hf, B, full);
    if (full.cols) {
      Buf<int64_t> dptr(ctx, full.cols + 1), dsplit(ctx, full.cols);
      ctx->to_dev(dptr.p, full.ptr.data(), full.cols + 1);
      LAUNCH(ctx, k_split_rows, ceil_div(full.cols, 256), 256, 0, dptr.p, (long long)full.cols, full.row.p,
             (int)Kold, dsplit.p);
      split.resize(full.cols);
      ctx->to_host(split.data(), dsplit.p, full.cols);
      ctx->sync();
    }
  }
  std::vector<int64_t> ocol(oc), optr(oc + 1, 0);
  if (oc) {
    ctx->to_host(ocol.data(), core.col.p, oc);
    ctx->to_host(optr.data(), core.ptr.p, oc + 1);
    ctx->sync();
  }
  // merged column list: old columns and bottom-left columns (ascending ids)
  std::vector<int64_t> ncol, nptr(1, 0), sbeg, scnt, dbeg;
  long long i = 0, j = 0;
  const long long fc = full.cols;
  auto bl_count = [&](long long c) { return full.ptr[c + 1] - split[c]; };
  while (i < oc || j < fc) {
    if (j < fc && bl_count(j) == 0) { ++j; continue; }
    const bool take_old = j == fc || (i < oc && ocol[i] <= full.col_id[j]);
    const bool take_bl = i == oc || (j < fc && full.col_id[j] <= ocol[i]);
    const int64_t cid = take_old ? ocol[i] : full.col_id[j];
    int64_t n = 0;
    if (take_old) n += optr[i + 1] - optr[i];
    if (take_bl) n += bl_count(j);
    ncol.push_back(cid);
    nptr.push_back(nptr.back() + n);
    if (take_old) {
      sbeg.push_back(optr[i]);
      scnt.push_back(optr[i + 1] - optr[i]);
      dbeg.push_back(nptr[nptr.size() - 2]);
      ++i;
    }
    if (take_bl) ++j;
  }
  const long long n_old_segs = (long long)sbeg.size();
  // bottom-left segments (sources in `full`)
  std::vector<int64_t> bsb, bcnt, bdb;
  {
    long long jj = 0;
    for (size_t c = 0; c < ncol.size(); ++c) {
      while (jj < fc && full.col_id[jj] < ncol[c]) ++jj;
      if (jj < fc && full.col_id[jj] == ncol[c] && bl_count(jj) > 0) {
        const int64_t olen = (nptr[c + 1] - nptr[c]) - bl_count(jj);
        bsb.push_back(split[jj]);
        bcnt.push_back(bl_count(jj));
        bdb.push_back(nptr[c] + olen);
      }
    }
  }
  const long long nmid = (long long)ncol.size();
  for (long long s2 = 0; s2 < sc.cols; ++s2) {
    ncol.push_back(sc.col_id[s2] + col_offset);
    nptr.push_back(nptr.back() + (sc.ptr[s2 + 1] - sc.ptr[s2]));
  }
  DevCore nw;
  nw.cols = (int64_t)ncol.size();
  nw.nnz = nptr.back();
  nw.col.alloc(ctx, nw.cols + 1);
  nw.ptr.alloc(ctx, nw.cols + 1);
  nw.row.alloc(ctx, nw.nnz + 1);
  nw.val.alloc(ctx, nw.nnz + 1);
  if (nw.cols) ctx->to_dev(nw.col.p, ncol.data(), nw.cols);
  ctx->to_dev(nw.ptr.p, nptr.data(), nw.cols + 1);
  auto copy = [&](const std::vector<int64_t>& sb, const std::vector<int64_t>& cn, const std::vector<int64_t>& db,
                  const int32_t* srow, const double* sval) {
    const long long ns = (long long)sb.size();
    if (!ns) return;
    Buf<int64_t> a(ctx, ns), b(ctx, ns), c(ctx, ns);
    ctx->to_dev(a.p, sb.data(), ns);
    ctx->to_dev(b.p, cn.data(), ns);
    ctx->to_dev(c.p, db.data(), ns);
    LAUNCH(ctx, k_copy_segs, ceil_div((uint64_t)ns * 32, 256), 256, 0, a.p, b.p, c.p, ns, srow, sval, nw.row.p,
           nw.val.p);
    ctx->sync();
  };
  if (n_old_segs) copy(sbeg, scnt, dbeg, core.row.p, core.val.p);
  if (!bsb.empty()) copy(bsb, bcnt, bdb, full.row.p, full.val.p);
  if (sc.nnz) {
    const int64_t d = nptr[nmid];
    CUDA_OK(cudaMemcpyAsync(nw.row.p + d, sc.row.p, sc.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
    CUDA_OK(cudaMemcpyAsync(nw.val.p + d, sc.val.p, sc.nnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
  }
  ctx->sync();
  core = std::move(nw);
}

double core_drift(Ctx* ctx, const DevCore& core, const Fibers& hf, const Basis& B) {
  Core ex;  // expected = R^T X_hist (transpose_times(R, matricize(history)))
  compute_core(ctx, hf, B, ex);
  const long long oc = core.cols, ec = ex.cols;
  std::vector<int64_t> ocol(oc), optr(oc + 1, 0);
  if (oc) {
    ctx->to_host(ocol.data(), core.col.p, oc);
    ctx->to_host(optr.data(), core.ptr.p, oc + 1);
    ctx->sync();
  }
  std::vector<int64_t> ca, cb, toff(1, 0);
  long long i = 0, j = 0;
  while (i < oc || j < ec) {
    const bool ta = j == ec || (i < oc && ocol[i] <= ex.col_id[j]);
    const bool tb = i == oc || (j < ec && ex.col_id[j] <= ocol[i]);
    int64_t n = 0;
    if (ta) n += optr[i + 1] - optr[i];
    if (tb) n += ex.ptr[j + 1] - ex.ptr[j];
    ca.push_back(ta ? i++ : -1);
    cb.push_back(tb ? j++ : -1);
    toff.push_back(toff.back() + n);
  }
  const long long nu = (long long)ca.size();
  const int64_t nt = toff.back();
  if (nt == 0) return 0.0;
  Buf<int64_t> dca(ctx, nu), dcb(ctx, nu), dto(ctx, nu + 1), dep(ctx, ec + 1);
  ctx->to_dev(dca.p, ca.data(), nu);
  ctx->to_dev(dcb.p, cb.data(), nu);
  ctx->to_dev(dto.p, toff.data(), nu + 1);
  ctx->to_dev(dep.p, ex.ptr.data(), ec + 1);
  Buf<double> terms(ctx, nt), cum(ctx, nt), tot(ctx, 1);
  const int32_t* erow = ex.nnz ? ex.row.p : nullptr;
  const double* eval = ex.nnz ? ex.val.p : nullptr;
  LAUNCH(ctx, k_drift_terms, ceil_div(nu, 128), 128, 0, dca.p, dcb.p, nu, core.ptr.p, core.row.p, core.val.p,
         dep.p, erow, eval, dto.p, terms.p);
  seq_cumsum(ctx, terms.p, nt, nullptr, tot.p);  // sq: the reference's sequential order, exactly
  double sq = 0.0;
  ctx->to_host(&sq, tot.p, 1);
  ctx->sync();
  ctx->check_flags("core_drift");
  return std::sqrt(sq);
}

}  // namespace ctdgpu

namespace ctdgpu {

void chain_product(Ctx* ctx, const Basis& B, const double* u, int A, const int64_t* dptr, const int32_t* drow,
                   const double* dval, const DevCore& core, Core& out) {
  const int64_t K = B.K;
  const long long oc = core.cols;
  out = Core{};
  out.rows = A;
  if (A == 0 || K == 0 || oc == 0) return;
  Buf<double> left(ctx, (size_t)A * K);
  std::vector<int32_t> f(A);
  for (int a = 0; a < A; ++a) f[a] = a;
  Buf<int32_t> fib(ctx, A);
  ctx->to_dev(fib.p, f.data(), A);
  chain_left(ctx, fib.p, A, dptr, drow, dval, B, K, u, left.p);
  // ((dR^T R) U) C column by column (ctd_dynamic.cpp:249-267): counts, then
  // the entries at their offsets (k_bottom_left writes row K + a at
  // nptr[w] + (column length) + rank, so nptr is shifted back by the length)
  Buf<long long> blc(ctx, oc + 1);
  const unsigned wgrid = ceil_div((uint64_t)oc * 32, 256);
  LAUNCH(ctx, k_bottom_left, wgrid, 256, 0, 0, core.ptr.p, core.row.p, core.val.p, oc, left.p, A, (int)K, blc.p,
         (const int64_t*)nullptr, (int32_t*)nullptr, (double*)nullptr);
  std::vector<long long> cnt(oc);
  std::vector<int64_t> optr(oc + 1);
  ctx->to_host(cnt.data(), blc.p, oc);
  ctx->to_host(optr.data(), core.ptr.p, oc + 1);
  ctx->sync();
  std::vector<int64_t> adj(oc + 1);
  int64_t tot = 0;
  out.ptr.push_back(0);
  for (long long w = 0; w < oc; ++w) {
    adj[w] = tot - (optr[w + 1] - optr[w]);
    if (cnt[w]) {
      out.col_id.push_back(w);
      out.ptr.push_back(tot + cnt[w]);
    }
    tot += cnt[w];
  }
  adj[oc] = tot;
  out.cols = (int64_t)out.col_id.size();
  out.nnz = tot;
  out.row.alloc(ctx, tot + 1);
  out.val.alloc(ctx, tot + 1);
  if (tot) {
    Buf<int64_t> nptr(ctx, oc + 1);
    ctx->to_dev(nptr.p, adj.data(), oc + 1);
    LAUNCH(ctx, k_bottom_left, wgrid, 256, 0, 1, core.ptr.p, core.row.p, core.val.p, oc, left.p, A, (int)K,
           (long long*)nullptr, nptr.p, out.row.p, out.val.p);
    ctx->sync();
  }
}

}  // namespace ctdgpu
