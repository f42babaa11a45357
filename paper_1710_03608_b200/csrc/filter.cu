// Linear-independence filter + U recurrence (FiberBasis::try_append_fiber,
// fiber_basis.cpp:43-109), replayed bit-exactly on the device.
//
// The loop over candidates is inherently sequential (each accept changes R
// and U), so it runs as ONE persistent cooperative kernel over all SMs with
// a software grid barrier between dependent phases.  Per candidate n:
//   P0 (if n-1 was accepted) U <- [[U + y y^T/d, -y/d], [-y^T/d, 1/d]]
//      elementwise over (K+1)^2 (fiber_basis.cpp:92-106); append x_{n-1} to R,
//      to R's row index and to the first-appearance row order.
//   P1 y = U g, one thread per row, each a sequential fl() chain in column
//      order (DenseMatrix::matvec, dense_matrix.cpp:42-47).  g = R^T x comes
//      from a Gram table precomputed in parallel before the loop: every g_k
//      is a sorted-merge dot product (gram_coeffs, fiber_basis.cpp:21-41)
//      whose only nonzero terms are the common rows in ascending order, so
//      a dense-lookup chain over c_k's rows adds exactly the same terms.
//   P2 z_r = sum_k y_k R[r,k] per row of R in ascending k (the reference's
//      scatter order, :56-65); the squared residual terms are laid out in the
//      reference's summation order: x's rows ascending, then R's rows in
//      first-touch order (:66-77).
//   P3 every CTA computes res^2 = the exact sequential sum of those terms
//      (seqsum.cuh) redundantly — no barrier needed after it — and takes the
//      decision sqrt(res^2) <= eps sqrt(|x|^2) (:79) and the delta guard
//      (:83-88).
// All arithmetic that restates the reference uses __dmul_rn/__dadd_rn/
// __ddiv_rn (no FMA), so kept fibers, delta and U are bit-identical.
#include <algorithm>
#include <cmath>

#include "filter.cuh"
#include "gridsum.cuh"
#include "radix.cuh"
#include "seqsum.cuh"

namespace ctdgpu {

Basis::Basis(Ctx* c, int64_t d) : ctx(c), dim(d) {
  rowbase.alloc(c, d + 1);
  rowbase.zero();
  rowlen.alloc(c, d + 1);
  rowlen.zero();
  sr_list.alloc(c, d + 1);
  sr_pos.alloc(c, d + 1);
  CUDA_OK(cudaMemsetAsync(sr_pos.p, 0xff, (d + 1) * sizeof(int32_t), c->stream));
  sr_n.alloc(c, 1);
  sr_n.zero();
  tag.alloc(c, d + 1);
  tag.zero();
  zd.alloc(c, 2 * (d + 1));
  kf.alloc(c, d + 1);
  rptr.alloc(c, 1);
  rptr.zero();
}

void basis_load(Basis& B, int64_t K, const int64_t* col_ptr, const int64_t* rows, const double* vals,
                const double* u) {
  Ctx* ctx = B.ctx;
  if (B.K != 0) fail(CTD_ERR_ARGUMENT, "basis_load needs an empty basis");
  const int64_t nnz = col_ptr[K], dim = B.dim;
  if (col_ptr[0] != 0 || nnz < 0) fail(CTD_ERR_ARGUMENT, "malformed column pointers");
  // R's CSC
  B.kcap = K;
  B.rptr.alloc(ctx, K + 1);
  ctx->to_dev(B.rptr.p, col_ptr, K + 1);
  std::vector<int32_t> r32(nnz > 0 ? nnz : 1);
  std::vector<int32_t> cnt(dim + 1, 0);
  for (int64_t k = 0; k < K; ++k) {
    if (col_ptr[k + 1] < col_ptr[k]) fail(CTD_ERR_ARGUMENT, "malformed column pointers");
    for (int64_t t = col_ptr[k]; t < col_ptr[k + 1]; ++t) {
      if (rows[t] < 0 || rows[t] >= dim) fail(CTD_ERR_SHAPE, "row index outside the fiber length");
      if (t > col_ptr[k] && rows[t] <= rows[t - 1]) fail(CTD_ERR_ARGUMENT, "rows must ascend within a column");
      r32[t] = (int32_t)rows[t];
      ++cnt[rows[t]];
    }
  }
  B.rcap = std::max<int64_t>(nnz, 1);
  B.rrow.alloc(ctx, B.rcap);
  B.rval.alloc(ctx, B.rcap);
  if (nnz) {
    ctx->to_dev(B.rrow.p, r32.data(), nnz);
    ctx->to_dev(B.rval.p, vals, nnz);
  }
  B.rnnz = nnz;
  // row index: per row, the columns containing it in ascending k
  std::vector<int64_t> base(dim + 1, 0);
  for (int64_t r = 0; r < dim; ++r) base[r + 1] = base[r] + ((cnt[r] + 3) & ~3);
  const int64_t ricap = base[dim] + 4;
  std::vector<int32_t> ek(ricap, 0), fill(dim, 0);
  std::vector<double> ev(ricap, 0.0);
  for (int64_t k = 0; k < K; ++k)
    for (int64_t t = col_ptr[k]; t < col_ptr[k + 1]; ++t) {
      const int64_t r = rows[t], p = base[r] + fill[r]++;
      ek[p] = (int32_t)k;
      ev[p] = vals[t];
    }
  B.ricap = ricap;
  B.rek.alloc(ctx, ricap);
  B.rev.alloc(ctx, ricap);
  ctx->to_dev(B.rek.p, ek.data(), ricap);
  ctx->to_dev(B.rev.p, ev.data(), ricap);
  ctx->to_dev(B.rowbase.p, base.data(), dim + 1);
  ctx->to_dev(B.rowlen.p, cnt.data(), dim);
  // U
  B.LD = (K + 2) & ~int64_t(1);
  if (u && K) {
    B.U.alloc(ctx, (size_t)B.LD * B.LD);
    CUDA_OK(cudaMemcpy2DAsync(B.U.p, B.LD * sizeof(double), u, K * sizeof(double), K * sizeof(double), K,
                              cudaMemcpyHostToDevice, ctx->stream));
  }
  B.K = K;
  ctx->sync();
}

namespace {

template <typename T>
__device__ __forceinline__ T ldg_cg(const T* p) { return __ldcg(p); }

// ---------------------------------------------------------------------------
// Preparation kernels.
__global__ void k_cand_stats(Cands c, long long* total_len) {
  long long s = 0;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < c.n;
       i += (long long)gridDim.x * blockDim.x)
    s += c.len[i];
  s = warp_sum(s);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd((unsigned long long*)total_len, (unsigned long long)s);
}

// per-row count of candidate entries (for row-index capacity)
__global__ void k_count_rows(Cands c, int32_t* cnt) {
  const long long cand = blockIdx.x;
  if (cand >= c.n) return;
  const long long off = c.off[cand];
  for (int t = threadIdx.x; t < c.len[cand]; t += blockDim.x) atomicAdd(&cnt[c.row[off + t]], 1);
}

__global__ void k_row_caps(const int32_t* rowlen, const int32_t* cnt, long long dim, long long* cap) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  // multiples of 4 entries: every row segment is 16-byte aligned for the
  // filter's bulk (TMA) copies, which may read up to 3 entries past the end
  if (r < dim) cap[r] = ((long long)rowlen[r] + cnt[r] + 3) & ~3ll;
}

__global__ void k_excl_scan_ll(const long long* in, long long n, long long* out) {
  __shared__ long long sh[33];
  long long carry = 0;
  for (long long b0 = 0; b0 < n; b0 += (long long)blockDim.x * 4) {
    long long v[4], s = 0;
    const long long base = b0 + (long long)threadIdx.x * 4;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      v[k] = (base + k < n) ? in[base + k] : 0;
      s += v[k];
    }
    long long tot;
    long long pre = block_excl_sum<long long>(s, sh, &tot) + carry;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      if (base + k < n) out[base + k] = pre;
      pre += v[k];
    }
    carry += tot;
  }
  if (threadIdx.x == 0) out[n] = carry;
}

__global__ void k_copy_rows(const long long* oldbase, const long long* newbase, const int32_t* rowlen,
                            const int32_t* ok, const double* ov, int32_t* nk, double* nv, long long dim) {
  // warp per row, lanes over its entries
  const long long r = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (r >= dim) return;
  const int lane = threadIdx.x & 31;
  const long long a = oldbase[r], b = newbase[r];
  const int L = rowlen[r];
  for (int t = lane; t < L; t += 32) {
    nk[b + t] = ok[a + t];
    nv[b + t] = ov[a + t];
  }
}

// W[:, col] = 0 (the panel's scratch column before a new batch: the last
// candidate of the previous batch may have left its residual there)
__global__ void k_zero_col(double* W, long long ld, long long dim, long long col) {
  const long long r = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (r < dim) W[r * ld + col] = 0.0;
}

__global__ void k_copy_u(const double* src, long long ld_src, double* dst, long long ld_dst, long long k) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= k * k) return;
  const long long i = e / k, j = e % k;
  dst[i * ld_dst + j] = src[i * ld_src + j];
}

// x_sq = SparseVec::squared_norm (sparse_matrix.cpp:10-14), exact sequential.
__global__ void __launch_bounds__(256) k_xsq(Cands c, double* xsq, unsigned* flags) {
  __shared__ SeqSumSmem S;
  const long long cand = blockIdx.x;
  if (cand >= c.n) return;
  const double* v = c.val + c.off[cand];
  auto get = [v](long long i) { return dsqr(v[i]); };
  bool bad = false;
  const double s = block_exact_sum(get, c.len[cand], S, &bad);
  if (threadIdx.x == 0) {
    xsq[cand] = s;
    if (bad) atomicOr(flags, FLAG_SEQSUM);
  }
}

// Dense candidate matrix D[row][cand] (dim x n), zeroed beforehand.
// The candidates as a dense table in 32-column chunks: D[(bc * dim + r) * 32 +
// (cand & 31)], bc = cand / 32, so one chunk (dim x 32 doubles) is contiguous
// and the Gram pass can keep it L2-resident while every left vector streams
// through it.
__global__ void k_dense_cands(Cands c, double* D, long long dim, const int32_t* pos) {
  const long long cand = blockIdx.x;
  if (cand >= c.n) return;
  const long long off = c.off[cand];
  const long long q = pos ? pos[cand] : cand;  // column of the table
  double* Dc = D + (q >> 5) * dim * 32 + (q & 31);
  for (int t = threadIdx.x; t < c.len[cand]; t += blockDim.x) Dc[(long long)c.row[off + t] * 32] = c.val[off + t];
}

// G[a][b] = merge-dot(left column a, candidate b) for b > a_min(a):
// sequential over the left column's rows ascending; D lookups are exactly 0
// off the common support, and adding fl(v*0) = +-0 never changes the sum.
__global__ void k_gram(const int64_t* lptr_off, const int32_t* llen, const int64_t* lptr, int use_ptr,
                       const int32_t* lrow, const double* lval, long long nleft, const double* D,
                       long long dim, long long n, long long bc0, long long nbc, const int32_t* perm, double* G) {
  // One warp per (left vector a, 32-column chunk bc of the table), lane =
  // column (candidate perm[j]).  g[a][b] is the sum over a's entries in order
  // (the reference's merge order) of x_a[r] * x_b[r]; loads run 4 entries
  // ahead of the add chain.
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long a = warp % nleft;
  const long long bc = bc0 + warp / nleft;
  if (bc >= bc0 + nbc) return;
  const int lane = threadIdx.x & 31;
  const long long j = bc * 32 + lane;  // table column
  long long off, len;
  if (use_ptr) {
    off = lptr[a];
    len = lptr[a + 1] - off;
  } else {
    off = lptr_off[a];
    len = llen[a];
  }
  const double* Dc = D + bc * dim * 32 + lane;
  double s = 0.0;
  long long t = 0;
  for (; t + 4 <= len; t += 4) {
    const int r0 = lrow[off + t], r1 = lrow[off + t + 1], r2 = lrow[off + t + 2], r3 = lrow[off + t + 3];
    const double x0 = lval[off + t], x1 = lval[off + t + 1], x2 = lval[off + t + 2], x3 = lval[off + t + 3];
    const double d0 = Dc[(long long)r0 * 32], d1 = Dc[(long long)r1 * 32];
    const double d2 = Dc[(long long)r2 * 32], d3 = Dc[(long long)r3 * 32];
    s = dadd(s, dmul(x0, d0));
    s = dadd(s, dmul(x1, d1));
    s = dadd(s, dmul(x2, d2));
    s = dadd(s, dmul(x3, d3));
  }
  for (; t < len; ++t) s = dadd(s, dmul(lval[off + t], Dc[(long long)lrow[off + t] * 32]));
  if (j < n) G[a * n + (perm ? perm[j] : j)] = s;
}

// The candidate Gram table g[a][b] (a < b), symmetric in its pair: the sum
// runs over the rows the two fibers share, ascending, of x_a[r] * x_b[r]
// (both merge orders of the reference visit the same rows in the same order,
// and rows present in one fiber only add +-0).  So each pair walks the
// SHORTER fiber: the candidates are ranked by length (perm: rank -> cand, the
// table's columns in rank order) and warp (i, chunk) walks candidate perm[i]
// against the 32 ranked columns j > i of the chunk.  The chain of a pair is
// min(len) long instead of len(a); warps start at the longest i.
__global__ void __launch_bounds__(256, 3) k_gram_sym(Cands c, const int32_t* perm, const double* D, long long dim, long long n,
                           long long nbw, double* G) {
  // Chunk-major: blockIdx.y picks a PAIR of 32-column chunks (the widest-ranked,
  // i.e. those with the most and longest partners, first) and blockIdx.x the
  // walked fibers i < their columns, longest first.  All resident warps then
  // gather from a few chunks (dim x 32 doubles each, 25.6 MB at C5), which
  // stay in L2, instead of sweeping the whole table per walked fiber.
  // The kernel is bound by L1 wavefronts / LSU write-back (ncu at C5: l1tex
  // 83-91 %, DRAM 9-14 %): a walked entry costs three write-back cycles for its
  // row and value however they reach the 32 lanes (uniform loads and shuffles
  // measured the same) plus two per 256-byte gather.  So a warp feeds TWO
  // chunks from one walk.
  const long long bc1 = nbw - 1 - 2 * (long long)blockIdx.y;  // upper chunk
  const long long bc0 = bc1 - 1;                              // lower chunk (absent when bc1 == 0)
  const long long ni = bc1 * 32 + 31 < n ? bc1 * 32 + 31 : n;  // i < the upper chunk's last column
  const long long i = ni - 1 - (((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  if (i < 0) return;
  const bool lower = bc0 >= 0 && i < bc0 * 32 + 31;  // the lower chunk has columns above i too
  const int lane = threadIdx.x & 31;
  const int a = perm[i];
  const long long off = c.off[a], len = c.len[a];
  const int32_t* __restrict__ cr = c.row + off;
  const double* __restrict__ cv = c.val + off;
  const double* D1 = D + bc1 * dim * 32 + lane;
  const double* D0 = lower ? D + bc0 * dim * 32 + lane : D1;
  double s1 = 0.0, s0 = 0.0;
  // 32 walked entries per round: lane u loads entry t + u (coalesced), and the
  // entries reach every lane in order by shuffles, eight gathers in flight per chunk
  for (long long t = 0; t < len; t += 32) {
    const int rem = (int)min(32ll, len - t);
    const int rl = lane < rem ? cr[t + lane] : 0;
    const double xl = lane < rem ? cv[t + lane] : 0.0;
    int u0 = 0;
    for (; u0 + 8 <= rem; u0 += 8) {
      int r[8];
      double x[8], d[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        r[u] = __shfl_sync(0xffffffffu, rl, u0 + u);
        x[u] = __shfl_sync(0xffffffffu, xl, u0 + u);
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) d[u] = D1[(long long)r[u] * 32];
      if (lower) {
        double e[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) e[u] = D0[(long long)r[u] * 32];
#pragma unroll
        for (int u = 0; u < 8; ++u) s0 = dadd(s0, dmul(x[u], e[u]));
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) s1 = dadd(s1, dmul(x[u], d[u]));
    }
    for (; u0 < rem; ++u0) {
      const long long r = (long long)__shfl_sync(0xffffffffu, rl, u0) * 32;
      const double x = __shfl_sync(0xffffffffu, xl, u0);
      s1 = dadd(s1, dmul(x, D1[r]));
      if (lower) s0 = dadd(s0, dmul(x, D0[r]));
    }
  }
  const long long j1 = bc1 * 32 + lane;
  if (j1 < n && j1 > i) {
    const long long b = perm[j1];
    const long long lo = a < b ? a : b, hi = a < b ? b : a;
    G[lo * n + hi] = s1;
  }
  const long long j0 = bc0 * 32 + lane;
  if (lower && j0 > i) {
    const long long b = perm[j0];
    const long long lo = a < b ? a : b, hi = a < b ? b : a;
    G[lo * n + hi] = s0;
  }
}

// ---------------------------------------------------------------------------
// The persistent filter kernel.
struct FArgs {
  int n_u;
  int K0;
  long long dim;
  long long LD;
  Cands c;
  const double* xsq;
  const double* Gc;  // [n_u][n_u] candidate x candidate (a < b)
  const double* Gb;  // [K0][n_u] basis x candidate
  double eps;
  double* U;
  int64_t* rptr;
  int32_t* rrow;
  double* rval;
  long long rnnz0;
  const int64_t* rowbase;
  int32_t* rowlen;
  int32_t* rek;
  double* rev;
  int32_t* sr_list;
  int32_t* sr_pos;
  int* sr_n;
  uint32_t* tag;
  uint32_t tag_base;
  double* zd;
  int32_t* kf;
  double* term;      // [dim]
  double* term2;     // [dim] slow-path ordered terms
  uint32_t* skey;    // [4*dim] slow-path sort scratch
  double* ybuf0;
  double* ybuf1;
  int* kept_cand;
  int* slow;         // [n_u] per-candidate slow-path flag
  int32_t* accepted;
  int32_t* degenerate;
  double* delta;
  double* res_out;
  double* y_last;
  long long* final_K;
  long long* final_rnnz;
  unsigned* bar;
  unsigned* flags;
  long long* trace;  // optional [n_u][kTraceW] clock64 stamps from CTA 0 (CTD_FILTER_TRACE)
  SliceSum* ssum;    // [grid] residual-sum slice summaries
  SliceDirect* sdir; // [grid * kSliceDirects]
  int* nfallback;    // exact-sum self-check failures (sequential fallback taken)
  double* gscr;      // [grid][LD+1] per-CTA g staging when K exceeds shared memory
  int kvec;          // largest K whose g / y vectors are staged in shared memory
  SliceLoc* sloc;    // [grid] published approximate slice sums (epoch-flagged)
  unsigned* sflag;   // [grid] slice-summary epoch flags
  double* W;         // optional [dim][Wld] orthonormal panel R T (error pass), column k written at accept k
  long long Wld;
  // resumable segments (speculative rejection batches, spec.cu)
  int n_begin;       // first candidate of this launch
  int Kstart;        // basis size at n_begin
  long long rnnz_start;
  int prev_n0;       // last exactly processed candidate before n_begin (a rejection), or -1
  int exit_run;      // return after this many consecutive rejections (0: never)
  int* next_out;     // first unprocessed candidate (n_u when done)
  long long* chk;    // [grid][2] checked builds: per-CTA (K, rnnz) after grid barrier 1
};

constexpr int kTraceW = 32;  // clock64 slots per candidate
constexpr int kSpecRun = 2;  // consecutive rejections that hand over to the batch certifier
__device__ __forceinline__ void stamp(long long* tr, int n, int k) {
  if (tr && blockIdx.x == 0 && threadIdx.x == 0) tr[(long long)n * kTraceW + k] = clock64();
}

#include "filter_kernel.cuh"

}  // namespace

void filter_batch(Basis& B, const Cands& c, double eps, BatchOut& out, bool want_y) {
  Ctx* ctx = B.ctx;
  const int64_t n = c.n;
  out = BatchOut{};
  if (n == 0) return;
  if (n >= (1ll << 31)) fail(CTD_ERR_ARGUMENT, "too many candidates");
  // ---- sizes
  ctx->phase_begin(PH_FILTER_PREP);
  Buf<long long> tl(ctx, 1);
  tl.zero();
  LAUNCH(ctx, k_cand_stats, std::min<unsigned>(ceil_div(n, 256), 1024), 256, 0, c, tl.p);
  const long long total_len = ctx->read1(tl.p);
  const int64_t K0 = B.K;
  // ---- capacities: U, R columns, R entries
  if (B.LD < K0 + n) {
    B.Wok = false;  // the panel follows U's capacity; rebuilt only from an empty basis
    B.W = Buf<double>();
    const int64_t nld = (std::max<int64_t>(K0 + n, B.LD * 2) + 1) & ~int64_t(1);  // even: 16-byte rows
    Buf<double> nu(ctx, (size_t)nld * nld);
    if (K0 > 0)
      LAUNCH(ctx, k_copy_u, ceil_div(K0 * K0, 256), 256, 0, B.U.p, (long long)B.LD, nu.p,
             (long long)nld, (long long)K0);
    B.U = std::move(nu);
    B.LD = nld;
  }
  if (B.kcap < K0 + n) {
    const int64_t nk = std::max<int64_t>(K0 + n, B.kcap * 2);
    Buf<int64_t> np(ctx, nk + 1);
    CUDA_OK(cudaMemcpyAsync(np.p, B.rptr.p, (K0 + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, ctx->stream));
    B.rptr = std::move(np);
    B.kcap = nk;
  }
  if (B.rcap < B.rnnz + total_len) {
    const int64_t nr = std::max<int64_t>(B.rnnz + total_len, B.rcap * 2);
    Buf<int32_t> nrow(ctx, nr);
    Buf<double> nval(ctx, nr);
    if (B.rnnz) {
      CUDA_OK(cudaMemcpyAsync(nrow.p, B.rrow.p, B.rnnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, ctx->stream));
      CUDA_OK(cudaMemcpyAsync(nval.p, B.rval.p, B.rnnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    }
    B.rrow = std::move(nrow);
    B.rval = std::move(nval);
    B.rcap = nr;
  }
  // ---- row index with room for every candidate entry
  {
    const long long dim = B.dim;
    Buf<int32_t> cnt(ctx, dim + 1);
    cnt.zero();
    LAUNCH(ctx, k_count_rows, (unsigned)n, 128, 0, c, cnt.p);
    Buf<int64_t> cap(ctx, dim + 1), nbase(ctx, dim + 1);
    LAUNCH(ctx, k_row_caps, ceil_div(dim, 256), 256, 0, B.rowlen.p, cnt.p, dim, (long long*)cap.p);
    LAUNCH(ctx, k_excl_scan_ll, 1, 1024, 0, (const long long*)cap.p, dim, (long long*)nbase.p);
    const int64_t ncap = B.rnnz + total_len + 3 * dim + 4;
    Buf<int32_t> nk(ctx, ncap);
    Buf<double> nv(ctx, ncap);
    if (B.rnnz)
      LAUNCH(ctx, k_copy_rows, ceil_div(dim * 32, 256), 256, 0, (const long long*)B.rowbase.p,
             (const long long*)nbase.p, B.rowlen.p, B.rek.p, B.rev.p, nk.p, nv.p, dim);
    B.rowbase = std::move(nbase);
    B.rek = std::move(nk);
    B.rev = std::move(nv);
    B.ricap = ncap;
  }
  // ---- per-candidate |x|^2, Gram tables
  Buf<double> xsq(ctx, n);
  LAUNCH(ctx, k_xsq, (unsigned)n, 256, 0, c, xsq.p, ctx->d_flags);
  // candidates ranked by length (stable): the Gram pairs walk the shorter fiber
  const long long nbw = (n + 31) / 32;
  std::vector<int32_t> hlen(n), perm(n), rank(n);
  ctx->to_host(hlen.data(), c.len, n);
  ctx->sync();
  for (int64_t q = 0; q < n; ++q) perm[q] = (int32_t)q;
  std::stable_sort(perm.begin(), perm.end(), [&](int32_t x, int32_t y) { return hlen[x] < hlen[y]; });
  for (int64_t q = 0; q < n; ++q) rank[perm[q]] = (int32_t)q;
  Buf<int32_t> dperm(ctx, n), drank(ctx, n);
  ctx->to_dev(dperm.p, perm.data(), n);
  ctx->to_dev(drank.p, rank.data(), n);
  Buf<double> D(ctx, (size_t)B.dim * nbw * 32);
  D.zero();
  LAUNCH(ctx, k_dense_cands, (unsigned)n, 128, 0, c, D.p, (long long)B.dim, (const int32_t*)drank.p);
  Buf<double> Gc(ctx, (size_t)n * n);
  LAUNCH(ctx, k_gram_sym, dim3(ceil_div(n * 32, 256), (unsigned)((nbw + 1) / 2)), 256, 0, c, (const int32_t*)dperm.p, D.p,
         (long long)B.dim, (long long)n, nbw, Gc.p);
  // kept fibers x candidates: warp (k, chunk of ranked columns)
  Buf<double> Gb(ctx, K0 > 0 ? (size_t)K0 * n : 1);
  if (K0 > 0)
    LAUNCH(ctx, k_gram, ceil_div(K0 * nbw * 32, 256), 256, 0, (const int64_t*)nullptr, (const int32_t*)nullptr,
           B.rptr.p, 1, B.rrow.p, B.rval.p, (long long)K0, D.p, (long long)B.dim, (long long)n, 0ll, nbw,
           (const int32_t*)dperm.p, Gb.p);
  D.reset();
  // ---- persistent kernel
  Buf<double> term(ctx, B.dim + 1), term2(ctx, B.dim + 1);
  Buf<uint32_t> skey(ctx, 4 * (B.dim + 1));
  Buf<double> y0(ctx, B.LD + 1), y1(ctx, B.LD + 1), ylast(ctx, B.LD + 1);
  Buf<int> kept(ctx, n), slow(ctx, n);
  slow.zero();
  Buf<int32_t> acc(ctx, n), deg(ctx, n);
  Buf<double> dl(ctx, n), res(ctx, n);
  Buf<long long> fK(ctx, 1), fR(ctx, 1);
  FArgs fa{};
  fa.n_u = (int)n;
  fa.K0 = (int)K0;
  fa.dim = B.dim;
  fa.LD = B.LD;
  // the orthonormal panel for the error pass (relerr.cu): started with an
  // empty basis, kept while U's capacity holds
  static const bool no_w = getenv("CTD_NO_WPANEL") != nullptr;  // the two-panel error pass only
  if (K0 == 0 && B.want_panel && !no_w && (double)B.dim * (double)B.LD * 8.0 <= kWPanelBytes) {
    B.W.alloc(ctx, (size_t)B.dim * B.LD);
    B.W.zero();
    B.Wok = true;
    B.Wscale.clear();
  }
  if (B.Wok) {
    fa.W = B.W.p;
    fa.Wld = B.LD;
    if (K0 > 0) LAUNCH(ctx, k_zero_col, ceil_div((uint64_t)B.dim, 256), 256, 0, B.W.p, (long long)B.LD, (long long)B.dim,
                       (long long)K0);
  }
  fa.c = c;
  fa.xsq = xsq.p;
  fa.Gc = Gc.p;
  fa.Gb = Gb.p;
  fa.eps = eps;
  fa.U = B.U.p;
  fa.rptr = B.rptr.p;
  fa.rrow = B.rrow.p;
  fa.rval = B.rval.p;
  fa.rnnz0 = B.rnnz;
  fa.rowbase = B.rowbase.p;
  fa.rowlen = B.rowlen.p;
  fa.rek = B.rek.p;
  fa.rev = B.rev.p;
  fa.sr_list = B.sr_list.p;
  fa.sr_pos = B.sr_pos.p;
  fa.sr_n = B.sr_n.p;
  fa.tag = B.tag.p;
  fa.tag_base = B.tag_base;
  fa.zd = B.zd.p;
  fa.kf = B.kf.p;
  fa.term = term.p;
  fa.term2 = term2.p;
  fa.skey = skey.p;
  fa.ybuf0 = y0.p;
  fa.ybuf1 = y1.p;
  fa.kept_cand = kept.p;
  fa.slow = slow.p;
  fa.accepted = acc.p;
  fa.degenerate = deg.p;
  fa.delta = dl.p;
  fa.res_out = res.p;
  fa.y_last = want_y ? ylast.p : nullptr;
  fa.final_K = fK.p;
  fa.final_rnnz = fR.p;
  fa.bar = ctx->d_bar;
  fa.flags = ctx->d_flags;
  Buf<SliceSum> ssum(ctx, ctx->sm_count);
  Buf<SliceDirect> sdir(ctx, (size_t)ctx->sm_count * kSliceDirects);
  fa.ssum = ssum.p;
  fa.sdir = sdir.p;
  Buf<double> gscr(ctx, (size_t)ctx->sm_count * (B.LD + 1));
  fa.gscr = gscr.p;
  // CTD_FILTER_KVEC (tests) lowers the shared-memory staging limit to exercise
  // the global-operand path at small K
  static const int kvec_env = getenv("CTD_FILTER_KVEC") ? atoi(getenv("CTD_FILTER_KVEC")) : 0;
  fa.kvec = (kvec_env > 0 && kvec_env < kVec) ? kvec_env : kVec;
  Buf<SliceLoc> sloc(ctx, ctx->sm_count);
  sloc.zero();
  Buf<unsigned> sflag(ctx, (size_t)ctx->sm_count * kFlagStride);
  sflag.zero();
  fa.sloc = sloc.p;
  fa.sflag = sflag.p;
  Buf<int> nfb(ctx, 1);
  nfb.zero();
  fa.nfallback = nfb.p;
  const char* trace_env = getenv("CTD_FILTER_TRACE");
  Buf<long long> tbuf;
  if (trace_env && *trace_env == '1') {
    tbuf.alloc(ctx, (size_t)n * kTraceW);
    tbuf.zero();
    tbuf.zero();
    fa.trace = tbuf.p;
  }
  ctx->zero(ctx->d_bar, 2 * sizeof(unsigned));
  int per_sm = 0;
  const size_t dsmem = kFilterSmem;
  static unsigned long long attr_done = 0;
  if (first_on_device(&attr_done, ctx->device))
    CUDA_OK(cudaFuncSetAttribute(k_filter, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)dsmem));
  CUDA_OK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_filter, kFThreads, dsmem));
  if (per_sm < 1) fail(CTD_ERR_DEVICE, "filter kernel cannot be resident");
  unsigned grid = (unsigned)ctx->sm_count;  // one CTA per SM
  if (const char* ge = getenv("CTD_FILTER_GRID")) {  // experiment hook: fewer CTAs
    const int gv = atoi(ge);
    if (gv > 0 && gv < (int)grid) grid = (unsigned)gv;
  }
  Buf<long long> chk(ctx, 2 * (size_t)grid);  // read only by checked builds
  fa.chk = chk.p;
  void* args[] = {&fa};
  // Exact kernel segments; after kSpecRun consecutive rejections the kernel
  // returns and the following candidates are certified in batches
  // (spec.cu) until one needs the exact path again.
  Buf<int> dnext(ctx, 1);
  fa.next_out = dnext.p;
  fa.n_begin = 0;
  fa.Kstart = (int)K0;
  fa.rnnz_start = B.rnnz;
  fa.prev_n0 = -1;
  static const bool no_spec = getenv("CTD_NO_SPEC") != nullptr;
  fa.exit_run = (!no_spec && !want_y && n > kSpecRun) ? kSpecRun : 0;
  int64_t spec_b = 64;
  ctx->phase_end();
  ctx->phase_begin(PH_FILTER);
  for (;;) {
    CUDA_OK(cudaLaunchCooperativeKernel((const void*)k_filter, dim3(grid), dim3(kFThreads), args, dsmem,
                                        ctx->stream));
    ctx->launches++;
    if (!fa.exit_run) break;
    int nx = 0;
    long long kk = 0, rr = 0;
    ctx->to_host(&nx, dnext.p, 1);
    ctx->to_host(&kk, fK.p, 1);
    ctx->to_host(&rr, fR.p, 1);
    ctx->sync();
    if (nx >= n) break;
    int64_t pos = nx;
    for (;;) {
      const int64_t L = spec_certify(B, c, xsq.p, Gb.p, Gc.p, kept.p, K0, kk, pos, spec_b, eps, acc.p, deg.p, dl.p,
                                     res.p);
      out.n_spec += L;
      pos += L;
      if (pos >= n) break;
      if (L < spec_b) {  // the next batch sized to the run just seen
        spec_b = std::min<int64_t>(4096, std::max<int64_t>(32, 2 * L + 32));
        break;
      }
      spec_b = std::min<int64_t>(spec_b * 2, 4096);
    }
    if (pos >= n) break;
    fa.n_begin = (int)pos;
    fa.Kstart = (int)kk;
    fa.rnnz_start = rr;
    fa.prev_n0 = nx - 1;
    ctx->zero(ctx->d_bar, 2 * sizeof(unsigned));
  }
  ctx->phase_end();
  // ---- results
  out.accepted.resize(n);
  out.degenerate.resize(n);
  out.delta.resize(n);
  out.res_sq.resize(n);
  out.x_sq.resize(n);
  std::vector<int> slowv(n);
  long long newK = 0, newR = 0;
  ctx->to_host(out.accepted.data(), acc.p, n);
  ctx->to_host(out.degenerate.data(), deg.p, n);
  ctx->to_host(out.delta.data(), dl.p, n);
  ctx->to_host(out.res_sq.data(), res.p, n);
  ctx->to_host(out.x_sq.data(), xsq.p, n);
  ctx->to_host(slowv.data(), slow.p, n);
  ctx->to_host(&newK, fK.p, 1);
  ctx->to_host(&newR, fR.p, 1);
  int srn = 0;
  ctx->to_host(&srn, B.sr_n.p, 1);
  if (want_y) {
    out.y_last.resize(K0 + n);
    ctx->to_host(out.y_last.data(), ylast.p, K0 + n);
  }
  ctx->sync();
  if (fa.trace) {
    std::vector<long long> tr((size_t)n * kTraceW);
    ctx->to_host(tr.data(), tbuf.p, (size_t)n * kTraceW);
    ctx->sync();
    const char* names[] = {"append", "stage", "rows", "bar1", "P2", "bar2", "tstage", "xsum", "decide"};
    double sum[9] = {0};
    for (int64_t i = 0; i < n; ++i)
      for (int k = 0; k < 9; ++k) sum[k] += (double)(tr[i * kTraceW + k + 1] - tr[i * kTraceW + k]);
    fprintf(stderr, "[filter trace] fallbacks=%d\n", ctx->read1(nfb.p));
    fprintf(stderr, "[filter trace] n=%lld cycles/candidate:", (long long)n);
    for (int k = 0; k < 9; ++k) fprintf(stderr, " %s=%.0f", names[k], sum[k] / n);
    fprintf(stderr, "\n");
    for (int64_t i = 0; i < n; i += std::max<int64_t>(1, n / 8)) {
      fprintf(stderr, "  cand %lld:", (long long)i);
      for (int k = 0; k < 9; ++k) fprintf(stderr, " %lld", tr[i * kTraceW + k + 1] - tr[i * kTraceW + k]);
      // P2 detail: staging, first row, remaining rows (CTA 0 warp 0)
      fprintf(stderr, " | P2: stage=%lld row0=%lld rest=%lld | P3: bar=%lld combine=%lld",
              tr[i * kTraceW + 10] - tr[i * kTraceW + 4], tr[i * kTraceW + 11] - tr[i * kTraceW + 10],
              tr[i * kTraceW + 5] - tr[i * kTraceW + 11], tr[i * kTraceW + 12] - tr[i * kTraceW + 7],
              tr[i * kTraceW + 8] - tr[i * kTraceW + 12]);
      fprintf(stderr, " | P1 cons-wait=%lld cons-chain=%lld", tr[i * kTraceW + 13], tr[i * kTraceW + 11]);
      // warp_grid_sum stages (CTA 0 lane 0), slots 16..26
      fprintf(stderr, " | P3:");
      for (int k = 17; k <= 24; ++k)
        if (tr[i * kTraceW + k] && tr[i * kTraceW + k - 1]) fprintf(stderr, " %lld", tr[i * kTraceW + k] - tr[i * kTraceW + k - 1]);
      fprintf(stderr, " directs=%lld | P1 prod wait=%lld compute=%lld probe=%lld", tr[i * kTraceW + 25],
              tr[i * kTraceW + 28], tr[i * kTraceW + 29], tr[i * kTraceW + 27]);
      fprintf(stderr, " | uncertified div=%lld", tr[i * kTraceW + 30]);
      fprintf(stderr, " | P2 chain wait=%lld work=%lld", tr[i * kTraceW + 26], tr[i * kTraceW + 27]);
      fprintf(stderr, " | P2 ring: setup=%lld chain=%lld steps=%lld groups=%lld", tr[i * kTraceW + 14] - tr[i * kTraceW + 10],
              tr[i * kTraceW + 15] - tr[i * kTraceW + 14], tr[i * kTraceW + 31] / 1000, tr[i * kTraceW + 31] % 1000);
      fprintf(stderr, "\n");
    }
  }
  ctx->check_flags("filter");
  int64_t k_at_last = K0;
  for (int64_t i = 0; i < n; ++i) {
    if (out.accepted[i]) out.kept_cand.push_back((int32_t)i);
    if (slowv[i]) out.slow_path = true;
    if (i < n - 1 && out.accepted[i]) ++k_at_last;
  }
  if (want_y) out.y_last.resize(k_at_last);
  if (B.Wok) {
    // W's columns hold the accepted candidates' residuals x - z; the error
    // pass weighs column k by 1/delta_k (W = R T, T's column (-y, 1)/sqrt(delta))
    B.Wscale.resize(K0);
    for (int64_t i = 0; i < n; ++i)
      if (out.accepted[i]) B.Wscale.push_back(1.0 / out.delta[i]);
    B.Wsc.alloc(ctx, B.Wscale.size() + 1);
    if (!B.Wscale.empty()) ctx->to_dev(B.Wsc.p, B.Wscale.data(), B.Wscale.size());
  }
  B.K = newK;
  B.rnnz = newR;
  B.srn = srn;
  B.tag_base += (uint32_t)n + 1u;
}

void basis_u(const Basis& B, double* u) {
  if (B.K == 0) return;
  CUDA_OK(cudaMemcpy2DAsync(u, B.K * sizeof(double), B.U.p, B.LD * sizeof(double), B.K * sizeof(double),
                            B.K, cudaMemcpyDeviceToHost, B.ctx->stream));
  B.ctx->sync();
}

void basis_r(const Basis& B, int64_t* col_ptr, int64_t* rows, double* vals) {
  Ctx* ctx = B.ctx;
  if (col_ptr) ctx->to_host(col_ptr, B.rptr.p, B.K + 1);
  if (rows && B.rnnz) {
    std::vector<int32_t> r(B.rnnz);
    ctx->to_host(r.data(), B.rrow.p, B.rnnz);
    ctx->sync();
    for (int64_t i = 0; i < B.rnnz; ++i) rows[i] = r[i];
  }
  if (vals) ctx->to_host(vals, B.rval.p, B.rnnz);
  ctx->sync();
}

}  // namespace ctdgpu
