// FP64 tensor-core GEMM (DMMA) and the polar orthonormalization the error
// pass builds its projector from (relerr.cu).
//
// The reference evaluates |X - (R U) C|^2 column by column (evaluation.cpp:
// 88-122).  With Q an orthonormal basis of span(R) and S = Q^T R U R^T Q,
//   |x - R U R^T x|^2 = |x|^2 - |Q^T x|^2 + |(I - S) Q^T x|^2
// exactly, and I - S is similar to U G - I (G = R^T R), i.e. the inverse's
// backward error, so the last term is second order in it (~1e-16 and below
// on every config).  The pass therefore needs only |X|^2 - sum_j |Q^T x_j|^2,
// whose terms are sums of squares (no cancellation inside a fiber), where the
// identity |X|^2 - <X, R U R^T X> would carry U's first-order rounding
// (relerr.cu).  Q = A (A^T A)^(-1/2) from a near-orthonormal A
// spanning R: the filter's residual panel (W = R T, U = T T^T) when kept,
// else R with unit columns.  All the O(n K^2) work is GEMM on DMMA
// (mma.sync.m8n8k4.f64), the one place on the path large enough for tensor
// cores.
#include "ortho.cuh"

#include <cmath>
#include <cstdio>
#include <cstdlib>

namespace ctdgpu {

namespace {

constexpr int BM = 64, BN = 64, BK = 16, LDSM = BM + 8;  // +8: conflict-free fragment loads

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// One 64x64 tile of C per CTA (4 warps, 32x32 each = 4x4 DMMA fragments),
// K-slices of 16 double-buffered through shared memory.  blockIdx.z selects
// a split of the reduction range; with `partial` the raw sums go to
// C + z*M*N (ldc = N) for k_reduce_splits.
template <bool TA, bool ABS>
__global__ void __launch_bounds__(128) k_gemm(long long M, long long N, long long Kr, const double* __restrict__ A,
                                              long long lda, const double* __restrict__ B, long long ldb,
                                              double* __restrict__ C, long long ldc, long long kchunk, double alpha,
                                              double beta, double gamma, int partial) {
  __shared__ double As[2][BK][LDSM];
  __shared__ double Bs[2][BK][LDSM];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const long long m0 = (long long)blockIdx.y * BM, n0 = (long long)blockIdx.x * BN;
  const long long kbeg = (long long)blockIdx.z * kchunk;
  const long long kend = min(Kr, kbeg + kchunk);
  const int wm = (warp >> 1) * 32, wn = (warp & 1) * 32;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  double ra[8], rb[8];
  auto load = [&](long long k0) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 128 * i;
      if (TA) {
        const long long gk = k0 + (e >> 6), gm = m0 + (e & 63);
        ra[i] = (gk < kend && gm < M) ? A[gk * lda + gm] : 0.0;
      } else {
        const long long gm = m0 + (e >> 4), gk = k0 + (e & 15);
        ra[i] = (gk < kend && gm < M) ? A[gm * lda + gk] : 0.0;
      }
      const long long gk = k0 + (e >> 6), gn = n0 + (e & 63);
      rb[i] = (gk < kend && gn < N) ? B[gk * ldb + gn] : 0.0;
      if (ABS) {
        ra[i] = fabs(ra[i]);
        rb[i] = fabs(rb[i]);
      }
    }
  };
  auto store = [&](int buf) {
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int e = tid + 128 * i;
      if (TA) As[buf][e >> 6][e & 63] = ra[i];
      else As[buf][e & 15][e >> 4] = ra[i];
      Bs[buf][e >> 6][e & 63] = rb[i];
    }
  };
  int buf = 0;
  if (kbeg < kend) {
    load(kbeg);
    store(0);
  }
  __syncthreads();
  for (long long k0 = kbeg; k0 < kend; k0 += BK) {
    const bool more = k0 + BK < kend;
    if (more) load(k0 + BK);
#pragma unroll
    for (int kk = 0; kk < BK; kk += 4) {
      double a[4], b[4];
      const int kr = kk + (lane & 3);
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[buf][kr][wm + 8 * i + (lane >> 2)];
#pragma unroll
      for (int j = 0; j < 4; ++j) b[j] = Bs[buf][kr][wn + 8 * j + (lane >> 2)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma(acc[i][j], a[i], b[j]);
    }
    if (more) store(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const long long row = m0 + wm + 8 * i + (lane >> 2);
    if (row >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j)
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const long long col = n0 + wn + 8 * j + 2 * (lane & 3) + h;
        if (col >= N) continue;
        if (partial) {
          C[(long long)blockIdx.z * M * N + row * N + col] = acc[i][j][h];
        } else {
          double v = alpha * acc[i][j][h];
          if (beta != 0.0) v += beta * C[row * ldc + col];
          if (row == col) v += gamma;
          C[row * ldc + col] = v;
        }
      }
  }
}

__global__ void k_reduce_splits(const double* part, int splits, long long M, long long N, double* C, long long ldc,
                                double alpha, double beta, double gamma) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= M * N) return;
  const long long row = e / N, col = e - row * N;
  double s = 0.0;
  for (int z = 0; z < splits; ++z) s += part[(long long)z * M * N + e];
  double v = alpha * s;
  if (beta != 0.0) v += beta * C[row * ldc + col];
  if (row == col) v += gamma;
  C[row * ldc + col] = v;
}

// partial[b] = {sum (H - I)^2, sum H^2} over a grid-stride share of H (K x K).
__global__ void k_defect(const double* H, long long K, double* partial) {
  __shared__ double sh[33];
  double e = 0.0, h = 0.0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < K * K;
       t += (long long)gridDim.x * blockDim.x) {
    const long long r = t / K, c = t - r * K;
    const double v = H[t];
    const double d = (r == c) ? v - 1.0 : v;
    e = __fma_rn(d, d, e);
    h = __fma_rn(v, v, h);
  }
  e = block_sum<double>(e, sh);
  h = block_sum<double>(h, sh);
  if (threadIdx.x == 0) {
    partial[2 * blockIdx.x] = e;
    partial[2 * blockIdx.x + 1] = h;
  }
}

__global__ void k_defect_final(const double* partial, int nb, double* out) {
  __shared__ double sh[33];
  double e = 0.0, h = 0.0;
  for (int b = threadIdx.x; b < nb; b += blockDim.x) {
    e += partial[2 * b];
    h += partial[2 * b + 1];
  }
  e = block_sum<double>(e, sh);
  h = block_sum<double>(h, sh);
  if (threadIdx.x == 0) {
    out[0] = e;
    out[1] = h;
  }
}

// E = H - I (in place on T), and M += I - E/2 (M already holds 3/8 E^2 or 0).
__global__ void k_ns_coeffs(const double* H, long long K, double* E, double* Mx, int have_sq) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= K * K) return;
  const long long r = t / K, c = t - r * K;
  const double e = (r == c) ? H[t] - 1.0 : H[t];
  E[t] = e;
  const double m = (have_sq ? Mx[t] : 0.0) - 0.5 * e + ((r == c) ? 1.0 : 0.0);
  Mx[t] = m;
}

__global__ void k_scale_all(double* A, long long n, long long K, long long lda, double s) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const long long r = t / K, c = t - r * K;
  A[r * lda + c] *= s;
}

__global__ void k_copy_panel(const double* src, double* dst, long long n, long long K, long long lda) {
  const long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n * K) return;
  const long long r = t / K, c = t - r * K;
  dst[r * lda + c] = src[r * lda + c];
}

}  // namespace

void gemm_f64(Ctx* ctx, bool trans_a, int64_t M, int64_t N, int64_t Kr, const double* A, int64_t lda,
              const double* B, int64_t ldb, double* C, int64_t ldc, double alpha, double beta, double gamma,
              bool abs_operands) {
  if (M <= 0 || N <= 0) return;
  const int64_t tiles = ((M + BM - 1) / BM) * ((N + BN - 1) / BN);
  const int64_t want = (int64_t)ctx->sm_count * 4;
  int64_t splits = 1;
  if (tiles < want && Kr >= 8 * BK) {
    splits = std::min<int64_t>((want + tiles - 1) / tiles, 32);
    splits = std::min<int64_t>(splits, (Kr + 8 * BK - 1) / (8 * BK));
  }
  int64_t kchunk = (Kr + splits - 1) / splits;
  kchunk = (kchunk + BK - 1) / BK * BK;
  splits = std::max<int64_t>(1, (Kr + kchunk - 1) / std::max<int64_t>(kchunk, 1));
  const dim3 grid((unsigned)((N + BN - 1) / BN), (unsigned)((M + BM - 1) / BM), (unsigned)splits);
  Buf<double> part;
  double* out = C;
  long long ldo = ldc;
  if (splits > 1) {
    part.alloc(ctx, (size_t)splits * M * N);
    out = part.p;
    ldo = N;
  }
  const int is_part = splits > 1 ? 1 : 0;
  if (trans_a && !abs_operands)
    LAUNCH(ctx, (k_gemm<true, false>), grid, 128, 0, (long long)M, (long long)N, (long long)Kr, A, (long long)lda, B,
           (long long)ldb, out, ldo, (long long)kchunk, alpha, beta, gamma, is_part);
  else if (trans_a)
    LAUNCH(ctx, (k_gemm<true, true>), grid, 128, 0, (long long)M, (long long)N, (long long)Kr, A, (long long)lda, B,
           (long long)ldb, out, ldo, (long long)kchunk, alpha, beta, gamma, is_part);
  else if (!abs_operands)
    LAUNCH(ctx, (k_gemm<false, false>), grid, 128, 0, (long long)M, (long long)N, (long long)Kr, A, (long long)lda,
           B, (long long)ldb, out, ldo, (long long)kchunk, alpha, beta, gamma, is_part);
  else
    LAUNCH(ctx, (k_gemm<false, true>), grid, 128, 0, (long long)M, (long long)N, (long long)Kr, A, (long long)lda,
           B, (long long)ldb, out, ldo, (long long)kchunk, alpha, beta, gamma, is_part);
  if (splits > 1)
    LAUNCH(ctx, k_reduce_splits, ceil_div((uint64_t)M * N, 256), 256, 0, part.p, (int)splits, (long long)M,
           (long long)N, C, (long long)ldc, alpha, beta, gamma);
}

double frob_defect(Ctx* ctx, const double* H, int64_t K) {
  const unsigned nb = (unsigned)std::min<int64_t>(ctx->sm_count * 2, ceil_div((uint64_t)K * K, 256));
  Buf<double> dp(ctx, 2 * (size_t)nb), dv(ctx, 2);
  LAUNCH(ctx, k_defect, nb, 256, 0, H, (long long)K, dp.p);
  LAUNCH(ctx, k_defect_final, 1, 256, 0, dp.p, (int)nb, dv.p);
  double hv[2];
  ctx->to_host(hv, dv.p, 2);
  ctx->sync();
  return std::sqrt(hv[0]);
}

double frob_norm(Ctx* ctx, const double* H, int64_t K) {
  const unsigned nb = (unsigned)std::min<int64_t>(ctx->sm_count * 2, ceil_div((uint64_t)K * K, 256));
  Buf<double> dp(ctx, 2 * (size_t)nb), dv(ctx, 2);
  LAUNCH(ctx, k_defect, nb, 256, 0, H, (long long)K, dp.p);
  LAUNCH(ctx, k_defect_final, 1, 256, 0, dp.p, (int)nb, dv.p);
  double hv[2];
  ctx->to_host(hv, dv.p, 2);
  ctx->sync();
  return std::sqrt(hv[1]);
}

int orthonormalize(Ctx* ctx, double* A, int64_t n, int64_t K, int64_t lda, double* defect, int max_iter) {
  *defect = 0.0;
  if (K == 0 || n == 0) return 0;
  Buf<double> H(ctx, (size_t)K * K), E(ctx, (size_t)K * K), Mx(ctx, (size_t)K * K);
  Buf<double> A2(ctx, (size_t)n * lda);
  const unsigned nb = (unsigned)std::min<int64_t>(ctx->sm_count * 2, ceil_div((uint64_t)K * K, 256));
  Buf<double> dp(ctx, 2 * (size_t)nb), dv(ctx, 2);
  bool scaled = false;
  for (int it = 0; it < max_iter; ++it) {
    gemm_f64(ctx, true, K, K, n, A, lda, A, lda, H.p, K, 1.0, 0.0, 0.0);  // H = A^T A
    LAUNCH(ctx, k_defect, nb, 256, 0, H.p, (long long)K, dp.p);
    LAUNCH(ctx, k_defect_final, 1, 256, 0, dp.p, (int)nb, dv.p);
    double hv[2];
    ctx->to_host(hv, dv.p, 2);
    ctx->sync();
    const double e = std::sqrt(hv[0]);
    static const bool trace = getenv("CTD_ORTHO_TRACE") != nullptr;
    if (trace) fprintf(stderr, "[ortho] n=%lld K=%lld it=%d |A^T A - I|_F=%.3e |A^T A|_F=%.3e\n", (long long)n,
                       (long long)K, it, e, std::sqrt(hv[1]));
    if (!std::isfinite(e)) fail(CTD_ERR_NUMERIC, "orthonormalize: non-finite Gram matrix");
    if (!scaled && e > 0.5) {
      // |A|_2^2 <= |A^T A|_F: scale so every singular value is <= 1, where
      // sigma -> sigma p(sigma^2 - 1) increases monotonically to 1
      scaled = true;
      LAUNCH(ctx, k_scale_all, ceil_div((uint64_t)n * K, 256), 256, 0, A, (long long)n, (long long)K,
             (long long)lda, 1.0 / std::sqrt(std::sqrt(hv[1])));
      continue;
    }
    scaled = true;
    *defect = e;
    if (e < 1e-13) return it;  // orthonormal to rounding already
    const bool sq = e > 1e-8;  // the 3/8 E^2 term is below rounding under 1e-8
    if (sq) {
      LAUNCH(ctx, k_ns_coeffs, ceil_div((uint64_t)K * K, 256), 256, 0, H.p, (long long)K, E.p, Mx.p, 0);
      // Mx currently I - E/2; rebuild as 3/8 E^2 + I - E/2
      gemm_f64(ctx, false, K, K, K, E.p, K, E.p, K, Mx.p, K, 0.375, 1.0, 0.0);
    } else {
      LAUNCH(ctx, k_ns_coeffs, ceil_div((uint64_t)K * K, 256), 256, 0, H.p, (long long)K, E.p, Mx.p, 0);
    }
    gemm_f64(ctx, false, n, K, K, A, lda, Mx.p, K, A2.p, lda, 1.0, 0.0, 0.0);  // A2 = A M
    LAUNCH(ctx, k_copy_panel, ceil_div((uint64_t)n * K, 256), 256, 0, A2.p, A, (long long)n, (long long)K,
           (long long)lda);
    if (e < 1e-5) return it + 1;  // the defect after this step is O(e^3)
  }
  fail(CTD_ERR_NUMERIC, "orthonormalize: Newton-Schulz did not converge (rank-deficient R?)");
}

}  // namespace ctdgpu
