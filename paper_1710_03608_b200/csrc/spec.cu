// Speculative rejection batches for the independence filter.
//
// try_append_fiber (fiber_basis.cpp:43-109) is sequential because every
// accept changes R and U; a rejection changes nothing.  When the persistent
// filter kernel sees a run of rejections (the basis has saturated, as at C4
// after K = I_alpha, or a CTD-D slab adds little), it returns, and the next b
// candidates are evaluated together against the unchanged (R, U) -- in the
// reference's own operation order, so every y and z below is bit-identical to
// what try_append_fiber computes for that candidate:
//   g_c  the exact Gram table (gram_coeffs, fiber_basis.cpp:21-41),
//   y_c = U g_c, one sequential fl() chain per (row, candidate) in column
//        order (DenseMatrix::matvec, dense_matrix.cpp:42-47),
//   z_c = R y_c, per (row of R, candidate) a chain over the row's kept
//        columns in ascending k, skipping y_k == 0 (fiber_basis.cpp:56-65),
// and the residual terms fl((x_r - z_r)^2) / fl(z_r^2) are those the
// reference sums (:66-77).  Only their ORDER of summation differs, so for
// non-negative terms |res_ref - res| <= 2 gamma_n res, and a candidate is
// certified rejected when even res (1 + 2 gamma_n) clears the threshold
// sqrt(res) <= eps sqrt(|x|^2) (:79) with a few ulps to spare.  Certified
// rejections are exactly what the reference decides (accepted = degenerate =
// 0, delta = 0; the residual is a diagnostic); the first candidate that is not
// certified goes back to the exact kernel.
#include "filter.cuh"

namespace ctdgpu {

namespace {

// G[k][c] = g_k of candidate pos + c: the Gram table entries the exact
// kernel reads (basis columns k < K0 from Gb, appended candidates from Gc).
__global__ void k_spec_g(double* G, long long b, long long K, long long K0, long long nu, long long pos,
                         const double* Gb, const double* Gc, const int* kept_cand) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K * b) return;
  const long long k = e / b, c = e - k * b;
  const long long n = pos + c;
  double g = 0.0;
  if (n < nu) g = (k < K0) ? Gb[k * nu + n] : Gc[(long long)kept_cand[k - K0] * nu + n];
  G[e] = g;
}

// Xd[r][c] = x_{pos+c}[r] (Xd zeroed).
__global__ void k_spec_dense_x(Cands c, long long pos, long long b, double* Xd) {
  const long long j = blockIdx.x;
  if (j >= b || pos + j >= c.n) return;
  const long long off = c.off[pos + j];
  for (int t = threadIdx.x; t < c.len[pos + j]; t += blockDim.x) Xd[(long long)c.row[off + t] * b + j] = c.val[off + t];
}

// y[i][c] = U[i][:] . g_c as the reference's matvec chain (warp per row i
// and 32 candidates; U's row is a broadcast, G's row coalesced).
__global__ void k_spec_y(const double* U, long long LD, long long K, const double* G, long long b, double* Y) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nch = (b + 31) >> 5;
  const long long i = warp / nch;
  if (i >= K) return;
  const long long c = (warp - i * nch) * 32 + (threadIdx.x & 31);
  const bool act = c < b;
  const double* ur = U + i * LD;
  double s = 0.0;
  long long j = 0;
  for (; j + 8 <= K; j += 8) {
    double p[8];
#pragma unroll
    for (int u = 0; u < 8; ++u) p[u] = dmul(__ldg(ur + j + u), act ? G[(j + u) * b + c] : 0.0);
#pragma unroll
    for (int u = 0; u < 8; ++u) s = dadd(s, p[u]);
  }
  for (; j < K; ++j) s = dadd(s, dmul(__ldg(ur + j), act ? G[j * b + c] : 0.0));
  if (act) Y[i * b + c] = s;
}

// Warp per row r, lanes across candidates: z_r in the reference's scatter
// order, then the row's residual term, summed per candidate (order-free:
// the terms are >= 0 and exact; the bound in k_spec_decide covers the order).
__global__ void k_spec_res(long long dim, long long b, const int64_t* rowbase, const int32_t* rowlen,
                           const int32_t* rek, const double* rev, const double* Y, const double* Xd, double* res) {
  const long long warp = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const long long nw = ((long long)gridDim.x * blockDim.x) >> 5;
  const int lane = threadIdx.x & 31;
  for (long long c0 = 0; c0 < b; c0 += 32) {
    const long long c = c0 + lane;
    const bool act = c < b;
    double rs = 0.0;
    for (long long r = warp; r < dim; r += nw) {
      const long long base = rowbase[r];
      const int L = rowlen[r];
      double z = 0.0;
      for (int t = 0; t < L; ++t) {
        const double yk = act ? Y[(long long)rek[base + t] * b + c] : 0.0;
        if (yk != 0.0) z = dadd(z, dmul(yk, rev[base + t]));
      }
      if (act) {
        const double x = Xd[r * b + c];  // stored values are never 0: x != 0 <=> r in supp(x)
        rs += (x != 0.0) ? dsqr(dsub(x, z)) : dsqr(z);
      }
    }
    if (act && rs != 0.0) atomicAdd(&res[c], rs);
  }
}

__global__ void k_spec_decide(long long b, long long pos, long long nu, const double* res, const double* xsq,
                              double eps, double grow, int* cert) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= b) return;
  if (pos + c >= nu) {
    cert[c] = 0;
    return;
  }
  // res_ref <= res * grow; sqrt and the product eps * sqrt(|x|^2) round by
  // at most an ulp each: keep 8 ulps of room
  const double lhs = sqrt(res[c] * grow) * (1.0 + 8.0 * 1.1102230246251565e-16);
  const double rhs = eps * sqrt(xsq[pos + c]) * (1.0 - 8.0 * 1.1102230246251565e-16);
  cert[c] = (lhs <= rhs) ? 1 : 0;
}

__global__ void k_spec_commit(long long pos, long long L, const double* res, int32_t* acc, int32_t* deg, double* dl,
                              double* res_out) {
  const long long c = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (c >= L) return;
  acc[pos + c] = 0;
  deg[pos + c] = 0;
  dl[pos + c] = 0.0;
  res_out[pos + c] = res[c];
}

}  // namespace

int64_t spec_certify(Basis& B, const Cands& c, const double* xsq, const double* Gb, const double* Gc,
                     const int* kept_cand, int64_t K0, int64_t K, int64_t pos, int64_t b, double eps, int32_t* acc,
                     int32_t* deg, double* dl, double* res_out) {
  Ctx* ctx = B.ctx;
  const int64_t nu = c.n;
  b = std::min<int64_t>(b, nu - pos);
  if (b <= 0 || K == 0) return 0;
  const int64_t dim = B.dim;
  Buf<double> G(ctx, (size_t)K * b), Y(ctx, (size_t)K * b), Xd(ctx, (size_t)dim * b);
  Buf<double> res(ctx, b);
  Buf<int> cert(ctx, b);
  res.zero();
  Xd.zero();
  LAUNCH(ctx, k_spec_g, ceil_div((uint64_t)K * b, 256), 256, 0, G.p, (long long)b, (long long)K, (long long)K0,
         (long long)nu, (long long)pos, Gb, Gc, kept_cand);
  LAUNCH(ctx, k_spec_dense_x, (unsigned)b, 128, 0, c, (long long)pos, (long long)b, Xd.p);
  const long long ywarps = (long long)K * ((b + 31) / 32);
  LAUNCH(ctx, k_spec_y, ceil_div((uint64_t)ywarps * 32, 256), 256, 0, B.U.p, (long long)B.LD, (long long)K, G.p,
         (long long)b, Y.p);
  const unsigned grid = (unsigned)std::min<int64_t>(ceil_div((uint64_t)dim * 32, 256), (int64_t)ctx->sm_count * 16);
  LAUNCH(ctx, k_spec_res, grid, 256, 0, (long long)dim, (long long)b, B.rowbase.p, B.rowlen.p, B.rek.p, B.rev.p, Y.p,
         Xd.p, res.p);
  // n terms summed in another order (plus the per-warp partial sums): the
  // reference's sum is within a factor 1 +- 2 gamma_n of ours
  const double u = 1.1102230246251565e-16;
  const double n_terms = (double)dim + 64.0;
  const double gam = n_terms * u / (1.0 - n_terms * u);
  LAUNCH(ctx, k_spec_decide, ceil_div((uint64_t)b, 128), 128, 0, (long long)b, (long long)pos, (long long)nu, res.p,
         xsq, eps, 1.0 + 2.0 * gam, cert.p);
  std::vector<int> hc(b);
  ctx->to_host(hc.data(), cert.p, b);
  ctx->sync();
  int64_t L = 0;
  while (L < b && hc[L]) ++L;
  if (L > 0)
    LAUNCH(ctx, k_spec_commit, ceil_div((uint64_t)L, 128), 128, 0, (long long)pos, (long long)L, res.p, acc, deg, dl,
           res_out);
  return L;
}

}  // namespace ctdgpu
