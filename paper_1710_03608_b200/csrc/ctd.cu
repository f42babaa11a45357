// Orchestration of Algorithm 1 (CTD-S, ctd_static.cpp:19-50) and
// Algorithm 2 (CTD-D step, ctd_dynamic.cpp:149-229) on the device.
#include <chrono>
#include <cstdio>
#include <cstdlib>

#include "cdf.cuh"
#include "ctd.cuh"
#include "relerr.cuh"
#include "sample.cuh"

namespace ctdgpu {

namespace {

__global__ void k_make_cands(const int32_t* uniq, const int* n_u, const int64_t* fptr, int64_t* off,
                             int32_t* len) {
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= *n_u) return;
  const int f = uniq[i];
  off[i] = fptr[f];
  len[i] = (int32_t)(fptr[f + 1] - fptr[f]);
}

__global__ void k_gather_cols(const int32_t* fib, long long n, const int64_t* fcol, int64_t* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = fcol[fib[i]];
}

// Front end shared by CTD-S and the CTD-D step: law, draws, dedup, filter.
struct Front {
  std::vector<int64_t> drawn, unique;
  std::vector<int32_t> unique_fib;  // fiber index (into the Fibers) of each unique candidate
  BatchOut bo;
  double total = 0.0;
};

void front_end(Ctx* ctx, const Fibers& fb, Basis& basis, int64_t s, double eps, uint64_t seed,
               Front& fr, bool trace) {
  const int64_t F = fb.F;
  Buf<double> probs(ctx, F + 1), cum(ctx, F + 1), total(ctx, 1);
  {
    PhaseScope ps(ctx, PH_LAW);
    sampling_law(ctx, fb.norm.p, F, total.p, probs.p, cum.p, ctx->d_flags);
  }
  Buf<int32_t> drawn(ctx, s), uniq(ctx, s);
  Buf<int> nu(ctx, 1);
  {
    PhaseScope ps(ctx, PH_SAMPLE);
    draw_fibers(ctx, cum.p, F, s, seed, drawn.p);
    dedup_first(ctx, drawn.p, s, uniq.p, nu.p);
  }
  int n_u = 0;
  ctx->to_host(&n_u, nu.p, 1);
  ctx->to_host(&fr.total, total.p, 1);
  ctx->sync();
  ctx->check_flags("sampling");
  Buf<int64_t> coff(ctx, n_u + 1);
  Buf<int32_t> clen(ctx, n_u + 1);
  if (n_u > 0) LAUNCH(ctx, k_make_cands, ceil_div(n_u, 256), 256, 0, uniq.p, nu.p, fb.ptr.p, coff.p, clen.p);
  Cands c;
  c.n = n_u;
  c.off = coff.p;
  c.len = clen.p;
  c.row = fb.row.p;
  c.val = fb.val.p;
  filter_batch(basis, c, eps, fr.bo, false);
  // column ids of the draws / unique candidates (host trace)
  Buf<int64_t> cols(ctx, s + 1);
  if (trace) {
    fr.drawn.resize(s);
    LAUNCH(ctx, k_gather_cols, ceil_div(s, 256), 256, 0, drawn.p, (long long)s, fb.col.p, cols.p);
    ctx->to_host(fr.drawn.data(), cols.p, s);
    ctx->sync();
  }
  fr.unique.resize(n_u);
  fr.unique_fib.resize(n_u);
  if (n_u > 0) {
    ctx->to_host(fr.unique_fib.data(), uniq.p, n_u);
    LAUNCH(ctx, k_gather_cols, ceil_div(n_u, 256), 256, 0, uniq.p, (long long)n_u, fb.col.p, cols.p);
    ctx->to_host(fr.unique.data(), cols.p, n_u);
    ctx->sync();
  }
}

void check_ctd_s_args(const Tensor& x, int mode, int64_t s, double eps) {
  // ctd_static.cpp:21-27
  if (x.nnz == 0) fail(CTD_ERR_EMPTY_INPUT, "cannot decompose an empty tensor");
  if (mode < 0 || mode >= x.order)
    fail(CTD_ERR_ARGUMENT, "mode " + std::to_string(mode) + " out of range for order " +
                               std::to_string(x.order));
  if (s < 1) fail(CTD_ERR_ARGUMENT, "sample size must be at least 1");
  if (!(eps > 0.0)) fail(CTD_ERR_ARGUMENT, "epsilon must be positive");
}

// History append (concatenate_time, ctd_dynamic.cpp:87-105): plane k of the
// history holds mode k's indices; the time coordinate is shifted by t_add.
struct IdxPlanes {
  const int32_t* p[kMaxOrder];
};
__global__ void k_hist_append(IdxPlanes src, const double* sval, long long nnz, int order, long long t_add,
                              int32_t* didx, long long hcap, double* dval, long long at) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  for (int k = 0; k < order; ++k)
    didx[(long long)k * hcap + at + i] = src.p[k][i] + (k == order - 1 ? (int32_t)t_add : 0);
  dval[at + i] = sval[i];
}

void history_append(Stream& st, const Tensor& x, long long t_add) {
  Ctx* ctx = st.ctx;
  const long long need_n = st.hnnz + x.nnz;
  if (need_n > st.hcap) {
    const long long ncap = std::max<long long>(need_n, 2 * st.hcap + 1024);
    Buf<int32_t> ni(ctx, (size_t)ncap * st.order);
    Buf<double> nv(ctx, ncap);
    for (int k = 0; k < st.order && st.hnnz; ++k)
      CUDA_OK(cudaMemcpyAsync(ni.p + (size_t)k * ncap, st.hidx.p + (size_t)k * st.hcap, st.hnnz * sizeof(int32_t),
                              cudaMemcpyDeviceToDevice, ctx->stream));
    if (st.hnnz)
      CUDA_OK(cudaMemcpyAsync(nv.p, st.hval.p, st.hnnz * sizeof(double), cudaMemcpyDeviceToDevice, ctx->stream));
    st.hidx = std::move(ni);
    st.hval = std::move(nv);
    st.hcap = ncap;
  }
  if (x.nnz) {
    IdxPlanes pl{};
    for (int k = 0; k < x.order; ++k) pl.p[k] = x.idx[k];
    LAUNCH(ctx, k_hist_append, ceil_div(x.nnz, 256), 256, 0, pl, x.val, (long long)x.nnz, x.order, t_add,
           st.hidx.p, (long long)st.hcap, st.hval.p, (long long)st.hnnz);
  }
  st.hnnz = need_n;
}

}  // namespace

Tensor Stream::history() const {
  Tensor h;
  h.ctx = ctx;
  h.order = order;
  for (int k = 0; k + 1 < order; ++k) h.shape[k] = slab_shape[k];
  h.shape[order - 1] = t;
  h.nnz = hnnz;
  for (int k = 0; k < order; ++k) h.idx[k] = hidx.p ? hidx.p + (size_t)k * hcap : nullptr;
  h.val = hval.p;
  return h;
}

void stream_core_sync(Stream& st) {
  for (const CoreRecord& r : st.pending) core_apply(st.ctx, st.core, r);
  st.pending.clear();
  st.arena.clear();
  st.pending_entries = st.pending_bytes = 0;
}

double stream_core_drift(Stream& st) {
  // ctd_dynamic.cpp:271-273
  if (!(st.keep_history || st.exact_core)) fail(CTD_ERR_ARGUMENT, "core drift requires retained history");
  stream_core_sync(st);
  Fibers hf;
  matricize(st.ctx, st.history(), st.mode, hf);
  return core_drift(st.ctx, st.core, hf, *st.basis);
}

void build_law(Ctx* ctx, const Tensor& x, int mode, Law& law) {
  matricize(ctx, x, mode, law.fb);
  if (law.fb.nnz == 0) fail(CTD_ERR_EMPTY_INPUT, "column distribution of an all-zero matrix");
  const int64_t F = law.fb.F;
  law.probs.alloc(ctx, F + 1);
  law.cum.alloc(ctx, F + 1);
  law.total.alloc(ctx, 1);
  sampling_law(ctx, law.fb.norm.p, F, law.total.p, law.probs.p, law.cum.p, ctx->d_flags);
  ctx->sync();
  ctx->check_flags("column_distribution");
}

void run_ctd_s(Ctx* ctx, const Tensor& x, int mode, int64_t s, double eps, uint64_t seed,
               unsigned flags, Factors& out) {
  check_ctd_s_args(x, mode, s, eps);
  out.ctx = ctx;
  out.order = x.order;
  out.mode = mode;
  for (int k = 0; k < x.order; ++k) out.shape[k] = x.shape[k];
  out.eps = eps;
  out.seed = seed;
  Fibers fb;
  static const bool htrace = getenv("CTD_HOST_TRACE") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  {
    PhaseScope ps(ctx, PH_MATRICIZE);
    matricize(ctx, x, mode, fb);
  }
  const auto h1 = std::chrono::steady_clock::now();
  out.F = fb.F;
  out.cols = fb.cols;
  out.rows = fb.rows;
  out.integer_exact = fb.integer_exact;
  out.basis = std::make_unique<Basis>(ctx, fb.rows);
  out.basis->want_panel = (flags & (CTD_GPU_WITH_ERROR | CTD_GPU_KEEP_PANEL)) != 0;
  Front fr;
  front_end(ctx, fb, *out.basis, s, eps, seed, fr, true);
  out.total = fr.total;
  out.drawn = std::move(fr.drawn);
  out.unique = std::move(fr.unique);
  out.accepted = fr.bo.accepted;
  out.degenerate = fr.bo.degenerate;
  out.delta = fr.bo.delta;
  out.slow_path = fr.bo.slow_path;
  for (int32_t k : fr.bo.kept_cand) out.kept_flat.push_back(out.unique[k]);
  for (size_t i = 0; i < fr.bo.res_sq.size(); ++i) {
    const double xs = fr.bo.x_sq[i];
    if (xs > 0.0 && fr.bo.res_sq[i] > 0.0) {
      const double m = std::fabs(std::log10(std::sqrt(fr.bo.res_sq[i] / xs) / eps));
      out.min_margin = std::min(out.min_margin, m);
    }
  }
  const auto h2 = std::chrono::steady_clock::now();
  if (flags & CTD_GPU_WITH_ERROR) {
    PhaseScope ps(ctx, PH_ERROR);
    out.rel_error = relative_error(ctx, fb, *out.basis);
  }
  if (flags & CTD_GPU_WITH_CORE) {  // factors.C = compute_core(x, R, mode) (ctd_static.cpp:47)
    PhaseScope ps(ctx, PH_CORE);
    compute_core(ctx, fb, *out.basis, out.core);
    out.has_core = true;
  }
  if (htrace) {
    const auto h3 = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "[ctd_s host] matricize=%.3f front=%.3f error=%.3f ms\n", ms(h0, h1), ms(h1, h2),
            ms(h2, h3));
  }
}

void stream_init(Ctx* ctx, const Tensor& hist, int mode, int64_t s, double eps, uint64_t seed,
                 unsigned flags, Stream& out) {
  // ctd_dynamic.cpp:133-136
  if (hist.order < 2) fail(CTD_ERR_ARGUMENT, "a stream needs at least one non-time mode");
  if (mode < 0 || mode >= hist.order - 1) fail(CTD_ERR_ARGUMENT, "mode must precede the time mode");
  Factors f;
  out.keep_history = (flags & CTD_GPU_KEEP_HISTORY) != 0;
  out.exact_core = (flags & CTD_GPU_EXACT_CORE) != 0;
  out.with_core = (flags & (CTD_GPU_WITH_CORE | CTD_GPU_KEEP_HISTORY | CTD_GPU_EXACT_CORE | CTD_GPU_LAZY_CORE)) != 0;
  out.lazy_core = (flags & CTD_GPU_LAZY_CORE) != 0 && !out.exact_core;
  run_ctd_s(ctx, hist, mode, s, eps, seed, out.with_core ? CTD_GPU_WITH_CORE : 0, f);
  if (out.with_core) core_from_static(ctx, f.core, out.core);  // matricize(f.C, mode) (:141)
  out.ctx = ctx;
  out.order = hist.order;
  out.mode = mode;
  for (int k = 0; k + 1 < hist.order; ++k) out.slab_shape[k] = hist.shape[k];
  out.t = hist.shape[hist.order - 1];
  out.eps = eps;
  out.seed = seed;
  out.basis = std::move(f.basis);
  out.kept_flat = std::move(f.kept_flat);
  if (out.keep_history || out.exact_core) history_append(out, hist, 0);  // :143
}

void stream_step(Stream& st, const Tensor& slab, int64_t d) {
  // ctd_dynamic.cpp:151-158
  if (slab.order != st.order) fail(CTD_ERR_SHAPE, "slab order does not match the stream");
  for (int k = 0; k + 1 < st.order; ++k)
    if (slab.shape[k] != st.slab_shape[k]) fail(CTD_ERR_SHAPE, "slab extents do not match the stream");
  if (slab.shape[st.order - 1] != 1) fail(CTD_ERR_SHAPE, "slab must have time extent 1");
  if (d < 1) fail(CTD_ERR_ARGUMENT, "sample size must be at least 1");
  Ctx* ctx = st.ctx;
  if (slab.nnz > 0) {  // :173-188
    Fibers fb;
    matricize(ctx, slab, st.mode, fb);
    // snapshot U^(t) for the core update (:165-167)
    const int64_t Kold = st.basis->K;
    Buf<double>& uold = st.uold;
    if (st.with_core && Kold) {
      if (uold.n < (size_t)Kold * Kold) uold.alloc(ctx, (size_t)Kold * Kold * 3 / 2 + 1);  // amortized growth
      CUDA_OK(cudaMemcpy2DAsync(uold.p, Kold * sizeof(double), st.basis->U.p, st.basis->LD * sizeof(double),
                                Kold * sizeof(double), Kold, cudaMemcpyDeviceToDevice, ctx->stream));
    }
    Front fr;
    front_end(ctx, fb, *st.basis, d, st.eps, st.seed ^ (uint64_t)st.t, fr, false);
    std::vector<int32_t> appended;
    for (int32_t k : fr.bo.kept_cand) {
      st.kept_flat.push_back(fr.unique[k] + st.t * fb.cols);
      appended.push_back(fr.unique_fib[k]);
    }
    PhaseScope ps(ctx, PH_CORE);
    if (st.exact_core && !appended.empty()) {  // :207-211
      Fibers hf;
      matricize(ctx, st.history(), st.mode, hf);
      core_step_exact(ctx, st.core, fb, hf, *st.basis, Kold, st.t * fb.cols);
    } else if (st.lazy_core) {
      st.pending.emplace_back();
      core_record(ctx, fb, *st.basis, Kold, uold.p, appended, st.t * fb.cols, &st.arena, st.pending.back());
      const CoreRecord& r = st.pending.back();
      st.pending_entries += r.nnz;
      st.pending_bytes += 12 * r.nnz + 8 * (int64_t)r.A * r.Kold;
    } else if (st.with_core) {
      core_step(ctx, st.core, fb, *st.basis, Kold, uold.p, appended, st.t * fb.cols);
    }
  }
  if (st.keep_history || st.exact_core) history_append(st, slab, st.t);  // :225-226
  st.t += 1;  // :227
}

}  // namespace ctdgpu
