// extern "C" boundary (include/ctd_gpu.h).  Every entry point converts
// internal failures into the reference ErrorClass codes.
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <string>

#include "cdf.cuh"
#include "ctd.cuh"
#include "relerr.cuh"
#include "sample.cuh"

using namespace ctdgpu;

struct ctd_gpu_ctx {
  Ctx c;
};
struct ctd_gpu_tensor {
  Tensor t;
};
struct ctd_gpu_factors {
  Factors f;
};
struct ctd_gpu_basis {
  Ctx* ctx;
  std::unique_ptr<Basis> b;
};
struct ctd_gpu_stream {
  Stream s;
};
struct ctd_gpu_shard {
  Ctx* ctx;
  Fibers fb;                       // the shard's bucketed fibers, resident in HBM
  std::vector<int64_t> col, ptr;   // host copies for owner lookups
  Buf<double> cum;                 // this shard's segment of the global CDF (ctd_gpu_shard_cdf)
  Buf<int> last_pos;               // last fiber with p > 0, or -1
  double cum_lo = 0.0, cum_hi = 0.0;
  Core core;                       // this shard's core columns (ctd_gpu_shard_core)
  bool has_core = false;
};
struct ctd_gpu_csc {
  Ctx* ctx;
  Core c;               // columns with entries; row/val on the device
  int32_t row_shift = 0;  // subtracted from the stored rows on export
};
struct ctd_gpu_core_shard {
  Ctx* ctx;
  DevCore core;       // this rank's columns of the stream's Eq. 13 core
  Buf<double> uold;   // U^(t) snapshot (Kold x Kold) taken by _begin
  int64_t Kold = -1;
};

namespace {

thread_local std::string g_last_error;

template <typename F>
int guarded(F&& f) {
  try {
    f();
    return CTD_OK;
  } catch (const Fail& e) {
    g_last_error = e.msg;
    return e.code;
  } catch (const std::bad_alloc&) {
    g_last_error = "host allocation failed";
    return CTD_ERR_DEVICE;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return CTD_ERR_DEVICE;
  }
}

void need(const void* p, const char* what) {
  if (!p) fail(CTD_ERR_ARGUMENT, std::string(what) + " is NULL");
}

// Every entry point runs on its context's device, whatever the calling
// thread's current device is (several contexts on several devices may share
// one process).
void bind_device(const Ctx* c) {
  if (!c) return;
  int cur = -1;
  CUDA_OK(cudaGetDevice(&cur));
  if (cur != c->device) CUDA_OK(cudaSetDevice(c->device));
}

__global__ void k_narrow(const int64_t* in, long long nnz, int order, int32_t* out, unsigned* flags) {
  const long long e = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= nnz * order) return;
  const long long i = e / order;
  const int k = (int)(e - i * order);
  const int64_t v = in[e];
  if (v < 0 || v > 0x7fffffffLL) atomicOr(flags, FLAG_BOUNDS);
  out[(long long)k * nnz + i] = (int32_t)v;
}

void check_shape(int order, const int64_t* shape) {
  if (order < 0 || order > kMaxOrder) fail(CTD_ERR_ARGUMENT, "tensor order out of range");
  for (int k = 0; k < order; ++k) {
    if (shape[k] < 0) fail(CTD_ERR_ARGUMENT, "tensor extent must be non-negative");
    if (shape[k] > 0x7fffffffLL) fail(CTD_ERR_SHAPE, "tensor extent exceeds the int32 index range");
  }
}

}  // namespace

namespace ctdgpu {

// dist.cu's view of the boundary objects (its own entry points report
// through the same thread-local message as every other entry point).
Ctx* ctx_of(ctd_gpu_ctx* c) { return c ? &c->c : nullptr; }
int report_error(int code, const std::string& msg) {
  g_last_error = msg;
  return code;
}
int64_t tensor_extent(const ctd_gpu_tensor* t, int mode) {
  return (t && mode >= 0 && mode < t->t.order) ? t->t.shape[mode] : -1;
}
bool shard_col_range(const ctd_gpu_shard* s, int64_t* first, int64_t* last) {
  if (!s || s->col.empty()) return false;
  *first = s->col.front();
  *last = s->col.back();
  return true;
}

void Ctx::check_flags(const char* where) {
  unsigned f = 0;
  CUDA_OK(cudaMemcpyAsync(&f, d_flags, sizeof(unsigned), cudaMemcpyDeviceToHost, stream));
  CUDA_OK(cudaStreamSynchronize(stream));
  if (!f) return;
  CUDA_OK(cudaMemsetAsync(d_flags, 0, sizeof(unsigned), stream));
  const std::string w(where);
  if (f & FLAG_BOUNDS) fail(CTD_ERR_SHAPE, w + ": tensor entry index out of bounds");
  if (f & FLAG_DUPLICATE)
    fail(CTD_ERR_ARGUMENT, w + ": duplicate coordinates (input is not a normalized SparseTensor)");
  if (f & FLAG_ZERO) fail(CTD_ERR_ARGUMENT, w + ": stored zero (input is not a normalized SparseTensor)");
  if (f & FLAG_EMPTY) fail(CTD_ERR_EMPTY_INPUT, w + ": sampling from an all-zero distribution");
  if (f & FLAG_OVERFLOW) fail(CTD_ERR_NUMERIC, w + ": internal capacity exceeded");
  // FLAG_SEQSUM: a self-check failed and the sequential fallback ran; the
  // result is still exact.  Nothing to report.
}

}  // namespace ctdgpu

extern "C" {

const char* ctd_gpu_last_error(void) { return g_last_error.c_str(); }
const char* ctd_gpu_version(void) { return "ctd_gpu 0.1 (sm_100a)"; }

int ctd_gpu_ctx_create(int device, void* stream, ctd_gpu_ctx** out) {
  return guarded([&] {
    need(out, "out");
    auto h = std::make_unique<ctd_gpu_ctx>();
    Ctx& c = h->c;
    c.device = device;
    CUDA_OK(cudaSetDevice(device));
    c.stream = static_cast<cudaStream_t>(stream);
    CUDA_OK(cudaDeviceGetAttribute(&c.sm_count, cudaDevAttrMultiProcessorCount, device));
    int coop = 0;
    CUDA_OK(cudaDeviceGetAttribute(&coop, cudaDevAttrCooperativeLaunch, device));
    if (!coop) fail(CTD_ERR_DEVICE, "device does not support cooperative launch");
    cudaMemPool_t pool;
    CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, device));
    uint64_t thr = UINT64_MAX;
    CUDA_OK(cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr));
    // Prewarm the stream-ordered pool so steady-state calls never map memory
    // (CTD_GPU_POOL_MB, default 1024: buffers below Ctx::kBigBytes; the pool keeps it).
    {
      size_t mb = 1024;
      if (const char* e = getenv("CTD_GPU_POOL_MB")) mb = (size_t)atoll(e);
      size_t free_b = 0, total_b = 0;
      CUDA_OK(cudaMemGetInfo(&free_b, &total_b));
      mb = std::min(mb, free_b / 4 / (1 << 20));
      if (mb > 0) {
        void* p = nullptr;
        CUDA_OK(cudaMallocAsync(&p, mb << 20, c.stream));
        CUDA_OK(cudaFreeAsync(p, c.stream));
        CUDA_OK(cudaStreamSynchronize(c.stream));
      }
    }
    CUDA_OK(cudaMalloc(&c.d_flags, sizeof(unsigned)));
    CUDA_OK(cudaMalloc(&c.d_bar, 4 * sizeof(unsigned)));
    CUDA_OK(cudaMemset(c.d_flags, 0, sizeof(unsigned)));
    CUDA_OK(cudaMemset(c.d_bar, 0, 4 * sizeof(unsigned)));
    ctx_register(&h->c, true);
    *out = h.release();
  });
}

int ctd_gpu_ctx_set_stream(ctd_gpu_ctx* ctx, void* stream) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    CUDA_OK(cudaStreamSynchronize(ctx->c.stream));  // cached blocks are reused in stream order
    ctx->c.stream = static_cast<cudaStream_t>(stream);
  });
}

int ctd_gpu_ctx_trim(ctd_gpu_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    ctx->c.big_trim();
    cudaMemPool_t pool;
    CUDA_OK(cudaDeviceGetDefaultMemPool(&pool, ctx->c.device));
    CUDA_OK(cudaStreamSynchronize(ctx->c.stream));
    CUDA_OK(cudaMemPoolTrimTo(pool, 0));
  });
}

int ctd_gpu_ctx_synchronize(ctd_gpu_ctx* ctx) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    ctx->c.sync();
  });
}

int ctd_gpu_ctx_destroy(ctd_gpu_ctx* ctx) {
  return guarded([&] {
    if (!ctx) return;
    cudaStreamSynchronize(ctx->c.stream);
    ctx_register(&ctx->c, false);
    ctx->c.big_release_all();
    cudaFree(ctx->c.d_flags);
    cudaFree(ctx->c.d_bar);
    delete ctx;
  });
}

int64_t ctd_gpu_ctx_launches(const ctd_gpu_ctx* ctx) { return ctx ? ctx->c.launches : -1; }

int ctd_gpu_ctx_set_timing(ctd_gpu_ctx* ctx, int enable) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    ctx->c.phase_flush();
    ctx->c.timing = enable != 0;
  });
}

int ctd_gpu_ctx_phase_times(ctd_gpu_ctx* ctx, double* ms, int64_t* counts, int reset) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    ctx->c.phase_flush();
    for (int i = 0; i < Ctx::kPhases; ++i) {
      if (ms) ms[i] = ctx->c.phase_ms[i];
      if (counts) counts[i] = ctx->c.phase_n[i];
      if (reset) {
        ctx->c.phase_ms[i] = 0;
        ctx->c.phase_n[i] = 0;
      }
    }
  });
}

const char* ctd_gpu_phase_name(int i) {
  static const char* names[] = {"matricize", "law", "sample", "filter_prep", "filter", "error", "h2d", "core"};
  return (i >= 0 && i < Ctx::kPhases) ? names[i] : "";
}

int ctd_gpu_tensor_from_host(ctd_gpu_ctx* ctx, int order, const int64_t* shape, int64_t nnz,
                             const int64_t* indices, const double* values, ctd_gpu_tensor** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(out, "out");
    if (order > 0) need(shape, "shape");
    if (nnz < 0) fail(CTD_ERR_SHAPE, "index data does not match entry count");
    if (order == 0 && nnz > 0) fail(CTD_ERR_SHAPE, "entries supplied for an order-0 tensor");
    check_shape(order, shape);
    Ctx* c = &ctx->c;
    auto h = std::make_unique<ctd_gpu_tensor>();
    Tensor& t = h->t;
    t.ctx = c;
    t.order = order;
    t.nnz = nnz;
    for (int k = 0; k < order; ++k) t.shape[k] = shape[k];
    t.own_idx.alloc(c, (size_t)nnz * order + 1);
    t.own_val.alloc(c, nnz + 1);
    if (nnz > 0) {
      need(indices, "indices");
      need(values, "values");
      PhaseScope ps(c, PH_H2D);
      Buf<int64_t> raw(c, (size_t)nnz * order);
      c->to_dev(raw.p, indices, (size_t)nnz * order);
      c->to_dev(t.own_val.p, values, nnz);
      LAUNCH(c, k_narrow, ceil_div((uint64_t)nnz * order, 256), 256, 0, raw.p, (long long)nnz, order,
             t.own_idx.p, c->d_flags);
      c->check_flags("SparseTensor");
    }
    for (int k = 0; k < order; ++k) t.idx[k] = t.own_idx.p + (size_t)k * nnz;
    t.val = t.own_val.p;
    *out = h.release();
  });
}

int ctd_gpu_tensor_from_device(ctd_gpu_ctx* ctx, int order, const int64_t* shape, int64_t nnz,
                               const int32_t* const* mode_indices, const double* values,
                               ctd_gpu_tensor** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(out, "out");
    if (order > 0) need(shape, "shape");
    if (nnz < 0) fail(CTD_ERR_SHAPE, "index data does not match entry count");
    check_shape(order, shape);
    auto h = std::make_unique<ctd_gpu_tensor>();
    Tensor& t = h->t;
    t.ctx = &ctx->c;
    t.order = order;
    t.nnz = nnz;
    for (int k = 0; k < order; ++k) {
      t.shape[k] = shape[k];
      t.idx[k] = mode_indices ? mode_indices[k] : nullptr;
      if (nnz > 0) need(t.idx[k], "mode_indices[k]");
    }
    t.val = values;
    if (nnz > 0) need(values, "values");
    *out = h.release();
  });
}

int64_t ctd_gpu_tensor_nnz(const ctd_gpu_tensor* t) { return t ? t->t.nnz : -1; }

int ctd_gpu_tensor_destroy(ctd_gpu_tensor* t) {
  return guarded([&] { delete t; });
}

int ctd_gpu_matricize(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* x, int mode, int64_t* n_fibers,
                      int64_t* fiber_col, int64_t* fiber_ptr, int32_t* rows, double* vals,
                      double* sq_norms) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(x, "x");
    Ctx* c = &ctx->c;
    Fibers fb;
    matricize(c, x->t, mode, fb);
    if (n_fibers) *n_fibers = fb.F;
    if (fiber_col) c->to_host(fiber_col, fb.col.p, fb.F);
    if (fiber_ptr) c->to_host(fiber_ptr, fb.ptr.p, fb.F + 1);
    if (rows) c->to_host(rows, fb.row.p, fb.nnz);
    if (vals) c->to_host(vals, fb.val.p, fb.nnz);
    if (sq_norms) c->to_host(sq_norms, fb.norm.p, fb.F);
    c->sync();
  });
}

int ctd_gpu_column_distribution(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* x, int mode,
                                double* total_sq_norm, double* probs, double* cumulative) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(x, "x");
    Ctx* c = &ctx->c;
    Law law;
    build_law(c, x->t, mode, law);
    if (total_sq_norm) c->to_host(total_sq_norm, law.total.p, 1);
    if (probs) c->to_host(probs, law.probs.p, law.fb.F);
    if (cumulative) c->to_host(cumulative, law.cum.p, law.fb.F);
    c->sync();
  });
}

// A host CSC (SparseMatrix layout: col_ptr[cols+1], rows ascending per
// column) uploaded as the nonempty columns' fibers.
static void fibers_from_csc(Ctx* c, int64_t rows, int64_t cols, const int64_t* col_ptr, const int64_t* row_idx,
                            const double* vals, Fibers& fb) {
  if (rows < 0 || cols < 0) fail(CTD_ERR_ARGUMENT, "matrix extents must be non-negative");
  if (rows > 0x7fffffffLL) fail(CTD_ERR_SHAPE, "matrix row count exceeds the int32 index range");
  need(col_ptr, "col_ptr");
  const int64_t nnz = col_ptr[cols];
  std::vector<int64_t> col, ptr;
  std::vector<int32_t> r32(nnz > 0 ? nnz : 1);
  for (int64_t j = 0; j < cols; ++j) {
    if (col_ptr[j + 1] < col_ptr[j]) fail(CTD_ERR_ARGUMENT, "col_ptr must be non-decreasing");
    if (col_ptr[j + 1] > col_ptr[j]) {
      col.push_back(j);
      ptr.push_back(col_ptr[j]);
    }
  }
  ptr.push_back(nnz);
  for (int64_t t = 0; t < nnz; ++t) {
    if (row_idx[t] < 0 || row_idx[t] >= rows) fail(CTD_ERR_SHAPE, "row index out of range");
    r32[t] = (int32_t)row_idx[t];
  }
  fb.rows = rows;
  fb.cols = cols;
  fb.nnz = nnz;
  fb.F = (int64_t)col.size();
  fb.col.alloc(c, fb.F + 1);
  fb.ptr.alloc(c, fb.F + 1);
  fb.row.alloc(c, nnz + 1);
  fb.val.alloc(c, nnz + 1);
  c->to_dev(fb.col.p, col.data(), fb.F);
  c->to_dev(fb.ptr.p, ptr.data(), fb.F + 1);
  c->to_dev(fb.row.p, r32.data(), nnz);
  c->to_dev(fb.val.p, vals, nnz);
  fiber_norms(c, fb);
  c->check_flags("column_sq_norms");
}

int ctd_gpu_column_sq_norms_csc(ctd_gpu_ctx* ctx, int64_t rows, int64_t cols, const int64_t* col_ptr,
                                const int64_t* row_idx, const double* vals, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(out, "out");
    Ctx* c = &ctx->c;
    Fibers fb;
    fibers_from_csc(c, rows, cols, col_ptr, row_idx, vals, fb);
    std::vector<int64_t> col(fb.F);
    std::vector<double> nrm(fb.F);
    c->to_host(col.data(), fb.col.p, fb.F);
    c->to_host(nrm.data(), fb.norm.p, fb.F);
    c->sync();
    std::fill(out, out + cols, 0.0);
    for (int64_t f = 0; f < fb.F; ++f) out[col[f]] = nrm[f];
  });
}

int ctd_gpu_column_distribution_csc(ctd_gpu_ctx* ctx, int64_t rows, int64_t cols, const int64_t* col_ptr,
                                    const int64_t* row_idx, const double* vals, double* total_sq_norm,
                                    double* probs) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    Ctx* c = &ctx->c;
    Fibers fb;
    fibers_from_csc(c, rows, cols, col_ptr, row_idx, vals, fb);
    if (fb.F == 0) fail(CTD_ERR_EMPTY_INPUT, "column distribution of a matrix without nonzero entries");  // sampling.cpp:22-23
    Buf<double> pr(c, fb.F + 1), cum(c, fb.F + 1), tot(c, 1);
    sampling_law(c, fb.norm.p, fb.F, tot.p, pr.p, cum.p, c->d_flags);
    c->check_flags("column_distribution");
    std::vector<int64_t> col(fb.F);
    std::vector<double> p(fb.F);
    c->to_host(col.data(), fb.col.p, fb.F);
    c->to_host(p.data(), pr.p, fb.F);
    if (total_sq_norm) c->to_host(total_sq_norm, tot.p, 1);
    c->sync();
    if (probs) {
      std::fill(probs, probs + cols, 0.0);
      for (int64_t f = 0; f < fb.F; ++f) probs[col[f]] = p[f];
    }
  });
}

int ctd_gpu_sample_with_replacement(ctd_gpu_ctx* ctx, const double* probs, int64_t n, int64_t count,
                                    uint64_t seed, int64_t* out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    if (count < 0) fail(CTD_ERR_ARGUMENT, "sample count must be non-negative");  // sampling.cpp:36
    if (count == 0) return;
    need(out, "out");
    Ctx* c = &ctx->c;
    if (n <= 0) fail(CTD_ERR_EMPTY_INPUT, "sampling from an all-zero distribution");
    need(probs, "probs");
    Buf<double> p(c, n), cum(c, n);
    c->to_dev(p.p, probs, n);
    clamped_cdf(c, p.p, n, cum.p, c->d_flags);
    c->check_flags("sample_with_replacement");
    Buf<int64_t> d(c, count);
    draw_columns(c, cum.p, n, count, seed, d.p);
    c->to_host(out, d.p, count);
    c->sync();
  });
}

int ctd_gpu_seq_cumsum(ctd_gpu_ctx* ctx, const double* x, int64_t n, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    if (n <= 0) return;
    need(x, "x");
    need(out, "out");
    Ctx* c = &ctx->c;
    Buf<double> d(c, n), o(c, n), t(c, 1);
    c->to_dev(d.p, x, n);
    seq_cumsum(c, d.p, n, o.p, t.p);
    c->to_host(out, o.p, n);
    c->sync();
  });
}

int ctd_gpu_unique_first_occurrence(ctd_gpu_ctx* ctx, const int64_t* drawn, int64_t n, int64_t* out,
                                    int64_t* n_out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(n_out, "n_out");
    *n_out = 0;
    if (n <= 0) return;
    need(drawn, "drawn");
    need(out, "out");
    Ctx* c = &ctx->c;
    Buf<int64_t> in(c, n), o(c, n);
    Buf<int> nu(c, 1);
    c->to_dev(in.p, drawn, n);
    dedup_first64(c, in.p, n, o.p, nu.p);
    int k = c->read1(nu.p);
    c->to_host(out, o.p, k);
    c->sync();
    *n_out = k;
  });
}

int ctd_gpu_ctd_s(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* x, int mode, int64_t sample_size, double epsilon,
                  uint64_t seed, unsigned flags, ctd_gpu_factors** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(x, "x");
    need(out, "out");
    auto h = std::make_unique<ctd_gpu_factors>();
    run_ctd_s(&ctx->c, x->t, mode, sample_size, epsilon, seed, flags, h->f);
    ctx->c.phase_flush();
    *out = h.release();
  });
}

int ctd_gpu_factors_info_get(const ctd_gpu_factors* f, ctd_gpu_factors_info* info) {
  return guarded([&] {
    need(f, "factors");
    bind_device(f->f.ctx);
    need(info, "info");
    const Factors& F = f->f;
    std::memset(info, 0, sizeof(*info));
    info->kept = (int64_t)F.kept_flat.size();
    info->r_rows = F.rows;
    info->r_nnz = F.basis ? F.basis->rnnz : 0;
    info->c_nnz = F.has_core ? F.core.nnz : 0;
    info->n_drawn = (int64_t)F.drawn.size();
    info->n_unique = (int64_t)F.unique.size();
    info->n_fibers = F.F;
    info->n_cols = F.cols;
    info->mode = F.mode;
    info->order = F.order;
    info->epsilon = F.eps;
    info->seed = F.seed;
    info->total_sq_norm = F.total;
    info->relative_error = F.rel_error;
    info->min_margin = F.min_margin;
    info->integer_exact = F.integer_exact;
    info->u_nnz = -1;  // computed on demand by ctd_gpu_factors_u callers
  });
}

int ctd_gpu_factors_kept_flat(const ctd_gpu_factors* f, int64_t* out) {
  return guarded([&] {
    need(f, "factors");
    bind_device(f->f.ctx);
    need(out, "out");
    std::memcpy(out, f->f.kept_flat.data(), f->f.kept_flat.size() * sizeof(int64_t));
  });
}

int ctd_gpu_factors_r(const ctd_gpu_factors* f, int64_t* col_ptr, int64_t* rows, double* vals) {
  return guarded([&] {
    need(f, "factors");
    bind_device(f->f.ctx);
    basis_r(*f->f.basis, col_ptr, rows, vals);
  });
}

int ctd_gpu_factors_u(const ctd_gpu_factors* f, double* u) {
  return guarded([&] {
    need(f, "factors");
    bind_device(f->f.ctx);
    need(u, "u");
    basis_u(*f->f.basis, u);
  });
}

int ctd_gpu_factors_core(const ctd_gpu_factors* f, int64_t* c_cols, int64_t* col_id, int64_t* col_ptr,
                         int64_t* rows, double* vals) {
  return guarded([&] {
    need(f, "factors");
    bind_device(f->f.ctx);
    const Factors& F = f->f;
    if (!F.has_core) fail(CTD_ERR_ARGUMENT, "factors were computed without CTD_GPU_WITH_CORE");
    const Core& c = F.core;
    if (c_cols) *c_cols = c.cols;
    if (col_id && c.cols) std::memcpy(col_id, c.col_id.data(), c.cols * sizeof(int64_t));
    if (col_ptr) std::memcpy(col_ptr, c.ptr.data(), (c.cols + 1) * sizeof(int64_t));
    if (c.nnz && (rows || vals)) {
      Ctx* cx = F.ctx;
      if (vals) cx->to_host(vals, c.val.p, c.nnz);
      std::vector<int32_t> r32(rows ? c.nnz : 0);
      if (rows) cx->to_host(r32.data(), c.row.p, c.nnz);
      cx->sync();
      for (int64_t i = 0; rows && i < c.nnz; ++i) rows[i] = r32[i];
    }
  });
}

int ctd_gpu_factors_trace(const ctd_gpu_factors* f, int64_t* drawn, int64_t* unique, int32_t* accepted,
                          int32_t* degenerate, double* delta) {
  return guarded([&] {
    need(f, "factors");
    bind_device(f->f.ctx);
    const Factors& F = f->f;
    if (drawn) std::memcpy(drawn, F.drawn.data(), F.drawn.size() * sizeof(int64_t));
    if (unique) std::memcpy(unique, F.unique.data(), F.unique.size() * sizeof(int64_t));
    if (accepted) std::memcpy(accepted, F.accepted.data(), F.accepted.size() * sizeof(int32_t));
    if (degenerate) std::memcpy(degenerate, F.degenerate.data(), F.degenerate.size() * sizeof(int32_t));
    if (delta) std::memcpy(delta, F.delta.data(), F.delta.size() * sizeof(double));
  });
}

int ctd_gpu_factors_destroy(ctd_gpu_factors* f) {
  return guarded([&] { delete f; });
}

int ctd_gpu_relative_error(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* x, ctd_gpu_factors* f, double* out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(x, "x");
    need(f, "factors");
    bind_device(f->f.ctx);
    need(out, "out");
    Factors& F = f->f;
    if (x->t.order != F.order) fail(CTD_ERR_SHAPE, "factor shape does not match the tensor");
    for (int k = 0; k < F.order; ++k)
      if (x->t.shape[k] != F.shape[k]) fail(CTD_ERR_SHAPE, "factor shape does not match the tensor");
    Fibers fb;
    {
      PhaseScope ps(&ctx->c, PH_MATRICIZE);
      matricize(&ctx->c, x->t, F.mode, fb);
    }
    {
      PhaseScope ps(&ctx->c, PH_ERROR);
      *out = (F.has_core && F.core_from_stream) ? relative_error_core(&ctx->c, fb, *F.basis, F.core)
                                                : relative_error(&ctx->c, fb, *F.basis);
    }
    ctx->c.phase_flush();
  });
}

int ctd_gpu_memory_usage(const ctd_gpu_tensor* x, const ctd_gpu_factors* f, double* out) {
  return guarded([&] {
    need(x, "x");
    need(f, "factors");
    bind_device(f->f.ctx);
    need(out, "out");
    if (x->t.nnz == 0) fail(CTD_ERR_METRIC, "memory usage undefined for an empty tensor");  // evaluation.cpp:125-126
    const Factors& F = f->f;
    if (!F.has_core) fail(CTD_ERR_ARGUMENT, "memory_usage needs nnz(C): compute the factors with CTD_GPU_WITH_CORE");
    // (nnz(C) + nnz(U) + nnz(R)) / nnz(X), nnz(U) = exact nonzeros (dense_matrix.cpp:24-29)
    const int64_t K = F.basis ? F.basis->K : 0;
    std::vector<double> u((size_t)K * K);
    if (K) basis_u(*F.basis, u.data());
    int64_t u_nnz = 0;
    for (double v : u) u_nnz += (v != 0.0);
    const int64_t r_nnz = F.basis ? F.basis->rnnz : 0;
    *out = (double)(F.core.nnz + u_nnz + r_nnz) / (double)x->t.nnz;
  });
}

int ctd_gpu_basis_create(ctd_gpu_ctx* ctx, int64_t dim, ctd_gpu_basis** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(out, "out");
    if (dim < 0) fail(CTD_ERR_ARGUMENT, "basis dimension must be non-negative");
    auto h = std::make_unique<ctd_gpu_basis>();
    h->ctx = &ctx->c;
    h->b = std::make_unique<Basis>(&ctx->c, dim);
    h->b->want_panel = true;  // error partials over shards use the orthonormal panel (relerr.cu)
    *out = h.release();
  });
}

int ctd_gpu_basis_destroy(ctd_gpu_basis* b) {
  return guarded([&] { delete b; });
}

int64_t ctd_gpu_basis_size(const ctd_gpu_basis* b) { return b ? b->b->K : -1; }

int ctd_gpu_basis_try_append(ctd_gpu_basis* b, int64_t dim, int64_t nnz, const int64_t* idx, const double* val,
                             double epsilon, int32_t* accepted, int32_t* degenerate, double* delta, double* y) {
  return guarded([&] {
    need(b, "basis");
    bind_device(b->ctx);
    Basis& B = *b->b;
    Ctx* c = b->ctx;
    if (dim != B.dim) fail(CTD_ERR_SHAPE, "fiber length does not match basis");  // fiber_basis.cpp:45
    if (nnz < 0) fail(CTD_ERR_ARGUMENT, "negative nnz");
    std::vector<int32_t> r32(nnz > 0 ? nnz : 1);
    for (int64_t i = 0; i < nnz; ++i) {
      if (idx[i] < 0 || idx[i] >= dim) fail(CTD_ERR_SHAPE, "fiber index out of range");
      r32[i] = (int32_t)idx[i];
    }
    Buf<int32_t> drow(c, nnz + 1), dlen(c, 1);
    Buf<double> dval(c, nnz + 1);
    Buf<int64_t> doff(c, 1);
    const int64_t zero = 0;
    const int32_t len = (int32_t)nnz;
    c->to_dev(drow.p, r32.data(), nnz);
    if (nnz) c->to_dev(dval.p, val, nnz);
    c->to_dev(doff.p, &zero, 1);
    c->to_dev(dlen.p, &len, 1);
    Cands cd;
    cd.n = 1;
    cd.off = doff.p;
    cd.len = dlen.p;
    cd.row = drow.p;
    cd.val = dval.p;
    BatchOut bo;
    const int64_t k_before = B.K;
    filter_batch(B, cd, epsilon, bo, y != nullptr);
    if (accepted) *accepted = bo.accepted[0];
    if (degenerate) *degenerate = bo.degenerate[0];
    if (delta) *delta = bo.delta[0];
    if (y) std::memcpy(y, bo.y_last.data(), (size_t)k_before * sizeof(double));
  });
}

// ---- sharded CTD-S building blocks ----------------------------

int ctd_gpu_sample_fibers(ctd_gpu_ctx* ctx, int64_t n_fibers, const int64_t* fiber_col, const double* sq_norms,
                          int64_t sample_size, uint64_t seed, double* total_sq_norm, int64_t* unique,
                          int64_t* n_unique) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(unique, "unique");
    need(n_unique, "n_unique");
    if (sample_size < 1) fail(CTD_ERR_ARGUMENT, "sample size must be at least 1");  // sampling.cpp:36
    if (n_fibers < 0) fail(CTD_ERR_ARGUMENT, "negative fiber count");
    if (n_fibers == 0) fail(CTD_ERR_EMPTY_INPUT, "column distribution of an all-zero matrix");  // :22-23
    need(fiber_col, "fiber_col");
    need(sq_norms, "sq_norms");
    for (int64_t i = 1; i < n_fibers; ++i)
      if (fiber_col[i] <= fiber_col[i - 1]) fail(CTD_ERR_ARGUMENT, "fiber columns must be strictly ascending");
    Ctx* c = &ctx->c;
    const int64_t F = n_fibers;
    Buf<double> norm(c, F + 1), probs(c, F + 1), cum(c, F + 1), total(c, 1);
    c->to_dev(norm.p, sq_norms, F);
    {
      PhaseScope ps(c, PH_LAW);
      sampling_law(c, norm.p, F, total.p, probs.p, cum.p, c->d_flags);
    }
    Buf<int32_t> drawn(c, sample_size), uniq(c, sample_size);
    Buf<int> nu(c, 1);
    {
      PhaseScope ps(c, PH_SAMPLE);
      draw_fibers(c, cum.p, F, sample_size, seed, drawn.p);
      dedup_first(c, drawn.p, sample_size, uniq.p, nu.p);
    }
    int n_u = 0;
    c->to_host(&n_u, nu.p, 1);
    if (total_sq_norm) c->to_host(total_sq_norm, total.p, 1);
    c->sync();
    c->check_flags("sampling");
    std::vector<int32_t> u32(n_u > 0 ? n_u : 1);
    if (n_u) c->to_host(u32.data(), uniq.p, n_u);
    c->sync();
    for (int i = 0; i < n_u; ++i) unique[i] = fiber_col[u32[i]];
    *n_unique = n_u;
    c->phase_flush();
  });
}

namespace {
// device-side candidate checks: rows inside [0, dim) (FLAG_BOUNDS) and
// strictly ascending within a candidate (FLAG_DUPLICATE: not normalized)
__global__ void k_check_cands(Cands c, long long dim, unsigned* flags) {
  const long long k = blockIdx.x;
  if (k >= c.n) return;
  const long long off = c.off[k];
  const int len = c.len[k];
  bool oob = false, ord = false;
  for (int i = threadIdx.x; i < len; i += blockDim.x) {
    const int r = c.row[off + i];
    oob |= r < 0 || r >= dim;
    if (i > 0) ord |= r <= c.row[off + i - 1];
  }
  if (__syncthreads_or(oob) && threadIdx.x == 0) atomicOr(flags, FLAG_BOUNDS);
  if (__syncthreads_or(ord) && threadIdx.x == 0) atomicOr(flags, FLAG_DUPLICATE);
}
}  // namespace

int ctd_gpu_basis_append_batch_device(ctd_gpu_basis* b, int64_t n, const int64_t* cand_ptr, const int32_t* rows,
                                      const double* vals, double epsilon, int32_t* accepted, int32_t* degenerate,
                                      double* delta) {
  return guarded([&] {
    need(b, "basis");
    bind_device(b->ctx);
    if (n < 0) fail(CTD_ERR_ARGUMENT, "negative candidate count");
    if (n == 0) return;
    need(cand_ptr, "cand_ptr");
    Basis& B = *b->b;
    Ctx* c = b->ctx;
    if (cand_ptr[0] != 0) fail(CTD_ERR_ARGUMENT, "cand_ptr[0] must be 0");
    std::vector<int32_t> len(n);
    std::vector<int64_t> off(n);
    for (int64_t k = 0; k < n; ++k) {
      if (cand_ptr[k + 1] < cand_ptr[k]) fail(CTD_ERR_ARGUMENT, "cand_ptr must be non-decreasing");
      if (cand_ptr[k + 1] - cand_ptr[k] >= (int64_t(1) << 31)) fail(CTD_ERR_ARGUMENT, "candidate too long");
      off[k] = cand_ptr[k];
      len[k] = (int32_t)(cand_ptr[k + 1] - cand_ptr[k]);
    }
    if (cand_ptr[n] > 0) {
      need(rows, "rows");
      need(vals, "vals");
    }
    Buf<int32_t> dlen(c, n);
    Buf<int64_t> doff(c, n);
    c->to_dev(doff.p, off.data(), n);
    c->to_dev(dlen.p, len.data(), n);
    Cands cd;
    cd.n = n;
    cd.off = doff.p;
    cd.len = dlen.p;
    cd.row = rows;
    cd.val = vals;
    // the host path's checks (fiber_basis.cpp:45; rows ascending) on the device
    LAUNCH(c, k_check_cands, (unsigned)n, 128, 0, cd, (long long)B.dim, c->d_flags);
    c->check_flags("basis_append_batch_device");
    BatchOut bo;
    {
      PhaseScope ps(c, PH_FILTER);
      filter_batch(B, cd, epsilon, bo, false);
    }
    for (int64_t k = 0; k < n; ++k) {
      if (accepted) accepted[k] = bo.accepted[k];
      if (degenerate) degenerate[k] = bo.degenerate[k];
      if (delta) delta[k] = bo.delta[k];
    }
    c->phase_flush();
  });
}

int ctd_gpu_basis_append_batch(ctd_gpu_basis* b, int64_t n, const int64_t* cand_ptr, const int64_t* rows,
                               const double* vals, double epsilon, int32_t* accepted, int32_t* degenerate,
                               double* delta) {
  return guarded([&] {
    need(b, "basis");
    bind_device(b->ctx);
    if (n < 0) fail(CTD_ERR_ARGUMENT, "negative candidate count");
    if (n == 0) return;
    need(cand_ptr, "cand_ptr");
    Basis& B = *b->b;
    Ctx* c = b->ctx;
    if (cand_ptr[0] != 0) fail(CTD_ERR_ARGUMENT, "cand_ptr[0] must be 0");
    const int64_t nnz = cand_ptr[n];
    std::vector<int32_t> r32(nnz > 0 ? nnz : 1), len(n);
    std::vector<int64_t> off(n);
    for (int64_t k = 0; k < n; ++k) {
      if (cand_ptr[k + 1] < cand_ptr[k]) fail(CTD_ERR_ARGUMENT, "cand_ptr must be non-decreasing");
      if (cand_ptr[k + 1] - cand_ptr[k] >= (int64_t(1) << 31)) fail(CTD_ERR_ARGUMENT, "candidate too long");
      off[k] = cand_ptr[k];
      len[k] = (int32_t)(cand_ptr[k + 1] - cand_ptr[k]);
      for (int64_t i = cand_ptr[k]; i < cand_ptr[k + 1]; ++i) {
        if (rows[i] < 0 || rows[i] >= B.dim) fail(CTD_ERR_SHAPE, "fiber index out of range");  // :45
        if (i > cand_ptr[k] && rows[i] <= rows[i - 1]) fail(CTD_ERR_ARGUMENT, "fiber rows must ascend");
        r32[i] = (int32_t)rows[i];
      }
    }
    Buf<int32_t> drow(c, nnz + 1), dlen(c, n);
    Buf<double> dval(c, nnz + 1);
    Buf<int64_t> doff(c, n);
    if (nnz) {
      c->to_dev(drow.p, r32.data(), nnz);
      c->to_dev(dval.p, vals, nnz);
    }
    c->to_dev(doff.p, off.data(), n);
    c->to_dev(dlen.p, len.data(), n);
    Cands cd;
    cd.n = n;
    cd.off = doff.p;
    cd.len = dlen.p;
    cd.row = drow.p;
    cd.val = dval.p;
    BatchOut bo;
    {
      PhaseScope ps(c, PH_FILTER);
      filter_batch(B, cd, epsilon, bo, false);
    }
    for (int64_t k = 0; k < n; ++k) {
      if (accepted) accepted[k] = bo.accepted[k];
      if (degenerate) degenerate[k] = bo.degenerate[k];
      if (delta) delta[k] = bo.delta[k];
    }
    c->phase_flush();
  });
}

int64_t ctd_gpu_basis_r_nnz(const ctd_gpu_basis* b) { return b ? b->b->rnnz : -1; }

int ctd_gpu_basis_r(const ctd_gpu_basis* b, int64_t* col_ptr, int64_t* rows, double* vals) {
  return guarded([&] {
    need(b, "basis");
    bind_device(b->ctx);
    need(col_ptr, "col_ptr");
    basis_r(*b->b, col_ptr, rows, vals);
  });
}

int ctd_gpu_basis_error_partials(ctd_gpu_ctx* ctx, const ctd_gpu_basis* b, const ctd_gpu_tensor* x, int mode,
                                 double* x_sq, double* cross) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(b, "basis");
    bind_device(b->ctx);
    need(x, "x");
    need(x_sq, "x_sq");
    need(cross, "cross");
    if (mode < 0 || mode >= x->t.order) fail(CTD_ERR_ARGUMENT, "mode out of range");
    if (x->t.shape[mode] != b->b->dim) fail(CTD_ERR_SHAPE, "fiber length does not match basis");
    Fibers fb;
    {
      PhaseScope ps(&ctx->c, PH_MATRICIZE);
      matricize(&ctx->c, x->t, mode, fb);
    }
    {
      PhaseScope ps(&ctx->c, PH_ERROR);
      error_partials(&ctx->c, fb, *b->b, x_sq, cross);
    }
    ctx->c.phase_flush();
  });
}

namespace {
// copies candidate k's entries [src[k], src[k]+len[k]) to [dst[k], ...)
__global__ void k_gather_fibers(const int64_t* src, const int64_t* dst, const int64_t* len, const int32_t* row,
                                const double* val, int64_t* orow, double* oval) {
  const int k = blockIdx.x;
  const int64_t s = src[k], d = dst[k], n = len[k];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    orow[d + i] = row[s + i];
    oval[d + i] = val[s + i];
  }
}
__global__ void k_gather_fibers32(const int64_t* src, const int64_t* dst, const int64_t* len, const int32_t* row,
                                  const double* val, int32_t* orow, double* oval) {
  const int k = blockIdx.x;
  const int64_t s = src[k], d = dst[k], n = len[k];
  for (int64_t i = threadIdx.x; i < n; i += blockDim.x) {
    orow[d + i] = row[s + i];
    oval[d + i] = val[s + i];
  }
}
}  // namespace

int ctd_gpu_shard_create(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* x, int mode, ctd_gpu_shard** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(x, "x");
    need(out, "out");
    if (mode < 0 || mode >= x->t.order) fail(CTD_ERR_ARGUMENT, "mode out of range");
    auto h = std::make_unique<ctd_gpu_shard>();
    h->ctx = &ctx->c;
    {
      PhaseScope ps(&ctx->c, PH_MATRICIZE);
      matricize(&ctx->c, x->t, mode, h->fb);
    }
    const int64_t F = h->fb.F;
    h->col.resize(F);
    h->ptr.resize(F + 1);
    if (F) ctx->c.to_host(h->col.data(), h->fb.col.p, F);
    ctx->c.to_host(h->ptr.data(), h->fb.ptr.p, F + 1);
    ctx->c.sync();
    ctx->c.phase_flush();
    *out = h.release();
  });
}

int64_t ctd_gpu_shard_n_fibers(const ctd_gpu_shard* s) { return s ? s->fb.F : -1; }

int ctd_gpu_shard_fibers(const ctd_gpu_shard* s, int64_t* fiber_col, double* sq_norms) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    const int64_t F = s->fb.F;
    if (fiber_col && F) std::memcpy(fiber_col, s->col.data(), F * sizeof(int64_t));
    if (sq_norms && F) {
      s->ctx->to_host(sq_norms, s->fb.norm.p, F);
      s->ctx->sync();
    }
  });
}

int ctd_gpu_shard_gather(const ctd_gpu_shard* s, int64_t n, const int64_t* cols, int64_t* cand_ptr,
                         int64_t* rows, double* vals) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    need(cand_ptr, "cand_ptr");
    if (n < 0) fail(CTD_ERR_ARGUMENT, "negative count");
    std::vector<int64_t> src(n), len(n);
    cand_ptr[0] = 0;
    for (int64_t k = 0; k < n; ++k) {
      const auto it = std::lower_bound(s->col.begin(), s->col.end(), cols[k]);
      if (it == s->col.end() || *it != cols[k]) fail(CTD_ERR_ARGUMENT, "fiber not held by this shard");
      const int64_t f = it - s->col.begin();
      src[k] = s->ptr[f];
      len[k] = s->ptr[f + 1] - s->ptr[f];
      cand_ptr[k + 1] = cand_ptr[k] + len[k];
    }
    if (!rows || !vals || n == 0 || cand_ptr[n] == 0) return;
    Ctx* c = s->ctx;
    const int64_t tot = cand_ptr[n];
    Buf<int64_t> dsrc(c, n), ddst(c, n), dlen(c, n), orow(c, tot);
    Buf<double> oval(c, tot);
    c->to_dev(dsrc.p, src.data(), n);
    c->to_dev(ddst.p, cand_ptr, n);
    c->to_dev(dlen.p, len.data(), n);
    LAUNCH(c, k_gather_fibers, (unsigned)n, 128, 0, dsrc.p, ddst.p, dlen.p, s->fb.row.p, s->fb.val.p, orow.p,
           oval.p);
    c->to_host(rows, orow.p, tot);
    c->to_host(vals, oval.p, tot);
    c->sync();
  });
}

int ctd_gpu_shard_gather_device(const ctd_gpu_shard* s, int64_t n, const int64_t* cols, int64_t* cand_ptr,
                                int32_t* rows, double* vals) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    need(cand_ptr, "cand_ptr");
    if (n < 0) fail(CTD_ERR_ARGUMENT, "negative count");
    std::vector<int64_t> src(n), len(n);
    cand_ptr[0] = 0;
    for (int64_t k = 0; k < n; ++k) {
      const auto it = std::lower_bound(s->col.begin(), s->col.end(), cols[k]);
      if (it == s->col.end() || *it != cols[k]) fail(CTD_ERR_ARGUMENT, "fiber not held by this shard");
      const int64_t f = it - s->col.begin();
      src[k] = s->ptr[f];
      len[k] = s->ptr[f + 1] - s->ptr[f];
      cand_ptr[k + 1] = cand_ptr[k] + len[k];
    }
    if (!rows || !vals || n == 0 || cand_ptr[n] == 0) return;
    Ctx* c = s->ctx;
    Buf<int64_t> dsrc(c, n), ddst(c, n), dlen(c, n);
    c->to_dev(dsrc.p, src.data(), n);
    c->to_dev(ddst.p, cand_ptr, n);
    c->to_dev(dlen.p, len.data(), n);
    LAUNCH(c, k_gather_fibers32, (unsigned)n, 128, 0, dsrc.p, ddst.p, dlen.p, s->fb.row.p, s->fb.val.p, rows, vals);
    c->sync();
  });
}

int ctd_gpu_shard_find(const ctd_gpu_shard* s, int64_t n, const int64_t* cols, int64_t* pos) {
  return guarded([&] {
    need(s, "shard");
    if (n < 0) fail(CTD_ERR_ARGUMENT, "negative count");
    if (n == 0) return;
    need(cols, "cols");
    need(pos, "pos");
    for (int64_t k = 0; k < n; ++k) {
      const auto it = std::lower_bound(s->col.begin(), s->col.end(), cols[k]);
      pos[k] = (it != s->col.end() && *it == cols[k]) ? (int64_t)(it - s->col.begin()) : -1;
    }
  });
}

int ctd_gpu_shard_gather_into(const ctd_gpu_shard* s, int64_t n, const int64_t* cols, const int64_t* dst_off,
                              int32_t* rows, double* vals) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    if (n < 0) fail(CTD_ERR_ARGUMENT, "negative count");
    if (n == 0) return;
    need(cols, "cols");
    need(dst_off, "dst_off");
    std::vector<int64_t> src(n), len(n);
    int64_t tot = 0;
    for (int64_t k = 0; k < n; ++k) {
      const auto it = std::lower_bound(s->col.begin(), s->col.end(), cols[k]);
      if (it == s->col.end() || *it != cols[k]) fail(CTD_ERR_ARGUMENT, "fiber not held by this shard");
      if (dst_off[k] < 0) fail(CTD_ERR_ARGUMENT, "negative destination offset");
      const int64_t f = it - s->col.begin();
      src[k] = s->ptr[f];
      len[k] = s->ptr[f + 1] - s->ptr[f];
      tot += len[k];
    }
    if (tot == 0) return;
    need(rows, "rows");
    need(vals, "vals");
    Ctx* c = s->ctx;
    Buf<int64_t> dsrc(c, n), ddst(c, n), dlen(c, n);
    c->to_dev(dsrc.p, src.data(), n);
    c->to_dev(ddst.p, dst_off, n);
    c->to_dev(dlen.p, len.data(), n);
    LAUNCH(c, k_gather_fibers32, (unsigned)n, 128, 0, dsrc.p, ddst.p, dlen.p, s->fb.row.p, s->fb.val.p, rows, vals);
    c->sync();
  });
}

int ctd_gpu_shard_error_partials(const ctd_gpu_shard* s, const ctd_gpu_basis* b, double* x_sq, double* cross) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    need(b, "basis");
    bind_device(b->ctx);
    need(x_sq, "x_sq");
    need(cross, "cross");
    if (s->fb.rows != b->b->dim) fail(CTD_ERR_SHAPE, "fiber length does not match basis");
    PhaseScope ps(s->ctx, PH_ERROR);
    error_partials(s->ctx, s->fb, *b->b, x_sq, cross);
  });
}

int ctd_gpu_shard_core(ctd_gpu_shard* s, const ctd_gpu_basis* b, int64_t* c_cols, int64_t* c_nnz) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    need(b, "basis");
    if (s->fb.rows != b->b->dim) fail(CTD_ERR_SHAPE, "fiber length does not match basis");
    PhaseScope ps(s->ctx, PH_CORE);
    s->core = Core{};
    compute_core(s->ctx, s->fb, *b->b, s->core);
    s->has_core = true;
    if (c_cols) *c_cols = s->core.cols;
    if (c_nnz) *c_nnz = s->core.nnz;
  });
}

int ctd_gpu_shard_core_copy(const ctd_gpu_shard* s, int64_t* col_id, int64_t* col_ptr, int64_t* rows,
                            double* vals) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    if (!s->has_core) fail(CTD_ERR_ARGUMENT, "ctd_gpu_shard_core was not called on this shard");
    const Core& c = s->core;
    if (col_id && c.cols) std::memcpy(col_id, c.col_id.data(), c.cols * sizeof(int64_t));
    if (col_ptr) std::memcpy(col_ptr, c.ptr.data(), (c.cols + 1) * sizeof(int64_t));
    if (c.nnz && (rows || vals)) {
      if (vals) s->ctx->to_host(vals, c.val.p, c.nnz);
      std::vector<int32_t> r32(rows ? c.nnz : 0);
      if (rows) s->ctx->to_host(r32.data(), c.row.p, c.nnz);
      s->ctx->sync();
      for (int64_t i = 0; rows && i < c.nnz; ++i) rows[i] = r32[i];
    }
  });
}

// ---- compute_core / chain_product on caller-provided operands ----------------
int ctd_gpu_compute_core(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* x, int mode, int64_t r_rows, int64_t r_cols,
                         const int64_t* r_col_ptr, const int64_t* r_row, const double* r_val, ctd_gpu_csc** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(x, "x");
    need(out, "out");
    need(r_col_ptr, "r_col_ptr");
    Ctx* c = &ctx->c;
    if (mode < 0 || mode >= x->t.order) fail(CTD_ERR_ARGUMENT, "mode out of range");
    // ctd_static.cpp:14-15
    if (r_rows != x->t.shape[mode]) fail(CTD_ERR_SHAPE, "fiber matrix rows do not match the tensor extent");
    if (r_cols < 0) fail(CTD_ERR_ARGUMENT, "negative column count");
    PhaseScope ps(c, PH_CORE);
    Fibers fb;
    matricize(c, x->t, mode, fb);
    Basis B(c, r_rows);
    basis_load(B, r_cols, r_col_ptr, r_row, r_val, nullptr);
    auto h = std::make_unique<ctd_gpu_csc>();
    h->ctx = c;
    compute_core(c, fb, B, h->c);
    *out = h.release();
  });
}

int ctd_gpu_chain_product(ctd_gpu_ctx* ctx, int64_t dim, int64_t a_cols, const int64_t* dr_col_ptr,
                          const int64_t* dr_row, const double* dr_val, int64_t k, const int64_t* r_col_ptr,
                          const int64_t* r_row, const double* r_val, const double* u, int64_t c_cols,
                          const int64_t* c_col_ptr, const int64_t* c_row, const double* c_val, ctd_gpu_csc** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(out, "out");
    need(dr_col_ptr, "dr_col_ptr");
    need(r_col_ptr, "r_col_ptr");
    need(c_col_ptr, "c_col_ptr");
    Ctx* c = &ctx->c;
    if (dim < 0 || a_cols < 0 || k < 0 || c_cols < 0) fail(CTD_ERR_ARGUMENT, "negative extent");
    if (k > 0) need(u, "u");
    if (a_cols >= (1ll << 31)) fail(CTD_ERR_ARGUMENT, "too many appended columns");
    PhaseScope ps(c, PH_CORE);
    Basis B(c, dim);
    basis_load(B, k, r_col_ptr, r_row, r_val, u);
    // dR on the device (rows ascending within a column, inside dim)
    const int64_t dn = dr_col_ptr[a_cols];
    std::vector<int32_t> d32(dn > 0 ? dn : 1);
    for (int64_t a = 0; a < a_cols; ++a)
      for (int64_t t = dr_col_ptr[a]; t < dr_col_ptr[a + 1]; ++t) {
        if (dr_row[t] < 0 || dr_row[t] >= dim) fail(CTD_ERR_SHAPE, "dR row outside the fiber length");
        d32[t] = (int32_t)dr_row[t];
      }
    Buf<int64_t> dptr(c, a_cols + 1);
    Buf<int32_t> drow(c, dn + 1);
    Buf<double> dval(c, dn + 1);
    c->to_dev(dptr.p, dr_col_ptr, a_cols + 1);
    if (dn) {
      c->to_dev(drow.p, d32.data(), dn);
      c->to_dev(dval.p, dr_val, dn);
    }
    // C on the device (k rows)
    const int64_t cn = c_col_ptr[c_cols];
    std::vector<int32_t> c32(cn > 0 ? cn : 1);
    for (int64_t t = 0; t < cn; ++t) {
      if (c_row[t] < 0 || c_row[t] >= k) fail(CTD_ERR_SHAPE, "core row outside the basis size");
      c32[t] = (int32_t)c_row[t];
    }
    DevCore core;
    core.cols = c_cols;
    core.nnz = cn;
    core.ptr.alloc(c, c_cols + 1);
    core.row.alloc(c, cn + 1);
    core.val.alloc(c, cn + 1);
    c->to_dev(core.ptr.p, c_col_ptr, c_cols + 1);
    if (cn) {
      c->to_dev(core.row.p, c32.data(), cn);
      c->to_dev(core.val.p, c_val, cn);
    }
    Buf<double> ud(c, k > 0 ? (size_t)k * k : 1);
    if (k) c->to_dev(ud.p, u, (size_t)k * k);
    auto h = std::make_unique<ctd_gpu_csc>();
    h->ctx = c;
    h->row_shift = (int32_t)k;  // chain_product stores the rows as k + a
    chain_product(c, B, ud.p, (int)a_cols, dptr.p, drow.p, dval.p, core, h->c);
    c->sync();
    *out = h.release();
  });
}

int ctd_gpu_csc_info(const ctd_gpu_csc* m, int64_t* rows, int64_t* n_cols, int64_t* nnz) {
  return guarded([&] {
    need(m, "csc");
    if (rows) *rows = m->c.rows;
    if (n_cols) *n_cols = m->c.cols;
    if (nnz) *nnz = m->c.nnz;
  });
}

int ctd_gpu_csc_copy(const ctd_gpu_csc* m, int64_t* col_id, int64_t* col_ptr, int64_t* rows, double* vals) {
  return guarded([&] {
    need(m, "csc");
    bind_device(m->ctx);
    const Core& c = m->c;
    if (col_id && c.cols) std::memcpy(col_id, c.col_id.data(), c.cols * sizeof(int64_t));
    if (col_ptr) std::memcpy(col_ptr, c.ptr.data(), (c.cols + 1) * sizeof(int64_t));
    if (c.nnz && (rows || vals)) {
      if (vals) m->ctx->to_host(vals, c.val.p, c.nnz);
      std::vector<int32_t> r32(rows ? c.nnz : 0);
      if (rows) m->ctx->to_host(r32.data(), c.row.p, c.nnz);
      m->ctx->sync();
      for (int64_t i = 0; rows && i < c.nnz; ++i) rows[i] = (int64_t)r32[i] - m->row_shift;
    }
  });
}

int ctd_gpu_csc_destroy(ctd_gpu_csc* m) {
  return guarded([&] {
    if (!m) return;
    bind_device(m->ctx);
    delete m;
  });
}

// ---- CTD-D core over fiber-range shards ---------------------------------------
int ctd_gpu_core_shard_create(ctd_gpu_shard* hist, const ctd_gpu_basis* b, ctd_gpu_core_shard** out) {
  return guarded([&] {
    need(hist, "shard");
    need(b, "basis");
    need(out, "out");
    bind_device(hist->ctx);
    if (hist->fb.rows != b->b->dim) fail(CTD_ERR_SHAPE, "fiber length does not match basis");
    PhaseScope ps(hist->ctx, PH_CORE);
    auto c = std::make_unique<ctd_gpu_core_shard>();
    c->ctx = hist->ctx;
    Core st;
    compute_core(hist->ctx, hist->fb, *b->b, st);  // init_stream's core (ctd_dynamic.cpp:129-147)
    core_from_static(hist->ctx, st, c->core);
    *out = c.release();
  });
}

int ctd_gpu_core_shard_begin(ctd_gpu_core_shard* c, const ctd_gpu_basis* b) {
  return guarded([&] {
    need(c, "core shard");
    need(b, "basis");
    bind_device(c->ctx);
    const Basis& B = *b->b;
    c->Kold = B.K;
    if (B.K) {
      if (c->uold.n < (size_t)B.K * B.K) c->uold.alloc(c->ctx, (size_t)B.K * B.K * 3 / 2 + 1);
      CUDA_OK(cudaMemcpy2DAsync(c->uold.p, B.K * sizeof(double), B.U.p, B.LD * sizeof(double), B.K * sizeof(double),
                                B.K, cudaMemcpyDeviceToDevice, c->ctx->stream));
    }
  });
}

int ctd_gpu_core_shard_step(ctd_gpu_core_shard* c, const ctd_gpu_shard* slab, const ctd_gpu_basis* b,
                            int64_t col_offset) {
  return guarded([&] {
    need(c, "core shard");
    need(slab, "shard");
    need(b, "basis");
    bind_device(c->ctx);
    if (c->Kold < 0) fail(CTD_ERR_ARGUMENT, "ctd_gpu_core_shard_begin was not called before this step");
    if (slab->fb.rows != b->b->dim) fail(CTD_ERR_SHAPE, "fiber length does not match basis");
    if (b->b->K < c->Kold) fail(CTD_ERR_ARGUMENT, "the basis shrank since ctd_gpu_core_shard_begin");
    PhaseScope ps(c->ctx, PH_CORE);
    // Eq. 13 on this rank's columns: its old columns gain the bottom-left rows
    // ((dR^T R) U) C, its slab columns are R_new^T dX_p; dR from the basis
    core_step(c->ctx, c->core, slab->fb, *b->b, c->Kold, c->uold.p, {}, col_offset, true);
    c->Kold = -1;
  });
}

int ctd_gpu_core_shard_copy(const ctd_gpu_core_shard* c, int64_t* c_cols, int64_t* c_nnz, int64_t* col_id,
                            int64_t* col_ptr, int64_t* rows, double* vals) {
  return guarded([&] {
    need(c, "core shard");
    bind_device(c->ctx);
    const DevCore& d = c->core;
    if (c_cols) *c_cols = d.cols;
    if (c_nnz) *c_nnz = d.nnz;
    Ctx* cx = c->ctx;
    if (col_id && d.cols) cx->to_host(col_id, d.col.p, d.cols);
    if (col_ptr) cx->to_host(col_ptr, d.ptr.p, d.cols + 1);
    if (d.nnz && (rows || vals)) {
      if (vals) cx->to_host(vals, d.val.p, d.nnz);
      std::vector<int32_t> r32(rows ? d.nnz : 0);
      if (rows) cx->to_host(r32.data(), d.row.p, d.nnz);
      cx->sync();
      for (int64_t i = 0; rows && i < d.nnz; ++i) rows[i] = r32[i];
    }
    cx->sync();
  });
}

int ctd_gpu_core_shard_destroy(ctd_gpu_core_shard* c) {
  return guarded([&] {
    if (!c) return;
    bind_device(c->ctx);
    delete c;
  });
}

// ---- the sampling law chained across fiber-range shards ---------------------
namespace {

// cum[0..n] of [start, x[0], ..., x[n-1]]: the reference's sequential sum
// resumed from `start` (the running value at the end of the earlier shards).
void seq_from(Ctx* c, double start, const double* x, int64_t n, Buf<double>& ext, double* end) {
  ext.alloc(c, n + 1);
  c->to_dev(ext.p, &start, 1);
  if (n > 0)
    CUDA_OK(cudaMemcpyAsync(ext.p + 1, x, n * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
  Buf<double> out(c, n + 1), tot(c, 1);
  seq_cumsum(c, ext.p, n + 1, out.p, tot.p);
  *end = c->read1(tot.p);
  ext = std::move(out);
}

__global__ void k_shard_draw(const uint64_t* raw, long long count, double lo, double hi, const double* cum,
                             long long F, const int64_t* fcol, int64_t* out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= count) return;
  const double u = (double)(raw[i] >> 11) * (1.0 / 9007199254740992.0);  // sampling.cpp:15-17
  int64_t col = -1;
  if (u >= lo && u < hi) {  // upper_bound (sampling.cpp:59-61) lands in this shard
    long long a = 0, b = F;
    while (a < b) {
      const long long m = (a + b) >> 1;
      if (cum[m] > u) b = m;
      else a = m + 1;
    }
    col = a < F ? fcol[a] : -1;
  }
  out[i] = col;
}

}  // namespace

int ctd_gpu_shard_seq_total(const ctd_gpu_shard* s, double start, double* total) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    need(total, "total");
    Buf<double> ext;
    seq_from(s->ctx, start, s->fb.norm.p, s->fb.F, ext, total);
  });
}

int ctd_gpu_shard_cdf(ctd_gpu_shard* s, double total, double start, double* end, int* has_positive) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    need(end, "end");
    if (!(total > 0.0)) fail(CTD_ERR_EMPTY_INPUT, "sampling from an all-zero distribution");
    Ctx* c = s->ctx;
    const int64_t F = s->fb.F;
    Buf<double> pr(c, F + 1), dt(c, 1);
    c->to_dev(dt.p, &total, 1);
    s->last_pos.alloc(c, 1);
    probs_from_norms(c, s->fb.norm.p, F, dt.p, pr.p, s->last_pos.p);
    Buf<double> ext;
    seq_from(c, start, pr.p, F, ext, end);
    s->cum.alloc(c, F + 1);
    if (F > 0) CUDA_OK(cudaMemcpyAsync(s->cum.p, ext.p + 1, F * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    const int lp = c->read1(s->last_pos.p);
    if (has_positive) *has_positive = lp >= 0;
    s->cum_lo = start;
    s->cum_hi = *end;
  });
}

int ctd_gpu_shard_clamp(ctd_gpu_shard* s) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    if (!s->cum.p || !s->last_pos.p) fail(CTD_ERR_ARGUMENT, "ctd_gpu_shard_cdf first");
    clamp_from(s->ctx, s->cum.p, s->fb.F, s->last_pos.p);
    s->cum_hi = 1.0;
  });
}

int ctd_gpu_shard_draw(const ctd_gpu_shard* s, int64_t count, uint64_t seed, int64_t* cols) {
  return guarded([&] {
    need(s, "shard");
    bind_device(s->ctx);
    if (count < 0) fail(CTD_ERR_ARGUMENT, "sample count must be non-negative");
    if (count == 0) return;
    need(cols, "cols");
    if (!s->cum.p) fail(CTD_ERR_ARGUMENT, "ctd_gpu_shard_cdf first");
    Ctx* c = s->ctx;
    Buf<uint64_t> raw(c, count);
    mt19937_64(c, seed, count, raw.p);
    Buf<int64_t> out(c, count);
    LAUNCH(c, k_shard_draw, ceil_div(count, 256), 256, 0, raw.p, (long long)count, s->cum_lo, s->cum_hi, s->cum.p,
           (long long)s->fb.F, s->fb.col.p, out.p);
    c->to_host(cols, out.p, count);
    c->sync();
  });
}

int ctd_gpu_shard_destroy(ctd_gpu_shard* s) {
  return guarded([&] { delete s; });
}

int ctd_gpu_basis_u(const ctd_gpu_basis* b, double* u) {
  return guarded([&] {
    need(b, "basis");
    bind_device(b->ctx);
    need(u, "u");
    basis_u(*b->b, u);
  });
}

int ctd_gpu_stream_init(ctd_gpu_ctx* ctx, const ctd_gpu_tensor* historical, int mode, int64_t sample_size,
                        double epsilon, uint64_t seed, unsigned flags, ctd_gpu_stream** out) {
  return guarded([&] {
    need(ctx, "ctx");
    bind_device(&ctx->c);
    need(historical, "historical");
    need(out, "out");
    auto h = std::make_unique<ctd_gpu_stream>();
    stream_init(&ctx->c, historical->t, mode, sample_size, epsilon, seed, flags, h->s);
    *out = h.release();
  });
}

int ctd_gpu_stream_step(ctd_gpu_stream* s, const ctd_gpu_tensor* slab, int64_t sample_size) {
  return guarded([&] {
    need(s, "stream");
    bind_device(s->s.ctx);
    need(slab, "slab");
    stream_step(s->s, slab->t, sample_size);
  });
}

int64_t ctd_gpu_stream_t(const ctd_gpu_stream* s) { return s ? s->s.t : -1; }
int64_t ctd_gpu_stream_n_kept(const ctd_gpu_stream* s) { return s ? (int64_t)s->s.kept_flat.size() : -1; }

int ctd_gpu_stream_factors(ctd_gpu_stream* s, ctd_gpu_factors** out) {
  return guarded([&] {
    need(s, "stream");
    bind_device(s->s.ctx);
    need(out, "out");
    // Snapshot: kept ids and a copy of the basis (R, U).
    auto h = std::make_unique<ctd_gpu_factors>();
    Factors& F = h->f;
    const Stream& S = s->s;
    F.ctx = S.ctx;
    F.order = S.order;
    F.mode = S.mode;
    for (int k = 0; k + 1 < S.order; ++k) F.shape[k] = S.slab_shape[k];
    F.shape[S.order - 1] = S.t;
    F.eps = S.eps;
    F.seed = S.seed;
    F.rows = S.basis->dim;
    F.kept_flat = S.kept_flat;
    // copy the basis state needed by the accessors (R, U)
    auto nb = std::make_unique<Basis>(S.ctx, S.basis->dim);
    const Basis& B = *S.basis;
    Ctx* c = S.ctx;
    nb->K = B.K;
    nb->LD = B.K > 0 ? B.K : 1;
    nb->U.alloc(c, (size_t)nb->LD * nb->LD);
    if (B.K)
      CUDA_OK(cudaMemcpy2DAsync(nb->U.p, B.K * sizeof(double), B.U.p, B.LD * sizeof(double), B.K * sizeof(double),
                                B.K, cudaMemcpyDeviceToDevice, c->stream));
    nb->kcap = B.K;
    nb->rptr.alloc(c, B.K + 1);
    CUDA_OK(cudaMemcpyAsync(nb->rptr.p, B.rptr.p, (B.K + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice, c->stream));
    nb->rnnz = nb->rcap = B.rnnz;
    nb->rrow.alloc(c, B.rnnz + 1);
    nb->rval.alloc(c, B.rnnz + 1);
    if (B.rnnz) {
      CUDA_OK(cudaMemcpyAsync(nb->rrow.p, B.rrow.p, B.rnnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(nb->rval.p, B.rval.p, B.rnnz * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    // R's row index (relative_error's R U panel reads it)
    if (B.rowbase.p && B.ricap > 0) {
      nb->ricap = B.ricap;
      nb->rowbase.alloc(c, B.dim + 1);
      nb->rowlen.alloc(c, B.dim + 1);
      nb->rek.alloc(c, B.ricap);
      nb->rev.alloc(c, B.ricap);
      CUDA_OK(cudaMemcpyAsync(nb->rowbase.p, B.rowbase.p, (B.dim + 1) * sizeof(int64_t), cudaMemcpyDeviceToDevice,
                              c->stream));
      CUDA_OK(cudaMemcpyAsync(nb->rowlen.p, B.rowlen.p, B.dim * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                              c->stream));
      CUDA_OK(cudaMemcpyAsync(nb->rek.p, B.rek.p, B.ricap * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
      CUDA_OK(cudaMemcpyAsync(nb->rev.p, B.rev.p, B.ricap * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
    }
    F.basis = std::move(nb);
    if (S.with_core) {  // StreamState::factors folds the core (:114-127); kept matricized here
      stream_core_sync(s->s);
      const DevCore& dc = S.core;
      Core& cc = F.core;
      cc.rows = B.K;
      cc.cols = dc.cols;
      cc.nnz = dc.nnz;
      cc.col_id.resize(dc.cols);
      cc.ptr.resize(dc.cols + 1);
      if (dc.cols) c->to_host(cc.col_id.data(), dc.col.p, dc.cols);
      c->to_host(cc.ptr.data(), dc.ptr.p, dc.cols + 1);
      cc.row.alloc(c, dc.nnz + 1);
      cc.val.alloc(c, dc.nnz + 1);
      if (dc.nnz) {
        CUDA_OK(cudaMemcpyAsync(cc.row.p, dc.row.p, dc.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, c->stream));
        CUDA_OK(cudaMemcpyAsync(cc.val.p, dc.val.p, dc.nnz * sizeof(double), cudaMemcpyDeviceToDevice, c->stream));
      }
      c->sync();
      F.has_core = true;
      F.core_from_stream = true;
    }
    *out = h.release();
  });
}

int ctd_gpu_stream_core_drift(ctd_gpu_stream* s, double* out) {
  return guarded([&] {
    need(s, "stream");
    bind_device(s->s.ctx);
    need(out, "out");
    *out = stream_core_drift(s->s);
  });
}

int ctd_gpu_stream_core_pending(const ctd_gpu_stream* s, int64_t* records, int64_t* entries, int64_t* bytes) {
  return guarded([&] {
    need(s, "stream");
    need(records, "records");
    need(entries, "entries");
    need(bytes, "bytes");
    *records = (int64_t)s->s.pending.size();
    *entries = s->s.pending_entries;
    *bytes = s->s.pending_bytes;
  });
}

int ctd_gpu_stream_core_sync(ctd_gpu_stream* s) {
  return guarded([&] {
    need(s, "stream");
    bind_device(s->s.ctx);
    stream_core_sync(s->s);
  });
}

int ctd_gpu_stream_destroy(ctd_gpu_stream* s) {
  return guarded([&] { delete s; });
}

}  // extern "C"
