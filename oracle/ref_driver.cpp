// TEST INFRASTRUCTURE ONLY — never linked into or called by the product path.
//
// extern "C" driver around the *unmodified* reference library compiled from
// /root/reference/proj/core/src (see oracle/Makefile).  It lets the pytest
// parity suite and bench.py's cpu_baseline leg call the reference's own
// public C++ API (ctd::ctd_s, ctd::init_stream, ctd::ctd_d_step, ...) through
// ctypes.  Every function here only marshals arguments; all arithmetic is the
// reference's.
//
// Errors: every entry point returns 0 or the reference ErrorClass value
// (error.hpp:11-19) of the exception it caught; 99 = any other exception.

#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "ctd/ctd_dynamic.hpp"
#include "ctd/ctd_static.hpp"
#include "ctd/ddos.hpp"
#include "ctd/factor_io.hpp"
#include "ctd/error.hpp"
#include "ctd/evaluation.hpp"
#include "ctd/fiber_basis.hpp"
#include "ctd/sampling.hpp"
#include "ctd/stream_harness.hpp"
#include "ctd/tensor_ops.hpp"

using namespace ctd;

namespace {
thread_local std::string g_msg;

template <typename F>
int guard(F&& f) {
  try {
    f();
    return 0;
  } catch (const ctd::Error& e) {
    g_msg = e.what();
    return static_cast<int>(e.error_class());
  } catch (const std::exception& e) {
    g_msg = e.what();
    return 99;
  }
}

// Flattened view of an LRFactors (or of a front-end trace) for ctypes.
struct Factors {
  LRFactors f;
  // front-end trace (only filled by ref_frontend)
  std::vector<index_t> drawn, unique;
  std::vector<int> accepted, degenerate;
  std::vector<double> delta;
  std::vector<double> norms, probs;
  double total = 0.0;
  double seconds = 0.0;
};
}  // namespace

extern "C" {

const char* ref_last_error() { return g_msg.c_str(); }

// ---- SparseTensor --------------------------------------------------------
int ref_tensor_new(int order, const int64_t* shape, int64_t nnz,
                   const int64_t* idx, const double* vals, void** out) {
  return guard([&] {
    std::vector<index_t> sh(shape, shape + order);
    std::vector<index_t> ix(idx, idx + nnz * order);
    std::vector<double> v(vals, vals + nnz);
    *out = new SparseTensor(std::move(sh), std::move(ix), std::move(v));
  });
}
void ref_tensor_free(void* t) { delete static_cast<SparseTensor*>(t); }
int64_t ref_tensor_nnz(void* t) { return static_cast<SparseTensor*>(t)->nnz(); }
void ref_tensor_data(void* t, int64_t* idx, double* vals) {
  auto* x = static_cast<SparseTensor*>(t);
  std::memcpy(idx, x->indices().data(), x->indices().size() * sizeof(int64_t));
  std::memcpy(vals, x->values().data(), x->values().size() * sizeof(double));
}

// ---- matricize / norms / sampling (tensor_ops.cpp, sampling.cpp) ---------
// matricize(x, mode) -> CSC; caller passes col_ptr[cols+1], row[nnz], val[nnz].
int ref_matricize(void* t, int mode, int64_t* col_ptr, int64_t* rows,
                  double* vals, double* sq_norms) {
  return guard([&] {
    const SparseMatrix m = matricize(*static_cast<SparseTensor*>(t), mode);
    const auto& cp = m.column_pointers();
    for (size_t i = 0; i < cp.size(); ++i) col_ptr[i] = static_cast<int64_t>(cp[i]);
    std::memcpy(rows, m.row_indices().data(), m.nnz() * sizeof(int64_t));
    std::memcpy(vals, m.values().data(), m.nnz() * sizeof(double));
    if (sq_norms) {
      const auto n = column_sq_norms(m);
      std::memcpy(sq_norms, n.data(), n.size() * sizeof(double));
    }
  });
}

int ref_column_distribution(void* t, int mode, double* probs, double* total) {
  return guard([&] {
    const SparseMatrix m = matricize(*static_cast<SparseTensor*>(t), mode);
    const ColumnDistribution d = column_distribution(m);
    std::memcpy(probs, d.probabilities.data(), d.probabilities.size() * sizeof(double));
    *total = d.total_sq_norm;
  });
}

int ref_sample_with_replacement(const double* probs, int64_t n, double total,
                                int64_t count, uint64_t seed, int64_t* out) {
  return guard([&] {
    ColumnDistribution d;
    d.probabilities.assign(probs, probs + n);
    d.total_sq_norm = total;
    const auto drawn = sample_with_replacement(d, count, seed);
    std::memcpy(out, drawn.data(), drawn.size() * sizeof(int64_t));
  });
}

int ref_unique_first_occurrence(const int64_t* in, int64_t n, int64_t* out,
                                int64_t* n_out) {
  return guard([&] {
    const auto u = unique_first_occurrence(std::span<const index_t>(in, n));
    std::memcpy(out, u.data(), u.size() * sizeof(int64_t));
    *n_out = static_cast<int64_t>(u.size());
  });
}

// ---- FiberBasis (fiber_basis.cpp) ----------------------------------------
int ref_basis_new(int64_t dim, void** out) {
  return guard([&] { *out = new FiberBasis(dim); });
}
void ref_basis_free(void* b) { delete static_cast<FiberBasis*>(b); }
int64_t ref_basis_size(void* b) { return static_cast<FiberBasis*>(b)->size(); }
void ref_basis_u(void* b, double* u) {
  const auto& m = static_cast<FiberBasis*>(b)->inverse_gram();
  std::memcpy(u, m.data().data(), m.data().size() * sizeof(double));
}
int ref_basis_try_append(void* b, int64_t dim, int64_t nnz, const int64_t* idx,
                         const double* val, double eps, int* accepted,
                         int* degenerate, double* delta, double* y) {
  return guard([&] {
    SparseVec x;
    x.dim = dim;
    x.idx.assign(idx, idx + nnz);
    x.val.assign(val, val + nnz);
    auto* basis = static_cast<FiberBasis*>(b);
    const auto r = basis->try_append_fiber(x, eps);
    *accepted = r.accepted;
    *degenerate = r.degenerate;
    *delta = r.delta;
    if (y) std::memcpy(y, r.y.data(), r.y.size() * sizeof(double));
  });
}

// ---- ctd_s (ctd_static.cpp) ---------------------------------------------
int ref_ctd_s(void* t, int mode, int64_t s, double eps, uint64_t seed,
              void** out) {
  return guard([&] {
    auto fx = std::make_unique<Factors>();
    const auto t0 = std::chrono::steady_clock::now();
    fx->f = ctd_s(*static_cast<SparseTensor*>(t), mode, s, eps, seed);
    fx->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    *out = fx.release();
  });
}

// Public-API composition of ctd_s minus compute_core (the reference's own
// test idiom, test_ctd_static.cpp:88-120): matricize -> column_distribution
// -> sample_with_replacement -> unique_first_occurrence -> FiberBasis loop.
// Records every decision so parity can be checked candidate by candidate.
int ref_frontend(void* t, int mode, int64_t s, double eps, uint64_t seed,
                 void** out) {
  return guard([&] {
    const SparseTensor& x = *static_cast<SparseTensor*>(t);
    auto fx = std::make_unique<Factors>();
    const auto t0 = std::chrono::steady_clock::now();
    const SparseMatrix unfolded = matricize(x, mode);
    const ColumnDistribution dist = column_distribution(unfolded);
    fx->drawn = sample_with_replacement(dist, s, seed);
    fx->unique = unique_first_occurrence(fx->drawn);
    FiberBasis basis(unfolded.rows());
    for (index_t j : fx->unique) {
      const auto r = basis.try_append_fiber(unfolded.column(j), eps);
      fx->accepted.push_back(r.accepted);
      fx->degenerate.push_back(r.degenerate);
      fx->delta.push_back(r.delta);
      if (r.accepted) fx->f.kept_fibers.push_back(make_fiber_id(x.shape(), mode, j));
    }
    fx->f.R = basis.to_matrix();
    fx->f.U = basis.inverse_gram();
    fx->seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    fx->f.mode = mode;
    fx->f.epsilon = eps;
    fx->f.seed = seed;
    fx->total = dist.total_sq_norm;
    fx->probs = dist.probabilities;
    *out = fx.release();
  });
}

void ref_factors_free(void* f) { delete static_cast<Factors*>(f); }
double ref_factors_seconds(void* f) { return static_cast<Factors*>(f)->seconds; }
int64_t ref_factors_kept(void* f) { return static_cast<Factors*>(f)->f.kept_count(); }
int64_t ref_factors_r_rows(void* f) { return static_cast<Factors*>(f)->f.R.rows(); }
int64_t ref_factors_r_nnz(void* f) { return static_cast<Factors*>(f)->f.R.nnz(); }
int64_t ref_factors_c_nnz(void* f) { return static_cast<Factors*>(f)->f.C.nnz(); }
int ref_factors_c_order(void* f) { return static_cast<Factors*>(f)->f.C.order(); }
void ref_factors_c_shape(void* f, int64_t* shape) {
  const auto& s = static_cast<Factors*>(f)->f.C.shape();
  for (size_t i = 0; i < s.size(); ++i) shape[i] = s[i];
}
void ref_factors_kept_flat(void* f, int64_t* out) {
  const auto& k = static_cast<Factors*>(f)->f.kept_fibers;
  for (size_t i = 0; i < k.size(); ++i) out[i] = k[i].flat;
}
void ref_factors_kept_coords(void* f, int64_t* out) {
  const auto& k = static_cast<Factors*>(f)->f.kept_fibers;
  size_t p = 0;
  for (const auto& id : k)
    for (auto c : id.coords) out[p++] = c;
}
void ref_factors_r(void* f, int64_t* col_ptr, int64_t* rows, double* vals) {
  const auto& r = static_cast<Factors*>(f)->f.R;
  const auto& cp = r.column_pointers();
  for (size_t i = 0; i < cp.size(); ++i) col_ptr[i] = static_cast<int64_t>(cp[i]);
  std::memcpy(rows, r.row_indices().data(), r.nnz() * sizeof(int64_t));
  std::memcpy(vals, r.values().data(), r.nnz() * sizeof(double));
}
void ref_factors_u(void* f, double* u) {
  const auto& m = static_cast<Factors*>(f)->f.U;
  std::memcpy(u, m.data().data(), m.data().size() * sizeof(double));
}
void ref_factors_c(void* f, int64_t* idx, double* vals) {
  const auto& c = static_cast<Factors*>(f)->f.C;
  std::memcpy(idx, c.indices().data(), c.indices().size() * sizeof(int64_t));
  std::memcpy(vals, c.values().data(), c.values().size() * sizeof(double));
}
int64_t ref_trace_len(void* f, int which) {
  auto* x = static_cast<Factors*>(f);
  return which == 0 ? (int64_t)x->drawn.size() : (int64_t)x->unique.size();
}
void ref_trace(void* f, int64_t* drawn, int64_t* unique, int* accepted,
               int* degenerate, double* delta) {
  auto* x = static_cast<Factors*>(f);
  std::memcpy(drawn, x->drawn.data(), x->drawn.size() * sizeof(int64_t));
  std::memcpy(unique, x->unique.data(), x->unique.size() * sizeof(int64_t));
  std::memcpy(accepted, x->accepted.data(), x->accepted.size() * sizeof(int));
  std::memcpy(degenerate, x->degenerate.data(), x->degenerate.size() * sizeof(int));
  std::memcpy(delta, x->delta.data(), x->delta.size() * sizeof(double));
}
double ref_trace_total(void* f) { return static_cast<Factors*>(f)->total; }

// ---- evaluation (evaluation.cpp) -----------------------------------------
int ref_relative_error(void* t, void* f, double* out) {
  return guard([&] {
    *out = relative_error(*static_cast<SparseTensor*>(t), static_cast<Factors*>(f)->f);
  });
}
int ref_memory_usage(void* t, void* f, double* out) {
  return guard([&] {
    *out = memory_usage(*static_cast<SparseTensor*>(t), static_cast<Factors*>(f)->f);
  });
}

// ---- CTD-D (ctd_dynamic.cpp) ---------------------------------------------
// Hooks of the GPU drop-in (paper_1710_03608_b200/shim): absent (null) in the
// plain CPU library.  The drop-in refreshes a StreamState's basis / core /
// history from the device lazily; these accessors read the fields directly.
extern "C" void ctd_shim_sync_state(void* state) __attribute__((weak));
extern "C" void ctd_shim_release_state(void* state) __attribute__((weak));
static StreamState* synced(void* s) {
  if (ctd_shim_sync_state) ctd_shim_sync_state(s);
  return static_cast<StreamState*>(s);
}
int ref_init_stream(void* hist, int mode, int64_t s, double eps, uint64_t seed,
                    int keep_history, int exact_core, void** out) {
  return guard([&] {
    *out = new StreamState(init_stream(*static_cast<SparseTensor*>(hist), mode, s,
                                       eps, seed, keep_history != 0, exact_core != 0));
  });
}
void ref_stream_free(void* s) {
  if (ctd_shim_release_state) ctd_shim_release_state(s);
  delete static_cast<StreamState*>(s);
}
int ref_stream_step(void* s, void* slab, int64_t d, double* seconds) {
  return guard([&] {
    auto* st = static_cast<StreamState*>(s);
    const auto t0 = std::chrono::steady_clock::now();
    *st = ctd_d_step(std::move(*st), *static_cast<SparseTensor*>(slab), d);
    if (seconds)
      *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
  });
}
int64_t ref_stream_t(void* s) { return static_cast<StreamState*>(s)->t; }
int ref_stream_factors(void* s, void** out) {
  return guard([&] {
    auto fx = std::make_unique<Factors>();
    fx->f = static_cast<StreamState*>(s)->factors();
    *out = fx.release();
  });
}
// Matricized core (basis.size() x t*slab_columns) as CSC.
int64_t ref_stream_core_nnz(void* s) { return synced(s)->core.nnz(); }
int64_t ref_stream_core_rows(void* s) { return synced(s)->core.rows(); }
int64_t ref_stream_core_cols(void* s) { return synced(s)->core.cols(); }
void ref_stream_core(void* s, int64_t* col_ptr, int64_t* rows, double* vals) {
  const auto& c = synced(s)->core;
  const auto& cp = c.column_pointers();
  for (size_t i = 0; i < cp.size(); ++i) col_ptr[i] = static_cast<int64_t>(cp[i]);
  std::memcpy(rows, c.row_indices().data(), c.nnz() * sizeof(int64_t));
  std::memcpy(vals, c.values().data(), c.nnz() * sizeof(double));
}
int ref_core_drift(void* s, double* out) {
  return guard([&] { *out = core_drift(*static_cast<StreamState*>(s)); });
}

// ---- stream harness (stream_harness.cpp) ----------------------------------
// Per-step reports of run_stream; arrays hold at least time-extent + 1 entries;
// mean4 = {error, memory, seconds, kept} of result.mean.
int ref_run_stream(void* t, int mode, int64_t s, int64_t d, double split, double eps, uint64_t seed,
                   int exact_core, int64_t* nsteps, int64_t* step, double* err, double* mem, double* secs,
                   int64_t* kept, double* mean4) {
  return guard([&] {
    HarnessOptions o;
    o.mode = mode;
    o.sample_size = s;
    if (d > 0) o.step_samples = d;
    o.split = split;
    o.epsilon = eps;
    o.seed = seed;
    o.exact_core = exact_core != 0;
    const StreamRunResult r = run_stream(*static_cast<SparseTensor*>(t), o);
    *nsteps = static_cast<int64_t>(r.steps.size());
    for (size_t i = 0; i < r.steps.size(); ++i) {
      step[i] = r.steps[i].step;
      err[i] = r.steps[i].eval.relative_error;
      mem[i] = r.steps[i].eval.memory_usage;
      secs[i] = r.steps[i].eval.wall_time_seconds;
      kept[i] = r.steps[i].eval.kept_fibers;
    }
    mean4[0] = r.mean.relative_error;
    mean4[1] = r.mean.memory_usage;
    mean4[2] = r.mean.wall_time_seconds;
    mean4[3] = static_cast<double>(r.mean.kept_fibers);
  });
}
int ref_tsv_line(int64_t step, double err, double secs, double mem, int64_t kept, char* buf, int64_t cap) {
  return guard([&] {
    EvalReport e;
    e.relative_error = err;
    e.wall_time_seconds = secs;
    e.memory_usage = mem;
    e.kept_fibers = kept;
    const std::string line = step < 0 ? tsv_header() : tsv_line(step, e);
    std::snprintf(buf, static_cast<size_t>(cap), "%s", line.c_str());
  });
}

// ---- factor bundles (factor_io.cpp) and DDoS post-processing (ddos.cpp) ----
int ref_save_factors(void* f, const char* dir) {
  return guard([&] { save_factors(static_cast<Factors*>(f)->f, dir); });
}
int ref_load_factors(const char* dir, void** out) {
  return guard([&] {
    auto fx = std::make_unique<Factors>();
    fx->f = load_factors(dir);
    *out = fx.release();
  });
}
// flagged candidates; arrays hold at least kept-count entries
int ref_detect_ddos(void* f, int64_t* n, int64_t* dst, int64_t* bin, double* norm) {
  return guard([&] {
    const auto c = detect_ddos(static_cast<Factors*>(f)->f);
    *n = static_cast<int64_t>(c.size());
    for (size_t i = 0; i < c.size(); ++i) {
      dst[i] = c[i].dst;
      bin[i] = c[i].bin;
      norm[i] = c[i].norm;
    }
  });
}
int ref_decompose_online(void* t, int mode, int64_t d, double eps, uint64_t seed, void** out) {
  return guard([&] {
    auto fx = std::make_unique<Factors>();
    fx->f = decompose_online(*static_cast<SparseTensor*>(t), mode, d, eps, seed);
    *out = fx.release();
  });
}

}  // extern "C"

// compute_core / chain_product on caller-given operands (test driver for the
// drop-in's compute_core and chain_product wrappers)
namespace {
SparseMatrix csc_of(int64_t rows, int64_t cols, const int64_t* cp, const int64_t* r, const double* v) {
  std::vector<index_t> ri, ci;
  std::vector<double> vv;
  for (int64_t j = 0; j < cols; ++j)
    for (int64_t t = cp[j]; t < cp[j + 1]; ++t) {
      ri.push_back(r[t]);
      ci.push_back(j);
      vv.push_back(v[t]);
    }
  return SparseMatrix(rows, cols, std::move(ri), std::move(ci), std::move(vv));
}
}  // namespace

extern "C" {
int ref_compute_core(void* t, int mode, int64_t r_rows, int64_t r_cols, const int64_t* cp, const int64_t* rows,
                     const double* vals, void** out) {
  return guard([&] {
    const SparseMatrix R = csc_of(r_rows, r_cols, cp, rows, vals);
    *out = new SparseTensor(compute_core(*static_cast<SparseTensor*>(t), R, mode));
  });
}
int ref_chain_product(int64_t dr_rows, int64_t a, const int64_t* dcp, const int64_t* drow, const double* dval,
                      int64_t r_rows, int64_t k, const int64_t* rcp, const int64_t* rrow, const double* rval,
                      int64_t u_rows, int64_t u_cols, const double* u, int64_t c_rows, int64_t c_cols,
                      const int64_t* ccp, const int64_t* crow, const double* cval, void** out) {
  return guard([&] {
    const SparseMatrix dR = csc_of(dr_rows, a, dcp, drow, dval);
    const SparseMatrix R = csc_of(r_rows, k, rcp, rrow, rval);
    DenseMatrix U(u_rows, u_cols);
    for (int64_t i = 0; i < u_rows; ++i)
      for (int64_t j = 0; j < u_cols; ++j) U.at(i, j) = u[i * u_cols + j];
    const SparseMatrix Cm = csc_of(c_rows, c_cols, ccp, crow, cval);
    *out = new SparseMatrix(chain_product(dR, R, U, Cm));
  });
}
void ref_matrix_free(void* m) { delete static_cast<SparseMatrix*>(m); }
void ref_matrix_shape(void* m, int64_t* rows, int64_t* cols, int64_t* nnz) {
  const auto* M = static_cast<SparseMatrix*>(m);
  *rows = M->rows();
  *cols = M->cols();
  *nnz = M->nnz();
}
void ref_matrix_data(void* m, int64_t* col_ptr, int64_t* rows, double* vals) {
  const auto* M = static_cast<SparseMatrix*>(m);
  const auto& cp = M->column_pointers();
  for (size_t j = 0; j < cp.size(); ++j) col_ptr[j] = (int64_t)cp[j];
  for (size_t t = 0; t < M->row_indices().size(); ++t) {
    rows[t] = M->row_indices()[t];
    vals[t] = M->values()[t];
  }
}
}
