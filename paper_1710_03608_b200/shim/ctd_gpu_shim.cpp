// Drop-in for the reference C++ API (proj/core, namespace ctd): the hot-path
// entry points re-pointed at libctd_gpu.so through the C-ABI in
// include/ctd_gpu.h.  Compiled against the reference's own headers and linked
// into the reference library with `ld --wrap=<mangled name>` for each symbol
// below (shim/Makefile), so every caller (stream_harness, ddos, tests, the
// Python/ctypes drivers) runs on the B200 without a source change; see
// INTEGRATION.md.
//
// Entry points replaced (reference declarations, include/ctd/...):
//   ctd_s                    ctd_static.hpp:22-24   (src/ctd_static.cpp:19-50)
//   init_stream              ctd_dynamic.hpp:42-45  (src/ctd_dynamic.cpp:129-147)
//   ctd_d_step               ctd_dynamic.hpp:57-58  (src/ctd_dynamic.cpp:149-229)
//   StreamState::factors     ctd_dynamic.hpp:38     (src/ctd_dynamic.cpp:114-127)
//   core_drift               ctd_dynamic.hpp:66     (src/ctd_dynamic.cpp:271-301)
//   relative_error           evaluation.hpp:39      (src/evaluation.cpp:88-122)
//   matricize                tensor_ops.hpp:21      (src/tensor_ops.cpp:118-135)
//   column_sq_norms          tensor_ops.hpp:39      (src/tensor_ops.cpp:194-202)
//   column_distribution      sampling.hpp:20        (src/sampling.cpp:21-31)
//   sample_with_replacement  sampling.hpp:27-28     (src/sampling.cpp:33-64)
//   unique_first_occurrence  sampling.hpp:31        (src/sampling.cpp:66-78)
//   compute_core             ctd_static.hpp:28      (src/ctd_static.cpp:12-17)
//   chain_product            ctd_dynamic.hpp:61-62  (src/ctd_dynamic.cpp:231-269)
// FiberBasis stays reference code: callers drive it one candidate at a time
// and read its STL members directly; the batched GPU filter is reached
// through ctd_s / init_stream / ctd_d_step above.
// memory_usage (evaluation.cpp:124-129) stays reference code: it counts the
// nonzeros of host objects the caller already holds.
//
// Device state: a CTD-D stream lives on the GPU (ctd_gpu_stream), keyed by
// the heap buffer of StreamState::kept_fibers (which survives the reference's
// move-in / return-out idiom).  ctd_d_step updates only t and kept_fibers;
// the basis, the matricized core and the retained history are refreshed from
// the device when the caller asks for them (factors(), core_drift(), or
// ctd_shim_sync_state() for code that reads the fields directly), so a step
// costs no O(core) or O(history) host copy.  Factors produced on the device
// stay registered (bounded LRU) so relative_error on them runs on the GPU;
// anything else falls back to the reference code (__real_).
// Errors: the C-ABI status is the reference ErrorClass; it is rethrown as the
// matching ctd::*Error with ctd_gpu_last_error()'s message.
#include <cstdint>
#include <list>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "ctd/ctd_dynamic.hpp"
#include "ctd/ctd_static.hpp"
#include "ctd/evaluation.hpp"
#include "ctd/sampling.hpp"
#include "ctd/error.hpp"
#include "ctd/factors.hpp"
#include "ctd/fiber_basis.hpp"
#include "ctd/tensor_ops.hpp"
#include "ctd_gpu.h"

namespace ctd {

namespace {

void rethrow(int st) {
  if (st == CTD_OK) return;
  const std::string m = ctd_gpu_last_error();
  switch (st) {
    case CTD_ERR_ARGUMENT: throw ArgumentError(m);
    case CTD_ERR_SHAPE: throw ShapeError(m);
    case CTD_ERR_EMPTY_INPUT: throw EmptyInputError(m);
    case CTD_ERR_METRIC: throw MetricError(m);
    // device / numeric failures (CTD_ERR_DEVICE, CTD_ERR_NUMERIC) have no
    // reference class: the status is carried through as the exit code.
    default: throw Error(static_cast<ErrorClass>(st), "libctd_gpu: " + m);
  }
}

ctd_gpu_ctx* context() {
  static ctd_gpu_ctx* c = [] {
    ctd_gpu_ctx* p = nullptr;
    rethrow(ctd_gpu_ctx_create(0, nullptr, &p));
    return p;
  }();
  return c;
}

struct Tensor {
  ctd_gpu_tensor* h = nullptr;
  explicit Tensor(const SparseTensor& x) {
    rethrow(ctd_gpu_tensor_from_host(context(), x.order(), x.shape().data(), x.nnz(), x.indices().data(),
                                     x.values().data(), &h));
  }
  ~Tensor() { ctd_gpu_tensor_destroy(h); }
};

struct Factors {
  ctd_gpu_factors* h = nullptr;
  ctd_gpu_factors_info info{};
  ~Factors() {
    if (h) ctd_gpu_factors_destroy(h);
  }
  void load_info() { rethrow(ctd_gpu_factors_info_get(h, &info)); }
  ctd_gpu_factors* release() {
    ctd_gpu_factors* p = h;
    h = nullptr;
    return p;
  }

  std::vector<int64_t> kept_flat() const {
    std::vector<int64_t> v(info.kept);
    if (info.kept) rethrow(ctd_gpu_factors_kept_flat(h, v.data()));
    return v;
  }
  SparseMatrix r() const {
    std::vector<int64_t> cp(info.kept + 1), rows(info.r_nnz);
    std::vector<double> vals(info.r_nnz);
    rethrow(ctd_gpu_factors_r(h, cp.data(), rows.data(), vals.data()));
    std::vector<index_t> ri, ci;
    ri.reserve(info.r_nnz);
    ci.reserve(info.r_nnz);
    for (int64_t k = 0; k < info.kept; ++k)
      for (int64_t t = cp[k]; t < cp[k + 1]; ++t) {
        ri.push_back(rows[t]);
        ci.push_back(k);
      }
    return SparseMatrix(info.r_rows, info.kept, std::move(ri), std::move(ci), std::move(vals));
  }
  DenseMatrix u() const {
    DenseMatrix m(info.kept, info.kept);
    std::vector<double> flat((size_t)info.kept * info.kept);
    if (info.kept) rethrow(ctd_gpu_factors_u(h, flat.data()));
    for (int64_t i = 0; i < info.kept; ++i)
      for (int64_t j = 0; j < info.kept; ++j) m.at(i, j) = flat[(size_t)i * info.kept + j];
    return m;
  }
  // the matricized core as a SparseMatrix with `cols` columns
  SparseMatrix core(index_t cols) const {
    int64_t nc = 0;
    rethrow(ctd_gpu_factors_core(h, &nc, nullptr, nullptr, nullptr, nullptr));
    std::vector<int64_t> col(nc), ptr(nc + 1), rows(info.c_nnz);
    std::vector<double> vals(info.c_nnz);
    rethrow(ctd_gpu_factors_core(h, &nc, col.data(), ptr.data(), rows.data(), vals.data()));
    std::vector<index_t> ri(rows.begin(), rows.end()), ci;
    ci.reserve(info.c_nnz);
    for (int64_t c = 0; c < nc; ++c)
      for (int64_t t = ptr[c]; t < ptr[c + 1]; ++t) ci.push_back(col[c]);
    return SparseMatrix(info.kept, cols, std::move(ri), std::move(ci), std::move(vals));
  }
};

index_t other_extents(const std::vector<index_t>& shape, int mode) {
  index_t p = 1;
  for (size_t k = 0; k < shape.size(); ++k)
    if ((int)k != mode) p *= shape[k];
  return p;
}

// GPU stream handles, keyed by the heap buffer of StreamState::kept_fibers:
// moving a StreamState (the reference's pass-by-value / return idiom) keeps
// that buffer, so the key follows the state through ctd_d_step calls.
struct StreamEntry {
  ctd_gpu_stream* s = nullptr;
  bool stale = false;                 // basis / core / t not refreshed since a step
  std::vector<SparseTensor> pending;  // slabs not yet appended to state.history
};
std::mutex g_mu;
std::unordered_map<const void*, StreamEntry> g_streams;

// Factors computed on the device, keyed like streams by kept_fibers' buffer;
// the last kFactorsKept stay resident for relative_error.
constexpr size_t kFactorsKept = 8;
std::list<std::pair<const void*, ctd_gpu_factors*>> g_factors;

void register_factors(const LRFactors& f, ctd_gpu_factors* h) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto it = g_factors.begin(); it != g_factors.end(); ++it)
    if (it->first == f.kept_fibers.data()) {
      ctd_gpu_factors_destroy(it->second);
      g_factors.erase(it);
      break;
    }
  g_factors.emplace_front(f.kept_fibers.data(), h);
  while (g_factors.size() > kFactorsKept) {
    ctd_gpu_factors_destroy(g_factors.back().second);
    g_factors.pop_back();
  }
}

ctd_gpu_factors* find_factors(const LRFactors& f) {
  std::lock_guard<std::mutex> lk(g_mu);
  for (auto& e : g_factors)
    if (e.first == f.kept_fibers.data() && !f.kept_fibers.empty()) return e.second;
  return nullptr;
}

SparseTensor append_time(const SparseTensor& head, const SparseTensor& slab) {
  std::vector<index_t> shape = head.shape();
  const size_t tm = shape.size() - 1;
  const index_t off = shape[tm];
  shape[tm] += slab.extent((int)tm);
  std::vector<index_t> idx = head.indices();
  std::vector<double> val = head.values();
  for (index_t i = 0; i < slab.nnz(); ++i) {
    const auto e = slab.index(i);
    for (size_t k = 0; k < e.size(); ++k) idx.push_back(k == tm ? e[k] + off : e[k]);
    val.push_back(slab.value(i));
  }
  return SparseTensor(std::move(shape), std::move(idx), std::move(val));
}

// The state's basis, core, t and history from the device (lazily, g_mu held).
void sync_locked(StreamState& st, StreamEntry& e) {
  if (e.stale) {
    Factors f;
    rethrow(ctd_gpu_stream_factors(e.s, &f.h));
    f.load_info();
    st.basis = FiberBasis(f.r(), f.u());
    st.t = ctd_gpu_stream_t(e.s);
    st.core = f.core(st.t * st.slab_columns());
    e.stale = false;
  }
  if (st.history && !e.pending.empty()) {
    for (const auto& slab : e.pending) st.history = append_time(*st.history, slab);
    e.pending.clear();
  }
}

StreamEntry* find_stream_locked(const StreamState& st) {
  auto it = g_streams.find(st.kept_fibers.data());
  return it == g_streams.end() ? nullptr : &it->second;
}

}  // namespace

}  // namespace ctd

using namespace ctd;

extern "C" {

LRFactors __wrap__ZN3ctd5ctd_sERKNS_12SparseTensorEildm(const SparseTensor& x, int mode, index_t sample_size,
                                                       double epsilon, std::uint64_t seed) {
  Tensor t(x);
  Factors f;
  rethrow(ctd_gpu_ctd_s(context(), t.h, mode, sample_size, epsilon, seed, CTD_GPU_WITH_CORE | CTD_GPU_KEEP_PANEL,
                        &f.h));
  f.load_info();
  LRFactors out;
  out.mode = mode;
  out.epsilon = epsilon;
  out.seed = seed;
  for (int64_t j : f.kept_flat()) out.kept_fibers.push_back(make_fiber_id(x.shape(), mode, j));
  out.R = f.r();
  out.U = f.u();
  std::vector<index_t> cshape = x.shape();
  cshape[(size_t)mode] = f.info.kept;
  out.C = fold(f.core(other_extents(x.shape(), mode)), mode, cshape);
  register_factors(out, f.release());
  return out;
}

StreamState __wrap__ZN3ctd11init_streamERKNS_12SparseTensorEildmbb(const SparseTensor& historical, int mode,
                                                                  index_t sample_size, double epsilon,
                                                                  std::uint64_t seed, bool keep_history,
                                                                  bool exact_core) {
  Tensor t(historical);
  ctd_gpu_stream* s = nullptr;
  // keep_history / exact_core: the device stream keeps its own history (the
  // bottom-left block, ctd_dynamic.cpp:207-211, and core_drift); the host
  // copy is appended lazily on sync
  // the core is kept as per-step records and assembled when read (bit-identical)
  const unsigned flags = CTD_GPU_WITH_CORE | CTD_GPU_LAZY_CORE | (exact_core ? CTD_GPU_EXACT_CORE : 0u) |
                        (keep_history ? CTD_GPU_KEEP_HISTORY : 0u);
  rethrow(ctd_gpu_stream_init(context(), t.h, mode, sample_size, epsilon, seed, flags, &s));
  StreamState st{FiberBasis(historical.extent(mode)), SparseMatrix(0, 0), historical.shape(), mode, 0, epsilon,
                 seed, {}};
  st.slab_shape.pop_back();
  st.kept_fibers.reserve(1);  // a stable, non-null key buffer
  {
    Factors f;
    rethrow(ctd_gpu_stream_factors(s, &f.h));
    f.load_info();
    for (int64_t j : f.kept_flat()) st.kept_fibers.push_back(make_fiber_id(historical.shape(), mode, j));
    st.basis = FiberBasis(f.r(), f.u());
    st.t = ctd_gpu_stream_t(s);
    st.core = f.core(st.t * st.slab_columns());
  }
  st.exact_core = exact_core;
  if (keep_history || exact_core) st.history = historical;  // ctd_dynamic.cpp:143
  std::lock_guard<std::mutex> lk(g_mu);
  g_streams[st.kept_fibers.data()].s = s;
  return st;
}

StreamState __wrap__ZN3ctd10ctd_d_stepENS_11StreamStateERKNS_12SparseTensorEl(StreamState state,
                                                                             const SparseTensor& slab,
                                                                             index_t sample_size) {
  StreamEntry e;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_streams.find(state.kept_fibers.data());
    if (it == g_streams.end())
      throw ArgumentError("stream state was not created by the GPU init_stream (or was copied)");
    e = std::move(it->second);
    g_streams.erase(it);
  }
  const int64_t before = (int64_t)state.kept_fibers.size();
  {
    Tensor t(slab);
    const int st = ctd_gpu_stream_step(e.s, t.h, sample_size);
    if (st != CTD_OK) {
      std::lock_guard<std::mutex> lk(g_mu);
      g_streams[state.kept_fibers.data()] = std::move(e);
      rethrow(st);
    }
  }
  // kept ids (flat ids on the grown shape, ctd_dynamic.cpp:184-185) and t now;
  // basis, core and history when asked for (sync_locked)
  {
    Factors f;
    rethrow(ctd_gpu_stream_factors(e.s, &f.h));
    f.load_info();
    std::vector<int64_t> flat(f.info.kept);
    if (f.info.kept) rethrow(ctd_gpu_factors_kept_flat(f.h, flat.data()));
    std::vector<index_t> grown(state.slab_shape);
    grown.push_back(ctd_gpu_stream_t(e.s));
    for (int64_t k = before; k < (int64_t)flat.size(); ++k)
      state.kept_fibers.push_back(make_fiber_id(grown, state.mode, flat[k]));
  }
  state.t = ctd_gpu_stream_t(e.s);
  e.stale = true;
  if (state.history) e.pending.push_back(slab);  // ctd_dynamic.cpp:225-226, appended on sync
  std::lock_guard<std::mutex> lk(g_mu);
  g_streams[state.kept_fibers.data()] = std::move(e);
  return state;
}

LRFactors __real__ZNK3ctd11StreamState7factorsEv(const StreamState* self);
LRFactors __wrap__ZNK3ctd11StreamState7factorsEv(const StreamState* self) {
  ctd_gpu_stream* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (StreamEntry* e = find_stream_locked(*self)) s = e->s;
  }
  if (!s) return __real__ZNK3ctd11StreamState7factorsEv(self);
  // the device snapshot (ctd_dynamic.cpp:114-127): R, U, the core folded
  // with time extent t, the state's kept fibers
  Factors f;
  rethrow(ctd_gpu_stream_factors(s, &f.h));
  f.load_info();
  LRFactors out;
  out.mode = self->mode;
  out.epsilon = self->epsilon;
  out.seed = self->seed;
  out.kept_fibers = self->kept_fibers;
  out.R = f.r();
  out.U = f.u();
  std::vector<index_t> shape(self->slab_shape);
  const index_t t = ctd_gpu_stream_t(s);
  shape.push_back(t);
  std::vector<index_t> cshape = shape;
  cshape[(size_t)self->mode] = f.info.kept;
  out.C = fold(f.core(t * self->slab_columns()), self->mode, cshape);
  register_factors(out, f.release());
  return out;
}

double __real__ZN3ctd10core_driftERKNS_11StreamStateE(const StreamState& state);
double __wrap__ZN3ctd10core_driftERKNS_11StreamStateE(const StreamState& state) {
  ctd_gpu_stream* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    if (StreamEntry* e = find_stream_locked(state)) s = e->s;
  }
  if (!s) return __real__ZN3ctd10core_driftERKNS_11StreamStateE(state);
  double out = 0.0;
  rethrow(ctd_gpu_stream_core_drift(s, &out));
  return out;
}

double __real__ZN3ctd14relative_errorERKNS_12SparseTensorERKNS_9LRFactorsE(const SparseTensor& x,
                                                                         const LRFactors& f);
double __wrap__ZN3ctd14relative_errorERKNS_12SparseTensorERKNS_9LRFactorsE(const SparseTensor& x,
                                                                         const LRFactors& f) {
  ctd_gpu_factors* h = find_factors(f);
  if (!h) return __real__ZN3ctd14relative_errorERKNS_12SparseTensorERKNS_9LRFactorsE(x, f);
  Tensor t(x);
  double out = 0.0;
  rethrow(ctd_gpu_relative_error(context(), t.h, h, &out));
  return out;
}

SparseMatrix __wrap__ZN3ctd9matricizeERKNS_12SparseTensorEi(const SparseTensor& x, int mode) {
  Tensor t(x);
  int64_t F = 0;
  rethrow(ctd_gpu_matricize(context(), t.h, mode, &F, nullptr, nullptr, nullptr, nullptr, nullptr));
  std::vector<int64_t> col(F), ptr(F + 1);
  std::vector<int32_t> r32(x.nnz());
  std::vector<double> vals(x.nnz());
  rethrow(ctd_gpu_matricize(context(), t.h, mode, &F, col.data(), ptr.data(), r32.data(), vals.data(), nullptr));
  std::vector<index_t> ri(r32.begin(), r32.end()), ci;
  ci.reserve(x.nnz());
  for (int64_t f = 0; f < F; ++f)
    for (int64_t q = ptr[f]; q < ptr[f + 1]; ++q) ci.push_back(col[f]);
  return SparseMatrix(x.extent(mode), other_extents(x.shape(), mode), std::move(ri), std::move(ci), std::move(vals));
}

std::vector<double> __wrap__ZN3ctd15column_sq_normsERKNS_12SparseMatrixE(const SparseMatrix& m) {
  const auto& cp = m.column_pointers();
  std::vector<int64_t> cp64(cp.begin(), cp.end());
  std::vector<double> out((size_t)m.cols());
  rethrow(ctd_gpu_column_sq_norms_csc(context(), m.rows(), m.cols(), cp64.data(), m.row_indices().data(),
                                      m.values().data(), out.data()));
  return out;
}

ColumnDistribution __wrap__ZN3ctd19column_distributionERKNS_12SparseMatrixE(const SparseMatrix& m) {
  const auto& cp = m.column_pointers();
  std::vector<int64_t> cp64(cp.begin(), cp.end());
  ColumnDistribution d;
  d.probabilities.assign((size_t)m.cols(), 0.0);
  rethrow(ctd_gpu_column_distribution_csc(context(), m.rows(), m.cols(), cp64.data(), m.row_indices().data(),
                                          m.values().data(), &d.total_sq_norm, d.probabilities.data()));
  return d;
}

std::vector<index_t> __wrap__ZN3ctd23sample_with_replacementERKNS_18ColumnDistributionElm(
    const ColumnDistribution& dist, index_t count, std::uint64_t seed) {
  std::vector<index_t> out(count > 0 ? (size_t)count : 0);
  rethrow(ctd_gpu_sample_with_replacement(context(), dist.probabilities.data(), (int64_t)dist.probabilities.size(),
                                          count, seed, out.data()));
  return out;
}

std::vector<index_t> __wrap__ZN3ctd23unique_first_occurrenceESt4spanIKlLm18446744073709551615EE(
    std::span<const index_t> drawn) {
  std::vector<index_t> out(drawn.size());
  int64_t n = 0;
  rethrow(ctd_gpu_unique_first_occurrence(context(), drawn.data(), (int64_t)drawn.size(), out.data(), &n));
  out.resize((size_t)n);
  return out;
}

namespace {
// A ctd_gpu_csc result as a reference SparseMatrix with `rows` x `cols`.
SparseMatrix from_csc(ctd_gpu_csc* h, index_t rows, index_t cols) {
  struct Guard {
    ctd_gpu_csc* h;
    ~Guard() { ctd_gpu_csc_destroy(h); }
  } g{h};
  int64_t r = 0, nc = 0, nz = 0;
  rethrow(ctd_gpu_csc_info(h, &r, &nc, &nz));
  std::vector<int64_t> col(nc), ptr(nc + 1), rr(nz);
  std::vector<double> vals(nz);
  rethrow(ctd_gpu_csc_copy(h, col.data(), ptr.data(), rr.data(), vals.data()));
  std::vector<index_t> ri(rr.begin(), rr.end()), ci;
  ci.reserve(nz);
  for (int64_t c = 0; c < nc; ++c)
    for (int64_t t = ptr[c]; t < ptr[c + 1]; ++t) ci.push_back(col[c]);
  return SparseMatrix(rows, cols, std::move(ri), std::move(ci), std::move(vals));
}
std::vector<int64_t> ptr64(const SparseMatrix& m) {
  const auto& cp = m.column_pointers();
  return std::vector<int64_t>(cp.begin(), cp.end());
}
}  // namespace

SparseTensor __wrap__ZN3ctd12compute_coreERKNS_12SparseTensorERKNS_12SparseMatrixEi(const SparseTensor& x,
                                                                                 const SparseMatrix& r, int mode) {
  if (mode < 0 || mode >= x.order())
    throw ArgumentError("mode " + std::to_string(mode) + " out of range for order " + std::to_string(x.order()));
  if (r.rows() != x.extent(mode)) throw ShapeError("fiber matrix rows do not match the tensor extent");  // :14-15
  Tensor t(x);
  const auto cp = ptr64(r);
  ctd_gpu_csc* h = nullptr;
  rethrow(ctd_gpu_compute_core(context(), t.h, mode, r.rows(), r.cols(), cp.data(), r.row_indices().data(),
                               r.values().data(), &h));
  std::vector<index_t> cshape = x.shape();
  cshape[(size_t)mode] = r.cols();
  return fold(from_csc(h, r.cols(), other_extents(x.shape(), mode)), mode, cshape);
}

SparseMatrix __wrap__ZN3ctd13chain_productERKNS_12SparseMatrixES2_RKNS_11DenseMatrixES2_(const SparseMatrix& delta_r,
                                                                                      const SparseMatrix& r,
                                                                                      const DenseMatrix& u,
                                                                                      const SparseMatrix& core) {
  if (delta_r.rows() != r.rows()) throw ShapeError("inner dimensions differ");  // transpose_times, :55
  if (r.cols() != u.rows() || u.cols() != core.rows())
    throw ShapeError("chain product dimension mismatch");  // :234-235
  const index_t k = r.cols();
  std::vector<double> uf((size_t)k * (size_t)k);
  for (index_t i = 0; i < k; ++i)
    for (index_t j = 0; j < k; ++j) uf[(size_t)i * (size_t)k + (size_t)j] = u.at(i, j);
  const auto dcp = ptr64(delta_r), rcp = ptr64(r), ccp = ptr64(core);
  ctd_gpu_csc* h = nullptr;
  rethrow(ctd_gpu_chain_product(context(), r.rows(), delta_r.cols(), dcp.data(), delta_r.row_indices().data(),
                                delta_r.values().data(), k, rcp.data(), r.row_indices().data(), r.values().data(),
                                uf.data(), core.cols(), ccp.data(), core.row_indices().data(), core.values().data(),
                                &h));
  return from_csc(h, delta_r.cols(), core.cols());
}

// For callers that read StreamState::basis / core / history directly (the
// reference's own test driver does): bring them up to date from the device.
void ctd_shim_sync_state(void* state) {
  auto& st = *static_cast<StreamState*>(state);
  std::lock_guard<std::mutex> lk(g_mu);
  if (StreamEntry* e = find_stream_locked(st)) sync_locked(st, *e);
}

// Releases the device stream behind a state the caller is about to destroy.
void ctd_shim_release_state(void* state) {
  auto& st = *static_cast<StreamState*>(state);
  std::lock_guard<std::mutex> lk(g_mu);
  auto it = g_streams.find(st.kept_fibers.data());
  if (it == g_streams.end()) return;
  ctd_gpu_stream_destroy(it->second.s);
  g_streams.erase(it);
}

}  // extern "C"
