// Drop-in for the reference C++ API (proj/core, namespace ctd): the hot-path
// entry points re-pointed at libctd_gpu.so through the C-ABI in
// include/ctd_gpu.h.  Compiled against the reference's own headers and linked
// into the reference library with
//
//   -Wl,--wrap=_ZN3ctd5ctd_sERKNS_12SparseTensorEildm                (ctd_s)
//   -Wl,--wrap=_ZN3ctd11init_streamERKNS_12SparseTensorEildmbb       (init_stream)
//   -Wl,--wrap=_ZN3ctd10ctd_d_stepENS_11StreamStateERKNS_12SparseTensorEl  (ctd_d_step)
//
// so every caller (stream_harness, ddos, tests, the Python/ctypes drivers)
// runs on the B200 without a source change; see oracle/Makefile `dropin` and
// INTEGRATION.md.  Everything else (SparseTensor, SparseMatrix, DenseMatrix,
// FiberBasis, fold, relative_error, memory_usage, ...) stays reference code.
//
// Entry points replaced (reference declarations):
//   ctd_s        include/ctd/ctd_static.hpp:22-24   (src/ctd_static.cpp:19-50)
//   init_stream  include/ctd/ctd_dynamic.hpp:42-45  (src/ctd_dynamic.cpp:129-147)
//   ctd_d_step   include/ctd/ctd_dynamic.hpp:57-58  (src/ctd_dynamic.cpp:149-229)
// Errors: the C-ABI status is the reference ErrorClass; it is rethrown as the
// matching ctd::*Error with ctd_gpu_last_error()'s message.
#include <cstdint>
#include <mutex>
#include <string>
#include <unordered_map>
#include <utility>
#include <vector>

#include "ctd/ctd_dynamic.hpp"
#include "ctd/ctd_static.hpp"
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
std::mutex g_mu;
std::unordered_map<const void*, ctd_gpu_stream*> g_streams;

void fill_state(StreamState& st, ctd_gpu_stream* s, int64_t kept_before) {
  Factors f;
  rethrow(ctd_gpu_stream_factors(s, &f.h));
  f.load_info();
  const auto flat = f.kept_flat();
  std::vector<index_t> grown(st.slab_shape);
  grown.push_back(ctd_gpu_stream_t(s));
  for (int64_t k = kept_before; k < (int64_t)flat.size(); ++k)
    st.kept_fibers.push_back(make_fiber_id(grown, st.mode, flat[k]));
  st.basis = FiberBasis(f.r(), f.u());
  st.core = f.core(ctd_gpu_stream_t(s) * st.slab_columns());
  st.t = ctd_gpu_stream_t(s);
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

}  // namespace

}  // namespace ctd

using namespace ctd;

extern "C" {

LRFactors __wrap__ZN3ctd5ctd_sERKNS_12SparseTensorEildm(const SparseTensor& x, int mode, index_t sample_size,
                                                       double epsilon, std::uint64_t seed) {
  Tensor t(x);
  Factors f;
  rethrow(ctd_gpu_ctd_s(context(), t.h, mode, sample_size, epsilon, seed, CTD_GPU_WITH_CORE, &f.h));
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
  return out;
}

StreamState __wrap__ZN3ctd11init_streamERKNS_12SparseTensorEildmbb(const SparseTensor& historical, int mode,
                                                                  index_t sample_size, double epsilon,
                                                                  std::uint64_t seed, bool keep_history,
                                                                  bool exact_core) {
  Tensor t(historical);
  ctd_gpu_stream* s = nullptr;
  // exact_core: the device stream keeps its own history for the bottom-left
  // block (ctd_dynamic.cpp:207-211); the host copy below serves core_drift
  const unsigned flags = CTD_GPU_WITH_CORE | (exact_core ? CTD_GPU_EXACT_CORE : 0u);
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
  g_streams[st.kept_fibers.data()] = s;
  return st;
}

StreamState __wrap__ZN3ctd10ctd_d_stepENS_11StreamStateERKNS_12SparseTensorEl(StreamState state,
                                                                             const SparseTensor& slab,
                                                                             index_t sample_size) {
  ctd_gpu_stream* s = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_mu);
    auto it = g_streams.find(state.kept_fibers.data());
    if (it == g_streams.end())
      throw ArgumentError("stream state was not created by the GPU init_stream (or was copied)");
    s = it->second;
    g_streams.erase(it);
  }
  const int64_t before = (int64_t)state.kept_fibers.size();
  {
    Tensor t(slab);
    const int st = ctd_gpu_stream_step(s, t.h, sample_size);
    if (st != CTD_OK) {
      std::lock_guard<std::mutex> lk(g_mu);
      g_streams[state.kept_fibers.data()] = s;
      rethrow(st);
    }
  }
  fill_state(state, s, before);
  if (state.history) state.history = append_time(*state.history, slab);
  std::lock_guard<std::mutex> lk(g_mu);
  g_streams[state.kept_fibers.data()] = s;
  return state;
}

}  // extern "C"
