#pragma once
#include "core.cuh"
#include "stream_core.cuh"
#include <cmath>
#include <memory>
#include <vector>

#include "bucket.cuh"
#include "filter.cuh"

namespace ctdgpu {

// LRFactors (factors.hpp:32-47) + the run trace used for parity.
struct Factors {
  Ctx* ctx = nullptr;
  int order = 0, mode = 0;
  int64_t shape[kMaxOrder] = {0};
  double eps = 0;
  uint64_t seed = 0;
  int64_t F = 0, cols = 0, rows = 0;
  std::vector<int64_t> drawn, unique, kept_flat;
  std::vector<int32_t> accepted, degenerate;
  std::vector<double> delta;
  std::unique_ptr<Basis> basis;
  double total = 0.0;
  double rel_error = NAN;
  double min_margin = INFINITY;
  bool integer_exact = false;
  bool slow_path = false;
  bool has_core = false;  // CTD_GPU_WITH_CORE: C_(mode) = R^T X_(mode)
  bool core_from_stream = false;  // C(t) of a CTD-D stream: relative_error uses it explicitly
  Core core;
};

// Algorithm 1 (ctd_static.cpp:19-50) minus compute_core; with
// CTD_GPU_WITH_ERROR also the relative-error pass.
void run_ctd_s(Ctx* ctx, const Tensor& x, int mode, int64_t s, double eps, uint64_t seed,
               unsigned flags, Factors& out);

// The pieces of the front end, exposed for parity tests.
struct Law {
  Fibers fb;
  Buf<double> probs, cum, total;
};
void build_law(Ctx* ctx, const Tensor& x, int mode, Law& law);

// StreamState (ctd_dynamic.hpp:18-39).
struct Stream {
  Ctx* ctx = nullptr;
  int order = 0, mode = 0;
  int64_t slab_shape[kMaxOrder] = {0};
  int64_t t = 0;
  double eps = 0;
  uint64_t seed = 0;
  std::unique_ptr<Basis> basis;
  std::vector<int64_t> kept_flat;
  bool with_core = false;  // CTD_GPU_WITH_CORE: maintain the Eq. 13 core
  DevCore core;
  // CTD_GPU_LAZY_CORE: each step records its core inputs (CoreRecord) and the
  // records are applied when the core is read (stream_core_sync)
  bool lazy_core = false;
  std::vector<CoreRecord> pending;
  CoreArena arena;
  int64_t pending_entries = 0, pending_bytes = 0;  // slab-column entries; 12/entry + 8 per left value
  Buf<double> uold;  // U^(t) snapshot for the core update (capacity grows)
  // retained raw history (StreamState::history, ctd_dynamic.hpp:28-32): the
  // concatenated slabs as device COO, `order` planes of hcap int32 indices
  bool keep_history = false, exact_core = false;
  Buf<int32_t> hidx;
  Buf<double> hval;
  int64_t hnnz = 0, hcap = 0;
  Tensor history() const;
};

double stream_core_drift(Stream& st);
// Applies the lazily recorded core updates (a no-op for an eager stream).
void stream_core_sync(Stream& st);

void stream_init(Ctx* ctx, const Tensor& hist, int mode, int64_t s, double eps, uint64_t seed,
                 unsigned flags, Stream& out);
void stream_step(Stream& st, const Tensor& slab, int64_t d);

}  // namespace ctdgpu
