#pragma once
#include <future>
#include <utility>
#include <vector>

#include "core.cuh"

namespace ctdgpu {

// The CTD-D stream's matricized core (StreamState::core, ctd_dynamic.hpp:18-39)
// as compressed CSC on the device: col[cols] global column ids ascending,
// ptr[cols+1], row[nnz] kept-fiber index ascending within a column, val[nnz].
struct DevCore {
  int64_t cols = 0, nnz = 0;
  Buf<int64_t> col, ptr;
  Buf<int32_t> row;
  Buf<double> val;
};

void core_from_static(Ctx* ctx, const Core& c, DevCore& out);

// The inputs of one core update, computed when the step runs (they depend on
// the basis and U of that moment) and applied to the core later: the slab's
// columns R_new^T dX (top-right + bottom-right) and the chain product's dense
// left factor W = (dR^T R_old) U_old (A x Kold), which the bottom-left block
// applies to the core as it stood before the step (the
// block-append core with the bottom-left kept as W and expanded lazily).
// Bump allocator over large device chunks for the records: they are kept
// until the core is read, so per-record pool allocations would fragment the
// stream-ordered pool and grow it at every step.  Chunks come from
// cudaMalloc: growing the stream-ordered pool by 1 GB costs ~12 ms (47 ms
// worst) on a B200, cudaMalloc ~0.6 ms (tools/alloc_probe.cu).
struct CoreArena {
  std::vector<std::pair<char*, size_t>> chunks;
  size_t used = 0;
  // the next chunk, allocated on a helper thread once the current one is half
  // used, so a step rarely waits on cudaMalloc (50-140 ms under load: the
  // stream's p99)
  std::future<std::pair<char*, size_t>> next;
  static constexpr size_t chunk_bytes = size_t(1) << 30;  // smallest chunk
  CoreArena() = default;
  CoreArena(const CoreArena&) = delete;
  CoreArena& operator=(const CoreArena&) = delete;
  ~CoreArena() { clear(); }
  void* take(Ctx* ctx, size_t bytes);
  void clear();  // synchronizes the device (cudaFree)
  size_t bytes() const;
};

struct CoreRecord {
  // slab columns R_new^T dX: col_id/ptr on the host, row/val in the arena
  int64_t cols = 0, nnz = 0;
  std::vector<int64_t> col_id, ptr;
  const int32_t* row = nullptr;
  const double* val = nullptr;
  const double* left = nullptr;  // [A][Kold] in the arena
  Core own_sc;                   // without an arena: the record owns its blocks
  Buf<double> own_left;
  int A = 0;
  int64_t Kold = 0;
  int64_t col_offset = 0;
};
// dr_from_basis: the appended fibers dR are read from the basis itself (its
// columns Kold..K-1, identical data) instead of fb -- a rank of a sharded
// stream owns only its part of the slab, while the basis is replicated.
void core_record(Ctx* ctx, const Fibers& fb, const Basis& B, int64_t Kold, const double* uold,
                 const std::vector<int32_t>& appended_fib, int64_t col_offset, CoreArena* arena,
                 CoreRecord& out, bool dr_from_basis = false);
void core_apply(Ctx* ctx, DevCore& core, const CoreRecord& rec);

// chain_product(dR, R, U, C) (ctd_dynamic.cpp:231-269) on its own: B holds R
// (its K columns and row index) and u U (K x K row-major, device), dR is A
// columns (dptr/drow/dval, device CSC over B.dim rows), core is C (K rows).
// out: the A x core.cols product over the columns that keep an entry; its
// rows are stored as K + a (the bottom-left block's rows in the grown core).
void chain_product(Ctx* ctx, const Basis& B, const double* u, int A, const int64_t* dptr, const int32_t* drow,
                   const double* dval, const DevCore& core, Core& out);

// One ctd_d_step core update (Eq. 13) = core_record + core_apply.  B is the basis after this step's
// appends, Kold its size before them and uold (Kold x Kold, row-major) U
// before them; appended_fib the appended candidates' fiber indices into fb in
// acceptance order; col_offset = t * slab_columns.
void core_step(Ctx* ctx, DevCore& core, const Fibers& fb, const Basis& B, int64_t Kold, const double* uold,
               const std::vector<int32_t>& appended_fib, int64_t col_offset, bool dr_from_basis = false);

// exact_core variant (ctd_dynamic.cpp:207-211): the bottom-left block is
// dR^T X_hist (transpose_times over the retained history's matricization hf,
// columns in the core's time-extended space) instead of the chain product;
// it may add entries to columns that are empty in the old core.
void core_step_exact(Ctx* ctx, DevCore& core, const Fibers& fb, const Fibers& hf, const Basis& B, int64_t Kold,
                     int64_t col_offset);

// core_drift (ctd_dynamic.cpp:271-301): sqrt of the sequential sum, over the
// columns ascending and each column's merged rows, of (c - e)^2 / c^2 / e^2
// between the maintained core and R^T X_hist.
double core_drift(Ctx* ctx, const DevCore& core, const Fibers& hf, const Basis& B);

}  // namespace ctdgpu
