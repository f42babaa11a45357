/* ctd_gpu.h — C-ABI of the B200-native CTD-S / CTD-D hot path.
 *
 * Drop-in boundary for the reference's proj/core C++ entry points (paths
 * relative to /root/reference/proj/core).  Each function below names the
 * reference interface it replaces.  Plain pointers and sizes only: no CUDA,
 * torch or C++ types cross this boundary (a cudaStream_t travels as void*).
 *
 * Status codes: 0 = ok, otherwise the reference ErrorClass value
 * (include/ctd/error.hpp:11-19) of the exception the reference would throw,
 * or CTD_ERR_DEVICE / CTD_ERR_NUMERIC for failures the CPU code cannot have.
 * ctd_gpu_last_error() returns the message of the last failure on the
 * calling thread.
 *
 * Threading: calls on one context are not
 * re-entrant; independent contexts may run concurrently on separate streams.
 * Results are deterministic: identical inputs give bit-identical kept fibers,
 * U and sampled ids on every run and every GPU count.
 */
#ifndef CTD_GPU_H
#define CTD_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum ctd_gpu_status {
  CTD_OK = 0,
  CTD_ERR_ARGUMENT = 1,    /* ArgumentError   error.hpp:32-35 */
  CTD_ERR_SHAPE = 2,       /* ShapeError      error.hpp:37-40 */
  CTD_ERR_EMPTY_INPUT = 3, /* EmptyInputError error.hpp:42-45 */
  CTD_ERR_PARSE = 4,       /* ParseError (unused on this path) */
  CTD_ERR_METRIC = 5,      /* MetricError     error.hpp:61-64 */
  CTD_ERR_ORACLE = 6,      /* OracleError (unused on this path) */
  CTD_ERR_IO = 7,          /* IoError (unused on this path) */
  CTD_ERR_DEVICE = 8,      /* CUDA / NCCL failure, out of device memory */
  CTD_ERR_NUMERIC = 9      /* internal exact-arithmetic self-check failed */
};

/* ctd_s flags */
#define CTD_GPU_WITH_ERROR 0x1u /* also run the relative-error pass (evaluation.cpp:88-122) */
#define CTD_GPU_WITH_CORE 0x2u  /* also materialize C = X x_mode R^T (ctd_static.cpp:12-17) */
#define CTD_GPU_KEEP_PANEL 0x4u /* keep the orthonormal panel W = R T for a later ctd_gpu_relative_error
                                   (implied by CTD_GPU_WITH_ERROR; ~2% of the filter's time) */
/* ctd_gpu_stream_init flags (init_stream's keep_history / exact_core,
   ctd_dynamic.hpp:42-45); both imply CTD_GPU_WITH_CORE */
#define CTD_GPU_KEEP_HISTORY 0x8u /* retain the raw history on the device (core_drift) */
#define CTD_GPU_EXACT_CORE 0x10u  /* bottom-left block from the history (ctd_dynamic.cpp:207-211) */
#define CTD_GPU_LAZY_CORE 0x20u   /* maintain the Eq. 13 core as recorded blocks (the slab's columns and the
                                     chain product's left factor (dR^T R) U per step), applied when the core
                                     is read (stream factors, core_drift); implies CTD_GPU_WITH_CORE */

typedef struct ctd_gpu_ctx ctd_gpu_ctx;         /* device, stream, scratch pool */
typedef struct ctd_gpu_tensor ctd_gpu_tensor;   /* SparseTensor (sparse_tensor.hpp:17-60) resident in HBM */
typedef struct ctd_gpu_factors ctd_gpu_factors; /* LRFactors (factors.hpp:32-47) + run trace */
typedef struct ctd_gpu_basis ctd_gpu_basis;     /* FiberBasis (fiber_basis.hpp:21-61) */
typedef struct ctd_gpu_stream ctd_gpu_stream;   /* StreamState (ctd_dynamic.hpp:18-39) */

const char *ctd_gpu_last_error(void);
const char *ctd_gpu_version(void);

/* ---- context ------------------------------------------------------------ */
/* stream: a cudaStream_t (NULL = legacy default stream).  All work of the
 * context is ordered on that stream. */
int ctd_gpu_ctx_create(int device, void *stream, ctd_gpu_ctx **out);
int ctd_gpu_ctx_set_stream(ctd_gpu_ctx *ctx, void *stream);
/* Returns the context's cached device blocks and the stream-ordered pool's
   unused reserve to the driver (for other allocators in the process, e.g.
   torch.cuda.empty_cache's counterpart). */
int ctd_gpu_ctx_trim(ctd_gpu_ctx *ctx);
int ctd_gpu_ctx_synchronize(ctd_gpu_ctx *ctx);
int ctd_gpu_ctx_destroy(ctd_gpu_ctx *ctx);
/* Launch counter of this library's kernels on the context (for bench.py). */
int64_t ctd_gpu_ctx_launches(const ctd_gpu_ctx *ctx);
/* Live per-phase timing with CUDA events recorded on the context stream
 * (bench.py's roofline): 8 phases, names from ctd_gpu_phase_name(i). */
int ctd_gpu_ctx_set_timing(ctd_gpu_ctx *ctx, int enable);
int ctd_gpu_ctx_phase_times(ctd_gpu_ctx *ctx, double *ms, int64_t *counts, int reset);
const char *ctd_gpu_phase_name(int i);

/* ---- tensors (SparseTensor, sparse_tensor.hpp:27-28) --------------------- */
/* Host COO exactly as SparseTensor::indices()/values() hold it: nnz*order
 * int64 coordinates row-concatenated, lexicographically sorted and coalesced
 * (a normalized SparseTensor).  Copied host->device and narrowed to int32 on
 * the device after a range check (ShapeError if any extent >= 2^31). */
int ctd_gpu_tensor_from_host(ctd_gpu_ctx *ctx, int order, const int64_t *shape,
                             int64_t nnz, const int64_t *indices,
                             const double *values, ctd_gpu_tensor **out);
/* Device-resident COO, structure of arrays: mode_indices[k] is a device
 * pointer to nnz int32 coordinates of mode k; values a device pointer to nnz
 * doubles.  The pointers are borrowed (not copied, not freed). */
int ctd_gpu_tensor_from_device(ctd_gpu_ctx *ctx, int order, const int64_t *shape,
                               int64_t nnz, const int32_t *const *mode_indices,
                               const double *values, ctd_gpu_tensor **out);
int64_t ctd_gpu_tensor_nnz(const ctd_gpu_tensor *t);
int ctd_gpu_tensor_destroy(ctd_gpu_tensor *t);

/* ---- tensor_ops / sampling pieces (parity surface) ---------------------- */
/* matricize + column_sq_norms (tensor_ops.hpp:21,39; tensor_ops.cpp:118-135,
 * 194-202).  Writes the mode-`mode` matricization in *compressed* CSC form:
 * only the nonempty fibers.  n_fibers receives F; fiber_col[F] the column
 * ids j, fiber_ptr[F+1] the offsets, rows[nnz]/vals[nnz] the entries in
 * (column,row) order, sq_norms[F] the exact squared norms.  Any output
 * pointer may be NULL; sizes: F <= nnz. */
int ctd_gpu_matricize(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *x, int mode,
                      int64_t *n_fibers, int64_t *fiber_col, int64_t *fiber_ptr,
                      int32_t *rows, double *vals, double *sq_norms);
/* column_distribution (sampling.hpp:20, sampling.cpp:21-31) restricted to
 * the nonempty fibers (every other column has probability exactly 0), and
 * the clamped cumulative array sample_with_replacement builds
 * (sampling.cpp:42-54), both bit-exact.  probs/cumulative have F entries. */
int ctd_gpu_column_distribution(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *x,
                                int mode, double *total_sq_norm, double *probs,
                                double *cumulative);
/* column_sq_norms (tensor_ops.hpp:39, tensor_ops.cpp:194-202) and
 * column_distribution (sampling.hpp:20, sampling.cpp:21-31) of a host matrix
 * in the reference's SparseMatrix layout (col_ptr[cols+1], rows ascending
 * per column, no stored zeros): out/probs have `cols` entries, bit-exact. */
int ctd_gpu_column_sq_norms_csc(ctd_gpu_ctx *ctx, int64_t rows, int64_t cols,
                                const int64_t *col_ptr, const int64_t *row_idx,
                                const double *vals, double *out);
int ctd_gpu_column_distribution_csc(ctd_gpu_ctx *ctx, int64_t rows, int64_t cols,
                                    const int64_t *col_ptr, const int64_t *row_idx,
                                    const double *vals, double *total_sq_norm,
                                    double *probs);
/* sample_with_replacement (sampling.hpp:27-28) over a host probability
 * vector of n columns (zero entries allowed). */
int ctd_gpu_sample_with_replacement(ctd_gpu_ctx *ctx, const double *probs,
                                    int64_t n, int64_t count, uint64_t seed,
                                    int64_t *out);
/* The exact sequential running sum used for the CDF, |x|^2 and the residual:
 * out[i] = fl(out[i-1] + x[i]) bit-exactly, x[i] >= 0 (host buffers). */
int ctd_gpu_seq_cumsum(ctd_gpu_ctx *ctx, const double *x, int64_t n, double *out);
/* unique_first_occurrence (sampling.hpp:31). */
int ctd_gpu_unique_first_occurrence(ctd_gpu_ctx *ctx, const int64_t *drawn,
                                    int64_t n, int64_t *out, int64_t *n_out);

/* ---- CTD-S (ctd_static.hpp:22-24) --------------------------------------- */
int ctd_gpu_ctd_s(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *x, int mode,
                  int64_t sample_size, double epsilon, uint64_t seed,
                  unsigned flags, ctd_gpu_factors **out);

typedef struct {
  int64_t kept;        /* s~ = kept_count()                     */
  int64_t r_rows;      /* I_alpha                                */
  int64_t r_nnz;       /* nnz(R)                                 */
  int64_t c_nnz;       /* nnz(C) (0 unless CTD_GPU_WITH_CORE)    */
  int64_t n_drawn;     /* s                                      */
  int64_t n_unique;    /* s'                                     */
  int64_t n_fibers;    /* F = nonempty mode-alpha fibers of X    */
  int64_t n_cols;      /* N_alpha                                */
  int64_t u_nnz;       /* exact nonzeros of U (dense_matrix.cpp:24-29) */
  int mode;
  int order;
  double epsilon;
  uint64_t seed;
  double total_sq_norm; /* |X|_F^2 as column_distribution computes it */
  double relative_error; /* NaN unless CTD_GPU_WITH_ERROR */
  double min_margin;     /* min |log10(ratio/eps)| over decisions */
  int integer_exact;     /* 1 if the exact-integer fast paths were used */
} ctd_gpu_factors_info;

int ctd_gpu_factors_info_get(const ctd_gpu_factors *f, ctd_gpu_factors_info *info);
/* FiberId.flat of every kept fiber, acceptance order (factors.hpp:17-22). */
int ctd_gpu_factors_kept_flat(const ctd_gpu_factors *f, int64_t *out);
/* R as CSC (kept+1, r_nnz, r_nnz), acceptance order (fiber_basis.cpp:111-124). */
int ctd_gpu_factors_r(const ctd_gpu_factors *f, int64_t *col_ptr, int64_t *rows,
                      double *vals);
/* U, kept x kept row-major (factors.hpp:34). */
int ctd_gpu_factors_u(const ctd_gpu_factors *f, double *u);
/* C_(mode) = R^T X_(mode) as CSC with kept rows and N_alpha columns
 * (compressed: only nonempty columns, c_cols receives their count). */
int ctd_gpu_factors_core(const ctd_gpu_factors *f, int64_t *c_cols,
                         int64_t *col_id, int64_t *col_ptr, int64_t *rows,
                         double *vals);
/* Run trace for parity: drawn[s], unique[s'], and per unique candidate the
 * try_append_fiber outcome (fiber_basis.hpp:30-37).  Any pointer may be NULL. */
int ctd_gpu_factors_trace(const ctd_gpu_factors *f, int64_t *drawn, int64_t *unique,
                          int32_t *accepted, int32_t *degenerate, double *delta);
int ctd_gpu_factors_destroy(ctd_gpu_factors *f);

/* relative_error (evaluation.hpp:39) of X against factors computed from it. */
int ctd_gpu_relative_error(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *x,
                           ctd_gpu_factors *f, double *out);
/* memory_usage (evaluation.hpp:42); needs CTD_GPU_WITH_CORE. */
int ctd_gpu_memory_usage(const ctd_gpu_tensor *x, const ctd_gpu_factors *f,
                         double *out);

/* ---- FiberBasis (fiber_basis.hpp:21-61) --------------------------------- */
int ctd_gpu_basis_create(ctd_gpu_ctx *ctx, int64_t dim, ctd_gpu_basis **out);
int ctd_gpu_basis_destroy(ctd_gpu_basis *b);
int64_t ctd_gpu_basis_size(const ctd_gpu_basis *b);
/* try_append_fiber (fiber_basis.cpp:43-109): host sparse vector (sorted
 * unique idx, no zeros).  y receives U R^T x (size() entries, may be NULL). */
int ctd_gpu_basis_try_append(ctd_gpu_basis *b, int64_t dim, int64_t nnz,
                             const int64_t *idx, const double *val, double epsilon,
                             int32_t *accepted, int32_t *degenerate, double *delta,
                             double *y);
int ctd_gpu_basis_u(const ctd_gpu_basis *b, double *u);

/* ---- sharded CTD-S building blocks (multi-GPU) ---------------
 * Each rank matricizes its own fiber range (ctd_gpu_matricize), the fibers'
 * global column ids and exact squared norms are all-gathered, every rank
 * draws the same sample, candidates are all-gathered from their owners, the
 * filter runs replicated, and the error partials are all-reduced.
 * (The reference entry points these compose: column_distribution +
 * sample_with_replacement + unique_first_occurrence, sampling.cpp:21-78;
 * FiberBasis::try_append_fiber, fiber_basis.cpp:43-109; relative_error,
 * evaluation.cpp:88-122.) */
/* Law, draws and dedup over the nonempty fibers given by host arrays
 * (fiber_col strictly ascending global column ids, sq_norms their exact
 * squared norms): bit-exact with column_distribution /
 * sample_with_replacement / unique_first_occurrence over all N_alpha columns
 * (the absent columns have probability exactly 0).  unique[sample_size]
 * receives the unique drawn column ids in first-occurrence order. */
int ctd_gpu_sample_fibers(ctd_gpu_ctx *ctx, int64_t n_fibers, const int64_t *fiber_col,
                          const double *sq_norms, int64_t sample_size, uint64_t seed,
                          double *total_sq_norm, int64_t *unique, int64_t *n_unique);
/* try_append_fiber for n candidates in order (host CSC: cand_ptr[n+1], rows
 * ascending per candidate, values without zeros); per-candidate outcomes. */
int ctd_gpu_basis_append_batch(ctd_gpu_basis *b, int64_t n, const int64_t *cand_ptr,
                               const int64_t *rows, const double *vals, double epsilon,
                               int32_t *accepted, int32_t *degenerate, double *delta);
/* R of the basis as CSC (size()+1, r_nnz, r_nnz), acceptance order. */
/* The same with the candidates' rows (int32) and values in DEVICE memory
 * (e.g. assembled by a device all-gather); cand_ptr stays on the host.  The
 * row range / ascending checks run on the device. */
int ctd_gpu_basis_append_batch_device(ctd_gpu_basis *b, int64_t n, const int64_t *cand_ptr,
                                      const int32_t *rows, const double *vals, double epsilon,
                                      int32_t *accepted, int32_t *degenerate, double *delta);
int64_t ctd_gpu_basis_r_nnz(const ctd_gpu_basis *b);
int ctd_gpu_basis_r(const ctd_gpu_basis *b, int64_t *col_ptr, int64_t *rows, double *vals);
/* A shard of X bucketed once and kept resident: its fibers' global column
 * ids and exact squared norms (for the all-gather), owner-side gathers of
 * candidate fibers, and the error partials over its fibers. */
typedef struct ctd_gpu_shard ctd_gpu_shard;
int ctd_gpu_shard_create(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *x, int mode,
                         ctd_gpu_shard **out);
int64_t ctd_gpu_shard_n_fibers(const ctd_gpu_shard *s);
int ctd_gpu_shard_fibers(const ctd_gpu_shard *s, int64_t *fiber_col, double *sq_norms);
/* cand_ptr[n+1] always; rows/vals (cand_ptr[n] entries) when non-NULL.
 * Every cols[k] must be a fiber of this shard (ArgumentError otherwise). */
int ctd_gpu_shard_gather(const ctd_gpu_shard *s, int64_t n, const int64_t *cols,
                         int64_t *cand_ptr, int64_t *rows, double *vals);
/* The same with rows (int32) / vals written to DEVICE memory (cand_ptr on
 * the host): the owner's half of a device-resident candidate all-gather. */
int ctd_gpu_shard_gather_device(const ctd_gpu_shard *s, int64_t n, const int64_t *cols,
                                int64_t *cand_ptr, int32_t *rows, double *vals);
int ctd_gpu_shard_error_partials(const ctd_gpu_shard *s, const ctd_gpu_basis *b,
                                 double *x_sq, double *cross);
int ctd_gpu_shard_destroy(ctd_gpu_shard *s);
/* The core columns of this shard's fibers, C_p = R^T X_p (compute_core,
 * ctd_static.cpp:12-17, tensor_ops.cpp:27-59): C is column-sharded exactly like
 * X (a core column j is fiber j's), so every rank computes its own columns from
 * the replicated basis with no exchange.  The shard
 * keeps C_p resident; _core_copy exports it like ctd_gpu_factors_core (column
 * ids ascending, rows = kept-column index ascending within a column). */
int ctd_gpu_shard_core(ctd_gpu_shard *s, const ctd_gpu_basis *b, int64_t *c_cols, int64_t *c_nnz);
/* compute_core (ctd_static.hpp:28, ctd_static.cpp:12-17) for a caller-given R
 * (CSC, r_cols columns over r_rows = x's extent in `mode`, rows ascending):
 * C_(mode) = R^T X_(mode), entries with |c| < 1e-14 dropped.  The result is a
 * ctd_gpu_csc: K = r_cols rows, only the columns of X_(mode) that keep an
 * entry (their ids j); fold it with the reference's fold() for the tensor. */
typedef struct ctd_gpu_csc ctd_gpu_csc;
int ctd_gpu_compute_core(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *x, int mode, int64_t r_rows, int64_t r_cols,
                         const int64_t *r_col_ptr, const int64_t *r_row, const double *r_val, ctd_gpu_csc **out);
/* chain_product (ctd_dynamic.hpp:61-62, ctd_dynamic.cpp:231-269):
 * ((dR^T R) U) C for dR (a_cols columns), R (k columns; both over `dim` rows),
 * U (k x k row-major) and C (k rows, c_cols columns): a_cols x c_cols, only the
 * columns that keep an entry (ids = C's column index), |v| < 1e-14 dropped, in
 * the reference's operation order. */
int ctd_gpu_chain_product(ctd_gpu_ctx *ctx, int64_t dim, int64_t a_cols, const int64_t *dr_col_ptr,
                          const int64_t *dr_row, const double *dr_val, int64_t k, const int64_t *r_col_ptr,
                          const int64_t *r_row, const double *r_val, const double *u, int64_t c_cols,
                          const int64_t *c_col_ptr, const int64_t *c_row, const double *c_val, ctd_gpu_csc **out);
int ctd_gpu_csc_info(const ctd_gpu_csc *m, int64_t *rows, int64_t *n_cols, int64_t *nnz);
int ctd_gpu_csc_copy(const ctd_gpu_csc *m, int64_t *col_id, int64_t *col_ptr, int64_t *rows, double *vals);
int ctd_gpu_csc_destroy(ctd_gpu_csc *m);

/* The CTD-D core over fiber-range shards (core tiles stay
 * column-sharded): a rank's columns of StreamState::core (ctd_dynamic.hpp:18-39).
 * _create: init_stream's core of the rank's history shard (ctd_dynamic.cpp:
 * 129-147); per ctd_d_step (:149-229): _begin before the filter (snapshots U^(t),
 * :165-167), _step after it (Eq. 13: the old columns gain the bottom-left rows
 * chain_product(dR, R, U, C) (:190-222, :231-269), the slab's columns are
 * R_new^T dX_p (transpose_times, :188,:219); dR is read from the replicated
 * basis).  Every column of the stream's core is computed by exactly one rank,
 * from its own data and the replicated basis: no exchange. */
typedef struct ctd_gpu_core_shard ctd_gpu_core_shard;
int ctd_gpu_core_shard_create(ctd_gpu_shard *hist, const ctd_gpu_basis *b, ctd_gpu_core_shard **out);
int ctd_gpu_core_shard_begin(ctd_gpu_core_shard *c, const ctd_gpu_basis *b);
int ctd_gpu_core_shard_step(ctd_gpu_core_shard *c, const ctd_gpu_shard *slab, const ctd_gpu_basis *b,
                            int64_t col_offset);
int ctd_gpu_core_shard_copy(const ctd_gpu_core_shard *c, int64_t *c_cols, int64_t *c_nnz, int64_t *col_id,
                            int64_t *col_ptr, int64_t *rows, double *vals);
int ctd_gpu_core_shard_destroy(ctd_gpu_core_shard *c);
int ctd_gpu_shard_core_copy(const ctd_gpu_shard *s, int64_t *col_id, int64_t *col_ptr, int64_t *rows,
                            double *vals);
/* The sampling law chained across the shards' ascending fiber ranges instead
 * of all-gathering every fiber (column_distribution / sample_with_replacement,
 * sampling.cpp:21-64, whose sums are sequential over the columns):
 *   seq_total: the sequential sum of this shard's squared norms resumed from
 *     `start` (the running value after the earlier shards) -> *total;
 *   cdf: p = n / total and this shard's segment of the cumulative array
 *     resumed from `start` (kept on the shard); *end is its last value and
 *     *has_positive whether any p > 0;
 *   clamp: the tail clamp to 1.0 from the last positive p (the shard holding
 *     the global last positive column calls it);
 *   draw: the replicated mt19937_64(seed) uniforms; cols[i] = the fiber
 *     upper_bound selects when it lies in this shard, else -1. */
int ctd_gpu_shard_seq_total(const ctd_gpu_shard *s, double start, double *total);
int ctd_gpu_shard_cdf(ctd_gpu_shard *s, double total, double start, double *end, int *has_positive);
int ctd_gpu_shard_clamp(ctd_gpu_shard *s);
int ctd_gpu_shard_draw(const ctd_gpu_shard *s, int64_t count, uint64_t seed, int64_t *cols);
/* relative_error's two sums over the fibers of x (one shard):
 * x_sq = |X_p|^2 and cross = sum_j x_j^T (R U R^T) x_j; after summing the
 * shards, rel = (x_sq - cross) / x_sq. */
int ctd_gpu_basis_error_partials(ctd_gpu_ctx *ctx, const ctd_gpu_basis *b,
                                 const ctd_gpu_tensor *x, int mode, double *x_sq,
                                 double *cross);
/* pos[k] = the shard-local fiber index of global column cols[k], or -1 when
 * this shard does not hold it (owner lookup for the candidate exchange). */
int ctd_gpu_shard_find(const ctd_gpu_shard *s, int64_t n, const int64_t *cols, int64_t *pos);
/* Owner-side candidate gather straight into a draw-order layout in DEVICE
 * memory: fiber cols[k] (held by this shard) is written to rows/vals
 * [dst_off[k], dst_off[k] + its length).  dst_off stays on the host. */
int ctd_gpu_shard_gather_into(const ctd_gpu_shard *s, int64_t n, const int64_t *cols,
                              const int64_t *dst_off, int32_t *rows, double *vals);

/* ---- multi-GPU CTD-S driven from C++  -------------------------
 * ctd_s (ctd_static.cpp:19-50) over fiber-range shards with the whole host
 * orchestration inside this library: one process (or thread) per GPU, each
 * holding its fiber range of X in the GLOBAL index space.  Every exchange is
 * an in-place all-reduce (sum) of a DEVICE buffer on the context's stream:
 *   - range check and global fiber count (a slot per rank);
 *   - the sequential law, chained rank to rank (one double per hop);
 *   - the draws (each is resolved by exactly one owner; others add 0);
 *   - candidate lengths and payload, written by the owners into the
 *     draw-order layout (others add 0: integer sums of bit patterns, exact);
 *   - relative_error's partials, summed in rank order on the host.
 * The filter then runs replicated, so every rank ends with the same kept
 * ids, R and U, bit-identical to ctd_gpu_ctd_s on the whole tensor.
 * Communicators:
 *   - NCCL (libnccl.so.2 is dlopen'ed on first use, preferring the copy the
 *     process already loaded): rank 0 makes the 128-byte id, the caller
 *     ships it to the other ranks by any means, each rank calls _nccl_create;
 *   - host callbacks (gloo, MPI, tests): allreduce_sum receives a HOST copy
 *     of the buffer (dtype 0 = int32, 1 = int64) and sums it in place over
 *     the ranks; return 0 on success. */
typedef struct ctd_gpu_comm ctd_gpu_comm;
typedef int (*ctd_gpu_allreduce_fn)(void *user, void *buf, int64_t n, int dtype);
int ctd_gpu_comm_nccl_unique_id(unsigned char id[128]);
int ctd_gpu_comm_nccl_create(ctd_gpu_ctx *ctx, int world, int rank, const unsigned char id[128],
                             ctd_gpu_comm **out);
int ctd_gpu_comm_host_create(ctd_gpu_ctx *ctx, int world, int rank, ctd_gpu_allreduce_fn allreduce_sum,
                             void *user, ctd_gpu_comm **out);
int ctd_gpu_comm_world(const ctd_gpu_comm *c, int *world, int *rank);
int ctd_gpu_comm_destroy(ctd_gpu_comm *c);

typedef struct ctd_gpu_sharded ctd_gpu_sharded;
typedef struct {
  int64_t n_fibers;      /* global nonempty fibers */
  int64_t n_unique;      /* unique drawn fibers (candidates) */
  int64_t n_kept;        /* accepted candidates = kept_fibers.size() */
  int64_t r_nnz;         /* nnz(R) */
  int64_t cand_nnz;      /* entries of the candidate layout */
  int64_t local_fibers;  /* this rank's nonempty fibers */
  int64_t core_cols;     /* CTD_GPU_WITH_CORE: this rank's core columns and entries */
  int64_t core_nnz;
  double total_sq_norm;  /* |X|^2 in the law's sequential order */
  double relative_error; /* CTD_GPU_WITH_ERROR, else NaN */
} ctd_gpu_sharded_info;
/* flags: CTD_GPU_WITH_ERROR; CTD_GPU_WITH_CORE keeps this rank's core
 * columns on the shard (ctd_gpu_sharded_shard + ctd_gpu_shard_core_copy). */
int ctd_gpu_ctd_s_sharded(ctd_gpu_ctx *ctx, ctd_gpu_comm *comm, const ctd_gpu_tensor *local, int mode,
                          int64_t sample_size, double epsilon, uint64_t seed, unsigned flags,
                          ctd_gpu_sharded **out);
int ctd_gpu_sharded_info_get(const ctd_gpu_sharded *r, ctd_gpu_sharded_info *info);
/* kept[n_kept] (acceptance order); unique[n_unique] with per-candidate
 * accepted / degenerate / delta (any may be NULL). */
int ctd_gpu_sharded_kept(const ctd_gpu_sharded *r, int64_t *kept);
int ctd_gpu_sharded_trace(const ctd_gpu_sharded *r, int64_t *unique, int32_t *accepted,
                          int32_t *degenerate, double *delta);
/* Borrowed handles owned by the result: the replicated basis (R, U via
 * ctd_gpu_basis_r / ctd_gpu_basis_u) and this rank's shard. */
ctd_gpu_basis *ctd_gpu_sharded_basis(ctd_gpu_sharded *r);
ctd_gpu_shard *ctd_gpu_sharded_shard(ctd_gpu_sharded *r);
int ctd_gpu_sharded_destroy(ctd_gpu_sharded *r);

/* ---- CTD-D (ctd_dynamic.hpp:42-58) -------------------------------------- */
int ctd_gpu_stream_init(ctd_gpu_ctx *ctx, const ctd_gpu_tensor *historical,
                        int mode, int64_t sample_size, double epsilon,
                        uint64_t seed, unsigned flags, ctd_gpu_stream **out);
/* ctd_d_step: one slab of time extent 1. */
int ctd_gpu_stream_step(ctd_gpu_stream *s, const ctd_gpu_tensor *slab,
                        int64_t sample_size);
int64_t ctd_gpu_stream_t(const ctd_gpu_stream *s);
/* kept_fibers.size() (-1 for a null stream). */
int64_t ctd_gpu_stream_n_kept(const ctd_gpu_stream *s);
/* Snapshot of the stream's factors (kept ids, R, U; core when maintained). */
int ctd_gpu_stream_factors(ctd_gpu_stream *s, ctd_gpu_factors **out);
/* core_drift (ctd_dynamic.hpp:64-66, ctd_dynamic.cpp:271-301): |C - R^T X_hist|_F
   against the retained history (CTD_GPU_KEEP_HISTORY or CTD_GPU_EXACT_CORE;
   otherwise CTD_ERR_ARGUMENT like the reference's ArgumentError). */
int ctd_gpu_stream_core_drift(ctd_gpu_stream *s, double *out);
/* CTD_GPU_LAZY_CORE: the recorded, not yet applied core updates (records,
   slab-column entries, and bytes = 12 per entry + 8 per left-factor value);
   ctd_gpu_stream_core_sync applies them (factors and core_drift do so
   themselves).  No reference counterpart: the reference applies every update
   inside ctd_d_step (ctd_dynamic.cpp:149-229). */
int ctd_gpu_stream_core_pending(const ctd_gpu_stream *s, int64_t *records, int64_t *entries,
                                int64_t *bytes);
int ctd_gpu_stream_core_sync(ctd_gpu_stream *s);
int ctd_gpu_stream_destroy(ctd_gpu_stream *s);

#ifdef __cplusplus
}
#endif
#endif /* CTD_GPU_H */
