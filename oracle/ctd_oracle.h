/* TEST INFRASTRUCTURE ONLY — the CPU restatement ("port") of the reference
 * CTD-S / CTD-D hot path used as the parity checker.  Only tests/,
 * __graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference legs
 * may load it.  The product (libctd_gpu.so) never links or calls it.
 *
 * Pinning: tests/test_oracle_pin.py checks every function here against the
 * unmodified reference compiled into oracle/_ref/libctdref.so and against the
 * known-answer vectors of the reference's own unit tests; tests/golden/ holds
 * fixtures produced by the reference itself (tests/golden/make_golden.py).
 *
 * Conventions: int64 indices like the reference (sparse_tensor.hpp:10),
 * CSC matrices as (col_ptr[cols+1], row[nnz], val[nnz]), dense matrices
 * row-major.  Status codes are the reference ErrorClass values
 * (error.hpp:11-19): 0 ok, 1 argument, 2 shape, 3 empty_input, 5 metric. */
#ifndef CTD_ORACLE_H
#define CTD_ORACLE_H
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  int64_t rows, cols, nnz;
  int64_t *col_ptr, *row;
  double *val;
} cto_csc;

void cto_csc_free(cto_csc *m);

/* matricize (tensor_ops.cpp:118-135) + SparseMatrix COO ctor
 * (sparse_matrix.cpp:22-67): column id by fiber_strides (:106-116). */
int cto_matricize(int order, const int64_t *shape, int64_t nnz,
                  const int64_t *idx, const double *val, int mode, cto_csc *out);

/* column_sq_norms (tensor_ops.cpp:194-202). */
void cto_column_sq_norms(const cto_csc *m, double *out);

/* column_distribution (sampling.cpp:21-31); probs has m->cols entries. */
int cto_column_distribution(const cto_csc *m, double *probs, double *total);

/* sample_with_replacement (sampling.cpp:33-64). */
int cto_sample_with_replacement(const double *probs, int64_t n, int64_t count,
                                uint64_t seed, int64_t *out);

/* unique_first_occurrence (sampling.cpp:66-78); returns the unique count. */
int64_t cto_unique_first_occurrence(const int64_t *in, int64_t n, int64_t *out);

/* std::mt19937_64 restated (seed, then `count` raw outputs). */
void cto_mt19937_64(uint64_t seed, int64_t count, uint64_t *out);

/* FiberBasis (fiber_basis.cpp). */
typedef struct cto_basis cto_basis;
cto_basis *cto_basis_new(int64_t dim);
void cto_basis_free(cto_basis *b);
int64_t cto_basis_size(const cto_basis *b);
const double *cto_basis_u(const cto_basis *b); /* size() x size() row-major */
int cto_basis_try_append(cto_basis *b, int64_t dim, int64_t nnz,
                         const int64_t *idx, const double *val, double eps,
                         int *accepted, int *degenerate, double *delta,
                         double *y /* size() entries or NULL */);
/* R (acceptance order) as CSC. */
void cto_basis_r(const cto_basis *b, cto_csc *out);

/* Algorithm 1 front end (ctd_static.cpp:29-47): matricize, distribution,
 * draws, dedup, filter.  Outputs are malloc'd arrays owned by the struct. */
typedef struct {
  int64_t n_drawn, n_unique, kept;
  int64_t *drawn, *unique, *kept_flat;
  int *accepted, *degenerate;
  double *delta;
  double total;
  cto_basis *basis;
} cto_frontend;
int cto_ctd_s_frontend(int order, const int64_t *shape, int64_t nnz,
                       const int64_t *idx, const double *val, int mode,
                       int64_t s, double eps, uint64_t seed, cto_frontend *out);
void cto_frontend_free(cto_frontend *f);

/* compute_core matricized: C_(mode) = R^T X_(mode) with the 1e-14 drop
 * (ctd_static.cpp:12-17 -> tensor_ops.cpp:27-59). */
int cto_core_matricized(const cto_csc *x_mat, const cto_csc *r, cto_csc *out);

/* relative_error (evaluation.cpp:88-122) from the matricized tensor, the
 * tensor's x_sq (sequential over values in tensor order), R, U and C_(mode). */
int cto_relative_error(const cto_csc *x_mat, double x_sq, const cto_csc *r,
                       const double *u, const cto_csc *core, double *out);

/* Double-double restatements of relative_error (relerr_dd.c): the error
 * numerator column by column over the fibers of x (any subset of X's
 * columns), and the whole-tensor value through the exact expansion
 * |X|^2 - <U, N> + tr((U G - I) U N), N = C C^T, G = R^T R. */
int cto_relerr_dd_direct(const cto_csc *x, const cto_csc *r, const double *u,
                         double *err_hi, double *err_lo, double *xsq_hi, double *xsq_lo);
int cto_relerr_dd_full(const cto_csc *x, const cto_csc *r, const double *u, double *out,
                       double *num_hi, double *num_lo);

/* The filter loop (ctd_static.cpp:40-44 over try_append_fiber) from an empty
 * basis, multi-threaded but bit-identical to cto_basis_try_append
 * (filter_par.c).  u_out holds n*n doubles; *k_out receives K. */
int cto_filter_par(int64_t dim, int64_t n, const int64_t *cand_ptr, const int64_t *rows, const double *vals,
                   double eps, int *accepted, int *degenerate, double *delta, int64_t *k_out, double *u_out);

/* CTD-D (ctd_dynamic.cpp).  The stream keeps R/U (basis), the matricized core
 * and the kept flat ids. */
typedef struct cto_stream cto_stream;
int cto_stream_init(int order, const int64_t *shape, int64_t nnz,
                    const int64_t *idx, const double *val, int mode, int64_t s,
                    double eps, uint64_t seed, cto_stream **out);
int cto_stream_init2(int order, const int64_t *shape, int64_t nnz,
                     const int64_t *idx, const double *val, int mode, int64_t s,
                     double eps, uint64_t seed, int no_core, cto_stream **out);
int cto_stream_step(cto_stream *st, int order, const int64_t *shape,
                    int64_t nnz, const int64_t *idx, const double *val,
                    int64_t d);
void cto_stream_free(cto_stream *st);
int64_t cto_stream_t(const cto_stream *st);
int64_t cto_stream_kept(const cto_stream *st);
const int64_t *cto_stream_kept_flat(const cto_stream *st);
const cto_basis *cto_stream_basis(const cto_stream *st);
const cto_csc *cto_stream_core(const cto_stream *st);

#ifdef __cplusplus
}
#endif
#endif
