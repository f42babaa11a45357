/* TEST INFRASTRUCTURE ONLY — CPU restatement of the reference CTD-S / CTD-D
 * hot path (see ctd_oracle.h for the contract and how it is pinned).  Every
 * function restates the reference operation order so that integer, index and
 * floating-point results are bit-identical; the file:line in each comment is
 * the reference code it follows (paths relative to proj/core/src/).
 * Compiled with -O2 -ffp-contract=off (oracle/Makefile): no FMA contraction. */
#include "ctd_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

#define DROP_TOL 1e-14 /* kDropTolerance, tensor_ops.hpp:13 */

static void *xmalloc(size_t n) { return malloc(n ? n : 1); }
static void *xcalloc(size_t n, size_t s) { return calloc(n ? n : 1, s ? s : 1); }

void cto_csc_free(cto_csc *m) {
  free(m->col_ptr);
  free(m->row);
  free(m->val);
  memset(m, 0, sizeof(*m));
}

/* ---------------------------------------------------------------------------
 * COO -> CSC.  SparseMatrix(rows, cols, row, col, val) sorts a permutation by
 * (col, row) and sums duplicates, dropping exact zeros (sparse_matrix.cpp:
 * 38-66).  Restated as a stable counting sort by column followed by a stable
 * insertion/merge sort by row inside each column; for coalesced input the
 * order is identical (keys are unique), for duplicates the sum runs in input
 * order. */
typedef struct { int64_t row; int64_t pos; } rowpos;

static void merge_sort_rows(rowpos *a, rowpos *tmp, int64_t n) {
  if (n < 2) return;
  if (n <= 16) {
    for (int64_t i = 1; i < n; ++i) {
      rowpos v = a[i];
      int64_t j = i;
      while (j > 0 && a[j - 1].row > v.row) { a[j] = a[j - 1]; --j; }
      a[j] = v;
    }
    return;
  }
  int64_t h = n / 2;
  merge_sort_rows(a, tmp, h);
  merge_sort_rows(a + h, tmp, n - h);
  int64_t i = 0, j = h, k = 0;
  while (i < h && j < n) tmp[k++] = (a[j].row < a[i].row) ? a[j++] : a[i++];
  while (i < h) tmp[k++] = a[i++];
  while (j < n) tmp[k++] = a[j++];
  memcpy(a, tmp, (size_t)n * sizeof(rowpos));
}

static int csc_from_coo(int64_t rows, int64_t cols, int64_t count,
                        const int64_t *row, const int64_t *col,
                        const double *val, cto_csc *out) {
  if (rows < 0 || cols < 0) return 1;
  for (int64_t i = 0; i < count; ++i)
    if (row[i] < 0 || row[i] >= rows || col[i] < 0 || col[i] >= cols) return 2;
  int64_t *cnt = xcalloc((size_t)cols + 1, sizeof(int64_t));
  for (int64_t i = 0; i < count; ++i) cnt[col[i] + 1]++;
  for (int64_t c = 0; c < cols; ++c) cnt[c + 1] += cnt[c];
  rowpos *perm = xmalloc((size_t)count * sizeof(rowpos));
  rowpos *tmp = xmalloc((size_t)count * sizeof(rowpos));
  int64_t *cur = xmalloc((size_t)(cols + 1) * sizeof(int64_t));
  memcpy(cur, cnt, (size_t)(cols + 1) * sizeof(int64_t));
  for (int64_t i = 0; i < count; ++i) {
    rowpos rp = {row[i], i};
    perm[cur[col[i]]++] = rp;
  }
  free(cur);
  out->rows = rows;
  out->cols = cols;
  out->col_ptr = xcalloc((size_t)cols + 1, sizeof(int64_t));
  out->row = xmalloc((size_t)count * sizeof(int64_t));
  out->val = xmalloc((size_t)count * sizeof(double));
  int64_t w = 0;
  for (int64_t c = 0; c < cols; ++c) {
    int64_t b = cnt[c], e = cnt[c + 1];
    merge_sort_rows(perm + b, tmp, e - b);
    int64_t i = b;
    while (i < e) {
      int64_t r = perm[i].row;
      double sum = val[perm[i].pos];
      int64_t j = i + 1;
      while (j < e && perm[j].row == r) { sum += val[perm[j].pos]; ++j; }
      if (sum != 0.0) { out->row[w] = r; out->val[w] = sum; ++w; }
      i = j;
    }
    out->col_ptr[c + 1] = w;
  }
  out->nnz = w;
  free(cnt);
  free(perm);
  free(tmp);
  return 0;
}

/* fiber_strides (tensor_ops.cpp:106-116) + matricize (:118-135). */
int cto_matricize(int order, const int64_t *shape, int64_t nnz,
                  const int64_t *idx, const double *val, int mode,
                  cto_csc *out) {
  if (mode < 0 || mode >= order) return 1; /* check_mode, tensor_ops.cpp:12-16 */
  int64_t strides[64];
  int64_t acc = 1;
  for (int k = 0; k < order; ++k) {
    if (k == mode) { strides[k] = 0; continue; }
    strides[k] = acc;
    acc *= shape[k];
  }
  int64_t cols = acc;
  int64_t *row = xmalloc((size_t)nnz * sizeof(int64_t));
  int64_t *col = xmalloc((size_t)nnz * sizeof(int64_t));
  for (int64_t i = 0; i < nnz; ++i) {
    int64_t j = 0;
    for (int k = 0; k < order; ++k) j += idx[i * order + k] * strides[k];
    row[i] = idx[i * order + mode];
    col[i] = j;
  }
  int st = csc_from_coo(shape[mode], cols, nnz, row, col, val, out);
  free(row);
  free(col);
  return st;
}

/* column_sq_norms (tensor_ops.cpp:194-202): sequential per column. */
void cto_column_sq_norms(const cto_csc *m, double *out) {
  for (int64_t j = 0; j < m->cols; ++j) {
    double s = 0.0;
    for (int64_t t = m->col_ptr[j]; t < m->col_ptr[j + 1]; ++t)
      s += m->val[t] * m->val[t];
    out[j] = s;
  }
}

/* column_distribution (sampling.cpp:21-31). */
int cto_column_distribution(const cto_csc *m, double *probs, double *total) {
  if (m->nnz == 0) return 3; /* EmptyInputError, :22-23 */
  cto_column_sq_norms(m, probs);
  double t = 0.0;
  for (int64_t j = 0; j < m->cols; ++j) t += probs[j];
  for (int64_t j = 0; j < m->cols; ++j) probs[j] /= t;
  *total = t;
  return 0;
}

/* std::mt19937_64 (the generator sampling.cpp:56 instantiates). */
#define MT_N 312
#define MT_M 156
typedef struct { uint64_t mt[MT_N]; int i; } mt64;
static void mt64_seed(mt64 *g, uint64_t seed) {
  g->mt[0] = seed;
  for (int i = 1; i < MT_N; ++i)
    g->mt[i] = 6364136223846793005ULL * (g->mt[i - 1] ^ (g->mt[i - 1] >> 62)) + (uint64_t)i;
  g->i = MT_N;
}
static uint64_t mt64_next(mt64 *g) {
  const uint64_t UM = 0xFFFFFFFF80000000ULL, LM = 0x7FFFFFFFULL, A = 0xB5026F5AA96619E9ULL;
  if (g->i >= MT_N) {
    for (int k = 0; k < MT_N; ++k) {
      uint64_t y = (g->mt[k] & UM) | (g->mt[(k + 1) % MT_N] & LM);
      g->mt[k] = g->mt[(k + MT_M) % MT_N] ^ (y >> 1) ^ ((y & 1ULL) ? A : 0ULL);
    }
    g->i = 0;
  }
  uint64_t x = g->mt[g->i++];
  x ^= (x >> 29) & 0x5555555555555555ULL;
  x ^= (x << 17) & 0x71D67FFFEDA60000ULL;
  x ^= (x << 37) & 0xFFF7EEE000000000ULL;
  x ^= x >> 43;
  return x;
}
void cto_mt19937_64(uint64_t seed, int64_t count, uint64_t *out) {
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t i = 0; i < count; ++i) out[i] = mt64_next(&g);
}

/* sample_with_replacement (sampling.cpp:33-64). */
int cto_sample_with_replacement(const double *p, int64_t n, int64_t count,
                                uint64_t seed, int64_t *out) {
  if (count < 0) return 1;
  if (count == 0) return 0;
  double *cum = xmalloc((size_t)n * sizeof(double));
  double acc = 0.0;
  int64_t last_positive = n;
  for (int64_t i = 0; i < n; ++i) { /* :45-49 */
    acc += p[i];
    cum[i] = acc;
    if (p[i] > 0.0) last_positive = i;
  }
  if (last_positive == n) { free(cum); return 3; } /* :50-51 */
  for (int64_t i = last_positive; i < n; ++i) cum[i] = 1.0; /* :54 */
  mt64 g;
  mt64_seed(&g, seed);
  for (int64_t k = 0; k < count; ++k) {
    const double u = (double)(mt64_next(&g) >> 11) * 0x1.0p-53; /* uniform01 :15-17 */
    int64_t lo = 0, hi = n; /* std::upper_bound: first cum > u */
    while (lo < hi) {
      int64_t mid = lo + (hi - lo) / 2;
      if (u < cum[mid]) hi = mid; else lo = mid + 1;
    }
    out[k] = lo;
  }
  free(cum);
  return 0;
}

/* unique_first_occurrence (sampling.cpp:66-78). */
static int cmp_i64(const void *a, const void *b) {
  int64_t x = *(const int64_t *)a, y = *(const int64_t *)b;
  return (x > y) - (x < y);
}
int64_t cto_unique_first_occurrence(const int64_t *in, int64_t n, int64_t *out) {
  int64_t *seen = xmalloc((size_t)n * sizeof(int64_t));
  int64_t ns = 0, nu = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (ns && bsearch(&in[i], seen, (size_t)ns, sizeof(int64_t), cmp_i64)) continue;
    int64_t p = ns; /* sorted insert */
    while (p > 0 && seen[p - 1] > in[i]) { seen[p] = seen[p - 1]; --p; }
    seen[p] = in[i];
    ++ns;
    out[nu++] = in[i];
  }
  free(seen);
  return nu;
}

/* ---------------------------------------------------------------------------
 * FiberBasis (fiber_basis.cpp). */
struct cto_basis {
  int64_t dim, k, cap;
  int64_t *len;
  int64_t **idx;
  double **val;
  double *u; /* k x k row-major */
};

cto_basis *cto_basis_new(int64_t dim) {
  cto_basis *b = xcalloc(1, sizeof(cto_basis));
  b->dim = dim;
  return b;
}
void cto_basis_free(cto_basis *b) {
  if (!b) return;
  for (int64_t i = 0; i < b->k; ++i) { free(b->idx[i]); free(b->val[i]); }
  free(b->idx); free(b->val); free(b->len); free(b->u);
  free(b);
}
int64_t cto_basis_size(const cto_basis *b) { return b->k; }
const double *cto_basis_u(const cto_basis *b) { return b->u; }

int cto_basis_try_append(cto_basis *b, int64_t dim, int64_t nnz,
                         const int64_t *xi, const double *xv, double eps,
                         int *accepted, int *degenerate, double *delta,
                         double *y_out) {
  if (dim != b->dim) return 2; /* :45 */
  const int64_t k = b->k;
  *accepted = 0; *degenerate = 0; *delta = 0.0;
  double x_sq = 0.0; /* SparseVec::squared_norm, sparse_matrix.cpp:10-14 */
  for (int64_t t = 0; t < nnz; ++t) x_sq += xv[t] * xv[t];
  /* gram_coeffs (:21-41): sorted merge per kept column. */
  double *g = xcalloc((size_t)k, sizeof(double));
  for (int64_t c = 0; c < k; ++c) {
    const int64_t *ci = b->idx[c];
    const double *cv = b->val[c];
    double s = 0.0;
    int64_t a = 0, q = 0;
    while (a < b->len[c] && q < nnz) {
      if (ci[a] < xi[q]) ++a;
      else if (ci[a] > xi[q]) ++q;
      else { s += cv[a] * xv[q]; ++a; ++q; }
    }
    g[c] = s;
  }
  /* y = U g, DenseMatrix::matvec (dense_matrix.cpp:38-49). */
  double *y = xcalloc((size_t)k, sizeof(double));
  for (int64_t r = 0; r < k; ++r) {
    double s = 0.0;
    const double *row = b->u + r * k;
    for (int64_t c = 0; c < k; ++c) s += row[c] * g[c];
    y[r] = s;
  }
  if (y_out) memcpy(y_out, y, (size_t)k * sizeof(double));
  /* z = R y with touched list (:54-65), residual (:66-77). */
  double *z = xcalloc((size_t)b->dim, sizeof(double));
  int64_t tcap = 16, tn = 0;
  int64_t *touched = xmalloc((size_t)tcap * sizeof(int64_t));
  for (int64_t c = 0; c < k; ++c) {
    const double yk = y[c];
    if (yk == 0.0) continue;
    for (int64_t t = 0; t < b->len[c]; ++t) {
      const int64_t r = b->idx[c][t];
      if (z[r] == 0.0) {
        if (tn == tcap) { tcap *= 2; touched = realloc(touched, (size_t)tcap * sizeof(int64_t)); }
        touched[tn++] = r;
      }
      z[r] += yk * b->val[c][t];
    }
  }
  double res_sq = 0.0;
  for (int64_t t = 0; t < nnz; ++t) {
    const double d = xv[t] - z[xi[t]];
    res_sq += d * d;
    z[xi[t]] = 0.0;
  }
  for (int64_t t = 0; t < tn; ++t) {
    const double zr = z[touched[t]];
    res_sq += zr * zr;
    z[touched[t]] = 0.0;
  }
  free(z); free(touched); free(g);
  if (sqrt(res_sq) <= eps * sqrt(x_sq)) { free(y); return 0; } /* :79 */
  const double dl = res_sq; /* :83-88 */
  if (!(dl > 0.0) || !isfinite(dl) || !isfinite(1.0 / dl)) {
    *degenerate = 1;
    free(y);
    return 0;
  }
  *accepted = 1;
  *delta = dl;
  /* Block update (:92-106). */
  double *next = xcalloc((size_t)(k + 1) * (size_t)(k + 1), sizeof(double));
  const int64_t n1 = k + 1;
  for (int64_t i = 0; i < k; ++i) {
    const double yi = y[i];
    for (int64_t j = 0; j <= i; ++j) {
      const double v = b->u[i * k + j] + yi * y[j] / dl;
      next[i * n1 + j] = v;
      next[j * n1 + i] = v;
    }
    next[i * n1 + k] = -yi / dl;
    next[k * n1 + i] = -yi / dl;
  }
  next[k * n1 + k] = 1.0 / dl;
  free(b->u);
  b->u = next;
  if (b->k == b->cap) {
    b->cap = b->cap ? 2 * b->cap : 16;
    b->len = realloc(b->len, (size_t)b->cap * sizeof(int64_t));
    b->idx = realloc(b->idx, (size_t)b->cap * sizeof(int64_t *));
    b->val = realloc(b->val, (size_t)b->cap * sizeof(double *));
  }
  b->len[k] = nnz;
  b->idx[k] = xmalloc((size_t)nnz * sizeof(int64_t));
  b->val[k] = xmalloc((size_t)nnz * sizeof(double));
  memcpy(b->idx[k], xi, (size_t)nnz * sizeof(int64_t));
  memcpy(b->val[k], xv, (size_t)nnz * sizeof(double));
  b->k = k + 1;
  free(y);
  return 0;
}

/* FiberBasis::to_matrix (fiber_basis.cpp:111-124). */
void cto_basis_r(const cto_basis *b, cto_csc *out) {
  int64_t nnz = 0;
  for (int64_t c = 0; c < b->k; ++c) nnz += b->len[c];
  out->rows = b->dim;
  out->cols = b->k;
  out->nnz = nnz;
  out->col_ptr = xcalloc((size_t)b->k + 1, sizeof(int64_t));
  out->row = xmalloc((size_t)nnz * sizeof(int64_t));
  out->val = xmalloc((size_t)nnz * sizeof(double));
  int64_t w = 0;
  for (int64_t c = 0; c < b->k; ++c) {
    memcpy(out->row + w, b->idx[c], (size_t)b->len[c] * sizeof(int64_t));
    memcpy(out->val + w, b->val[c], (size_t)b->len[c] * sizeof(double));
    w += b->len[c];
    out->col_ptr[c + 1] = w;
  }
}

/* ---------------------------------------------------------------------------
 * Sampling + filter loop shared by CTD-S (ctd_static.cpp:29-44) and the CTD-D
 * step (ctd_dynamic.cpp:173-187).  kept_flat receives j + flat_offset. */
static int sample_and_filter(const cto_csc *m, int64_t s, double eps,
                             uint64_t seed, cto_basis *basis,
                             int64_t flat_offset, cto_frontend *f) {
  double *probs = xmalloc((size_t)m->cols * sizeof(double));
  int st = cto_column_distribution(m, probs, &f->total);
  if (st) { free(probs); return st; }
  f->drawn = xmalloc((size_t)s * sizeof(int64_t));
  f->n_drawn = s;
  st = cto_sample_with_replacement(probs, m->cols, s, seed, f->drawn);
  free(probs);
  if (st) return st;
  f->unique = xmalloc((size_t)s * sizeof(int64_t));
  f->n_unique = cto_unique_first_occurrence(f->drawn, s, f->unique);
  f->accepted = xcalloc((size_t)f->n_unique, sizeof(int));
  f->degenerate = xcalloc((size_t)f->n_unique, sizeof(int));
  f->delta = xcalloc((size_t)f->n_unique, sizeof(double));
  f->kept_flat = xmalloc((size_t)f->n_unique * sizeof(int64_t));
  f->kept = 0;
  for (int64_t u = 0; u < f->n_unique; ++u) {
    const int64_t j = f->unique[u];
    const int64_t b = m->col_ptr[j], e = m->col_ptr[j + 1];
    st = cto_basis_try_append(basis, m->rows, e - b, m->row + b, m->val + b, eps,
                              &f->accepted[u], &f->degenerate[u], &f->delta[u], NULL);
    if (st) return st;
    if (f->accepted[u]) f->kept_flat[f->kept++] = j + flat_offset;
  }
  return 0;
}

void cto_frontend_free(cto_frontend *f) {
  free(f->drawn); free(f->unique); free(f->kept_flat);
  free(f->accepted); free(f->degenerate); free(f->delta);
  cto_basis_free(f->basis);
  memset(f, 0, sizeof(*f));
}

/* ctd_s validation (ctd_static.cpp:21-27) + front end (:29-47). */
int cto_ctd_s_frontend(int order, const int64_t *shape, int64_t nnz,
                       const int64_t *idx, const double *val, int mode,
                       int64_t s, double eps, uint64_t seed, cto_frontend *out) {
  memset(out, 0, sizeof(*out));
  if (nnz == 0) return 3;
  if (mode < 0 || mode >= order) return 1;
  if (s < 1) return 1;
  if (!(eps > 0.0)) return 1;
  cto_csc m;
  int st = cto_matricize(order, shape, nnz, idx, val, mode, &m);
  if (st) return st;
  out->basis = cto_basis_new(m.rows);
  st = sample_and_filter(&m, s, eps, seed, out->basis, 0, out);
  cto_csc_free(&m);
  return st;
}

/* ---------------------------------------------------------------------------
 * compute_core matricized (tensor_ops.cpp:27-59 with m = R^T): per column j of
 * X, per nonzero (r, v) ascending, per entry of R's row r ascending in k. */
static void csc_transpose(const cto_csc *a, cto_csc *out) {
  /* SparseMatrix::transposed (sparse_matrix.cpp:79-92): rows<->cols, sorted. */
  int64_t *r = xmalloc((size_t)a->nnz * sizeof(int64_t));
  int64_t *c = xmalloc((size_t)a->nnz * sizeof(int64_t));
  for (int64_t j = 0; j < a->cols; ++j)
    for (int64_t t = a->col_ptr[j]; t < a->col_ptr[j + 1]; ++t) { r[t] = j; c[t] = a->row[t]; }
  csc_from_coo(a->cols, a->rows, a->nnz, r, c, a->val, out);
  free(r);
  free(c);
}

typedef struct { int64_t n, cap; int64_t *r, *c; double *v; } triples;
static void tri_push(triples *t, int64_t r, int64_t c, double v) {
  if (t->n == t->cap) {
    t->cap = t->cap ? 2 * t->cap : 1024;
    t->r = realloc(t->r, (size_t)t->cap * sizeof(int64_t));
    t->c = realloc(t->c, (size_t)t->cap * sizeof(int64_t));
    t->v = realloc(t->v, (size_t)t->cap * sizeof(double));
  }
  t->r[t->n] = r; t->c[t->n] = c; t->v[t->n] = v; t->n++;
}
static int tri_to_csc(triples *t, int64_t rows, int64_t cols, cto_csc *out) {
  int st = csc_from_coo(rows, cols, t->n, t->r, t->c, t->v, out);
  free(t->r); free(t->c); free(t->v);
  memset(t, 0, sizeof(*t));
  return st;
}

int cto_core_matricized(const cto_csc *x, const cto_csc *r, cto_csc *out) {
  if (r->rows != x->rows) return 2; /* ctd_static.cpp:14-15 */
  cto_csc rt;
  csc_transpose(r, &rt); /* n_mode_product_impl :94 */
  double *acc = xcalloc((size_t)rt.rows + 1, sizeof(double));
  int64_t *touched = xmalloc(((size_t)rt.rows + 1) * 4 * sizeof(int64_t));
  int64_t tcap = (rt.rows + 1) * 4;
  triples tr = {0};
  for (int64_t j = 0; j < x->cols; ++j) {
    int64_t tn = 0;
    for (int64_t t = x->col_ptr[j]; t < x->col_ptr[j + 1]; ++t) {
      const int64_t row = x->row[t];
      const double xv = x->val[t];
      for (int64_t u = rt.col_ptr[row]; u < rt.col_ptr[row + 1]; ++u) {
        const int64_t k = rt.row[u];
        if (acc[k] == 0.0) {
          if (tn == tcap) { tcap *= 2; touched = realloc(touched, (size_t)tcap * sizeof(int64_t)); }
          touched[tn++] = k;
        }
        acc[k] += rt.val[u] * xv;
      }
    }
    for (int64_t q = 0; q < tn; ++q) {
      const double v = acc[touched[q]];
      if (fabs(v) >= DROP_TOL) tri_push(&tr, touched[q], j, v);
      acc[touched[q]] = 0.0;
    }
  }
  free(acc);
  free(touched);
  cto_csc_free(&rt);
  return tri_to_csc(&tr, r->cols, x->cols, out);
}

/* relative_error (evaluation.cpp:88-122) with dense_product (:32-43). */
int cto_relative_error(const cto_csc *x, double x_sq, const cto_csc *r,
                       const double *u, const cto_csc *core, double *out) {
  if (x_sq == 0.0) return 5;
  const int64_t rows = x->rows, k = r->cols;
  double *proj = xcalloc((size_t)rows * (size_t)(k ? k : 1), sizeof(double));
  for (int64_t c0 = 0; c0 < k; ++c0)
    for (int64_t t = r->col_ptr[c0]; t < r->col_ptr[c0 + 1]; ++t)
      for (int64_t c = 0; c < k; ++c)
        proj[r->row[t] * k + c] += r->val[t] * u[c0 * k + c];
  double *recon = xcalloc((size_t)rows, sizeof(double));
  double err = 0.0;
  for (int64_t j = 0; j < x->cols; ++j) {
    if (core->col_ptr[j] == core->col_ptr[j + 1]) {
      for (int64_t t = x->col_ptr[j]; t < x->col_ptr[j + 1]; ++t) err += x->val[t] * x->val[t];
      continue;
    }
    memset(recon, 0, (size_t)rows * sizeof(double));
    for (int64_t t = core->col_ptr[j]; t < core->col_ptr[j + 1]; ++t)
      for (int64_t q = 0; q < rows; ++q) recon[q] += proj[q * k + core->row[t]] * core->val[t];
    for (int64_t t = x->col_ptr[j]; t < x->col_ptr[j + 1]; ++t) recon[x->row[t]] -= x->val[t];
    for (int64_t q = 0; q < rows; ++q) err += recon[q] * recon[q];
  }
  free(proj);
  free(recon);
  *out = err / x_sq;
  return 0;
}

/* ---------------------------------------------------------------------------
 * CTD-D (ctd_dynamic.cpp). */
struct cto_stream {
  int no_core; /* front end only: kept ids and the basis, no Eq. 13 core */
  cto_basis *basis;
  cto_csc core; /* C_(alpha): basis.size() x t*slab_cols */
  int order;     /* order of the slab / stream tensor (time mode last) */
  int64_t slab_shape[64];
  int mode;
  int64_t t;
  double eps;
  uint64_t seed;
  int64_t kept, kept_cap;
  int64_t *kept_flat;
};

static void push_kept(cto_stream *st, int64_t flat) {
  if (st->kept == st->kept_cap) {
    st->kept_cap = st->kept_cap ? 2 * st->kept_cap : 64;
    st->kept_flat = realloc(st->kept_flat, (size_t)st->kept_cap * sizeof(int64_t));
  }
  st->kept_flat[st->kept++] = flat;
}

/* transpose_times (ctd_dynamic.cpp:53-85): A^T B by pairwise sorted merges. */
static int transpose_times(const cto_csc *a, const cto_csc *b, cto_csc *out) {
  if (a->rows != b->rows) return 2;
  triples tr = {0};
  for (int64_t i = 0; i < a->cols; ++i) {
    for (int64_t j = 0; j < b->cols; ++j) {
      double s = 0.0;
      int64_t p = a->col_ptr[i], q = b->col_ptr[j];
      const int64_t pe = a->col_ptr[i + 1], qe = b->col_ptr[j + 1];
      while (p < pe && q < qe) {
        if (a->row[p] < b->row[q]) ++p;
        else if (a->row[p] > b->row[q]) ++q;
        else { s += a->val[p] * b->val[q]; ++p; ++q; }
      }
      if (fabs(s) >= DROP_TOL) tri_push(&tr, i, j, s);
    }
  }
  return tri_to_csc(&tr, a->cols, b->cols, out);
}

/* chain_product (ctd_dynamic.cpp:231-269), strictly left to right. */
static int chain_product(const cto_csc *dr, const cto_csc *r, const double *u,
                         int64_t uk, const cto_csc *core, cto_csc *out) {
  cto_csc gram;
  int st = transpose_times(dr, r, &gram);
  if (st) return st;
  if (gram.cols != uk || uk != core->rows) { cto_csc_free(&gram); return 2; }
  const int64_t lr = gram.rows;
  double *left = xcalloc((size_t)lr * (size_t)(uk ? uk : 1), sizeof(double));
  for (int64_t j = 0; j < gram.cols; ++j)
    for (int64_t t = gram.col_ptr[j]; t < gram.col_ptr[j + 1]; ++t)
      for (int64_t c = 0; c < uk; ++c)
        left[gram.row[t] * uk + c] += gram.val[t] * u[j * uk + c];
  double *acc = xcalloc((size_t)lr, sizeof(double));
  triples tr = {0};
  for (int64_t j = 0; j < core->cols; ++j) {
    if (core->col_ptr[j] == core->col_ptr[j + 1]) continue;
    memset(acc, 0, (size_t)lr * sizeof(double));
    for (int64_t t = core->col_ptr[j]; t < core->col_ptr[j + 1]; ++t)
      for (int64_t i = 0; i < lr; ++i) acc[i] += left[i * uk + core->row[t]] * core->val[t];
    for (int64_t i = 0; i < lr; ++i)
      if (fabs(acc[i]) >= DROP_TOL) tri_push(&tr, i, j, acc[i]);
  }
  free(left);
  free(acc);
  cto_csc_free(&gram);
  return tri_to_csc(&tr, lr, core->cols, out);
}

/* assemble_blocks (ctd_dynamic.cpp:18-50): per-column concatenation, since
 * top-block rows precede bottom-block rows in (col,row) order. */
static void assemble(const cto_csc *tl, const cto_csc *tr, const cto_csc *bl,
                     const cto_csc *br, cto_csc *out) {
  const int64_t top = tl->rows, bot = bl ? bl->rows : 0;
  const int64_t lc = tl->cols, rc = tr->cols;
  const int64_t nnz = tl->nnz + tr->nnz + (bl ? bl->nnz + br->nnz : 0);
  out->rows = top + bot;
  out->cols = lc + rc;
  out->nnz = nnz;
  out->col_ptr = xcalloc((size_t)(lc + rc) + 1, sizeof(int64_t));
  out->row = xmalloc((size_t)nnz * sizeof(int64_t));
  out->val = xmalloc((size_t)nnz * sizeof(double));
  int64_t w = 0;
  for (int64_t j = 0; j < lc + rc; ++j) {
    const cto_csc *a = j < lc ? tl : tr;
    const cto_csc *b = bl ? (j < lc ? bl : br) : NULL;
    const int64_t jj = j < lc ? j : j - lc;
    for (int64_t t = a->col_ptr[jj]; t < a->col_ptr[jj + 1]; ++t) { out->row[w] = a->row[t]; out->val[w++] = a->val[t]; }
    if (b)
      for (int64_t t = b->col_ptr[jj]; t < b->col_ptr[jj + 1]; ++t) { out->row[w] = b->row[t] + top; out->val[w++] = b->val[t]; }
    out->col_ptr[j + 1] = w;
  }
}

/* init_stream (ctd_dynamic.cpp:129-147): ctd_s on the history, core =
 * matricize(compute_core(...)). */
int cto_stream_init(int order, const int64_t *shape, int64_t nnz,
                    const int64_t *idx, const double *val, int mode, int64_t s,
                    double eps, uint64_t seed, cto_stream **out) {
  return cto_stream_init2(order, shape, nnz, idx, val, mode, s, eps, seed, 0, out);
}

/* init_stream with an optional front-end-only state (no_core): the kept ids
 * and the basis evolve exactly as in ctd_d_step, the core is not kept (for
 * parity checks of long streams, where the reference's core does not fit). */
int cto_stream_init2(int order, const int64_t *shape, int64_t nnz,
                     const int64_t *idx, const double *val, int mode, int64_t s,
                     double eps, uint64_t seed, int no_core, cto_stream **out) {
  if (order < 2) return 1;
  if (mode < 0 || mode >= order - 1) return 1;
  cto_frontend f;
  int st = cto_ctd_s_frontend(order, shape, nnz, idx, val, mode, s, eps, seed, &f);
  if (st) { cto_frontend_free(&f); return st; }
  cto_stream *S = xcalloc(1, sizeof(cto_stream));
  S->basis = f.basis;
  f.basis = NULL;
  S->order = order;
  for (int k = 0; k < order - 1; ++k) S->slab_shape[k] = shape[k];
  S->mode = mode;
  S->t = shape[order - 1];
  S->eps = eps;
  S->seed = seed;
  for (int64_t i = 0; i < f.kept; ++i) push_kept(S, f.kept_flat[i]);
  cto_frontend_free(&f);
  S->no_core = no_core;
  if (no_core) {
    *out = S;
    return 0;
  }
  cto_csc xm, r;
  cto_matricize(order, shape, nnz, idx, val, mode, &xm);
  cto_basis_r(S->basis, &r);
  st = cto_core_matricized(&xm, &r, &S->core);
  cto_csc_free(&xm);
  cto_csc_free(&r);
  if (st) { cto_stream_free(S); return st; }
  *out = S;
  return 0;
}

/* ctd_d_step (ctd_dynamic.cpp:149-229). */
int cto_stream_step(cto_stream *S, int order, const int64_t *shape,
                    int64_t nnz, const int64_t *idx, const double *val,
                    int64_t d) {
  if (order != S->order) return 2;
  for (int k = 0; k < order - 1; ++k)
    if (shape[k] != S->slab_shape[k]) return 2;
  if (shape[order - 1] != 1) return 2;
  if (d < 1) return 1;
  cto_csc delta;
  int st = cto_matricize(order, shape, nnz, idx, val, S->mode, &delta);
  if (st) return st;
  const int64_t delta_cols = delta.cols;
  cto_csc r_old;
  memset(&r_old, 0, sizeof(r_old));
  const int64_t k_old = S->basis->k;
  double *u_old = NULL;
  if (!S->no_core) {
    cto_basis_r(S->basis, &r_old); /* :165 */
    u_old = xmalloc((size_t)(k_old * k_old) * sizeof(double) + 8);
    if (k_old) memcpy(u_old, S->basis->u, (size_t)(k_old * k_old) * sizeof(double));
  }
  int64_t kept_before = S->kept;
  if (delta.nnz > 0) { /* :173-188 */
    cto_frontend f;
    memset(&f, 0, sizeof(f));
    st = sample_and_filter(&delta, d, S->eps, S->seed ^ (uint64_t)S->t, S->basis,
                           S->t * delta_cols, &f);
    if (!st)
      for (int64_t i = 0; i < f.kept; ++i) push_kept(S, f.kept_flat[i]);
    f.basis = NULL;
    cto_frontend_free(&f);
    if (st) { cto_csc_free(&delta); cto_csc_free(&r_old); free(u_old); return st; }
  }
  if (S->no_core) {
    S->t += 1;
    cto_csc_free(&delta);
    return 0;
  }
  cto_csc top_right;
  transpose_times(&r_old, &delta, &top_right); /* :190 */
  cto_csc next;
  const int64_t n_app = S->kept - kept_before;
  if (n_app == 0) { /* :192-196 */
    assemble(&S->core, &top_right, NULL, NULL, &next);
  } else { /* :198-222 */
    cto_csc full_r, dr, bl, br;
    cto_basis_r(S->basis, &full_r);
    /* dR = the appended columns (the last n_app columns of R). */
    dr.rows = full_r.rows;
    dr.cols = n_app;
    const int64_t off = full_r.col_ptr[k_old];
    dr.nnz = full_r.nnz - off;
    dr.col_ptr = xmalloc((size_t)(n_app + 1) * sizeof(int64_t));
    for (int64_t c = 0; c <= n_app; ++c) dr.col_ptr[c] = full_r.col_ptr[k_old + c] - off;
    dr.row = xmalloc((size_t)dr.nnz * sizeof(int64_t) + 8);
    dr.val = xmalloc((size_t)dr.nnz * sizeof(double) + 8);
    memcpy(dr.row, full_r.row + off, (size_t)dr.nnz * sizeof(int64_t));
    memcpy(dr.val, full_r.val + off, (size_t)dr.nnz * sizeof(double));
    cto_csc_free(&full_r);
    chain_product(&dr, &r_old, u_old, k_old, &S->core, &bl);
    transpose_times(&dr, &delta, &br);
    assemble(&S->core, &top_right, &bl, &br, &next);
    cto_csc_free(&dr);
    cto_csc_free(&bl);
    cto_csc_free(&br);
  }
  cto_csc_free(&S->core);
  S->core = next;
  S->t += 1;
  cto_csc_free(&top_right);
  cto_csc_free(&delta);
  cto_csc_free(&r_old);
  free(u_old);
  return 0;
}

void cto_stream_free(cto_stream *S) {
  if (!S) return;
  cto_basis_free(S->basis);
  cto_csc_free(&S->core);
  free(S->kept_flat);
  free(S);
}
int64_t cto_stream_t(const cto_stream *S) { return S->t; }
int64_t cto_stream_kept(const cto_stream *S) { return S->kept; }
const int64_t *cto_stream_kept_flat(const cto_stream *S) { return S->kept_flat; }
const cto_basis *cto_stream_basis(const cto_stream *S) { return S->basis; }
const cto_csc *cto_stream_core(const cto_stream *S) { return &S->core; }
