/* TEST INFRASTRUCTURE ONLY — a multi-threaded restatement of the
 * independence-filter loop (FiberBasis::try_append_fiber, fiber_basis.cpp:
 * 43-109, driven as ctd_static.cpp:40-44), bit-identical to the sequential
 * port (cto_basis_try_append in ctd_oracle.c) and therefore to the reference.
 * It exists so the GPU's every decision, delta and U can be checked at C5
 * (c = 10000, K ~ 3000, fibers of 1e4-1e5 entries), where the sequential
 * loop would take hours.  Every floating-point result keeps the reference's
 * operation order; only independent chains run in parallel:
 *   g_k    one chain per kept column k over its rows ascending, adding
 *          R[r,k] x_r where x_r != 0: the terms and order of the sorted merge
 *          in gram_coeffs (:21-41);
 *   y_i    one chain per row of U in column order (DenseMatrix::matvec,
 *          dense_matrix.cpp:42-47);
 *   z_r    one chain per row of R over its kept columns ascending with
 *          y_k != 0 (the scatter of :54-65, seen per row);
 *   res^2  sequential: x's rows in order, then the touched rows ordered by
 *          (first column with y_k != 0, row) -- the order the reference's
 *          `touched` list has (a row re-pushed after z returns to 0 adds 0);
 *   U      the block update (:92-106) row by row.
 * Compiled -O2 -ffp-contract=off like the rest of the oracle; threads:
 * CTO_THREADS (default: all cores). */
#define _POSIX_C_SOURCE 200809L
#include <math.h>
#include <pthread.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#include "ctd_oracle.h"

typedef struct {
  int64_t dim, n, K;
  const int64_t *cptr, *crow;
  const double *cval;
  double eps;
  int *acc, *deg;
  double *delta;
  /* basis */
  int64_t **cidx;
  double **cv;
  int64_t *clen;
  double *u, *unext; /* K x K and (K+1) x (K+1), leading dimension ld */
  int64_t ld;
  /* R's row index: per row, kept columns ascending */
  int64_t *rcap, *rlen;
  int64_t **rk;
  double **rv;
  /* per-candidate scratch */
  double *xd;    /* dense x */
  int64_t *xmk;  /* candidate id marking xd entries */
  double *g, *y, *z;
  int64_t *kfirst;
  /* current candidate */
  int64_t cur;
  int accepted_now;
  double dl;
  int nth;
  pthread_barrier_t bar;
} fp_state;

typedef struct {
  fp_state *S;
  int tid;
} fp_arg;

static void range(int64_t n, int tid, int nth, int64_t *a, int64_t *b) {
  *a = n * tid / nth;
  *b = n * (tid + 1) / nth;
}

static void *fp_worker(void *p) {
  fp_arg *A = p;
  fp_state *S = A->S;
  const int tid = A->tid, nth = S->nth;
  for (int64_t n = 0; n < S->n; ++n) {
    const int64_t K = S->K;
    int64_t a, b;
    /* g_k = R_k . x (gram_coeffs order) */
    range(K, tid, nth, &a, &b);
    for (int64_t k = a; k < b; ++k) {
      double s = 0.0;
      const int64_t *ri = S->cidx[k];
      const double *rvv = S->cv[k];
      for (int64_t t = 0; t < S->clen[k]; ++t) {
        const int64_t r = ri[t];
        if (S->xmk[r] == n) s += rvv[t] * S->xd[r];
      }
      S->g[k] = s;
    }
    pthread_barrier_wait(&S->bar);
    /* y = U g (matvec) */
    for (int64_t i = a; i < b; ++i) {
      double s = 0.0;
      const double *row = S->u + i * S->ld;
      for (int64_t c = 0; c < K; ++c) s += row[c] * S->g[c];
      S->y[i] = s;
    }
    pthread_barrier_wait(&S->bar);
    /* z_r over R's row index, k ascending, y_k != 0; the first such k */
    range(S->dim, tid, nth, &a, &b);
    for (int64_t r = a; r < b; ++r) {
      double s = 0.0;
      int64_t kf = -1;
      for (int64_t t = 0; t < S->rlen[r]; ++t) {
        const int64_t k = S->rk[r][t];
        const double yk = S->y[k];
        if (yk == 0.0) continue;
        if (kf < 0) kf = k;
        s += yk * S->rv[r][t];
      }
      S->z[r] = s;
      S->kfirst[r] = kf;
    }
    pthread_barrier_wait(&S->bar);
    if (tid == 0) {
      /* residual in the reference's order, decision (:66-88) */
      const int64_t x0 = S->cptr[n], x1 = S->cptr[n + 1];
      double x_sq = 0.0;
      for (int64_t t = x0; t < x1; ++t) x_sq += S->cval[t] * S->cval[t];
      double res = 0.0;
      for (int64_t t = x0; t < x1; ++t) {
        const double d = S->cval[t] - S->z[S->crow[t]];
        res += d * d;
      }
      /* touched rows not in x, ordered by (kfirst, r): counting sort on kfirst */
      int64_t *cnt = calloc((size_t)K + 1, sizeof(int64_t));
      int64_t nt = 0;
      for (int64_t r = 0; r < S->dim; ++r)
        if (S->kfirst[r] >= 0 && S->xmk[r] != n) { cnt[S->kfirst[r] + 1]++; ++nt; }
      for (int64_t k = 0; k < K; ++k) cnt[k + 1] += cnt[k];
      int64_t *ord = malloc((size_t)(nt ? nt : 1) * sizeof(int64_t));
      for (int64_t r = 0; r < S->dim; ++r)
        if (S->kfirst[r] >= 0 && S->xmk[r] != n) ord[cnt[S->kfirst[r]]++] = r;
      for (int64_t q = 0; q < nt; ++q) {
        const double zr = S->z[ord[q]];
        res += zr * zr;
      }
      free(cnt);
      free(ord);
      S->acc[n] = 0;
      S->deg[n] = 0;
      S->delta[n] = 0.0;
      S->accepted_now = 0;
      if (!(sqrt(res) <= S->eps * sqrt(x_sq))) {
        if (!(res > 0.0) || !isfinite(res) || !isfinite(1.0 / res)) {
          S->deg[n] = 1;
        } else {
          S->acc[n] = 1;
          S->delta[n] = res;
          S->accepted_now = 1;
          S->dl = res;
        }
      }
    }
    pthread_barrier_wait(&S->bar);
    if (S->accepted_now) {
      /* block update (:92-106), rows i: lower triangle from U, mirrored */
      const double dl = S->dl;
      const int64_t ld = S->ld;
      range(K, tid, nth, &a, &b);
      for (int64_t i = a; i < b; ++i) {
        const double yi = S->y[i];
        for (int64_t j = 0; j <= i; ++j) {
          const double v = S->u[i * ld + j] + yi * S->y[j] / dl;
          S->unext[i * ld + j] = v;
          S->unext[j * ld + i] = v;
        }
        S->unext[i * ld + K] = -yi / dl;
        S->unext[K * ld + i] = -yi / dl;
      }
      if (tid == 0) S->unext[K * ld + K] = 1.0 / dl;
    }
    pthread_barrier_wait(&S->bar);
    if (tid == 0) {
      if (S->accepted_now) {
        double *t = S->u;
        S->u = S->unext;
        S->unext = t;
        const int64_t x0 = S->cptr[n], len = S->cptr[n + 1] - x0;
        S->clen[K] = len;
        S->cidx[K] = (int64_t *)(S->crow + x0);
        S->cv[K] = (double *)(S->cval + x0);
        for (int64_t t = 0; t < len; ++t) {
          const int64_t r = S->crow[x0 + t];
          if (S->rlen[r] == S->rcap[r]) {
            S->rcap[r] = S->rcap[r] ? 2 * S->rcap[r] : 8;
            S->rk[r] = realloc(S->rk[r], (size_t)S->rcap[r] * sizeof(int64_t));
            S->rv[r] = realloc(S->rv[r], (size_t)S->rcap[r] * sizeof(double));
          }
          S->rk[r][S->rlen[r]] = K;
          S->rv[r][S->rlen[r]] = S->cval[x0 + t];
          S->rlen[r]++;
        }
        S->K = K + 1;
      }
      /* mark the next candidate's rows */
      if (n + 1 < S->n)
        for (int64_t t = S->cptr[n + 1]; t < S->cptr[n + 2]; ++t) {
          S->xd[S->crow[t]] = S->cval[t];
          S->xmk[S->crow[t]] = n + 1;
        }
    }
    pthread_barrier_wait(&S->bar);
  }
  return NULL;
}

/* The filter loop over n candidates (CSC cand_ptr[n+1], rows ascending per
 * candidate) from an empty basis.  Outputs per candidate, the final K and
 * U (K x K row-major into u_out, which holds n*n doubles). */
int cto_filter_par(int64_t dim, int64_t n, const int64_t *cand_ptr, const int64_t *rows, const double *vals,
                   double eps, int *accepted, int *degenerate, double *delta, int64_t *k_out, double *u_out) {
  fp_state S;
  memset(&S, 0, sizeof(S));
  S.dim = dim;
  S.n = n;
  S.cptr = cand_ptr;
  S.crow = rows;
  S.cval = vals;
  S.eps = eps;
  S.acc = accepted;
  S.deg = degenerate;
  S.delta = delta;
  S.ld = n + 1;
  S.u = calloc((size_t)S.ld * (size_t)S.ld, sizeof(double));
  S.unext = calloc((size_t)S.ld * (size_t)S.ld, sizeof(double));
  S.cidx = calloc((size_t)n + 1, sizeof(int64_t *));
  S.cv = calloc((size_t)n + 1, sizeof(double *));
  S.clen = calloc((size_t)n + 1, sizeof(int64_t));
  S.rcap = calloc((size_t)dim, sizeof(int64_t));
  S.rlen = calloc((size_t)dim, sizeof(int64_t));
  S.rk = calloc((size_t)dim, sizeof(int64_t *));
  S.rv = calloc((size_t)dim, sizeof(double *));
  S.xd = calloc((size_t)dim, sizeof(double));
  S.xmk = malloc((size_t)dim * sizeof(int64_t));
  for (int64_t r = 0; r < dim; ++r) S.xmk[r] = -1;
  S.g = calloc((size_t)n + 1, sizeof(double));
  S.y = calloc((size_t)n + 1, sizeof(double));
  S.z = calloc((size_t)dim, sizeof(double));
  S.kfirst = calloc((size_t)dim, sizeof(int64_t));
  for (int64_t t = 0; n > 0 && t < cand_ptr[1]; ++t) {
    S.xd[rows[t]] = vals[t];
    S.xmk[rows[t]] = 0;
  }
  const char *e = getenv("CTO_THREADS");
  long nth = e ? atol(e) : sysconf(_SC_NPROCESSORS_ONLN);
  if (nth < 1) nth = 1;
  if (nth > 64) nth = 64;
  S.nth = (int)nth;
  pthread_barrier_init(&S.bar, NULL, (unsigned)nth);
  pthread_t th[64];
  fp_arg args[64];
  for (int t = 0; t < nth; ++t) {
    args[t].S = &S;
    args[t].tid = t;
    if (t) pthread_create(&th[t], NULL, fp_worker, &args[t]);
  }
  fp_worker(&args[0]);
  for (int t = 1; t < nth; ++t) pthread_join(th[t], NULL);
  pthread_barrier_destroy(&S.bar);
  *k_out = S.K;
  for (int64_t i = 0; i < S.K; ++i)
    for (int64_t j = 0; j < S.K; ++j) u_out[i * S.K + j] = S.u[i * S.ld + j];
  for (int64_t r = 0; r < dim; ++r) {
    free(S.rk[r]);
    free(S.rv[r]);
  }
  free(S.u); free(S.unext); free(S.cidx); free(S.cv); free(S.clen); free(S.rcap); free(S.rlen);
  free(S.rk); free(S.rv); free(S.xd); free(S.xmk); free(S.g); free(S.y); free(S.z); free(S.kfirst);
  return 0;
}
