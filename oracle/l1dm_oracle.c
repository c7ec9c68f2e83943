/*
 * l1dm_oracle.c — CPU ORACLE for the l1 distance-matrix block product Y = A·Z.
 *
 * TEST INFRASTRUCTURE ONLY.  Nothing in the product path (the CUDA library
 * under paper_2210_15114_b200/csrc and its Python binding) may include, link
 * or call this file.  Only tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs use it.  It shares no code, header,
 * table or constant with the CUDA path.
 *
 * What it computes (PAPER.md = /root/reference/PAPER.md):
 *   A_ij = f(x_i, x_j),  f(x,y) = ||x - y||_1 = sum_k |x_k - y_k|     (§2)
 *   Y = A·Z, one column of Z at a time                               (Lemma matrixmult)
 *
 * Modes (each an independent route to the same numbers):
 *   oracle_brute      — the definition written out, O(n^2 (d+m))        (P:149, P:171 first equality)
 *   oracle_alg1       — Alg. 1 "Preprocessing": per coordinate, the sorted
 *                       array T_i and the order pi^i it induces
 *   oracle_alg2       — Alg. 2 "matrix-vector Query for p=1", literally:
 *                       B_i, C_i inclusive partial sums in sorted order,
 *                       q = position, S1..S4, z(k) += x_k(i)(S3-S4)+S2-S1
 *   oracle_hist       — integer alphabets only: the definition regrouped by
 *                       coordinate value, evaluated exactly in int64
 *   oracle_rows       — the definition for a chosen set of rows (full-size spot checks)
 *   oracle_brute_lp   — l_p^p, the definition: sum_j z_j sum_k |x_ik - x_jk|^p
 *                       ("A_ij = ||x_i - x_j||_p^p", Thm. odd_p)
 *   oracle_lp_sorted  — odd p, SPEC S:150-158's construction over Alg. 1's order, written
 *                       in Alg. 2's shape: per coordinate and power t, inclusive partial
 *                       sums in sorted order of z_j x_j^(p-t); per point, below/above split
 *                       at its position; y_k += sum_t C(p,t) (-1)^(p-t) x_k^t (below - above)
 *   oracle_brute_tv   — TV(x, y) = (1/2) sum_k |x_k - y_k|, the definition (Thm. tv)
 *   oracle_brute_bilinear — A_ij = x_i^T M x_j, the definition (Thm. maha)
 *   oracle_bilinear_alg   — Algs. 7-8 step by step: S = [M x_j]_j (d x n), v = S y,
 *                           z(k) = <x_k, v>
 *   oracle_l2_embed   — Thm. l2embed: X'[i][r] = (1/(beta k)) sum_j G[r][j] x_ij,
 *                       beta = sqrt(2/pi), rounded to fp32 (the l1 engine's input type)
 *   oracle_brute_l2   — sum_j z_j ||x_i - x_j||_2, the exact l2 product (definition)
 *   oracle_lp_even    — even p, Alg. "query_p_even" step by step with the
 *                       corrections of SPEC S:140-146 (the text drops y_j and C(p,t) and
 *                       starts t at 1): S_{i,t} = C(p,t) (-1)^(p-t) sum_j y_j x_j(i)^(p-t),
 *                       z(k) = sum_i sum_{t=0}^{p} x_k(i)^t S_{i,t}
 *
 * Precision: inputs are fp32 (BASELINE.json); every sum is accumulated in
 * x86 80-bit long double ("fp64 or better", reading R6) and
 * rounded to fp64 at the end.  Products/differences of fp32 values are
 * exact in long double.
 *
 * Parallelism: independent outputs (rows, columns) are split over POSIX
 * threads.  No sum is split across threads, so the result does not depend
 * on the thread count.  That is the only liberty taken over the paper's
 * loop order; see the notes at each function.
 *
 * Status: every function is pinned by tests/test_oracle_pins.py (see the
 * pin table in DESIGN.md §3).  No function is "parity unpinned".
 */
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdlib.h>
#include <string.h>
#include <unistd.h>

#define ORACLE_OK 0
#define ORACLE_EINVAL -1
#define ORACLE_ENOMEM -2
#define ORACLE_ENOTINT -3

typedef long double acc_t;

/* ------------------------------------------------------------------ */
/* tiny thread pool helper: run fn(arg, lo, hi) on [0, count) in chunks */
/* ------------------------------------------------------------------ */
typedef void (*range_fn)(void *arg, int64_t lo, int64_t hi);
typedef struct {
  range_fn fn;
  void *arg;
  int64_t count;
  int64_t next;
  int64_t grain;
  pthread_mutex_t mu;
} pool_job;

static void *pool_worker(void *p) {
  pool_job *job = (pool_job *)p;
  for (;;) {
    pthread_mutex_lock(&job->mu);
    int64_t lo = job->next;
    job->next += job->grain;
    pthread_mutex_unlock(&job->mu);
    if (lo >= job->count) break;
    int64_t hi = lo + job->grain;
    if (hi > job->count) hi = job->count;
    job->fn(job->arg, lo, hi);
  }
  return NULL;
}

static int resolve_threads(int nthreads) {
  if (nthreads > 0) return nthreads;
  long c = sysconf(_SC_NPROCESSORS_ONLN);
  return c > 0 ? (int)c : 1;
}

static void run_parallel(range_fn fn, void *arg, int64_t count, int64_t grain, int nthreads) {
  nthreads = resolve_threads(nthreads);
  if (grain < 1) grain = 1;
  pool_job job;
  job.fn = fn;
  job.arg = arg;
  job.count = count;
  job.next = 0;
  job.grain = grain;
  pthread_mutex_init(&job.mu, NULL);
  if (nthreads == 1 || count <= grain) {
    pool_worker(&job);
  } else {
    pthread_t *th = (pthread_t *)malloc(sizeof(pthread_t) * (size_t)nthreads);
    int started = 0;
    for (int t = 0; t < nthreads; ++t)
      if (pthread_create(&th[t], NULL, pool_worker, &job) == 0) ++started;
    if (started == 0) pool_worker(&job);
    for (int t = 0; t < started; ++t) pthread_join(th[t], NULL);
    free(th);
  }
  pthread_mutex_destroy(&job.mu);
}

int oracle_num_threads(int nthreads) { return resolve_threads(nthreads); }

/* ------------------------------------------------------------------ */
/* BRUTE: the definition.  Y[i][c] = sum_j Z[j][c] * sum_k |X[i][k]-X[j][k]|
 * P:149 (f = ||x-y||_1) and P:171 ((Ay)(k) = sum_j y_j ||x_k - x_j||_1).   */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d, ldx;
  const float *Z; int64_t m, ldz;
  double *Y; int64_t ldy;
  const int64_t *rows;   /* NULL: rows 0..n-1 */
} brute_args;

static void brute_rows(void *p, int64_t lo, int64_t hi) {
  brute_args *a = (brute_args *)p;
  acc_t *acc = (acc_t *)malloc(sizeof(acc_t) * (size_t)a->m);
  for (int64_t t = lo; t < hi; ++t) {
    int64_t i = a->rows ? a->rows[t] : t;
    for (int64_t c = 0; c < a->m; ++c) acc[c] = 0.0L;
    const float *xi = a->X + i * a->ldx;
    for (int64_t j = 0; j < a->n; ++j) {
      const float *xj = a->X + j * a->ldx;
      acc_t dist = 0.0L;                                  /* ||x_i - x_j||_1 */
      for (int64_t k = 0; k < a->d; ++k) dist += fabsl((acc_t)xi[k] - (acc_t)xj[k]);
      const float *zj = a->Z + j * a->ldz;
      for (int64_t c = 0; c < a->m; ++c) acc[c] += dist * (acc_t)zj[c];
    }
    double *yt = a->Y + t * a->ldy;                       /* row t of the output block */
    for (int64_t c = 0; c < a->m; ++c) yt[c] = (double)acc[c];
  }
  free(acc);
}

/* All rows: Y is n x m (ld = m). */
int oracle_brute(const float *X, int64_t n, int64_t d, const float *Z, int64_t m,
                 double *Y, int nthreads) {
  if (!X || !Z || !Y || n < 1 || d < 1 || m < 1) return ORACLE_EINVAL;
  brute_args a = {X, n, d, d, Z, m, m, Y, m, NULL};
  run_parallel(brute_rows, &a, n, 4, nthreads);
  return ORACLE_OK;
}

/* Selected rows (full-size spot checks): Yrows is nr x m, row t = output row rows[t]. */
int oracle_rows(const float *X, int64_t n, int64_t d, const float *Z, int64_t m,
                const int64_t *rows, int64_t nr, double *Yrows, int nthreads) {
  if (!X || !Z || !Yrows || !rows || n < 1 || d < 1 || m < 1 || nr < 0) return ORACLE_EINVAL;
  for (int64_t t = 0; t < nr; ++t)
    if (rows[t] < 0 || rows[t] >= n) return ORACLE_EINVAL;
  brute_args a = {X, n, d, d, Z, m, m, Yrows, m, rows};
  run_parallel(brute_rows, &a, nr, 1, nthreads);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Alg. 1: for i in [d]: T_i <- sorted array of the i-th
 * coordinates.  We also keep the order pi^i induced by T_i, which
 * Alg. 2 needs for "the order induced by T_i".  Ties are broken
 * by point index (a stable sort), reading R3.
 * T and order are d x n, coordinate-major: T[i*n + r], order[i*n + r].     */
/* ------------------------------------------------------------------ */
typedef struct { float v; uint32_t idx; } keyed;

static int cmp_keyed(const void *pa, const void *pb) {
  const keyed *a = (const keyed *)pa, *b = (const keyed *)pb;
  if (a->v < b->v) return -1;
  if (a->v > b->v) return 1;
  return (a->idx > b->idx) - (a->idx < b->idx);   /* equal values: by index */
}

typedef struct {
  const float *X; int64_t n, d;
  float *T; uint32_t *order;
} alg1_args;

static void alg1_coords(void *p, int64_t lo, int64_t hi) {
  alg1_args *a = (alg1_args *)p;
  keyed *buf = (keyed *)malloc(sizeof(keyed) * (size_t)a->n);
  for (int64_t i = lo; i < hi; ++i) {
    for (int64_t j = 0; j < a->n; ++j) {
      buf[j].v = a->X[j * a->d + i];
      buf[j].idx = (uint32_t)j;
    }
    qsort(buf, (size_t)a->n, sizeof(keyed), cmp_keyed);
    for (int64_t r = 0; r < a->n; ++r) {
      if (a->T) a->T[i * a->n + r] = buf[r].v;
      a->order[i * a->n + r] = buf[r].idx;
    }
  }
  free(buf);
}

int oracle_alg1(const float *X, int64_t n, int64_t d, float *T, uint32_t *order, int nthreads) {
  if (!X || !order || n < 1 || d < 1 || n > 0xFFFFFFFFLL) return ORACLE_EINVAL;
  for (int64_t t = 0; t < n * d; ++t)
    if (!isfinite(X[t])) return ORACLE_EINVAL;
  alg1_args a = {X, n, d, T, order};
  run_parallel(alg1_coords, &a, d, 1, nthreads);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Alg. 2, one query column y = Z[:, c] per task:
 *   for i in [d]:
 *     B_i = partial sums of y_j x_j(i) in the order induced by T_i
 *     C_i = partial sums of y_j        in the order induced by T_i
 *   for k in [n]: for i in [d]:
 *     q  = position of x_k(i) in the order of T_i
 *     S1 = B_i[q]; S2 = B_i[n]-B_i[q]; S3 = C_i[q]; S4 = C_i[n]-C_i[q]
 *     z(k) += x_k(i) (S3 - S4) + S2 - S1
 * Partial sums are inclusive and 1-based: B[q] = sum over sorted positions
 * 1..q, B[0] = 0 (reading R2).  Positions q are 1-based.
 *
 * Loop order: the paper builds every B_i, C_i first and then runs k-outer,
 * i-inner.  We run i-outer and k-inner so that only one coordinate's B_i,
 * C_i is held at a time.  Each z(k) still receives its terms in the order
 * i = 1..d, each term computed from identical operands, so the arithmetic
 * is the same as the paper's loop order.                                   */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d;
  const uint32_t *order;        /* Alg. 1 output, d x n */
  const float *Z; int64_t m;
  double *Y;                    /* n x m */
} alg2_args;

static void alg2_columns(void *p, int64_t lo, int64_t hi) {
  alg2_args *a = (alg2_args *)p;
  const int64_t n = a->n;
  acc_t *B = (acc_t *)malloc(sizeof(acc_t) * (size_t)(n + 1));
  acc_t *C = (acc_t *)malloc(sizeof(acc_t) * (size_t)(n + 1));
  uint32_t *pos = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  acc_t *z = (acc_t *)malloc(sizeof(acc_t) * (size_t)n);
  for (int64_t c = lo; c < hi; ++c) {
    for (int64_t k = 0; k < n; ++k) z[k] = 0.0L;                 /* z <- 0^n */
    for (int64_t i = 0; i < a->d; ++i) {
      const uint32_t *pi = a->order + i * n;
      B[0] = 0.0L;
      C[0] = 0.0L;
      for (int64_t q = 1; q <= n; ++q) {
        int64_t j = pi[q - 1];                                   /* point at sorted position q */
        acc_t yj = (acc_t)a->Z[j * a->m + c];
        acc_t xji = (acc_t)a->X[j * a->d + i];
        B[q] = B[q - 1] + yj * xji;                              /* partial sums of y_j x_j(i) */
        C[q] = C[q - 1] + yj;                                    /* partial sums of y_j */
        pos[j] = (uint32_t)q;                                    /* position of x_j(i) in T_i */
      }
      for (int64_t k = 0; k < n; ++k) {
        int64_t q = pos[k];
        acc_t S1 = B[q];
        acc_t S2 = B[n] - B[q];
        acc_t S3 = C[q];
        acc_t S4 = C[n] - C[q];
        acc_t xki = (acc_t)a->X[k * a->d + i];
        z[k] += xki * (S3 - S4) + S2 - S1;
      }
    }
    for (int64_t k = 0; k < n; ++k) a->Y[k * a->m + c] = (double)z[k];
  }
  free(B);
  free(C);
  free(pos);
  free(z);
}

int oracle_alg2(const float *X, int64_t n, int64_t d, const uint32_t *order,
                const float *Z, int64_t m, double *Y, int nthreads) {
  if (!X || !order || !Z || !Y || n < 1 || d < 1 || m < 1) return ORACLE_EINVAL;
  alg2_args a = {X, n, d, order, Z, m, Y};
  run_parallel(alg2_columns, &a, m, 1, nthreads);
  return ORACLE_OK;
}

/* Alg. 2 restricted to a coordinate range [k0, k1): the partial product over
 * those coordinates, sum_{i in [k0,k1)} of Alg. 2's per-coordinate term.
 * Used for the coordinate-sharding pins (swap of sums).  `order` is
 * the full d x n Alg. 1 output.                                            */
int oracle_alg2_range(const float *X, int64_t n, int64_t d, const uint32_t *order,
                      int64_t k0, int64_t k1, const float *Z, int64_t m, double *Y,
                      int nthreads) {
  if (!X || !order || !Z || !Y || n < 1 || d < 1 || m < 1 || k0 < 0 || k1 > d || k0 >= k1)
    return ORACLE_EINVAL;
  /* A sub-problem on the column slice: copy X[:, k0:k1] and order[k0:k1]. */
  int64_t dd = k1 - k0;
  float *Xs = (float *)malloc(sizeof(float) * (size_t)(n * dd));
  if (!Xs) return ORACLE_ENOMEM;
  for (int64_t j = 0; j < n; ++j)
    for (int64_t i = 0; i < dd; ++i) Xs[j * dd + i] = X[j * d + k0 + i];
  int rc = oracle_alg2(Xs, n, dd, order + k0 * n, Z, m, Y, nthreads);
  free(Xs);
  return rc;
}

/* ------------------------------------------------------------------ */
/* HIST: integer alphabets {0..M} (BASELINE.json config 5: 0..255), with
 * integer-valued Z.  The definition regrouped by coordinate value:
 *   Y[i][c] = sum_k sum_v |x_ik - v| * H_k[v][c],  H_k[v][c] = sum_{j: x_jk = v} Z[j][c]
 * Every quantity is an integer, so int64 arithmetic is exact (the caller
 * guarantees |Y| < 2^63; config 5 stays below 2^40).  No sort is used.
 * Returns ORACLE_ENOTINT if X or Z is not integer-valued / out of range.   */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d;
  const float *Z; int64_t m;
  int64_t M;
  int64_t *Y;   /* n x m */
} hist_args;

static void hist_columns(void *p, int64_t lo, int64_t hi) {
  hist_args *a = (hist_args *)p;
  const int64_t V = a->M + 1;
  int64_t *H = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
  int64_t *F = (int64_t *)malloc(sizeof(int64_t) * (size_t)V);
  for (int64_t c = lo; c < hi; ++c) {
    for (int64_t i = 0; i < a->n; ++i) a->Y[i * a->m + c] = 0;
    for (int64_t k = 0; k < a->d; ++k) {
      for (int64_t v = 0; v < V; ++v) H[v] = 0;
      for (int64_t j = 0; j < a->n; ++j)
        H[(int64_t)a->X[j * a->d + k]] += (int64_t)a->Z[j * a->m + c];
      for (int64_t u = 0; u < V; ++u) {                /* F[u] = sum_v |u - v| H[v] */
        int64_t s = 0;
        for (int64_t v = 0; v < V; ++v) s += (u > v ? u - v : v - u) * H[v];
        F[u] = s;
      }
      for (int64_t i = 0; i < a->n; ++i) a->Y[i * a->m + c] += F[(int64_t)a->X[i * a->d + k]];
    }
  }
  free(H);
  free(F);
}

int oracle_hist(const float *X, int64_t n, int64_t d, const float *Z, int64_t m, int64_t M,
                int64_t *Y, int nthreads) {
  if (!X || !Z || !Y || n < 1 || d < 1 || m < 1 || M < 0 || M > 65535) return ORACLE_EINVAL;
  for (int64_t t = 0; t < n * d; ++t) {
    float x = X[t];
    if (!(x >= 0.0f && x <= (float)M) || x != floorf(x)) return ORACLE_ENOTINT;
  }
  for (int64_t t = 0; t < n * m; ++t) {
    float z = Z[t];
    if (!isfinite(z) || z != floorf(z) || fabsf(z) > 16777216.0f) return ORACLE_ENOTINT;
  }
  hist_args a = {X, n, d, Z, m, M, Y};
  run_parallel(hist_columns, &a, m, 1, nthreads);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* l_p^p (A_ij = ||x_i - x_j||_p^p; Thm. odd_p P:485-487 for odd p; any p >= 1 here).
 * The definition: Y[i][c] = sum_j Z[j][c] * sum_k |X[i][k] - X[j][k]|^p, long double.      */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d;
  const float *Z; int64_t m;
  int p;
  double scale;          /* 1 for l_p^p; 1/2 for TV (p = 1) */
  double *Y;
  const int64_t *rows;   /* NULL: rows 0..n-1; else output row t is point rows[t] */
} lp_args;

static acc_t powi_l(acc_t a, int p) {
  acc_t r = 1.0L;
  for (int q = 0; q < p; ++q) r *= a;
  return r;
}

static void brute_lp_rows(void *pa, int64_t lo, int64_t hi) {
  lp_args *a = (lp_args *)pa;
  acc_t *acc = (acc_t *)malloc(sizeof(acc_t) * (size_t)a->m);
  for (int64_t t = lo; t < hi; ++t) {
    const int64_t i = a->rows ? a->rows[t] : t;
    for (int64_t c = 0; c < a->m; ++c) acc[c] = 0.0L;
    const float *xi = a->X + i * a->d;
    for (int64_t j = 0; j < a->n; ++j) {
      const float *xj = a->X + j * a->d;
      acc_t dist = 0.0L;                                  /* ||x_i - x_j||_p^p */
      for (int64_t k = 0; k < a->d; ++k) dist += powi_l(fabsl((acc_t)xi[k] - (acc_t)xj[k]), a->p);
      dist *= (acc_t)a->scale;
      const float *zj = a->Z + j * a->m;
      for (int64_t c = 0; c < a->m; ++c) acc[c] += dist * (acc_t)zj[c];
    }
    for (int64_t c = 0; c < a->m; ++c) a->Y[t * a->m + c] = (double)acc[c];
  }
  free(acc);
}

int oracle_brute_lp(const float *X, int64_t n, int64_t d, const float *Z, int64_t m, int p,
                    double *Y, int nthreads) {
  if (!X || !Z || !Y || n < 1 || d < 1 || m < 1 || p < 1) return ORACLE_EINVAL;
  lp_args a = {X, n, d, Z, m, p, 1.0, Y, NULL};
  run_parallel(brute_lp_rows, &a, n, 4, nthreads);
  return ORACLE_OK;
}

/* Selected rows of the l_p^p definition (full-size spot checks): Yrows is nr x m. */
int oracle_rows_lp(const float *X, int64_t n, int64_t d, const float *Z, int64_t m, int p,
                   const int64_t *rows, int64_t nr, double *Yrows, int nthreads) {
  if (!X || !Z || !Yrows || !rows || n < 1 || d < 1 || m < 1 || p < 1 || nr < 0)
    return ORACLE_EINVAL;
  for (int64_t t = 0; t < nr; ++t)
    if (rows[t] < 0 || rows[t] >= n) return ORACLE_EINVAL;
  lp_args a = {X, n, d, Z, m, p, 1.0, Yrows, rows};
  run_parallel(brute_lp_rows, &a, nr, 1, nthreads);
  return ORACLE_OK;
}

/* TV (Thm. tv): TV(x, y) = (1/2) ||x - y||_1 for distributions x, y. */
int oracle_brute_tv(const float *X, int64_t n, int64_t d, const float *Z, int64_t m, double *Y,
                    int nthreads) {
  if (!X || !Z || !Y || n < 1 || d < 1 || m < 1) return ORACLE_EINVAL;
  lp_args a = {X, n, d, Z, m, 1, 0.5, Y, NULL};
  run_parallel(brute_lp_rows, &a, n, 4, nthreads);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Odd p with the sort (the paper omits the proof).  For odd p,
 * |a - b|^p = sign(a - b) (a - b)^p and (x_k - x_j)^p = sum_t C(p,t) x_k^t (-x_j)^(p-t), so
 * with the points split at x_k's position in T_i (below: x_j <= x_k, above: x_j > x_k):
 *   sum_j z_j |x_k(i) - x_j(i)|^p
 *     = sum_t C(p,t) (-1)^(p-t) x_k(i)^t [ sum_below z_j x_j(i)^(p-t) - sum_above z_j x_j(i)^(p-t) ].
 * In Alg. 2's shape: for each t, B_t[q] = inclusive partial sums over sorted
 * positions 1..q of z_j x_j(i)^(p-t); q = position of x_k(i); below = B_t[q] (self included:
 * it contributes (x_k - x_k)^p = 0), above = B_t[n] - B_t[q].  `order` is Alg. 1's output.  */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d;
  const uint32_t *order;
  const float *Z; int64_t m;
  int p;
  double *Y;
} lps_args;

static void lp_sorted_columns(void *pa, int64_t lo, int64_t hi) {
  lps_args *a = (lps_args *)pa;
  const int64_t n = a->n;
  const int p = a->p;
  acc_t *B = (acc_t *)malloc(sizeof(acc_t) * (size_t)(n + 1) * (size_t)(p + 1));
  uint32_t *pos = (uint32_t *)malloc(sizeof(uint32_t) * (size_t)n);
  acc_t *z = (acc_t *)malloc(sizeof(acc_t) * (size_t)n);
  acc_t binom[16];
  binom[0] = 1.0L;                                   /* C(p, t), t = 0..p */
  for (int t = 1; t <= p; ++t) binom[t] = binom[t - 1] * (acc_t)(p - t + 1) / (acc_t)t;
  for (int64_t c = lo; c < hi; ++c) {
    for (int64_t k = 0; k < n; ++k) z[k] = 0.0L;
    for (int64_t i = 0; i < a->d; ++i) {
      const uint32_t *pi = a->order + i * n;
      for (int t = 0; t <= p; ++t) B[(size_t)t * (n + 1)] = 0.0L;
      for (int64_t q = 1; q <= n; ++q) {
        int64_t j = pi[q - 1];                       /* point at sorted position q */
        acc_t yj = (acc_t)a->Z[j * a->m + c];
        acc_t xji = (acc_t)a->X[j * a->d + i];
        for (int t = 0; t <= p; ++t) {
          acc_t *Bt = B + (size_t)t * (n + 1);
          Bt[q] = Bt[q - 1] + yj * powi_l(xji, p - t);
        }
        pos[j] = (uint32_t)q;
      }
      for (int64_t k = 0; k < n; ++k) {
        int64_t q = pos[k];
        acc_t xki = (acc_t)a->X[k * a->d + i];
        acc_t sum = 0.0L;
        for (int t = 0; t <= p; ++t) {
          const acc_t *Bt = B + (size_t)t * (n + 1);
          acc_t below = Bt[q], above = Bt[n] - Bt[q];
          acc_t sgn = ((p - t) & 1) ? -1.0L : 1.0L;  /* (-1)^(p-t) */
          sum += binom[t] * sgn * powi_l(xki, t) * (below - above);
        }
        z[k] += sum;
      }
    }
    for (int64_t k = 0; k < n; ++k) a->Y[k * a->m + c] = (double)z[k];
  }
  free(B);
  free(pos);
  free(z);
}

int oracle_lp_sorted(const float *X, int64_t n, int64_t d, const uint32_t *order,
                     const float *Z, int64_t m, int p, double *Y, int nthreads) {
  if (!X || !order || !Z || !Y || n < 1 || d < 1 || m < 1 || p < 1 || p > 15 || !(p & 1))
    return ORACLE_EINVAL;
  lps_args a = {X, n, d, order, Z, m, p, Y};
  run_parallel(lp_sorted_columns, &a, m, 1, nthreads);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Even p: Alg. "query_p_even" with SPEC S:140-146's corrections, one column of Z
 * at a time (Lemma matrixmult).  Line "Compute all the values S_{i,t}" then the loop over k.  */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d;
  const float *Z; int64_t m;
  int p;
  double *Y;
} lpe_args;

static void lp_even_columns(void *pa, int64_t lo, int64_t hi) {
  lpe_args *a = (lpe_args *)pa;
  const int p = a->p;
  acc_t *S = (acc_t *)malloc(sizeof(acc_t) * (size_t)a->d * (size_t)(p + 1));
  acc_t binom[32];
  binom[0] = 1.0L;
  for (int t = 1; t <= p; ++t) binom[t] = binom[t - 1] * (acc_t)(p - t + 1) / (acc_t)t;
  for (int64_t c = lo; c < hi; ++c) {
    for (int64_t i = 0; i < a->d; ++i)                 /* S_{i,t} for all i, t */
      for (int t = 0; t <= p; ++t) {
        acc_t sum = 0.0L;
        for (int64_t j = 0; j < a->n; ++j)
          sum += (acc_t)a->Z[j * a->m + c] * powi_l((acc_t)a->X[j * a->d + i], p - t);
        acc_t sgn = ((p - t) & 1) ? -1.0L : 1.0L;
        S[i * (p + 1) + t] = binom[t] * sgn * sum;
      }
    for (int64_t k = 0; k < a->n; ++k) {               /* z(k) = sum_i sum_t x_k(i)^t S_{i,t} */
      acc_t z = 0.0L;
      for (int64_t i = 0; i < a->d; ++i)
        for (int t = 0; t <= p; ++t) z += powi_l((acc_t)a->X[k * a->d + i], t) * S[i * (p + 1) + t];
      a->Y[k * a->m + c] = (double)z;
    }
  }
  free(S);
}

int oracle_lp_even(const float *X, int64_t n, int64_t d, const float *Z, int64_t m, int p,
                   double *Y, int nthreads) {
  if (!X || !Z || !Y || n < 1 || d < 1 || m < 1 || p < 2 || p > 30 || (p & 1))
    return ORACLE_EINVAL;
  lpe_args a = {X, n, d, Z, m, p, Y};
  run_parallel(lp_even_columns, &a, m, 1, nthreads);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Thm. maha: f(x, y) = x^T M y.  The definition, row by row: Y[i][c] =
 * sum_j Z[j][c] x_i^T M x_j (M: d x d, row-major, fp64).                                    */
/* ------------------------------------------------------------------ */
typedef struct {
  const float *X; int64_t n, d;
  const double *M;
  const float *Z; int64_t m;
  double *Y;
} bil_args;

static void bilinear_rows(void *pa, int64_t lo, int64_t hi) {
  bil_args *a = (bil_args *)pa;
  const int64_t d = a->d;
  acc_t *xm = (acc_t *)malloc(sizeof(acc_t) * (size_t)d);   /* x_i^T M */
  acc_t *acc = (acc_t *)malloc(sizeof(acc_t) * (size_t)a->m);
  for (int64_t i = lo; i < hi; ++i) {
    for (int64_t l = 0; l < d; ++l) {
      acc_t s = 0.0L;
      for (int64_t k = 0; k < d; ++k) s += (acc_t)a->X[i * d + k] * (acc_t)a->M[k * d + l];
      xm[l] = s;
    }
    for (int64_t c = 0; c < a->m; ++c) acc[c] = 0.0L;
    for (int64_t j = 0; j < a->n; ++j) {
      acc_t f = 0.0L;                                     /* x_i^T M x_j */
      for (int64_t l = 0; l < d; ++l) f += xm[l] * (acc_t)a->X[j * d + l];
      for (int64_t c = 0; c < a->m; ++c) acc[c] += f * (acc_t)a->Z[j * a->m + c];
    }
    for (int64_t c = 0; c < a->m; ++c) a->Y[i * a->m + c] = (double)acc[c];
  }
  free(xm);
  free(acc);
}

int oracle_brute_bilinear(const float *X, int64_t n, int64_t d, const double *M, const float *Z,
                          int64_t m, double *Y, int nthreads) {
  if (!X || !M || !Z || !Y || n < 1 || d < 1 || m < 1) return ORACLE_EINVAL;
  bil_args a = {X, n, d, M, Z, m, Y};
  run_parallel(bilinear_rows, &a, n, 4, nthreads);
  return ORACLE_OK;
}

/* Algs. 7-8: Preprocessing S <- d x n matrix with j-th column M x_j; Query v <- S y,
 * z(k) <- <x_k, v>.  One column of Z at a time (Lemma matrixmult).  Single-threaded: small n. */
int oracle_bilinear_alg(const float *X, int64_t n, int64_t d, const double *M, const float *Z,
                        int64_t m, double *Y) {
  if (!X || !M || !Z || !Y || n < 1 || d < 1 || m < 1) return ORACLE_EINVAL;
  acc_t *S = (acc_t *)malloc(sizeof(acc_t) * (size_t)d * (size_t)n);
  acc_t *v = (acc_t *)malloc(sizeof(acc_t) * (size_t)d);
  if (!S || !v) {
    free(S);
    free(v);
    return ORACLE_ENOMEM;
  }
  for (int64_t j = 0; j < n; ++j)                 /* S[:, j] = M x_j */
    for (int64_t k = 0; k < d; ++k) {
      acc_t s = 0.0L;
      for (int64_t l = 0; l < d; ++l) s += (acc_t)M[k * d + l] * (acc_t)X[j * d + l];
      S[k * n + j] = s;
    }
  for (int64_t c = 0; c < m; ++c) {
    for (int64_t k = 0; k < d; ++k) {             /* v = S y */
      acc_t s = 0.0L;
      for (int64_t j = 0; j < n; ++j) s += S[k * n + j] * (acc_t)Z[j * m + c];
      v[k] = s;
    }
    for (int64_t kk = 0; kk < n; ++kk) {          /* z(k) = <x_k, v> */
      acc_t s = 0.0L;
      for (int64_t k = 0; k < d; ++k) s += (acc_t)X[kk * d + k] * v[k];
      Y[kk * m + c] = (double)s;
    }
  }
  free(S);
  free(v);
  return ORACLE_OK;
}

/* ------------------------------------------------------------------ */
/* Thm. l2embed: T(x)_r = (1 / (beta k)) sum_j G_rj x_j, beta = sqrt(2/pi), long
 * double, rounded to fp32.  G is k x d (the caller's N(0,1) draws).                          */
/* ------------------------------------------------------------------ */
int oracle_l2_embed(const float *X, int64_t n, int64_t d, const float *G, int64_t k, float *Xp) {
  if (!X || !G || !Xp || n < 1 || d < 1 || k < 1) return ORACLE_EINVAL;
  const acc_t beta = sqrtl(2.0L / 3.14159265358979323846264338327950288L);
  const acc_t scale = 1.0L / (beta * (acc_t)k);
  for (int64_t i = 0; i < n; ++i)
    for (int64_t r = 0; r < k; ++r) {
      acc_t s = 0.0L;
      for (int64_t j = 0; j < d; ++j) s += (acc_t)G[r * d + j] * (acc_t)X[i * d + j];
      Xp[i * k + r] = (float)(double)(s * scale);
    }
  return ORACLE_OK;
}

/* The exact l2 distance product: Y[i][c] = sum_j Z[j][c] ||x_i - x_j||_2 (definition). */
static void brute_l2_rows(void *pa, int64_t lo, int64_t hi) {
  lp_args *a = (lp_args *)pa;
  acc_t *acc = (acc_t *)malloc(sizeof(acc_t) * (size_t)a->m);
  for (int64_t i = lo; i < hi; ++i) {
    for (int64_t c = 0; c < a->m; ++c) acc[c] = 0.0L;
    for (int64_t j = 0; j < a->n; ++j) {
      acc_t s = 0.0L;
      for (int64_t k = 0; k < a->d; ++k) {
        acc_t t = (acc_t)a->X[i * a->d + k] - (acc_t)a->X[j * a->d + k];
        s += t * t;
      }
      const acc_t dist = sqrtl(s);
      for (int64_t c = 0; c < a->m; ++c) acc[c] += dist * (acc_t)a->Z[j * a->m + c];
    }
    for (int64_t c = 0; c < a->m; ++c) a->Y[i * a->m + c] = (double)acc[c];
  }
  free(acc);
}

int oracle_brute_l2(const float *X, int64_t n, int64_t d, const float *Z, int64_t m, double *Y,
                    int nthreads) {
  if (!X || !Z || !Y || n < 1 || d < 1 || m < 1) return ORACLE_EINVAL;
  lp_args a = {X, n, d, Z, m, 2, 1.0, Y, NULL};
  run_parallel(brute_l2_rows, &a, n, 4, nthreads);
  return ORACLE_OK;
}
