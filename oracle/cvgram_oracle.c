/*
 * cvgram CPU ORACLE — TEST INFRASTRUCTURE ONLY.
 *
 * A plain-C restatement of the reference's all-fold cross-validation XᵀX/XᵀY
 * path (arXiv 2401.13185, reference tree /root/reference/proj).  Only
 * tests/, __graft_entry__.smoke() and bench.py's cpu_baseline / --impl
 * reference legs may load this library, and only as the checker or the timed
 * CPU baseline.  The product path (paper_2401_13185_b200) never calls it.
 *
 * The reference cannot be compiled here (Eigen3, Catch2 and CLI11 are absent,
 * SURVEY.md §8c), so this file restates it.  Three engines:
 *
 *   R64  orc_fast_*      faithful fp64 Algorithm 7 (fast.hpp:19-152), the same
 *                        formula shapes: mean-based training_mean, reciprocal-
 *                        scaled radicand with clamp and exact zero->1,
 *                        outer-product-then-times-N_t, divide by the product.
 *   B64  orc_baseline_*  faithful fp64 Algorithms 2/4/6 (baseline.hpp:17-97):
 *                        extract T, center, scale, then multiply.
 *   RLD  orc_truth_*     "truth": Algorithm 7 in long double (64-bit mantissa)
 *                        in a basis shifted by the fp64-rounded global column
 *                        mean, so no catastrophic cancellation.  This is what
 *                        the 1e-10 (fp64) and 1e-4 (fp32) parity gates compare
 *                        against (SURVEY.md §7 hard part 1).
 *
 * Parity pinning: the reference ships no fixture files; its known-answer tests
 * are hand-computed values inside the Catch2 sources (test_fast.cpp,
 * test_core.cpp, test_baseline.cpp, test_partition.cpp, acceptance.cpp).  They
 * are transcribed into tests/golden/reference_kats.json and checked against
 * this file by tests/test_reference_kats.py.  The seeded generator is
 * std::mt19937_64 (standard-specified; pinned by its 10000th output).
 *
 * Eigen's GEMM summation order is unspecified, so R64/B64
 * agree with the reference only to its own tolerances; RLD is the exactness
 * anchor.
 */
#define _GNU_SOURCE
#include <float.h>
#include <math.h>
#include <pthread.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_internal.h"

#define ORC_OK 0
#define ORC_E_DIMENSION 1
#define ORC_E_PARTITION 2
#define ORC_E_SCALABILITY 3
#define ORC_E_INVALID_ARG 4
#define ORC_E_OOM 6

/* PreprocessConfig bit order of enumerate_configs (combos.hpp:33-45). */
#define CX 8u
#define CY 4u
#define SX 2u
#define SY 1u
#define ANY_CENTER(c) (((c) & (CX | CY)) != 0)
#define ANY_SCALE(c) (((c) & (SX | SY)) != 0)
#define ANY(c) (((c) & 15u) != 0)

static void set_err(char* err, size_t len, const char* msg) {
  if (err && len) {
    strncpy(err, msg, len - 1);
    err[len - 1] = 0;
  }
}

/* ------------------------------------------------------------------------- */
/* std::mt19937_64 (random.hpp:14-18 relies on it being standard-specified).  */
/* ------------------------------------------------------------------------- */
typedef struct {
  uint64_t mt[312];
  int idx;
} orc_rng;

void orc_rng_seed(orc_rng* r, uint64_t seed) {
  r->mt[0] = seed;
  for (int i = 1; i < 312; ++i)
    r->mt[i] = 6364136223846793005ULL * (r->mt[i - 1] ^ (r->mt[i - 1] >> 62)) + (uint64_t)i;
  r->idx = 312;
}

uint64_t orc_rng_next(orc_rng* r) {
  if (r->idx >= 312) {
    for (int i = 0; i < 312; ++i) {
      uint64_t x = (r->mt[i] & 0xFFFFFFFF80000000ULL) | (r->mt[(i + 1) % 312] & 0x7FFFFFFFULL);
      uint64_t xa = x >> 1;
      if (x & 1ULL) xa ^= 0xB5026F5AA96619E9ULL;
      r->mt[i] = r->mt[(i + 156) % 312] ^ xa;
    }
    r->idx = 0;
  }
  uint64_t y = r->mt[r->idx++];
  y ^= (y >> 29) & 0x5555555555555555ULL;
  y ^= (y << 17) & 0x71D67FFFEDA60000ULL;
  y ^= (y << 37) & 0xFFF7EEE000000000ULL;
  y ^= y >> 43;
  return y;
}

orc_rng* orc_rng_new(uint64_t seed) {
  orc_rng* r = (orc_rng*)malloc(sizeof(orc_rng));
  if (r) orc_rng_seed(r, seed);
  return r;
}
void orc_rng_free(orc_rng* r) { free(r); }

/* uniform01, random.hpp:16-18 */
double orc_uniform01(orc_rng* r) { return (double)(orc_rng_next(r) >> 11) * 0x1.0p-53; }

/* random_dataset, random.hpp:21-27: row-major X first, then Y. */
void orc_random_dataset(orc_rng* r, int64_t n, int64_t k, int64_t m, double* x, double* y) {
  for (int64_t i = 0; i < n * k; ++i) x[i] = orc_uniform01(r);
  for (int64_t i = 0; i < n * m; ++i) y[i] = orc_uniform01(r);
}

/* random_partitioning, random.hpp:38-50: labels 1+(i mod p), Fisher-Yates. */
void orc_random_partitioning(orc_rng* r, int64_t n, int32_t p, int32_t* labels) {
  for (int64_t i = 0; i < n; ++i) labels[i] = 1 + (int32_t)(i % p);
  for (int64_t i = n - 1; i > 0; --i) {
    int64_t j = (int64_t)(orc_rng_next(r) % (uint64_t)(i + 1));
    int32_t t = labels[i];
    labels[i] = labels[j];
    labels[j] = t;
  }
}

/* ------------------------------------------------------------------------- */
/* Partition predicates, partition.hpp:21-90                                  */
/* ------------------------------------------------------------------------- */
int orc_validate_partitioning(const int32_t* labels, int64_t n, int32_t p, char* err, size_t len) {
  char buf[256];
  if (p < 2) {
    snprintf(buf, sizeof buf, "fold count must be at least 2, got %d", p);
    set_err(err, len, buf);
    return ORC_E_PARTITION;
  }
  if ((int64_t)p > n) {
    snprintf(buf, sizeof buf, "fold count %d exceeds sample count %lld", p, (long long)n);
    set_err(err, len, buf);
    return ORC_E_PARTITION;
  }
  char* seen = (char*)calloc((size_t)p, 1);
  if (!seen) return ORC_E_OOM;
  for (int64_t i = 0; i < n; ++i) {
    int32_t l = labels[i];
    if (l < 1 || l > p) {
      snprintf(buf, sizeof buf, "label %d at sample %lld is outside {1..%d}", l, (long long)(i + 1), p);
      set_err(err, len, buf);
      free(seen);
      return ORC_E_PARTITION;
    }
    seen[l - 1] = 1;
  }
  for (int32_t f = 1; f <= p; ++f)
    if (!seen[f - 1]) {
      snprintf(buf, sizeof buf, "fold %d is empty", f);
      set_err(err, len, buf);
      free(seen);
      return ORC_E_PARTITION;
    }
  free(seen);
  return ORC_OK;
}

int orc_check_scalable(const int32_t* labels, int64_t n, int32_t p, char* err, size_t len) {
  int64_t* sz = (int64_t*)calloc((size_t)p, sizeof(int64_t));
  if (!sz) return ORC_E_OOM;
  for (int64_t i = 0; i < n; ++i) sz[labels[i] - 1]++;
  for (int32_t f = 1; f <= p; ++f)
    if (n - sz[f - 1] < 2) {
      char buf[256];
      snprintf(buf, sizeof buf, "fold %d leaves a training partition of %lld rows; scaling needs at least 2", f,
               (long long)(n - sz[f - 1]));
      set_err(err, len, buf);
      free(sz);
      return ORC_E_SCALABILITY;
    }
  free(sz);
  return ORC_OK;
}

/* build_validation_partitions (partition.hpp:61-68) as CSR: rows[offsets[f]..offsets[f+1]) ascending. */
void orc_build_validation_partitions(const int32_t* labels, int64_t n, int32_t p, int64_t* rows, int64_t* offsets) {
  memset(offsets, 0, sizeof(int64_t) * (size_t)(p + 1));
  for (int64_t i = 0; i < n; ++i) offsets[labels[i]]++;
  for (int32_t f = 0; f < p; ++f) offsets[f + 1] += offsets[f];
  int64_t* fill = (int64_t*)malloc(sizeof(int64_t) * (size_t)p);
  for (int32_t f = 0; f < p; ++f) fill[f] = offsets[f];
  for (int64_t i = 0; i < n; ++i) rows[fill[labels[i] - 1]++] = i;
  free(fill);
}

/* complement_rows, partition.hpp:71-83 */
int64_t orc_complement_rows(const int64_t* v, int64_t nv, int64_t n, int64_t* t_out) {
  int64_t next = 0, nt = 0;
  for (int64_t i = 0; i < n; ++i) {
    if (next < nv && v[next] == i)
      ++next;
    else
      t_out[nt++] = i;
  }
  return nt;
}

/* ------------------------------------------------------------------------- */
/* Thread pool: detail::parallel_for, threading.hpp:12-26 (strided).          */
/* ------------------------------------------------------------------------- */

typedef struct {
  orc_task_fn fn;
  void* ctx;
  int64_t count;
  int workers;
  int w;
} orc_worker;

static void* orc_worker_main(void* arg) {
  orc_worker* wk = (orc_worker*)arg;
  for (int64_t i = wk->w; i < wk->count; i += wk->workers) wk->fn(wk->ctx, i);
  return NULL;
}

void orc_parallel_for(int64_t count, int n_threads, orc_task_fn fn, void* ctx) {
  if (n_threads <= 1 || count <= 1) {
    for (int64_t i = 0; i < count; ++i) fn(ctx, i);
    return;
  }
  int workers = (int)(count < n_threads ? count : n_threads);
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
  orc_worker* wk = (orc_worker*)malloc(sizeof(orc_worker) * (size_t)workers);
  for (int w = 0; w < workers; ++w) {
    wk[w] = (orc_worker){fn, ctx, count, workers, w};
    pthread_create(&th[w], NULL, orc_worker_main, &wk[w]);
  }
  for (int w = 0; w < workers; ++w) pthread_join(th[w], NULL);
  free(th);
  free(wk);
}

/* ------------------------------------------------------------------------- */
/* core.hpp:116-156                                                           */
/* ------------------------------------------------------------------------- */
int orc_hadamard_outer_divide(const double* mat, int64_t rows, int64_t cols, const double* l, int64_t nl,
                              const double* r, int64_t nr, double* out, char* err, size_t len) {
  if (nl != rows || nr != cols) {
    set_err(err, len, "divisor vector lengths must match matrix shape");
    return ORC_E_DIMENSION;
  }
  for (int64_t i = 0; i < nl; ++i)
    if (!(l[i] > 0.0)) {
      set_err(err, len, "hadamard_outer_divide: non-positive left divisor");
      return ORC_E_INVALID_ARG;
    }
  for (int64_t j = 0; j < nr; ++j)
    if (!(r[j] > 0.0)) {
      set_err(err, len, "hadamard_outer_divide: non-positive right divisor");
      return ORC_E_INVALID_ARG;
    }
  for (int64_t i = 0; i < rows; ++i)
    for (int64_t j = 0; j < cols; ++j) out[i * cols + j] = mat[i * cols + j] / (l[i] * r[j]);
  return ORC_OK;
}

double orc_max_rel_diff(const double* a, const double* b, int64_t len, double floor_) {
  double worst = 0.0;
  for (int64_t i = 0; i < len; ++i) {
    double d = fmax(fmax(fabs(a[i]), fabs(b[i])), floor_);
    double v = fabs(a[i] - b[i]) / d;
    if (v > worst || isnan(v)) worst = isnan(v) ? INFINITY : v;
  }
  return worst;
}

double orc_rel_frobenius_dist(const double* a, const double* b, int64_t len, double floor_) {
  long double na = 0, nb = 0, nd = 0;
  for (int64_t i = 0; i < len; ++i) {
    na += (long double)a[i] * a[i];
    nb += (long double)b[i] * b[i];
    long double d = (long double)a[i] - b[i];
    nd += d * d;
  }
  double den = fmax(fmax(sqrt((double)na), sqrt((double)nb)), floor_);
  return sqrt((double)nd) / den;
}

/* ------------------------------------------------------------------------- */
/* R64: Algorithm 7 exactly as fast.hpp writes it.                            */
/* ------------------------------------------------------------------------- */
typedef struct {
  int64_t n, k, m;
  double *xtx, *xty, *sum_x, *sum_y, *mean_x, *mean_y, *sumsq_x, *sumsq_y;
} orc_cache;

static void colsum(const double* a, int64_t rows, int64_t cols, double* out) {
  memset(out, 0, sizeof(double) * (size_t)cols);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; ++j) out[j] += a[r * cols + j];
}
static void colsumsq(const double* a, int64_t rows, int64_t cols, double* out) {
  memset(out, 0, sizeof(double) * (size_t)cols);
  for (int64_t r = 0; r < rows; ++r)
    for (int64_t j = 0; j < cols; ++j) out[j] += a[r * cols + j] * a[r * cols + j];
}

/* precompute_global, fast.hpp:19-36.  Unused vectors are left untouched (the
 * reference leaves them empty); the caller passes NULL or ignores them. */
int orc_precompute_global(const double* x, const double* y, int64_t n, int64_t k, int64_t m, uint32_t cfg,
                          double* xtx, double* xty, double* sum_x, double* sum_y, double* mean_x, double* mean_y,
                          double* sumsq_x, double* sumsq_y, int n_threads) {
  orc_gemm_tn(x, k, k, x, k, k, n, xtx, k, 1, n_threads);
  orc_gemm_tn(x, k, k, y, m, m, n, xty, m, 0, n_threads);
  if (ANY(cfg)) {
    colsum(x, n, k, sum_x);
    colsum(y, n, m, sum_y);
    for (int64_t j = 0; j < k; ++j) mean_x[j] = sum_x[j] / (double)n;
    for (int64_t j = 0; j < m; ++j) mean_y[j] = sum_y[j] / (double)n;
  }
  if (ANY_SCALE(cfg)) {
    colsumsq(x, n, k, sumsq_x);
    colsumsq(y, n, m, sumsq_y);
  }
  return ORC_OK;
}

/* training_mean, fast.hpp:40-47 */
int orc_training_mean(const double* g, const double* v, int64_t len, int64_t n, int64_t n_val, double* out, char* err,
                      size_t errlen) {
  if (n_val >= n) {
    set_err(err, errlen, "training_mean: validation rows cover the dataset");
    return ORC_E_INVALID_ARG;
  }
  const double nt = (double)(n - n_val);
  const double a = (double)n / nt, b = (double)n_val / nt;
  for (int64_t j = 0; j < len; ++j) {
    double t1 = a * g[j];
    double t2 = b * v[j];
    out[j] = t1 - t2;
  }
  return ORC_OK;
}

/* training_std, fast.hpp:53-69 */
int orc_training_std(const double* mean_t, const double* sum_t, const double* sumsq_t, int64_t len, int64_t n_train,
                     double* out, char* err, size_t errlen) {
  if (n_train < 2) {
    set_err(err, errlen, "training_std: need at least 2 training rows");
    return ORC_E_SCALABILITY;
  }
  const double scale = 1.0 / (double)(n_train - 1);
  for (int64_t j = 0; j < len; ++j) {
    double t1 = -2.0 * mean_t[j];
    t1 = t1 * sum_t[j];
    double t2 = (double)n_train * mean_t[j];
    t2 = t2 * mean_t[j];
    double s = t1 + t2;
    s = s + sumsq_t[j];
    double rad = scale * s;
    if (rad < 0.0) rad = 0.0;
    const double sd = sqrt(rad);
    out[j] = (sd == 0.0) ? 1.0 : sd;
  }
  return ORC_OK;
}

/* Per-fold outputs; any pointer may be NULL. */
typedef struct {
  double *xtx, *xty, *mean_x, *mean_y, *std_x, *std_y;
  int64_t *n_train, *n_val;
} orc_out;

/* fold_products, fast.hpp:73-130 */
static int fold_products_r64(const orc_cache* c, const double* x, const double* y, const int64_t* v_rows,
                             int64_t n_val, uint32_t cfg, double* xtx_t, double* xty_t, double* mx_t, double* my_t,
                             double* sx_t, double* sy_t, int64_t* n_train_out, int64_t* n_val_out, char* err,
                             size_t errlen) {
  const int64_t n = c->n, k = c->k, m = c->m;
  if (n_val == 0) {
    set_err(err, errlen, "fold_products: empty validation partition");
    return ORC_E_INVALID_ARG;
  }
  if (n_val >= n) {
    set_err(err, errlen, "fold_products: degenerate fold covers all rows");
    return ORC_E_INVALID_ARG;
  }
  const int64_t n_train = n - n_val;
  if (ANY_SCALE(cfg) && n_train < 2) {
    set_err(err, errlen, "fold_products: scaling needs at least 2 training rows");
    return ORC_E_SCALABILITY;
  }
  double* xv = (double*)malloc(sizeof(double) * (size_t)(n_val * k));
  double* yv = (double*)malloc(sizeof(double) * (size_t)(n_val * m));
  double* g = (double*)malloc(sizeof(double) * (size_t)(k * (k > m ? k : m)));
  double* tmp = (double*)malloc(sizeof(double) * (size_t)(4 * (k + m) + 4));
  double* mean_x = mx_t ? mx_t : (double*)malloc(sizeof(double) * (size_t)k);
  double* mean_y = my_t ? my_t : (double*)malloc(sizeof(double) * (size_t)m);
  double* std_x = sx_t ? sx_t : (double*)malloc(sizeof(double) * (size_t)k);
  double* std_y = sy_t ? sy_t : (double*)malloc(sizeof(double) * (size_t)m);
  if (!xv || !yv || !g || !tmp || !mean_x || !mean_y || !std_x || !std_y) return ORC_E_OOM;
  for (int64_t i = 0; i < n_val; ++i) {  /* gather_rows, partition.hpp:85-90 */
    memcpy(xv + i * k, x + v_rows[i] * k, sizeof(double) * (size_t)k);
    memcpy(yv + i * m, y + v_rows[i] * m, sizeof(double) * (size_t)m);
  }
  if (n_train_out) *n_train_out = n_train;
  if (n_val_out) *n_val_out = n_val;
  orc_gemm_tn(xv, k, k, xv, k, k, n_val, g, k, 1, 1);
  for (int64_t i = 0; i < k * k; ++i) xtx_t[i] = c->xtx[i] - g[i];
  orc_gemm_tn(xv, k, k, yv, m, m, n_val, g, m, 0, 1);
  for (int64_t i = 0; i < k * m; ++i) xty_t[i] = c->xty[i] - g[i];

  double* sum_xv = tmp;
  double* sum_yv = tmp + k;
  double* mv = tmp + k + m;
  int rc = ORC_OK;
  if (ANY(cfg)) {
    colsum(xv, n_val, k, sum_xv);
    colsum(yv, n_val, m, sum_yv);
    for (int64_t j = 0; j < k; ++j) mv[j] = sum_xv[j] / (double)n_val;
    rc = orc_training_mean(c->mean_x, mv, k, n, n_val, mean_x, err, errlen);
    for (int64_t j = 0; j < m; ++j) mv[j] = sum_yv[j] / (double)n_val;
    if (!rc) rc = orc_training_mean(c->mean_y, mv, m, n, n_val, mean_y, err, errlen);
  }
  const double nt = (double)n_train;
  if (!rc && (cfg & CX))
    for (int64_t i = 0; i < k; ++i)
      for (int64_t j = 0; j < k; ++j) {
        double o = mean_x[i] * mean_x[j];
        double s = nt * o;
        xtx_t[i * k + j] -= s;
      }
  if (!rc && ANY_CENTER(cfg))
    for (int64_t i = 0; i < k; ++i)
      for (int64_t j = 0; j < m; ++j) {
        double o = mean_x[i] * mean_y[j];
        double s = nt * o;
        xty_t[i * m + j] -= s;
      }
  if (!rc && (cfg & SX)) {
    double* s_t = mv;
    double* q = mv + k;
    colsumsq(xv, n_val, k, q);
    for (int64_t j = 0; j < k; ++j) {
      s_t[j] = c->sum_x[j] - sum_xv[j];
      q[j] = c->sumsq_x[j] - q[j];
    }
    rc = orc_training_std(mean_x, s_t, q, k, n_train, std_x, err, errlen);
    if (!rc) rc = orc_hadamard_outer_divide(xtx_t, k, k, std_x, k, std_x, k, xtx_t, err, errlen);
  }
  if (!rc && (cfg & SY)) {
    double* s_t = mv;
    double* q = mv + m;
    colsumsq(yv, n_val, m, q);
    for (int64_t j = 0; j < m; ++j) {
      s_t[j] = c->sum_y[j] - sum_yv[j];
      q[j] = c->sumsq_y[j] - q[j];
    }
    rc = orc_training_std(mean_y, s_t, q, m, n_train, std_y, err, errlen);
  }
  if (!rc && ANY_SCALE(cfg)) {
    double* l = (double*)malloc(sizeof(double) * (size_t)k);
    double* r = (double*)malloc(sizeof(double) * (size_t)m);
    for (int64_t i = 0; i < k; ++i) l[i] = (cfg & SX) ? std_x[i] : 1.0;
    for (int64_t j = 0; j < m; ++j) r[j] = (cfg & SY) ? std_y[j] : 1.0;
    rc = orc_hadamard_outer_divide(xty_t, k, m, l, k, r, m, xty_t, err, errlen);
    free(l);
    free(r);
  }
  free(xv);
  free(yv);
  free(g);
  free(tmp);
  if (!mx_t) free(mean_x);
  if (!my_t) free(mean_y);
  if (!sx_t) free(std_x);
  if (!sy_t) free(std_y);
  return rc;
}

/* Single-fold entry point for tests (fast.hpp:73-75) given a caller-held cache. */
int orc_fold_products(const double* x, const double* y, int64_t n, int64_t k, int64_t m, const double* c_xtx,
                      const double* c_xty, const double* c_sum_x, const double* c_sum_y, const double* c_mean_x,
                      const double* c_mean_y, const double* c_sumsq_x, const double* c_sumsq_y,
                      const int64_t* v_rows, int64_t n_val, uint32_t cfg, double* xtx_t, double* xty_t,
                      double* mean_x_t, double* mean_y_t, double* std_x_t, double* std_y_t, int64_t* n_train,
                      char* err, size_t errlen) {
  orc_cache c = {n, k, m, (double*)c_xtx, (double*)c_xty, (double*)c_sum_x, (double*)c_sum_y,
                 (double*)c_mean_x, (double*)c_mean_y, (double*)c_sumsq_x, (double*)c_sumsq_y};
  return fold_products_r64(&c, x, y, v_rows, n_val, cfg, xtx_t, xty_t, mean_x_t, mean_y_t, std_x_t, std_y_t,
                           n_train, NULL, err, errlen);
}

typedef struct {
  const orc_cache* c;
  const double *x, *y;
  const int64_t *rows, *offsets;
  uint32_t cfg;
  orc_out o;
  int* rc;
  char** errs;
} r64_fold_job;

static void r64_fold_fn(void* ctx, int64_t f) {
  r64_fold_job* j = (r64_fold_job*)ctx;
  const int64_t k = j->c->k, m = j->c->m;
  char err[256] = {0};
  j->rc[f] = fold_products_r64(j->c, j->x, j->y, j->rows + j->offsets[f], j->offsets[f + 1] - j->offsets[f], j->cfg,
                               j->o.xtx + f * k * k, j->o.xty + f * k * m, j->o.mean_x ? j->o.mean_x + f * k : NULL,
                               j->o.mean_y ? j->o.mean_y + f * m : NULL, j->o.std_x ? j->o.std_x + f * k : NULL,
                               j->o.std_y ? j->o.std_y + f * m : NULL, j->o.n_train ? j->o.n_train + f : NULL,
                               j->o.n_val ? j->o.n_val + f : NULL, err, sizeof err);
  if (j->rc[f]) j->errs[f] = strdup(err);
}

static int run_checks(int64_t n, int64_t k, int64_t m, const int32_t* labels, int64_t n_labels, int32_t p,
                      uint32_t cfg, char* err, size_t errlen) {
  if (n < 2 || k < 1 || m < 1) {
    set_err(err, errlen, n < 2 ? "need at least 2 samples" : "x and y must each have at least one column");
    return ORC_E_DIMENSION;
  }
  if (n_labels != n) { /* fast.hpp:137-138 */
    set_err(err, errlen, "partitioning length does not match sample count");
    return ORC_E_DIMENSION;
  }
  int rc = orc_validate_partitioning(labels, n, p, err, errlen);
  if (rc) return rc;
  if (ANY_SCALE(cfg)) return orc_check_scalable(labels, n, p, err, errlen);
  return ORC_OK;
}

static int collect_fold_errors(int32_t p, int* rc, char** errs, char* err, size_t errlen) {
  int out = ORC_OK;
  for (int32_t f = 0; f < p; ++f) {
    if (rc[f] && !out) {
      out = rc[f];
      set_err(err, errlen, errs[f] ? errs[f] : "fold failed");
    }
    free(errs[f]);
  }
  return out;
}

/* run_all_folds, fast.hpp:133-152.  Outputs are [p][...] contiguous. */
int orc_fast_all_folds(const double* x, const double* y, int64_t n, int64_t k, int64_t m, const int32_t* labels,
                       int64_t n_labels, int32_t p, uint32_t cfg, int n_threads, double* xtx, double* xty,
                       double* mean_x, double* mean_y, double* std_x, double* std_y, int64_t* n_train,
                       int64_t* n_val, char* err, size_t errlen) {
  int rc = run_checks(n, k, m, labels, n_labels, p, cfg, err, errlen);
  if (rc) return rc;
  orc_cache c = {n, k, m, NULL, NULL, NULL, NULL, NULL, NULL, NULL, NULL};
  c.xtx = (double*)malloc(sizeof(double) * (size_t)(k * k));
  c.xty = (double*)malloc(sizeof(double) * (size_t)(k * m));
  double* vec = (double*)malloc(sizeof(double) * (size_t)(3 * (k + m)));
  c.sum_x = vec;
  c.sum_y = vec + k;
  c.mean_x = vec + k + m;
  c.mean_y = vec + 2 * k + m;
  c.sumsq_x = vec + 2 * (k + m);
  c.sumsq_y = vec + 3 * k + 2 * m;
  orc_precompute_global(x, y, n, k, m, cfg, c.xtx, c.xty, c.sum_x, c.sum_y, c.mean_x, c.mean_y, c.sumsq_x,
                        c.sumsq_y, n_threads);
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p + 1));
  orc_build_validation_partitions(labels, n, p, rows, offsets);
  int* frc = (int*)calloc((size_t)p, sizeof(int));
  char** errs = (char**)calloc((size_t)p, sizeof(char*));
  r64_fold_job job = {&c, x, y, rows, offsets, cfg, {xtx, xty, mean_x, mean_y, std_x, std_y, n_train, n_val}, frc,
                      errs};
  orc_parallel_for(p, n_threads, r64_fold_fn, &job);
  rc = collect_fold_errors(p, frc, errs, err, errlen);
  free(frc);
  free(errs);
  free(rows);
  free(offsets);
  free(c.xtx);
  free(c.xty);
  free(vec);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* B64: baseline engine, baseline.hpp:17-97                                   */
/* ------------------------------------------------------------------------- */
int orc_baseline_single_fold(const double* x, const double* y, int64_t n, int64_t k, int64_t m,
                             const int64_t* v_rows, int64_t n_val, uint32_t cfg, double* xtx_t, double* xty_t,
                             double* mean_x_t, double* mean_y_t, double* std_x_t, double* std_y_t,
                             int64_t* n_train_out, char* err, size_t errlen) {
  int64_t* t_rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)(n > 0 ? n : 1));
  int64_t nt = orc_complement_rows(v_rows, n_val, n, t_rows);
  if (n_val == 0 || nt == 0) {
    free(t_rows);
    set_err(err, errlen, "a fold needs both validation and training rows");
    return ORC_E_PARTITION;
  }
  if (ANY_SCALE(cfg) && nt < 2) {
    free(t_rows);
    set_err(err, errlen, "scaling needs at least 2 training rows");
    return ORC_E_SCALABILITY;
  }
  double* xt = (double*)malloc(sizeof(double) * (size_t)(nt * k));
  double* yt = (double*)malloc(sizeof(double) * (size_t)(nt * m));
  for (int64_t i = 0; i < nt; ++i) {
    memcpy(xt + i * k, x + t_rows[i] * k, sizeof(double) * (size_t)k);
    memcpy(yt + i * m, y + t_rows[i] * m, sizeof(double) * (size_t)m);
  }
  if (n_train_out) *n_train_out = nt;
  double* mx = (double*)malloc(sizeof(double) * (size_t)k);
  double* my = (double*)malloc(sizeof(double) * (size_t)m);
  double* sdx = (double*)malloc(sizeof(double) * (size_t)k);
  double* sdy = (double*)malloc(sizeof(double) * (size_t)m);
  if (ANY(cfg)) { /* column_means, baseline.hpp:17-19 */
    colsum(xt, nt, k, mx);
    colsum(yt, nt, m, my);
    for (int64_t j = 0; j < k; ++j) mx[j] /= (double)nt;
    for (int64_t j = 0; j < m; ++j) my[j] /= (double)nt;
  }
  /* sample_std two-pass, baseline.hpp:23-36 */
  for (int side = 0; side < 2; ++side) {
    if (!(cfg & (side ? SY : SX))) continue;
    const double* a = side ? yt : xt;
    const double* mu = side ? my : mx;
    double* sd_out = side ? sdy : sdx;
    int64_t cols = side ? m : k;
    for (int64_t j = 0; j < cols; ++j) {
      double acc = 0.0;
      for (int64_t i = 0; i < nt; ++i) {
        const double d = a[i * cols + j] - mu[j];
        acc += d * d;
      }
      double sd = sqrt(acc / ((double)nt - 1.0));
      sd_out[j] = (sd == 0.0) ? 1.0 : sd;
    }
  }
  if (cfg & CX)
    for (int64_t i = 0; i < nt; ++i)
      for (int64_t j = 0; j < k; ++j) xt[i * k + j] -= mx[j];
  if (cfg & CY)
    for (int64_t i = 0; i < nt; ++i)
      for (int64_t j = 0; j < m; ++j) yt[i * m + j] -= my[j];
  if (cfg & SX)
    for (int64_t i = 0; i < nt; ++i)
      for (int64_t j = 0; j < k; ++j) xt[i * k + j] /= sdx[j];
  if (cfg & SY)
    for (int64_t i = 0; i < nt; ++i)
      for (int64_t j = 0; j < m; ++j) yt[i * m + j] /= sdy[j];
  orc_gemm_tn(xt, k, k, xt, k, k, nt, xtx_t, k, 1, 1);
  orc_gemm_tn(xt, k, k, yt, m, m, nt, xty_t, m, 0, 1);
  if (mean_x_t && ANY(cfg)) memcpy(mean_x_t, mx, sizeof(double) * (size_t)k);
  if (mean_y_t && ANY(cfg)) memcpy(mean_y_t, my, sizeof(double) * (size_t)m);
  if (std_x_t && (cfg & SX)) memcpy(std_x_t, sdx, sizeof(double) * (size_t)k);
  if (std_y_t && (cfg & SY)) memcpy(std_y_t, sdy, sizeof(double) * (size_t)m);
  free(t_rows);
  free(xt);
  free(yt);
  free(mx);
  free(my);
  free(sdx);
  free(sdy);
  return ORC_OK;
}

typedef struct {
  const double *x, *y;
  int64_t n, k, m;
  const int64_t *rows, *offsets;
  uint32_t cfg;
  orc_out o;
  int* rc;
  char** errs;
} base_fold_job;

static void base_fold_fn(void* ctx, int64_t f) {
  base_fold_job* j = (base_fold_job*)ctx;
  const int64_t k = j->k, m = j->m;
  char err[256] = {0};
  j->rc[f] = orc_baseline_single_fold(
      j->x, j->y, j->n, k, m, j->rows + j->offsets[f], j->offsets[f + 1] - j->offsets[f], j->cfg,
      j->o.xtx + f * k * k, j->o.xty + f * k * m, j->o.mean_x ? j->o.mean_x + f * k : NULL,
      j->o.mean_y ? j->o.mean_y + f * m : NULL, j->o.std_x ? j->o.std_x + f * k : NULL,
      j->o.std_y ? j->o.std_y + f * m : NULL, j->o.n_train ? j->o.n_train + f : NULL, err, sizeof err);
  if (j->o.n_val) j->o.n_val[f] = j->offsets[f + 1] - j->offsets[f];
  if (j->rc[f]) j->errs[f] = strdup(err);
}

int orc_baseline_all_folds(const double* x, const double* y, int64_t n, int64_t k, int64_t m, const int32_t* labels,
                           int64_t n_labels, int32_t p, uint32_t cfg, int n_threads, double* xtx, double* xty,
                           double* mean_x, double* mean_y, double* std_x, double* std_y, int64_t* n_train,
                           int64_t* n_val, char* err, size_t errlen) {
  int rc = run_checks(n, k, m, labels, n_labels, p, cfg, err, errlen);
  if (rc) return rc;
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p + 1));
  orc_build_validation_partitions(labels, n, p, rows, offsets);
  int* frc = (int*)calloc((size_t)p, sizeof(int));
  char** errs = (char**)calloc((size_t)p, sizeof(char*));
  base_fold_job job = {x, y, n, k, m, rows, offsets, cfg, {xtx, xty, mean_x, mean_y, std_x, std_y, n_train, n_val},
                       frc, errs};
  orc_parallel_for(p, n_threads, base_fold_fn, &job);
  rc = collect_fold_errors(p, frc, errs, err, errlen);
  free(frc);
  free(errs);
  free(rows);
  free(offsets);
  return rc;
}

/* ------------------------------------------------------------------------- */
/* RLD: long-double truth.  Algorithm 7 (fast.hpp) in a globally shifted      */
/* basis z = x - c, c = fp64-rounded global column mean, all accumulation in  */
/* long double.  Inputs may be fp64 or fp32 (widened: the fp32 config is      */
/* checked against fp64 truth, BASELINE.json configs[3]).                     */
/* ------------------------------------------------------------------------- */
typedef long double ld;

static inline ld load_val(const void* base, int f32, int64_t idx) {
  return f32 ? (ld)((const float*)base)[idx] : (ld)((const double*)base)[idx];
}

#define TRUTH_PANEL 64
#define TRUTH_IB 32 /* Gram rows per task */

typedef struct {
  const void *x, *y;
  int f32;
  int64_t n, k, m, w; /* w = k + m */
  const int64_t *rows, *offsets;
  const ld* shift; /* [w] */
  ld* gv;          /* [p][k][w] validation Gram in shifted basis (upper part, c >= i) */
  ld* sv;          /* [p][w] */
  ld* qv;          /* [p][w] */
  int64_t nib;     /* Gram row blocks per fold */
  int64_t ntasks;
  int64_t next;    /* dynamic task counter */
} truth_job;

/* One task = (fold f, Gram rows [i_lo, i_hi)): rows of g are disjoint across tasks, so the
 * (fold, row block) tasks run in any order with a fixed per-entry summation order (row panels
 * in ascending order, 4 interleaved partial sums per panel). */
static void truth_task(truth_job* j, int64_t t) {
  const int64_t k = j->k, m = j->m, w = j->w;
  const int64_t f = t / j->nib, ib = t % j->nib;
  const int64_t i_lo = ib * TRUTH_IB, i_hi = i_lo + TRUTH_IB < k ? i_lo + TRUTH_IB : k;
  const int64_t beg = j->offsets[f], end = j->offsets[f + 1];
  const int64_t c0 = ib == 0 ? 0 : i_lo; /* columns this task reads (row block 0 also owns the sums) */
  const int64_t wc = w - c0;
  ld* g = j->gv + f * k * w;
  ld* s = j->sv + f * w;
  ld* q = j->qv + f * w;
  for (int64_t i = i_lo; i < i_hi; ++i)
    for (int64_t c = i; c < w; ++c) g[i * w + c] = 0;
  if (ib == 0) {
    memset(s, 0, sizeof(ld) * (size_t)w);
    memset(q, 0, sizeof(ld) * (size_t)w);
  }
  ld* zp = (ld*)malloc(sizeof(ld) * (size_t)(wc * TRUTH_PANEL)); /* panel transposed: zp[col - c0][r] */
  for (int64_t r0 = beg; r0 < end; r0 += TRUTH_PANEL) {
    const int64_t rr = end - r0 < TRUTH_PANEL ? end - r0 : TRUTH_PANEL;
    for (int64_t r = 0; r < rr; ++r) {
      const int64_t row = j->rows[r0 + r];
      for (int64_t c = c0; c < w; ++c)
        zp[(c - c0) * TRUTH_PANEL + r] =
            (c < k ? load_val(j->x, j->f32, row * k + c) : load_val(j->y, j->f32, row * m + (c - k))) - j->shift[c];
    }
    if (ib == 0)
      for (int64_t c = 0; c < w; ++c) {
        ld a = 0, b = 0;
        for (int64_t r = 0; r < rr; ++r) {
          a += zp[c * TRUTH_PANEL + r];
          b += zp[c * TRUTH_PANEL + r] * zp[c * TRUTH_PANEL + r];
        }
        s[c] += a;
        q[c] += b;
      }
    for (int64_t i = i_lo; i < i_hi; ++i) {
      const ld* zi = zp + (i - c0) * TRUTH_PANEL;
      for (int64_t c = i; c < w; ++c) {
        const ld* zc = zp + (c - c0) * TRUTH_PANEL;
        ld a0 = 0, a1 = 0, a2 = 0, a3 = 0;
        int64_t r = 0;
        for (; r + 4 <= rr; r += 4) {
          a0 += zi[r] * zc[r];
          a1 += zi[r + 1] * zc[r + 1];
          a2 += zi[r + 2] * zc[r + 2];
          a3 += zi[r + 3] * zc[r + 3];
        }
        for (; r < rr; ++r) a0 += zi[r] * zc[r];
        g[i * w + c] += (a0 + a1) + (a2 + a3);
      }
    }
  }
  free(zp);
}

static void* truth_worker(void* arg) {
  truth_job* j = (truth_job*)arg;
  for (;;) {
    const int64_t t = __atomic_fetch_add(&j->next, 1, __ATOMIC_RELAXED);
    if (t >= j->ntasks) break;
    truth_task(j, t);
  }
  return NULL;
}

/* Per-configuration epilogue of RLD (fast.hpp:94-128 in long double, shifted basis). */
static void truth_epilogue(const truth_job* j, int32_t p, const ld* gt, const ld* st, const ld* qt, uint32_t cfg,
                           double* xtx, double* xty, double* mean_x, double* mean_y, double* std_x, double* std_y,
                           int64_t* n_train, int64_t* n_val) {
  const int64_t n = j->n, k = j->k, m = j->m, w = j->w;
  const ld* shift = j->shift;
  ld* mz = (ld*)malloc(sizeof(ld) * (size_t)w);
  ld* sd = (ld*)malloc(sizeof(ld) * (size_t)w);
  ld* sT = (ld*)malloc(sizeof(ld) * (size_t)w);
  for (int32_t f = 0; f < p; ++f) {
    const int64_t nv = j->offsets[f + 1] - j->offsets[f], nt = n - nv;
    const ld ntl = (ld)nt;
    if (n_train) n_train[f] = nt;
    if (n_val) n_val[f] = nv;
    for (int64_t c = 0; c < w; ++c) {
      sT[c] = st[c] - j->sv[f * w + c];
      const ld qT = qt[c] - j->qv[f * w + c];
      mz[c] = sT[c] / ntl;
      ld rad = (qT - sT[c] * mz[c]) / (ntl - 1);
      /* exact-zero rule of training_std (fast.hpp:66-67): a training column
       * whose variance is below long-double resolution is constant. */
      if (rad <= 64 * LDBL_EPSILON * (qT / (ntl - 1))) rad = 0;
      ld sq = sqrtl(rad);
      sd[c] = sq == 0 ? 1 : sq;
    }
    if (ANY(cfg)) {
      if (mean_x)
        for (int64_t c = 0; c < k; ++c) mean_x[f * k + c] = (double)(shift[c] + mz[c]);
      if (mean_y)
        for (int64_t c = 0; c < m; ++c) mean_y[f * m + c] = (double)(shift[k + c] + mz[k + c]);
    }
    if ((cfg & SX) && std_x)
      for (int64_t c = 0; c < k; ++c) std_x[f * k + c] = (double)sd[c];
    if ((cfg & SY) && std_y)
      for (int64_t c = 0; c < m; ++c) std_y[f * m + c] = (double)sd[k + c];
    const ld* g = j->gv + f * k * w;
    for (int64_t i = 0; i < k; ++i)
      for (int64_t c = i; c < w; ++c) {
        ld v = gt[i * w + c] - g[i * w + c];
        const int is_x = c < k;
        const int centered = is_x ? (cfg & CX) != 0 : ANY_CENTER(cfg);
        if (centered)
          v -= ntl * mz[i] * mz[c];
        else
          v += shift[i] * sT[c] + sT[i] * shift[c] + ntl * shift[i] * shift[c];
        if (is_x) {
          if (cfg & SX) v /= sd[i] * sd[c];
          xtx[f * k * k + i * k + c] = (double)v;
          xtx[f * k * k + c * k + i] = (double)v;
        } else {
          if (ANY_SCALE(cfg)) v /= ((cfg & SX) ? sd[i] : 1) * ((cfg & SY) ? sd[c] : 1);
          xty[f * k * m + i * m + (c - k)] = (double)v;
        }
      }
  }
  free(mz);
  free(sd);
  free(sT);
}

/* RLD for n_cfg configurations from ONE long-double Gram pass.  Outputs are [n_cfg][p][...]. */
int orc_truth_all_folds_multi(const void* x, const void* y, int is_f32, int64_t n, int64_t k, int64_t m,
                              const int32_t* labels, int64_t n_labels, int32_t p, const uint32_t* cfgs, int n_cfg,
                              int n_threads, double* xtx, double* xty, double* mean_x, double* mean_y, double* std_x,
                              double* std_y, int64_t* n_train, int64_t* n_val, char* err, size_t errlen) {
  for (int c = 0; c < n_cfg; ++c) {
    int rc = run_checks(n, k, m, labels, n_labels, p, cfgs[c], err, errlen);
    if (rc) return rc;
  }
  const int64_t w = k + m;
  ld* shift = (ld*)malloc(sizeof(ld) * (size_t)w);
  for (int64_t c = 0; c < w; ++c) {
    ld acc = 0;
    for (int64_t r = 0; r < n; ++r)
      acc += c < k ? load_val(x, is_f32, r * k + c) : load_val(y, is_f32, r * m + (c - k));
    shift[c] = (ld)(double)(acc / (ld)n); /* fp64-rounded: z = x - c is exact for near-constant columns */
  }
  int64_t* rows = (int64_t*)malloc(sizeof(int64_t) * (size_t)n);
  int64_t* offsets = (int64_t*)malloc(sizeof(int64_t) * (size_t)(p + 1));
  orc_build_validation_partitions(labels, n, p, rows, offsets);
  ld* gv = (ld*)malloc(sizeof(ld) * (size_t)(p * k * w));
  ld* sv = (ld*)malloc(sizeof(ld) * (size_t)(p * w));
  ld* qv = (ld*)malloc(sizeof(ld) * (size_t)(p * w));
  if (!shift || !rows || !offsets || !gv || !sv || !qv) return ORC_E_OOM;
  const int64_t nib = (k + TRUTH_IB - 1) / TRUTH_IB;
  truth_job job = {x, y, is_f32, n, k, m, w, rows, offsets, shift, gv, sv, qv, nib, (int64_t)p * nib, 0};
  const int workers = n_threads < 1 ? 1 : (int64_t)n_threads < job.ntasks ? n_threads : (int)job.ntasks;
  pthread_t* th = (pthread_t*)malloc(sizeof(pthread_t) * (size_t)workers);
  for (int t = 0; t < workers; ++t) pthread_create(&th[t], NULL, truth_worker, &job);
  for (int t = 0; t < workers; ++t) pthread_join(th[t], NULL);
  free(th);
  /* totals: folds in ascending order */
  ld* gt = (ld*)calloc((size_t)(k * w), sizeof(ld));
  ld* st = (ld*)calloc((size_t)w, sizeof(ld));
  ld* qt = (ld*)calloc((size_t)w, sizeof(ld));
  for (int32_t f = 0; f < p; ++f) {
    for (int64_t i = 0; i < k; ++i)
      for (int64_t c = i; c < w; ++c) gt[i * w + c] += gv[f * k * w + i * w + c];
    for (int64_t c = 0; c < w; ++c) {
      st[c] += sv[f * w + c];
      qt[c] += qv[f * w + c];
    }
  }
  for (int c = 0; c < n_cfg; ++c) {
    const int64_t o = (int64_t)c * p;
    truth_epilogue(&job, p, gt, st, qt, cfgs[c], xtx + o * k * k, xty + o * k * m, mean_x ? mean_x + o * k : NULL,
                   mean_y ? mean_y + o * m : NULL, std_x ? std_x + o * k : NULL, std_y ? std_y + o * m : NULL,
                   n_train, n_val);
  }
  free(gt);
  free(st);
  free(qt);
  free(shift);
  free(rows);
  free(offsets);
  free(gv);
  free(sv);
  free(qv);
  return ORC_OK;
}

int orc_truth_all_folds(const void* x, const void* y, int is_f32, int64_t n, int64_t k, int64_t m,
                        const int32_t* labels, int64_t n_labels, int32_t p, uint32_t cfg, int n_threads,
                        double* xtx, double* xty, double* mean_x, double* mean_y, double* std_x, double* std_y,
                        int64_t* n_train, int64_t* n_val, char* err, size_t errlen) {
  return orc_truth_all_folds_multi(x, y, is_f32, n, k, m, labels, n_labels, p, &cfg, 1, n_threads, xtx, xty, mean_x,
                                   mean_y, std_x, std_y, n_train, n_val, err, errlen);
}

int orc_version(void) { return 1; }
