/*
 * cvgram CPU ORACLE — TEST INFRASTRUCTURE ONLY (see cvgram_oracle.c header).
 * Cache-blocked fp64 GEMM standing in for Eigen's x.transpose() * y
 * (fast.hpp:23-24, 91-92; baseline.hpp:72-73).  Compiled with FMA
 * contraction; Eigen's own summation order is unspecified.
 */
#include <math.h>
#include <stdlib.h>
#include <string.h>

#include "oracle_internal.h"

/* ------------------------------------------------------------------------- */
/* fp64 GEMM C = AᵀB over `rows` rows (stands in for Eigen's x.transpose()*y). */
/* A: rows x ka (pitch lda), B: rows x nb (pitch ldb), C: ka x nb (pitch ldc). */
/* Cache-blocked, register-tiled, AVX-512 or AVX2 picked at run time.         */
/* ------------------------------------------------------------------------- */
typedef double v8d __attribute__((vector_size(64), aligned(8), may_alias));
typedef double v4d __attribute__((vector_size(32), aligned(8), may_alias));

#define ROW_PANEL 192

__attribute__((target("avx512f,fma"))) static void mk_avx512(const double* A, int64_t lda, const double* B,
                                                             int64_t ldb, int64_t rows, double* C, int64_t ldc) {
  /* 4 x 16 block of C */
  v8d c00 = {0}, c01 = {0}, c10 = {0}, c11 = {0}, c20 = {0}, c21 = {0}, c30 = {0}, c31 = {0};
  for (int64_t r = 0; r < rows; ++r) {
    const double* a = A + r * lda;
    const double* b = B + r * ldb;
    v8d b0 = *(const v8d*)b, b1 = *(const v8d*)(b + 8);
    double a0 = a[0], a1 = a[1], a2 = a[2], a3 = a[3];
    c00 += a0 * b0; c01 += a0 * b1;
    c10 += a1 * b0; c11 += a1 * b1;
    c20 += a2 * b0; c21 += a2 * b1;
    c30 += a3 * b0; c31 += a3 * b1;
  }
  *(v8d*)(C) += c00; *(v8d*)(C + 8) += c01;
  *(v8d*)(C + ldc) += c10; *(v8d*)(C + ldc + 8) += c11;
  *(v8d*)(C + 2 * ldc) += c20; *(v8d*)(C + 2 * ldc + 8) += c21;
  *(v8d*)(C + 3 * ldc) += c30; *(v8d*)(C + 3 * ldc + 8) += c31;
}

__attribute__((target("avx2,fma"))) static void mk_avx2(const double* A, int64_t lda, const double* B, int64_t ldb,
                                                        int64_t rows, double* C, int64_t ldc) {
  /* 4 x 16 block of C as two 4 x 8 halves (12 ymm accumulators would spill). */
  for (int h = 0; h < 2; ++h) {
    v4d c00 = {0}, c01 = {0}, c10 = {0}, c11 = {0}, c20 = {0}, c21 = {0}, c30 = {0}, c31 = {0};
    for (int64_t r = 0; r < rows; ++r) {
      const double* a = A + r * lda;
      const double* b = B + r * ldb + 8 * h;
      v4d b0 = *(const v4d*)b, b1 = *(const v4d*)(b + 4);
      double a0 = a[0], a1 = a[1], a2 = a[2], a3 = a[3];
      c00 += a0 * b0; c01 += a0 * b1;
      c10 += a1 * b0; c11 += a1 * b1;
      c20 += a2 * b0; c21 += a2 * b1;
      c30 += a3 * b0; c31 += a3 * b1;
    }
    double* c = C + 8 * h;
    *(v4d*)(c) += c00; *(v4d*)(c + 4) += c01;
    *(v4d*)(c + ldc) += c10; *(v4d*)(c + ldc + 4) += c11;
    *(v4d*)(c + 2 * ldc) += c20; *(v4d*)(c + 2 * ldc + 4) += c21;
    *(v4d*)(c + 3 * ldc) += c30; *(v4d*)(c + 3 * ldc + 4) += c31;
  }
}

static int g_have_avx512 = -1;

static void mk_scalar(const double* A, int64_t lda, int64_t ni, const double* B, int64_t ldb, int64_t nj,
                      int64_t rows, double* C, int64_t ldc) {
  for (int64_t i = 0; i < ni; ++i)
    for (int64_t j = 0; j < nj; ++j) {
      double s = 0.0;
      for (int64_t r = 0; r < rows; ++r) s += A[r * lda + i] * B[r * ldb + j];
      C[i * ldc + j] += s;
    }
}

/* C[i0:i1, :nb] += A[:, i0:i1]ᵀ B ; if sym (A==B), only blocks with j >= i-block start. */
static void gemm_tn_range(const double* A, int64_t lda, int64_t i0, int64_t i1, const double* B, int64_t ldb,
                          int64_t nb, int64_t rows, double* C, int64_t ldc, int sym) {
  if (g_have_avx512 < 0) g_have_avx512 = __builtin_cpu_supports("avx512f") ? 1 : 0;
  for (int64_t r0 = 0; r0 < rows; r0 += ROW_PANEL) {
    int64_t rr = rows - r0 < ROW_PANEL ? rows - r0 : ROW_PANEL;
    const double* Ap = A + r0 * lda;
    const double* Bp = B + r0 * ldb;
    for (int64_t i = i0; i < i1; i += 4) {
      int64_t ni = i1 - i < 4 ? i1 - i : 4;
      int64_t jstart = sym ? (i / 16) * 16 : 0;
      for (int64_t j = jstart; j < nb; j += 16) {
        int64_t nj = nb - j < 16 ? nb - j : 16;
        if (ni == 4 && nj == 16) {
          if (g_have_avx512)
            mk_avx512(Ap + i, lda, Bp + j, ldb, rr, C + i * ldc + j, ldc);
          else
            mk_avx2(Ap + i, lda, Bp + j, ldb, rr, C + i * ldc + j, ldc);
        } else {
          mk_scalar(Ap + i, lda, ni, Bp + j, ldb, nj, rr, C + i * ldc + j, ldc);
        }
      }
    }
  }
}

typedef struct {
  const double *A, *B;
  int64_t lda, ldb, ka, nb, rows, ldc;
  double* C;
  int sym;
  int64_t nparts;
  const int64_t* bounds;
} gemm_job;

static void gemm_job_fn(void* ctx, int64_t t) {
  gemm_job* j = (gemm_job*)ctx;
  gemm_tn_range(j->A, j->lda, j->bounds[t], j->bounds[t + 1], j->B, j->ldb, j->nb, j->rows, j->C, j->ldc, j->sym);
}

/* C = AᵀB (overwrites C).  sym: B == A and nb == ka; mirrors the lower triangle. */
void orc_gemm_tn(const double* A, int64_t lda, int64_t ka, const double* B, int64_t ldb, int64_t nb,
                    int64_t rows, double* C, int64_t ldc, int sym, int n_threads) {
  for (int64_t i = 0; i < ka; ++i) memset(C + i * ldc, 0, sizeof(double) * (size_t)nb);
  int parts = n_threads < 1 ? 1 : n_threads;
  if (ka < 4 * parts) parts = (int)((ka + 3) / 4);
  if (parts < 1) parts = 1;
  int64_t* bounds = (int64_t*)malloc(sizeof(int64_t) * (size_t)(parts + 1));
  /* balance by work: symmetric work in row i ~ (ka - i) */
  bounds[0] = 0;
  for (int t = 1; t < parts; ++t) {
    double f = (double)t / parts;
    int64_t b = sym ? (int64_t)(ka * (1.0 - sqrt(1.0 - f))) : (int64_t)(ka * f);
    b = (b / 4) * 4;
    if (b < bounds[t - 1]) b = bounds[t - 1];
    bounds[t] = b;
  }
  bounds[parts] = ka;
  gemm_job job = {A, B, lda, ldb, ka, nb, rows, ldc, C, sym, parts, bounds};
  orc_parallel_for(parts, parts, gemm_job_fn, &job);
  free(bounds);
  if (sym)
    for (int64_t i = 0; i < ka; ++i)
      for (int64_t j = 0; j < i; ++j) C[i * ldc + j] = C[j * ldc + i];
}

