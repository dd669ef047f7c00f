/* Internal declarations shared by the oracle translation units (test infrastructure only). */
#pragma once
#include <stdint.h>

typedef void (*orc_task_fn)(void* ctx, int64_t i);
/* detail::parallel_for, threading.hpp:12-26 (strided worker assignment). */
void orc_parallel_for(int64_t count, int n_threads, orc_task_fn fn, void* ctx);
/* C = AᵀB over `rows` rows; sym => B == A, lower triangle mirrored. */
void orc_gemm_tn(const double* A, int64_t lda, int64_t ka, const double* B, int64_t ldb, int64_t nb,
                 int64_t rows, double* C, int64_t ldc, int sym, int n_threads);
