/*
 * cvgram_b200.h — C ABI of the B200-native all-fold cross-validation XᵀX/XᵀY
 * engine (arXiv 2401.13185, reference: /root/reference/proj/include/cvgram).
 *
 * Plain pointers and sizes only; no torch or CUDA types cross this boundary
 * (streams travel as void*).  Every entry point names the reference interface
 * it replaces.  All calls are synchronous unless stated otherwise; host-pointer
 * entry points copy in and out themselves.  There is no CPU fallback: without
 * a usable sm_100a device every compute call returns CVG_E_CUDA.
 *
 * Status codes map onto the reference's exception types (core.hpp:20-32,
 * exit codes at cvgram_cli.cpp:264-276).  On failure `err` receives the
 * reference's message text (partition.hpp:21-58, fast.hpp:43,56,78-82,137-141,
 * core.hpp:38-44,119-125).
 *
 * Configuration masks use the bit order of enumerate_configs
 * (combos.hpp:33-45): center_x = 8, center_y = 4, scale_x = 2, scale_y = 1.
 */
#ifndef CVGRAM_B200_H_
#define CVGRAM_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define CVG_OK 0
#define CVG_E_DIMENSION 1   /* cvgram::dimension_error   (core.hpp:20-22)  */
#define CVG_E_PARTITION 2   /* cvgram::partition_error   (core.hpp:24-26)  */
#define CVG_E_SCALABILITY 3 /* cvgram::scalability_error (core.hpp:30-32)  */
#define CVG_E_INVALID_ARG 4 /* std::invalid_argument (fast.hpp:43,78-79; core.hpp:122,125) */
#define CVG_E_CUDA 5        /* device missing / kernel or copy failure       */
#define CVG_E_OOM 6         /* device allocation failure                     */
#define CVG_E_NCCL 7        /* NCCL unavailable or a collective failed (multi-device contexts) */

#define CVG_DTYPE_F64 0 /* fp64 inputs, fp64 DMMA Gram (BASELINE configs 0,1,2,4) */
#define CVG_DTYPE_F32 1 /* fp32 inputs (BASELINE config 3)                          */

#define CVG_CENTER_X 8u
#define CVG_CENTER_Y 4u
#define CVG_SCALE_X 2u
#define CVG_SCALE_Y 1u

typedef struct cvg_context cvg_context; /* device, stream, memory pool        */
typedef struct cvg_plan cvg_plan;       /* one partitioning over owned folds */
typedef struct cvg_global cvg_global;   /* device state behind a GlobalCache */

/* ---------------------------------------------------------------- context */
int cvg_version(void);
/* Binds `device` (CUDA ordinal).  Fails with CVG_E_CUDA if it is not sm_100. */
int cvg_context_create(int device, cvg_context** out, char* err, size_t errlen);
void cvg_context_destroy(cvg_context* ctx);
/* A context over n_gpus devices of this node (the reference's run_all_folds(..., n_threads) knob,
 * threading.hpp:12-26, as GPUs).  cvg_run_all_folds on it shards the folds across the devices: each rank owns
 * a node of the canonical fold tree (cvg_fold_range), copies only its row shard over its own PCIe link when
 * p >= n_gpus (rows then move to their fold's owner over NVLink), and the ranks exchange one partial Gram
 * (all-gather); outputs are bit-identical to one device for power-of-two n_gpus.  One host thread per device;
 * the exchanges use NCCL (loaded at run time; CVG_E_NCCL if it cannot be) over distinct devices, or device
 * copies when dev_ids repeats a device (a one-GPU emulation) or CVG_EXCHANGE=peer.  A run whose folds all hold
 * <= 32 rows (leave-one-out scale) stays on dev_ids[0]: one device forms such folds' Grams in its epilogue, a
 * summation order rank plans do not share.  Every other entry point runs on dev_ids[0]. */
int cvg_context_create_multi(int n_gpus, const int* dev_ids, cvg_context** out, char* err, size_t errlen);
/* Devices of a context (1 for cvg_context_create). */
int cvg_context_device_count(const cvg_context* ctx);
/* Exchange backend of a multi-device context: 1 NCCL, 2 device copies, 0 single device. */
int cvg_context_exchange(const cvg_context* ctx);
/* Subsequent work is issued on `stream` (a cudaStream_t; NULL = the context's
 * own non-blocking stream; cudaStreamLegacy = the legacy default stream). */
int cvg_context_set_stream(cvg_context* ctx, void* stream);
/* Number of kernels this context has launched (for the bench's gpu_launches). */
int64_t cvg_context_launch_count(const cvg_context* ctx);
/* Per-kernel-class device timing with CUDA events on the launching stream.
 * Classes: 0 bucketing, 1 reorder (K1), 2 fold Gram (K2), 3 tree sums (K4),
 * 4 fold stats, 5 products (K5).  enable != 0 starts recording (and clears);
 * cvg_context_kernel_times synchronizes and returns total ms and launch counts
 * per class (arrays of CVG_KERNEL_CLASSES). */
#define CVG_KERNEL_CLASSES 6
int cvg_context_enable_timing(cvg_context* ctx, int enable);
int cvg_context_kernel_times(cvg_context* ctx, double* ms, int64_t* launches);

/* ------------------------------------------------- host validation (no GPU) */
/* DatasetPair invariants, core.hpp:37-45. */
int cvg_validate_dataset(const double* x, const double* y, int64_t n, int64_t k, int64_t m, int64_t y_rows,
                         char* err, size_t errlen);
/* validate_partitioning, partition.hpp:21-45: CVG_E_PARTITION with the first violated clause. */
int cvg_validate_partitioning(const int32_t* labels, int64_t n, int32_t p, char* err, size_t errlen);
/* check_scalable, partition.hpp:48-58: CVG_E_SCALABILITY. */
int cvg_check_scalable(const int32_t* labels, int64_t n, int32_t p, char* err, size_t errlen);
/* Canonical fold ownership for `rank` of `world` (a node of the fixed fold-sum
 * tree, so results are bit-identical for every power-of-two world size). */
int cvg_fold_range(int32_t p, int32_t rank, int32_t world, int32_t* begin, int32_t* end);

/* ------------------------------------------------------------ the hot path */
/* run_all_folds (fast.hpp:133-152) for n_cfg configurations at once: one Gram
 * pass serves every configuration.  Host buffers in and out.
 *   x: n x k row-major, y: n x m row-major, element type `dtype`.
 *   labels: n 1-based fold ids (Partitioning::labels), p folds.
 *   xtx: [n_cfg][p][k][k], xty: [n_cfg][p][k][m]  (fp64, caller-allocated)
 *   mean_x/mean_y/std_x/std_y: [n_cfg][p][k|m] or NULL; entries the reference
 *     leaves empty for a configuration (FoldStats, core.hpp:95-105) are not written.
 *   n_train/n_val: [p] or NULL. */
int cvg_run_all_folds(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                      const int32_t* labels, int64_t n_labels, int32_t p, const uint32_t* cfg_masks, int32_t n_cfg,
                      double* xtx, double* xty, double* mean_x, double* mean_y, double* std_x, double* std_y,
                      int64_t* n_train, int64_t* n_val, char* err, size_t errlen);

/* run_all_folds streamed in fold batches (a lazy per-fold generator for
 * leave-one-out-scale P, where the P*K*(K+M) outputs cannot all exist at once).
 * `fn` is called once per batch of folds [fold_lo, fold_hi) (0-based, ascending)
 * with host buffers valid only during the call:
 *   xtx [n_cfg][nb][k][k], xty [n_cfg][nb][k][m]  (nb = fold_hi - fold_lo)
 *   mean_x, std_x [nb][k], mean_y, std_y [nb][m]  (training statistics, every entry filled)
 *   n_train, n_val [nb]
 * A nonzero return from `fn` stops the run early (CVG_OK is still returned).
 * Same values, bit for bit, as cvg_run_all_folds. */
typedef int (*cvg_fold_batch_fn)(int32_t fold_lo, int32_t fold_hi, const double* xtx, const double* xty,
                                 const double* mean_x, const double* mean_y, const double* std_x, const double* std_y,
                                 const int64_t* n_train, const int64_t* n_val, void* user);
int cvg_run_all_folds_stream(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                             const int32_t* labels, int64_t n_labels, int32_t p, const uint32_t* cfg_masks,
                             int32_t n_cfg, int32_t batch, cvg_fold_batch_fn fn, void* user, char* err, size_t errlen);

/* ------------------------------- device-resident staged API (bench, multi-GPU) */
/* A plan owns folds [fold_begin, fold_end) of a p-fold partitioning of n rows. */
int cvg_plan_create(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t fold_begin,
                    int32_t fold_end, cvg_plan** out, char* err, size_t errlen);
void cvg_plan_destroy(cvg_plan* plan);
/* Rank mode: this plan is rank `rank` of `world` and owns its node of the
 * canonical fold tree (cvg_fold_range's descent; when more ranks than folds
 * remain, one fold's segment range is split further — P < G).  Decided at
 * bind time; query it with cvg_plan_assignment.  Outputs are bit-identical to
 * one GPU for power-of-two world sizes. */
int cvg_plan_create_rank(cvg_context* ctx, int dtype, int64_t n, int64_t k, int64_t m, int32_t p, int32_t rank,
                         int32_t world, cvg_plan** out, char* err, size_t errlen);
/* Folds this plan emits after bind: [fold_begin, fold_end) (empty when this
 * rank shares a fold whose outputs another rank of its group emits). */
int cvg_plan_assignment(const cvg_plan* plan, int32_t* fold_begin, int32_t* fold_end);
/* Device labels (n int32, 1-based).  Validates them (partition.hpp:21-45, and
 * check_scalable when require_scalable != 0) and builds the fold-bucketed row
 * order on the device (build_validation_partitions, partition.hpp:61-68). */
int cvg_plan_bind_labels(cvg_plan* plan, const int32_t* d_labels, int require_scalable, char* err, size_t errlen);
/* Gram pass over the owned folds: reorder+shift, segmented fold Gram,
 * deterministic fold sums.  d_x: n rows with pitch ldx elements, d_y pitch ldy.
 * shift: host pointer to k+m values, or NULL for row 0 of (x | y). */
int cvg_plan_gram(cvg_plan* plan, const void* d_x, int64_t ldx, const void* d_y, int64_t ldy, const double* shift,
                  char* err, size_t errlen);
/* cvg_plan_gram over COMPACTED inputs (multi-GPU row exchange): d_x / d_y hold
 * n_compact rows, and original row i (of the n the labels describe) is compact
 * row d_row_map[i] (device int64[n]; -1 = not present).  Every row of the
 * plan's owned folds / segments must be present.  `shift` (k+m host values) is
 * required: row 0 of the full data need not be present.  Same results, bit for
 * bit, as cvg_plan_gram over the full x / y. */
int cvg_plan_gram_mapped(cvg_plan* plan, const void* d_x, int64_t ldx, const void* d_y, int64_t ldy,
                         const int64_t* d_row_map, int64_t n_compact, const double* shift, char* err, size_t errlen);
/* cvg_plan_finish for the emitted folds [fold_lo, fold_hi) only (0-based fold ids
 * inside [fold_begin, fold_end)); outputs are packed for that range
 * ([n_cfg][fold_hi - fold_lo][k][k] ...), so P x K x K outputs can be streamed
 * through bounded buffers (leave-one-out at scale).  Same values as the
 * corresponding slice of cvg_plan_finish. */
int cvg_plan_finish_range(cvg_plan* plan, const double* d_rank_partials, int32_t n_ranks, const uint32_t* cfg_masks,
                          int32_t n_cfg, int32_t fold_lo, int32_t fold_hi, double* d_xtx, double* d_xty,
                          double* d_mean_x, double* d_mean_y, double* d_std_x, double* d_std_y, char* err,
                          size_t errlen);
/* This plan's contribution to the cross-rank fold sum (its node of the fold
 * tree): *count doubles, copied into device buffer d_dst when it is non-NULL. */
int cvg_plan_partial(cvg_plan* plan, double* d_dst, int64_t* count);
/* Epilogue for the owned folds.  d_rank_partials: [n_ranks][count] device
 * buffer holding every rank's cvg_plan_partial in rank order (an all-gather),
 * or NULL when this plan owns all folds.  Device outputs, fold-major over the
 * owned folds: xtx [n_cfg][n_owned][k][k], xty [n_cfg][n_owned][k][m], stats
 * [n_owned][k|m] (configuration-independent; NULL to skip). */
int cvg_plan_finish(cvg_plan* plan, const double* d_rank_partials, int32_t n_ranks, const uint32_t* cfg_masks,
                    int32_t n_cfg, double* d_xtx, double* d_xty, double* d_mean_x, double* d_mean_y,
                    double* d_std_x, double* d_std_y, char* err, size_t errlen);
/* Per-fold validation counts of the bound labels (host array of p). */
int cvg_plan_fold_counts(const cvg_plan* plan, int64_t* counts);

/* ----------------------------------- GlobalCache / single-fold entry points */
/* precompute_global (fast.hpp:19-36): uploads the data, runs the Gram over all
 * rows and keeps the shifted-basis products on the device for fold_products. */
int cvg_global_create(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k, int64_t m,
                      cvg_global** out, char* err, size_t errlen);
void cvg_global_destroy(cvg_global* g);
/* GlobalCache fields for configuration `cfg`; vectors the reference leaves
 * empty for cfg (fast.hpp:25-34) are not written.  Any pointer may be NULL. */
int cvg_global_export(cvg_global* g, uint32_t cfg, double* xtx, double* xty, double* sum_x, double* sum_y,
                      double* mean_x, double* mean_y, double* sum_sq_x, double* sum_sq_y, char* err,
                      size_t errlen);
/* fold_products (fast.hpp:73-130) for validation rows v_rows (0-based, ascending). */
int cvg_global_fold_products(cvg_global* g, const int64_t* v_rows, int64_t n_val, uint32_t cfg, double* xtx_t,
                             double* xty_t, double* mean_x_t, double* mean_y_t, double* std_x_t, double* std_y_t,
                             int64_t* n_train, char* err, size_t errlen);

/* ------------------------------------------ baseline engine (baseline.hpp) */
/* baseline_fold_products (baseline.hpp:79-97) on the device: every fold's
 * training rows are contracted directly in their own mean-centered basis (two
 * passes: training means, then the Gram of x - mean), with no downdate; the
 * independent engine `cvgram verify` checks the fast path against.
 * Same argument layout as cvg_run_all_folds.  Cost: Θ(P·N·K(K+M)). */
int cvg_baseline_fold_products(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k,
                               int64_t m, const int32_t* labels, int64_t n_labels, int32_t p,
                               const uint32_t* cfg_masks, int32_t n_cfg, double* xtx, double* xty, double* mean_x,
                               double* mean_y, double* std_x, double* std_y, int64_t* n_train, int64_t* n_val,
                               char* err, size_t errlen);
/* baseline_single_fold (baseline.hpp:42-76) for validation rows v_rows (0-based, ascending). */
int cvg_baseline_single_fold(cvg_context* ctx, int dtype, const void* x, const void* y, int64_t n, int64_t k,
                             int64_t m, const int64_t* v_rows, int64_t n_val, uint32_t cfg, double* xtx_t,
                             double* xty_t, double* mean_x_t, double* mean_y_t, double* std_x_t, double* std_y_t,
                             int64_t* n_train, char* err, size_t errlen);

/* ------------------------------------------ seeded test data (random.hpp) */
/* An opaque std::mt19937_64 stream (random.hpp:14-18; standard-specified, so
 * seeds reproduce the reference's test data bit for bit). */
typedef struct cvg_rng cvg_rng;
cvg_rng* cvg_rng_create(uint64_t seed);
void cvg_rng_destroy(cvg_rng* rng);
uint64_t cvg_rng_next(cvg_rng* rng);
/* uniform01, random.hpp:16-18 */
double cvg_rng_uniform01(cvg_rng* rng);
/* random_dataset, random.hpp:21-27 (row-major X first, then Y). */
void cvg_random_dataset(cvg_rng* rng, int64_t n, int64_t k, int64_t m, double* x, double* y);
/* random_partitioning, random.hpp:38-50 (balanced labels, Fisher-Yates). */
void cvg_random_partitioning(cvg_rng* rng, int64_t n, int32_t p, int32_t* labels);
/* The same two generators over a caller-owned 64-bit engine: next(state) returns its next
 * draw.  The C++ header (cvgram/random.hpp) passes the caller's std::mt19937_64 through
 * these, so the seeded-data contract has one implementation.  cvg_uniform01_bits maps one
 * draw to [0, 1) (random.hpp:16-18). */
typedef uint64_t (*cvg_next_fn)(void* state);
double cvg_uniform01_bits(uint64_t draw);
void cvg_random_dataset_fn(cvg_next_fn next, void* state, int64_t n, int64_t k, int64_t m, double* x, double* y);
void cvg_random_partitioning_fn(cvg_next_fn next, void* state, int64_t n, int32_t p, int32_t* labels);

/* ------------------------------------------- small vector kernels (fast.hpp) */
/* training_mean, fast.hpp:40-47 (on the device). */
int cvg_training_mean(cvg_context* ctx, const double* global_mean, const double* val_mean, int64_t len, int64_t n,
                      int64_t n_val, double* out, char* err, size_t errlen);
/* training_std, fast.hpp:53-69 (on the device). */
int cvg_training_std(cvg_context* ctx, const double* mean_t, const double* sum_t, const double* sum_sq_t,
                     int64_t len, int64_t n_train, double* out, char* err, size_t errlen);
/* hadamard_outer_divide, core.hpp:116-130 (on the device). */
int cvg_hadamard_outer_divide(cvg_context* ctx, const double* mat, int64_t rows, int64_t cols, const double* left,
                              int64_t n_left, const double* right, int64_t n_right, double* out, char* err,
                              size_t errlen);

/* ------------------------------------------------- pinned host output buffers */
/* Page-locked host memory from a process-wide pool (64 KB granularity): output arrays allocated here receive
 * cvg_run_all_folds' device-to-host copies at full PCIe speed, and a freed block is reused by the next
 * allocation of a similar size (no cudaHostAlloc, no first-touch page faults).  CVG_E_OOM if no block. */
int cvg_host_alloc(size_t bytes, void** out);
void cvg_host_free(void* p);

/* ------------------------------------------------------------- self-tests */
/* The epilogue's branch-free fp64 division (the scaled outputs' one division by the product,
 * core.hpp:128) against the hardware-correct div.rn.f64 over n hashed operand pairs (NaN/inf/subnormal
 * patterns, quotients near 1, underflow/overflow edges).  *mismatches = fast-path quotients whose bits
 * differ (must be 0), *fast = quotients the fast path accepted. */
int cvg_selftest_division(cvg_context* ctx, int64_t n, uint64_t seed, int64_t* mismatches, int64_t* fast);

#ifdef __cplusplus
}
#endif
#endif /* CVGRAM_B200_H_ */
