// Internal declarations of the cvgram B200 engine (kernels + host orchestration).
//
// HBM layout:
//   Z      [zrows][kp] fp64   fold-bucketed, shifted rows z = [x - c | y - d | 1 | 0...];
//                             each owned fold is a contiguous block padded with zero
//                             rows to a multiple of kRowStep; kp = roundup(k+m+1, 64).
//   part   [nseg][kp][kp]     per-segment Gram partials (upper 64x64 tiles only);
//                             a segment is <= kChunkRows rows of one fold.
//   foldG  [nmulti][kp][kp]   fold Grams of folds with > 1 segment (fixed-order sums).
//   local  [kp][kp]           this plan's fold-tree node (the cross-rank exchange unit).
//   total  [kp][kp]           the whole-data Gram in the shifted basis.
// Column k+m of Z is all ones on real rows, so Gram[j][k+m] is the column sum and
// Gram[j][j] the sum of squares: the per-fold statistics ride in the Gram pass.
#pragma once

#include <atomic>
#include <cstdio>

#include <cuda_runtime.h>
#include <stdint.h>

#include <string>
#include <vector>

namespace cvg {

constexpr int kTile = 64;          // Gram / epilogue tile edge (columns)
constexpr int kRowStep = 32;       // rows per pipeline stage; fold blocks pad to this
// max rows per fp64 segment (a fixed constant => a deterministic split; folds are cut into equal
// segments, Plan::seg_rows).  8192 vs 32768: c1 10.70 vs 10.81 ms (two even CTAs per fold fill the
// last wave better), c4 45.4 vs 45.8.
constexpr int64_t kChunkRows = 8192;
// fp32 segments (fp16 hi/lo operands: 4 B per Z element, half of fp64's): c3 sweep of the total step
// with the kind::f16 Gram: 8192 -> 27.8 ms, 12288 -> 26.7, 16384 -> 26.4, 24576 -> 25.3, 32768 -> 25.1,
// 49152 -> 25.8, 65536 -> 25.2 (the fold tree shrinks from 1.30 to 0.19 ms; the Gram is flat within noise
// up to 32768 rows).  A multiple of every fp16 row group (64 / 128 / 256).
constexpr int64_t kChunkRowsF32 = 32768;
// 3xTF32 operands (CVG_FP32_KIND=tf32, 8 B per element): 32768 -> 44.9 ms, 16384 -> 44.5, 12288 -> 42.9,
// 8192 -> 44.2 on c3 (shorter segments re-read less from DRAM; the tree over more partials eats the rest).
constexpr int64_t kChunkRowsTf32 = 12288;
// int8-slice fp64 Gram (default fp64 kind): exact int32 TMEM sums need S * 2^14 * rows < 2^31 for base-256
// digits in [-128, 127] (rows < 21,845 at S = 6); the exponent is per (segment, column).
constexpr int64_t kChunkRowsI8 = 16384;
constexpr int kTileF32 = 128;             // tcgen05 tile edge (M = N = 128)
constexpr int kTileRowsPerWarp = 1024; // rows per warp in the bucketing passes (at least)
// Bound on the bucketing's tile x fold counter table (int32): 2^26 counters = 256 MB.  Past it
// (leave-one-out-scale P) tiles grow by powers of two, so memory stays O(N + P), not O(N P / 1024).
constexpr int64_t kMaxTileCounters = int64_t(1) << 26;

// Checked builds (make CHECKED=1 -> _build_checked/, selected with CVG_LIB_VARIANT=checked):
// device-side bounds assertions on every index the kernels derive (row maps,
// segment ranges, tile coordinates, scatter positions).  A failed check prints
// the site and traps, which surfaces as CVG_E_CUDA.  compute-sanitizer is not
// available on this pool, so this build + the GPU suite is the bounds evidence.
#ifndef CVG_CHECKED
#define CVG_CHECKED 0
#endif
#if CVG_CHECKED
#define CVG_DCHECK(cond)                                                                                   \
  do {                                                                                                     \
    if (!(cond)) {                                                                                         \
      printf("CVG_DCHECK failed: %s at %s:%d block %d thread %d\n", #cond, __FILE__, __LINE__, (int)blockIdx.x, \
             (int)threadIdx.x);                                                                            \
      __trap();                                                                                            \
    }                                                                                                      \
  } while (0)
#else
#define CVG_DCHECK(cond) \
  do {                   \
  } while (0)
#endif

struct Status {
  int code = 0;
  std::string msg;
  bool ok() const { return code == 0; }
  static Status Ok() { return {}; }
  static Status Err(int c, std::string m) { return {c, std::move(m)}; }
};

// ------------------------------------------------------------------ kernels
// Bucketing (build_validation_partitions, partition.hpp:61-68) on the device.
int64_t bucket_tile_rows(int64_t n, int32_t p);  // rows per bucketing tile (>= kTileRowsPerWarp)
void launch_tile_histogram(const int32_t* labels, int64_t n, int32_t p, int32_t* tile_counts,
                           unsigned long long* bad_row, cudaStream_t s);
void launch_tile_scan(int32_t* tile_counts, int64_t ntiles, int32_t p, int64_t* fold_counts, cudaStream_t s);
// Rows at fold-relative bucketed positions outside [win_lo, win_hi) are dropped
// (a rank owning only part of one fold's segments).
void launch_scatter(const int32_t* labels, int64_t n, int32_t p, int32_t fold_begin, int32_t fold_end,
                    int32_t* tile_offsets, const int64_t* fold_zbase, int64_t win_lo, int64_t win_hi, int64_t* src_row,
                    int64_t zrows, cudaStream_t s);

// out[r] = map[src_row[r]] (-1 for padding rows); *bad = 1 if a bound row is unmapped.
void launch_remap_rows(const int64_t* src_row, int64_t zrows, const int64_t* map, int64_t n_map, int64_t n_compact,
                       int64_t* out, int* bad, cudaStream_t s);
// K1: gather + shift + ones column + zero padding (+ finiteness flag).
void launch_reorder(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                    const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc,
                    const double* shift, double* z, int* nonfinite, cudaStream_t s);
void launch_shift_from_row0(int dtype, const void* x, const void* y, int64_t k, int64_t m, double* shift,
                            cudaStream_t s);

// K2: segmented fold Gram, fp64 DMMA.  One CTA per (segment, upper tile).
struct GramTask {
  int64_t zrow;  // first Z row of the segment
  int64_t rows;  // padded row count (multiple of kRowStep)
};
void launch_gram_f64(const double* z, int64_t kp, int64_t zrows, const GramTask* segs, int64_t nseg,
                     const int2* tiles, int ntiles, double* part, cudaStream_t s);

// K4: fixed-order (midpoint-tree) sums of kp x kp matrices over upper tiles.  One op is a node S(a, b) of a
// midpoint tree evaluated down to depth kTreeFanDepth in registers: its inputs are the node's frontier at that
// depth, left to right (leaves, or nodes computed by deeper ops), and
//   S(size) = in  if depth == kTreeFanDepth or size == 1,  else S(size / 2) + S(size - size / 2)
// -- the same additions, in the same order, as the unfused binary tree; size 0 zeroes d.
constexpr int kTreeFanDepth = 4;
constexpr int kTreeFanIn = 1 << kTreeFanDepth;
struct TreeOp {
  const double* in[kTreeFanIn];
  double* d;
  int size;  // leaves under the node (the recursion's shape)
};
void launch_tree_ops(const TreeOp* ops, int nops, int64_t kp, const int2* tiles, int ntiles, cudaStream_t s);
// g[0] = NaN when *flag has bit 0 set (non-finite input seen by K1): the flag rides in the partial.
void launch_poison_if_flag(const int* flag, double* g, cudaStream_t s);

// K5: epilogue.
struct FoldStatsDev {
  double* mz;   // [nfold][kp] training mean in the shifted basis (padding columns: 0)
  double* sT;   // [nfold][kp] training column sums (shifted; padding: 0)
  double* sd;   // [nfold][kp] training std (zero -> 1; padding: 1)
};  // rows of kp (a multiple of 64): every 64-column slice is a whole, 16-byte aligned 512 B copy
// Small-fold mode (every fold <= kSmallFoldRows rows, e.g. leave-one-out): no per-fold Gram partials; a fold's
// Gram entries are formed in the epilogue from its rows of Z (z: zrows x kp, rows zbase[f] .. + n_val[f]).
constexpr int kSmallFoldRows = 32;
struct SmallFolds {
  const double* z = nullptr;       // null: fold Grams come from foldG
  const int64_t* zbase = nullptr;  // first Z row of each fold
};
void launch_fold_stats(const double* total, const double* const* foldG, const int64_t* n_val, int nfold, int64_t n,
                       int64_t k, int64_t m, int64_t kp, const double* shift, FoldStatsDev st, double* mean_x,
                       double* mean_y, double* std_x, double* std_y, int* nonfinite, cudaStream_t s,
                       SmallFolds sf = SmallFolds());
// tiles[0, ndiag) are the diagonal tiles; returns the number of kernels launched.
int launch_products(const double* total, const double* const* foldG, const int64_t* n_val, int nfold, int64_t n,
                    int64_t k, int64_t m, int64_t kp, const double* shift, FoldStatsDev st, const int2* tiles,
                    int ntiles, int ndiag, const uint32_t* cfgs, int ncfg, double* xtx, double* xty, cudaStream_t s,
                    SmallFolds sf = SmallFolds());
// div_rn_fast vs __ddiv_rn over n hashed operand pairs: counts[0] += mismatches, counts[1] += fast-path quotients.
void launch_selftest_division(uint64_t seed, int64_t n, unsigned long long* counts, cudaStream_t s);
void launch_unshift_global(const double* total, int64_t n, int64_t k, int64_t m, int64_t kp, const double* shift,
                           double* xtx, double* xty, double* sum, double* sumsq, double* mean, cudaStream_t s);
void launch_training_mean(const double* g, const double* v, int64_t len, int64_t n, int64_t nv, double* out,
                          cudaStream_t s);
void launch_training_std(const double* mt, const double* st, const double* qt, int64_t len, int64_t nt,
                         double* out, cudaStream_t s);
void launch_hadamard(const double* mat, int64_t rows, int64_t cols, const double* l, const double* r, double* out,
                     cudaStream_t s);

// Tile list of the symmetric Gram (ti <= tj), plus the diagonal/ones tiles of
// Y-only column blocks, for tile edge `edge`.  The 64-tile list drives the
// reductions and the epilogue; the fp32 Gram uses the 128-tile list.
std::vector<int2> gram_tiles(int64_t k, int64_t m, int64_t kp, int edge = kTile);

// K1T + K2' (fp32 inputs): bucket/shift/split into TF32 hi + lo, transposed in
// 32-row blocks;
// then the tcgen05 kind::tf32 Gram (3 products: hi·hi + hi·lo + lo·hi).
void launch_reorder_split_t(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                            const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                            const double* shift, float* zt_hi, float* zt_lo, int* nonfinite, cudaStream_t s);
// K1H + K2h (fp32 inputs, default): bucket/shift, per-(G-row group, column) power-of-two
// scaling, fp16 hi + lo split into Zh[row / 64][col][64]; then the tcgen05 kind::f16 Gram
// (3 products, fp32 TMEM chunks of one row group, exact unscale into fp64).  k_gram_f16.cu.
bool launch_reorder_split_h(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                            const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                            int64_t nsrc, const double* shift, int group_rows, void* zh_hi, void* zh_lo,
                            float* unscale, int* nonfinite, cudaStream_t s);
bool launch_gram_f16s(const void* zh_hi, const void* zh_lo, const float* unscale, int group_rows, int64_t zrows,
                      int64_t kp, const GramTask* segs, int64_t nseg, const int2* tiles128, int ntiles, double* part,
                      cudaStream_t s);
bool launch_gram_tf32(const float* zt_hi, const float* zt_lo, int64_t zrows, int64_t kp, const GramTask* segs,
                      int64_t nseg, const int2* tiles128, int ntiles, double* part, int nterms, cudaStream_t s);

// K1Q + K2q (fp64, CVG_FP64_KIND=i8; k_gram_i8.cu): per-(segment, column) exponents from the
// segment's max |z| (segmax), then bucket/shift/scale/cut into `slices` int8 digits laid out
// Zq[t][row / 64][col][64]; the tcgen05 kind::i8 Gram sums the slice pairs t + u < slices into
// int32 TMEM and drains each (segment, 128 x 64 tile) once into the fp64 partial.
// blkseg[b]: segment of Z's 64-row block b.  tiles: {I, J | write mask << 16}.
// segmax must be zeroed before (bits of max |z| per (segment, column); atomicMax).  stride > 1: the
// max over rows 0, stride, 2 stride, ... of each segment (the exponents then keep 2x headroom);
// only != null: just the segments with only[seg] set (the exact pass, on top of the sampled max).
void launch_segmax(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                   const int64_t* src_row, const GramTask* segs, int64_t nseg, int64_t max_seg_rows, int64_t kp,
                   int64_t c_begin, int64_t c_end, int64_t nsrc, const double* shift, int stride, const int* only,
                   unsigned long long* segmax, cudaStream_t s);
// ovf != null (sampled exponents): a value outside the digits' range sets ovf[its segment];
// ovf == null: sets *nonfinite.
bool launch_reorder_q(int dtype, int slices, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k,
                      int64_t m, const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                      int64_t nsrc, const double* shift, const int* blkseg, const unsigned long long* segmax,
                      int headroom, int* ovf, int8_t* zq, int* nonfinite, cudaStream_t s, int64_t blk_lo = 0,
                      int64_t blk_hi = -1, int max_sms = 0, int direct_ctas_per_sm = 0, unsigned* seg_ready = nullptr);
// direct_ctas_per_sm > 0: the register-only cut (no shared-memory tile, no TMA) on that many persistent CTAs per
// SM; it counts every finished 64-row block into seg_ready[its segment] (release) when seg_ready != null.
//
// Segments [seg_base, seg_base + nseg) of segs (absolute indices into segs / segmax / part); max_ctas > 0 caps
// the persistent grid.  lean: the 96-register kernel that shares its SM with a cut CTA; seg_ready + abort_flag:
// each item waits for its segment's block count from a concurrent cut (k_gram_i8.cu).
bool launch_gram_i8(int slices, const int8_t* zq, const unsigned long long* segmax, int headroom, int64_t zrows,
                    int64_t kp, const GramTask* segs, int64_t nseg, const int2* tiles, int ntiles, double* part,
                    cudaStream_t s, int64_t seg_base = 0, int max_ctas = 0, int lean = 0,
                    const unsigned* seg_ready = nullptr, int* abort_flag = nullptr, int32_t* split_ws = nullptr,
                    unsigned* split_cnt = nullptr, int64_t min_seg_rows = 0);
// split_ws (gram_i8_split_ws_bytes(SM count) bytes) + split_cnt (SM count words): the items past the grid's last
// full round are cut into row parts whose exact int32 sums are added by the part that finishes last (bit-identical
// to the unsplit item); min_seg_rows bounds the split so every part keeps a few stages.
size_t gram_i8_split_ws_bytes(int ctas);

// Function attributes are per device (one process may drive several: cvg_context_create_multi) but never
// change: a launcher sets them the first time it runs on a device.  `done` is the launcher's own static mask
// (bit = device ordinal, devices beyond 63 simply set them every time).
inline bool first_on_device(std::atomic<uint64_t>& done) {
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev > 63) return true;
  const uint64_t bit = 1ull << dev;
  return !(done.fetch_or(bit, std::memory_order_relaxed) & bit);
}

inline int64_t round_up(int64_t a, int64_t b) { return (a + b - 1) / b * b; }
inline int64_t padded_cols(int64_t k, int64_t m, int dtype = 0) {
  return round_up(k + m + 1, dtype == 1 ? kTileF32 : kTile);
}

}  // namespace cvg
