// Fold bucketing on the device: a stable counting sort of rows by fold label.
// Replaces build_validation_partitions (partition.hpp:61-68) + gather_rows
// (partition.hpp:85-90, called at fast.hpp:84-85): instead of P row lists and P
// gathered copies, every owned fold becomes one contiguous, zero-padded block of
// the Z matrix, rows in ascending original order (the reference's Algorithm 1
// order), so the Gram reads each fold with plain sequential tiles.
//
// Three passes, all integer work, bit-exact by construction:
//   1. tile histogram: one warp per tile (1024 rows, or more when P is large: the
//      tile x fold table stays <= 2^26 counters) counts its labels (warp
//      __match_any_sync groups equal labels; the group leader owns the update,
//      so no atomics and no contention).  Out-of-range labels record the first
//      offending row (validate_partitioning's first violated clause,
//      partition.hpp:34-38).
//   2. per-fold exclusive scan over tiles (one CTA per fold).
//   3. stable scatter: same warp/tile walk, rank = popc(peers below me).
#include "cvg_internal.cuh"

namespace cvg {
namespace {

// P <= kSmemFolds: each warp keeps its tile's row of counters / offsets in shared memory (the read-modify-
// write per 32 labels is then a shared-memory round trip, not a global one; c1: 35 -> ~5 us per pass).
constexpr int kSmemFolds = 1024;
constexpr int kBucketThreads = 256;
constexpr int kBatch = 8;  // labels loaded ahead per lane

__global__ void tile_histogram_kernel(const int32_t* __restrict__ labels, int64_t n, int32_t p, int64_t tile_rows,
                                      int32_t* __restrict__ tile_counts, unsigned long long* __restrict__ bad) {
  extern __shared__ int32_t s_cnt[];
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = warp * tile_rows;
  const bool in_smem = p <= kSmemFolds;
  int32_t* counts = in_smem ? s_cnt + (threadIdx.x >> 5) * p : tile_counts + warp * p;
  if (in_smem) {  // global counters are zeroed by the caller; shared ones here
    for (int f = lane; f < p; f += 32) counts[f] = 0;
    __syncwarp();
  }
  if (row0 >= n) return;
  const int64_t row_end = min(n, row0 + tile_rows);
  // kBatch label loads in flight per lane: the walk itself is a chain of shared-memory round trips, so it
  // must not also wait for one global load per 32 labels (c1: 30 -> ~12 us per pass)
  for (int64_t base0 = row0; base0 < row_end; base0 += 32 * kBatch) {
    int32_t lab[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int64_t row = base0 + 32 * b + lane;
      lab[b] = row < row_end ? __ldg(labels + row) : 0;
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int64_t row = base0 + 32 * b + lane;
      const bool live = row < row_end;
      const int32_t label = lab[b];
      const bool good = live && label >= 1 && label <= p;
      if (live && !good) atomicMin(bad, (unsigned long long)row);
      const unsigned act = __ballot_sync(0xffffffffu, good);
      if (good) {
        const unsigned peers = __match_any_sync(act, label);
        if (lane == __ffs(peers) - 1) counts[label - 1] += __popc(peers);
      }
      __syncwarp();
    }
  }
  if (in_smem) {
    int32_t* g = tile_counts + warp * p;
    for (int f = lane; f < p; f += 32) g[f] = counts[f];
  }
}

// One CTA per fold: exclusive scan of its tile counts (in place) + fold total.
__global__ void tile_scan_kernel(int32_t* __restrict__ tile_counts, int64_t ntiles, int32_t p,
                                 int64_t* __restrict__ fold_counts) {
  const int32_t f = blockIdx.x;
  __shared__ int64_t warp_sums[32];
  const int64_t per = (ntiles + blockDim.x - 1) / blockDim.x;
  const int64_t t0 = threadIdx.x * per, t1 = min(ntiles, t0 + per);
  int64_t local = 0;
  for (int64_t t = t0; t < t1; ++t) local += tile_counts[t * p + f];
  // block exclusive scan of `local`
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t incl = local;
  for (int o = 1; o < 32; o <<= 1) {
    int64_t v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) warp_sums[wid] = incl;
  __syncthreads();
  if (wid == 0) {
    const int nw = blockDim.x >> 5;
    int64_t v = lane < nw ? warp_sums[lane] : 0;
    for (int o = 1; o < 32; o <<= 1) {
      int64_t u = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += u;
    }
    if (lane < nw) warp_sums[lane] = v;  // inclusive over warps
  }
  __syncthreads();
  int64_t run = (wid ? warp_sums[wid - 1] : 0) + incl - local;
  for (int64_t t = t0; t < t1; ++t) {
    const int32_t c = tile_counts[t * p + f];
    tile_counts[t * p + f] = (int32_t)run;
    run += c;
  }
  if (threadIdx.x == blockDim.x - 1) fold_counts[f] = run;
}

// Consumes tile_offsets: each warp owns its tile's row of per-fold offsets and
// advances it as it walks the tile, so ranks stay stable without atomics.
__global__ void scatter_kernel(const int32_t* __restrict__ labels, int64_t n, int32_t p, int64_t tile_rows,
                               int32_t fold_begin,
                               int32_t fold_end, int32_t* __restrict__ tile_offsets,
                               const int64_t* __restrict__ fold_zbase, int64_t win_lo, int64_t win_hi,
                               int64_t* __restrict__ src_row, int64_t zrows) {
  extern __shared__ int32_t s_run[];
  const int64_t warp = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  const int64_t row0 = warp * tile_rows;
  if (row0 >= n) return;
  const bool in_smem = p <= kSmemFolds;
  int32_t* run = tile_offsets + warp * p;
  if (in_smem) {  // the offsets are consumed here: advance a shared copy
    int32_t* sr = s_run + (threadIdx.x >> 5) * p;
    for (int f = lane; f < p; f += 32) sr[f] = run[f];
    __syncwarp();
    run = sr;
  }
  const int64_t row_end = min(n, row0 + tile_rows);
  for (int64_t base0 = row0; base0 < row_end; base0 += 32 * kBatch) {
    int32_t lab[kBatch];
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int64_t row = base0 + 32 * b + lane;
      lab[b] = row < row_end ? __ldg(labels + row) : 0;
    }
#pragma unroll
    for (int b = 0; b < kBatch; ++b) {
      const int64_t row = base0 + 32 * b + lane;
      const bool live = row < row_end;
      const int32_t label = lab[b];
      const bool own = live && label > fold_begin && label <= fold_end;
      const unsigned act = __ballot_sync(0xffffffffu, own);
      int32_t before = 0;
      unsigned peers = 0;
      if (own) {
        peers = __match_any_sync(act, label);
        before = run[label - 1];
        const int rank = __popc(peers & ((1u << lane) - 1u));
        const int64_t pos = before + rank;  // position within the fold's bucketed rows
        if (pos >= win_lo && pos < win_hi) {
          const int64_t dst = fold_zbase[label - 1 - fold_begin] + pos - win_lo;
          CVG_DCHECK(dst >= 0 && dst < zrows);
          src_row[dst] = row;
        }
      }
      __syncwarp();
      if (own && lane == __ffs(peers) - 1) run[label - 1] = before + __popc(peers);
      __syncwarp();
    }
  }
}

// Row map for compacted inputs (multi-GPU row exchange): Z row r reads compact
// row map[src_row[r]]; a bound row the map does not cover sets *bad.
__global__ void remap_rows_kernel(const int64_t* __restrict__ src_row, int64_t zrows, const int64_t* __restrict__ map,
                                  int64_t n_map, int64_t n_compact, int64_t* __restrict__ out, int* __restrict__ bad) {
  const int64_t r = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (r >= zrows) return;
  const int64_t src = src_row[r];
  int64_t v = -1;
  if (src >= 0) {
    v = src < n_map ? map[src] : -1;
    if (v < 0 || v >= n_compact) {
      atomicExch(bad, 1);
      v = -1;
    }
  }
  out[r] = v;
}

}  // namespace

void launch_remap_rows(const int64_t* src_row, int64_t zrows, const int64_t* map, int64_t n_map, int64_t n_compact,
                       int64_t* out, int* bad, cudaStream_t s) {
  if (zrows <= 0) return;
  remap_rows_kernel<<<(unsigned)((zrows + 255) / 256), 256, 0, s>>>(src_row, zrows, map, n_map, n_compact, out, bad);
}

int64_t bucket_tile_rows(int64_t n, int32_t p) {
  int64_t r = kTileRowsPerWarp;
  while (((n + r - 1) / r) * (int64_t)p > kMaxTileCounters && r < n) r *= 2;
  return r;
}

void launch_tile_histogram(const int32_t* labels, int64_t n, int32_t p, int32_t* tile_counts,
                           unsigned long long* bad, cudaStream_t s) {
  const int64_t tile_rows = bucket_tile_rows(n, p);
  const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
  const int threads = kBucketThreads;
  const int64_t blocks = (ntiles * 32 + threads - 1) / threads;
  const size_t smem = p <= kSmemFolds ? sizeof(int32_t) * (threads / 32) * p : 0;
  tile_histogram_kernel<<<(unsigned)blocks, threads, smem, s>>>(labels, n, p, tile_rows, tile_counts, bad);
}

void launch_tile_scan(int32_t* tile_counts, int64_t ntiles, int32_t p, int64_t* fold_counts, cudaStream_t s) {
  tile_scan_kernel<<<p, 256, 0, s>>>(tile_counts, ntiles, p, fold_counts);
}

void launch_scatter(const int32_t* labels, int64_t n, int32_t p, int32_t fold_begin, int32_t fold_end,
                    int32_t* tile_offsets, const int64_t* fold_zbase, int64_t win_lo, int64_t win_hi, int64_t* src_row,
                    int64_t zrows, cudaStream_t s) {
  const int64_t tile_rows = bucket_tile_rows(n, p);
  const int64_t ntiles = (n + tile_rows - 1) / tile_rows;
  const int threads = kBucketThreads;
  const int64_t blocks = (ntiles * 32 + threads - 1) / threads;
  const size_t smem = p <= kSmemFolds ? sizeof(int32_t) * (threads / 32) * p : 0;
  scatter_kernel<<<(unsigned)blocks, threads, smem, s>>>(labels, n, p, tile_rows, fold_begin, fold_end, tile_offsets, fold_zbase,
                                                      win_lo, win_hi, src_row, zrows);
}

}  // namespace cvg
