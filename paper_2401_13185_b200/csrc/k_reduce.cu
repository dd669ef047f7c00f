// K4: deterministic fixed-order sums of kp x kp Gram matrices (HBM-bound).
//
// The reference forms the whole-data XᵀX/XᵀY directly (fast.hpp:23-24); here
// they are the sum of the per-fold Grams, and a fold's Gram is the sum of its
// segments.  Every such sum uses one canonical shape — the midpoint tree
//     S(a, b) = S(a, mid) + S(mid, b),  mid = a + (b - a) / 2,  S(a, a+1) = v[a]
// — so the result never depends on scheduling, thread count or (for power-of-
// two world sizes) on how folds are split across GPUs: a rank's fold range is a
// node of this tree (cvg_fold_range) and the cross-rank combine evaluates the
// tree's top levels.  This keeps the reference's bitwise thread-count
// invariance (threading.hpp:8-10, test_fast.cpp:217-229).  No float atomics.
//
// Only the tiles the Gram wrote are touched.  One CTA per (tile, group).
#include "cvg_internal.cuh"

namespace cvg {
namespace {

__device__ double tree_sum(const double* const* __restrict__ src, int a, int b, int64_t off) {
  if (b <= a) return 0.0;
  if (b - a == 1) return src[a][off];
  const int mid = a + (b - a) / 2;
  return __dadd_rn(tree_sum(src, a, mid, off), tree_sum(src, mid, b, off));
}

__global__ void __launch_bounds__(256) tree_sum_kernel(const double* const* __restrict__ srcs,
                                                       const int32_t* __restrict__ src_begin,
                                                       double* const* __restrict__ dsts, int64_t kp,
                                                       const int2* __restrict__ tiles) {
  const int2 tile = tiles[blockIdx.x];
  const int grp = blockIdx.y;
  const int a = src_begin[grp], b = src_begin[grp + 1];
  double* dst = dsts[grp];
  const int c = threadIdx.x & 63;
  for (int r = threadIdx.x >> 6; r < kTile; r += 4) {
    const int64_t off = ((int64_t)tile.x * kTile + r) * kp + (int64_t)tile.y * kTile + c;
    dst[off] = tree_sum(srcs, a, b, off);
  }
}

}  // namespace

void launch_tree_sum(const double* const* srcs, const int32_t* src_begin, int ngroups, double* const* dsts,
                     int64_t kp, const int2* tiles, int ntiles, cudaStream_t s) {
  if (ngroups <= 0 || ntiles <= 0) return;
  dim3 grid((unsigned)ntiles, (unsigned)ngroups);
  tree_sum_kernel<<<grid, 256, 0, s>>>(srcs, src_begin, dsts, kp, tiles);
}

}  // namespace cvg
