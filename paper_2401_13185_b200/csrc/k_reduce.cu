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
// The host flattens the trees into levels of independent ops (TreeProgram, engine.cu); an op evaluates a node
// down to kTreeFanDepth levels in registers (up to 16 inputs) -- the same additions in the same order, so four
// tree levels cost one pass (intermediate nodes are not written and re-read; configs[1]'s 100-fold tree is 2
// launches instead of 6).  Each level is one launch over (tile, op) with 16-byte loads, streaming at HBM speed.
// Only the tiles the Gram wrote are touched.
#include "cvg_internal.cuh"

namespace cvg {
namespace {

__device__ __forceinline__ double2 ld2(const double* p) { return *reinterpret_cast<const double2*>(p); }

// S(size) of the op's subtree at depth kTreeFanDepth - D, consuming inputs left to right.  The op (and so every
// branch on size) is uniform across the CTA.
template <int D>
__device__ __forceinline__ double2 tree_node(const TreeOp* __restrict__ op, int size, int& idx, int64_t off) {
  if constexpr (D == 0) {
    return ld2(op->in[idx++] + off);
  } else {
    if (size == 1) return ld2(op->in[idx++] + off);
    const int l = size / 2;
    const double2 a = tree_node<D - 1>(op, l, idx, off);
    const double2 b = tree_node<D - 1>(op, size - l, idx, off);
    return make_double2(__dadd_rn(a.x, b.x), __dadd_rn(a.y, b.y));
  }
}

__global__ void __launch_bounds__(256) tree_op_kernel(const TreeOp* __restrict__ ops, int64_t kp,
                                                      const int2* __restrict__ tiles) {
  const int2 tile = tiles[blockIdx.x];
  const TreeOp* op = ops + blockIdx.y;
  const int size = op->size;
  double* d = op->d;
  CVG_DCHECK(d != nullptr && size >= 0);
  CVG_DCHECK(tile.x >= 0 && tile.x <= tile.y && (int64_t)(tile.y + 1) * kTile <= kp);
  const int c2 = (threadIdx.x & 31) * 2;  // column pair within the tile
  // gridDim.z row slices of the tile: a level with few ops (a tree's top) still spreads over the SMs
  const int rows = kTile / (int)gridDim.z, r0 = (int)blockIdx.z * rows;
#pragma unroll 2
  for (int r = r0 + (threadIdx.x >> 5); r < r0 + rows; r += 8) {
    const int64_t off = ((int64_t)tile.x * kTile + r) * kp + (int64_t)tile.y * kTile + c2;
    int idx = 0;
    const double2 v = size > 0 ? tree_node<kTreeFanDepth>(op, size, idx, off) : make_double2(0.0, 0.0);
    *reinterpret_cast<double2*>(d + off) = v;
  }
}

// A plan whose K1 flagged a non-finite input writes NaN into its node's (0, 0) entry, so the flag
// travels with the partial through the cross-rank exchange and every rank's fold statistics
// (which test the total's diagonal) report it -- not only the rank that owns the bad rows.
__global__ void poison_if_flag_kernel(const int* __restrict__ flag, double* __restrict__ g) {
  if (*flag & 1) g[0] = __longlong_as_double(0x7ff8000000000000ll);
}

}  // namespace

void launch_poison_if_flag(const int* flag, double* g, cudaStream_t s) { poison_if_flag_kernel<<<1, 1, 0, s>>>(flag, g); }

void launch_tree_ops(const TreeOp* ops, int nops, int64_t kp, const int2* tiles, int ntiles, cudaStream_t s) {
  if (nops <= 0 || ntiles <= 0) return;
  int slices = 1;  // 8 .. 64 rows per CTA: at least ~4 CTAs per SM while the level is small
  while (slices < 8 && (int64_t)ntiles * nops * slices < 600) slices *= 2;
  for (int o = 0; o < nops; o += 65535) {  // gridDim.y <= 65535 (a level of a leave-one-out tree can hold N ops)
    dim3 grid((unsigned)ntiles, (unsigned)(nops - o < 65535 ? nops - o : 65535), (unsigned)slices);
    tree_op_kernel<<<grid, 256, 0, s>>>(ops + o, kp, tiles);
  }
}

}  // namespace cvg
