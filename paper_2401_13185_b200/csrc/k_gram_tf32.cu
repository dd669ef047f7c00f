// K1T + K2': the fp32-input fold Gram on the 5th-generation tensor cores
// (tcgen05.mma kind::tf32, TMEM accumulators, TMA-fed shared-memory ring).
//
// BASELINE.json configs[3] (fp32 inputs, fp32 accumulation on tensor cores,
// 1e-4 against the fp64 oracle).  TF32 keeps 11 significant bits, so each
// shifted value is split z = hi + lo with hi, lo TF32-exact (round to
// nearest) and every product is formed as hi·hi + hi·lo + lo·hi ("3xTF32",
// ~2^-22 relative per term) into an fp32 TMEM accumulator.  The tensor core's
// fp32 accumulation drifts linearly with chain length (measured: 3e-5 relative
// after 16384 rows, 5e-6 after 512), so the accumulator is double-buffered in
// TMEM and drained into fp64 registers every 128 rows while the MMAs continue
// in the other buffer; partials leave as fp64 and all later sums (K4) and the
// epilogue (K5) are fp64.
//
// K1T writes the bucketed, shifted, split operand transposed in 32-row blocks,
// Zt[row / 32][col][row % 32], so both MMA operands are K-major (contraction
// over rows is the contiguous axis) and every 32-row block is one contiguous
// run of kp x 128 B.  One 3-D TMA box {32 rows, 128 columns, 1 block} = 128
// rows of 128 B, 128B-swizzled: the canonical K-major SWIZZLE_128B UMMA layout
// (SBO = 1024 B).  Measured alternatives: a [col][row] transpose (multi-MB
// column pitch) halves the Gram's speed; row-major Z with MN-major operands
// (SWIZZLE_128B_BASE32B) costs the Gram 9%.
//
// K2' roles (10 warps, 1 CTA per SM, 192 KB of stages, 256 TMEM columns):
//   warp 0      TMA producer: hi/lo slabs of both column tiles per 32-row stage
//   warp 1      TMEM owner + MMA issuer (one elected thread), ping-pong accumulators
//   warps 2..9  drain every 128 rows: tcgen05.ld 128 lanes x 64 columns each, fp64 sums,
//               write the fp64 partial at the end
#include <cuda.h>

#include "cvg_internal.cuh"
#include "tc_util.cuh"

namespace cvg {
namespace {

using namespace tc;

constexpr int TT = 128;                       // tile edge (M = N = 128)
constexpr int KS = 32;                        // rows per stage = 128 B of fp32
constexpr int NST = 3;                        // pipeline stages
constexpr int kOpBytes = TT * KS * 4;         // 16 KB per operand slab
constexpr int kStageBytes = 4 * kOpBytes;     // A_hi, A_lo, B_hi, B_lo
constexpr int kSmemTf32 = NST * kStageBytes + 1024;  // + alignment slack
constexpr int kDrainSteps = 4;                // 128 rows per fp32 accumulation chunk
constexpr int kEpiWarps = 8;                  // 4 TMEM lane quarters x 2 column halves
constexpr int kThreads = 64 + 32 * kEpiWarps;


// kind::tf32, fp32 accumulate, both operands K-major, M = N = 128.
constexpr uint32_t kIdescTf32 = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(TT >> 3) << 17) |
                                ((uint32_t)(TT >> 4) << 24);

__device__ __forceinline__ void mma_tf32(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescTf32), "r"(accumulate));
}

__global__ void __launch_bounds__(kThreads, 1)
    gram_tf32_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                     const GramTask* __restrict__ segs, const int2* __restrict__ tiles, int ntiles, int64_t kp,
                     double* __restrict__ part, int nterms) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;

  const int seg = blockIdx.x / ntiles;
  const int2 tile0 = tiles[blockIdx.x - seg * ntiles];
  const int2 tile = make_int2(uniform(tile0.x), uniform(tile0.y));
  const bool diag = tile.x == tile.y;
  const GramTask task0 = segs[seg];
  const GramTask task{uniform(task0.zrow), uniform(task0.rows)};
  CVG_DCHECK(task.zrow % KS == 0 && task.rows % KS == 0 && task.rows > 0);
  CVG_DCHECK(tile.x >= 0 && tile.x <= tile.y && (int64_t)(tile.y + 1) * TT <= kp);
  const int nsteps = (int)(task.rows / KS);
  const int nchunks = (nsteps + kDrainSteps - 1) / kDrainSteps;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&acc_full[b], 1);
      mbar_init(&acc_empty[b], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(2 * TT));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_d = uniform(tmem_base);

  auto op = [&](int s, int which) { return smem + s * kStageBytes + which * kOpBytes; };  // 0 Ahi 1 Alo 2 Bhi 3 Blo

  if (warp == 0) {  // ---- TMA producer (whole warp waits; one elected lane issues)
    const uint32_t bytes = (uint32_t)kOpBytes * (nterms == 3 ? 2u : 1u) * (diag ? 1u : 2u);
    for (int it = 0; it < nsteps; ++it) {
      const int s = it % NST;
      const uint32_t ph = (uint32_t)(it / NST) & 1u;
      mbar_wait(&empty_bar[s], ph ^ 1u);
      const int blk = (int)(task.zrow / KS) + it;  // 32-row block index
      if (elect_one()) {
        mbar_expect_tx(&full_bar[s], bytes);
        tma_load_3d(op(s, 0), &map_hi, &full_bar[s], 0, tile.x * TT, blk);
        if (nterms == 3) tma_load_3d(op(s, 1), &map_lo, &full_bar[s], 0, tile.x * TT, blk);
        if (!diag) {
          tma_load_3d(op(s, 2), &map_hi, &full_bar[s], 0, tile.y * TT, blk);
          if (nterms == 3) tma_load_3d(op(s, 3), &map_lo, &full_bar[s], 0, tile.y * TT, blk);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // ---- MMA issuer (whole warp waits; one elected lane issues), accumulator b = chunk & 1
    for (int it = 0; it < nsteps; ++it) {
      const int chunk = it / kDrainSteps, b = chunk & 1;
      const bool first = it % kDrainSteps == 0;
      if (first && chunk >= 2) mbar_wait(&acc_empty[b], (uint32_t)((chunk >> 1) - 1) & 1u);  // drained
      const int s = it % NST;
      const uint32_t ph = (uint32_t)(it / NST) & 1u;
      mbar_wait(&full_bar[s], ph);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t acc = tmem_d + (uint32_t)(b * TT);
      const uint64_t a_hi = kmajor_sw128_desc(op(s, 0)), a_lo = kmajor_sw128_desc(op(s, 1));
      const uint64_t b_hi = diag ? a_hi : kmajor_sw128_desc(op(s, 2));
      const uint64_t b_lo = diag ? a_lo : kmajor_sw128_desc(op(s, 3));
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < KS / 8; ++k) {  // K = 8 tf32 = 32 B per MMA: +2 in 16-byte descriptor units
          const uint64_t dk = 2ull * k;
          mma_tf32(acc, a_hi + dk, b_hi + dk, (first && k == 0) ? 0u : 1u);
          if (nterms == 3) {
            mma_tf32(acc, a_hi + dk, b_lo + dk, 1u);
            mma_tf32(acc, a_lo + dk, b_hi + dk, 1u);
          }
        }
        mma_commit(&empty_bar[s]);  // frees the stage once these MMAs have read it
        if (it % kDrainSteps == kDrainSteps - 1 || it == nsteps - 1) mma_commit(&acc_full[b]);
      }
      __syncwarp();
    }
  } else {  // ---- drain warps: fp32 TMEM chunks -> fp64 registers -> fp64 partial
    const int q = warp & 3;            // TMEM lanes [32q, 32q + 32) (hardware: warp id mod 4)
    const int h = (warp - 2) >> 2;     // columns [64h, 64h + 64)
    double acc64[64];
#pragma unroll
    for (int j = 0; j < 64; ++j) acc64[j] = 0.0;
    for (int chunk = 0; chunk < nchunks; ++chunk) {
      const int b = chunk & 1;
      mbar_wait(&acc_full[b], (uint32_t)(chunk >> 1) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int c0 = 0; c0 < 64; c0 += 32) {
        uint32_t r[32];
        tmem_ld32(tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)(b * TT + 64 * h + c0), r);
#pragma unroll
        for (int j = 0; j < 32; ++j) acc64[c0 + j] += (double)__uint_as_float(r[j]);
      }
      asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[b]);
    }
    const int64_t row = (int64_t)tile.x * TT + 32 * q + lane;
    double* out = part + (int64_t)seg * kp * kp + row * kp + (int64_t)tile.y * TT + 64 * h;
#pragma unroll
    for (int j = 0; j < 64; j += 2) *reinterpret_cast<double2*>(out + j) = make_double2(acc64[j], acc64[j + 1]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_d), "r"(2 * TT));
  }
}


// TF32 round-to-nearest of an fp32 value (low 13 mantissa bits cleared).
__device__ __forceinline__ float tf32_rn(float v) {
  uint32_t u = __float_as_uint(v);
  if ((u & 0x7f800000u) != 0x7f800000u) u = (u + 0x1000u) & 0xffffe000u;
  return __uint_as_float(u);
}

// K1T: bucket, shift, TF32-split, transpose into Zt[block][col][32] (HBM-bound).
// One CTA per 32 bucketed rows, 128-column chunks through a padded shared-memory
// transpose; each column's 32 rows leave as 128 B, a warp covering 4 adjacent
// columns = 512 contiguous bytes.  The split is pure fp32: fl(x - c) is within 2^-24 of z and
// hi / lo are exact (an fp64 convert chain made this pass compute-bound, ~2.6 TB/s).
constexpr int kK1tCols = 128;

template <typename T>
__global__ void __launch_bounds__(256) reorder_split_t_kernel(const T* __restrict__ x, int64_t ldx,
                                                              const T* __restrict__ y, int64_t ldy, int64_t k,
                                                              int64_t m, const int64_t* __restrict__ src_row,
                                                              int64_t zrows, int64_t kp, int64_t c_begin,
                                                              int64_t c_end, const double* __restrict__ shift,
                                                              float* __restrict__ zt_hi, float* __restrict__ zt_lo,
                                                              int* __restrict__ nonfinite) {
  __shared__ float s_hi[kK1tCols][33], s_lo[kK1tCols][33];
  __shared__ int64_t s_src[32];
  const int64_t blk = blockIdx.x;
  const int t = threadIdx.x;
  const int64_t w = k + m;
  if (t < 32) s_src[t] = blk * 32 + t < zrows ? src_row[blk * 32 + t] : -1;
  CVG_DCHECK(c_begin >= 0 && c_end <= kp && c_begin % kK1tCols == 0);
  __syncthreads();
  // Lane l owns columns c0 + l + 32e (e = 0..3) of rows r_lo + 8j: every load
  // instruction is one coalesced 128-byte row segment, and the transposed
  // shared-memory writes hit 32 distinct banks (bank = l + row).  The next
  // chunk's loads are issued before this chunk's stores drain.
  const int lane = t & 31;
  const int r_lo = t >> 5;  // rows r_lo + 8j, j = 0..3
  bool bad = false;
  auto load_chunk = [&](int64_t c0, float (&v)[4][4]) {
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t src = s_src[r_lo + 8 * j];
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int64_t ce = c0 + lane + 32 * e;
        float val = 0.f;
        if (src >= 0) {
          if (ce < k)
            val = (float)__ldg(x + src * ldx + ce);
          else if (ce < w)
            val = (float)__ldg(y + src * ldy + (ce - k));
        }
        v[j][e] = val;
      }
    }
  };
  float v[4][4];
  load_chunk(c_begin, v);
  for (int64_t c0 = c_begin; c0 < c_end; c0 += kK1tCols) {
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t ce = c0 + lane + 32 * e;
      const float sh = ce < w ? (float)__ldg(shift + ce) : 0.f;
      const int kind = ce < w ? 0 : (ce == w ? 1 : 2);  // data, ones column, padding
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int rr = r_lo + 8 * j;
        float z = 0.f;
        if (s_src[rr] >= 0) {
          if (kind == 0) {
            bad |= !isfinite(v[j][e]);
            z = v[j][e] - sh;
          } else if (kind == 1) {
            z = 1.f;  // ones column: column sums ride in the Gram
          }
        }
        const float hi = tf32_rn(z);
        s_hi[lane + 32 * e][rr] = hi;
        s_lo[lane + 32 * e][rr] = tf32_rn(z - hi);
      }
    }
    __syncthreads();
    if (c0 + kK1tCols < c_end) load_chunk(c0 + kK1tCols, v);  // in flight while the stores below drain
    // write: 8 threads per column (16 B each), 32 columns per pass
#pragma unroll
    for (int cc = t >> 3; cc < kK1tCols; cc += 32) {
      const int64_t col = c0 + cc;
      const int r4 = (t & 7) * 4;
      if (col < c_end) {
        const int64_t off = (blk * kp + col) * 32 + r4;  // Zt[block][col][row % 32]
        *reinterpret_cast<float4*>(zt_hi + off) =
            make_float4(s_hi[cc][r4], s_hi[cc][r4 + 1], s_hi[cc][r4 + 2], s_hi[cc][r4 + 3]);
        *reinterpret_cast<float4*>(zt_lo + off) =
            make_float4(s_lo[cc][r4], s_lo[cc][r4 + 1], s_lo[cc][r4 + 2], s_lo[cc][r4 + 3]);
      }
    }
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && (t & 31) == 0) atomicOr(nonfinite, 1);
}

bool make_map(CUtensorMap* map, const float* base, int64_t zrows, int64_t kp, int box_cols = TT) {
  return make_blocked_map(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, base, 4, zrows, kp, box_cols);
}

}  // namespace

void launch_reorder_split_t(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                            const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                            const double* shift, float* zt_hi, float* zt_lo, int* nonfinite, cudaStream_t s) {
  dim3 grid((unsigned)((zrows + 31) / 32));
  if (dtype == 0)
    reorder_split_t_kernel<double><<<grid, 256, 0, s>>>((const double*)x, ldx, (const double*)y, ldy, k, m, src_row,
                                                        zrows, kp, c_begin, c_end, shift, zt_hi, zt_lo, nonfinite);
  else
    reorder_split_t_kernel<float><<<grid, 256, 0, s>>>((const float*)x, ldx, (const float*)y, ldy, k, m, src_row,
                                                       zrows, kp, c_begin, c_end, shift, zt_hi, zt_lo, nonfinite);
}

bool launch_gram_tf32(const float* zt_hi, const float* zt_lo, int64_t zrows, int64_t kp, const GramTask* segs,
                      int64_t nseg, const int2* tiles128, int ntiles, double* part, int nterms, cudaStream_t s) {
  CUtensorMap mh, ml;
  if (!make_map(&mh, zt_hi, zrows, kp) || !make_map(&ml, zt_lo, zrows, kp)) return false;
  cudaFuncSetAttribute(gram_tf32_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemTf32);
  const int64_t blocks = nseg * (int64_t)ntiles;
  if (blocks > 0) gram_tf32_kernel<<<(unsigned)blocks, kThreads, kSmemTf32, s>>>(mh, ml, segs, tiles128, ntiles, kp, part, nterms);
  return true;
}

}  // namespace cvg

