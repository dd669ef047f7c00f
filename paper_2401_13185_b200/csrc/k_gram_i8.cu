// K1Q + K2q: the fp64 fold Gram on tcgen05 kind::i8 (exact int8 slices, Ozaki-style).
//
// sm_100 has no fp64 tcgen05 kind; the DMMA path (k_gram_f64.cu) tops out at the
// FP64 tensor rate (~37 TFLOP/s).  The int8 tensor rate is ~4.5 POPS, so each
// shifted fp64 value is cut into S signed 7-bit digits and the Gram is formed from
// exact integer products:
//
//   per (segment, column) exponent e:  w = z * 2^e  with  max |w| in [32, 64)
//   w ~= d_0 + d_1 2^-7 + ... + d_{S-1} 2^-7(S-1),   |d_t| <= 64  (int8)
//   sum_rows w_a w_b ~= sum_{t+u <= S-1} 2^-7(t+u) sum_rows d_t[a] d_u[b]
//
// Every digit is exact (d_t = round-to-nearest of the exact residual, which is
// formed without error in fp64), every int8 x int8 product and its int32 TMEM sum
// is exact (|sum| <= S * 4096 * rows < 2^31 for rows <= kChunkRowsI8), and the
// drain turns the S diagonal accumulators into fp64 with one rounding per step of a
// fixed Horner chain.  The only approximation is the digit cut: each w keeps
// 7(S-1) + 6 bits below its column's segment maximum (relative error <= 2^-7(S-1)-1
// of that maximum), and the dropped products t + u >= S weigh <= S 2^-7S of
// max|w_a| max|w_b|.  S = 7 keeps the error at the level of fp64 accumulation
// itself (~1e-15 relative to the column norms).
//
// The exponent is a function of the segment's rows only (segmax_kernel), so a
// segment's partial -- and every sum built from the partials -- is bit-identical
// on 1, 2, 4 or 8 GPUs, through the host-streaming or the device-resident entry.
//
// Layout: Zq[t][row / 64][col][row % 64] int8: 64 rows of a column = 64 B, one
// SWIZZLE_64B K-major atom row.  One 4-D TMA box {64 rows, 128 | 64 columns, 1
// block, S slices} loads every slice of an operand for one 64-row stage.
//
// K2q roles (10 warps, 1 CTA per SM, one (segment, 128 x 64 output tile) per CTA):
//   warp 0      TMA producer: A (128 Gram rows) and B (64 Gram columns) slices
//   warp 1      TMEM owner + MMA issuer: S(S+1)/2 slice pairs x 2 K-steps per stage,
//               pair (t, u) into accumulator t + u (S x 64 int32 TMEM columns)
//   warps 2..9  drain once per tile: Horner over the S accumulators, exact unscale
#include "cvg_internal.cuh"
#include "tc_util.cuh"

namespace cvg {
namespace {

using namespace tc;

constexpr int QA = 128;                 // A tile: Gram rows (MMA M)
constexpr int QB = 64;                  // B tile: Gram columns (MMA N)
constexpr int QK = 64;                  // rows per stage = 64 B of int8 (one SW64 atom row)
constexpr int kQEpiWarps = 8;           // 4 TMEM lane quarters x 2 column halves
constexpr int kQThreads = 64 + 32 * kQEpiWarps;

template <int S>
struct QCfg {
  static constexpr int kA = QA * QK;                      // 8 KB per slice
  static constexpr int kB = QB * QK;                      // 4 KB per slice
  static constexpr int kStage = S * (kA + kB);
  static constexpr int kNst = (227 * 1024 - 2048) / kStage;  // 3 stages for S = 6, 2 for S = 7
  static constexpr int kSmem = kNst * kStage + 1024;
};

// kind::i8, signed A and B, int32 accumulate, both K-major, M = 128, N = 64.
constexpr uint32_t kIdescI8 =
    (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(QB >> 3) << 17) | ((uint32_t)(QA >> 4) << 24);

// CU: A-operand collector use -- 0 none, 1 fill, 2 use, 3 lastuse (consecutive MMAs of one A slice
// keep it in the collector instead of re-reading shared memory).
template <int CU>
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
#define CVG_MMA_I8(Q)                                                       \
  asm volatile(                                                             \
      "{\n"                                                                 \
      ".reg .pred p;\n"                                                     \
      "setp.ne.b32 p, %4, 0;\n"                                             \
      "tcgen05.mma.cta_group::1.kind::i8" Q " [%0], %1, %2, %3, p;\n"       \
      "}\n" ::"r"(tmem_d),                                                  \
      "l"(a), "l"(b), "r"(kIdescI8), "r"(accumulate))
  if constexpr (CU == 1)
    CVG_MMA_I8(".collector::a::fill");
  else if constexpr (CU == 2)
    CVG_MMA_I8(".collector::a::use");
  else if constexpr (CU == 3)
    CVG_MMA_I8(".collector::a::lastuse");
  else
    CVG_MMA_I8("");
#undef CVG_MMA_I8
}

#ifndef CVG_I8_COLLECTOR
#define CVG_I8_COLLECTOR 1
#endif

// pair (t, u) into accumulator t + u; A slice t held in the collector across its u run
template <int S, int T, int U>
__device__ __forceinline__ void mma_pairs(uint32_t tmem_d, uint64_t a, uint64_t b0, uint64_t b_step, bool first) {
  if constexpr (T + U < S) {
    constexpr int last = S - 1 - T;
    constexpr int cu = !CVG_I8_COLLECTOR || last == 0 ? 0 : U == 0 ? 1 : U == last ? 3 : 2;
    mma_i8<cu>(tmem_d + (uint32_t)((T + U) * QB), a, b0 + U * b_step, (first && T == 0) ? 0u : 1u);
    mma_pairs<S, T, U + 1>(tmem_d, a, b0, b_step, first);
  }
}
template <int S, int T>
__device__ __forceinline__ void mma_slices(uint32_t tmem_d, uint64_t a0, uint64_t a_step, uint64_t b0, uint64_t b_step,
                                           bool first) {
  if constexpr (T < S) {
    mma_pairs<S, T, 0>(tmem_d, a0 + T * a_step, b0, b_step, first);
    mma_slices<S, T + 1>(tmem_d, a0, a_step, b0, b_step, first);
  }
}

// K-major, 64B-swizzled operand: 8-row atoms of 512 B (SBO), version 1 (sm_100), layout 4 = SWIZZLE_64B.
__device__ __forceinline__ uint64_t kmajor_sw64_desc(const void* tile) {
  const uint64_t addr = smem_u32(tile);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | ((512ull >> 4) << 32) | (1ull << 46) | (4ull << 61);
}

__device__ __forceinline__ void tma_load_4d(void* dst, const CUtensorMap* map, uint64_t* bar, int c0, int c1, int c2,
                                            int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1, {%3, %4, %5, %6}], "
      "[%2];\n" ::"r"(smem_u32(dst)),
      "l"(map), "r"(smem_u32(bar)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

// int32 -> fp64 exactly, without the XU conversion unit: 2^52 + 2^31 + v has v in its low word.
__device__ __forceinline__ double i2d_exact(uint32_t v) {
  return __hiloint2double(0x43300000, (int)(v ^ 0x80000000u)) - 4503601774854144.0;  // 2^52 + 2^31
}

__device__ __forceinline__ double pow2(int e) {  // 2^e for e in [-1022, 1023]
  return __hiloint2double((1023 + e) << 20, 0);
}

// tiles[i] = {I, J | wmask << 16}: rows 128I .. +128 (Z columns), columns 64J .. +64; wmask bit h:
// the 64 x 64 sub-tile of rows 128I + 64h is needed downstream (an upper 64-tile of the plan).
template <int S>
__global__ void __launch_bounds__(kQThreads, 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
                   const int* __restrict__ segexp, const GramTask* __restrict__ segs, const int2* __restrict__ tiles,
                   int ntiles, int64_t kp, double* __restrict__ part) {
  using C = QCfg<S>;
  constexpr int NST = C::kNst;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], acc_full;
  __shared__ uint32_t tmem_base;

  const int seg = blockIdx.x / ntiles;
  const int2 tile0 = tiles[blockIdx.x - seg * ntiles];
  const int ti = uniform(tile0.x), tj = uniform(tile0.y & 0xffff), wmask = uniform(tile0.y >> 16);
  // B inside A's 128 columns (tj == 2ti or 2ti + 1): B is a slice of the A stage, no B load
  const int inner = tj - 2 * ti;
  const bool self = inner == 0 || inner == 1;
  const GramTask task0 = segs[seg];
  const GramTask task{uniform(task0.zrow), uniform(task0.rows)};
  CVG_DCHECK(task.zrow % QK == 0 && task.rows % QK == 0 && task.rows > 0);
  CVG_DCHECK(ti >= 0 && 2 * ti <= tj && (int64_t)tj * QB < kp);
  const int nsteps = (int)(task.rows / QK);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&acc_full, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t tmem_d = uniform(tmem_base);

  auto opA = [&](int s) { return smem + s * C::kStage; };
  auto opB = [&](int s) { return smem + s * C::kStage + S * C::kA; };

  if (warp == 0) {  // ---- TMA producer (whole warp waits; one elected lane issues)
    const uint32_t bytes = (uint32_t)(S * C::kA + (self ? 0 : S * C::kB));
    for (int it = 0; it < nsteps; ++it) {
      const int s = it % NST;
      mbar_wait(&empty_bar[s], ((uint32_t)(it / NST) & 1u) ^ 1u);
      const int blk = (int)(task.zrow / QK) + it;
      if (elect_one()) {
        mbar_expect_tx(&full_bar[s], bytes);
        tma_load_4d(opA(s), &map_a, &full_bar[s], 0, ti * QA, blk, 0);
        if (!self) tma_load_4d(opB(s), &map_b, &full_bar[s], 0, tj * QB, blk, 0);
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // ---- MMA issuer
    for (int it = 0; it < nsteps; ++it) {
      const int s = it % NST;
      mbar_wait(&full_bar[s], (uint32_t)(it / NST) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint64_t a0 = kmajor_sw64_desc(opA(s));
      const uint64_t b0 = self ? kmajor_sw64_desc(opA(s) + inner * QB * QK) : kmajor_sw64_desc(opB(s));
      const uint64_t a_step = (uint64_t)(C::kA >> 4), b_step = (uint64_t)((self ? C::kA : C::kB) >> 4);
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < QK / 32; ++k)  // K = 32 int8 = 32 B per MMA: +2 in 16-byte descriptor units
          mma_slices<S, 0>(tmem_d, a0 + 2ull * k, a_step, b0 + 2ull * k, b_step, it == 0 && k == 0);
        mma_commit(&empty_bar[s]);  // frees the stage once these MMAs have read it
        if (it == nsteps - 1) mma_commit(&acc_full);
      }
      __syncwarp();
    }
  } else {  // ---- drain: Horner over the diagonal accumulators, exact unscale, fp64 partial
    const int dw = warp - 2;
    const int q = warp & 3;  // TMEM lanes [32q, 32q + 32) (hardware: warp id mod 4)
    const int h = dw >> 2;   // columns [32h, 32h + 32) of the 64-wide tile
    const int64_t row = (int64_t)ti * QA + 32 * q + lane;  // this thread's Gram row (a Z column)
    const int64_t col0 = (int64_t)tj * QB + 32 * h;
    const bool write = row < kp && ((wmask >> (q >> 1)) & 1);
    const int* ex = segexp + (int64_t)seg * kp;
    const double urow = pow2(-ex[row < kp ? row : 0]);
    const double ucol = pow2(-ex[col0 + lane]);  // lane j holds column col0 + j's factor
    mbar_wait(&acc_full, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    double* out = part + (int64_t)seg * kp * kp + row * kp + col0;
#pragma unroll
    for (int c0 = 0; c0 < 32; c0 += 16) {
      double f[16];
      {
        uint32_t r[16];
        tmem_ld16(tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)((S - 1) * QB + 32 * h + c0), r);
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = i2d_exact(r[j]);
      }
#pragma unroll
      for (int d = S - 2; d >= 0; --d) {
        uint32_t r[16];
        tmem_ld16(tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)(d * QB + 32 * h + c0), r);
#pragma unroll
        for (int j = 0; j < 16; ++j) f[j] = fma(f[j], 0x1p-7, i2d_exact(r[j]));  // f * 2^-7 exact
      }
      if (write) {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {
          const double u0 = __shfl_sync(0xffffffffu, ucol, c0 + j), u1 = __shfl_sync(0xffffffffu, ucol, c0 + j + 1);
          *reinterpret_cast<double2*>(out + c0 + j) = make_double2(f[j] * urow * u0, f[j + 1] * urow * u1);
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; j += 2) {  // keep the shuffles converged
          __shfl_sync(0xffffffffu, ucol, c0 + j);
          __shfl_sync(0xffffffffu, ucol, c0 + j + 1);
        }
      }
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_d), "r"(512));
  }
}

// ---------------------------------------------------------------------------
// Segment column maxima: segexp[seg][c] = e with max |z| * 2^e in [32, 64) over the
// segment's rows (z = shifted value; ones column 1; padding columns / rows 0 -> e = 0).
// One CTA per (segment, 64-column chunk); warp w reads rows w, w + 16, ...; lane
// holds columns 2 lane, 2 lane + 1 (one 16-byte load per row when aligned).
constexpr int kSmThreads = 512;

template <typename T>
__global__ void __launch_bounds__(kSmThreads) segmax_kernel(const T* __restrict__ x, int64_t ldx,
                                                            const T* __restrict__ y, int64_t ldy, int64_t k,
                                                            int64_t m, const int64_t* __restrict__ src_row,
                                                            const GramTask* __restrict__ segs, int64_t kp,
                                                            int64_t c_begin, int64_t nsrc,
                                                            const double* __restrict__ shift, int* __restrict__ segexp) {
  __shared__ double s_max[kSmThreads / 32][64];
  const int seg = blockIdx.x;
  const int64_t c0 = c_begin + 64 * (int64_t)blockIdx.y;
  const GramTask task = segs[seg];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t wd = k + m;
  const int64_t ca = c0 + 2 * lane, cb = ca + 1;
  const double sa = ca < wd ? shift[ca] : 0.0, sb = cb < wd ? shift[cb] : 0.0;
  const bool vec = sizeof(T) == 8 && cb < k && (ldx % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  double ma = 0.0, mb = 0.0;
  auto val = [&](const T* xr, const T* yr, int64_t c, double sh) -> double {
    if (c < k) return __dsub_rn((double)__ldg(xr + c), sh);
    if (c < wd) return __dsub_rn((double)__ldg(yr + (c - k)), sh);
    return c == wd ? 1.0 : 0.0;
  };
  for (int64_t r = w; r < task.rows; r += kSmThreads / 32) {
    const int64_t src = src_row[task.zrow + r];
    CVG_DCHECK(src < nsrc && src >= -1);
    if (src < 0) continue;
    const T* xr = x + src * ldx;
    const T* yr = y + src * ldy;
    double va, vb;
    if (vec) {
      const double2 p = __ldg(reinterpret_cast<const double2*>(xr + ca));
      va = __dsub_rn(p.x, sa);
      vb = __dsub_rn(p.y, sb);
    } else {
      va = val(xr, yr, ca, sa);
      vb = val(xr, yr, cb, sb);
    }
    ma = fmax(ma, fabs(va));  // NaN is dropped by fmax; K1Q flags non-finite inputs
    mb = fmax(mb, fabs(vb));
  }
  s_max[w][2 * lane] = ma;
  s_max[w][2 * lane + 1] = mb;
  __syncthreads();
  if (threadIdx.x < 64) {
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < kSmThreads / 32; ++i) mx = fmax(mx, s_max[i][threadIdx.x]);
    int e = 0;
    if (mx > 0.0 && isfinite(mx)) {
      const int be = (int)((__double_as_longlong(mx) >> 52) & 0x7ff);  // 0 for subnormal maxima
      e = min(1023, 5 - (be - 1023));
    }
    segexp[(int64_t)seg * kp + c0 + threadIdx.x] = e;
  }
}

// ---------------------------------------------------------------------------
// K1Q: bucket, shift, scale by the segment exponent, cut into S int8 digits, transpose
// into Zq[t][blk][col][64].  One CTA per 64-row block, 64-column chunks.  Warp w holds
// rows 4w .. 4w + 3 (row quad w) of columns 2 lane, 2 lane + 1; a thread packs its 4 rows'
// digits of one column into one 32-bit word.  Shared tile: word (t, col, quad) at
// (t * 64 + col) * 17 + quad (stride 17: the transposed writes are at most 2-way
// conflicted); the write-out stores 4-byte words, a warp covering 2 columns x 64 B.
constexpr int kQ1Threads = 512;  // 16 warps = 16 row quads
constexpr int kQ1Stride = 17;

template <typename T, int S>
__global__ void __launch_bounds__(kQ1Threads, 2)
    reorder_q_kernel(const T* __restrict__ x, int64_t ldx, const T* __restrict__ y, int64_t ldy, int64_t k, int64_t m,
                     const int64_t* __restrict__ src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                     int64_t nsrc, const double* __restrict__ shift, const int* __restrict__ blkseg,
                     const int* __restrict__ segexp, int8_t* __restrict__ zq, int* __restrict__ nonfinite) {
  __shared__ uint32_t s_q[S * 64 * kQ1Stride];
  __shared__ int64_t s_src[QK];
  const int64_t blk = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int64_t wd = k + m;
  CVG_DCHECK(c_begin >= 0 && c_end <= kp && c_begin % 64 == 0 && zrows % QK == 0);
  if (t < QK) {
    const int64_t src = src_row[blk * QK + t];
    CVG_DCHECK(src < nsrc && src >= -1);
    s_src[t] = src;
  }
  const int seg = blkseg[blk];
  __syncthreads();
  int64_t src4[4];
  bool all_real = true;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    src4[i] = s_src[4 * w + i];
    all_real &= src4[i] >= 0;
  }
  const bool vec_ok = sizeof(T) == 8 && (ldx % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  bool bad = false;
  const int64_t zslice = zrows * kp;  // bytes per digit slice
  for (int64_t c0 = c_begin; c0 < c_end; c0 += 64) {
    const int64_t ca = c0 + 2 * lane;
    double v[4][2];
    if (all_real && vec_ok && ca + 1 < k) {
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        const double2 p = __ldg(reinterpret_cast<const double2*>(x + src4[i] * ldx + ca));
        v[i][0] = p.x;
        v[i][1] = p.y;
      }
    } else {
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int e = 0; e < 2; ++e) {
          const int64_t c = ca + e;
          double val = 0.0;
          if (src4[i] >= 0) {
            if (c < k)
              val = (double)__ldg(x + src4[i] * ldx + c);
            else if (c < wd)
              val = (double)__ldg(y + src4[i] * ldy + (c - k));
            else if (c == wd)
              val = 1.0;
          }
          v[i][e] = val;
        }
    }
#pragma unroll
    for (int e = 0; e < 2; ++e) {
      const int64_t c = ca + e;
      const double sh = c < wd ? shift[c] : 0.0;
      const double sc = pow2(segexp[(int64_t)seg * kp + c]);
      uint32_t word[S];
#pragma unroll
      for (int d = 0; d < S; ++d) word[d] = 0;
#pragma unroll
      for (int i = 0; i < 4; ++i) {
        double z = v[i][e];
        if (src4[i] >= 0 && c < wd) {
          bad |= !isfinite(z);
          z = __dsub_rn(z, sh);
        }
        // r = z * 2^e exactly; digit d = r rounded to a multiple of 2^-7d (ties to even),
        // read from the low word of r + 1.5 * 2^(52 - 7d); the residual r - digit is exact.
        double r = z * sc;
#pragma unroll
        for (int d = 0; d < S; ++d) {
          const double magic = 0x1.8p52 * (d == 0 ? 1.0 : d == 1 ? 0x1p-7 : d == 2 ? 0x1p-14 : d == 3 ? 0x1p-21
                                                       : d == 4 ? 0x1p-28 : d == 5 ? 0x1p-35 : d == 6 ? 0x1p-42 : 0x1p-49);
          const double tt = __dadd_rn(r, magic);
          const double dg = __dsub_rn(tt, magic);
          r = __dsub_rn(r, dg);
          word[d] |= ((uint32_t)__double2loint(tt) & 0xffu) << (8 * i);
        }
      }
      const int col = 2 * lane + e;
#pragma unroll
      for (int d = 0; d < S; ++d) s_q[(d * 64 + col) * kQ1Stride + w] = word[d];
    }
    __syncthreads();
    // write-out: (d, col, quad) words; consecutive threads -> consecutive quads of a column
    const int64_t ncols = c_end - c0 < 64 ? c_end - c0 : 64;
    for (int i = t; i < S * 64 * 16; i += kQ1Threads) {
      const int quad = i & 15, col = (i >> 4) & 63, d = i >> 10;
      if (col >= ncols) continue;
      const uint32_t wv = s_q[(d * 64 + col) * kQ1Stride + quad];
      *reinterpret_cast<uint32_t*>(zq + d * zslice + (blk * kp + c0 + col) * QK + 4 * quad) = wv;
    }
    __syncthreads();
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
}

template <int S>
bool launch_gram_i8_s(const int8_t* zq, const int* segexp, int64_t zrows, int64_t kp, const GramTask* segs,
                      int64_t nseg, const int2* tiles, int ntiles, double* part, cudaStream_t s) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  CUtensorMap ma, mb;
  const cuuint64_t dims[4] = {(cuuint64_t)QK, (cuuint64_t)kp, (cuuint64_t)(zrows / QK), (cuuint64_t)S};
  const cuuint64_t strides[3] = {(cuuint64_t)QK, (cuuint64_t)kp * QK, (cuuint64_t)zrows * kp};
  const cuuint32_t box_a[4] = {(cuuint32_t)QK, (cuuint32_t)QA, 1, (cuuint32_t)S};
  const cuuint32_t box_b[4] = {(cuuint32_t)QK, (cuuint32_t)QB, 1, (cuuint32_t)S};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  if (enc(&ma, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(zq), dims, strides, box_a, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  if (enc(&mb, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(zq), dims, strides, box_b, estr,
          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS)
    return false;
  cudaFuncSetAttribute(gram_i8_kernel<S>, cudaFuncAttributeMaxDynamicSharedMemorySize, QCfg<S>::kSmem);
  const int64_t blocks = nseg * (int64_t)ntiles;
  if (blocks > 0)
    gram_i8_kernel<S><<<(unsigned)blocks, kQThreads, QCfg<S>::kSmem, s>>>(ma, mb, segexp, segs, tiles, ntiles, kp,
                                                                          part);
  return true;
}

template <typename T, int S>
void launch_k1q(const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m, const int64_t* src_row,
                int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc, const double* shift,
                const int* blkseg, const int* segexp, int8_t* zq, int* nonfinite, cudaStream_t s) {
  reorder_q_kernel<T, S><<<(unsigned)(zrows / QK), kQ1Threads, 0, s>>>(
      (const T*)x, ldx, (const T*)y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, blkseg, segexp, zq,
      nonfinite);
}

}  // namespace

void launch_segmax(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                   const int64_t* src_row, const GramTask* segs, int64_t nseg, int64_t kp, int64_t c_begin,
                   int64_t c_end, int64_t nsrc, const double* shift, int* segexp, cudaStream_t s) {
  if (nseg <= 0 || c_end <= c_begin) return;
  const dim3 grid((unsigned)nseg, (unsigned)((c_end - c_begin) / 64));
  if (dtype == 0)
    segmax_kernel<double><<<grid, kSmThreads, 0, s>>>((const double*)x, ldx, (const double*)y, ldy, k, m, src_row,
                                                      segs, kp, c_begin, nsrc, shift, segexp);
  else
    segmax_kernel<float><<<grid, kSmThreads, 0, s>>>((const float*)x, ldx, (const float*)y, ldy, k, m, src_row, segs,
                                                     kp, c_begin, nsrc, shift, segexp);
}

void launch_reorder_q(int dtype, int slices, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k,
                      int64_t m, const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                      int64_t nsrc, const double* shift, const int* blkseg, const int* segexp, int8_t* zq,
                      int* nonfinite, cudaStream_t s) {
  if (zrows <= 0 || c_end <= c_begin) return;
#define CVG_K1Q(T, S) \
  launch_k1q<T, S>(x, ldx, y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, blkseg, segexp, zq, nonfinite, s)
  if (dtype == 0) {
    if (slices == 6) CVG_K1Q(double, 6);
    else CVG_K1Q(double, 7);
  } else {
    if (slices == 6) CVG_K1Q(float, 6);
    else CVG_K1Q(float, 7);
  }
#undef CVG_K1Q
}

bool launch_gram_i8(int slices, const int8_t* zq, const int* segexp, int64_t zrows, int64_t kp, const GramTask* segs,
                    int64_t nseg, const int2* tiles, int ntiles, double* part, cudaStream_t s) {
  return slices == 6 ? launch_gram_i8_s<6>(zq, segexp, zrows, kp, segs, nseg, tiles, ntiles, part, s)
                     : launch_gram_i8_s<7>(zq, segexp, zrows, kp, segs, nseg, tiles, ntiles, part, s);
}

}  // namespace cvg
