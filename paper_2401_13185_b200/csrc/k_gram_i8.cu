// K1Q + K2q: the fp64 fold Gram on tcgen05 kind::i8 (exact int8 slices, Ozaki-style).
//
// sm_100 has no fp64 tcgen05 kind; the DMMA path (k_gram_f64.cu) tops out at the
// FP64 tensor rate (~37 TFLOP/s).  The int8 tensor rate is ~4.5 POPS, so each
// shifted fp64 value is cut into S signed base-256 digits and the Gram is formed
// from exact integer products:
//
//   per (segment, column) exponent e:  w = z * 2^e  with  |w| < 127
//   w ~= d_0 + d_1 2^-8 + ... + d_{S-1} 2^-8(S-1),   d_t in [-128, 127]  (int8)
//   sum_rows w_a w_b ~= sum_{t+u <= S-1} 2^-8(t+u) sum_rows d_t[a] d_u[b]
//
// The digits are exact (the bytes of V = round(w 2^8(S-1)) + offset), every int8 x
// int8 product and its int32 TMEM sum is exact (|sum| <= S * 2^14 * rows < 2^31 for
// rows <= kChunkRowsI8), and the drain turns the S diagonal accumulators into fp64
// with one rounding per step of a fixed Horner chain.  The only approximation is the
// digit cut: each w keeps 8(S-1) + 6..7 bits below its column's segment maximum, and
// the dropped products t + u >= S weigh <= S 2^-8S of max|w_a| max|w_b|.  S = 6 (48
// bits, 21 slice pairs) keeps the error at the level of fp64 accumulation itself
// (~1e-14 relative to the column norms).
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
//               pair (t, u) into accumulator t + u (S x 64 int32 TMEM columns); the pairs of
//               one A slice with adjacent B slices are one MMA of N = 64 .. 256
//   warps 2..9  drain once per tile: Horner over the S accumulators, exact unscale
#include <atomic>
#include <type_traits>
#include <cstdlib>

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

// KS rows per pipeline stage: 64 (one SW64 atom row of a 64-row block) or 32 (half of it, SW32):
// S = 7 fits 2 stages of 64 rows (84 KB each) or 5 of 32 rows (42 KB).
template <int S, int KS, int kMaxSt = 8>
struct QCfg {
  static constexpr int kA = QA * KS;                      // per slice
  static constexpr int kB = QB * KS;
  static constexpr int kStage = S * (kA + kB);
  static constexpr int kNst = (227 * 1024 - 2048) / kStage < kMaxSt ? (227 * 1024 - 2048) / kStage : kMaxSt;
  static constexpr int kSmem = kNst * kStage + 1024;
};

// kind::i8, signed A and B, int32 accumulate, both K-major, M = 128, N = 64 * NS.
template <int NS>
constexpr uint32_t idesc_i8() {
  return (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(NS * QB >> 3) << 17) | ((uint32_t)(QA >> 4) << 24);
}

// CU: A-operand collector use -- 0 none, 1 fill, 2 use, 3 lastuse (consecutive MMAs of one A slice
// keep it in the collector instead of re-reading shared memory).
template <int CU, int NS>
__device__ __forceinline__ void mma_i8(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
#define CVG_MMA_I8(Q)                                                       \
  asm volatile(                                                             \
      "{\n"                                                                 \
      ".reg .pred p;\n"                                                     \
      "setp.ne.b32 p, %4, 0;\n"                                             \
      "tcgen05.mma.cta_group::1.kind::i8" Q " [%0], %1, %2, %3, p;\n"       \
      "}\n" ::"r"(tmem_d),                                                  \
      "l"(a), "l"(b), "r"(idesc_i8<NS>()), "r"(accumulate))
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

// Pairs (t, u), u = 0 .. S-1-t, go into accumulators t + u, which sit side by side in TMEM
// (accumulator d = columns 64d .. 64d + 63), and the B slices u sit side by side in shared
// memory (one 64-column K-major tile each, SBO-uniform): so NS consecutive pairs are ONE
// MMA with N = 64 NS (NS <= 4, N <= 256) -- 10 MMAs per K-step instead of 28 for S = 7.
// A slice t stays in the collector across its run.
template <int S, int T, int U0, int LEN = S - T>
__device__ __forceinline__ void mma_runs(uint32_t tmem_d, uint64_t a, uint64_t b0, uint64_t b_step, bool first) {
  if constexpr (U0 < LEN) {
    constexpr int NS = (LEN - U0) < 4 ? (LEN - U0) : 4;
    constexpr bool only = U0 == 0 && NS == LEN;  // the whole run is one MMA
    constexpr int cu = !CVG_I8_COLLECTOR || only ? 0 : U0 == 0 ? 1 : U0 + NS == LEN ? 3 : 2;
    mma_i8<cu, NS>(tmem_d + (uint32_t)((T + U0) * QB), a, b0 + U0 * b_step, (first && T == 0) ? 0u : 1u);
    mma_runs<S, T, U0 + NS, LEN>(tmem_d, a, b0, b_step, first);
  }
}
// Accumulators: S diagonals t + u <= S-1, plus (S even) the square pair (S/2, S/2) of diagonal S: the
// dropped pairs t + u >= S are zero-mean products of independent digits except these squares, so
// keeping the first one removes the truncation's bias on the Gram diagonal (the next, diagonal S+2,
// weighs 2^-16 less).
template <int S>
constexpr int kNAcc = S + (S % 2 == 0 ? 1 : 0);

template <int S, int T>
__device__ __forceinline__ void mma_slices(uint32_t tmem_d, uint64_t a0, uint64_t a_step, uint64_t b0, uint64_t b_step,
                                           bool first) {
  if constexpr (T < S) {
    if constexpr (S % 2 == 0 && T == S / 2) {
      // the square pair (S/2, S/2) into accumulator S, adjacent to the run's last one: after the first
      // K-step (which must start accumulator S from zero on its own) it extends the run by one slice
      if (first) {
        mma_runs<S, T, 0>(tmem_d, a0 + T * a_step, b0, b_step, first);
        mma_i8<0, 1>(tmem_d + (uint32_t)(S * QB), a0 + T * a_step, b0 + T * b_step, 0u);
      } else {
        mma_runs<S, T, 0, S - T + 1>(tmem_d, a0 + T * a_step, b0, b_step, first);
      }
    } else {
      mma_runs<S, T, 0>(tmem_d, a0 + T * a_step, b0, b_step, first);
    }
    mma_slices<S, T + 1>(tmem_d, a0, a_step, b0, b_step, first);
  }
}

// K-major swizzled operand with KS-byte rows: 8-row atoms of 8 KS bytes (SBO), version 1 (sm_100);
// layout 4 = SWIZZLE_64B (KS = 64), 6 = SWIZZLE_32B (KS = 32).
template <int KS>
__device__ __forceinline__ uint64_t kmajor_sw_desc(const void* tile) {
  const uint64_t addr = smem_u32(tile);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(8 * KS >> 4) << 32) | (1ull << 46) |
         ((KS == 64 ? 4ull : 6ull) << 61);
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

// 256-bit global store (sm_100): four doubles, 32-byte aligned
__device__ __forceinline__ void stg_v4_f64(double* p, double a, double b, double c, double d) {
  asm volatile("st.global.v4.f64 [%0], {%1, %2, %3, %4};\n" ::"l"(p), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

__device__ __forceinline__ double pow2(int e) {  // 2^e for e in [-1022, 1023]
  return __hiloint2double((1023 + e) << 20, 0);
}

// The segment exponent of a column whose max |z| is mx: max |z| 2^e in [63.5, 127), so every
// value is representable by the offset digits (|w| < 127 < 128 - 128/255); with `headroom` (mx is
// the max over a row sample) in [31.75, 63.5), so values up to 2x the sampled max still fit
// (larger ones are caught by K1Q and the segment is redone from its exact max).  e = 0 for an
// all-zero (or non-finite) column.  ilogb / scalbn keep subnormal maxima exact: e spans
// [-1018, 1080], so the cut scales in two power-of-two steps (cut_scales) and the drain
// unscales through unscale() -- no 2^e ever has to be a normal double.
__device__ __forceinline__ int seg_exponent(double mx, int headroom) {
  const uint64_t bits = (uint64_t)__double_as_longlong(mx);
  const int ex = (int)(bits >> 52);  // sign + biased exponent: 1 .. 2046 for a positive normal max
  if (ex >= 1 && ex <= 2046) {
    // normal: ilogb = ex - 1023 and scalbn(mx, e) = 1.f * 2^(5 | 6), which reaches 63.5 (127) iff
    // 1.f >= 1 + 63/64, i.e. the top 6 fraction bits are all ones -- no libm calls on the hot path
    return (headroom ? 5 : 6) - (ex - 1023) - (int)(((bits >> 46) & 63) == 63);
  }
  if (!(mx > 0.0) || !isfinite(mx)) return 0;
  int e = (headroom ? 5 : 6) - ilogb(mx);  // subnormal max
  if (scalbn(mx, e) >= (headroom ? 63.5 : 127.0)) --e;
  return e;
}

// z 2^(e + 8(S-1)) as (z * pre) * sc: pre = 2^a (1 unless the exponent exceeds 1000), sc = 2^(e + 8(S-1) - a);
// z * pre is exact (a power-of-two step up that stays below 2^-900), so the fma's single rounding is
// the only one -- the same bits as one fma by 2^(e + 8(S-1)) wherever that factor is a normal double.
struct CutScale {
  double pre, sc;
};
__device__ __forceinline__ CutScale cut_scales(int e_digits) {
  const int a = e_digits > 1000 ? e_digits - 1000 : 0;
  return CutScale{pow2(a), pow2(e_digits - a)};
}

// f 2^-E, E = e_row + e_col in [-2036, 2160]: one exact multiply by a normal power of two when
// |E| <= 1022 (every realistic column pair), else scalbn (correct rounding into subnormals / to inf).
__device__ __forceinline__ double unscale(double f, int E) {
  return (E <= 1022 && E >= -1022) ? f * pow2(-E) : scalbn(f, -E);
}

// Items: tiles[i] = {a0 | a1 << 16, c | mode0 << 16 | mode1 << 18}.  B = the 64 Gram columns of block c; A = two
// 64-row halves, half h = Z columns of block a_h (64 a_h .. +64); mode 1: the half's 64 x 64 result is the upper
// tile (a_h, c) (a_h <= c), stored as is; mode 2: a_h > c, it is the transpose of the upper tile (c, a_h), stored
// transposed; mode 0: unused half (not loaded, not stored).  An aligned item (a1 = a0 + 1, a0 even, both used)
// loads A with one TMA box of 128 columns; other items load each used half slice by slice.  The host cover
// (engine.cu i8_items) produces every needed upper tile exactly once with at most one unused half, where 128-row
// aligned tiles left a 64 x 64 sub-tile below the diagonal on every diagonal tile (c1: 18 items instead of 20).
//
// Persistent: one CTA per SM walks the (segment, tile) items round-robin (item = blockIdx.x + i gridDim.x,
// segment-major, so the CTAs running at once share a segment's digits in L2).  The TMA ring runs on across
// items -- the next item's first stages load while this one drains -- and TMEM is allocated once; the MMA warp
// starts an item once the drain warps have read the previous item's accumulators (tmem_empty).  A launch per
// item paid its TMEM allocation, barrier setup and pipeline fill every time: ~9 us per item, which dominated
// short folds (the paper's P = 1000 at N = 1e5: 20,000 items of 2 K-steps).
//
// LEAN (the Gram that runs beside the direct cut): the drain reads its accumulators 8 columns at a time and the
// kernel is held to 96 registers (launch bounds of two CTAs per SM; shared memory admits one), so a 256-thread
// cut CTA fits on the same SM; the TMA producer acquires seg_ready[seg] (one count per cut 64-row block) before
// an item's first stage.  A producer that waits longer than kReadyTimeoutNs sets *abort_flag and stops
// waiting (so does every other producer): the launch then finishes on whatever digits are there and the host
// redoes the pass serially -- the cut does not depend on the Gram, so a missing co-residency cannot hang.
__device__ __forceinline__ unsigned ld_acquire_u32(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];\n" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long global_ns() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;\n" : "=l"(t));
  return t;
}
constexpr unsigned long long kReadyTimeoutNs = 1000000000ull;

template <int S, int KS, int kMaxSt = 8, bool LEAN = false>
__global__ void __launch_bounds__(kQThreads, LEAN ? 2 : 1)
    gram_i8_kernel(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_a64,
                   const __grid_constant__ CUtensorMap map_b,
                   const unsigned long long* __restrict__ segmax, const GramTask* __restrict__ segs,
                   const int2* __restrict__ tiles, int ntiles, int64_t nitems, int64_t seg_base, int64_t kp,
                   double* __restrict__ part, int headroom, const unsigned* __restrict__ seg_ready,
                   int* __restrict__ abort_flag, int64_t split_from, int split_f, int32_t* __restrict__ split_ws,
                   unsigned* __restrict__ split_cnt) {
  using C = QCfg<S, KS, kMaxSt>;
  constexpr int NST = C::kNst;
  constexpr int kPer = QK / KS;  // stages per 64-row block
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], acc_full, tmem_empty;
  __shared__ uint32_t tmem_base;
  __shared__ bool s_last;  // tail split: this CTA's part arrived last
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t G = gridDim.x;

  if (threadIdx.x == 0) {
    for (int s = 0; s < NST; ++s) {
      mbar_init(&full_bar[s], 1);
      mbar_init(&empty_bar[s], 1);
    }
    mbar_init(&acc_full, 1);
    mbar_init(&tmem_empty, kQEpiWarps);
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
  // item -> (segment, A halves a0 / a1, B block c, half modes)
  // Tail split (split_f > 1): the items past the last full round of the grid (virtual indices >= split_from) are
  // each cut into split_f row parts, so the partial last round fills the SMs with short parts instead of running
  // a few whole items.  A part accumulates its rows' exact int32 sums and dumps them; the part that arrives last
  // adds all dumps -- integer adds, so the order does not matter and the total is the un-split item's own
  // accumulator, bit for bit -- and drains as usual.  Nobody waits for anybody.
  int tail = -1, rpart = 0;  // tail item index (else -1) and row part of the item decoded last
  int st0 = 0, st1 = 0;      // its stage range
  auto item = [&](int64_t it, int& seg, int& a0, int& a1, int& c, int& modes, GramTask& task) {
    tail = -1;
    rpart = 0;
    if (split_f > 1 && it >= split_from) {
      const int64_t v = it - split_from;
      tail = (int)(v / split_f);
      rpart = (int)(v - (int64_t)tail * split_f);
      it = split_from + tail;
    }
    const int64_t sl = it / ntiles;  // segment within this launch's range [seg_base, seg_base + nitems / ntiles)
    seg = (int)(seg_base + sl);
    const int2 tile0 = tiles[it - sl * ntiles];
    a0 = uniform(tile0.x & 0xffff);
    a1 = uniform(tile0.x >> 16);
    c = uniform(tile0.y & 0xffff);
    modes = uniform(tile0.y >> 16);
    const GramTask task0 = segs[seg];
    task = GramTask{uniform(task0.zrow), uniform(task0.rows)};
    CVG_DCHECK(task.zrow % QK == 0 && task.rows % QK == 0 && task.rows > 0);
    CVG_DCHECK((int64_t)c * QB < kp && (int64_t)a0 * QB < kp && (int64_t)a1 * QB < kp && (modes & 3) != 0);
    const int nst = (int)(task.rows / KS);
    st0 = tail < 0 ? 0 : (int)((int64_t)nst * rpart / split_f);
    st1 = tail < 0 ? nst : (int)((int64_t)nst * (rpart + 1) / split_f);
    CVG_DCHECK(st1 > st0);
  };

  if (warp == 0) {  // ---- TMA producer (whole warp waits; one elected lane issues)
    int64_t g = 0;  // stage-ring position, continuous across items
    for (int64_t it = blockIdx.x; it < nitems; it += G) {
      int seg, a0, a1, c, modes;
      GramTask task;
      item(it, seg, a0, a1, c, modes, task);
      const bool use0 = (modes & 3) != 0, use1 = ((modes >> 2) & 3) != 0;
      const bool aligned = use0 && use1 && a1 == a0 + 1 && (a0 & 1) == 0;
      const uint32_t bytes = (uint32_t)(S * ((use0 + use1) * (C::kA / 2) + C::kB));
      if (seg_ready) {  // the concurrent cut has published every 64-row block of this segment
        const unsigned need = (unsigned)(task.rows / QK);
        if (ld_acquire_u32(seg_ready + seg) < need) {
          const unsigned long long t0 = global_ns();
          while (ld_acquire_u32(seg_ready + seg) < need) {
            __nanosleep(256);
            if (*reinterpret_cast<volatile int*>(abort_flag)) break;
            if (global_ns() - t0 > kReadyTimeoutNs) {
              atomicExch(abort_flag, 1);
              break;
            }
          }
        }
        asm volatile("fence.proxy.async.global;\n" ::: "memory");  // generic-proxy digits -> TMA reads
        __syncwarp();
      }
      for (int st = st0; st < st1; ++st, ++g) {
        const int s = (int)(g % NST);
        mbar_wait(&empty_bar[s], ((uint32_t)(g / NST) & 1u) ^ 1u);
        const int blk = (int)(task.zrow / QK) + st / kPer, r0 = (st % kPer) * KS;
        if (elect_one()) {
          mbar_expect_tx(&full_bar[s], bytes);
          if (aligned) {
            tma_load_4d(opA(s), &map_a, &full_bar[s], r0, a0 * QB, blk, 0);
          } else {
#pragma unroll
            for (int t = 0; t < S; ++t) {
              if (use0) tma_load_4d(opA(s) + t * C::kA, &map_a64, &full_bar[s], r0, a0 * QB, blk, t);
              if (use1) tma_load_4d(opA(s) + t * C::kA + C::kA / 2, &map_a64, &full_bar[s], r0, a1 * QB, blk, t);
            }
          }
          tma_load_4d(opB(s), &map_b, &full_bar[s], r0, c * QB, blk, 0);
        }
        __syncwarp();
      }
    }
  } else if (warp == 1) {  // ---- MMA issuer
    int64_t g = 0;
    int t = 0;  // items of this CTA
    for (int64_t it = blockIdx.x; it < nitems; it += G, ++t) {
      int seg, a0, a1, c, modes;
      GramTask task;
      item(it, seg, a0, a1, c, modes, task);
      if (t > 0) {  // the drain warps have read the previous item's accumulators
        mbar_wait(&tmem_empty, (uint32_t)(t - 1) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      }
      for (int st = st0; st < st1; ++st, ++g) {
        const int s = (int)(g % NST);
        mbar_wait(&full_bar[s], (uint32_t)(g / NST) & 1u);
        asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
        const uint64_t a0 = kmajor_sw_desc<KS>(opA(s));
        const uint64_t b0 = kmajor_sw_desc<KS>(opB(s));
        const uint64_t a_step = (uint64_t)(C::kA >> 4), b_step = (uint64_t)(C::kB >> 4);
        if (elect_one()) {
#pragma unroll
          for (int k = 0; k < KS / 32; ++k)  // K = 32 int8 = 32 B per MMA: +2 in 16-byte descriptor units
            mma_slices<S, 0>(tmem_d, a0 + 2ull * k, a_step, b0 + 2ull * k, b_step, st == st0 && k == 0);
          mma_commit(&empty_bar[s]);  // frees the stage once these MMAs have read it
          if (st == st1 - 1) mma_commit(&acc_full);
        }
        __syncwarp();
      }
    }
  } else {  // ---- drain: Horner over the diagonal accumulators, exact unscale, fp64 partial
    const int dw = warp - 2;
    const int q = warp & 3;  // TMEM lanes [32q, 32q + 32) (hardware: warp id mod 4)
    const int h = dw >> 2;   // columns [32h, 32h + 32) of the 64-wide tile
    int t = 0;
    for (int64_t it = blockIdx.x; it < nitems; it += G, ++t) {
      int seg, a0, a1, c, modes;
      GramTask task;
      item(it, seg, a0, a1, c, modes, task);
      const int half = q >> 1;  // TMEM lanes 0-63: A half 0, 64-127: half 1
      const int mode = (modes >> (2 * half)) & 3;
      const int64_t row = (int64_t)(half ? a1 : a0) * QB + 32 * (q & 1) + lane;  // this thread's Gram row (a Z column)
      const int64_t col0 = (int64_t)c * QB + 32 * h;
      const unsigned long long* mx = segmax + (int64_t)seg * kp;
      const int erow = seg_exponent(__longlong_as_double((long long)mx[row]), headroom);
      const int ecol = seg_exponent(__longlong_as_double((long long)mx[col0 + lane]), headroom);  // lane j: column col0 + j
      mbar_wait(&acc_full, (uint32_t)t & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      double* out = part + (int64_t)seg * kp * kp + row * kp + col0;
      double* out_t = part + (int64_t)seg * kp * kp + col0 * kp + row;  // mode 2: element (row, col0 + j) at (col0 + j, row)
      constexpr int DB = LEAN ? 8 : 16;  // accumulator columns per batch
      constexpr int NACC = kNAcc<S>;
      // TMEM -> registers: all accumulators' DB columns in one batch of loads (one wait: the MMAs restart sooner)
      auto load_acc = [&](uint32_t (&r)[NACC][DB], int c0) {
#pragma unroll
        for (int d = 0; d < NACC; ++d) {
          const uint32_t ta = tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)(d * QB + 32 * h + c0);
          if constexpr (LEAN) tmem_ld8_nowait(ta, r[d]);
          else tmem_ld16_nowait(ta, r[d]);
        }
        tmem_ld_wait();
      };
      auto release_tmem = [&]() {  // every accumulator column of this thread has been read: the MMA warp may go on
        asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) mbar_arrive(&tmem_empty);
      };
      // exact Horner over the diagonal accumulators, unscale, store this thread's DB entries of its row
      auto emit = [&](uint32_t (&r)[NACC][DB], int c0) {
        double f[DB];
#pragma unroll
        for (int j = 0; j < DB; ++j) f[j] = i2d_exact(r[NACC - 1][j]);
#pragma unroll
        for (int d = NACC - 2; d >= 0; --d)
#pragma unroll
          for (int j = 0; j < DB; ++j) f[j] = fma(f[j], 0x1p-8, i2d_exact(r[d][j]));  // f * 2^-8 exact
        if (mode == 1) {
#pragma unroll
          for (int j = 0; j < DB; j += 4) {  // 32-byte stores: a lane's row segment is whole sectors
            const int e0 = __shfl_sync(0xffffffffu, ecol, c0 + j), e1 = __shfl_sync(0xffffffffu, ecol, c0 + j + 1);
            const int e2 = __shfl_sync(0xffffffffu, ecol, c0 + j + 2), e3 = __shfl_sync(0xffffffffu, ecol, c0 + j + 3);
            stg_v4_f64(out + c0 + j, unscale(f[j], erow + e0), unscale(f[j + 1], erow + e1), unscale(f[j + 2], erow + e2),
                       unscale(f[j + 3], erow + e3));
          }
        } else if (mode == 2) {
#pragma unroll
          for (int j = 0; j < DB; j += 2) {  // transposed: the warp's 32 rows are 256 contiguous bytes of one row
            const int e0 = __shfl_sync(0xffffffffu, ecol, c0 + j), e1 = __shfl_sync(0xffffffffu, ecol, c0 + j + 1);
            out_t[(int64_t)(c0 + j) * kp] = unscale(f[j], erow + e0);
            out_t[(int64_t)(c0 + j + 1) * kp] = unscale(f[j + 1], erow + e1);
          }
        } else {
#pragma unroll
          for (int j = 0; j < DB; j += 2) {  // keep the shuffles converged
            __shfl_sync(0xffffffffu, ecol, c0 + j);
            __shfl_sync(0xffffffffu, ecol, c0 + j + 1);
          }
        }
      };
      if (tail < 0) {
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += DB) {
          uint32_t r[NACC][DB];
          load_acc(r, c0);
          if (c0 == 32 - DB) release_tmem();
          emit(r, c0);
        }
      } else {
        // a row part of a tail item: dump the exact int32 sums ([accumulator][column][tile row], coalesced over
        // the lanes' rows); the part that arrives last adds every part's dump and drains
        constexpr int64_t kDump = (int64_t)NACC * QB * QA;
        int32_t* ws = split_ws + (int64_t)tail * split_f * kDump;
        const int trow = 32 * q + lane;
#pragma unroll
        for (int c0 = 0; c0 < 32; c0 += DB) {
          uint32_t r[NACC][DB];
          load_acc(r, c0);
          if (c0 == 32 - DB) release_tmem();
          int32_t* my = ws + (int64_t)rpart * kDump + (int64_t)(32 * h + c0) * QA + trow;
#pragma unroll
          for (int d = 0; d < NACC; ++d)
#pragma unroll
            for (int j = 0; j < DB; ++j) my[((int64_t)d * QB + j) * QA] = (int32_t)r[d][j];
        }
        __threadfence();
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kQEpiWarps) : "memory");  // the drain warps' dumps are out
        if (threadIdx.x == 64) {
          const unsigned prev = atomicAdd(split_cnt + tail, 1u);
          s_last = prev + 1u == (unsigned)split_f;
          if (s_last) split_cnt[tail] = 0u;  // ready for the next launch
        }
        asm volatile("bar.sync 1, %0;\n" ::"n"(32 * kQEpiWarps) : "memory");
        if (s_last) {
          __threadfence();
#pragma unroll
          for (int c0 = 0; c0 < 32; c0 += DB) {
            uint32_t r[NACC][DB];
#pragma unroll
            for (int d = 0; d < NACC; ++d)
#pragma unroll
              for (int j = 0; j < DB; ++j) r[d][j] = 0u;
            for (int pf = 0; pf < split_f; ++pf) {
              const int32_t* src = ws + (int64_t)pf * kDump + (int64_t)(32 * h + c0) * QA + trow;
#pragma unroll
              for (int d = 0; d < NACC; ++d)
#pragma unroll
                for (int j = 0; j < DB; ++j) r[d][j] += (uint32_t)__ldcg(src + ((int64_t)d * QB + j) * QA);
            }
            emit(r, c0);
          }
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
// Segment column maxima: segmax[seg][c] = max |z| over the segment's rows, as the bits of
// a non-negative double (so atomicMax on the bits is an exact, order-free max); z = shifted
// value, ones column 1, padding columns / rows 0.  Grid (segment, 64-column chunk, row
// slice of `slice` rows: 128 .. 1024, so small problems still spread over the SMs); warp w
// reads rows w, w + 8, ... four at a time (16-byte loads of columns 2 lane, 2 lane + 1); one
// atomicMax per column per CTA.  The buffer is zeroed first.
constexpr int kSmThreads = 256;

template <typename T>
__global__ void __launch_bounds__(kSmThreads) segmax_kernel(const T* __restrict__ x, int64_t ldx,
                                                            const T* __restrict__ y, int64_t ldy, int64_t k,
                                                            int64_t m, const int64_t* __restrict__ src_row,
                                                            const GramTask* __restrict__ segs, int64_t kp,
                                                            int64_t c_begin, int64_t nsrc,
                                                            const double* __restrict__ shift, int64_t slice,
                                                            int stride, const int* __restrict__ only,
                                                            unsigned long long* __restrict__ segmax) {
  constexpr int NW = kSmThreads / 32;
  __shared__ double s_max[NW][64];
  const int seg = blockIdx.x;
  if (only && !only[seg]) return;  // exact pass: only the segments whose sample fell short
  const int64_t c0 = c_begin + 64 * (int64_t)blockIdx.y;
  const GramTask task = segs[seg];
  // sampled row indices j (rows j * stride of the segment), sliced over blockIdx.z; a segment keeps at
  // least 512 sampled rows (short segments are scanned whole)
  stride = (int)max((int64_t)1, min((int64_t)stride, task.rows / 512));
  const int64_t nj = (task.rows + stride - 1) / stride;
  const int64_t r_begin = (int64_t)blockIdx.z * slice;
  const int64_t r_end = min(nj, r_begin + slice);
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int64_t wd = k + m;
  const int64_t ca = c0 + 2 * lane, cb = ca + 1;
  const double sa = ca < wd ? shift[ca] : 0.0, sb = cb < wd ? shift[cb] : 0.0;
  const bool vec = sizeof(T) == 8 && cb < k && (ldx % 2) == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  // a Y column pair (k even): one 16-byte load from y
  const bool yvec = sizeof(T) == 8 && ca >= k && cb < wd && (k % 2) == 0 && (ldy % 2) == 0 &&
                    (reinterpret_cast<uintptr_t>(y) & 15) == 0;
  const T* vbase = vec ? x + ca : yvec ? y + (ca - k) : nullptr;
  const int64_t vld = vec ? ldx : ldy;
  double ma = 0.0, mb = 0.0;
  auto val = [&](int64_t src, int64_t c, double sh) -> double {
    if (src < 0) return 0.0;
    if (c < k) return __dsub_rn((double)__ldg(x + src * ldx + c), sh);
    if (c < wd) return __dsub_rn((double)__ldg(y + src * ldy + (c - k)), sh);
    return c == wd ? 1.0 : 0.0;
  };
  for (int64_t r0 = r_begin + w; r0 < r_end; r0 += 4 * NW) {
    int64_t src[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t r = r0 + u * NW;
      src[u] = r < r_end ? src_row[task.zrow + r * stride] : -1;
      CVG_DCHECK(src[u] < nsrc && src[u] >= -1);
    }
    if (vbase) {
      double2 p[4];
#pragma unroll
      for (int u = 0; u < 4; ++u)
        p[u] = src[u] >= 0 ? __ldg(reinterpret_cast<const double2*>(vbase + src[u] * vld)) : make_double2(sa, sb);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ma = fmax(ma, fabs(__dsub_rn(p[u].x, sa)));  // NaN is dropped by fmax; K1Q flags non-finite inputs
        mb = fmax(mb, fabs(__dsub_rn(p[u].y, sb)));
      }
    } else {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        ma = fmax(ma, fabs(val(src[u], ca, sa)));
        mb = fmax(mb, fabs(val(src[u], cb, sb)));
      }
    }
  }
  s_max[w][2 * lane] = ma;
  s_max[w][2 * lane + 1] = mb;
  __syncthreads();
  if (threadIdx.x < 64) {
    double mx = 0.0;
#pragma unroll
    for (int i = 0; i < NW; ++i) mx = fmax(mx, s_max[i][threadIdx.x]);
    if (mx > 0.0) atomicMax(segmax + (int64_t)seg * kp + c0 + threadIdx.x, (unsigned long long)__double_as_longlong(mx));
  }
}

// ---------------------------------------------------------------------------
// K1Q: bucket, shift, scale by the segment exponent, cut into S int8 digits, write
// Zq[t][blk][col][64].  A CTA item is one 64-row block x 64 columns.  Warp w owns columns 8w .. 8w + 7 and
// runs on its own: it assembles its S x 8 columns x 64 rows of digits (S x 512 B) in its own shared-memory
// region in the operand's SWIZZLE_64B layout and sends them with its own TMA tensor store (8 contiguous 64 B
// lines per slice; double-buffered so the next chunk's loads and cuts overlap the store).  The only CTA
// barrier is one per 64-row block, publishing the row pointers of the block two ahead (triple-buffered), so
// the warps drift past one another's load latencies.  Lane (j, qq) = (lane >> 2, lane & 3) holds column 8w + j
// of the row quads qq, qq + 4, qq + 8, qq + 12 (16 rows; a warp load reads 64 contiguous bytes of 4 rows).
// Each thread packs a quad's 4 digits of one position into one word; with the SW64 XOR the 32 lanes' words
// land in 32 distinct banks.
//
// Digits: one fma gives V = round(z 2^(e + 8(S-1))) + O in the low 52 bits of
// tt = fma(z, 2^(e + 8(S-1)), 2^52 + O), O = 128 (1 + 256 + ... + 256^(S-1)) (0x80 in every byte),
// 0 <= V < 2^(8S); digit t (t = 0 most significant) is byte S-1-t of V minus 128 -- as int8, the
// byte XOR 0x80 -- so sum_t d_t 2^-8t = round(w 2^8(S-1)) 2^-8(S-1) exactly (|w| < 127, while the
// digits reach 128 - 128/255).  Four rows' digits of one byte position are one word of a 4 x 4
// byte transpose (8 byte permutes for bytes 0-3, 4 for bytes 4-5).
//
// Padding rows (src < 0) read through a row pointer aimed at the shift vector itself, so z = c_j - c_j = +0
// with no per-value select; the ones column takes the block's padding mask.
constexpr int kQ1Threads = 256;
constexpr int kQ1PQ = 4;  // row quads per thread
#ifndef CVG_K1Q_MIN_BLOCKS
#define CVG_K1Q_MIN_BLOCKS 2
#endif

template <int S>
struct DigitOffset {  // 128 * (256^S - 1) / 255: 0x80 in every byte of V
  static constexpr int64_t v = 128 * (((int64_t)1 << (8 * S)) - 1) / 255;
};

template <int S>
constexpr int k1q_region_bytes() {  // one warp's S x 512 B of digits, 1 KB aligned
  return (S * 512 + 1023) / 1024 * 1024;
}
template <int S>
constexpr int k1q_smem_bytes() {
  return 2 * 8 * k1q_region_bytes<S>() + 1024;
}

__device__ __forceinline__ void tma_store_4d(const CUtensorMap* map, const void* src, int c0, int c1, int c2, int c3) {
  asm volatile(
      "cp.async.bulk.tensor.4d.global.shared::cta.bulk_group [%0, {%2, %3, %4, %5}], [%1];\n" ::"l"(map),
      "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2), "r"(c3)
      : "memory");
}

//
// DIRECT (the cut that runs beside the Gram, one CTA per SM): no shared-memory tile and no TMA -- on an SM whose
// TMA queue and shared memory belong to a Gram CTA both would wait behind the Gram's operand stages.  A thread
// then holds two runs of 8 consecutive rows (8 qq .. + 7 and 32 + 8 qq ..), so the 4 lanes of a column write 32
// contiguous bytes of its 64-byte line per store instruction (whole sectors) straight from registers, and the
// CTA publishes each finished 64-row block with a release increment of its segment's counter (seg_ready),
// which the Gram's TMA producer acquires before the segment's first stage.  Same digits, bit for bit.
// Registers: an SM sub-partition (16K registers) holds 3 of the lean Gram's 10 warps (96 registers) and 2 of the
// direct cut's 8, so the cut must stay at 112 -- launch bounds of 2 x 288 threads make ptxas cap it there.
template <typename T, int S, bool DIRECT>
__global__ void __launch_bounds__(DIRECT ? 288 : kQ1Threads, CVG_K1Q_MIN_BLOCKS)
    reorder_q_kernel(const __grid_constant__ CUtensorMap map_out, const T* __restrict__ x, int64_t ldx,
                     const T* __restrict__ y, int64_t ldy, int64_t k, int64_t m, const int64_t* __restrict__ src_row,
                     int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc,
                     const double* __restrict__ shift, const int* __restrict__ blkseg,
                     const unsigned long long* __restrict__ segmax, int headroom, int* __restrict__ ovf,
                     int* __restrict__ nonfinite, int64_t blk_lo, int64_t blk_hi, int8_t* __restrict__ zq,
                     unsigned* __restrict__ seg_ready) {
  // Blocks [blk_lo, blk_hi) of Z.  map_out's box is {64, 8, 1, S}: one warp's columns.
  // Out of range: tt outside [2^52, 2^53) (a non-finite z, or w below the digits' range) or V >= 2^(7S)
  // (w above it).  With sampled exponents (ovf != null) that marks the block's segment for the exact
  // pass; otherwise (exact exponents, where only a non-finite z can get there) it is the
  // non-finite-input flag (DatasetPair's allFinite, core.hpp:43-44).
  static_assert(std::is_same<T, double>::value, "padding rows read the (double) shift through the row pointers");
  static_assert(8 * S <= 48, "digits must fit the 52-bit window");
  constexpr uint32_t kHiMask = 8 * S >= 32 ? (0xfff00000u | (0x000fffffu & ~((1u << (8 * S - 32)) - 1u))) : 0xffffffffu;
  constexpr uint32_t kLoMask = 8 * S >= 32 ? 0u : ~((1u << (8 * S)) - 1u);
  constexpr int kRegion = k1q_region_bytes<S>();
  constexpr int NV = 4 * kQ1PQ;
  extern __shared__ uint8_t k1q_raw[];
  uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(k1q_raw) + 1023) & ~uintptr_t(1023));
  __shared__ const double* s_row[3][2][QK];  // per block: X and Y row pointers (padding: the shift)
  __shared__ uint32_t s_pad[3][2];           // per block: padding-row mask
  __shared__ int s_seg[3];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int j = lane >> 2, qq = lane & 3;
  const int col = 8 * w + j;  // column within the 64-column chunk
  // row quad of batch pp: TMA tile: qq + 4 pp; DIRECT: 2 qq + (pp & 1) + 8 (pp >> 1) (8-row runs)
  auto quad = [&](int pp) { return DIRECT ? 2 * qq + (pp & 1) + 8 * (pp >> 1) : qq + 4 * pp; };
  const int64_t wd = k + m;
  CVG_DCHECK(c_begin >= 0 && c_end <= kp && c_begin % 64 == 0 && zrows % QK == 0);
  const int64_t nchunk = (c_end - c_begin) / 64;
  const int64_t nblk = blk_hi;
  CVG_DCHECK(blk_lo >= 0 && blk_hi <= zrows / QK);
  const int64_t grid = gridDim.x;
  const double C = 0x1p52 + (double)DigitOffset<S>::v;
  auto load_src = [&](int64_t b, int rb) {
    if (threadIdx.x < QK && b < nblk) {  // warps 0 and 1, whole
      const int64_t src = src_row[b * QK + threadIdx.x];
      CVG_DCHECK(src < nsrc && src >= -1);
      s_row[rb][0][threadIdx.x] = src < 0 ? shift : x + src * ldx;
      s_row[rb][1][threadIdx.x] = src < 0 || m == 0 ? shift + k : y + src * ldy;
      const uint32_t pm = __ballot_sync(0xffffffffu, src < 0);
      if (lane == 0) s_pad[rb][w] = pm;
      if (threadIdx.x == 0) s_seg[rb] = blkseg[b];
    }
  };
  // the next chunk's NV values, shift and sampled column max, loaded while the current chunk is cut and stored
  double v[NV], shn = 0.0;
  unsigned long long mxn = 0ull;
  auto load_chunk = [&](int rb, int64_t c0) {
    const int64_t c = c0 + col;
    mxn = __ldg(segmax + (int64_t)s_seg[rb] * kp + c);
    if (c < wd) {
      shn = __ldg(shift + c);
      const int h = c < k ? 0 : 1;
      const int64_t cc = c < k ? c : c - k;
#pragma unroll
      for (int pp = 0; pp < kQ1PQ; ++pp)
#pragma unroll
        for (int i = 0; i < 4; ++i) v[4 * pp + i] = __ldg(s_row[rb][h][4 * quad(pp) + i] + cc);
    } else {
      shn = 0.0;
      const uint64_t pad = s_pad[rb][0] | (uint64_t)s_pad[rb][1] << 32;
#pragma unroll
      for (int pp = 0; pp < kQ1PQ; ++pp)
#pragma unroll
        for (int i = 0; i < 4; ++i)
          v[4 * pp + i] = c == wd && !((pad >> (4 * quad(pp) + i)) & 1) ? 1.0 : 0.0;  // ones / padding
    }
  };
  int64_t blk = blk_lo + blockIdx.x;
  load_src(blk, 0);
  load_src(blk + grid, 1);
  __syncthreads();
  if (blk < nblk) load_chunk(0, c_begin);
  int buf = 0, rb = 0;
  uint32_t oor_hi = 0, oor_lo = 0;  // out-of-range bits of this block's values
  for (; blk < nblk; blk += grid, rb = rb == 2 ? 0 : rb + 1) {
    const int rn = rb == 2 ? 0 : rb + 1;
    const int seg = s_seg[rb];
    for (int64_t ch = 0; ch < nchunk; ++ch, buf ^= 1) {
      const int64_t c0 = c_begin + 64 * ch;
      const double sh = shn;
      const unsigned long long mxb = mxn;
      const CutScale cs = cut_scales(seg_exponent(__longlong_as_double((long long)mxb), headroom) + 8 * (S - 1));
      // a sampled max of 0 cannot scale the column: any nonzero value sends the segment to the exact pass
      const bool zero_col = ovf && mxb == 0ull;
      uint32_t lo[NV], hi[NV];
      if (cs.pre == 1.0 && !zero_col) {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          const double tt = fma(__dsub_rn(v[e], sh), cs.sc, C);
          lo[e] = (uint32_t)__double2loint(tt);
          hi[e] = (uint32_t)__double2hiint(tt);
          oor_hi |= hi[e] ^ 0x43300000u;
          oor_lo |= lo[e];
        }
      } else {
#pragma unroll
        for (int e = 0; e < NV; ++e) {
          double z = __dsub_rn(v[e], sh);
          if (cs.pre != 1.0) z = __dmul_rn(z, cs.pre);
          const double tt = fma(z, cs.sc, C);
          lo[e] = (uint32_t)__double2loint(tt);
          hi[e] = (uint32_t)__double2hiint(tt);
          oor_hi |= (hi[e] ^ 0x43300000u) | (zero_col && z != 0.0 ? 0x80000000u : 0u);
          oor_lo |= lo[e];
        }
      }
      // next chunk's loads in flight while this one is cut and stored
      if (ch + 1 < nchunk)
        load_chunk(rb, c0 + 64);
      else if (blk + grid < nblk)
        load_chunk(rn, c_begin);
      uint8_t* region = tiles + buf * (8 * kRegion) + w * kRegion;
      if constexpr (!DIRECT) {
        // this warp's previous TMA store from this buffer has finished reading shared memory
        if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 1;\n" ::: "memory");
        __syncwarp();
      }
      // DIRECT: this column's 64-byte line of slice 0; slices are zrows * kp bytes apart
      int8_t* line = zq + (blk * kp + c0 + col) * QK + 8 * qq;
      uint32_t prev[S];
#pragma unroll
      for (int pp = 0; pp < kQ1PQ; ++pp) {
        // quad q = qq + 4 pp of line j, SWIZZLE_64B: 16-byte chunk (q >> 2) ^ ((j >> 1) & 3)
        const int off = j * 64 + ((pp ^ ((j >> 1) & 3)) << 4) + (qq << 2);
        // 4 x 4 byte transposes: word b = byte b of the 4 rows' V (low word: bytes 0-3, high word: 4-5)
        const uint32_t* L = lo + 4 * pp;
        const uint32_t* H = hi + 4 * pp;
        uint32_t wb[8];
        {
          const uint32_t x0 = __byte_perm(L[0], L[1], 0x5140), x1 = __byte_perm(L[0], L[1], 0x7362);
          const uint32_t y0 = __byte_perm(L[2], L[3], 0x5140), y1 = __byte_perm(L[2], L[3], 0x7362);
          wb[0] = __byte_perm(x0, y0, 0x5410);
          wb[1] = __byte_perm(x0, y0, 0x7632);
          wb[2] = __byte_perm(x1, y1, 0x5410);
          wb[3] = __byte_perm(x1, y1, 0x7632);
        }
        if constexpr (S > 4) {
          const uint32_t x0 = __byte_perm(H[0], H[1], 0x5140), y0 = __byte_perm(H[2], H[3], 0x5140);
          wb[4] = __byte_perm(x0, y0, 0x5410);
          wb[5] = __byte_perm(x0, y0, 0x7632);
        }
        if constexpr (!DIRECT) {
#pragma unroll
          for (int d = 0; d < S; ++d)  // digit d = byte S-1-d; offset binary -> two's complement: ^ 0x80
            *reinterpret_cast<uint32_t*>(region + d * 512 + off) = wb[S - 1 - d] ^ 0x80808080u;
        } else if (pp & 1) {  // rows 8 qq + 32 (pp >> 1) .. + 7 of the line: two quads, 8 bytes
#pragma unroll
          for (int d = 0; d < S; ++d)
            *reinterpret_cast<uint2*>(line + (int64_t)d * zrows * kp + 32 * (pp >> 1)) =
                make_uint2(prev[d], wb[S - 1 - d] ^ 0x80808080u);
        } else {
#pragma unroll
          for (int d = 0; d < S; ++d) prev[d] = wb[S - 1 - d] ^ 0x80808080u;
        }
      }
      if constexpr (!DIRECT) {
        asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
        __syncwarp();
        if (lane == 0) {
          tma_store_4d(&map_out, region, 0, (int)c0 + 8 * w, (int)blk, 0);
          asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
        }
      }
    }
    const uint32_t oor = (oor_hi & kHiMask) | (oor_lo & kLoMask);
    if (__any_sync(0xffffffffu, oor != 0u) && lane == 0) atomicOr(ovf ? ovf + seg : nonfinite, 1);
    oor_hi = oor_lo = 0;
    // every warp is past its reads of the block before this one: its buffer takes the block two ahead
    load_src(blk + 2 * grid, rb == 0 ? 2 : rb - 1);
    if constexpr (DIRECT) asm volatile("fence.proxy.async.global;\n" ::: "memory");  // these digits are read by TMA
    __syncthreads();
    if constexpr (DIRECT) {
      if (threadIdx.x == 0 && seg_ready) {  // every thread's stores of this block precede the barrier
        __threadfence();
        atomicAdd(seg_ready + seg, 1u);
      }
    }
  }
  if constexpr (!DIRECT) {
    if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  }
}

// 4-D map over Zq: {64 rows, kp, zrows / 64, S} bytes, box {64, box_cols, 1, box_slices (default S)}, SWIZZLE_64B.
inline bool make_zq_map(CUtensorMap* map, const int8_t* zq, int64_t zrows, int64_t kp, int slices, int box_cols,
                        int box_rows = QK, int box_slices = 0) {
  EncodeTiledFn enc = encode_fn();
  if (!enc) return false;
  const cuuint64_t dims[4] = {(cuuint64_t)QK, (cuuint64_t)kp, (cuuint64_t)(zrows / QK), (cuuint64_t)slices};
  const cuuint64_t strides[3] = {(cuuint64_t)QK, (cuuint64_t)kp * QK, (cuuint64_t)zrows * kp};
  const cuuint32_t box[4] = {(cuuint32_t)box_rows, (cuuint32_t)box_cols, 1,
                             (cuuint32_t)(box_slices > 0 ? box_slices : slices)};
  const cuuint32_t estr[4] = {1, 1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_UINT8, 4, const_cast<int8_t*>(zq), dims, strides, box, estr,
             CU_TENSOR_MAP_INTERLEAVE_NONE, box_rows == 64 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

template <int S, int KS, bool LEAN>
bool launch_gram_i8_s(const int8_t* zq, const unsigned long long* segmax, int headroom, int64_t zrows, int64_t kp,
                      const GramTask* segs, int64_t seg_base, int64_t nseg, const int2* tiles, int ntiles, double* part,
                      int max_ctas, const unsigned* seg_ready, int* abort_flag, int32_t* split_ws, unsigned* split_cnt,
                      int64_t min_seg_rows, cudaStream_t s) {
  CUtensorMap ma, ma64, mb;
  if (!make_zq_map(&ma, zq, zrows, kp, S, QA, KS) || !make_zq_map(&ma64, zq, zrows, kp, S, QB, KS, 1) ||
      !make_zq_map(&mb, zq, zrows, kp, S, QB, KS))
    return false;
  using C = QCfg<S, KS, 8>;
  static std::atomic<uint64_t> attrs_done{0};  // one per <S, KS, LEAN> instantiation
  if (first_on_device(attrs_done))
    cudaFuncSetAttribute(gram_i8_kernel<S, KS, 8, LEAN>, cudaFuncAttributeMaxDynamicSharedMemorySize, C::kSmem);
  int dev = 0, sms = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int64_t nitems = nseg * (int64_t)ntiles;
  // persistent: one CTA per SM (1 fits: shared memory), or max_ctas
  const int64_t blocks = std::min<int64_t>(nitems, max_ctas > 0 ? std::min(max_ctas, sms) : sms);
  if (blocks <= 0) return true;
  // Tail split (kernel comment): the `tail` items past the last full round become tail * f row parts, at most one
  // more round of the grid; only when they fill at most half of it and every part keeps >= 4 stages.
  const int64_t tail = nitems % blocks;
  int64_t f = 1;
  if (split_ws && split_cnt && tail > 0 && 2 * tail <= blocks) {
    f = std::min<int64_t>(blocks / tail, 8);
    while (f > 1 && min_seg_rows / KS / f < 4) --f;
  }
  const int64_t split_from = nitems - tail;
  if (f > 1) cudaMemsetAsync(split_cnt, 0, sizeof(unsigned) * tail, s);
  gram_i8_kernel<S, KS, 8, LEAN><<<(unsigned)blocks, kQThreads, C::kSmem, s>>>(
      ma, ma64, mb, segmax, segs, tiles, ntiles, f > 1 ? split_from + tail * f : nitems, seg_base, kp, part, headroom,
      seg_ready, abort_flag, split_from, (int)f, split_ws, split_cnt);
  return true;
}

template <typename T, int S>
bool launch_k1q(const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m, const int64_t* src_row,
                int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc, const double* shift,
                const int* blkseg, const unsigned long long* segmax, int headroom, int* ovf, int8_t* zq, int* nonfinite,
                int64_t blk_lo, int64_t blk_hi, int max_sms, int direct_ctas_per_sm, unsigned* seg_ready,
                cudaStream_t s) {
  int dev = 0, sms_all = 0;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms_all, cudaDevAttrMultiProcessorCount, dev);
  if (direct_ctas_per_sm > 0) {  // the register-only cut (beside the Gram: one CTA per SM)
    CUtensorMap none{};
    const int64_t blocks = std::min<int64_t>(blk_hi - blk_lo, (int64_t)direct_ctas_per_sm * sms_all);
    if (blocks <= 0) return true;
    // same shared-memory carveout as the Gram it shares the SM with (an SM holds one configuration at a time)
    static std::atomic<uint64_t> direct_done{0};
    if (first_on_device(direct_done))
      cudaFuncSetAttribute(reorder_q_kernel<T, S, true>, cudaFuncAttributePreferredSharedMemoryCarveout,
                           cudaSharedmemCarveoutMaxShared);
    reorder_q_kernel<T, S, true><<<(unsigned)blocks, kQ1Threads, 0, s>>>(
        none, (const T*)x, ldx, (const T*)y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, blkseg, segmax,
        headroom, ovf, nonfinite, blk_lo, blk_hi, zq, seg_ready);
    return true;
  }
  CUtensorMap mo;
  if (!make_zq_map(&mo, zq, zrows, kp, S, 8)) return false;
  constexpr int smem = k1q_smem_bytes<S>();
  // grid-stride over one wave of resident CTAs.  Function attributes are per device (one process may drive
  // several: cvg_context_create_multi), so they are set on every launch; the occupancy query is cached per device.
  static std::atomic<int> wave_cache[64];
  static std::atomic<uint64_t> attrs_done{0};
  if (first_on_device(attrs_done))
    cudaFuncSetAttribute(reorder_q_kernel<T, S, false>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int wave = wave_cache[dev & 63].load(std::memory_order_relaxed);
  if (!wave) {
    int per_sm = 0;
    cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, reorder_q_kernel<T, S, false>, kQ1Threads, smem);
    wave = (per_sm > 0 ? per_sm : 1) * sms_all;
    wave_cache[dev & 63].store(wave, std::memory_order_relaxed);
  }
  if (max_sms > 0 && max_sms < sms_all) wave = wave / sms_all * max_sms;  // confine to max_sms SMs' worth
  const int64_t blocks = std::min<int64_t>(blk_hi - blk_lo, (int64_t)std::max(wave, 1));
  if (blocks <= 0) return true;
  reorder_q_kernel<T, S, false><<<(unsigned)blocks, kQ1Threads, smem, s>>>(
      mo, (const T*)x, ldx, (const T*)y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, blkseg, segmax,
      headroom, ovf, nonfinite, blk_lo, blk_hi, zq, nullptr);
  return true;
}

}  // namespace

void launch_segmax(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                   const int64_t* src_row, const GramTask* segs, int64_t nseg, int64_t max_seg_rows, int64_t kp,
                   int64_t c_begin, int64_t c_end, int64_t nsrc, const double* shift, int stride, const int* only,
                   unsigned long long* segmax, cudaStream_t s) {
  if (nseg <= 0 || c_end <= c_begin) return;
  // bound on any segment's sampled rows: segments below 1024 rows are scanned whole (stride 1), longer ones
  // keep >= 512 rows at a stride of at most `stride`
  max_seg_rows = std::max<int64_t>(std::min<int64_t>(max_seg_rows, 1024), (max_seg_rows + stride - 1) / stride) + 1;
  // row slices: ~4096+ CTAs in all, 128 .. 1024 rows each
  const int64_t nchunk = (c_end - c_begin) / 64;
  int64_t slice = 1024;
  while (slice > 128 && nseg * nchunk * ((max_seg_rows + slice - 1) / slice) < 4096) slice /= 2;
  const dim3 grid((unsigned)nseg, (unsigned)nchunk, (unsigned)((max_seg_rows + slice - 1) / slice));
  if (dtype == 0)
    segmax_kernel<double><<<grid, kSmThreads, 0, s>>>((const double*)x, ldx, (const double*)y, ldy, k, m, src_row,
                                                      segs, kp, c_begin, nsrc, shift, slice, stride, only, segmax);
  else
    segmax_kernel<float><<<grid, kSmThreads, 0, s>>>((const float*)x, ldx, (const float*)y, ldy, k, m, src_row, segs,
                                                     kp, c_begin, nsrc, shift, slice, stride, only, segmax);
}

bool launch_reorder_q(int dtype, int slices, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k,
                      int64_t m, const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                      int64_t nsrc, const double* shift, const int* blkseg, const unsigned long long* segmax,
                      int headroom, int* ovf, int8_t* zq, int* nonfinite, cudaStream_t s, int64_t blk_lo,
                      int64_t blk_hi, int max_sms, int direct_ctas_per_sm, unsigned* seg_ready) {
  if (zrows <= 0 || c_end <= c_begin) return true;
  if (blk_hi < 0) blk_hi = zrows / QK;
#define CVG_K1Q(T, S)                                                                                              \
  return launch_k1q<T, S>(x, ldx, y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, blkseg, segmax, \
                          headroom, ovf, zq, nonfinite, blk_lo, blk_hi, max_sms, direct_ctas_per_sm, seg_ready, s)
  (void)dtype;  // fp64 inputs only (fp32 inputs take the fp16-split Gram)
  if (slices == 5) CVG_K1Q(double, 5);
  CVG_K1Q(double, 6);
#undef CVG_K1Q
}

// Pipeline stage rows: 64 (SW64; S = 7 fits 2 stages of 84 KB) or, with CVG_I8_STAGE_ROWS=32, 32 (SW32; 5
// stages of 42 KB).  c1 Gram 2.94 vs 3.35 ms, c4 12.9 vs 16.0 ms: fewer, longer MMA runs per barrier win.
static int i8_stage_rows() {
  static const int v = [] {
    const char* e = std::getenv("CVG_I8_STAGE_ROWS");
    return e && std::atoi(e) == 32 ? 32 : 64;
  }();
  return v;
}

// Workspace of the tail split for a grid of `ctas` CTAs: one int32 dump per part (<= ctas parts) and one counter
// per tail item; 7 accumulators of 128 x 64 int32 per dump (S = 6).
size_t gram_i8_split_ws_bytes(int ctas) { return (size_t)ctas * (7 * QA * QB * sizeof(int32_t)); }

// lean != 0: the 96-register kernel that leaves room for a cut CTA on the same SM; seg_ready / abort_flag (both
// or neither): wait for the concurrent cut's per-segment block counts.
bool launch_gram_i8(int slices, const int8_t* zq, const unsigned long long* segmax, int headroom, int64_t zrows,
                    int64_t kp, const GramTask* segs, int64_t nseg, const int2* tiles, int ntiles, double* part,
                    cudaStream_t s, int64_t seg_base, int max_ctas, int lean, const unsigned* seg_ready,
                    int* abort_flag, int32_t* split_ws, unsigned* split_cnt, int64_t min_seg_rows) {
#define CVG_GRAM_I8(S, KS, LEAN)                                                                                \
  return launch_gram_i8_s<S, KS, LEAN>(zq, segmax, headroom, zrows, kp, segs, seg_base, nseg, tiles, ntiles, part, \
                                       max_ctas, seg_ready, abort_flag, split_ws, split_cnt, min_seg_rows, s)
  if (lean) {
    if (slices == 5) CVG_GRAM_I8(5, 64, true);
    CVG_GRAM_I8(6, 64, true);
  }
  if (i8_stage_rows() == 64) {
    if (slices == 5) CVG_GRAM_I8(5, 64, false);
    CVG_GRAM_I8(6, 64, false);
  }
  if (slices == 5) CVG_GRAM_I8(5, 32, false);
  CVG_GRAM_I8(6, 32, false);
#undef CVG_GRAM_I8
}

}  // namespace cvg
