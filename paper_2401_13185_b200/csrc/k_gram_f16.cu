// K1H + K2h: the fp32-input fold Gram on tcgen05 kind::f16 (the default fp32 path).
//
// BASELINE.json configs[3]: fp32 inputs, fp32 accumulation on tensor cores, 1e-4
// against the fp64 oracle.  Each shifted value z is split into two fp16 terms,
// z * 2^e = hi + lo (hi = fp16_rn(z * 2^e), lo = fp16_rn(z * 2^e - hi)), and every
// product is formed as hi·hi + hi·lo + lo·hi into an fp32 TMEM accumulator: the
// same 11 + 11 significant bits as the 3xTF32 split (k_gram_tf32.cu), at the
// kind::f16 rate (2x kind::tf32) and with half the operand bytes.
//
// fp16 has 5 exponent bits, so every value is scaled by a power of two first:
// one exponent e per (row group of G rows, column), chosen by K1H from the
// group's max |z| so the largest value lands in [2^14, 2^15).  Power-of-two
// scaling is exact, so the split keeps 22 bits of every value whose lo term is
// a normal fp16 (all values within 2^18 of their group's column max; smaller
// ones keep an absolute error below 2^-39 of that max).  A row group is also
// the Gram's fp32 accumulation chunk: the MMAs of one group accumulate in one
// TMEM buffer (products scaled by 2^(e_i + e_j)), and the drain warps unscale
// each element exactly while adding it to the fp64 accumulator:
//     acc64 += (double)(f * 2^-e_j) * 2^-e_i      (both multiplications exact).
// Segments and folds are padded to G rows so a group never straddles two
// segments; G (64, 128 or 256) is a plan constant, so results stay
// bit-identical across GPU counts.
//
// Layout: Zh[row / 64][col][row % 64] fp16 (hi and lo arrays): 64 rows of a
// column = 128 B, one SWIZZLE_128B K-major atom row; one 3-D TMA box {64 rows,
// 128 columns, 1 block} = 16 KB per operand slab.  unscale[row / G][col] = 2^-e.
//
// K2h roles (10 warps, 1 CTA per SM, 192 KB of stages, 256 TMEM columns):
//   warp 0      TMA producer: hi / lo slabs of both column tiles per 64-row stage
//   warp 1      TMEM owner + MMA issuer (one elected thread), ping-pong accumulators
//   warps 2..9  drain every row group: tcgen05.ld 128 lanes x 64 columns each, exact
//               unscale, fp64 sums, write the fp64 partial at the end
#include <cuda_fp16.h>

#include "cvg_internal.cuh"
#include "tc_util.cuh"

namespace cvg {
namespace {

using namespace tc;

constexpr int TT = 128;                         // tile edge (M = N = 128)
constexpr int KS = 64;                          // rows per stage = 128 B of fp16
constexpr int NST = 3;                          // pipeline stages
constexpr int kOpBytes = TT * KS * 2;           // 16 KB per operand slab
constexpr int kStageBytes = 4 * kOpBytes;       // A_hi, A_lo, B_hi, B_lo
constexpr int kSmemF16 = NST * kStageBytes + 1024;
constexpr int kEpiWarps = 8;                    // 4 TMEM lane quarters x 2 column halves
constexpr int kThreads = 64 + 32 * kEpiWarps;

// kind::f16 with fp16 A and B (format 0), fp32 accumulate, both K-major, M = N = 128.
constexpr uint32_t kIdescF16 = (1u << 4) | ((uint32_t)(TT >> 3) << 17) | ((uint32_t)(TT >> 4) << 24);

__device__ __forceinline__ void mma_f16(uint32_t tmem_d, uint64_t a, uint64_t b, uint32_t accumulate) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "setp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n"
      "}\n" ::"r"(tmem_d),
      "l"(a), "l"(b), "r"(kIdescF16), "r"(accumulate));
}

// Drain warps (both kernels): per row group, wait for the TMEM chunk, unscale it exactly
// ((double)(f * 2^-e_j) * 2^-e_i) into 64 fp64 accumulators per thread, release the buffer
// with `release(b)`; finally write this thread's 64 entries (Gram row rcol) to `out` (if any).
//
// fp32 -> fp64 without F2F: F2F.F64.F32 issues at ~4 per clock per SM (XU), which made
// the drain the kernel's bottleneck.  For t = f * 2^-e_j (fp32 bits u), the fp64 whose
// bits are (sign(u) | ((u & 0x7fffffff) >> 3), u << 29) is exactly t * 2^-896 (normal and
// subnormal t alike, +-0 stays +-0), so with M = 2^-e_i * 2^896,
//     acc = fma(D, M, acc)  ==  fma((double)t, 2^-e_i, acc)    (bit for bit)
// at 3 integer ops per element.
__device__ __forceinline__ double fp32_bits_scaled_signed(uint32_t u) {
  return __hiloint2double((int)((u & 0x80000000u) | ((u >> 3) & 0x0fffffffu)), (int)(u << 29));
}

template <typename Release>
__device__ __forceinline__ void drain_groups(uint32_t tmem_d, int q, int h, int lane, float* tab,
                                             const float* __restrict__ unscale, int64_t kp, int64_t g0, int64_t rcol,
                                             int64_t col0, int nchunks, uint64_t* acc_full, Release release,
                                             double* out) {
  // this group's factors: the lane's 2 table columns and its row; stepped by kp per group
  const bool row_ok = rcol < kp;  // a CTA-pair's row block past kp (odd block count) reads zeros
  const float* uc = unscale + g0 * kp + col0 + 2 * lane;
  const float* ur = unscale + g0 * kp + (row_ok ? rcol : 0);
  float2 cs = *reinterpret_cast<const float2*>(uc);
  float rs = *ur;
  double acc64[64];
#pragma unroll
  for (int j = 0; j < 64; ++j) acc64[j] = 0.0;
  for (int chunk = 0; chunk < nchunks; ++chunk) {
    const int b = chunk & 1;
    __syncwarp();
    *reinterpret_cast<float2*>(tab + 2 * lane) = cs;
    const double mrow = (double)rs * 0x1p+896;  // 2^-e_i * 2^896 (e_i in [-64, 64]: a normal double)
    if (chunk + 1 < nchunks) {  // next group's factors, in flight during this drain
      uc += kp;
      ur += kp;
      cs = *reinterpret_cast<const float2*>(uc);
      rs = *ur;
    }
    __syncwarp();
    mbar_wait(&acc_full[b], (uint32_t)(chunk >> 1) & 1u);
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
    for (int c0 = 0; c0 < 64; c0 += 16) {
      uint32_t r[16];
      tmem_ld16(tmem_d + ((uint32_t)(32 * q) << 16) + (uint32_t)(b * TT + 64 * h + c0), r);
#pragma unroll
      for (int j = 0; j < 16; j += 4) {
        const float4 s4 = *reinterpret_cast<const float4*>(tab + c0 + j);
        const float sc[4] = {s4.x, s4.y, s4.z, s4.w};
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const uint32_t u = __float_as_uint(__uint_as_float(r[j + i]) * sc[i]);
          acc64[c0 + j + i] = fma(fp32_bits_scaled_signed(u), mrow, acc64[c0 + j + i]);
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) release(b);
  }
  if (out) {
#pragma unroll
    for (int j = 0; j < 64; j += 2) *reinterpret_cast<double2*>(out + j) = make_double2(acc64[j], acc64[j + 1]);
  }
}

__global__ void __launch_bounds__(kThreads, 1)
    gram_f16s_kernel(const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo,
                     const float* __restrict__ unscale, int group_rows, const GramTask* __restrict__ segs,
                     const int2* __restrict__ tiles, int ntiles, int64_t kp, double* __restrict__ part) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  __shared__ __align__(8) uint64_t full_bar[NST], empty_bar[NST], acc_full[2], acc_empty[2];
  __shared__ uint32_t tmem_base;
  __shared__ __align__(16) float s_tab[kEpiWarps][64];  // per drain warp: its 64 column unscale factors

  const int seg = blockIdx.x / ntiles;
  const int2 tile0 = tiles[blockIdx.x - seg * ntiles];
  const int2 tile = make_int2(uniform(tile0.x), uniform(tile0.y));
  const bool diag = tile.x == tile.y;
  const GramTask task0 = segs[seg];
  const GramTask task{uniform(task0.zrow), uniform(task0.rows)};
  CVG_DCHECK(task.zrow % group_rows == 0 && task.rows % KS == 0 && task.rows > 0);
  CVG_DCHECK(tile.x >= 0 && tile.x <= tile.y && (int64_t)(tile.y + 1) * TT <= kp);
  const int nsteps = (int)(task.rows / KS);
  const int drain_steps = group_rows / KS;
  const int nchunks = (nsteps + drain_steps - 1) / drain_steps;
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
    const uint32_t bytes = (uint32_t)kOpBytes * 2u * (diag ? 1u : 2u);
    for (int it = 0; it < nsteps; ++it) {
      const int s = it % NST;
      const uint32_t ph = (uint32_t)(it / NST) & 1u;
      mbar_wait(&empty_bar[s], ph ^ 1u);
      const int blk = (int)(task.zrow / KS) + it;  // 64-row block index
      if (elect_one()) {
        mbar_expect_tx(&full_bar[s], bytes);
        tma_load_3d(op(s, 0), &map_hi, &full_bar[s], 0, tile.x * TT, blk);
        tma_load_3d(op(s, 1), &map_lo, &full_bar[s], 0, tile.x * TT, blk);
        if (!diag) {
          tma_load_3d(op(s, 2), &map_hi, &full_bar[s], 0, tile.y * TT, blk);
          tma_load_3d(op(s, 3), &map_lo, &full_bar[s], 0, tile.y * TT, blk);
        }
      }
      __syncwarp();
    }
  } else if (warp == 1) {  // ---- MMA issuer (whole warp waits; one elected lane issues), accumulator b = chunk & 1
    for (int it = 0; it < nsteps; ++it) {
      const int chunk = it / drain_steps, b = chunk & 1;
      const bool first = it % drain_steps == 0;
      if (first && chunk >= 2) mbar_wait(&acc_empty[b], (uint32_t)((chunk >> 1) - 1) & 1u);  // drained
      const int s = it % NST;
      mbar_wait(&full_bar[s], (uint32_t)(it / NST) & 1u);
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
      const uint32_t acc = tmem_d + (uint32_t)(b * TT);
      const uint64_t a_hi = kmajor_sw128_desc(op(s, 0)), a_lo = kmajor_sw128_desc(op(s, 1));
      const uint64_t b_hi = diag ? a_hi : kmajor_sw128_desc(op(s, 2));
      const uint64_t b_lo = diag ? a_lo : kmajor_sw128_desc(op(s, 3));
      if (elect_one()) {
#pragma unroll
        for (int k = 0; k < KS / 16; ++k) {  // K = 16 fp16 = 32 B per MMA: +2 in 16-byte descriptor units
          const uint64_t dk = 2ull * k;
          mma_f16(acc, a_hi + dk, b_hi + dk, (first && k == 0) ? 0u : 1u);
          mma_f16(acc, a_hi + dk, b_lo + dk, 1u);
          mma_f16(acc, a_lo + dk, b_hi + dk, 1u);
        }
        mma_commit(&empty_bar[s]);  // frees the stage once these MMAs have read it
        if (it % drain_steps == drain_steps - 1 || it == nsteps - 1) mma_commit(&acc_full[b]);
      }
      __syncwarp();
    }
  } else {  // ---- drain warps: scaled fp32 TMEM chunks -> exact unscale -> fp64 registers
    const int dw = warp - 2;
    const int q = warp & 3;  // TMEM lanes [32q, 32q + 32) (hardware: warp id mod 4)
    const int h = dw >> 2;   // columns [64h, 64h + 64)
    const int64_t rcol = (int64_t)tile.x * TT + 32 * q + lane;  // this thread's Gram row (a Z column)
    drain_groups(tmem_d, q, h, lane, s_tab[dw], unscale, kp, task.zrow / group_rows, rcol,
                 (int64_t)tile.y * TT + 64 * h, nchunks, acc_full, [&](int b) { mbar_arrive(&acc_empty[b]); },
                 part + (int64_t)seg * kp * kp + rcol * kp + (int64_t)tile.y * TT + 64 * h);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (warp == 1) {
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem_d), "r"(2 * TT));
  }
}

// K1H: bucket, shift, scale, fp16-split, transpose into Zh[block][col][64] (HBM-bound).
// One CTA per G bucketed rows, two CTAs per SM (one loads while the other
// computes); 64-column chunks.  Lane (h, cq) = (lane >> 4, lane & 15) holds the 4
// adjacent columns c0 + 4cq .. + 3 (one 16-byte load per row: a warp reads two
// 256-byte row segments) of the row pairs rp = 2w + h + 32j of warp w.  A column's
// group max is a 32-way reduction in shared memory; each (hi, lo) row pair is one
// 32-bit word of a column-major shared tile whose row-pair index is XOR-swizzled
// by the column quad (word = col * G/2 + (rp ^ 2(col >> 2))): the transposed
// writes hit 32 distinct banks and the write-out reads 16-byte blocks
// conflict-free, so the output leaves as 16-byte stores (a warp: 4 columns x 128 B
// contiguous).
constexpr int kK1hThreads = 512;
constexpr int kK1hWarps = kK1hThreads / 32;
constexpr int kK1hCols = 64;

template <int G>
constexpr int k1h_smem_bytes() {
  return 2 * kK1hCols * (G / 2) * 4 + 2 * kK1hWarps * kK1hCols * 4 + kK1hCols * 4 + G * 8;
}

template <typename T>
__device__ __forceinline__ void load4(const T* p, float (&v)[4]) {
  if constexpr (sizeof(T) == 4) {
    const float4 q = __ldg(reinterpret_cast<const float4*>(p));
    v[0] = q.x, v[1] = q.y, v[2] = q.z, v[3] = q.w;
  } else {
    const double2 a = __ldg(reinterpret_cast<const double2*>(p)), b = __ldg(reinterpret_cast<const double2*>(p) + 1);
    v[0] = (float)a.x, v[1] = (float)a.y, v[2] = (float)b.x, v[3] = (float)b.y;
  }
}

template <typename T, int G>
__global__ void __launch_bounds__(kK1hThreads, 2) reorder_split_h_kernel(
    const T* __restrict__ x, int64_t ldx, const T* __restrict__ y, int64_t ldy, int64_t k, int64_t m,
    const int64_t* __restrict__ src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc,
    const double* __restrict__ shift, __half* __restrict__ zh_hi, __half* __restrict__ zh_lo,
    float* __restrict__ unscale, int* __restrict__ nonfinite) {
  constexpr int S = G / 2;    // words (row pairs) per column
  constexpr int NJ = G / 64;  // row pairs per thread
  constexpr int kSlots = 2 * kK1hWarps;  // row-pair slots per 32 row pairs (= 32)
  extern __shared__ __align__(16) uint8_t k1h_smem[];
  uint32_t* s_hi = reinterpret_cast<uint32_t*>(k1h_smem);
  uint32_t* s_lo = s_hi + kK1hCols * S;
  float* s_max = reinterpret_cast<float*>(s_lo + kK1hCols * S);  // [slot][cols]
  float* s_scale = s_max + kSlots * kK1hCols;                     // [cols] 2^e
  int64_t* s_src = reinterpret_cast<int64_t*>(s_scale + kK1hCols);
  const int64_t grp = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int h = lane >> 4, cq = lane & 15;
  const int slot = 2 * w + h;  // this thread's row pairs: slot + 32j
  const int64_t wd = k + m;
  CVG_DCHECK(c_begin >= 0 && c_end <= kp && c_begin % kK1hCols == 0 && zrows % G == 0);
  for (int i = t; i < G; i += kK1hThreads) {
    const int64_t r = grp * G + i;
    const int64_t src = r < zrows ? src_row[r] : -1;
    CVG_DCHECK(src < nsrc);
    s_src[i] = src;
  }
  __syncthreads();
  bool all_real = true;
#pragma unroll
  for (int j = 0; j < NJ; ++j)
#pragma unroll
    for (int p = 0; p < 2; ++p) all_real &= s_src[2 * (slot + 32 * j) + p] >= 0;
  // 16-byte row loads need 16-byte aligned rows
  const bool vec_ok = (ldx * (int64_t)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  float nan_acc = 0.f;  // v * 0 is NaN exactly when v is not finite
  bool too_big = false;
  float v[NJ][2][4];
  // Fast chunks (every column an X column, every row real, aligned rows): no per-element checks.
  auto fast_chunk = [&](int64_t c0) { return all_real && vec_ok && c0 + kK1hCols <= k; };
  auto load_chunk = [&](int64_t c0) {
    if (fast_chunk(c0)) {
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int p = 0; p < 2; ++p)
          load4(x + (int64_t)(int32_t)s_src[2 * (slot + 32 * j) + p] * ldx + c0 + 4 * cq, v[j][p]);
      return;
    }
#pragma unroll
    for (int j = 0; j < NJ; ++j)
#pragma unroll
      for (int p = 0; p < 2; ++p) {
        const int64_t src = s_src[2 * (slot + 32 * j) + p];
#pragma unroll
        for (int e = 0; e < 4; ++e) {
          const int64_t ce = c0 + 4 * cq + e;
          float val = 0.f;
          if (src >= 0) {
            if (ce < k)
              val = (float)__ldg(x + src * ldx + ce);
            else if (ce < wd)
              val = (float)__ldg(y + src * ldy + (ce - k));
            else if (ce == wd)
              val = 1.f;  // ones column: column sums ride in the Gram
          }
          v[j][p][e] = val;
        }
      }
  };
  load_chunk(c_begin);
  for (int64_t c0 = c_begin; c0 < c_end; c0 += kK1hCols) {
    // shift; per-column max |z| over this thread's rows
    const bool fast = fast_chunk(c0);
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t ce = c0 + 4 * cq + e;
      const float sh = ce < wd ? (float)__ldg(shift + ce) : 0.f;  // ones / padding columns: no shift
      float mx = 0.f;
#pragma unroll
      for (int j = 0; j < NJ; ++j)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          nan_acc = fmaf(v[j][p][e], 0.f, nan_acc);
          const bool shifted = fast || (s_src[2 * (slot + 32 * j) + p] >= 0 && ce < wd);
          const float z = shifted ? v[j][p][e] - sh : v[j][p][e];
          v[j][p][e] = z;
          mx = fmaxf(mx, fabsf(z));
        }
      s_max[slot * kK1hCols + 4 * cq + e] = mx;
    }
    __syncthreads();
    if (t < kK1hCols) {
      float mx = 0.f;
#pragma unroll
      for (int i = 0; i < kSlots; ++i) mx = fmaxf(mx, s_max[i * kK1hCols + t]);
      // e: the group's max |z| scaled into [2^14, 2^15); zero / non-finite columns keep e = 0
      int ex = 0;
      if (mx > 0.f && isfinite(mx)) {
        const int be = (int)((__float_as_uint(mx) >> 23) & 0xff);
        ex = 14 - (be == 0 ? -127 : be - 127);
        too_big |= ex < -64;  // |z| >= 2^79: products beyond the fp32 accumulation range
        ex = max(-64, min(64, ex));
      }
      s_scale[t] = __uint_as_float((uint32_t)(127 + ex) << 23);
      unscale[grp * kp + c0 + t] = __uint_as_float((uint32_t)(127 - ex) << 23);
    }
    __syncthreads();
    // scale (exact) and split: hi = fp16_rn(z'), lo = fp16_rn(z' - hi); one word per row pair,
    // at col * S + (rp ^ 2cq) (col >> 2 == cq)
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int col = 4 * cq + e;
      const float sc = s_scale[col];
#pragma unroll
      for (int j = 0; j < NJ; ++j) {
        const float z0 = v[j][0][e] * sc, z1 = v[j][1][e] * sc;
        const __half2 hi = __floats2half2_rn(z0, z1);
        const float2 hf = __half22float2(hi);
        const __half2 lo = __floats2half2_rn(z0 - hf.x, z1 - hf.y);
        const int word = col * S + ((slot + 32 * j) ^ (2 * cq));
        s_hi[word] = *reinterpret_cast<const uint32_t*>(&hi);
        s_lo[word] = *reinterpret_cast<const uint32_t*>(&lo);
      }
    }
    __syncthreads();
    if (c0 + kK1hCols < c_end) load_chunk(c0 + kK1hCols);  // in flight while the stores below drain
    // write: task = (64-row block b, column quad q): lane i -> column 4q + i / 8, words 4(i % 8) .. + 3
    // of the block (16 B; a warp stores 4 columns x 128 B contiguous) for hi and for lo.
    const int mq = lane & 7, cl = lane >> 3;
#pragma unroll 2
    for (int task = w; task < (G / 64) * (kK1hCols / 4); task += kK1hWarps) {
      const int b = task / (kK1hCols / 4), q = task - b * (kK1hCols / 4);
      const int col = 4 * q + cl;
      // row pairs 32b + 4mq + r (r < 4) are stored at 32b + ((4mq + r) ^ 2q): one 16-B block, words permuted
      const int word = col * S + 32 * b + 4 * (mq ^ (q >> 1));
      const uint4 hv = *reinterpret_cast<const uint4*>(s_hi + word);
      const uint4 lv = *reinterpret_cast<const uint4*>(s_lo + word);
      const bool sw = q & 1;  // warp-uniform: words r ^ 2
      const uint4 ho = sw ? make_uint4(hv.z, hv.w, hv.x, hv.y) : hv;
      const uint4 lo = sw ? make_uint4(lv.z, lv.w, lv.x, lv.y) : lv;
      const int64_t off = ((grp * (G / 64) + b) * kp + c0 + col) * 32 + 4 * mq;  // words
      *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(zh_hi) + off) = ho;
      *reinterpret_cast<uint4*>(reinterpret_cast<uint32_t*>(zh_lo) + off) = lo;
    }
    __syncthreads();
  }
  // bit 0: a non-finite input; bit 1: a finite magnitude the fp32 accumulation cannot hold
  const unsigned bad = __ballot_sync(0xffffffffu, nan_acc != 0.f), big = __ballot_sync(0xffffffffu, too_big);
  if (lane == 0 && (bad | big)) atomicOr(nonfinite, (bad ? 1 : 0) | (big ? 2 : 0));
}

template <typename T, int G>
void launch_k1h(const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m, const int64_t* src_row,
                int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc, const double* shift,
                __half* zh_hi, __half* zh_lo, float* unscale, int* nonfinite, cudaStream_t s) {
  constexpr int smem = k1h_smem_bytes<G>();
  cudaFuncSetAttribute(reorder_split_h_kernel<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  reorder_split_h_kernel<T, G><<<(unsigned)(zrows / G), kK1hThreads, smem, s>>>(
      (const T*)x, ldx, (const T*)y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, zh_hi, zh_lo,
      unscale, nonfinite);
}

}  // namespace

void launch_reorder_split_h(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                            const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                            int64_t nsrc, const double* shift, int group_rows, void* zh_hi, void* zh_lo,
                            float* unscale, int* nonfinite, cudaStream_t s) {
  if (zrows <= 0 || c_end <= c_begin) return;
  __half* hi = static_cast<__half*>(zh_hi);
  __half* lo = static_cast<__half*>(zh_lo);
#define CVG_K1H(T, G)                                                                                         \
  launch_k1h<T, G>(x, ldx, y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, hi, lo, unscale, \
                   nonfinite, s)
  if (dtype == 0) {
    if (group_rows == 256) CVG_K1H(double, 256);
    else if (group_rows == 128) CVG_K1H(double, 128);
    else CVG_K1H(double, 64);
  } else {
    if (group_rows == 256) CVG_K1H(float, 256);
    else if (group_rows == 128) CVG_K1H(float, 128);
    else CVG_K1H(float, 64);
  }
#undef CVG_K1H
}

bool launch_gram_f16s(const void* zh_hi, const void* zh_lo, const float* unscale, int group_rows, int64_t zrows,
                      int64_t kp, const GramTask* segs, int64_t nseg, const int2* tiles128, int ntiles, double* part,
                      cudaStream_t s) {
  CUtensorMap mh, ml;
  if (!make_blocked_map(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, zh_hi, 2, zrows, kp, TT) ||
      !make_blocked_map(&ml, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, zh_lo, 2, zrows, kp, TT))
    return false;
  cudaFuncSetAttribute(gram_f16s_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemF16);
  const int64_t blocks = nseg * (int64_t)ntiles;
  if (blocks > 0)
    gram_f16s_kernel<<<(unsigned)blocks, kThreads, kSmemF16, s>>>(mh, ml, unscale, group_rows, segs, tiles128, ntiles,
                                                                   kp, part);
  return true;
}

}  // namespace cvg
