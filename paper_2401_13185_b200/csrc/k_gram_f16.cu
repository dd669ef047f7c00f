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
// One CTA per G bucketed rows; warp w owns the 8 columns c0 + 8w .. + 7 of every 64-column chunk over all G rows
// and runs on its own (the group's per-column exponent is a reduction within the warp), so the warps drift past
// one another's load latencies with no CTA barrier after the row indices are in.  Lane (rq, h) = (lane >> 1,
// lane & 1) holds columns 4h .. 4h + 3 of the row pairs rp = 16 i + rq (rows 2 rp, 2 rp + 1): a warp load reads
// 16 rows' 32-byte segments (whole sectors).  Each (hi, lo) row pair is one 32-bit word of the warp's shared
// tile [block][col][64 rows] in the SWIZZLE_128B layout (16-byte chunk (word >> 2) ^ col): the 32 lanes' words
// land in 32 distinct banks, and the tile leaves by one TMA tensor store per plane (4 KB at G = 256).
constexpr int kK1hThreads = 256;
constexpr int kK1hCols = 64;

template <int G>
constexpr int k1h_smem_bytes() {  // per warp: hi and lo planes of (G / 64) x 8 columns x 128 B
  return 8 * 2 * (G / 64) * 1024 + 1024;
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

__device__ __forceinline__ void tma_store_3d(const CUtensorMap* map, const void* src, int c0, int c1, int c2) {
  asm volatile("cp.async.bulk.tensor.3d.global.shared::cta.bulk_group [%0, {%2, %3, %4}], [%1];\n" ::"l"(map),
               "r"(smem_u32(src)), "r"(c0), "r"(c1), "r"(c2)
               : "memory");
}

template <typename T, int G>
__global__ void __launch_bounds__(kK1hThreads, 2) reorder_split_h_kernel(
    const __grid_constant__ CUtensorMap map_hi, const __grid_constant__ CUtensorMap map_lo, const T* __restrict__ x,
    int64_t ldx, const T* __restrict__ y, int64_t ldy, int64_t k, int64_t m, const int64_t* __restrict__ src_row,
    int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc, const double* __restrict__ shift,
    float* __restrict__ unscale, int* __restrict__ nonfinite) {
  // map_hi / map_lo: Zh planes as {64 rows, kp, zrows / 64} halves, box {64, 8, G / 64}, SWIZZLE_128B.
  constexpr int NB = G / 64;  // 64-row blocks per group
  constexpr int NI = G / 32;  // row-pair batches per thread
  extern __shared__ uint8_t k1h_raw[];
  uint8_t* tiles = reinterpret_cast<uint8_t*>((reinterpret_cast<uintptr_t>(k1h_raw) + 1023) & ~uintptr_t(1023));
  __shared__ int64_t s_src[G];
  const int64_t grp = blockIdx.x;
  const int t = threadIdx.x, lane = t & 31, w = t >> 5;
  const int h = lane & 1, rq = lane >> 1;
  const int64_t wd = k + m;
  CVG_DCHECK(c_begin >= 0 && c_end <= kp && c_begin % kK1hCols == 0 && zrows % G == 0);
  bool real = true;
  for (int i = t; i < G; i += kK1hThreads) {
    const int64_t r = grp * G + i;
    const int64_t src = r < zrows ? src_row[r] : -1;
    CVG_DCHECK(src < nsrc);
    s_src[i] = src;
    real &= src >= 0;
  }
  const bool all_real = __syncthreads_and(real);
  // 16-byte row loads need 16-byte aligned rows
  const bool vec_ok = (ldx * (int64_t)sizeof(T)) % 16 == 0 && (reinterpret_cast<uintptr_t>(x) & 15) == 0;
  uint8_t* plane_hi = tiles + w * (2 * NB * 1024);
  uint8_t* plane_lo = plane_hi + NB * 1024;
  float nan_acc = 0.f;  // v * 0 is NaN exactly when v is not finite
  bool too_big = false;
  for (int64_t c0 = c_begin; c0 < c_end; c0 += kK1hCols) {
    const int64_t cw = c0 + 8 * w;  // the warp's columns
    const int64_t cb = cw + 4 * h;  // this thread's
    // Fast warps (every column an X column, every row real, aligned rows): no per-element checks.
    const bool fast = all_real && vec_ok && cw + 8 <= k;
    float z[NI][2][4];
    if (fast) {
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int p = 0; p < 2; ++p) load4(x + (int64_t)(int32_t)s_src[32 * i + 2 * rq + p] * ldx + cb, z[i][p]);
    } else {
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          const int64_t src = s_src[32 * i + 2 * rq + p];
#pragma unroll
          for (int e = 0; e < 4; ++e) {
            const int64_t ce = cb + e;
            float val = 0.f;
            if (src >= 0) {
              if (ce < k)
                val = (float)__ldg(x + src * ldx + ce);
              else if (ce < wd)
                val = (float)__ldg(y + src * ldy + (ce - k));
              else if (ce == wd)
                val = 1.f;  // ones column: column sums ride in the Gram
            }
            z[i][p][e] = val;
          }
        }
    }
    // shift; per-column max |z| over the group's rows (this thread's, then the 16 lanes of its column half)
    float sc[4];
#pragma unroll
    for (int e = 0; e < 4; ++e) {
      const int64_t ce = cb + e;
      const float sh = ce < wd ? (float)__ldg(shift + ce) : 0.f;  // ones / padding columns: no shift
      float mx = 0.f;
#pragma unroll
      for (int i = 0; i < NI; ++i)
#pragma unroll
        for (int p = 0; p < 2; ++p) {
          nan_acc = fmaf(z[i][p][e], 0.f, nan_acc);
          const bool shifted = fast || (s_src[32 * i + 2 * rq + p] >= 0 && ce < wd);
          if (shifted) z[i][p][e] -= sh;
          mx = fmaxf(mx, fabsf(z[i][p][e]));
        }
#pragma unroll
      for (int o = 2; o < 32; o <<= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
      // e: the group's max |z| scaled into [2^14, 2^15); zero / non-finite columns keep e = 0
      int ex = 0;
      if (mx > 0.f && isfinite(mx)) {
        const int be = (int)((__float_as_uint(mx) >> 23) & 0xff);
        ex = 14 - (be == 0 ? -127 : be - 127);
        too_big |= ex < -64;  // |z| >= 2^79: products beyond the fp32 accumulation range
        ex = max(-64, min(64, ex));
      }
      sc[e] = __uint_as_float((uint32_t)(127 + ex) << 23);
      if (rq == 0) unscale[grp * kp + ce] = __uint_as_float((uint32_t)(127 - ex) << 23);
    }
    // this warp's previous TMA stores have finished reading its tile
    if (lane == 0) asm volatile("cp.async.bulk.wait_group.read 0;\n" ::: "memory");
    __syncwarp();
    // scale (exact) and split: hi = fp16_rn(z'), lo = fp16_rn(z' - hi); row pair rp = 16 i + rq is word
    // rp & 31 of block rp >> 5 = i >> 1, line (block, column 4h + e), 16-byte chunk (word >> 2) ^ column
#pragma unroll
    for (int i = 0; i < NI; ++i) {
      const int word = 16 * (i & 1) + rq;
#pragma unroll
      for (int e = 0; e < 4; ++e) {
        const int col = 4 * h + e;
        const float z0 = z[i][0][e] * sc[e], z1 = z[i][1][e] * sc[e];
        const __half2 hi = __floats2half2_rn(z0, z1);
        const float2 hf = __half22float2(hi);
        const __half2 lo = __floats2half2_rn(z0 - hf.x, z1 - hf.y);
        const int off = ((i >> 1) * 8 + col) * 128 + (((word >> 2) ^ col) << 4) + ((word & 3) << 2);
        *reinterpret_cast<uint32_t*>(plane_hi + off) = *reinterpret_cast<const uint32_t*>(&hi);
        *reinterpret_cast<uint32_t*>(plane_lo + off) = *reinterpret_cast<const uint32_t*>(&lo);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    __syncwarp();
    if (lane == 0) {
      tma_store_3d(&map_hi, plane_hi, 0, (int)cw, (int)(grp * NB));
      tma_store_3d(&map_lo, plane_lo, 0, (int)cw, (int)(grp * NB));
      asm volatile("cp.async.bulk.commit_group;\n" ::: "memory");
    }
  }
  if (lane == 0) asm volatile("cp.async.bulk.wait_group 0;\n" ::: "memory");
  // bit 0: a non-finite input; bit 1: a finite magnitude the fp32 accumulation cannot hold
  const unsigned bad = __ballot_sync(0xffffffffu, nan_acc != 0.f), big = __ballot_sync(0xffffffffu, too_big);
  if (lane == 0 && (bad | big)) atomicOr(nonfinite, (bad ? 1 : 0) | (big ? 2 : 0));
}

template <typename T, int G>
bool launch_k1h(const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m, const int64_t* src_row,
                int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc, const double* shift,
                __half* zh_hi, __half* zh_lo, float* unscale, int* nonfinite, cudaStream_t s) {
  CUtensorMap mh, ml;
  if (!make_blocked_map(&mh, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, zh_hi, 2, zrows, kp, 8, G / 64) ||
      !make_blocked_map(&ml, CU_TENSOR_MAP_DATA_TYPE_FLOAT16, zh_lo, 2, zrows, kp, 8, G / 64))
    return false;
  constexpr int smem = k1h_smem_bytes<G>();
  cudaFuncSetAttribute(reorder_split_h_kernel<T, G>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  reorder_split_h_kernel<T, G><<<(unsigned)(zrows / G), kK1hThreads, smem, s>>>(
      mh, ml, (const T*)x, ldx, (const T*)y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, unscale,
      nonfinite);
  return true;
}

}  // namespace

bool launch_reorder_split_h(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                            const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end,
                            int64_t nsrc, const double* shift, int group_rows, void* zh_hi, void* zh_lo,
                            float* unscale, int* nonfinite, cudaStream_t s) {
  if (zrows <= 0 || c_end <= c_begin) return true;
  __half* hi = static_cast<__half*>(zh_hi);
  __half* lo = static_cast<__half*>(zh_lo);
#define CVG_K1H(T, G)                                                                                         \
  return launch_k1h<T, G>(x, ldx, y, ldy, k, m, src_row, zrows, kp, c_begin, c_end, nsrc, shift, hi, lo, unscale, \
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
