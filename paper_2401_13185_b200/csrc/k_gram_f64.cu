// K2: segmented fold Gram in fp64 on the B200 FP64 tensor path (DMMA.8x8x4).
//
// For every segment s (<= kChunkRows rows of one fold, contiguous in Z) and
// every upper tile (ti <= tj) of the kp x kp Gram:
//     part[s][ti*64 + i][tj*64 + j] = sum_{r in s} Z[r][ti*64 + i] * Z[r][tj*64 + j]
// This is each validation partition's X_pᵀ[X_p | Y_p | 1] — the reference's
// per-fold `xv.transpose() * xv / * yv` (fast.hpp:91-92) plus its colwise sums
// and squares (fast.hpp:95-96, 110-119) — and the whole-data products of
// precompute_global (fast.hpp:23-24) are the fixed-order sum over folds (K4),
// so the data is contracted exactly once.  Symmetry: only ti <= tj tiles.
//
// Tensor path: sm_100 has no fp64 tcgen05 kind; `mma.sync.m8n8k4.f64` lowers to
// SASS DMMA.8x8x4, measured at 37.1 TFLOP/s on this B200 (profiles/r01_fp64_peaks.txt).
// CTA = 64x64 output tile, 8 warps (2 x 4), warp tile 32x16 = 4x2 DMMA tiles;
// a diagonal tile instead deals its 36 upper 8x8 blocks round-robin to the 8
// warps (no DMMA below the diagonal: c1 Gram 8.81 -> 8.31 ms, c4 36.4 -> 32.8).
// Operands: 32-row x 64-col slabs staged by cp.async (16 B) into a 3-stage ring
// synchronised by mbarriers (see gram_f64_kernel);
// the smem row pitch of 68 doubles makes the DMMA fragment loads conflict-free
// (lanes (g, t) read [t][g]: bank = 2(68t + g) mod 32 covers all 32 banks).
#include "cvg_internal.cuh"

namespace cvg {
namespace {

constexpr int BT = kTile;      // 64
constexpr int KC = kRowStep;   // 32 rows per stage
constexpr int STAGES = 3;
constexpr int LDS = BT + 4;    // smem pitch in doubles
constexpr int NT = 256;
constexpr int kSlab = KC * LDS;                 // doubles per operand slab
constexpr int kSmemBytes = STAGES * 2 * kSlab * 8;  // 104,448 B -> 2 CTAs / SM

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned s = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"(s), "l"(gmem));
}

__device__ __forceinline__ void dmma(double (&c)[2], double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};\n"
               : "+d"(c[0]), "+d"(c[1])
               : "d"(a), "d"(b));
}

// Pipeline: per-stage mbarriers instead of a CTA barrier per step.  Every
// thread's cp.asyncs for a stage arrive on full[stage] when they land
// (cp.async.mbarrier.arrive.noinc), each warp arrives on empty[stage] after its
// DMMAs, and a stage is refilled only once all 8 warps have left it, so warps
// drift up to one stage apart instead of re-aligning at every 32-row step
// (measured against __syncthreads per step: c1 Gram 9.13 -> 8.99 ms, c2 13.35
// -> 12.99, c4 36.77 -> 36.40; 6 stages of 16 rows were slower than 3 of 32).
__device__ __forceinline__ uint32_t smem_addr(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_wait_parity(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred P1;\nWAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
      "@P1 bra DONE_%=;\nbra WAIT_%=;\nDONE_%=:\n}\n" ::"r"(smem_addr(bar)),
      "r"(parity)
      : "memory");
}

// Diagonal tiles: the 36 upper 8x8 blocks (bi <= bj) of the 64x64 tile, dealt round-robin to the 8 warps
// (5 or 4 each) so no DMMA is spent below the diagonal.  Packed as bi * 8 + bj.
__constant__ unsigned char kDiagBlocks[40] = {
    0,  1,  2,  3,  4,  5,  6,  7,  9,  10, 11, 12, 13, 14, 15, 18, 19, 20, 21, 22,
    23, 27, 28, 29, 30, 31, 36, 37, 38, 39, 45, 46, 47, 54, 55, 63, 0,  0,  0,  0};

// Grid order: segment-major, tile fastest, so the CTAs of one segment run
// together and share its rows in L2 (ncu, c1: 4.9 GB DRAM for 4.1 GB of Z).
// (Running every diagonal tile after all off-diagonal ones, to end on cheap
// CTAs, saved nothing and re-read every segment: 8.8 GB.)
template <int KCm, int STm>
__global__ void __launch_bounds__(NT, 2)
    gram_f64_kernel(const double* __restrict__ z, int64_t kp, int64_t zrows, const GramTask* __restrict__ segs,
                    int64_t nseg, const int2* __restrict__ tiles, int ntiles, double* __restrict__ part) {
  constexpr int kSl = KCm * LDS;  // doubles per operand slab
  extern __shared__ __align__(128) double smem[];
  __shared__ __align__(8) uint64_t full[STm], empty[STm];
  const int seg = (int)(blockIdx.x / ntiles);
  const int2 tile = tiles[blockIdx.x - (int64_t)seg * ntiles];
  const int ti = tile.x, tj = tile.y;
  const bool diag = ti == tj;
  CVG_DCHECK(seg >= 0 && seg < nseg);
  const GramTask task = segs[seg];
  CVG_DCHECK(task.zrow >= 0 && task.rows % KCm == 0 && task.zrow + task.rows <= zrows);
  CVG_DCHECK(tile.x >= 0 && tile.x <= tile.y && (int64_t)(tile.y + 1) * BT <= kp);
  const double* zb = z + task.zrow * kp;
  const int nsteps = (int)(task.rows / KCm);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int g = lane >> 2, t4 = lane & 3;
  const int wi = (warp >> 2) * 32, wj = (warp & 3) * 16;
  // diagonal tiles: this warp's upper blocks b = warp, warp + 8, ... (< 36)
  const int nblk = diag ? (warp < 4 ? 5 : 4) : 0;
  int boff_a[5], boff_b[5];
#pragma unroll
  for (int u = 0; u < 5; ++u) {
    const int code = kDiagBlocks[u < nblk ? warp + 8 * u : 0];
    boff_a[u] = (code >> 3) * 8 + g;
    boff_b[u] = (code & 7) * 8 + g;
  }
  if (tid == 0) {
    for (int s = 0; s < STm; ++s) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&full[s])), "r"(NT));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_addr(&empty[s])), "r"(NT / 32));
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  __syncthreads();

  auto load_stage = [&](int step, int buf) {
    const double* src = zb + (int64_t)step * KCm * kp;
    double* dA = smem + buf * 2 * kSl;
    double* dB = dA + kSl;
#pragma unroll
    for (int q = 0; q < KCm * 32 / NT; ++q) {  // KCm rows x 32 16-byte chunks
      const int idx = tid + q * NT;
      const int r = idx >> 5, c = (idx & 31) * 2;
      cp_async16(dA + r * LDS + c, src + (int64_t)r * kp + ti * BT + c);
      if (!diag) cp_async16(dB + r * LDS + c, src + (int64_t)r * kp + tj * BT + c);
    }
    asm volatile("cp.async.mbarrier.arrive.noinc.shared::cta.b64 [%0];\n" ::"r"(smem_addr(&full[buf])) : "memory");
  };

  double acc[4][2][2];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 2; ++b) acc[a][b][0] = acc[a][b][1] = 0.0;
#pragma unroll
  for (int s = 0; s < STm - 1; ++s)
    if (s < nsteps) load_stage(s, s);
  for (int step = 0; step < nsteps; ++step) {
    const int buf = step % STm;
    mbar_wait_parity(&full[buf], (uint32_t)(step / STm) & 1u);
    if (diag) {
      const double* sA = smem + buf * 2 * kSl;
#pragma unroll
      for (int kk = 0; kk < KCm; kk += 4) {
        const double* pr = sA + (kk + t4) * LDS;
#pragma unroll
        for (int u = 0; u < 5; ++u)
          if (u < nblk) dmma(acc[u >> 1][u & 1], pr[boff_a[u]], pr[boff_b[u]]);
      }
    } else {
      const double* sA = smem + buf * 2 * kSl;
      const double* sB = sA + kSl;
#pragma unroll
      for (int kk = 0; kk < KCm; kk += 4) {
        const double* pa = sA + (kk + t4) * LDS + wi + g;
        const double* pb = sB + (kk + t4) * LDS + wj + g;
        double a[4], b[2];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi) a[mi] = pa[mi * 8];
#pragma unroll
        for (int ni = 0; ni < 2; ++ni) b[ni] = pb[ni * 8];
#pragma unroll
        for (int mi = 0; mi < 4; ++mi)
#pragma unroll
          for (int ni = 0; ni < 2; ++ni) dmma(acc[mi][ni], a[mi], b[ni]);
      }
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_addr(&empty[buf])) : "memory");
    const int nxt = step + STm - 1;
    if (nxt < nsteps) {
      const int nb = nxt % STm;  // last held step nxt - STm = step - 1
      if (nxt >= STm) mbar_wait_parity(&empty[nb], (uint32_t)((nxt - STm) / STm) & 1u);
      load_stage(nxt, nb);
    }
  }

  double* out = part + (int64_t)seg * kp * kp;
  if (diag) {
#pragma unroll
    for (int u = 0; u < 5; ++u)
      if (u < nblk) {
        const int64_t row = (int64_t)ti * BT + boff_a[u];
        const int64_t col = (int64_t)tj * BT + (boff_b[u] - g) + 2 * t4;
        *reinterpret_cast<double2*>(out + row * kp + col) = make_double2(acc[u >> 1][u & 1][0], acc[u >> 1][u & 1][1]);
      }
    // strictly-lower blocks are never read downstream; zero them so every partial is fully defined
    for (int lb = warp; lb < 64; lb += 8) {
      const int bi = lb >> 3, bj = lb & 7;
      if (bi <= bj) continue;
      const int64_t row = (int64_t)ti * BT + bi * 8 + g, col = (int64_t)tj * BT + bj * 8 + 2 * t4;
      *reinterpret_cast<double2*>(out + row * kp + col) = make_double2(0.0, 0.0);
    }
    return;
  }
#pragma unroll
  for (int mi = 0; mi < 4; ++mi)
#pragma unroll
    for (int ni = 0; ni < 2; ++ni) {
      const int64_t row = (int64_t)ti * BT + wi + mi * 8 + g;
      const int64_t col = (int64_t)tj * BT + wj + ni * 8 + 2 * t4;
      *reinterpret_cast<double2*>(out + row * kp + col) = make_double2(acc[mi][ni][0], acc[mi][ni][1]);
    }
}

}  // namespace

void launch_gram_f64(const double* z, int64_t kp, int64_t zrows, const GramTask* segs, int64_t nseg,
                     const int2* tiles, int ntiles, double* part, cudaStream_t s) {
  // per device (a process may drive several GPUs), so set it on every launch: a host-side call
  cudaFuncSetAttribute(gram_f64_kernel<KC, STAGES>, cudaFuncAttributeMaxDynamicSharedMemorySize, kSmemBytes);
  const int64_t blocks = nseg * (int64_t)ntiles;
  if (blocks <= 0) return;
  gram_f64_kernel<KC, STAGES><<<(unsigned)blocks, NT, kSmemBytes, s>>>(z, kp, zrows, segs, nseg, tiles, ntiles,
                                                                      part);
}

}  // namespace cvg
