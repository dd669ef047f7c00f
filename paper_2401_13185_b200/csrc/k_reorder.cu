// K1: build the fold-bucketed, shifted Gram operand Z (HBM-bound).
//
// Z[r] = [ x[src] - c | y[src] - d | 1 | 0 ... 0 ]   (kp columns, fp64)
// for each Z row r with source row src = src_row[r]; padding rows (src < 0) are
// all zero, including the ones column, so they contribute nothing.
//
// Replaces the per-fold gather_rows copies (partition.hpp:85-90 via
// fast.hpp:84-85) and the separate colwise sums (fast.hpp:25-34, 95-96,
// 110-119): the ones column turns column sums into Gram entries.  The shift
// (c | d) removes |mean| >> std conditioning from every downdate (SURVEY.md §7
// hard part 1) and is undone exactly in the epilogue.
//
// One warp per Z row; each lane streams 8-byte elements (x rows are not
// 16-byte aligned for odd k) with four loads in flight.  Algorithmic bytes per
// row: (k+m)*elt read + kp*8 written.  Also flags non-finite inputs
// (DatasetPair's allFinite check, core.hpp:43-44).
#include "cvg_internal.cuh"

namespace cvg {
namespace {

template <typename T>
__global__ void __launch_bounds__(256) reorder_kernel(const T* __restrict__ x, int64_t ldx, const T* __restrict__ y,
                                                      int64_t ldy, int64_t k, int64_t m,
                                                      const int64_t* __restrict__ src_row, int64_t zrows, int64_t kp,
                                                      int64_t c_begin, int64_t c_end, int64_t nsrc,
                                                      const double* __restrict__ shift, double* __restrict__ z,
                                                      int* __restrict__ nonfinite) {
  const int lane = threadIdx.x & 31;
  const int64_t warps = (int64_t(gridDim.x) * blockDim.x) >> 5;
  const int64_t w = k + m;
  bool bad = false;
  for (int64_t r = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) >> 5; r < zrows; r += warps) {
    const int64_t src = src_row[r];
    CVG_DCHECK(src < nsrc && src >= -1);
    CVG_DCHECK(c_begin >= 0 && c_end <= kp && c_begin % 64 == 0);
    double* zr = z + r * kp;
    if (src < 0) {
      for (int64_t c = c_begin + lane; c < c_end; c += 32) zr[c] = 0.0;
      continue;
    }
    const T* xr = x + src * ldx;
    const T* yr = y + src * ldy;
    for (int64_t c0 = c_begin; c0 < c_end; c0 += 128) {
      double v[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        double raw = 0.0;
        if (c < k)
          raw = (double)__ldg(xr + c);
        else if (c < w)
          raw = (double)__ldg(yr + (c - k));
        v[u] = raw;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t c = c0 + u * 32 + lane;
        if (c >= c_end) break;
        double out;
        if (c < w) {
          bad |= !isfinite(v[u]);
          out = __dsub_rn(v[u], shift[c]);
        } else {
          out = (c == w) ? 1.0 : 0.0;
        }
        zr[c] = out;
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
}

template <typename T>
__global__ void shift_row0_kernel(const T* __restrict__ x, const T* __restrict__ y, int64_t k, int64_t m,
                                  double* __restrict__ shift) {
  const int64_t c = int64_t(blockIdx.x) * blockDim.x + threadIdx.x;
  if (c < k)
    shift[c] = (double)x[c];
  else if (c < k + m)
    shift[c] = (double)y[c - k];
}

}  // namespace

void launch_reorder(int dtype, const void* x, int64_t ldx, const void* y, int64_t ldy, int64_t k, int64_t m,
                    const int64_t* src_row, int64_t zrows, int64_t kp, int64_t c_begin, int64_t c_end, int64_t nsrc,
                    const double* shift, double* z, int* nonfinite, cudaStream_t s) {
  const int threads = 256;
  int64_t blocks = (zrows * 32 + threads - 1) / threads;
  if (blocks > 148 * 16) blocks = 148 * 16;  // grid-stride: 16 CTAs (128 rows in flight) per SM
  if (blocks < 1) blocks = 1;
  if (dtype == 0)
    reorder_kernel<double><<<(unsigned)blocks, threads, 0, s>>>((const double*)x, ldx, (const double*)y, ldy, k, m,
                                                                src_row, zrows, kp, c_begin, c_end, nsrc, shift, z,
                                                                nonfinite);
  else
    reorder_kernel<float><<<(unsigned)blocks, threads, 0, s>>>((const float*)x, ldx, (const float*)y, ldy, k, m,
                                                               src_row, zrows, kp, c_begin, c_end, nsrc, shift, z,
                                                               nonfinite);
}

void launch_shift_from_row0(int dtype, const void* x, const void* y, int64_t k, int64_t m, double* shift,
                            cudaStream_t s) {
  const int threads = 256;
  const unsigned blocks = (unsigned)((k + m + threads - 1) / threads);
  if (dtype == 0)
    shift_row0_kernel<double><<<blocks, threads, 0, s>>>((const double*)x, (const double*)y, k, m, shift);
  else
    shift_row0_kernel<float><<<blocks, threads, 0, s>>>((const float*)x, (const float*)y, k, m, shift);
}

}  // namespace cvg
