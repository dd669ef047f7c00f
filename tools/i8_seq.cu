// The int8 Gram's MMA sequence on resident shared-memory operands (no TMA, no drain): how close does the
// 22-pair slice schedule of k_gram_i8.cu get to the issue-loop peak of tools/i8_peak.cu, and which part of
// the schedule (run merging, the A collector, the swizzle width) costs what.  One CTA per SM, one elected
// thread issues; useful ops = 22 pairs x 2 x 128 x 64 x 32 per K = 32 sub-step.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_seq tools/i8_seq.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

// K-major, rows of RB bytes: SW64 (RB = 64, 8-row atoms of 512 B) or SW128 (RB = 128, atoms of 1024 B)
template <int RB>
__device__ __forceinline__ uint64_t desc(uint32_t a) {
  return ((uint64_t)(a >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(8 * RB >> 4) << 32) | (1ull << 46) |
         ((RB == 128 ? 2ull : 4ull) << 61);
}

template <int N, int CU>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
#define I8(Q)                                                                                                         \
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8" Q " [%0], %1, %2, %3, p;\n}\n" \
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc))
  if constexpr (CU == 1) I8(".collector::a::fill");
  else if constexpr (CU == 2) I8(".collector::a::use");
  else if constexpr (CU == 3) I8(".collector::a::lastuse");
  else I8("");
#undef I8
}

// one K = 32 sub-step of the S = 6 schedule.  a/b: descriptors of slice 0; as/bs: slice strides (16 B units).
template <int V>
__device__ __forceinline__ void substep(uint32_t d, uint64_t a, uint64_t as, uint64_t b, uint64_t bs) {
  auto acc = [&](int L) { return d + (uint32_t)(64 * L); };
  constexpr bool C = V == 0 || V == 5;
  if constexpr (V == 0 || V == 1 || V == 5) {  // merged runs (k_gram_i8.cu)
    mma<256, C ? 1 : 0>(acc(0), a, b, 1);
    mma<128, C ? 3 : 0>(acc(4), a, b + 4 * bs, 1);
    mma<256, C ? 1 : 0>(acc(1), a + as, b, 1);
    mma<64, C ? 3 : 0>(acc(5), a + as, b + 4 * bs, 1);
    mma<256, 0>(acc(2), a + 2 * as, b, 1);
    mma<256, 0>(acc(3), a + 3 * as, b, 1);
    mma<128, 0>(acc(4), a + 4 * as, b, 1);
    mma<64, 0>(acc(5), a + 5 * as, b, 1);
  } else if constexpr (V == 2 || V == 3) {  // one N = 64 MMA per pair
#pragma unroll
    for (int t = 0; t < 6; ++t)
#pragma unroll
      for (int u = 0; u + t < 6; ++u) {
        const uint64_t aa = a + t * as, bb = b + u * bs;
        if (V == 3 && 6 - t > 1)
          (u == 0 ? mma<64, 1>(acc(t + u), aa, bb, 1) : u + t == 5 ? mma<64, 3>(acc(t + u), aa, bb, 1)
                                                                     : mma<64, 2>(acc(t + u), aa, bb, 1));
        else
          mma<64, 0>(acc(t + u), aa, bb, 1);
      }
    mma<64, 0>(acc(6), a + 3 * as, b + 3 * bs, 1);
  } else if constexpr (V == 4) {  // the same 1408 columns as N = 256 / 128 MMAs only
#pragma unroll
    for (int t = 0; t < 5; ++t) mma<256, 0>(acc(t % 2), a + t * as, b, 1);
    mma<128, 0>(acc(4), a + 5 * as, b, 1);
  }
}

// SPIN: 0 the other warps idle at the closing __syncthreads; 1 eight warps spin on the final mbarrier with
// try_wait (as the Gram's drain warps do on acc_full); 2 the same with a __nanosleep(SLEEP) backoff
template <int V, int RB, int CM = 0, bool WAITLAG = false, int SPIN = 0, int SLEEP = 0, bool RND = false>
__global__ void __launch_bounds__(320, 1) seq_loop(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar, ring[3];
  __shared__ uint32_t tbase;
  constexpr int kA = 128 * RB, kB = 64 * RB;
  // operand bytes: a fixed small pattern, or (RND) uniformly random bytes like real digit slices
  for (int i = threadIdx.x; i < 6 * (kA + kB) / 4; i += blockDim.x) {
    uint32_t h = (uint32_t)i * 2654435761u + blockIdx.x * 97u;
    h ^= h >> 15;
    h *= 2246822519u;
    h ^= h >> 13;
    ((int*)sm)[i] = RND ? (int)h : 0x01010101 * (i & 3);
  }
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    for (int i = 0; i < 3; ++i) asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&ring[i])));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t d = tbase;
  if (threadIdx.x == 0) {
    const uint64_t a = desc<RB>(smem_u32(sm)), b = desc<RB>(smem_u32(sm + 6 * kA));
    for (int it = 0; it < iters; ++it) {
#pragma unroll
      for (int k = 0; k < RB / 32; ++k) substep<V % 10>(d, a + 2 * k, kA >> 4, b + 2 * k, kB >> 4);
      if (CM > 0 && it % CM == CM - 1) {  // a commit per CM iterations (the kernel: one per 64-row stage)
        const int g = it / CM, s = g % 3;
        asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(
                         smem_u32(&ring[s]))
                     : "memory");
        if (WAITLAG && g >= 2) {  // like the ring: the group two back must be done before the next is issued
          const int s2 = (g - 2) % 3;
          const uint32_t ph = (uint32_t)((g - 2) / 3) & 1u;
          asm volatile("{\n.reg .pred P;\nW2:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], %1;\n@!P bra W2;\n}\n"
                       ::"r"(smem_u32(&ring[s2])), "r"(ph) : "memory");
        }
      }
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n"
                 ::"r"(smem_u32(&bar)) : "memory");
  } else if (SPIN > 0 && threadIdx.x >= 64) {
    for (;;) {
      uint32_t ok;
      asm volatile("{\n.reg .pred P;\nmbarrier.try_wait.parity.shared::cta.b64 P, [%1], 0;\nselp.b32 %0, 1, 0, P;\n}\n"
                   : "=r"(ok) : "r"(smem_u32(&bar)) : "memory");
      if (ok) break;
      if (SPIN == 2) __nanosleep(SLEEP);
    }
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(d));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (v == 0x7fffffff) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;\n" ::"r"(d));
  }
}

template <int V, int RB, int CM = 0, bool WAITLAG = false, int SPIN = 0, int SLEEP = 0, bool RND = false>
void run(const char* name, int sms, int iters) {
  const int smem = 6 * (128 + 64) * RB + 1024;
  cudaFuncSetAttribute(seq_loop<V, RB, CM, WAITLAG, SPIN, SLEEP, RND>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* sink;
  cudaMalloc(&sink, 4);
  seq_loop<V, RB, CM, WAITLAG, SPIN, SLEEP, RND><<<sms, 320, smem>>>(iters / 10, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 3; ++r) {
    cudaEventRecord(e0);
    seq_loop<V, RB, CM, WAITLAG, SPIN, SLEEP, RND><<<sms, 320, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double ops = 22.0 * 2 * 128 * 64 * 32 * (RB / 32) * (double)iters * sms;
  printf("{\"variant\": \"%s\", \"row_bytes\": %d, \"ms\": %.4f, \"useful_tops\": %.1f}\n", name, RB, best,
         ops / (best * 1e-3) / 1e12);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  run<0, 64, 1, true>("ring, pattern data", sms, 20000);
  run<0, 64, 1, true, 0, 0, true>("ring, random data", sms, 20000);
  run<0, 64, 1, true, 0, 0, true>("ring, random data (again)", sms, 60000);
  run<4, 64, 0, false, 0, 0, true>("5 x N=256 + N=128, random data", sms, 20000);
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
