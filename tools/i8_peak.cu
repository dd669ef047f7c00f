// int8 tensor-core (tcgen05.mma kind::i8) issue-loop peak on B200 (sm_100a): the
// roofline denominator for the int8-slice fp64 Gram (k_gram_i8.cu).  One CTA per SM,
// one elected thread issues back-to-back M = 128 MMAs (N = 64 .. 256, K = 32) from
// resident shared-memory operands into TMEM, so only the tensor pipe is measured.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/i8_peak tools/i8_peak.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t desc_sw64(const void* tile) {  // K-major SWIZZLE_64B, 8-row atoms of 512 B
  const uint64_t a = smem_u32(tile);
  return ((a >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(512 >> 4) << 32) | (1ull << 46) | (4ull << 61);
}

template <int N>
__device__ __forceinline__ void mma(uint32_t d, uint64_t a, uint64_t b, uint32_t acc) {
  constexpr uint32_t idesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  asm volatile("{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\ntcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n}\n"
               ::"r"(d), "l"(a), "l"(b), "r"(idesc), "r"(acc));
}

template <int N>
__global__ void __launch_bounds__(128, 1) i8_loop(int iters, int* sink) {
  extern __shared__ __align__(1024) uint8_t raw[];
  uint8_t* sm = (uint8_t*)(((uintptr_t)raw + 1023) & ~(uintptr_t)1023);
  __shared__ __align__(8) uint64_t bar;
  __shared__ uint32_t tbase;
  for (int i = threadIdx.x; i < (128 + 256) * 64 / 4; i += blockDim.x) ((int*)sm)[i] = 0x01010101 * (i & 3);
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  if (threadIdx.x < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;\n" ::"r"(smem_u32(&tbase)));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  const uint32_t d = tbase;
  if (threadIdx.x == 0) {
    const uint64_t a = desc_sw64(sm), b = desc_sw64(sm + 128 * 64);
    for (int it = 0; it < iters; ++it) {
      mma<N>(d, a, b, it > 0);
      mma<N>(d, a + 2, b + 2, 1u);
    }
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&bar))
                 : "memory");
    asm volatile("{\n.reg .pred P;\nW:\nmbarrier.try_wait.parity.shared::cta.b64 P, [%0], 0;\n@!P bra W;\n}\n"
                 ::"r"(smem_u32(&bar)) : "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (threadIdx.x < 32) {
    uint32_t v;
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x1.b32 {%0}, [%1];\n" : "=r"(v) : "r"(d));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    if (v == 0x7fffffff) sink[0] = v;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;\n" ::"r"(d));
  }
}

template <int N>
void run(int sms, int iters) {
  const int smem = (128 + 256) * 64 + 1024;
  cudaFuncSetAttribute(i8_loop<N>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
  int* sink;
  cudaMalloc(&sink, 4);
  i8_loop<N><<<sms, 128, smem>>>(iters / 10, sink);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    cudaEventRecord(e0);
    i8_loop<N><<<sms, 128, smem>>>(iters, sink);
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    best = ms < best ? ms : best;
  }
  const double ops = 2.0 * 128 * N * 64 * (double)iters * sms;  // two K = 32 MMAs per iteration
  printf("{\"kind\": \"i8\", \"M\": 128, \"N\": %d, \"ctas\": %d, \"iters\": %d, \"ms\": %.4f, \"tops\": %.1f}\n", N, sms,
         iters, best, ops / (best * 1e-3) / 1e12);
  cudaFree(sink);
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  for (int i = 0; i < 2; ++i) {
    run<64>(sms, 200000);
    run<128>(sms, 100000);
    run<256>(sms, 50000);
  }
  printf("status: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  return 0;
}
