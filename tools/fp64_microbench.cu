// FP64 pipe microbenchmark for B200 (sm_100a): DMMA.8x8x4 vs DFMA throughput.
// Used once to pick the Gram kernel's math path and to set the FP64 roofline
// denominator; results are committed under profiles/.
#include <cstdio>
#include <cuda_runtime.h>

template <int CHAINS>
__global__ void dmma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = seed - threadIdx.x * 1e-3;
  double c[CHAINS][2];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) { c[i][0] = 0; c[i][1] = 0; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i)
      asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
                   : "+d"(c[i][0]), "+d"(c[i][1]) : "d"(a), "d"(b));
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i][0] + c[i][1];
  if (s == 12345.678) out[0] = s;
}

template <int CHAINS>
__global__ void dfma_loop(double* out, int iters, double seed) {
  double a = seed + threadIdx.x * 1e-3, b = 1.0 - 1e-9 * threadIdx.x;
  double c[CHAINS];
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) c[i] = i;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int i = 0; i < CHAINS; ++i) c[i] = fma(c[i], b, a);
  }
  double s = 0;
#pragma unroll
  for (int i = 0; i < CHAINS; ++i) s += c[i];
  if (s == 12345.678) out[0] = s;
}

template <typename F>
float time_it(F f) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  f();  // warm
  cudaDeviceSynchronize();
  cudaEventRecord(e0);
  f();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  return ms;
}

int main() {
  double* out; cudaMalloc(&out, 8);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int iters = 20000;
  for (int warps : {4, 8, 16, 32}) {
    for (int blocks_per_sm : {1, 2}) {
      int grid = sms * blocks_per_sm, block = 32 * warps;
      float ms = time_it([&] { dmma_loop<8><<<grid, block>>>(out, iters, 1.0); });
      double flops = 2.0 * 256 * 8 * (double)iters * grid * warps;
      printf("DMMA chains=8 warps=%d bps=%d: %.3f ms  %.2f TFLOP/s\n", warps, blocks_per_sm, ms, flops / ms / 1e9);
    }
  }
  for (int warps : {8, 16, 32}) {
    int grid = sms * 2, block = 32 * warps;
    float ms = time_it([&] { dfma_loop<8><<<grid, block>>>(out, iters, 1.0); });
    double flops = 2.0 * 8 * (double)iters * grid * block;
    printf("DFMA chains=8 warps=%d bps=2: %.3f ms  %.2f TFLOP/s\n", warps, ms, flops / ms / 1e9);
  }
  cudaError_t e = cudaGetLastError();
  printf("status: %s\n", cudaGetErrorString(e));
  return 0;
}
