// Microbenchmark: shared-memory update throughput for random addresses
// (decides the counting-table design).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

template <int MODE>
__global__ void __launch_bounds__(512, 1) kern(int iters, uint32_t* out) {
  extern __shared__ uint32_t w[];           // 32768 words = 128 KiB
  for (int i = threadIdx.x; i < 32768; i += 512) w[i] = 0;
  __syncthreads();
  uint32_t s = hsh(blockIdx.x * 512 + threadIdx.x);
  uint32_t acc = 0;
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int u = 0; u < 8; ++u) {
      s = s * 1664525u + 1013904223u;
      const uint32_t x = (s >> 7) & 0x1FFFFFu;   // bit index in 2^21 bits (256 KiB) -> mask to 128 KiB
      const uint32_t b = x & 0xFFFFFu;           // 1M bits = 128 KiB
      if (MODE == 0) atomicOr(&w[b >> 5], 1u << (b & 31));                 // RED.OR
      if (MODE == 1) atomicAdd(&w[(b >> 3) & 32767], 1u << (8 * (b & 3)));  // RED.ADD byte lane
      if (MODE == 2) { uint8_t* p = (uint8_t*)w + ((b >> 3) & 131071); *p = *p + 1; }  // LDS/STS
      if (MODE == 3) acc += atomicAdd(&w[(b >> 3) & 32767], 1u);           // ATOMS with return
    }
  }
  __syncthreads();
  if (threadIdx.x == 0) out[blockIdx.x] = w[blockIdx.x & 32767] + acc;
}

int main() {
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint32_t* out; cudaMalloc(&out, 4 * sms);
  const int iters = 2000;
  const char* names[] = {"atomicOr (RED.OR)", "atomicAdd byte-lane (RED.ADD)", "plain byte RMW (LDS+STS)", "atomicAdd with return"};
  cudaFuncSetAttribute(kern<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(kern<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(kern<2>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  cudaFuncSetAttribute(kern<3>, cudaFuncAttributeMaxDynamicSharedMemorySize, 131072);
  for (int m = 0; m < 4; ++m) {
    cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
    for (int rep = 0; rep < 2; ++rep) {
      cudaEventRecord(a);
      if (m == 0) kern<0><<<sms, 512, 131072>>>(iters, out);
      if (m == 1) kern<1><<<sms, 512, 131072>>>(iters, out);
      if (m == 2) kern<2><<<sms, 512, 131072>>>(iters, out);
      if (m == 3) kern<3><<<sms, 512, 131072>>>(iters, out);
      cudaEventRecord(b); cudaEventSynchronize(b);
    }
    float ms; cudaEventElapsedTime(&ms, a, b);
    double ops = (double)sms * 512 * iters * 8;
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    printf("%-34s %8.3f ms  %7.2f Gop/s  %.3f cyc/op/SM (at %d MHz)\n", names[m], ms, ops / ms / 1e6,
           (ms * 1e-3 * clk * 1e3) / (ops / sms), clk / 1000);
  }
  printf("%s\n", cudaGetErrorString(cudaGetLastError()));
  return 0;
}
