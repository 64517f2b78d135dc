// Dependent fp64 add chain over float values in shared memory (the
// k_cluster_sums consumer): (a) LDS -> F2F -> DADD as chain_add compiles,
// (b) a batch converted one iteration ahead so only DADD -> DADD is serial.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/mbc tools/mb_chain_f2f.cu && /tmp/mbc
#include <cstdio>
#include <cuda_runtime.h>
__device__ __forceinline__ double chain_a(double acc, const float* tv, int rr, int st) {
  for (int q = 0; q + 64 <= rr; q += 64) {
    float a[32], b[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) a[u] = tv[(q + u) * st];
#pragma unroll
    for (int u = 0; u < 32; ++u) b[u] = tv[(q + 32 + u) * st];
#pragma unroll
    for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, (double)a[u]);
#pragma unroll
    for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, (double)b[u]);
  }
  return acc;
}
__device__ __forceinline__ double chain_b(double acc, const float* tv, int rr, int st) {
  double cur[16];
#pragma unroll
  for (int u = 0; u < 16; ++u) cur[u] = (double)tv[u * st];
  for (int q = 16; q <= rr; q += 16) {
    float raw[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) raw[u] = q + u < rr ? tv[(q + u) * st] : 0.f;
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, cur[u]);
#pragma unroll
    for (int u = 0; u < 16; ++u) cur[u] = (double)raw[u];
  }
  return acc;
}
template <int M>
__global__ void k(int reps, double* out) {
  __shared__ float tv[1024 * 8];
  for (int i = threadIdx.x; i < 1024 * 8; i += blockDim.x) tv[i] = 1.0f + i * 1e-3f;
  __syncthreads();
  double acc = 0.0;
  if (threadIdx.x < 8)
    for (int r = 0; r < reps; ++r)
      acc = M == 0 ? chain_a(acc, tv + threadIdx.x, 1024, 8) : chain_b(acc, tv + threadIdx.x, 1024, 8);
  out[threadIdx.x] = acc;
}
int main() {
  double* o; cudaMalloc(&o, 8 * 64);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int reps = 2000;
  for (int m = 0; m < 2; ++m) for (int t = 0; t < 2; ++t) {
    cudaEventRecord(a);
    if (m == 0) k<0><<<1, 32>>>(reps, o); else k<1><<<1, 32>>>(reps, o);
    cudaEventRecord(b); cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double adds = (double)reps * 1024;
    printf("%s: %.2f ns/add (%.1f cycles @ %d MHz)\n", m ? "pre-converted" : "chain_add    ", ms * 1e6 / adds,
           ms * 1e-3 * clk * 1e3 / adds, clk / 1000);
  }
  return 0;
}
