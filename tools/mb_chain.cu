// Micro-benchmark: cycles per element of a dependent fp64 add chain fed from
// shared memory (the k_cluster_sums / k_colmean_seq consumer loop), variants:
//  A: 64-wide float blocks, convert at the add;  B: convert a block to double first.
#include <cstdio>
#include <cuda_runtime.h>
template <int V>
__global__ void chain(const float* g, int n, int st, double* out, long long* cyc) {
  __shared__ float sm[64 * 8 * 4 + 32];
  for (int i = threadIdx.x; i < 64 * 8 * 4; i += blockDim.x) sm[i] = g[i];
  __syncthreads();
  const int lane = threadIdx.x;
  double acc = 0.0;
  long long t0 = clock64();
  for (int it = 0; it < n / 64; ++it) {
    const float* tv = sm + (it & 3) * 64 * st + lane;
    if (V == 0) {
      float a[32], b[32];
#pragma unroll
      for (int u = 0; u < 32; ++u) a[u] = tv[u * st];
#pragma unroll
      for (int u = 0; u < 32; ++u) b[u] = tv[(32 + u) * st];
#pragma unroll
      for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, (double)a[u]);
#pragma unroll
      for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, (double)b[u]);
    } else if (V == 1) {
      double a[16];
#pragma unroll
      for (int blk = 0; blk < 4; ++blk) {
#pragma unroll
        for (int u = 0; u < 16; ++u) a[u] = (double)tv[(blk * 16 + u) * st];
#pragma unroll
        for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, a[u]);
      }
    } else {
      // pure chain on registers (floor)
#pragma unroll
      for (int u = 0; u < 64; ++u) acc = __dadd_rn(acc, (double)(u + it));
    }
  }
  long long t1 = clock64();
  if (lane < 8) out[lane] = acc;
  if (lane == 0) *cyc = t1 - t0;
}
int main() {
  float* g; double* o; long long* c;
  cudaMalloc(&g, 64 * 8 * 4 * 4); cudaMemset(g, 0, 64 * 8 * 4 * 4);
  cudaMalloc(&o, 64); cudaMalloc(&c, 8);
  const int n = 64 * 4096;
  long long h;
  chain<0><<<1, 32>>>(g, n, 8, o, c);
  printf("launch: %s\n", cudaGetErrorString(cudaDeviceSynchronize()));
  cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("A float blocks, convert at add: %.2f cycles/elem\n", (double)h / n);
  chain<1><<<1, 32>>>(g, n, 8, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("B convert 16 first:             %.2f cycles/elem\n", (double)h / n);
  chain<2><<<1, 32>>>(g, n, 8, o, c); cudaMemcpy(&h, c, 8, cudaMemcpyDeviceToHost);
  printf("C register chain (floor):       %.2f cycles/elem\n", (double)h / n);
  return 0;
}
