// dependent fp64 add chain latency on one thread (k-means++ replay cost model)
#include <cstdio>
#include <cuda_runtime.h>
__global__ void chain(const double* x, int n, double* out) {
  double c = 0.0;
  for (int i = 0; i < n; i += 8) {
#pragma unroll
    for (int e = 0; e < 8; ++e) c = __dadd_rn(c, x[(i + e) & 1023]);
  }
  *out = c;
}
int main() {
  double *x, *o; cudaMalloc(&x, 8192); cudaMalloc(&o, 8); cudaMemset(x, 0, 8192);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  const int n = 1 << 24;
  chain<<<1, 1>>>(x, 1024, o);
  cudaEventRecord(a); chain<<<1, 1>>>(x, n, o); cudaEventRecord(b); cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("dependent DADD chain: %.2f ns/add  (%.1f cycles at %d MHz)\n", ms * 1e6 / n, ms * 1e-3 * clk * 1e3 / n, clk / 1000);
  return 0;
}
