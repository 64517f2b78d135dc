// Standalone check of the tcgen05 TF32 MMA path used by k_assign_tc:
// D[128 x N] = A[128 x 8] . B[N x 8]^T with the no-swizzle K-major layout.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ int tc_off(int row, int k) { return (row >> 3) * 64 + (k >> 2) * 32 + (row & 7) * 4 + (k & 3); }
__device__ __forceinline__ uint64_t tc_desc(const void* smem, uint32_t lbo, uint32_t sbo) {
  const uint64_t a = (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);
  return a | ((uint64_t)(lbo >> 4) << 16) | ((uint64_t)(sbo >> 4) << 32) | (1ull << 46);
}
template <int N>
__global__ void k(const float* A, const float* B, float* D, uint32_t lbo, uint32_t sbo) {
  __shared__ __align__(128) float As[128 * 8];
  __shared__ __align__(128) float Bs[N * 8];
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tbase;
  int tid = threadIdx.x;
  for (int t = 0; t < 8; ++t) As[tc_off(tid, t)] = A[tid * 8 + t];
  for (int e = tid; e < N * 8; e += 128) Bs[tc_off(e / 8, e % 8)] = B[e];
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;\n" ::"r"(smem_u32(&mbar)));
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tbase)), "r"(N < 32 ? 32 : N));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t tmem = tbase;
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(N >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  if (tid == 0) {
    uint64_t da = tc_desc(As, lbo, sbo), db = tc_desc(Bs, lbo, sbo);
    asm volatile("{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem), "l"(da), "l"(db), "r"(idesc), "r"(0u));
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar)) : "memory");
  }
  {
    uint32_t ok = 0;
    while (!ok) asm volatile("{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n selp.u32 %0, 1, 0, p;\n}\n" : "=r"(ok) : "r"(smem_u32(&mbar)) : "memory");
  }
  asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
  uint32_t trow = tmem + ((uint32_t)((tid / 32) * 32) << 16);
  for (int cb = 0; cb < N / 16; ++cb) {
    uint32_t r[16];
    asm volatile("tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
      : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15]) : "r"(trow + cb * 16));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
    for (int u = 0; u < 16; ++u) D[tid * N + cb * 16 + u] = __uint_as_float(r[u]);
  }
  asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(N < 32 ? 32 : N));
}
int main() {
  const int N = 64;
  float hA[128 * 8], hB[N * 8], hD[128 * N];
  for (int i = 0; i < 128 * 8; ++i) hA[i] = (float)((i * 7) % 13 - 6);
  for (int i = 0; i < N * 8; ++i) hB[i] = (float)((i * 5) % 11 - 5);
  float *A, *B, *D;
  cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&D, sizeof hD);
  cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice); cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
  uint32_t cfg[][2] = {{128, 256}, {256, 128}};
  for (auto& c : cfg) {
    cudaMemset(D, 0, sizeof hD);
    k<N><<<1, 128>>>(A, B, D, c[0], c[1]);
    cudaError_t e = cudaDeviceSynchronize();
    cudaMemcpy(hD, D, sizeof hD, cudaMemcpyDeviceToHost);
    int bad = 0; double maxerr = 0;
    for (int i = 0; i < 128; ++i) for (int j = 0; j < N; ++j) {
      double ref = 0; for (int t = 0; t < 8; ++t) ref += (double)hA[i * 8 + t] * hB[j * 8 + t];
      double er = hD[i * N + j] - ref; if (er < 0) er = -er; if (er > maxerr) maxerr = er; if (er > 1e-3) ++bad;
    }
    printf("lbo=%u sbo=%u: %s bad=%d maxerr=%g D[0][0..3]=%g %g %g %g\n", c[0], c[1], cudaGetErrorString(e), bad, maxerr, hD[0], hD[1], hD[2], hD[3]);
  }
  return 0;
}
