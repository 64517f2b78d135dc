// Microbenchmark: moving scattered 128-byte rows (the u8 re-rank gather,
// config 2: one row per candidate) into shared memory three ways.
//   bulk1  one elected thread per CTA issues a 1-D cp.async.bulk per row
//          into an mbarrier ring (TMA), a consumer warp reads each row
//   bulk32 the 32 lanes of a producer warp each issue one row's bulk copy
//   ldgsts cp.async 16 B (LDGSTS): 8 lanes per row, 4 rows per instruction,
//          a 2-stage ring per warp, 4 warps per CTA (what k_rerank_async does)
// Rows are drawn from `nrows` rows at random (nrows * 128 B: 32 MB stays in
// L2, 512 MB streams from HBM).  Prints rows/s and bytes/s.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/mb_bulk tools/mb_bulk.cu && tools/mb_bulk
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* b, unsigned c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, unsigned par) {
  uint32_t ok = 0;
  while (!ok)
    asm volatile("{ .reg .pred p; mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2; selp.u32 %0, 1, 0, p; }"
                 : "=r"(ok) : "r"(smem_u32(b)), "r"(par) : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ uint32_t hsh(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

constexpr int ST = 8, R = 32;   // ring: 8 stages of 32 rows (4 KB each)

// MODE 0: thread 0 of warp 1 issues; MODE 1: all 32 lanes of warp 1 issue
template <int MODE>
__global__ void __launch_bounds__(64) k_bulk(const uint8_t* __restrict__ X, uint32_t nrows, int tiles,
                                             uint32_t* out) {
  __shared__ __align__(128) uint8_t ring[ST][R][128];
  __shared__ uint64_t full[ST], empty[ST];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  if (threadIdx.x == 0) {
    for (int s = 0; s < ST; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  uint32_t acc = 0;
  if (w == 1) {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % ST;
      if (t >= ST) mbar_wait(&empty[s], ((t / ST) - 1) & 1);
      if (MODE == 0) {
        if (lane == 0) {
          mbar_expect_tx(&full[s], R * 128);
          for (int r = 0; r < R; ++r) {
            const uint32_t row = hsh(blockIdx.x * 7919u + t * 131u + r) % nrows;
            bulk(ring[s][r], X + (size_t)row * 128, 128, &full[s]);
          }
        }
      } else {
        if (lane == 0) mbar_expect_tx(&full[s], R * 128);
        __syncwarp();
        const uint32_t row = hsh(blockIdx.x * 7919u + t * 131u + lane) % nrows;
        bulk(ring[s][lane], X + (size_t)row * 128, 128, &full[s]);
      }
    }
  } else {
    for (int t = 0; t < tiles; ++t) {
      const int s = t % ST;
      mbar_wait(&full[s], (t / ST) & 1);
      acc += reinterpret_cast<const uint32_t*>(ring[s][lane])[lane & 31];
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[s]);
    }
  }
  if (acc == 0xFFFFFFFFu) out[0] = acc;
}

// LDGSTS: every warp streams its own tiles through a 2-stage ring
__global__ void __launch_bounds__(128) k_ldgsts(const uint8_t* __restrict__ X, uint32_t nrows, int tiles,
                                                uint32_t* out) {
  __shared__ __align__(128) uint8_t ring[4][2][R][144];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int r0 = lane / 8, cl = lane % 8;
  uint32_t acc = 0;
  auto issue = [&](int t) {
    const int s = t & 1;
#pragma unroll
    for (int j = 0; j < R / 4; ++j) {
      const int rr = j * 4 + r0;
      const uint32_t row = hsh((blockIdx.x * 4 + w) * 7919u + t * 131u + rr) % nrows;
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(&ring[w][s][rr][cl * 16])),
                   "l"(X + (size_t)row * 128 + cl * 16) : "memory");
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
  };
  issue(0);
  for (int t = 0; t < tiles; ++t) {
    if (t + 1 < tiles) issue(t + 1);
    else asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group 1;" ::: "memory");
    __syncwarp();
    acc += reinterpret_cast<const uint32_t*>(ring[w][t & 1][lane])[lane & 31];
    __syncwarp();
  }
  if (acc == 0xFFFFFFFFu) out[0] = acc;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  uint8_t* X;
  uint32_t* out;
  const size_t maxb = 512ull << 20;
  cudaMalloc(&X, maxb);
  cudaMemset(X, 1, maxb);
  cudaMalloc(&out, 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  for (size_t bytes : {32ull << 20, 512ull << 20}) {
    const uint32_t nrows = (uint32_t)(bytes / 128);
    for (int mode = 0; mode < 3; ++mode) {
      const int tiles = 2000;
      const int ctas = mode == 2 ? sms * 8 : sms * 16;   // ldgsts: 4 warps per CTA
      const double rows = (double)ctas * (mode == 2 ? 4 : 1) * tiles * R;
      for (int rep = 0; rep < 2; ++rep) {
        cudaEventRecord(a);
        if (mode == 0) k_bulk<0><<<ctas, 64>>>(X, nrows, tiles, out);
        else if (mode == 1) k_bulk<1><<<ctas, 64>>>(X, nrows, tiles, out);
        else k_ldgsts<<<ctas, 128>>>(X, nrows, tiles, out);
        cudaEventRecord(b);
        cudaEventSynchronize(b);
      }
      float ms = 0.f;
      cudaEventElapsedTime(&ms, a, b);
      const char* nm[3] = {"bulk1 ", "bulk32", "ldgsts"};
      printf("%s rows from %4zu MB: %7.2f G rows/s  %7.1f GB/s  (%.2f ms, err %s)\n", nm[mode], bytes >> 20,
             rows / ms / 1e6, rows * 128 / ms / 1e6, ms, cudaGetErrorString(cudaGetLastError()));
    }
  }
  return 0;
}
