// Shared helpers for the TaCo sm_100a kernels: status plumbing, launch
// accounting and the exact-order fp64 reductions the reference's numpy
// primitives use.
#pragma once

#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <cstdarg>
#include <cstdlib>
#include <cstdio>
#include <string>

#include "../../include/taco_b200.h"

namespace taco {

void set_error(const char* fmt, ...);
void count_launch(int n = 1);

struct Status {
  int code = TACO_OK;
};

#define TACO_CHECK_CUDA(expr)                                                       \
  do {                                                                              \
    cudaError_t _e = (expr);                                                        \
    if (_e != cudaSuccess) {                                                        \
      ::taco::set_error("CUDA error %s at %s:%d: %s", cudaGetErrorName(_e), __FILE__, \
                        __LINE__, cudaGetErrorString(_e));                          \
      return TACO_ERR_CUDA;                                                         \
    }                                                                               \
  } while (0)

#define TACO_LAUNCHED()                         \
  do {                                          \
    ::taco::count_launch();                     \
    TACO_CHECK_CUDA(cudaGetLastError());        \
  } while (0)

#define TACO_TRY(expr)              \
  do {                              \
    int _s = (expr);                \
    if (_s != TACO_OK) return _s;   \
  } while (0)

#define TACO_FAIL(code, ...)                  \
  do {                                        \
    ::taco::set_error(__VA_ARGS__);           \
    return (code);                            \
  } while (0)

inline int64_t ceil_div(int64_t a, int64_t b) { return (a + b - 1) / b; }

// ---------------------------------------------------------------- numerics
// numpy's einsum('ij,ij->i') inner loop for float64 as compiled into numpy
// 2.3 (baseline SSE2, no FMA): two lanes, 8-element blocks consumed in the
// order 6,4,2,0 (+lane), a zero-padded 2-wide tail, then lane0 + lane1.
// Every product and add is rounded separately (no contraction).
// Measured bit-identical to numpy for m in [1, 960].
template <typename Get>
__device__ __forceinline__ double einsum_sq(Get get, int m) {
  double a0 = 0.0, a1 = 0.0;
  int base = 0;
  for (; base + 8 <= m; base += 8) {
#pragma unroll
    for (int u = 3; u >= 0; --u) {
      double p0 = get(base + 2 * u);
      double p1 = get(base + 2 * u + 1);
      a0 = __dadd_rn(__dmul_rn(p0, p0), a0);
      a1 = __dadd_rn(__dmul_rn(p1, p1), a1);
    }
  }
  for (; base < m; base += 2) {
    double p0 = get(base);
    a0 = __dadd_rn(__dmul_rn(p0, p0), a0);
    if (base + 1 < m) {
      double p1 = get(base + 1);
      a1 = __dadd_rn(__dmul_rn(p1, p1), a1);
    }
  }
  return __dadd_rn(a0, a1);
}

// OpenBLAS dgemm (SkylakeX/Haswell kernels) accumulates each output as one
// FMA chain over k starting from 0 (measured for K <= 128).
template <typename GetA, typename GetB>
__device__ __forceinline__ double dot_fma(GetA a, GetB b, int m) {
  double acc = 0.0;
  for (int t = 0; t < m; ++t) acc = __fma_rn(a(t), b(t), acc);
  return acc;
}

// clustering._sq_dists (clustering.py:34-38): max((xsq - 2*dot) + csq, 0).
__device__ __forceinline__ double sq_dist_expand(double xsq, double dot, double csq) {
  double v = __dadd_rn(__dsub_rn(xsq, __dmul_rn(2.0, dot)), csq);
  return v > 0.0 ? v : 0.0;
}

__device__ __forceinline__ unsigned lane_id() { return threadIdx.x & 31u; }

// ---- mbarrier + 1-D TMA (cp.async.bulk) helpers
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, unsigned count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(count) : "memory");
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];\n" ::"r"(smem_u32(bar)) : "memory");
}
__device__ __forceinline__ bool mbar_try(uint64_t* bar, unsigned parity) {
  uint32_t ok;
  asm volatile(
      "{\n .reg .pred p;\n mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n selp.u32 %0, 1, 0, p;\n}\n"
      : "=r"(ok)
      : "r"(smem_u32(bar)), "r"(parity)
      : "memory");
  return ok != 0;
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, unsigned parity) {
  while (!mbar_try(bar, parity)) {
  }
}
// 1-D TMA: `bytes` (multiple of 16) from global to shared, completion counted on bar
__device__ __forceinline__ void tma_g2s(void* dst, const void* src, unsigned bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];\n" ::"r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

// expect `bytes` more transaction bytes without arriving (several producers
// may add to one phase before its single arrive)
__device__ __forceinline__ void mbar_add_tx(uint64_t* bar, unsigned bytes) {
  asm volatile("mbarrier.expect_tx.relaxed.cta.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}

}  // namespace taco
