// Cyclic Jacobi eigensolver on the GPU -- bit-exact with the reference's numpy
// jacobi_eigh rotation loop (spectral.py:155-195) and with the host
// restatement in jacobi.cpp.
//
// One cooperative kernel runs every sweep.  A and V live in global memory
// (L2-resident: 128 KB each at d = 128, 7.4 MB at d = 960).  Each round of
// the circle-method schedule (spectral.py:114-131) is three phases separated
// by grid-wide barriers:
//   1. every CTA recomputes the round's rotations (c, s) for the pairs with
//      A[p][q] != 0 into shared memory (d/2 pairs, cheap, no exchange needed);
//   2. row pass:    A[p,:] = c*A[p,:] - s*A[q,:],  A[q,:] = s*A[p,:] + c*A[q,:];
//   3. column pass: A[:,p], A[:,q] and V[:,p], V[:,q] likewise, A[p][q] and
//      A[q][p] set to 0.
// Pairs of a round are disjoint, so inside a pass every element is written by
// exactly one thread and the order of the element updates is irrelevant: every
// value is the same sequence of IEEE products and sums as numpy's elementwise
// ufuncs (no FMA contraction: explicit _rn intrinsics, --fmad=false).
// Before each sweep a grid-wide max of |off-diagonal| is compared with tol
// (spectral.py:161).  d <= JS_MAXD (160) takes the shared-memory variant below
// (one CTA, V rebuilt from the recorded rotations); larger d spreads over up
// to one CTA per SM.
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <vector>

#include "index.cuh"

namespace cg = cooperative_groups;

namespace taco {

constexpr int JT = 1024;
constexpr int JU = 8;   // row-pass items per thread with loads in flight together
constexpr int JC = 4;   // column-pass items (4 loads each)

struct JacobiArgs {
  double* A;
  double* V;
  const int16_t* sched;   // [rounds][d/2] pairs (p < q), -1 = dummy (odd d)
  int d, rounds, half;
  double tol;
  int max_sweeps;
  unsigned long long* maxbuf;   // [max_sweeps + 1] |off-diagonal| maxima (double bits)
  int* out;                     // [0] sweeps, [1] converged
};

__device__ __forceinline__ double ldA(const double* p) { return __ldcg(p); }

__global__ void __launch_bounds__(JT, 1) k_jacobi(JacobiArgs a) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ double jsh[];
  double* C = jsh;                         // [half]
  double* S = C + a.half;                  // [half]
  int* P = reinterpret_cast<int*>(S + a.half);
  int* Q = P + a.half;
  __shared__ double red[JT / 32];
  const int d = a.d;
  // 32-bit item indices throughout (d <= 32767 -> d*d < 2^30): the divisions
  // below are unsigned 32-bit, not the 64-bit software routine
  const unsigned gt = blockIdx.x * blockDim.x + threadIdx.x;
  const unsigned GT = gridDim.x * blockDim.x;
  const unsigned dd = (unsigned)d * (unsigned)d;
  const unsigned ud = (unsigned)d, uh = (unsigned)a.half;
  auto sync = [&]() {
    if (gridDim.x == 1) {
      __syncthreads();
    } else {
      __threadfence();
      grid.sync();
    }
  };
  auto offdiag_max = [&](int slot) -> double {
    double mx = 0.0;
    for (unsigned e = gt; e < dd; e += GT) {
      const unsigned i = e / ud, j = e - i * ud;
      if (i != j) mx = fmax(mx, fabs(ldA(a.A + e)));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = mx;
    __syncthreads();
    if (threadIdx.x == 0) {
      double w = 0.0;
      for (int k = 0; k < (int)(blockDim.x >> 5); ++k) w = fmax(w, red[k]);
      atomicMax(a.maxbuf + slot, (unsigned long long)__double_as_longlong(w));
    }
    sync();
    return __longlong_as_double((long long)__ldcg(a.maxbuf + slot));
  };
  int sweeps = 0, converged = 0;
  for (int sw = 0; sw < a.max_sweeps; ++sw) {
    if (offdiag_max(sw) <= a.tol) { converged = 1; break; }
    ++sweeps;
    for (int r = 0; r < a.rounds; ++r) {
      // 1. rotations of this round (every CTA, same values)
      const int16_t* pr = a.sched + (size_t)r * a.half * 2;
      for (int e = threadIdx.x; e < a.half; e += blockDim.x) {
        const int p = pr[2 * e], q = pr[2 * e + 1];
        P[e] = -1;
        if (p < 0) continue;
        const double apq = ldA(a.A + (size_t)p * d + q);
        if (apq == 0.0) continue;
        const double tau = __ddiv_rn(__dsub_rn(ldA(a.A + (size_t)q * d + q), ldA(a.A + (size_t)p * d + p)),
                                     __dmul_rn(2.0, apq));
        const double sg = tau < 0.0 ? -1.0 : 1.0;
        const double t = __ddiv_rn(sg, __dadd_rn(fabs(tau), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(tau, tau)))));
        const double c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
        C[e] = c;
        S[e] = __dmul_rn(t, c);
        P[e] = p;
        Q[e] = q;
      }
      __syncthreads();
      // 2. row pass (items: pair e, column x).  Items are disjoint, so each
      // thread loads JU items first and then computes/stores them (JU L2
      // round trips in flight instead of one at a time).
      const unsigned nrow = uh * ud;
      for (unsigned base = gt; base < nrow; base += GT * JU) {
        double av[JU], bv[JU];
        int ip[JU], ix[JU];
#pragma unroll
        for (int u = 0; u < JU; ++u) {
          const unsigned it = base + u * GT;
          ip[u] = -1;
          if (it < nrow) {
            const int e = (int)(it / ud), x = (int)(it - (unsigned)e * ud);
            ix[u] = x;
            const int p = P[e];
            if (p >= 0) {
              ip[u] = e;
              av[u] = ldA(a.A + (size_t)p * d + x);
              bv[u] = ldA(a.A + (size_t)Q[e] * d + x);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < JU; ++u) {
          if (ip[u] < 0) continue;
          const int e = ip[u], x = ix[u];
          const double c = C[e], s = S[e];
          a.A[(size_t)P[e] * d + x] = __dsub_rn(__dmul_rn(c, av[u]), __dmul_rn(s, bv[u]));
          a.A[(size_t)Q[e] * d + x] = __dadd_rn(__dmul_rn(s, av[u]), __dmul_rn(c, bv[u]));
        }
      }
      sync();
      // 3. column pass on A and V (items: row, pair), then A[p][q] = A[q][p] = 0
      for (unsigned base = gt; base < nrow; base += GT * JC) {
        double av[JC], bv[JC], va[JC], vb[JC];
        int ip[JC], ir[JC];
#pragma unroll
        for (int u = 0; u < JC; ++u) {
          const unsigned it = base + u * GT;
          ip[u] = -1;
          if (it < nrow) {
            const int row = (int)(it / uh), e = (int)(it - (unsigned)row * uh);
            ir[u] = row;
            const int p = P[e];
            if (p >= 0) {
              ip[u] = e;
              const int q = Q[e];
              av[u] = ldA(a.A + (size_t)row * d + p);
              bv[u] = ldA(a.A + (size_t)row * d + q);
              va[u] = ldA(a.V + (size_t)row * d + p);
              vb[u] = ldA(a.V + (size_t)row * d + q);
            }
          }
        }
#pragma unroll
        for (int u = 0; u < JC; ++u) {
          if (ip[u] < 0) continue;
          const int e = ip[u], row = ir[u];
          const int p = P[e], q = Q[e];
          const double c = C[e], s = S[e];
          double* ar = a.A + (size_t)row * d;
          const double np_ = __dsub_rn(__dmul_rn(av[u], c), __dmul_rn(bv[u], s));
          const double nq_ = __dadd_rn(__dmul_rn(av[u], s), __dmul_rn(bv[u], c));
          ar[p] = row == q ? 0.0 : np_;
          ar[q] = row == p ? 0.0 : nq_;
          double* vr = a.V + (size_t)row * d;
          vr[p] = __dsub_rn(__dmul_rn(va[u], c), __dmul_rn(vb[u], s));
          vr[q] = __dadd_rn(__dmul_rn(va[u], s), __dmul_rn(vb[u], c));
        }
      }
      sync();
    }
  }
  if (!converged) offdiag_max(a.max_sweeps);   // residual for the caller
  if (gt == 0) {
    a.out[0] = sweeps;
    a.out[1] = converged;
  }
}

// ---- d <= JS_MAXD: A lives in shared memory (rows padded to d+1 doubles so a
// column walk is conflict-free) and one CTA runs every sweep; the rotations of
// each round are recorded and V is rebuilt afterwards by k_jacobi_v, one warp
// per row of V (rows of V evolve independently: V[r,:] is rotated by every
// round's pairs in order, exactly the column pass of jacobi.cpp).
constexpr int JS_MAXD = 160;
struct JacobiSmemArgs {
  const double* A_in;
  double* A_out;
  const int16_t* sched;
  int d, rounds, half;
  double tol;
  int max_sweeps;
  int* rec_pq;      // [max_sweeps*rounds][half]: p | q << 16, -1 = no rotation
  double* rec_cs;   // [max_sweeps*rounds][half][2]
  int* out;         // [0] sweeps, [1] converged, [2] residual hi, [3] residual lo
};

__global__ void __launch_bounds__(JT, 1) k_jacobi_smem(JacobiSmemArgs a) {
  extern __shared__ double js[];
  const int d = a.d, ld = d + 1, half = a.half, tid = threadIdx.x;
  double* A = js;                              // [d][d+1]
  double* C = A + (size_t)d * ld;
  double* S = C + half;
  int* P = reinterpret_cast<int*>(S + half);
  int* Q = P + half;
  __shared__ double red[JT / 32];
  for (int e = tid; e < d * d; e += JT) A[(e / d) * ld + (e % d)] = a.A_in[e];
  __syncthreads();
  auto offdiag_max = [&]() -> double {
    double mx = 0.0;
    for (int e = tid; e < d * d; e += JT) {
      const int i = e / d, j = e - i * d;
      if (i != j) mx = fmax(mx, fabs(A[i * ld + j]));
    }
    for (int o = 16; o > 0; o >>= 1) mx = fmax(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if ((tid & 31) == 0) red[tid >> 5] = mx;
    __syncthreads();
    double w = 0.0;
    for (int k = 0; k < JT / 32; ++k) w = fmax(w, red[k]);
    __syncthreads();
    return w;
  };
  // thread -> (column/row x = tid % d, first pair tid / d, pair stride JT / d)
  const int x = tid % d, e0 = tid / d, es = JT / d;
  const bool xin = tid < es * d;
  int sweeps = 0, converged = 0, rec = 0;
  for (int sw = 0; sw < a.max_sweeps; ++sw) {
    if (offdiag_max() <= a.tol) { converged = 1; break; }
    ++sweeps;
    for (int r = 0; r < a.rounds; ++r, ++rec) {
      const int16_t* pr = a.sched + (size_t)r * half * 2;
      if (tid < half) {
        const int e = tid;
        const int p = pr[2 * e], q = pr[2 * e + 1];
        int pq = -1;
        double c = 1.0, sv = 0.0;
        if (p >= 0) {
          const double apq = A[p * ld + q];
          if (apq != 0.0) {
            const double tau = __ddiv_rn(__dsub_rn(A[q * ld + q], A[p * ld + p]), __dmul_rn(2.0, apq));
            const double sg = tau < 0.0 ? -1.0 : 1.0;
            const double t = __ddiv_rn(sg, __dadd_rn(fabs(tau), __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(tau, tau)))));
            c = __ddiv_rn(1.0, __dsqrt_rn(__dadd_rn(1.0, __dmul_rn(t, t))));
            sv = __dmul_rn(t, c);
            pq = p | (q << 16);
          }
        }
        P[e] = pq < 0 ? -1 : p;
        Q[e] = q;
        C[e] = c;
        S[e] = sv;
        a.rec_pq[(size_t)rec * half + e] = pq;
        a.rec_cs[((size_t)rec * half + e) * 2] = c;
        a.rec_cs[((size_t)rec * half + e) * 2 + 1] = sv;
      }
      __syncthreads();
      if (xin) {
        // row pass: A[p,x], A[q,x]
        for (int e = e0; e < half; e += es) {
          const int p = P[e];
          if (p < 0) continue;
          const int q = Q[e];
          const double c = C[e], sv = S[e];
          const double av = A[p * ld + x], bv = A[q * ld + x];
          A[p * ld + x] = __dsub_rn(__dmul_rn(c, av), __dmul_rn(sv, bv));
          A[q * ld + x] = __dadd_rn(__dmul_rn(sv, av), __dmul_rn(c, bv));
        }
      }
      __syncthreads();
      if (xin) {
        // column pass on row x: A[x,p], A[x,q]; A[p][q] = A[q][p] = 0
        double* ar = A + x * ld;
        for (int e = e0; e < half; e += es) {
          const int p = P[e];
          if (p < 0) continue;
          const int q = Q[e];
          const double c = C[e], sv = S[e];
          const double av = ar[p], bv = ar[q];
          const double np_ = __dsub_rn(__dmul_rn(av, c), __dmul_rn(bv, sv));
          const double nq_ = __dadd_rn(__dmul_rn(av, sv), __dmul_rn(bv, c));
          ar[p] = x == q ? 0.0 : np_;
          ar[q] = x == p ? 0.0 : nq_;
        }
      }
      __syncthreads();
    }
  }
  double res = 0.0;
  if (!converged) res = offdiag_max();
  for (int e = tid; e < d * d; e += JT) a.A_out[e] = A[(e / d) * ld + (e % d)];
  if (tid == 0) {
    a.out[0] = sweeps;
    a.out[1] = converged;
    a.out[4] = rec;
    memcpy(&a.out[2], &res, 8);
  }
}

// V = I rotated by every recorded round in order; one warp per row of V.
__global__ void k_jacobi_v(const int* __restrict__ rec_pq, const double* __restrict__ rec_cs,
                           const int* __restrict__ out, int d, int half, double* __restrict__ V) {
  extern __shared__ double vs[];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int row = blockIdx.x * (blockDim.x >> 5) + w;
  double* vr = vs + (size_t)w * d;
  if (row < d)
    for (int j = lane; j < d; j += 32) vr[j] = j == row ? 1.0 : 0.0;
  __syncwarp();
  if (row >= d) return;
  const int nrec = out[4];
  for (int r = 0; r < nrec; ++r) {
    for (int e = lane; e < half; e += 32) {
      const int pq = __ldg(rec_pq + (size_t)r * half + e);
      if (pq < 0) continue;
      const int p = pq & 0xffff, q = pq >> 16;
      const double c = __ldg(rec_cs + ((size_t)r * half + e) * 2), s = __ldg(rec_cs + ((size_t)r * half + e) * 2 + 1);
      const double va = vr[p], vb = vr[q];
      vr[p] = __dsub_rn(__dmul_rn(va, c), __dmul_rn(vb, s));
      vr[q] = __dadd_rn(__dmul_rn(va, s), __dmul_rn(vb, c));
    }
    __syncwarp();
  }
  for (int j = lane; j < d; j += 32) V[(size_t)row * d + j] = vr[j];
}

__global__ void k_eye(double* V, int d) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e < (int64_t)d * d) V[e] = (e / d) == (e % d) ? 1.0 : 0.0;
}

}  // namespace taco

using namespace taco;

extern "C" int taco_jacobi_sweeps_device(int device, double* A_h, double* V_h, int32_t d, double tol,
                                         int32_t max_sweeps, int32_t* sweeps_out, double* residual_out) {
  if (d < 0) TACO_FAIL(TACO_ERR_PARAMETER, "negative dimension");
  if (d > 32767) TACO_FAIL(TACO_ERR_PARAMETER, "dimension %d exceeds the device eigensolver limit", d);
  *sweeps_out = 0;
  *residual_out = 0.0;
  for (int i = 0; i < d; ++i)
    for (int j = 0; j < d; ++j) V_h[(size_t)i * d + j] = i == j ? 1.0 : 0.0;
  if (d <= 1) return TACO_OK;
  TACO_TRY(with_device(device));
  // circle-method schedule (spectral.py:114-131): ring of m = d + (d odd)
  const int m = d + (d & 1), half = m / 2, rounds = m - 1;
  std::vector<int16_t> sched((size_t)rounds * half * 2);
  std::vector<int> ring(m);
  for (int i = 0; i < m; ++i) ring[i] = i;
  for (int r = 0; r < rounds; ++r) {
    for (int i = 0; i < half; ++i) {
      int x = ring[i], y = ring[m - 1 - i];
      int16_t* o = &sched[((size_t)r * half + i) * 2];
      if (x < d && y < d) { o[0] = (int16_t)std::min(x, y); o[1] = (int16_t)std::max(x, y); }
      else { o[0] = -1; o[1] = -1; }
    }
    std::vector<int> nx(m);
    nx[0] = ring[0];
    nx[1] = ring[m - 1];
    for (int i = 1; i < m - 1; ++i) nx[i + 1] = ring[i];
    ring.swap(nx);
  }
  const size_t dd = (size_t)d * d;
  if (d <= JS_MAXD && !getenv("TACO_JACOBI_GLOBAL")) {
    DevBuf Ai, Ao, Vd, sch, rpq, rcs, out;
    const size_t nrec = (size_t)max_sweeps * rounds * half;
    TACO_TRY(Ai.ensure(8 * dd));
    TACO_TRY(Ao.ensure(8 * dd));
    TACO_TRY(Vd.ensure(8 * dd));
    TACO_TRY(sch.ensure(sizeof(int16_t) * sched.size()));
    TACO_TRY(rpq.ensure(sizeof(int) * nrec));
    TACO_TRY(rcs.ensure(2 * sizeof(double) * nrec));
    TACO_TRY(out.ensure(8 * sizeof(int)));
    cudaStream_t st = nullptr;
    TACO_CHECK_CUDA(cudaMemcpyAsync(Ai.p, A_h, 8 * dd, cudaMemcpyHostToDevice, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(sch.p, sched.data(), sizeof(int16_t) * sched.size(), cudaMemcpyHostToDevice, st));
    JacobiSmemArgs ja{Ai.as<double>(), Ao.as<double>(), sch.as<int16_t>(), d, rounds, half, tol, max_sweeps,
                      rpq.as<int>(), rcs.as<double>(), out.as<int>()};
    const size_t smem = sizeof(double) * ((size_t)d * (d + 1) + 2 * half) + sizeof(int) * 2 * half;
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_jacobi_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_jacobi_smem<<<1, JT, smem, st>>>(ja);
    TACO_LAUNCHED();
    const int wpb = 8;
    k_jacobi_v<<<(unsigned)ceil_div(d, wpb), 32 * wpb, sizeof(double) * wpb * d, st>>>(
        rpq.as<int>(), rcs.as<double>(), out.as<int>(), d, half, Vd.as<double>());
    TACO_LAUNCHED();
    int ho[8] = {0};
    TACO_CHECK_CUDA(cudaMemcpyAsync(ho, out.p, sizeof(ho), cudaMemcpyDeviceToHost, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(A_h, Ao.p, 8 * dd, cudaMemcpyDeviceToHost, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(V_h, Vd.p, 8 * dd, cudaMemcpyDeviceToHost, st));
    TACO_CHECK_CUDA(cudaStreamSynchronize(st));
    *sweeps_out = ho[0];
    if (!ho[1]) {
      double res;
      memcpy(&res, &ho[2], 8);
      *residual_out = res;
      if (res > tol)
        TACO_FAIL(TACO_ERR_CONVERGENCE,
                  "eigensolver hit the %d-sweep cap with off-diagonal residual %.3e above tolerance %.3e",
                  max_sweeps, res, tol);
    }
    return TACO_OK;
  }
  DevBuf A, V, sch, mx, out;
  TACO_TRY(A.ensure(8 * dd));
  TACO_TRY(V.ensure(8 * dd));
  TACO_TRY(sch.ensure(sizeof(int16_t) * sched.size()));
  TACO_TRY(mx.ensure(8 * (size_t)(max_sweeps + 1)));
  TACO_TRY(out.ensure(2 * sizeof(int)));
  cudaStream_t st = nullptr;
  TACO_CHECK_CUDA(cudaMemcpyAsync(A.p, A_h, 8 * dd, cudaMemcpyHostToDevice, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(sch.p, sched.data(), sizeof(int16_t) * sched.size(), cudaMemcpyHostToDevice, st));
  TACO_CHECK_CUDA(cudaMemsetAsync(mx.p, 0, 8 * (size_t)(max_sweeps + 1), st));
  k_eye<<<(unsigned)ceil_div((int64_t)dd, 256), 256, 0, st>>>(V.as<double>(), d);
  TACO_LAUNCHED();
  JacobiArgs ja;
  ja.A = A.as<double>();
  ja.V = V.as<double>();
  ja.sched = sch.as<int16_t>();
  ja.d = d;
  ja.rounds = rounds;
  ja.half = half;
  ja.tol = tol;
  ja.max_sweeps = max_sweeps;
  ja.maxbuf = mx.as<unsigned long long>();
  ja.out = out.as<int>();
  const size_t smem = (size_t)half * (2 * sizeof(double) + 2 * sizeof(int));
  TACO_CHECK_CUDA(cudaFuncSetAttribute(k_jacobi, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = 1;
  if (d > JS_MAXD) {
    int per_sm = 0, sms = 0, dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    TACO_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_jacobi, JT, smem));
    blocks = std::max(1, std::min(sms * std::max(per_sm, 1), (int)ceil_div((int64_t)half * d, JT)));
  }
  void* args[] = {&ja};
  TACO_CHECK_CUDA(cudaLaunchCooperativeKernel((void*)k_jacobi, dim3(blocks), dim3(JT), args, smem, st));
  count_launch();
  int ho[2] = {0, 0};
  unsigned long long res_bits = 0;
  TACO_CHECK_CUDA(cudaMemcpyAsync(ho, out.p, sizeof(ho), cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(&res_bits, mx.as<unsigned long long>() + max_sweeps, 8, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(A_h, A.p, 8 * dd, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(V_h, V.p, 8 * dd, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  *sweeps_out = ho[0];
  if (!ho[1]) {
    double res;
    memcpy(&res, &res_bits, 8);
    *residual_out = res;
    if (res > tol)
      TACO_FAIL(TACO_ERR_CONVERGENCE,
                "eigensolver hit the %d-sweep cap with off-diagonal residual %.3e above tolerance %.3e", max_sweeps,
                res, tol);
  }
  return TACO_OK;
}
