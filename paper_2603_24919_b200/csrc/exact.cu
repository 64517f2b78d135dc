// Index-free exact paths on the device.
//
// 1. Exact k-NN ground truth: the reference's
// dataio.compute_ground_truth (dataio.py:142-172) with its arithmetic --
//   xsq = einsum('ij,ij->i', X, X)            (numpy 2-lane einsum order)
//   G   = Q @ X.T                             (dgemm: one FMA chain over d)
//   d2  = max((xsq - 2 G) + qsq, 0)           (two roundings, as numpy evaluates)
//   top-k by (d2, id), dists = f32(sqrt(d2))
// Queries are processed in tiles of GT_QT: one pass over X computes the tile's
// full fp64 distance rows (each X row read once per tile, GT_QT FMA chains per
// thread), then one CTA per query radix-selects its k smallest (d2, id).
#include <algorithm>
#include <cmath>
#include <vector>

#include "index.cuh"

namespace taco {

constexpr int GT_QT = 32;     // queries per tile
constexpr int GT_NT = 256;    // threads per distance CTA
constexpr int GS_NT = 1024;   // threads per select CTA
constexpr int GS_MAXK = 1024;

__global__ void k_gt_qsq(const float* __restrict__ Q, int64_t nq, int d, double* __restrict__ Qd,
                         double* __restrict__ qsq) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  const float* r = Q + q * d;
  for (int t = 0; t < d; ++t) Qd[q * d + t] = (double)r[t];
  qsq[q] = einsum_sq([&](int t) { return (double)r[t]; }, d);
}

// D[qi * n + i] for the tile's qt queries (Qd rows q0 .. q0+qt-1)
__global__ void __launch_bounds__(GT_NT) k_gt_d2(const float* __restrict__ X, int64_t n, int d,
                                                  const double* __restrict__ Qd, const double* __restrict__ qsq,
                                                  int qt, double* __restrict__ D) {
  extern __shared__ double qs[];   // [GT_QT][d]
  for (int t = threadIdx.x; t < qt * d; t += GT_NT) qs[t] = Qd[t];
  __syncthreads();
  for (int64_t i = (int64_t)blockIdx.x * GT_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * GT_NT) {
    const float* xr = X + i * d;
    double acc[GT_QT];
#pragma unroll
    for (int q = 0; q < GT_QT; ++q) acc[q] = 0.0;
    double a0 = 0.0, a1 = 0.0;   // einsum lanes of xsq
    int b = 0;
    for (; b + 8 <= d; b += 8) {
      double p[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) p[u] = (double)xr[b + u];
#pragma unroll
      for (int u = 3; u >= 0; --u) {
        a0 = __dadd_rn(__dmul_rn(p[2 * u], p[2 * u]), a0);
        a1 = __dadd_rn(__dmul_rn(p[2 * u + 1], p[2 * u + 1]), a1);
      }
#pragma unroll
      for (int q = 0; q < GT_QT; ++q) {
        if (q < qt) {
          const double* qr = qs + q * d + b;
#pragma unroll
          for (int u = 0; u < 8; ++u) acc[q] = __fma_rn(qr[u], p[u], acc[q]);
        }
      }
    }
    for (; b < d; b += 2) {
      const double p0 = (double)xr[b];
      a0 = __dadd_rn(__dmul_rn(p0, p0), a0);
      double p1 = 0.0;
      if (b + 1 < d) {
        p1 = (double)xr[b + 1];
        a1 = __dadd_rn(__dmul_rn(p1, p1), a1);
      }
#pragma unroll
      for (int q = 0; q < GT_QT; ++q) {
        if (q < qt) {
          acc[q] = __fma_rn(qs[q * d + b], p0, acc[q]);
          if (b + 1 < d) acc[q] = __fma_rn(qs[q * d + b + 1], p1, acc[q]);
        }
      }
    }
    const double xsq = __dadd_rn(a0, a1);
#pragma unroll
    for (int q = 0; q < GT_QT; ++q) {
      if (q < qt) {
        double v = __dadd_rn(__dsub_rn(xsq, __dmul_rn(2.0, acc[q])), qsq[q]);
        D[(int64_t)q * n + i] = v > 0.0 ? v : 0.0;   // np.maximum(d2, 0): -0 and NaN handled like numpy below
      }
    }
  }
}

// k smallest (d2, id) of one distance row, ids implicit (= position).
__device__ void gt_radix(const unsigned long long* keys, int64_t n, int kk, bool by_id, unsigned long long key_eq,
                         unsigned long long& out, int& remain, unsigned& ties, unsigned* hist,
                         unsigned long long* s_pre, int* s_rem, unsigned* s_ties) {
  const int tid = threadIdx.x;
  if (tid == 0) { *s_pre = 0ull; *s_rem = kk; }
  __syncthreads();
  unsigned long long msk = 0ull;
  const int passes = by_id ? 4 : 8;   // ids < 2^32
  for (int p = 0; p < passes; ++p) {
    const int shift = (passes - 1 - p) * 8;
    for (int i = tid; i < 256; i += GS_NT) hist[i] = 0;
    __syncthreads();
    const unsigned long long pre = *s_pre;
    for (int64_t i = tid; i < n; i += GS_NT) {
      unsigned long long v;
      if (by_id) {
        if (keys[i] != key_eq) continue;
        v = (unsigned long long)i;
      } else {
        v = keys[i];
      }
      if ((v & msk) == pre) atomicAdd(&hist[(v >> shift) & 255ull], 1u);
    }
    __syncthreads();
    if (tid == 0) {
      const int rem = *s_rem;
      unsigned acc = 0;
      int dg = 0;
      for (; dg < 255; ++dg) {
        if (acc + hist[dg] >= (unsigned)rem) break;
        acc += hist[dg];
      }
      *s_rem = rem - (int)acc;
      *s_pre = pre | ((unsigned long long)dg << shift);
      *s_ties = hist[dg];   // after the last pass: how many keys equal the result
    }
    msk |= 255ull << shift;
    __syncthreads();
  }
  out = *s_pre;
  remain = *s_rem;
  ties = *s_ties;
  __syncthreads();
}

__global__ void __launch_bounds__(GS_NT) k_gt_select(const double* __restrict__ D, int64_t n, int k,
                                                      int32_t* __restrict__ ids, float* __restrict__ dists) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_pre;
  __shared__ int s_rem, s_fill;
  __shared__ unsigned s_ties;
  __shared__ unsigned long long skey[GS_MAXK];
  __shared__ int64_t sid[GS_MAXK];
  const int64_t q = blockIdx.x;
  const unsigned long long* keys = reinterpret_cast<const unsigned long long*>(D + q * n);
  // d2 >= +0 (clamped), so the bit patterns order like the values
  unsigned long long tau;
  int take;
  unsigned ties;
  gt_radix(keys, n, k, false, 0ull, tau, take, ties, hist, &s_pre, &s_rem, &s_ties);
  unsigned long long pi = ~0ull;   // largest id admitted among the d2 == tau ties (lower ids first)
  if (ties > (unsigned)take) {
    int dummy;
    unsigned t2;
    gt_radix(keys, n, take, true, tau, pi, dummy, t2, hist, &s_pre, &s_rem, &s_ties);
  }
  if (threadIdx.x == 0) s_fill = 0;
  __syncthreads();
  for (int64_t i = threadIdx.x; i < n; i += GS_NT) {
    const unsigned long long kv = keys[i];
    if (kv < tau || (kv == tau && (unsigned long long)i <= pi)) {
      const int slot = atomicAdd(&s_fill, 1);
      skey[slot] = kv;
      sid[slot] = i;
    }
  }
  __syncthreads();
  int P = 1;
  while (P < k) P <<= 1;
  for (int i = k + threadIdx.x; i < P; i += GS_NT) {
    skey[i] = ~0ull;
    sid[i] = INT64_MAX;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += GS_NT) {
        const int jx = i ^ stride;
        if (jx > i) {
          const bool up = (i & size) == 0;
          const unsigned long long ka = skey[i], kb = skey[jx];
          const int64_t pa = sid[i], pb = sid[jx];
          const bool gt = ka > kb || (ka == kb && pa > pb);
          if (gt == up) {
            skey[i] = kb; skey[jx] = ka;
            sid[i] = pb; sid[jx] = pa;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = threadIdx.x; i < k; i += GS_NT) {
    ids[q * k + i] = (int32_t)sid[i];
    dists[q * k + i] = (float)__dsqrt_rn(__longlong_as_double((long long)skey[i]));
  }
}

static int ground_truth_impl(int device, const float* X_d, int64_t n, int d, const float* Q_h, int64_t nq, int k,
                             int32_t* ids_h, float* dists_h) {
  if (n < 1 || d < 1) TACO_FAIL(TACO_ERR_PARAMETER, "dataset has zero rows or columns");
  if (nq < 1) TACO_FAIL(TACO_ERR_PARAMETER, "queries has zero rows");
  if (k < 1 || k > n) TACO_FAIL(TACO_ERR_PARAMETER, "k %d outside [1, %lld]", k, (long long)n);
  if (k > GS_MAXK) TACO_FAIL(TACO_ERR_PARAMETER, "ground truth supports k <= %d", GS_MAXK);
  const int qtm = (int)std::min<int64_t>(GT_QT, (200 * 1024) / (8 * (int64_t)d));   // queries per tile
  if (qtm < 1) TACO_FAIL(TACO_ERR_PARAMETER, "ground truth supports d <= %d", 200 * 1024 / 8);
  TACO_TRY(with_device(device));
  DevBuf Qf, Qd, qsq, D, oi, od;
  int rc = TACO_OK;
  do {
    if ((rc = Qf.ensure(sizeof(float) * (size_t)nq * d)) || (rc = Qd.ensure(sizeof(double) * (size_t)nq * d)) ||
        (rc = qsq.ensure(sizeof(double) * (size_t)nq)) || (rc = D.ensure(sizeof(double) * (size_t)GT_QT * n)) ||
        (rc = oi.ensure(sizeof(int32_t) * (size_t)nq * k)) || (rc = od.ensure(sizeof(float) * (size_t)nq * k)))
      break;
    const size_t smem = sizeof(double) * (size_t)qtm * d;
    if (cudaFuncSetAttribute(k_gt_d2, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
      set_error("ground truth: shared memory attribute");
      rc = TACO_ERR_CUDA;
      break;
    }
    cudaMemcpy(Qf.p, Q_h, sizeof(float) * (size_t)nq * d, cudaMemcpyHostToDevice);
    k_gt_qsq<<<(unsigned)ceil_div(nq, 128), 128>>>(Qf.as<float>(), nq, d, Qd.as<double>(), qsq.as<double>());
    count_launch();
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const unsigned grid = (unsigned)std::min<int64_t>(ceil_div(n, GT_NT), (int64_t)sms * 4);
    for (int64_t q0 = 0; q0 < nq; q0 += qtm) {
      const int qt = (int)std::min<int64_t>(qtm, nq - q0);
      k_gt_d2<<<grid, GT_NT, smem>>>(X_d, n, d, Qd.as<double>() + q0 * d, qsq.as<double>() + q0, qt, D.as<double>());
      k_gt_select<<<(unsigned)qt, GS_NT>>>(D.as<double>(), n, k, oi.as<int32_t>() + q0 * k, od.as<float>() + q0 * k);
      count_launch(2);
    }
    cudaMemcpy(ids_h, oi.p, sizeof(int32_t) * (size_t)nq * k, cudaMemcpyDeviceToHost);
    cudaMemcpy(dists_h, od.p, sizeof(float) * (size_t)nq * k, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; }
  } while (0);
  Qf.release(); Qd.release(); qsq.release(); D.release(); oi.release(); od.release();
  return rc;
}

// 2. SC-Linear exact collision counting (engine.py:290-321):
// per subspace j, d2_j(i) = einsum((f64 T[i, js:js+s] - f64 qt[js:js+s])^2);
// the ceil(alpha n) smallest (d2_j, id) collide; scores[i] = #subspaces.
// T element (i, c) lives at T[i * rs + c * cs] (row-major host copy or the
// index's dimension-major resident matrix).
__global__ void k_sc_d2(const float* __restrict__ T, int64_t n, int64_t rs, int64_t cs, int s,
                        const double* __restrict__ qt, double* __restrict__ D2) {
  const int j = blockIdx.y;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const float* base = T + i * rs + (int64_t)j * s * cs;
    const double* qj = qt + (int64_t)j * s;
    const double v = einsum_sq([&](int t) { return __dsub_rn((double)base[t * cs], qj[t]); }, s);
    D2[(int64_t)j * n + i] = v;   // a sum of squares: >= +0, bit patterns order like values
  }
}

__global__ void __launch_bounds__(GS_NT) k_sc_select(const double* __restrict__ D2, int64_t n, int collide,
                                                      unsigned long long* __restrict__ cut) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_pre;
  __shared__ int s_rem;
  __shared__ unsigned s_ties;
  const unsigned long long* keys = reinterpret_cast<const unsigned long long*>(D2 + (int64_t)blockIdx.x * n);
  unsigned long long tau, pi = ~0ull;
  int take;
  unsigned ties;
  gt_radix(keys, n, collide, false, 0ull, tau, take, ties, hist, &s_pre, &s_rem, &s_ties);
  if (ties > (unsigned)take) {
    int dummy;
    unsigned t2;
    gt_radix(keys, n, take, true, tau, pi, dummy, t2, hist, &s_pre, &s_rem, &s_ties);
  }
  if (threadIdx.x == 0) {
    cut[2 * blockIdx.x] = tau;
    cut[2 * blockIdx.x + 1] = pi;
  }
}

__global__ void k_sc_mark(const double* __restrict__ D2, int64_t n, int n_sub,
                          const unsigned long long* __restrict__ cut, uint8_t* __restrict__ scores) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    int c = 0;
    for (int j = 0; j < n_sub; ++j) {
      const unsigned long long kv = (unsigned long long)__double_as_longlong(D2[(int64_t)j * n + i]);
      c += kv < cut[2 * j] || (kv == cut[2 * j] && (unsigned long long)i <= cut[2 * j + 1]);
    }
    scores[i] = (uint8_t)c;
  }
}

static int sc_linear_impl(int device, const float* T_d, int64_t n, int64_t rs, int64_t cs, int n_sub, int s,
                          const float* qt_h, double alpha, uint8_t* scores_h) {
  if (n < 1) TACO_FAIL(TACO_ERR_PARAMETER, "empty transformed matrix");
  if (n_sub < 1 || n_sub > 255 || s < 1) TACO_FAIL(TACO_ERR_PARAMETER, "bad subspace layout %d x %d", n_sub, s);
  if (!(alpha > 0.0 && alpha <= 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "collision ratio %g outside (0, 1]", alpha);
  const int64_t collide = std::min<int64_t>(n, (int64_t)std::ceil(alpha * (double)n));   // engine.py:309
  std::vector<double> q64((size_t)n_sub * s);
  for (size_t t = 0; t < q64.size(); ++t) q64[t] = (double)qt_h[t];
  DevBuf qd, D2, cut, sc;
  int rc = TACO_OK;
  do {
    if ((rc = qd.ensure(sizeof(double) * q64.size())) || (rc = D2.ensure(sizeof(double) * (size_t)n_sub * n)) ||
        (rc = cut.ensure(16 * (size_t)n_sub)) || (rc = sc.ensure((size_t)n)))
      break;
    cudaMemcpy(qd.p, q64.data(), sizeof(double) * q64.size(), cudaMemcpyHostToDevice);
    int sms = 148;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device);
    const unsigned gx = (unsigned)std::min<int64_t>(ceil_div(n, 256), (int64_t)sms * 8);
    k_sc_d2<<<dim3(gx, (unsigned)n_sub), 256>>>(T_d, n, rs, cs, s, qd.as<double>(), D2.as<double>());
    k_sc_select<<<(unsigned)n_sub, GS_NT>>>(D2.as<double>(), n, (int)collide, cut.as<unsigned long long>());
    k_sc_mark<<<gx, 256>>>(D2.as<double>(), n, n_sub, cut.as<unsigned long long>(), sc.as<uint8_t>());
    count_launch(3);
    cudaMemcpy(scores_h, sc.p, (size_t)n, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; }
  } while (0);
  qd.release(); D2.release(); cut.release(); sc.release();
  return rc;
}

}  // namespace taco

using namespace taco;

extern "C" {

int taco_ground_truth(int device, const float* X_h, int64_t n, int32_t d, const float* Q_h, int64_t nq, int32_t k,
                      int32_t* ids_h, float* dists_h) {
  TACO_TRY(with_device(device));
  if (n < 1 || d < 1) TACO_FAIL(TACO_ERR_PARAMETER, "dataset has zero rows or columns");
  DevBuf X;
  TACO_TRY(X.ensure(sizeof(float) * (size_t)n * d));
  cudaError_t e = cudaMemcpy(X.p, X_h, sizeof(float) * (size_t)n * d, cudaMemcpyHostToDevice);
  int rc = e == cudaSuccess ? ground_truth_impl(device, X.as<float>(), n, d, Q_h, nq, k, ids_h, dists_h)
                            : (set_error("%s", cudaGetErrorString(e)), TACO_ERR_CUDA);
  X.release();
  return rc;
}

int taco_sc_linear_scores(int device, const float* T_h, int64_t n, int32_t n_sub, int32_t s, const float* qt_h,
                          double alpha, uint8_t* scores_h) {
  TACO_TRY(with_device(device));
  if (n < 1 || n_sub < 1 || s < 1) TACO_FAIL(TACO_ERR_PARAMETER, "empty transformed matrix");
  DevBuf T;
  TACO_TRY(T.ensure(sizeof(float) * (size_t)n * n_sub * s));
  cudaError_t e = cudaMemcpy(T.p, T_h, sizeof(float) * (size_t)n * n_sub * s, cudaMemcpyHostToDevice);
  int rc = e == cudaSuccess ? sc_linear_impl(device, T.as<float>(), n, (int64_t)n_sub * s, 1, n_sub, s, qt_h, alpha,
                                             scores_h)
                            : (set_error("%s", cudaGetErrorString(e)), TACO_ERR_CUDA);
  T.release();
  return rc;
}

int taco_sc_linear_scores_index(taco_index* idx, const float* qt_h, double alpha, uint8_t* scores_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_T) TACO_FAIL(TACO_ERR_STATE, "transformed matrix not resident");
  return sc_linear_impl(idx->device, idx->T.as<float>(), idx->n, 1, idx->n, idx->n_sub, idx->s, qt_h, alpha,
                        scores_h);
}

int taco_ground_truth_index(taco_index* idx, const float* Q_h, int64_t nq, int32_t k, int32_t* ids_h,
                            float* dists_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "base vectors are not resident");
  if (idx->n_global != idx->n) TACO_FAIL(TACO_ERR_STATE, "ground truth needs the whole dataset (not a shard)");
  return ground_truth_impl(idx->device, idx->X.as<float>(), idx->n, idx->d, Q_h, nq, k, ids_h, dists_h);
}

}  // extern "C"
