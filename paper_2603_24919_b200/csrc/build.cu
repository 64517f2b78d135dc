// TaCo index build on sm_100a.
//
//  covariance   k_nonfinite, k_colmean_seq (sequential fp64, bit-exact mean),
//               k_gram (split-K fp64 Gram tiles) + k_gram_reduce     spectral.py:94-111
//  transform    k_transform (index.cu)                                spectral.py:301-316
//  k-means++    k_xsq, k_pp_update (D^2 min + block sums), k_pp_search
//               (certified CDF search, exact numpy fallback)          clustering.py:41-54
//  Lloyd        k_assign (fp64 expansion, dgemm FMA order, first argmin),
//               k_lloyd_ctl, stable counting sort by label (k_label_*),
//               k_cluster_sums (sequential per-cluster fp64 sums in index
//               order == np.add.at), k_reseed                         clustering.py:86-107
//  cells        k_cell_hist / k_cell_offsets / k_cell_scatter: stable
//               counting sort by (l1,l2) into the chunk-major CSR     imi.py:70-81
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <vector>

#include "index.cuh"

namespace taco {

// ============================================================ covariance
__global__ void k_nonfinite(const float* __restrict__ X, int64_t total, int d,
                            unsigned long long* __restrict__ bad) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t e = i; e < total; e += stride) {
    if (!isfinite(X[e])) atomicMin(bad, (unsigned long long)(e / d));
  }
}

// numpy mean(axis=0) of a C-contiguous matrix: out = X[0]; out += X[r] for
// r = 1..n-1 (row-sequential), then / n.  Each of the block's first d
// threads runs one column's add chain over row tiles that the whole block
// stages in shared memory (double buffered).  One block per 1024 columns.
constexpr int CM_THREADS = 1024;
constexpr int CM_TILE_BYTES = 48 * 1024;
__global__ void __launch_bounds__(CM_THREADS) k_colmean_seq(const float* __restrict__ X, int64_t n, int d,
                                                            double* __restrict__ mean) {
  extern __shared__ float cm[];
  const int c0 = blockIdx.x * CM_THREADS;
  const int nc = min(CM_THREADS, d - c0);
  const int rows = max(1, CM_TILE_BYTES / (4 * nc));
  float* buf[2] = {cm, cm + (size_t)rows * nc};
  const int tid = threadIdx.x;
  const int64_t ntile = (n + rows - 1) / rows;
  auto load = [&](int64_t tb, float* dst) {
    const int64_t r0 = tb * rows;
    const int rr = (int)min((int64_t)rows, n - r0);
    for (int e = tid; e < rr * nc; e += CM_THREADS) {
      const int r = e / nc, c = e % nc;
      dst[e] = X[(r0 + r) * d + c0 + c];
    }
  };
  load(0, buf[0]);
  __syncthreads();
  double acc = 0.0;
  for (int64_t tb = 0; tb < ntile; ++tb) {
    if (tb + 1 < ntile) load(tb + 1, buf[(tb + 1) & 1]);
    if (tid < nc) {
      const float* tv = buf[tb & 1];
      const int rr = (int)min((int64_t)rows, n - tb * rows);
      int r = 0;
      if (tb == 0) { acc = (double)tv[tid]; r = 1; }
      for (; r < rr; ++r) acc = __dadd_rn(acc, (double)tv[r * nc + tid]);
    }
    __syncthreads();
  }
  if (tid < nc) mean[c0 + tid] = __ddiv_rn(acc, (double)n);
}

constexpr int GT = 64, GK = 16;
// partial[s] = sum over rows of split s of (x - mu)(x - mu)^T, 64x64 tile.
__global__ void __launch_bounds__(256) k_gram(const float* __restrict__ X, int64_t n, int d,
                                              const double* __restrict__ mean, int64_t rows_per,
                                              double* __restrict__ partial) {
  __shared__ double A[GK][GT + 1];
  __shared__ double B[GK][GT + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int i0 = blockIdx.x * GT, j0 = blockIdx.y * GT;
  const int64_t r0 = (int64_t)blockIdx.z * rows_per;
  const int64_t r1 = min(n, r0 + rows_per);
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int64_t rb = r0; rb < r1; rb += GK) {
    for (int e = threadIdx.x; e < GK * GT; e += 256) {
      const int kk = e / GT, cc = e % GT;
      const int64_t r = rb + kk;
      double va = 0.0, vb = 0.0;
      if (r < r1) {
        if (i0 + cc < d) va = __dsub_rn((double)X[r * d + i0 + cc], mean[i0 + cc]);
        if (j0 + cc < d) vb = __dsub_rn((double)X[r * d + j0 + cc], mean[j0 + cc]);
      }
      A[kk][cc] = va;
      B[kk][cc] = vb;
    }
    __syncthreads();
#pragma unroll 4
    for (int kk = 0; kk < GK; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = A[kk][ty + 16 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = B[kk][tx + 16 * u];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = __fma_rn(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
  double* P = partial + (size_t)blockIdx.z * d * d;
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    const int i = i0 + ty + 16 * x;
    if (i >= d) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      const int j = j0 + tx + 16 * y;
      if (j < d) P[(size_t)i * d + j] = acc[x][y];
    }
  }
}

__global__ void k_gram_reduce(const double* __restrict__ partial, int splits, int64_t dd,
                              double* __restrict__ G) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= dd) return;
  double acc = 0.0;
  for (int s = 0; s < splits; ++s) acc = __dadd_rn(acc, partial[(size_t)s * dd + e]);
  G[e] = acc;
}

// ================================================================ k-means
constexpr int PP_THREADS = 256;
constexpr int PP_PPT = 4;                       // points per thread in one block
constexpr int PP_BLOCK = PP_THREADS * PP_PPT;   // points per block-sum
constexpr double U0 = 1.1102230246251565e-16;   // 2^-53

static int g_force_replay = 0;   // test hook: always take the exact replay

struct HalfView {
  const float* X;   // dimension-major: X[t*n + i]
  int64_t n;
  int m;
  int k;
};

__global__ void k_xsq(HalfView h, double* __restrict__ xsq, double* __restrict__ xsqmax_blk) {
  __shared__ double red[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < h.n) {
    v = einsum_sq([&](int t) { return (double)h.X[(size_t)t * h.n + i]; }, h.m);
    xsq[i] = v;
  }
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = v;
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
    if (threadIdx.x == 0) xsqmax_blk[blockIdx.x] = w;
  }
}

// status layout (int64): [0] degenerate draw index (k if none), [1] fallbacks,
// [2] converged flag, [3] n_iter, [4] changed count
// D^2 update for centroid `ci` (= picks[ci]) and per-block sums of best.
__global__ void __launch_bounds__(PP_THREADS) k_pp_update(HalfView h, const double* __restrict__ xsq,
                                                          const int64_t* __restrict__ picks, int ci,
                                                          double* __restrict__ best,
                                                          double* __restrict__ C64,
                                                          double* __restrict__ bsum) {
  __shared__ double cv[64];
  __shared__ double red[PP_THREADS / 32];
  __shared__ double s_csq;
  const int64_t p = picks[ci];
  if (threadIdx.x < h.m) cv[threadIdx.x] = (double)h.X[(size_t)threadIdx.x * h.n + p];
  __syncthreads();
  if (threadIdx.x == 0) {
    s_csq = einsum_sq([&](int t) { return cv[t]; }, h.m);
    if (blockIdx.x == 0)
      for (int t = 0; t < h.m; ++t) C64[(size_t)ci * h.m + t] = cv[t];
  }
  __syncthreads();
  const double csq = s_csq;
  const int64_t b0 = (int64_t)blockIdx.x * PP_BLOCK + threadIdx.x;
  double s = 0.0;
#pragma unroll
  for (int u = 0; u < PP_PPT; ++u) {
    const int64_t i = b0 + (int64_t)u * PP_THREADS;
    if (i < h.n) {
      const double dot = dot_fma([&](int t) { return (double)h.X[(size_t)t * h.n + i]; },
                                 [&](int t) { return cv[t]; }, h.m);
      const double d2 = sq_dist_expand(xsq[i], dot, csq);
      double b = d2;
      if (ci > 0) {
        const double old = best[i];
        b = d2 < old ? d2 : old;
      }
      best[i] = b;
      s = __dadd_rn(s, b);
    }
  }
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < PP_THREADS / 32; ++w) t = __dadd_rn(t, red[w]);
    bsum[blockIdx.x] = t;
  }
}

// numpy pairwise summation (loops_utils.h.src, as measured in DESIGN.md §4):
// n < 8 sequential; n <= 128 eight strided accumulators combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail; else split at
// n2 = n/2 - (n/2)%8 and add the halves.  The leaves (ranges <= 128) depend
// only on n and are listed once on the host in depth-first order.
static void pairwise_leaves(int64_t off, int64_t len, std::vector<int64_t>& out) {
  if (len <= 128) {
    out.push_back(off);
    out.push_back(len);
    return;
  }
  int64_t n2 = len / 2;
  n2 -= n2 % 8;
  pairwise_leaves(off, n2, out);
  pairwise_leaves(off + n2, len - n2, out);
}

__device__ double np_leaf(const double* a, int64_t len) {
  if (len < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < len; ++i) r = __dadd_rn(r, a[i]);
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = a[j];
  int64_t i = 8;
  for (; i < len - (len % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], a[i + j]);
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < len; ++i) res = __dadd_rn(res, a[i]);
  return res;
}

// Combines the leaf sums (in depth-first order) exactly as the recursion does.
__device__ double np_combine(const double* leaf, int64_t n) {
  struct Fr { int64_t len; double left; int state; };
  Fr st[64];
  int sp = 0;
  int64_t li = 0;
  st[sp++] = {n, 0.0, 0};
  double ret = 0.0;
  while (sp > 0) {
    Fr& f = st[sp - 1];
    if (f.len <= 128) {
      ret = leaf[li++];
      --sp;
    } else {
      int64_t n2 = f.len / 2;
      n2 -= n2 % 8;
      if (f.state == 0) {
        f.state = 1;
        st[sp++] = {n2, 0.0, 0};
      } else if (f.state == 1) {
        f.left = ret;
        f.state = 2;
        st[sp++] = {f.len - n2, 0.0, 0};
      } else {
        ret = __dadd_rn(f.left, ret);
        --sp;
      }
    }
  }
  return ret;
}

// One CTA: chooses picks[ci+1] from best (after centroids 0..ci) and u.
// Fast path: fp64 prefix over block sums, locate the crossing, then certify
// that numpy's sequential cumsum/normalise/searchsorted (the reference's
// Generator.choice, clustering.py:48) cannot land elsewhere.  Otherwise
// replay numpy's arithmetic exactly (single thread).
constexpr int PS_THREADS = 1024;
constexpr int PS_TILE = 2048;   // doubles per staged tile of the replay chain
__global__ void __launch_bounds__(PS_THREADS) k_pp_search(HalfView h, const double* __restrict__ best,
                                                          const double* __restrict__ bsum, int64_t nb,
                                                          const double* __restrict__ uni,
                                                          const int64_t* __restrict__ forced,
                                                          double xsqmax, int ci,
                                                          int64_t* __restrict__ picks,
                                                          int64_t* __restrict__ status,
                                                          const int64_t* __restrict__ leaves, int64_t nleaves,
                                                          double* __restrict__ lsum, double* __restrict__ pbuf,
                                                          double* __restrict__ cbuf, int force_replay) {
  __shared__ double wsum[32];
  __shared__ double s_S;
  __shared__ int64_t s_blk;
  __shared__ double s_before;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int draw = ci + 1;                 // centroid index being chosen
  if (forced && forced[ci] >= 0) {
    if (tid == 0) picks[draw] = forced[ci];
    return;
  }
  // per-thread contiguous block-sum ranges, then a block scan (fixed order)
  const int64_t per = (nb + PS_THREADS - 1) / PS_THREADS;
  const int64_t a0 = (int64_t)tid * per, a1 = min(nb, a0 + per);
  double loc = 0.0;
  for (int64_t b = a0; b < a1; ++b) loc = __dadd_rn(loc, bsum[b]);
  double v = loc;
  for (int o = 1; o < 32; o <<= 1) {
    double x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = __dadd_rn(v, x);
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double w = wsum[lane];
    for (int o = 1; o < 32; o <<= 1) {
      double x = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w = __dadd_rn(w, x);
    }
    wsum[lane] = w;
    if (lane == 31) s_S = w;
  }
  if (tid == 0) s_blk = -1;
  __syncthreads();
  const double S = s_S;
  if (!(S > 0.0)) {
    // reference: total == 0 -> rng.integers(n); the host replays this draw
    if (tid == 0) {
      if (status[0] > draw) status[0] = draw;
      picks[draw] = 0;
    }
    return;
  }
  const double u = uni[ci];
  const double target = u * S;
  // thread whose range holds the first inclusive prefix > target
  double run = (wid ? wsum[wid - 1] : 0.0) + (v - loc);   // exclusive prefix (approx order ok: bounded)
  {
    double pre = run;
    for (int64_t b = a0; b < a1; ++b) {
      const double nx = __dadd_rn(pre, bsum[b]);
      if (nx > target && pre <= target) {
        s_blk = b;
        s_before = pre;
      }
      pre = nx;
    }
  }
  __syncthreads();
  __shared__ int s_ok;
  __shared__ double s_total;
  int64_t blk = s_blk;
  if (tid == 0) {
    int64_t kstar = -1;
    double Pk = 0.0, Pkm1 = 0.0;
    if (blk < 0) blk = nb - 1;   // rounding put the target at/after the end
    double pre = s_blk >= 0 ? s_before : S - bsum[blk];
    const int64_t i0 = blk * PP_BLOCK, i1 = min(h.n, i0 + PP_BLOCK);
    for (int64_t i = i0; i < i1; ++i) {
      const double nx = __dadd_rn(pre, best[i]);
      if (nx > target) { kstar = i; Pk = nx; Pkm1 = pre; break; }
      pre = nx;
    }
    if (kstar < 0) { kstar = i1 - 1; Pk = pre; Pkm1 = pre - best[kstar]; }
    // Error budget (rigorous, first order + slack): the reference's
    // cdf_k / cdf_last deviates from B_k/B_n by at most (k + n + 3)u
    // (sequential cumsum of k and n terms, p = b/T roundings, the division);
    // our fp64 prefix has <= ~1100u relative error (block tree + the final
    // in-block chain); the reference's best[] may differ from ours by the
    // rounding of its dgemv-ordered dot products: |delta d2| <= 8u(|x|+|c|)^2.
    const double n = (double)h.n;
    const double rel = ((double)kstar + n + 1200.0) * U0 * 1.05;
    const double absU = 32.0 * U0 * n * xsqmax;
    const double margin = rel * S + 2.0 * absU;
    s_ok = !force_replay && (Pk - target > margin) && (target - Pkm1 >= margin);
    if (s_ok) picks[draw] = kstar;
  }
  __syncthreads();
  if (s_ok) return;
  // ---- exact replay of Generator.choice(n, p=best/total) (clustering.py:48):
  // total = numpy pairwise sum; p = best/total; cdf = sequential cumsum;
  // idx = first i with fl(cdf_i / cdf_last) > u.  Everything but the cumsum
  // chain runs on all threads of the block.
  for (int64_t l = tid; l < nleaves; l += PS_THREADS) lsum[l] = np_leaf(best + leaves[2 * l], leaves[2 * l + 1]);
  __syncthreads();
  if (tid == 0) s_total = np_combine(lsum, h.n);
  __syncthreads();
  const double total = s_total;
  for (int64_t i = tid; i < h.n; i += PS_THREADS) pbuf[i] = __ddiv_rn(best[i], total);
  __syncthreads();
  // The sequential cumsum chain runs once on thread 0 over shared-memory tiles
  // that the rest of the block streams in (double buffered) and writes back
  // (cdf values -> cbuf); the crossing is then found by binary search.
  __shared__ double tile[2][PS_TILE];
  __shared__ double s_c;
  const int64_t ntile = (h.n + PS_TILE - 1) / PS_TILE;
  for (int64_t i = tid; i < min((int64_t)PS_TILE, h.n); i += PS_THREADS) tile[0][i] = pbuf[i];
  if (tid == 0) s_c = 0.0;
  __syncthreads();
  for (int64_t tb = 0; tb < ntile; ++tb) {
    const int64_t nb0 = (tb + 1) * PS_TILE;
    if (tid >= 32) {
      // write back the previous tile's cdf, prefetch the next tile
      if (tb > 0) {
        const int64_t pb0 = (tb - 1) * PS_TILE;
        for (int64_t i = tid - 32; i < PS_TILE && pb0 + i < h.n; i += PS_THREADS - 32)
          cbuf[pb0 + i] = tile[(tb + 1) & 1][i];
      }
      __syncwarp();
      for (int64_t i = tid - 32; i < PS_TILE && nb0 + i < h.n; i += PS_THREADS - 32)
        tile[(tb + 1) & 1][i] = pbuf[nb0 + i];
    } else if (tid == 0) {
      double* tv = tile[tb & 1];
      const int lim = (int)min((int64_t)PS_TILE, h.n - tb * PS_TILE);
      double c = s_c;
      int t = 0;
      for (; t + 8 <= lim; t += 8) {
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          c = __dadd_rn(c, tv[t + e]);
          tv[t + e] = c;
        }
      }
      for (; t < lim; ++t) {
        c = __dadd_rn(c, tv[t]);
        tv[t] = c;
      }
      s_c = c;
    }
    __syncthreads();
  }
  {
    const int64_t pb0 = (ntile - 1) * PS_TILE;
    for (int64_t i = tid; i < PS_TILE && pb0 + i < h.n; i += PS_THREADS) cbuf[pb0 + i] = tile[(ntile - 1) & 1][i];
  }
  __syncthreads();
  if (tid == 0) {
    const double last = s_c;                             // cdf[-1]
    // largest c with fl(c / last) <= u; searchsorted(cdf / last, u, 'right')
    // == first i with cdf_i > c_thr (fl(c/last) is monotone in c)
    double c_thr = __dmul_rn(u, last);
    // c_thr >= 0: neighbouring doubles are the bit patterns -1 / +1
    while (__ddiv_rn(c_thr, last) > u) c_thr = __longlong_as_double(__double_as_longlong(c_thr) - 1);
    while (true) {
      const double nx = __longlong_as_double(__double_as_longlong(c_thr) + 1);
      if (__ddiv_rn(nx, last) > u) break;
      c_thr = nx;
    }
    int64_t lo = -1, hi = h.n - 1;   // cbuf[hi] = last > c_thr; find first index > c_thr
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (cbuf[mid] > c_thr) hi = mid; else lo = mid;
    }
    picks[draw] = hi;
    status[1] += 1;
  }
}

// ------------------------------------------------------------------ Lloyd
constexpr int AS_THREADS = 256;
template <int MM>
__global__ void __launch_bounds__(AS_THREADS) k_assign(HalfView h, const double* __restrict__ xsq,
                                                       const double* __restrict__ C64,
                                                       const int32_t* __restrict__ lab,
                                                       int32_t* __restrict__ newlab,
                                                       double* __restrict__ pd, int iter,
                                                       int64_t* __restrict__ status,
                                                       double* __restrict__ hsum) {
  extern __shared__ double ash[];
  if (status[2]) return;
  const int m = h.m;
  double* C = ash;                    // k*m
  double* csq = ash + (size_t)h.k * m; // k
  __shared__ double red[AS_THREADS / 32];
  __shared__ int chg;
  for (int e = threadIdx.x; e < h.k * m; e += AS_THREADS) C[e] = C64[e];
  if (threadIdx.x == 0) chg = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < h.k; c += AS_THREADS)
    csq[c] = einsum_sq([&](int t) { return C[c * m + t]; }, m);
  __syncthreads();
  const int64_t i = (int64_t)blockIdx.x * AS_THREADS + threadIdx.x;
  double my = 0.0;
  int changed = 0;
  if (i < h.n) {
    double x[MM];
#pragma unroll
    for (int t = 0; t < MM; ++t) x[t] = t < m ? (double)h.X[(size_t)t * h.n + i] : 0.0;
    const double xs = xsq[i];
    double bd = 0.0;
    int bl = 0;
    for (int c = 0; c < h.k; ++c) {
      const double* cr = C + c * m;
      double acc = 0.0;
#pragma unroll
      for (int t = 0; t < MM; ++t)
        if (t < m) acc = __fma_rn(x[t], cr[t], acc);
      const double d2 = sq_dist_expand(xs, acc, csq[c]);
      if (c == 0 || d2 < bd) { bd = d2; bl = c; }
    }
    newlab[i] = bl;
    pd[i] = bd;
    my = bd;
    if (iter > 0 && lab[i] != bl) changed = 1;
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) atomicOr(&chg, 1);
  for (int o = 16; o > 0; o >>= 1) my = __dadd_rn(my, __shfl_xor_sync(0xffffffffu, my, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = my;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < AS_THREADS / 32; ++w) t = __dadd_rn(t, red[w]);
    hsum[blockIdx.x] = t;
    if (chg) atomicAdd((unsigned long long*)&status[4], 1ull);
  }
}

// history, convergence flag (clustering.py:90-93)
__global__ void k_lloyd_ctl(const double* __restrict__ hsum, int64_t nb, int iter,
                            int64_t* __restrict__ status, double* __restrict__ history,
                            int32_t* __restrict__ n_iter) {
  __shared__ double red[32];
  if (status[2]) return;
  double s = 0.0;
  for (int64_t b = threadIdx.x; b < nb; b += blockDim.x) s = __dadd_rn(s, hsum[b]);
  for (int o = 16; o > 0; o >>= 1) s = __dadd_rn(s, __shfl_xor_sync(0xffffffffu, s, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < (int)(blockDim.x >> 5); ++w) t = __dadd_rn(t, red[w]);
    history[iter] = t;
    *n_iter = iter + 1;
    status[3] = iter + 1;
    if (iter > 0 && status[4] == 0) status[2] = 1;
    status[4] = 0;
  }
}

constexpr int LT = 4096;  // points per label tile
__global__ void k_label_hist(int64_t n, int k, const int64_t* __restrict__ status,
                             const int32_t* __restrict__ newlab, int32_t* __restrict__ lab,
                             int32_t* __restrict__ lhist) {
  if (status[2]) return;
  __shared__ int cnt[256];
  for (int c = threadIdx.x; c < k; c += blockDim.x) cnt[c] = 0;
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * LT;
  const int64_t i1 = min(n, i0 + LT);
  for (int64_t i = i0 + threadIdx.x; i < i1; i += blockDim.x) {
    const int32_t l = newlab[i];
    lab[i] = l;
    atomicAdd(&cnt[l], 1);
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) lhist[(size_t)blockIdx.x * k + c] = cnt[c];
}

// loff[tile][c] = start of (cluster c, tile) in the label-sorted order; counts[c]
__global__ void k_label_offsets(int64_t ntiles, int k, const int64_t* __restrict__ status,
                                const int32_t* __restrict__ lhist, int64_t* __restrict__ loff,
                                int64_t* __restrict__ counts) {
  if (status[2]) return;
  __shared__ int64_t tot[256];
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    int64_t s = 0;
    for (int64_t t = 0; t < ntiles; ++t) s += lhist[(size_t)t * k + c];
    tot[c] = s;
    counts[c] = s;
  }
  __syncthreads();
  for (int c = threadIdx.x; c < k; c += blockDim.x) {
    int64_t base = 0;
    for (int c2 = 0; c2 < c; ++c2) base += tot[c2];
    for (int64_t t = 0; t < ntiles; ++t) {
      loff[(size_t)t * k + c] = base;
      base += lhist[(size_t)t * k + c];
    }
  }
}

// one warp per tile, rounds of 32 ascending points: stable ranks via match_any
__global__ void k_label_scatter(int64_t n, int k, const int64_t* __restrict__ status,
                                const int32_t* __restrict__ lab, const int64_t* __restrict__ loff,
                                int64_t* __restrict__ perm) {
  if (status[2]) return;
  __shared__ int64_t cur[256];
  for (int c = threadIdx.x; c < k; c += 32) cur[c] = loff[(size_t)blockIdx.x * k + c];
  __syncwarp();
  const int lane = threadIdx.x;
  const int64_t i0 = (int64_t)blockIdx.x * LT;
  const int64_t i1 = min(n, i0 + LT);
  for (int64_t r = i0; r < i1; r += 32) {
    const int64_t i = r + lane;
    const bool live = i < i1;
    const int l = live ? lab[i] : -1;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    const unsigned grp = __match_any_sync(0xffffffffu, l) & act;
    if (live) {
      const int rank = __popc(grp & ((1u << lane) - 1u));
      perm[cur[l] + rank] = i;
    }
    __syncwarp();
    if (live && lane == __ffs(grp) - 1) cur[l] += __popc(grp);
    __syncwarp();
  }
}

// xs[t][k] = X[t][perm[k]]: every cluster's values become one contiguous run
// (label-sorted, index order inside a label) for the sequential sums below.
__global__ void k_gather_sorted(HalfView h, const int64_t* __restrict__ status, const int64_t* __restrict__ perm,
                                float* __restrict__ xs) {
  if (status[2]) return;
  const int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= h.n) return;
  const int64_t p = perm[k];
  for (int t = 0; t < h.m; ++t) xs[(size_t)t * h.n + k] = h.X[(size_t)t * h.n + p];
}

// centroid = (sequential fp64 sum over the cluster's points in index order) / count
// -- np.add.at order (clustering.py:96).  One thread per (cluster, dim) runs
// the dependent add chain over a contiguous, prefetchable run of xs.
__global__ void k_cluster_sums(HalfView h, const int64_t* __restrict__ status,
                               const float* __restrict__ xs, const int64_t* __restrict__ counts,
                               double* __restrict__ C64) {
  if (status[2]) return;
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= h.k * h.m) return;
  const int c = e / h.m, t = e % h.m;
  const int64_t cnt = counts[c];
  if (cnt == 0) return;
  int64_t start = 0;
  for (int c2 = 0; c2 < c; ++c2) start += counts[c2];
  const float* x = xs + (size_t)t * h.n + start;
  double acc = 0.0;
  int64_t p = 0;
  for (; p + 16 <= cnt; p += 16) {
    float v[16];
#pragma unroll
    for (int u = 0; u < 16; ++u) v[u] = __ldg(x + p + u);
#pragma unroll
    for (int u = 0; u < 16; ++u) acc = __dadd_rn(acc, (double)v[u]);
  }
  for (; p < cnt; ++p) acc = __dadd_rn(acc, (double)x[p]);
  C64[(size_t)c * h.m + t] = __ddiv_rn(acc, (double)cnt);
}

// empty clusters (ascending): farthest point (first argmax of point_d2 with
// already-taken points at -1) becomes the centroid and moves its label.
__global__ void k_reseed(HalfView h, const int64_t* __restrict__ status,
                         const int64_t* __restrict__ counts, double* __restrict__ far,
                         int32_t* __restrict__ lab, double* __restrict__ C64) {
  if (status[2]) return;
  __shared__ double bv[32];
  __shared__ int64_t bi[32];
  for (int c = 0; c < h.k; ++c) {
    if (counts[c] != 0) continue;
    double v = -INFINITY;
    int64_t vi = INT64_MAX;
    for (int64_t i = threadIdx.x; i < h.n; i += blockDim.x) {
      const double f = far[i];
      if (f > v) { v = f; vi = i; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      const double ov = __shfl_xor_sync(0xffffffffu, v, o);
      const int64_t oi = __shfl_xor_sync(0xffffffffu, vi, o);
      if (ov > v || (ov == v && oi < vi)) { v = ov; vi = oi; }
    }
    if ((threadIdx.x & 31) == 0) { bv[threadIdx.x >> 5] = v; bi[threadIdx.x >> 5] = vi; }
    __syncthreads();
    if (threadIdx.x == 0) {
      double w = bv[0];
      int64_t wi = bi[0];
      for (int k2 = 1; k2 < (int)(blockDim.x >> 5); ++k2)
        if (bv[k2] > w || (bv[k2] == w && bi[k2] < wi)) { w = bv[k2]; wi = bi[k2]; }
      for (int t = 0; t < h.m; ++t) C64[(size_t)c * h.m + t] = (double)h.X[(size_t)t * h.n + wi];
      lab[wi] = c;
      far[wi] = -1.0;
    }
    __syncthreads();
  }
}

__global__ void k_centroids_out(const double* __restrict__ C64, int km, float* __restrict__ out) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e < km) out[e] = __double2float_rn(C64[e]);
}

__global__ void k_status_init(int64_t* status, int k) {
  status[0] = k;
  status[1] = 0;
  status[2] = 0;
  status[3] = 0;
  status[4] = 0;
}

struct KMeansRun {
  HalfView h;
  BuildScratch* s;
  int32_t* labels;     // n (device, output)
  double* history;     // iters (device)
  int32_t* n_iter;     // 1 (device)
  float* cent_out;     // k*m (device)
  int iters;
};

static int kmeans_enqueue(const KMeansRun& r, int64_t first, const double* uni_h,
                          const int64_t* forced_h, cudaStream_t st) {
  BuildScratch& s = *r.s;
  const HalfView h = r.h;
  const int64_t n = h.n;
  const int k = h.k;
  const int m = h.m;
  if (m > 32) TACO_FAIL(TACO_ERR_PARAMETER, "half width %d exceeds 32", m);
  if (k > 256) TACO_FAIL(TACO_ERR_PARAMETER, "codebook size %d exceeds 256", k);
  const int64_t nbx = ceil_div(n, 256);
  const int64_t nbp = ceil_div(n, PP_BLOCK);
  const int64_t nba = ceil_div(n, AS_THREADS);
  const int64_t ntile = ceil_div(n, LT);
  TACO_TRY(s.xsq.ensure(8 * n));
  TACO_TRY(s.best.ensure(8 * n));
  TACO_TRY(s.bsum.ensure(8 * std::max(nbp, nbx)));
  TACO_TRY(s.picks.ensure(8 * k));
  TACO_TRY(s.uni.ensure(8 * std::max(k, 1)));
  TACO_TRY(s.forced.ensure(8 * std::max(k, 1)));
  TACO_TRY(s.status.ensure(8 * 8));
  TACO_TRY(s.C64.ensure(8 * (size_t)k * m));
  TACO_TRY(s.newlab.ensure(4 * n));
  TACO_TRY(s.pd.ensure(8 * n));
  TACO_TRY(s.perm.ensure(8 * n));
  TACO_TRY(s.lhist.ensure(4 * (size_t)ntile * k));
  TACO_TRY(s.loff.ensure(8 * (size_t)ntile * k));
  TACO_TRY(s.ctl.ensure(8 * k));       // counts
  TACO_TRY(s.hsum.ensure(8 * nba));
  TACO_TRY(s.draws.ensure(8 * nbx));   // xsq block maxima
  if (s.leaves_n != n) {                // numpy pairwise leaves of an n-array (exact replay)
    std::vector<int64_t> lv;
    pairwise_leaves(0, n, lv);
    s.nleaves = (int64_t)lv.size() / 2;
    TACO_TRY(s.leaves.ensure(8 * lv.size()));
    TACO_CHECK_CUDA(cudaMemcpy(s.leaves.p, lv.data(), 8 * lv.size(), cudaMemcpyHostToDevice));
    s.leaves_n = n;
  }
  TACO_TRY(s.pbuf.ensure(8 * std::max<int64_t>(n, s.nleaves)));
  TACO_TRY(s.cbuf.ensure(std::max<size_t>(8 * n, 4 * (size_t)n * m)));   // replay cdf / sorted X
  // xsq + its maximum (bound for the certified draw)
  k_xsq<<<(unsigned)nbx, 256, 0, st>>>(h, s.xsq.as<double>(), s.draws.as<double>());
  TACO_LAUNCHED();
  std::vector<double> bm(nbx);
  TACO_CHECK_CUDA(cudaMemcpyAsync(bm.data(), s.draws.p, 8 * nbx, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  double xsqmax = 0.0;
  for (double v : bm) xsqmax = std::max(xsqmax, v);
  TACO_CHECK_CUDA(cudaMemcpyAsync(s.picks.p, &first, 8, cudaMemcpyHostToDevice, st));
  if (k > 1) {
    TACO_CHECK_CUDA(cudaMemcpyAsync(s.uni.p, uni_h, 8 * (k - 1), cudaMemcpyHostToDevice, st));
    if (forced_h)
      TACO_CHECK_CUDA(cudaMemcpyAsync(s.forced.p, forced_h, 8 * (k - 1), cudaMemcpyHostToDevice, st));
  }
  k_status_init<<<1, 1, 0, st>>>(s.status.as<int64_t>(), k);
  TACO_LAUNCHED();
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};
  if (getenv("TACO_DEBUG_TIMING")) {
    for (auto& e : ev) cudaEventCreate(&e);
    cudaEventRecord(ev[0], st);
  }
  for (int ci = 0; ci < k; ++ci) {
    k_pp_update<<<(unsigned)nbp, PP_THREADS, 0, st>>>(h, s.xsq.as<double>(), s.picks.as<int64_t>(), ci,
                                                      s.best.as<double>(), s.C64.as<double>(),
                                                      s.bsum.as<double>());
    TACO_LAUNCHED();
    if (ci + 1 < k) {
      k_pp_search<<<1, PS_THREADS, 0, st>>>(h, s.best.as<double>(), s.bsum.as<double>(), nbp,
                                            s.uni.as<double>(), forced_h ? s.forced.as<int64_t>() : nullptr,
                                            xsqmax, ci, s.picks.as<int64_t>(), s.status.as<int64_t>(),
                                            s.leaves.as<int64_t>(), s.nleaves, s.cbuf.as<double>(),
                                            s.pbuf.as<double>(), s.cbuf.as<double>(), g_force_replay);
      TACO_LAUNCHED();
    }
  }
  if (ev[1]) cudaEventRecord(ev[1], st);
  const size_t ash = sizeof(double) * ((size_t)k * m + k);
  auto* kas = m <= 8 ? k_assign<8> : m <= 16 ? k_assign<16> : k_assign<32>;
  if (ash > 48 * 1024)
    TACO_CHECK_CUDA(cudaFuncSetAttribute(kas, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ash));
  for (int it = 0; it < r.iters; ++it) {
    kas<<<(unsigned)nba, AS_THREADS, ash, st>>>(h, s.xsq.as<double>(), s.C64.as<double>(), r.labels,
                                                s.newlab.as<int32_t>(), s.pd.as<double>(), it,
                                                s.status.as<int64_t>(), s.hsum.as<double>());
    TACO_LAUNCHED();
    k_lloyd_ctl<<<1, 1024, 0, st>>>(s.hsum.as<double>(), nba, it, s.status.as<int64_t>(), r.history,
                                    r.n_iter);
    TACO_LAUNCHED();
    k_label_hist<<<(unsigned)ntile, 256, 0, st>>>(n, k, s.status.as<int64_t>(), s.newlab.as<int32_t>(),
                                                  r.labels, s.lhist.as<int32_t>());
    TACO_LAUNCHED();
    k_label_offsets<<<1, 256, 0, st>>>(ntile, k, s.status.as<int64_t>(), s.lhist.as<int32_t>(),
                                       s.loff.as<int64_t>(), s.ctl.as<int64_t>());
    TACO_LAUNCHED();
    k_label_scatter<<<(unsigned)ntile, 32, 0, st>>>(n, k, s.status.as<int64_t>(), r.labels,
                                                    s.loff.as<int64_t>(), s.perm.as<int64_t>());
    TACO_LAUNCHED();
    k_gather_sorted<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(h, s.status.as<int64_t>(), s.perm.as<int64_t>(),
                                                               s.cbuf.as<float>());
    TACO_LAUNCHED();
    k_cluster_sums<<<(unsigned)ceil_div((int64_t)k * m, 32), 32, 0, st>>>(
        h, s.status.as<int64_t>(), s.cbuf.as<float>(), s.ctl.as<int64_t>(), s.C64.as<double>());
    TACO_LAUNCHED();
    k_reseed<<<1, 1024, 0, st>>>(h, s.status.as<int64_t>(), s.ctl.as<int64_t>(), s.pd.as<double>(),
                                 r.labels, s.C64.as<double>());
    TACO_LAUNCHED();
  }
  k_centroids_out<<<(unsigned)ceil_div((int64_t)k * m, 256), 256, 0, st>>>(s.C64.as<double>(), k * m,
                                                                            r.cent_out);
  TACO_LAUNCHED();
  if (ev[2]) {
    cudaEventRecord(ev[2], st);
    s.ev[0] = ev[0]; s.ev[1] = ev[1]; s.ev[2] = ev[2];
  }
  return TACO_OK;
}

// ================================================================== cells
__global__ void k_cell_hist(const int32_t* __restrict__ l1, const int32_t* __restrict__ l2, int64_t n,
                            int kp, int64_t chunk, uint32_t* __restrict__ chist) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  const int key = l1[i] * kp + l2[i];
  atomicAdd(&chist[(size_t)(i / chunk) * kp * kp + key], 1u);
}

// per chunk: offs[c*K2 + cell] = c*CH + exclusive prefix within the chunk
__global__ void k_cell_offsets(const uint32_t* __restrict__ chist, int K2, int64_t nchunks, int64_t n,
                               int64_t chunk, uint32_t* __restrict__ offs) {
  __shared__ uint32_t wsum[32];
  const int64_t c = blockIdx.x;
  const uint32_t* hc = chist + (size_t)c * K2;
  const int per = (K2 + blockDim.x - 1) / blockDim.x;
  const int a0 = threadIdx.x * per, a1 = min(K2, a0 + per);
  uint32_t loc = 0;
  for (int e = a0; e < a1; ++e) loc += hc[e];
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t v = loc;
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += x;
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0u;
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t x = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += x;
    }
    wsum[lane] = w;
  }
  __syncthreads();
  uint32_t run = (uint32_t)(c * chunk) + (wid ? wsum[wid - 1] : 0u) + v - loc;
  for (int e = a0; e < a1; ++e) {
    offs[(size_t)c * K2 + e] = run;
    run += hc[e];
  }
  if (c == nchunks - 1 && threadIdx.x == 0) offs[(size_t)nchunks * K2] = (uint32_t)n;
}

__global__ void k_cell_sizes(const uint32_t* __restrict__ chist, int K2, int64_t nchunks,
                             int64_t* __restrict__ gsize) {
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= K2) return;
  int64_t s = 0;
  for (int64_t c = 0; c < nchunks; ++c) s += chist[(size_t)c * K2 + e];
  gsize[e] = s;
}

// one warp per chunk: stable scatter of ascending ids into their cells
__global__ void k_cell_scatter(const int32_t* __restrict__ l1, const int32_t* __restrict__ l2,
                               int64_t n, int kp, int64_t chunk, uint32_t* __restrict__ cursor,
                               uint32_t* __restrict__ ids) {
  const int lane = threadIdx.x;
  const int64_t c = blockIdx.x;
  const int K2 = kp * kp;
  uint32_t* cur = cursor + (size_t)c * K2;
  const int64_t i0 = c * chunk;
  const int64_t i1 = min(n, i0 + chunk);
  for (int64_t r = i0; r < i1; r += 32) {
    const int64_t i = r + lane;
    const bool live = i < i1;
    const int key = live ? l1[i] * kp + l2[i] : -1;
    const unsigned act = __ballot_sync(0xffffffffu, live);
    const unsigned grp = __match_any_sync(0xffffffffu, key) & act;
    uint32_t base = 0;
    const int leader = live ? __ffs(grp) - 1 : 0;
    if (live && lane == leader) base = atomicAdd(&cur[key], (uint32_t)__popc(grp));
    base = __shfl_sync(0xffffffffu, base, leader);
    if (live) ids[base + __popc(grp & ((1u << lane) - 1u))] = (uint32_t)i;
  }
}

}  // namespace taco

using namespace taco;

namespace {
int ensure_half_streams(taco_index* idx, int want) {
  while ((int)idx->half_streams.size() < want) {
    cudaStream_t s;
    TACO_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    idx->half_streams.push_back(s);
  }
  return TACO_OK;
}
}  // namespace

extern "C" {

static int covariance_impl(const float* Xd, int64_t n, int d, cudaStream_t st, double* mean_h,
                           double* gram_h, int64_t* bad_row) {
  DevBuf bad, mean, part, G;
  int rc = TACO_OK;
  do {
    if ((rc = bad.ensure(8)) || (rc = mean.ensure(8 * d)) || (rc = G.ensure(8 * (size_t)d * d))) break;
    unsigned long long init = ~0ull;
    cudaMemcpyAsync(bad.p, &init, 8, cudaMemcpyHostToDevice, st);
    k_nonfinite<<<1184, 256, 0, st>>>(Xd, n * d, d, bad.as<unsigned long long>());
    count_launch();
    unsigned long long b = 0;
    cudaMemcpyAsync(&b, bad.p, 8, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    *bad_row = b == ~0ull ? -1 : (int64_t)b;
    if (b != ~0ull) break;
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_colmean_seq, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         2 * CM_TILE_BYTES));
    k_colmean_seq<<<(unsigned)ceil_div(d, CM_THREADS), CM_THREADS, 2 * CM_TILE_BYTES, st>>>(Xd, n, d,
                                                                                          mean.as<double>());
    count_launch();
    const int tiles = (int)ceil_div(d, GT);
    int splits = (int)std::max<int64_t>(1, std::min<int64_t>(ceil_div(592, tiles * tiles), ceil_div(n, 256)));
    const int64_t rows_per = ceil_div(ceil_div(n, splits), GK) * GK;
    splits = (int)ceil_div(n, rows_per);
    if ((rc = part.ensure(8 * (size_t)splits * d * d))) break;
    k_gram<<<dim3(tiles, tiles, splits), 256, 0, st>>>(Xd, n, d, mean.as<double>(), rows_per,
                                                      part.as<double>());
    count_launch();
    const int64_t dd = (int64_t)d * d;
    k_gram_reduce<<<(unsigned)ceil_div(dd, 256), 256, 0, st>>>(part.as<double>(), splits, dd, G.as<double>());
    count_launch();
    cudaMemcpyAsync(mean_h, mean.p, 8 * d, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(gram_h, G.p, 8 * dd, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; }
  } while (0);
  bad.release(); mean.release(); part.release(); G.release();
  return rc;
}

int taco_fit_covariance(taco_index* idx, double* mean_h, double* gram_h, int64_t* bad_row) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "no data uploaded");
  return covariance_impl(idx->X.as<float>(), idx->n, idx->d, idx->stream, mean_h, gram_h, bad_row);
}

int taco_covariance(int device, const float* X_h, int64_t n, int32_t d, double* mean_h, double* gram_h,
                    int64_t* bad_row) {
  TACO_TRY(with_device(device));
  DevBuf X;
  TACO_TRY(X.ensure(4 * (size_t)n * d));
  cudaError_t e = cudaMemcpy(X.p, X_h, 4 * (size_t)n * d, cudaMemcpyHostToDevice);
  if (e != cudaSuccess) { X.release(); TACO_FAIL(TACO_ERR_CUDA, "%s", cudaGetErrorString(e)); }
  int rc = covariance_impl(X.as<float>(), n, d, nullptr, mean_h, gram_h, bad_row);
  X.release();
  return rc;
}

int taco_kmeans_all(taco_index* idx, const int64_t* first_h, const double* uniforms_h,
                    const int64_t* forced_h, int32_t* degenerate_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_T) TACO_FAIL(TACO_ERR_STATE, "transformed data not available");
  const int H = 2 * idx->n_sub;
  const int kp = idx->kp;
  const int64_t n = idx->n;
  if (n < kp) TACO_FAIL(TACO_ERR_INSUFFICIENT, "%lld points cannot fill %d clusters", (long long)n, kp);
  const int NS = std::min(H, 16);
  TACO_TRY(ensure_half_streams(idx, NS));
  if ((int)idx->bs.size() < NS) idx->bs.resize(NS);
  TACO_TRY(idx->labels.ensure(sizeof(int32_t) * (size_t)n * H));
  TACO_TRY(idx->hist.ensure(sizeof(double) * (size_t)H * std::max(idx->iters, 1)));
  TACO_TRY(idx->niter.ensure(sizeof(int32_t) * H));
  TACO_TRY(idx->cb1.ensure(sizeof(float) * (size_t)idx->n_sub * kp * idx->m1));
  TACO_TRY(idx->cb2.ensure(sizeof(float) * (size_t)idx->n_sub * kp * std::max(idx->m2, 1)));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  std::vector<int64_t> status_h(8);
  for (int w0 = 0; w0 < H; w0 += NS) {
    const int w1 = std::min(H, w0 + NS);
    for (int hh = w0; hh < w1; ++hh) {
      const int j = hh / 2, b = hh % 2;
      KMeansRun r;
      const int m = b ? idx->m2 : idx->m1;
      r.h.X = idx->T.as<float>() + (size_t)(j * idx->s + (b ? idx->m1 : 0)) * n;
      r.h.n = n;
      r.h.m = m;
      r.h.k = kp;
      r.s = &idx->bs[hh - w0];
      r.labels = idx->labels.as<int32_t>() + (size_t)hh * n;
      r.history = idx->hist.as<double>() + (size_t)hh * idx->iters;
      r.n_iter = idx->niter.as<int32_t>() + hh;
      r.cent_out = b ? idx->cb2.as<float>() + (size_t)j * kp * idx->m2 : idx->cb1.as<float>() + (size_t)j * kp * idx->m1;
      r.iters = idx->iters;
      TACO_TRY(kmeans_enqueue(r, first_h[hh], uniforms_h + (size_t)hh * std::max(kp - 1, 0),
                              forced_h ? forced_h + (size_t)hh * std::max(kp - 1, 0) : nullptr,
                              idx->half_streams[hh - w0]));
    }
    for (int hh = w0; hh < w1; ++hh) {
      cudaStream_t st = idx->half_streams[hh - w0];
      TACO_CHECK_CUDA(cudaMemcpyAsync(status_h.data(), idx->bs[hh - w0].status.p, 8 * 5, cudaMemcpyDeviceToHost, st));
      TACO_CHECK_CUDA(cudaStreamSynchronize(st));
      degenerate_h[hh] = (int32_t)status_h[0];
      BuildScratch& bs = idx->bs[hh - w0];
      if (bs.ev[2]) {
        float a = 0.f, b = 0.f;
        cudaEventElapsedTime(&a, bs.ev[0], bs.ev[1]);
        cudaEventElapsedTime(&b, bs.ev[1], bs.ev[2]);
        fprintf(stderr, "[taco] half %d: k-means++ %.1f ms (replays %lld), Lloyd %.1f ms (iters %lld)\n", hh, a,
                (long long)status_h[1], b, (long long)status_h[3]);
        for (auto& e : bs.ev) { cudaEventDestroy(e); e = nullptr; }
      }
    }
  }
  idx->has_cb = true;
  idx->has_labels = true;
  return TACO_OK;
}

int taco_build_cells(taco_index* idx) {
  TACO_TRY(index_check(idx));
  if (!idx->has_labels) TACO_FAIL(TACO_ERR_STATE, "labels not available");
  const int64_t n = idx->n, nc = idx->nchunks;
  const int kp = idx->kp, K2 = kp * kp;
  const size_t offs_len = (size_t)nc * K2 + 1;
  cudaStream_t st = idx->stream;
  for (auto s : idx->half_streams) TACO_CHECK_CUDA(cudaStreamSynchronize(s));
  TACO_TRY(idx->ids.ensure(sizeof(uint32_t) * (size_t)n * idx->n_sub));
  TACO_TRY(idx->offs.ensure(sizeof(uint32_t) * offs_len * idx->n_sub));
  TACO_TRY(idx->gsize.ensure(sizeof(int64_t) * (size_t)K2 * idx->n_sub));
  DevBuf chist, cursor;
  TACO_TRY(chist.ensure(sizeof(uint32_t) * (size_t)nc * K2));
  TACO_TRY(cursor.ensure(sizeof(uint32_t) * (size_t)nc * K2));
  for (int j = 0; j < idx->n_sub; ++j) {
    const int32_t* l1 = idx->labels.as<int32_t>() + (size_t)(2 * j) * n;
    const int32_t* l2 = idx->labels.as<int32_t>() + (size_t)(2 * j + 1) * n;
    uint32_t* offs = idx->offs.as<uint32_t>() + (size_t)j * offs_len;
    TACO_CHECK_CUDA(cudaMemsetAsync(chist.p, 0, sizeof(uint32_t) * (size_t)nc * K2, st));
    k_cell_hist<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(l1, l2, n, kp, idx->chunk, chist.as<uint32_t>());
    TACO_LAUNCHED();
    k_cell_offsets<<<(unsigned)nc, 1024, 0, st>>>(chist.as<uint32_t>(), K2, nc, n, idx->chunk, offs);
    TACO_LAUNCHED();
    if (idx->n_global == idx->n) {
      k_cell_sizes<<<(unsigned)ceil_div(K2, 256), 256, 0, st>>>(chist.as<uint32_t>(), K2, nc,
                                                               idx->gsize.as<int64_t>() + (size_t)j * K2);
      TACO_LAUNCHED();
    }
    TACO_CHECK_CUDA(cudaMemcpyAsync(cursor.p, offs, sizeof(uint32_t) * (size_t)nc * K2, cudaMemcpyDeviceToDevice, st));
    k_cell_scatter<<<(unsigned)nc, 32, 0, st>>>(l1, l2, n, kp, idx->chunk, cursor.as<uint32_t>(),
                                                idx->ids.as<uint32_t>() + (size_t)j * n);
    TACO_LAUNCHED();
  }
  cudaError_t e = cudaStreamSynchronize(st);
  chist.release();
  cursor.release();
  if (e != cudaSuccess) TACO_FAIL(TACO_ERR_CUDA, "%s", cudaGetErrorString(e));
  idx->has_cells = true;
  if (idx->n_global == idx->n) idx->has_gsize = true;
  return TACO_OK;
}

// local cell sizes of a shard (to be all-reduced into global sizes)
int taco_get_local_sizes(taco_index* idx, int64_t* sizes_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_cells) TACO_FAIL(TACO_ERR_STATE, "cells not built");
  const int64_t nc = idx->nchunks;
  const int K2 = idx->kp * idx->kp;
  const size_t offs_len = (size_t)nc * K2 + 1;
  std::vector<uint32_t> offs(offs_len);
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  for (int j = 0; j < idx->n_sub; ++j) {
    TACO_CHECK_CUDA(cudaMemcpy(offs.data(), idx->offs.as<uint32_t>() + (size_t)j * offs_len,
                               sizeof(uint32_t) * offs_len, cudaMemcpyDeviceToHost));
    for (int c = 0; c < K2; ++c) {
      int64_t s = 0;
      for (int64_t ch = 0; ch < nc; ++ch) s += offs[ch * K2 + c + 1] - offs[ch * K2 + c];
      sizes_h[(size_t)j * K2 + c] = s;
    }
  }
  return TACO_OK;
}

// Test hook: 1 = every k-means++ draw takes the exact numpy replay path.
int taco_debug_force_replay(int on) {
  g_force_replay = on ? 1 : 0;
  return TACO_OK;
}

int taco_kmeans(int device, const float* X_h, int64_t n, int32_t m, int32_t k, int32_t max_iter,
                int64_t first, const double* uniforms_h, const int64_t* forced_h, float* centroids_h,
                int32_t* labels_h, double* history_h, int32_t* n_iter_h, int32_t* degenerate_h) {
  TACO_TRY(with_device(device));
  if (k < 1) TACO_FAIL(TACO_ERR_PARAMETER, "cluster count must be positive, got %d", k);
  if (max_iter < 1) TACO_FAIL(TACO_ERR_PARAMETER, "iteration cap must be positive, got %d", max_iter);
  if (n < k) TACO_FAIL(TACO_ERR_INSUFFICIENT, "%lld points cannot fill %d clusters", (long long)n, k);
  // dimension-major copy
  std::vector<float> tr((size_t)n * m);
  for (int64_t i = 0; i < n; ++i)
    for (int t = 0; t < m; ++t) tr[(size_t)t * n + i] = X_h[(size_t)i * m + t];
  DevBuf X, lab, hist, nit, cent;
  BuildScratch s;
  int rc = TACO_OK;
  cudaStream_t st = nullptr;
  do {
    if ((rc = X.ensure(4 * tr.size())) || (rc = lab.ensure(4 * n)) || (rc = hist.ensure(8 * max_iter)) ||
        (rc = nit.ensure(4)) || (rc = cent.ensure(4 * (size_t)k * m)))
      break;
    cudaMemcpy(X.p, tr.data(), 4 * tr.size(), cudaMemcpyHostToDevice);
    KMeansRun r;
    r.h.X = X.as<float>();
    r.h.n = n;
    r.h.m = m;
    r.h.k = k;
    r.s = &s;
    r.labels = lab.as<int32_t>();
    r.history = hist.as<double>();
    r.n_iter = nit.as<int32_t>();
    r.cent_out = cent.as<float>();
    r.iters = max_iter;
    if ((rc = kmeans_enqueue(r, first, uniforms_h, forced_h, st))) break;
    std::vector<int64_t> status(5);
    cudaMemcpy(status.data(), s.status.p, 8 * 5, cudaMemcpyDeviceToHost);
    cudaMemcpy(centroids_h, cent.p, 4 * (size_t)k * m, cudaMemcpyDeviceToHost);
    cudaMemcpy(labels_h, lab.p, 4 * n, cudaMemcpyDeviceToHost);
    cudaMemcpy(history_h, hist.p, 8 * max_iter, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(n_iter_h, nit.p, 4, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    *degenerate_h = (int32_t)status[0];
  } while (0);
  X.release(); lab.release(); hist.release(); nit.release(); cent.release();
  DevBuf* sb[] = {&s.xsq, &s.best, &s.bsum, &s.picks, &s.uni, &s.forced, &s.status, &s.C64, &s.csq,
                  &s.newlab, &s.pd, &s.changed, &s.perm, &s.lhist, &s.loff, &s.ctl, &s.hsum, &s.draws,
                  &s.leaves, &s.pbuf, &s.cbuf};
  for (auto* b : sb) b->release();
  return rc;
}

}  // extern "C"
