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
#include <cstring>
#include <array>
#include <climits>
#include <ctime>
#include <cmath>
#include <cstdlib>
#include <mutex>
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
// r = 1..n-1 (row-sequential), then / n.  The add chain is inherently
// sequential per column, so the kernel is built to run at the dependent-DADD
// latency floor: one CTA per 32-column slab, warp 0 = the 32 chains (lane =
// column), warps 1..3 stream the slab's rows into an 8-stage shared-memory
// ring with cp.async (16-byte pieces when the slab is 16-byte aligned) so the
// chain never waits on HBM.  One __syncthreads per 128-row stage.
// One dependent fp64 add chain over rr floats at stride `st` in shared memory
// (acc += x_0, acc += x_1, ... in order).  Values are pulled into registers
// 64 at a time (both 32-halves issued before the first add), so the chain
// waits on LDS latency once per 64 adds and otherwise runs at the DADD
// latency (11 cycles on B200).
__device__ __forceinline__ double chain_add(double acc, const float* __restrict__ tv, int rr, int st) {
  int q = 0;
  for (; q + 64 <= rr; q += 64) {
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
  if (q + 32 <= rr) {
    float a[32];
#pragma unroll
    for (int u = 0; u < 32; ++u) a[u] = tv[(q + u) * st];
#pragma unroll
    for (int u = 0; u < 32; ++u) acc = __dadd_rn(acc, (double)a[u]);
    q += 32;
  }
  for (; q < rr; ++q) acc = __dadd_rn(acc, (double)tv[q * st]);
  return acc;
}

constexpr int CM_W = 32;          // columns per CTA
constexpr int CM_ROWS = 128;      // rows per stage
constexpr int CM_STAGES = 8;
constexpr int CM_THREADS = 128;   // 1 consumer warp + 3 producer warps
constexpr size_t CM_SMEM = sizeof(float) * CM_STAGES * CM_ROWS * CM_W;

__device__ __forceinline__ void cp_async4(void* s, const void* g) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cp_async16(void* s, const void* g) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;\n" ::"r"((unsigned)__cvta_generic_to_shared(s)), "l"(g));
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;\n" ::); }
template <int N>
__device__ __forceinline__ void cp_wait() { asm volatile("cp.async.wait_group %0;\n" ::"n"(N)); }

// Rows [r0, r1) of the chain; state[] carries each column's running sum
// between launches (r0 == 0 starts from X[0]), and the launch that reaches
// row n divides (the staged upload runs one launch per landed chunk).
__global__ void __launch_bounds__(CM_THREADS) k_colmean_seq(const float* __restrict__ X, int64_t r0g, int64_t r1g,
                                                            int64_t n, int d, double* __restrict__ state,
                                                            double* __restrict__ mean, int chained) {
  extern __shared__ __align__(16) float cm[];
  const int c0 = blockIdx.x * CM_W;
  const int nc = min(CM_W, d - c0);
  const int tid = threadIdx.x;
  const int64_t nrow = r1g - r0g;
  const int64_t ntile = (nrow + CM_ROWS - 1) / CM_ROWS;
  const bool vec = (d % 4 == 0) && (nc % 4 == 0) && ((reinterpret_cast<uintptr_t>(X) & 15) == 0);
  const int ptid = tid - 32;   // producer index (warps 1..3)
  auto load = [&](int64_t tb) {
    if (tb < ntile) {
      float* dst = cm + (size_t)(tb % CM_STAGES) * CM_ROWS * CM_W;
      const int64_t r0 = r0g + tb * CM_ROWS;
      const int rr = (int)min((int64_t)CM_ROWS, r1g - r0);
      if (vec) {
        const int per = nc / 4;
        for (int e = ptid; e < rr * per; e += CM_THREADS - 32) {
          const int r = e / per, q = e - r * per;
          cp_async16(dst + r * CM_W + 4 * q, X + (r0 + r) * d + c0 + 4 * q);
        }
      } else {
        for (int e = ptid; e < rr * nc; e += CM_THREADS - 32) {
          const int r = e / nc, c = e - r * nc;
          cp_async4(dst + r * CM_W + c, X + (r0 + r) * d + c0 + c);
        }
      }
    }
    cp_commit();
  };
  if (tid >= 32)
    for (int s = 0; s < CM_STAGES - 1; ++s) load(s);
  // chained: this device's row 0 continues a chain begun on an earlier shard
  double acc = ((r0g > 0 || chained) && tid < nc) ? state[c0 + tid] : 0.0;
  for (int64_t tb = 0; tb < ntile; ++tb) {
    if (tid >= 32) cp_wait<CM_STAGES - 2>();   // tile tb has landed (this thread's pieces)
    __syncthreads();                             // ... everyone's; slot (tb-1)%S is free
    if (tid >= 32) {
      load(tb + CM_STAGES - 1);
    } else if (tid < nc) {
      const float* tv = cm + (size_t)(tb % CM_STAGES) * CM_ROWS * CM_W + tid;
      const int rr = (int)min((int64_t)CM_ROWS, nrow - tb * CM_ROWS);
      if (tb == 0 && r0g == 0 && !chained) acc = chain_add((double)tv[0], tv + CM_W, rr - 1, CM_W);
      else acc = chain_add(acc, tv, rr, CM_W);
    }
  }
  if (tid < nc) {
    state[c0 + tid] = acc;
    if (r1g == n && mean) mean[c0 + tid] = __ddiv_rn(acc, (double)n);
  }
}

int launch_colmean(cudaStream_t st, const float* X, int64_t r0, int64_t r1, int64_t n, int d, double* state,
                   double* mean, int chained) {
  static bool attr = false;
  if (!attr) {
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_colmean_seq, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)CM_SMEM));
    attr = true;
  }
  if (r1 <= r0) return TACO_OK;
  k_colmean_seq<<<(unsigned)ceil_div(d, CM_W), CM_THREADS, CM_SMEM, st>>>(X, r0, r1, n, d, state, mean, chained);
  TACO_LAUNCHED();
  return TACO_OK;
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

// G += partial[0] + partial[1] + ... (sequential, in block order).  The Gram
// is a chain over fixed blocks of kGramBlock rows (the block partials are the
// only parallel part), so a point-sharded build whose shards start on block
// boundaries reproduces it exactly by carrying G from shard to shard.
__global__ void k_gram_accum(const double* __restrict__ partial, int splits, int64_t dd,
                             double* __restrict__ G) {
  const int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= dd) return;
  double acc = G[e];
  for (int s = 0; s < splits; ++s) acc = __dadd_rn(acc, partial[(size_t)s * dd + e]);
  G[e] = acc;
}

constexpr int64_t kGramBlock = 4096;   // rows per Gram partial (a multiple of GK)

// G (device, d x d, holding the carried-in sum) += the centred Gram of rows
// [0, n) of X, block by block; partial memory bounded by grouping blocks.
static int gram_chain(const float* X, int64_t n, int d, const double* mean_d, int64_t block_rows, double* G,
                      cudaStream_t st) {
  if (n <= 0) return TACO_OK;
  if (block_rows < GK || block_rows % GK) TACO_FAIL(TACO_ERR_PARAMETER, "Gram block of %lld rows", (long long)block_rows);
  const int tiles = (int)ceil_div(d, GT);
  const int64_t dd = (int64_t)d * d;
  const int64_t nblocks = ceil_div(n, block_rows);
  const int64_t group = std::max<int64_t>(1, std::min<int64_t>(nblocks, ((int64_t)1 << 30) / (8 * dd)));
  DevBuf part;
  TACO_TRY(part.ensure(8 * (size_t)group * dd));
  for (int64_t b0 = 0; b0 < nblocks; b0 += group) {
    const int64_t nb = std::min(group, nblocks - b0);
    const int64_t r0 = b0 * block_rows;
    const int64_t rows = std::min(n - r0, nb * block_rows);
    k_gram<<<dim3(tiles, tiles, (unsigned)nb), 256, 0, st>>>(X + (size_t)r0 * d, rows, d, mean_d, block_rows,
                                                            part.as<double>());
    count_launch();
    k_gram_accum<<<(unsigned)ceil_div(dd, 256), 256, 0, st>>>(part.as<double>(), (int)nb, dd, G);
    count_launch();
  }
  cudaError_t e = cudaStreamSynchronize(st);   // part is released below
  part.release();
  if (e != cudaSuccess) TACO_FAIL(TACO_ERR_CUDA, "%s", cudaGetErrorString(e));
  return TACO_OK;
}

// ================================================================ k-means
constexpr int PP_THREADS = 256;
constexpr int PP_PPT = 4;                       // points per thread in one block
constexpr int PP_BLOCK = PP_THREADS * PP_PPT;   // points per block-sum
constexpr double U0 = 1.1102230246251565e-16;   // 2^-53

static int g_force_replay = 0;   // test hook: always take the exact replay

static int g_num_sms() {
  static int sms = 0;
  if (!sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    if (sms <= 0) sms = 148;
  }
  return sms;
}

struct HalfView {
  const float* X;   // dimension-major: X[t*n + i]
  int64_t n;
  int m;
  int k;
};

__global__ void k_xsq(HalfView h, double* __restrict__ xsq, int64_t* __restrict__ status) {
  __shared__ double red[32], reds[32];
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  double v = 0.0;
  if (i < h.n) {
    v = einsum_sq([&](int t) { return (double)h.X[(size_t)t * h.n + i]; }, h.m);
    xsq[i] = v;
  }
  double sv = v;
  for (int o = 16; o > 0; o >>= 1) {
    v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
    sv += __shfl_xor_sync(0xffffffffu, sv, o);
  }
  if ((threadIdx.x & 31) == 0) {
    red[threadIdx.x >> 5] = v;
    reds[threadIdx.x >> 5] = sv;
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    double w = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0.0;
    double ws = threadIdx.x < (blockDim.x >> 5) ? reds[threadIdx.x] : 0.0;
    for (int o = 16; o > 0; o >>= 1) {
      w = fmax(w, __shfl_xor_sync(0xffffffffu, w, o));
      ws += __shfl_xor_sync(0xffffffffu, ws, o);
    }
    // non-negative doubles order like their bit patterns; the sum of xsq (a
    // bound input, any order) for the k-means++ certificate
    if (threadIdx.x == 0) {
      atomicMax(reinterpret_cast<unsigned long long*>(status + 5), (unsigned long long)__double_as_longlong(w));
      atomicAdd(reinterpret_cast<double*>(status + 8), ws);
    }
  }
}

// status layout (int64): [0] degenerate draw index (k if none), [1] fallbacks,
// [2] converged flag, [3] n_iter, [4] changed count, [5] max xsq (double bits)
// numpy pairwise summation (loops_utils.h.src, as measured in DESIGN.md §4):
// n < 8 sequential; n <= 128 eight strided accumulators combined
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) then the tail; else split at
// n2 = n/2 - (n/2)%8 and add the halves.  The leaves (ranges <= 128) depend
// only on n and are listed once on the host in depth-first order.
// The combine tree of that recursion: internal node = (left, right) ids over
// [0, nleaves) = leaves (DFS order) and nleaves + i = internal node i; nodes
// are ordered by height so a level-synchronous pass meets children first.
struct PwTree {
  std::vector<int32_t> left, right, level_start;
};
static int pw_build(int64_t len, int& leaf_ctr, std::vector<std::array<int32_t, 3>>& tmp) {
  // returns the node's temporary id: leaves -> (leaf index), internal -> -(1 + tmp index)
  if (len <= 128) return leaf_ctr++;
  int64_t n2 = len / 2;
  n2 -= n2 % 8;
  const int l = pw_build(n2, leaf_ctr, tmp);
  const int r = pw_build(len - n2, leaf_ctr, tmp);
  auto height = [&](int id) { return id >= 0 ? 0 : tmp[-1 - id][2]; };
  tmp.push_back({l, r, 1 + std::max(height(l), height(r))});
  return -(int)tmp.size();
}
static PwTree pairwise_tree(int64_t n) {
  PwTree t;
  std::vector<std::array<int32_t, 3>> tmp;
  int leaves = 0;
  pw_build(n, leaves, tmp);
  const int ni = (int)tmp.size();
  std::vector<int> order(ni);
  for (int i = 0; i < ni; ++i) order[i] = i;
  std::stable_sort(order.begin(), order.end(), [&](int a, int b) { return tmp[a][2] < tmp[b][2]; });
  std::vector<int> rank(ni);
  for (int i = 0; i < ni; ++i) rank[order[i]] = i;
  auto final_id = [&](int id) { return id >= 0 ? id : leaves + rank[-1 - id]; };
  int cur = 0;
  for (int i = 0; i < ni; ++i) {
    const auto& nd = tmp[order[i]];
    if (i == 0 || nd[2] != cur) { t.level_start.push_back(i); cur = nd[2]; }
    t.left.push_back(final_id(nd[0]));
    t.right.push_back(final_id(nd[1]));
  }
  t.level_start.push_back(ni);
  return t;
}

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
    for (int64_t i = 0; i < len; ++i) r = __dadd_rn(r, __ldcg(a + i));
    return r;
  }
  double r[8];
  for (int j = 0; j < 8; ++j) r[j] = __ldcg(a + j);
  int64_t i = 8;
  for (; i < len - (len % 8); i += 8)
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], __ldcg(a + i + j));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < len; ++i) res = __dadd_rn(res, __ldcg(a + i));
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

// numpy's sequential cumsum (np.add.accumulate) of p[0..n) reproduced
// bit-exactly by one CTA without the n-step dependent chain.  While the
// running value c stays in one binade [2^e, 2^(e+1)), every step
// fl(c + p_k) = c + g * round(p_k / g) with g = ulp = 2^(e-52) (c is a multiple
// of g), so the chain inside a binade is an exact int64 prefix sum of the
// rounded quotients q_k.  A parallel scan finds the first element that leaves
// the binade (c + g*Q_k >= 2^(e+1)) or whose quotient is an exact tie (round to
// even depends on the running value); that one element is added with a real
// fp64 add and the scan resumes from it.  There are ~log2(S / c_0) binade
// changes, so the work is one pass over p plus O(log n) short restarts.
constexpr int CX_V = 16;   // elements per thread per chunk
// The range form: c_k = fl(c_{k-1} + p_k) for k in [i0, i1), starting from
// c_in (started = false: the range begins the cumsum, c_{i0} = p_{i0}).  Writes
// cdf[k - i0] when cdf is non-null; returns the last value (every thread).
__device__ double cumsum_exact_range(const double* __restrict__ best, double total, int64_t i0, int64_t i1,
                                     double c_in, bool started, double* __restrict__ cdf) {
  // p_k = best_k / total (numpy's elementwise division), formed on the fly
  auto P = [&](int64_t k) { return __ddiv_rn(__ldcg(best + k), total); };
  __shared__ double s_crun;
  __shared__ long long s_i, s_stop, s_pq;
  __shared__ long long s_wq[32];
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NT = blockDim.x, NW = NT >> 5;
  if (tid == 0) {
    // head: sequential until the running value is a normal double well above underflow
    double c = c_in;
    int64_t i = i0;
    if (!started && i < i1) {
      c = P(i);
      if (cdf) cdf[0] = c;
      ++i;
    }
    while (i < i1 && !(c >= 0x1p-900)) {
      c = __dadd_rn(c, P(i));
      if (cdf) cdf[i - i0] = c;
      ++i;
    }
    s_crun = c;
    s_i = i;
    s_stop = LLONG_MAX;
  }
  __syncthreads();
  while (true) {
    const int64_t ib = s_i;
    if (ib >= i1) break;
    const double crun = s_crun;
    const int e = ilogb(crun);
    const double g = scalbn(1.0, e - 52), inv = scalbn(1.0, 52 - e);
    const long long Qlim = (long long)__dmul_rn(__dsub_rn(scalbn(1.0, e + 1), crun), inv);   // exact
    long long Qbase = 0;
    long long stop = LLONG_MAX;
    for (int64_t j0 = ib; j0 < i1; j0 += (int64_t)NT * CX_V) {
      long long lp[CX_V];
      long long tsum = 0;
      int tie = CX_V;
      double bv[CX_V];   // this thread's values: loads first (all in flight), then the quotients
#pragma unroll
      for (int v = 0; v < CX_V; ++v) {
        const int64_t k = j0 + (int64_t)tid * CX_V + v;
        bv[v] = k < i1 ? __ldcg(best + k) : 0.0;
      }
#pragma unroll
      for (int v = 0; v < CX_V; ++v) {
        const int64_t k = j0 + (int64_t)tid * CX_V + v;
        long long q = 0;
        if (k < i1) {
          const double t = __dmul_rn(__ddiv_rn(bv[v], total), inv);   // p_k, then exact power-of-two scaling
          if (t >= 0x1p60) {
            q = 1LL << 60;                         // certainly leaves the binade
          } else {
            const double fl = floor(t), fr = __dsub_rn(t, fl);
            q = (long long)fl + (fr > 0.5 ? 1 : 0);
            if (fr == 0.5 && tie == CX_V) tie = v;
          }
        }
        tsum += q;
        lp[v] = tsum;
      }
      // block exclusive scan of the thread totals
      long long incl = tsum;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_wq[wid] = incl;
      __syncthreads();
      if (wid == 0) {
        long long w = lane < NW ? s_wq[lane] : 0;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += y;
        }
        s_wq[lane] = w;
      }
      __syncthreads();
      const long long excl = Qbase + (wid ? s_wq[wid - 1] : 0) + (incl - tsum);
      const long long chunk_tot = s_wq[NW - 1];
#pragma unroll
      for (int v = 0; v < CX_V; ++v) {
        const int64_t k = j0 + (int64_t)tid * CX_V + v;
        if (k < i1 && (excl + lp[v] >= Qlim || v == tie)) {
          atomicMin(&s_stop, (long long)k);
          break;
        }
      }
      __syncthreads();
      stop = s_stop;
      {
        // the owner of the stop element records the quotient prefix before it
        const int64_t rel = stop - j0 - (int64_t)tid * CX_V;
        if (rel >= 0 && rel < CX_V) {
          long long pq = excl;
#pragma unroll
          for (int v = 0; v < CX_V; ++v)
            if (v < rel) pq = excl + lp[v];
          s_pq = pq;
        }
      }
      if (cdf) {
#pragma unroll
        for (int v = 0; v < CX_V; ++v) {
          const int64_t k = j0 + (int64_t)tid * CX_V + v;
          if (k < i1 && k < stop) cdf[k - i0] = __dadd_rn(crun, __dmul_rn((double)(excl + lp[v]), g));   // exact
        }
      }
      __syncthreads();   // s_wq / s_stop / s_pq, cdf visible
      if (stop != LLONG_MAX) break;
      Qbase += chunk_tot;
    }
    if (tid == 0) {
      if (stop == LLONG_MAX) {
        // ran to the end inside this binade: c = crun + g * Q (exact)
        s_crun = __dadd_rn(crun, __dmul_rn((double)Qbase, g));
        s_i = i1;
      } else {
        const double prev = __dadd_rn(crun, __dmul_rn((double)s_pq, g));   // exact (s_pq < Qlim)
        const double c = __dadd_rn(prev, P(stop));   // the element that leaves the binade (or ties)
        if (cdf) cdf[stop - i0] = c;
        s_crun = c;
        s_i = stop + 1;
        s_stop = LLONG_MAX;
      }
    }
    __syncthreads();
  }
  const double r = s_crun;
  __syncthreads();
  return r;
}

__device__ void cumsum_exact_block(const double* __restrict__ best, double total, int64_t n, double* __restrict__ cdf) {
  cumsum_exact_range(best, total, 0, n, 0.0, false, cdf);
}

// One CTA: chooses picks[ci+1] from best (after centroids 0..ci) and u.
// Fast path: fp64 prefix over block sums, locate the crossing, then certify
// that numpy's sequential cumsum/normalise/searchsorted (the reference's
// Generator.choice, clustering.py:48) cannot land elsewhere.  Otherwise
// replay numpy's arithmetic exactly (single thread).
constexpr int PS_TILE = 2048;   // doubles per staged tile of the replay chain
__device__ __forceinline__ void pp_search_body(HalfView h, const double* __restrict__ best,
                                                          const double* __restrict__ bsum, int64_t nb,
                                                          const double* __restrict__ uni,
                                                          const int64_t* __restrict__ forced,
                                                          int ci,
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
  const int NT = blockDim.x, NW = NT >> 5;
  const int draw = ci + 1;                 // centroid index being chosen
  if (forced && forced[ci] >= 0) {
    if (tid == 0) picks[draw] = forced[ci];
    return;
  }
  // per-thread contiguous block-sum ranges, then a block scan (fixed order)
  const int64_t per = (nb + NT - 1) / NT;
  const int64_t a0 = (int64_t)tid * per, a1 = min(nb, a0 + per);
  double loc = 0.0;
  for (int64_t b = a0; b < a1; ++b) loc = __dadd_rn(loc, __ldcg(bsum + b));
  double v = loc;
  for (int o = 1; o < 32; o <<= 1) {
    double x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v = __dadd_rn(v, x);
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    double w = lane < NW ? wsum[lane] : 0.0;
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
      const double nx = __dadd_rn(pre, __ldcg(bsum + b));
      if (nx > target && pre <= target) {
        s_blk = b;
        s_before = pre;
      }
      pre = nx;
    }
  }
  __syncthreads();
  __shared__ int s_ok;
  __shared__ double s_scan[PP_BLOCK];
  __shared__ int s_k;
  int64_t blk = s_blk;
  if (blk < 0) blk = nb - 1;   // rounding put the target at/after the end
  const double pre = s_blk >= 0 ? s_before : S - __ldcg(bsum + blk);
  const int64_t i0 = blk * PP_BLOCK, i1 = min(h.n, i0 + PP_BLOCK);
  {
    // in-block inclusive prefix of best[] (PP_BLOCK / NT consecutive values
    // per thread, then a block scan of the thread totals: a fp64 tree whose
    // error is far inside the certified budget below), then the first crossing
    constexpr int VPT_MAX = 8;
    const int vpt = PP_BLOCK / NT;
    double loc2[VPT_MAX];
    double tsum = 0.0;
#pragma unroll
    for (int e = 0; e < VPT_MAX; ++e) {
      if (e < vpt) {
        const int64_t i = i0 + (int64_t)tid * vpt + e;
        tsum = __dadd_rn(tsum, i < i1 ? __ldcg(best + i) : 0.0);
        loc2[e] = tsum;
      }
    }
    double sv = tsum;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, sv, o);
      if (lane >= o) sv = __dadd_rn(sv, y);
    }
    __syncthreads();   // wsum reuse
    if (lane == 31) wsum[wid] = sv;
    if (tid == 0) s_k = PP_BLOCK;
    __syncthreads();
    if (wid == 0) {
      double w = lane < NW ? wsum[lane] : 0.0;
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w = __dadd_rn(w, y);
      }
      wsum[lane] = w;
    }
    __syncthreads();
    const double prevlane = __shfl_up_sync(0xffffffffu, sv, 1);   // warp-inclusive prefix of lane - 1
    const double wbase = wid ? wsum[wid - 1] : 0.0;
    const double base = lane ? __dadd_rn(wbase, prevlane) : wbase;
#pragma unroll
    for (int e = 0; e < VPT_MAX; ++e) {
      if (e < vpt) {
        const int j = tid * vpt + e;
        const double pv = __dadd_rn(base, loc2[e]);
        s_scan[j] = pv;
        if (i0 + j < i1 && __dadd_rn(pre, pv) > target) atomicMin(&s_k, j);
      }
    }
    __syncthreads();
  }
  if (tid == 0) {
    int64_t kstar = -1;
    double Pk = 0.0, Pkm1 = 0.0;
    const int kk = s_k;
    if (kk < PP_BLOCK) {
      kstar = i0 + kk;
      Pk = __dadd_rn(pre, s_scan[kk]);
      Pkm1 = kk ? __dadd_rn(pre, s_scan[kk - 1]) : pre;
    } else {
      const int last = (int)(i1 - i0 - 1);
      kstar = i1 - 1;
      Pk = __dadd_rn(pre, s_scan[last]);
      Pkm1 = last ? __dadd_rn(pre, s_scan[last - 1]) : pre;
    }
    // Error budget (rigorous, first order + slack): the reference's
    // cdf_k / cdf_last deviates from B_k/B_n by at most (k + n + 3)u
    // (sequential cumsum of k and n terms, p = b/T roundings, the division);
    // our fp64 prefix has <= ~1100u relative error (block tree + the final
    // in-block chain); the reference's best[] may differ from ours by the
    // rounding of its dgemv-ordered dot products: |delta d2| <= 8u(|x|+|c|)^2.
    const double n = (double)h.n;
    const double rel = ((double)kstar + n + 1200.0) * U0 * 1.05;
    // |best_i(ours) - best_i(reference)| <= 16u (xsq_i + max csq of the chosen
    // centroids) (dgemv vs FMA-chain dot products, (|x|+|c|)^2 <= 2(xsq + csq)),
    // summed over the points: 16u (sum xsq + n csqmax); the sum of xsq carries a
    // 1e-9 relative slack for its own (order-free) rounding
    const double xsqsum = __longlong_as_double((long long)__ldcg(status + 8)) * (1.0 + 1e-9);
    const double csqmax = __longlong_as_double((long long)__ldcg(status + 9));
    const double absU = 16.0 * U0 * (xsqsum + n * csqmax);
    const double margin = rel * S + 2.0 * absU;
    s_ok = !force_replay && (Pk - target > margin) && (target - Pkm1 >= margin);
    if (s_ok) picks[draw] = kstar;
  }
  __syncthreads();
  if (!s_ok && tid == 0) status[7] = draw;   // undecided: k_pp_replay (next launch) replays numpy exactly
}

// numpy's pairwise sum of best (the total of Generator.choice's p): the
// leaves (<= 128 elements, 8 strided accumulators) summed by 8 lanes each (the
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree by xor shuffles, then the tail),
// thread `gt` of `gn` (a multiple of 32) taking leaves gt/8, gt/8 + gn/8, ...
__device__ void pw_leaf_sums(const double* __restrict__ best, const int64_t* __restrict__ leaves, int64_t nleaves,
                             double* __restrict__ lsum, int64_t gt, int64_t gn) {
  const int j = (int)(gt & 7);
  for (int64_t l0 = gt >> 3; l0 - (gt >> 3) < nleaves; l0 += gn / 8) {   // warp-uniform trip count
    const int64_t l = l0;
    double r = 0.0;
    int64_t off = 0, len = 0;
    if (l < nleaves) {
      off = leaves[2 * l];
      len = leaves[2 * l + 1];
      if (len >= 8) {
        // this lane's strided accumulator: all (<= 16) loads in flight, then the adds
        const double* a = best + off;
        const int nb8 = (int)(len / 8);
        double v[16];
#pragma unroll
        for (int t = 0; t < 16; ++t) v[t] = t < nb8 ? __ldcg(a + 8 * t + j) : 0.0;
        r = v[0];
#pragma unroll
        for (int t = 1; t < 16; ++t)
          if (t < nb8) r = __dadd_rn(r, v[t]);
      }
    }
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 1));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 2));
    r = __dadd_rn(r, __shfl_xor_sync(0xffffffffu, r, 4));
    if (l < nleaves && j == 0) {
      if (len < 8) {
        r = 0.0;
        for (int64_t i = 0; i < len; ++i) r = __dadd_rn(r, __ldcg(best + off + i));
      } else {
        for (int64_t i = len - (len % 8); i < len; ++i) r = __dadd_rn(r, __ldcg(best + off + i));
      }
      lsum[l] = r;
    }
  }
}

// the combine tree over the leaf sums, level by level (node lists from the
// host); one CTA, the leaf sums already visible to it; returns the total
__device__ double pw_combine(const int64_t* __restrict__ leaves, int64_t nleaves, double* __restrict__ lsum) {
  const int tid = threadIdx.x, NT = blockDim.x;
  const int32_t* tl = reinterpret_cast<const int32_t*>(leaves + 2 * nleaves);   // left[ni], right[ni], level_start[]
  const int ni = (int)(nleaves - 1);
  const int32_t* tr = tl + ni;
  const int32_t* lvs = tr + ni;
  for (int lv = 0; ni > 0; ++lv) {
    const int b0 = lvs[lv], b1 = lvs[lv + 1];
    for (int i = b0 + tid; i < b1; i += NT) lsum[nleaves + i] = __dadd_rn(__ldcg(lsum + tl[i]), __ldcg(lsum + tr[i]));
    __syncthreads();
    if (b1 == ni) break;
  }
  return ni > 0 ? __ldcg(lsum + nleaves + ni - 1) : __ldcg(lsum);
}

// The exact replay of Generator.choice(n, p=best/total) for draw ci + 1 when
// the certified search could not decide (status[7] == draw): its own launch of
// one 1024-thread CTA (4x the warps of a k_pp_step CTA to hide the latencies
// of the division / scan chain), a no-op otherwise.
constexpr int RP_THREADS = 1024;
__global__ void __launch_bounds__(RP_THREADS) k_pp_replay(HalfView h, const double* __restrict__ best,
                                                          const double* __restrict__ uni, int ci,
                                                          int64_t* __restrict__ picks, int64_t* __restrict__ status,
                                                          const int64_t* __restrict__ leaves, int64_t nleaves,
                                                          double* __restrict__ lsum, double* __restrict__ pbuf,
                                                          double* __restrict__ cbuf, int force_replay) {
  const int draw = ci + 1;
  if (__ldcg(status + 7) != draw) return;
  const int tid = threadIdx.x;
  const int NT = blockDim.x;
  const double u = uni[ci];
  __shared__ double s_total;
  // ---- exact replay of Generator.choice(n, p=best/total) (clustering.py:48):
  // total = numpy pairwise sum; p = best/total; cdf = sequential cumsum;
  // idx = first i with fl(cdf_i / cdf_last) > u.  Everything but the cumsum
  // chain runs on all threads of the block.
  // numpy pairwise total: 8 lanes per leaf (one per strided accumulator, the
  // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) tree by xor shuffles, then the tail),
  // then the combine tree level by level (node lists from the host)
  pw_leaf_sums(best, leaves, nleaves, lsum, tid, NT);
  __syncthreads();
  {
    const double t = pw_combine(leaves, nleaves, lsum);
    if (tid == 0) s_total = t;
    __syncthreads();
  }
  const double total = s_total;
  __shared__ double tile[2][PS_TILE];
  __shared__ double s_c;
  if (force_replay != 2) {
    cumsum_exact_block(best, total, h.n, cbuf);
    if (tid == 0) s_c = cbuf[h.n - 1];
    __syncthreads();
  } else {
  for (int64_t i = tid; i < h.n; i += NT) pbuf[i] = __ddiv_rn(__ldcg(best + i), total);
  __syncthreads();
  // (test hook force_replay == 2) the sequential cumsum chain on thread 0 over
  // shared-memory tiles the rest of the block streams in (double buffered)
  // and writes back (cdf values -> cbuf)
  const int64_t ntile = (h.n + PS_TILE - 1) / PS_TILE;
  for (int64_t i = tid; i < min((int64_t)PS_TILE, h.n); i += NT) tile[0][i] = pbuf[i];
  if (tid == 0) s_c = 0.0;
  __syncthreads();
  for (int64_t tb = 0; tb < ntile; ++tb) {
    const int64_t nb0 = (tb + 1) * PS_TILE;
    if (tid >= 32) {
      // write back the previous tile's cdf, prefetch the next tile
      if (tb > 0) {
        const int64_t pb0 = (tb - 1) * PS_TILE;
        for (int64_t i = tid - 32; i < PS_TILE && pb0 + i < h.n; i += NT - 32)
          cbuf[pb0 + i] = tile[(tb + 1) & 1][i];
      }
      __syncwarp();
      for (int64_t i = tid - 32; i < PS_TILE && nb0 + i < h.n; i += NT - 32)
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
    for (int64_t i = tid; i < PS_TILE && pb0 + i < h.n; i += NT) cbuf[pb0 + i] = tile[(ntile - 1) & 1][i];
  }
  __syncthreads();
  }   // sequential chain
  // the crossing is then found by binary search over cbuf
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
    status[7] = 0;
  }
}

// ---- the exact replay across the GPU (k_ppx_total, then k_ppx_quanta; both
// no-ops unless status[7] == draw).  The cumsum is cut into the k_pp_step
// tiles (PP_BLOCK points, their block sums in bsum).  k_ppx_total: the
// pairwise leaves over the grid, then its last CTA combines them into the total
// and predicts each tile's binade from an approximate prefix of the block sums
// (a tile whose approximate cdf range touches a binade edge gets none).
// k_ppx_quanta: the integer quotient sum Q_t = sum round(p_k / g_e) of every
// predicted tile (-1 on a tie or a quotient >= 2^52), then its last CTA walks
// the tiles in order with the exact running value c: a window of tiles whose
// predicted binade is c's and whose quotient prefix stays below the binade's
// end is one exact step c + g * Q (a block scan); any other tile runs through
// cumsum_exact_range.  tend[t] = the exact cdf after tile t; the crossing tile
// of u is then replayed element by element.  Same numbers as k_pp_replay.
constexpr int PX_THREADS = 512;
constexpr long long PX_NOBIN = LLONG_MIN;
__global__ void __launch_bounds__(256) k_ppx_total(HalfView h, const double* __restrict__ best, int ci,
                                                   int64_t* __restrict__ status, const int64_t* __restrict__ leaves,
                                                   int64_t nleaves, double* __restrict__ lsum,
                                                   const double* __restrict__ bsum, int64_t nb,
                                                   long long* __restrict__ tbin) {
  if (__ldcg(status + 7) != ci + 1) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NT = blockDim.x, NW = NT >> 5;
  pw_leaf_sums(best, leaves, nleaves, lsum, (int64_t)blockIdx.x * NT + tid, (int64_t)gridDim.x * NT);
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(reinterpret_cast<unsigned long long*>(status + 10), 1ull) == (unsigned long long)(gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  const double total = pw_combine(leaves, nleaves, lsum);
  if (tid == 0) {
    status[10] = 0;
    status[12] = __double_as_longlong(total);
  }
  // approximate exclusive / inclusive prefix of the block sums, NT tiles at a time
  __shared__ double s_w[32];
  __shared__ double s_base;
  if (tid == 0) s_base = 0.0;
  __syncthreads();
  // the reference's sequential cdf differs from the exact prefix by <= (n + 2) u
  // relative; the fp64 block sums and this scan by far less
  const double rel = 4.0 * ((double)h.n + 4096.0) * U0 + 1e-13;
  for (int64_t t0 = 0; t0 < nb; t0 += NT) {
    const int64_t t = t0 + tid;
    const double v = t < nb ? __ldcg(bsum + t) : 0.0;
    double incl = v;
    for (int o = 1; o < 32; o <<= 1) {
      const double y = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += y;
    }
    if (lane == 31) s_w[wid] = incl;
    __syncthreads();
    if (wid == 0) {
      double w = lane < NW ? s_w[lane] : 0.0;
      for (int o = 1; o < 32; o <<= 1) {
        const double y = __shfl_up_sync(0xffffffffu, w, o);
        if (lane >= o) w += y;
      }
      s_w[lane] = w;
    }
    __syncthreads();
    const double base = s_base;
    const double hi = base + (wid ? s_w[wid - 1] : 0.0) + incl;
    const double lo = hi - v;
    if (t < nb) {
      const double a = lo / total * (1.0 - rel), b = hi / total * (1.0 + rel);
      long long e = PX_NOBIN;
      if (a >= 0x1p-900 && ilogb(a) == ilogb(b)) e = ilogb(a);
      tbin[t] = e;
    }
    __syncthreads();
    if (tid == NT - 1) s_base = hi;
    __syncthreads();
  }
}

__global__ void __launch_bounds__(PX_THREADS) k_ppx_quanta(HalfView h, const double* __restrict__ best,
                                                           const double* __restrict__ uni, int ci,
                                                           int64_t* __restrict__ picks, int64_t* __restrict__ status,
                                                           int64_t nb, const long long* __restrict__ tbin,
                                                           long long* __restrict__ tq, double* __restrict__ tend,
                                                           double* __restrict__ cbuf) {
  const int draw = ci + 1;
  if (__ldcg(status + 7) != draw) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, NT = blockDim.x, NW = NT >> 5;
  const int64_t n = h.n;
  const double total = __longlong_as_double((long long)__ldcg(status + 12));
  // ---- quotient sums, one warp per tile
  for (int64_t t = (int64_t)blockIdx.x * NW + wid; t < nb; t += (int64_t)gridDim.x * NW) {
    const long long e = __ldcg(tbin + t);
    if (e == PX_NOBIN) {
      if (lane == 0) tq[t] = -1;
      continue;
    }
    const double inv = scalbn(1.0, 52 - (int)e);
    const int64_t k0 = t * PP_BLOCK, k1 = min(n, k0 + PP_BLOCK);
    long long q = 0;
    bool bad = false;
    for (int64_t k = k0 + lane; k < k1; k += 128) {
      double bv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) bv[u] = k + 32 * u < k1 ? __ldcg(best + k + 32 * u) : 0.0;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const double x = __dmul_rn(__ddiv_rn(bv[u], total), inv);
        if (x >= 0x1p52) {
          bad = true;
        } else {
          const double fl = floor(x), fr = __dsub_rn(x, fl);
          q += (long long)fl + (fr > 0.5 ? 1 : 0);
          bad |= fr == 0.5;
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) q += __shfl_xor_sync(0xffffffffu, q, o);
    bad = __any_sync(0xffffffffu, bad);
    if (lane == 0) tq[t] = bad ? -1 : q;
  }
  __shared__ int s_last;
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(reinterpret_cast<unsigned long long*>(status + 11), 1ull) == (unsigned long long)(gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  // ---- the ordered walk
  __shared__ double s_c;
  __shared__ int s_started;
  __shared__ long long s_t0;
  __shared__ int s_f;
  __shared__ long long s_w[32];
  __shared__ double s_cnew;
  if (tid == 0) {
    status[11] = 0;
    s_c = 0.0;
    s_started = 0;
    s_t0 = 0;
  }
  __syncthreads();
  while (true) {
    const int64_t t0 = s_t0;
    if (t0 >= nb) break;
    const double c = s_c;
    int64_t tel = t0;   // tile to run element by element
    if (s_started && c >= 0x1p-900) {
      const int e = ilogb(c);
      const double g = scalbn(1.0, e - 52);
      const long long Qlim = (long long)__dmul_rn(__dsub_rn(scalbn(1.0, e + 1), c), scalbn(1.0, 52 - e));
      const int64_t t = t0 + tid;
      const long long Q = t < nb ? __ldcg(tq + t) : -1;
      const bool ok = t < nb && Q >= 0 && __ldcg(tbin + t) == (long long)e;
      const long long qv = ok ? Q : 0;
      long long incl = qv;
      for (int o = 1; o < 32; o <<= 1) {
        const long long y = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += y;
      }
      if (lane == 31) s_w[wid] = incl;
      if (tid == 0) s_f = NT;
      __syncthreads();
      if (wid == 0) {
        long long w = lane < NW ? s_w[lane] : 0;
        for (int o = 1; o < 32; o <<= 1) {
          const long long y = __shfl_up_sync(0xffffffffu, w, o);
          if (lane >= o) w += y;
        }
        s_w[lane] = w;
      }
      __syncthreads();
      const long long P = (wid ? s_w[wid - 1] : 0) + incl;   // quotient prefix through tile t
      if (!(ok && P < Qlim)) atomicMin(&s_f, tid);
      __syncthreads();
      const int f = s_f;
      if (tid < f) tend[t] = __dadd_rn(c, __dmul_rn((double)P, g));   // exact
      if (f > 0 && tid == f - 1) s_cnew = __dadd_rn(c, __dmul_rn((double)P, g));
      __syncthreads();
      const double cn = f > 0 ? s_cnew : c;
      __syncthreads();
      if (f == NT || t0 + f >= nb) {
        if (tid == 0) {
          s_c = cn;
          s_t0 = t0 + f;
        }
        __syncthreads();
        continue;
      }
      tel = t0 + f;
      if (tid == 0) s_c = cn;
      __syncthreads();
    }
    const double cs = s_c;
    const bool st = s_started;
    const double ce = cumsum_exact_range(best, total, tel * PP_BLOCK, min(n, (tel + 1) * PP_BLOCK), cs, st, nullptr);
    if (tid == 0) {
      tend[tel] = ce;
      s_c = ce;
      s_started = 1;
      s_t0 = tel + 1;
    }
    __syncthreads();
  }
  // ---- the draw: first k with fl(cdf_k / last) > u
  __shared__ long long s_ts;
  __shared__ double s_thr;
  __shared__ int s_k;
  if (tid == 0) {
    const double u = uni[ci];
    const double last = s_c;
    double c_thr = __dmul_rn(u, last);
    while (__ddiv_rn(c_thr, last) > u) c_thr = __longlong_as_double(__double_as_longlong(c_thr) - 1);
    while (true) {
      const double nx = __longlong_as_double(__double_as_longlong(c_thr) + 1);
      if (__ddiv_rn(nx, last) > u) break;
      c_thr = nx;
    }
    int64_t lo = -1, hi = nb - 1;   // tend[nb-1] = last > c_thr: first tile whose end exceeds c_thr
    while (hi - lo > 1) {
      const int64_t mid = (lo + hi) >> 1;
      if (__ldcg(tend + mid) > c_thr) hi = mid; else lo = mid;
    }
    s_ts = hi;
    s_thr = c_thr;
    s_k = PP_BLOCK;
  }
  __syncthreads();
  const int64_t ts = s_ts;
  const int64_t k0 = ts * PP_BLOCK, k1 = min(n, k0 + PP_BLOCK);
  cumsum_exact_range(best, total, k0, k1, ts > 0 ? __ldcg(tend + ts - 1) : 0.0, ts > 0, cbuf);
  for (int64_t k = tid; k < k1 - k0; k += NT)
    if (__ldcg(cbuf + k) > s_thr) atomicMin(&s_k, (int)k);
  __syncthreads();
  if (tid == 0) {
    picks[draw] = k0 + min(s_k, (int)(k1 - k0 - 1));
    status[1] += 1;
    status[7] = 0;
  }
}

// One k-means++ draw in one launch: the D^2 update for centroid ci and the
// per-1024-point block sums, then the last CTA to finish (atomic ticket in
// status[6]) chooses picks[ci+1] with the certified search above.  The grid
// is persistent and sized so the concurrent halves share the SMs; a CTA of
// 256 threads walks its 1024-point blocks, 4 points per thread, reading each
// point's coordinates as float4s from the point-major copy.
template <int MP>
__global__ void __launch_bounds__(PP_THREADS, 3) k_pp_step(HalfView h, const float* __restrict__ xp,
                                                        const double* __restrict__ xsq, int ci,
                                                        double* __restrict__ best, double* __restrict__ C64,
                                                        double* __restrict__ bsum, int64_t nb,
                                                        const double* __restrict__ uni,
                                                        const int64_t* __restrict__ forced,
                                                        int64_t* __restrict__ picks, int64_t* __restrict__ status,
                                                        const int64_t* __restrict__ leaves, int64_t nleaves,
                                                        double* __restrict__ lsum, double* __restrict__ pbuf,
                                                        double* __restrict__ cbuf, int force_replay) {
  __shared__ double cv[MP];
  __shared__ double s_csq;
  __shared__ int s_last;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int m = h.m;
  const int64_t p = __ldcg(picks + ci);
  if (tid < MP) cv[tid] = tid < m ? (double)xp[(size_t)p * MP + tid] : 0.0;
  __syncthreads();
  if (tid == 0) {
    s_csq = einsum_sq([&](int t) { return cv[t]; }, m);
    if (blockIdx.x == 0) {
      for (int t = 0; t < m; ++t) C64[(size_t)ci * m + t] = cv[t];
      atomicMax(reinterpret_cast<unsigned long long*>(status + 9), (unsigned long long)__double_as_longlong(s_csq));
    }
  }
  __syncthreads();
  const double csq = s_csq;
  // Warp-granular: each warp owns whole 1024-point blocks (32 points per lane,
  // in batches with all loads in flight) and reduces them with shuffles, so no
  // CTA barrier sits between a block's loads and the next block's.
  const int64_t nwarps = (int64_t)gridDim.x * (PP_THREADS / 32);
  const int64_t gw = (int64_t)blockIdx.x * (PP_THREADS / 32) + wid;
  constexpr int UB = MP <= 8 ? 4 : MP <= 16 ? 2 : 1;   // points per lane per batch
  for (int64_t b = gw; b < nb; b += nwarps) {
    double part = 0.0;
    for (int u0 = 0; u0 < PP_BLOCK / 32; u0 += UB) {
      float xv[UB][MP];
      double ob[UB];
      int64_t ii[UB];
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        ii[u] = b * PP_BLOCK + (int64_t)(u0 + u) * 32 + lane;
        const bool live = ii[u] < h.n;
        const float4* src = reinterpret_cast<const float4*>(xp + (size_t)(live ? ii[u] : 0) * MP);
#pragma unroll
        for (int q = 0; q < MP / 4; ++q) {
          const float4 v = live ? __ldcs(src + q) : make_float4(0.f, 0.f, 0.f, 0.f);
          xv[u][4 * q] = v.x; xv[u][4 * q + 1] = v.y; xv[u][4 * q + 2] = v.z; xv[u][4 * q + 3] = v.w;
        }
        ob[u] = (live && ci > 0) ? best[ii[u]] : 0.0;
      }
#pragma unroll
      for (int u = 0; u < UB; ++u) {
        if (ii[u] < h.n) {
          double dot = 0.0;
#pragma unroll
          for (int t = 0; t < MP; ++t)
            if (t < m) dot = __fma_rn((double)xv[u][t], cv[t], dot);
          // xsq recomputed in the einsum order of k_xsq (bit-identical) instead of an 8 B/point read
          const double xs = einsum_sq([&](int t) { return (double)xv[u][t]; }, m);
          const double d2 = sq_dist_expand(xs, dot, csq);
          double bb = d2;
          if (ci > 0) {
            if (d2 < ob[u]) best[ii[u]] = d2; else bb = ob[u];
          } else {
            best[ii[u]] = d2;
          }
          part = __dadd_rn(part, bb);
        }
      }
    }
    for (int o = 16; o > 0; o >>= 1) part = __dadd_rn(part, __shfl_xor_sync(0xffffffffu, part, o));
    if (lane == 0) bsum[b] = part;
  }
  __syncthreads();
  if (tid == 0) {
    __threadfence();
    s_last = atomicAdd(reinterpret_cast<unsigned long long*>(status + 6), 1ull) ==
             (unsigned long long)(gridDim.x - 1);
  }
  __syncthreads();
  if (!s_last) return;
  __threadfence();
  if (tid == 0) status[6] = 0;   // ticket for the next draw (stream-ordered launch)
  if (ci + 1 < h.k)
    pp_search_body(h, best, bsum, nb, uni, forced, ci, picks, status, leaves, nleaves, lsum, pbuf, cbuf,
                   force_replay);
}

// ------------------------------------------------------------------ Lloyd
constexpr int AS_THREADS = 256;
constexpr int AS_CU = 4;   // centroids in flight per thread in k_assign
// Lloyd assignment (clustering.py:86-89): d2 = max((xsq - 2 x.c) + csq, 0)
// with x.c one FMA chain over t (dgemm order), first argmin.  Each thread
// owns PPT points so every centroid coordinate read from shared memory feeds
// PPT independent FMA chains (the kernel is fp64-issue bound).
template <int MM, int PPT>
__global__ void __launch_bounds__(AS_THREADS) k_assign(HalfView h, const double* __restrict__ xsq,
                                                       const double* __restrict__ C64,
                                                       const int32_t* __restrict__ lab,
                                                       int32_t* __restrict__ newlab,
                                                       double* __restrict__ pd, int iter,
                                                       int64_t* __restrict__ status,
                                                       double* __restrict__ hsum,
                                                       unsigned long long* __restrict__ cnt_cur,
                                                       unsigned long long* __restrict__ cnt_next) {
  extern __shared__ __align__(16) double ash[];
  __shared__ int lhist[256];
  if (status[2]) return;
  for (int c = threadIdx.x; c < h.k; c += AS_THREADS) lhist[c] = 0;
  if (blockIdx.x == 0)
    for (int c = threadIdx.x; c < h.k; c += AS_THREADS) cnt_next[c] = 0ull;
  const int m = h.m;
  // centroids at a compile-time stride MM, zero padded: a padded coordinate
  // adds fma(0, 0, acc) = acc exactly (up to the sign of a zero, which the
  // distance cannot see), so the inner loop has no bounds checks
  double* C = ash;                       // k*MM
  double* csq = ash + (size_t)h.k * MM;  // k
  __shared__ double red[AS_THREADS / 32];
  __shared__ int chg;
  for (int e = threadIdx.x; e < h.k * MM; e += AS_THREADS) {
    const int c = e / MM, t = e - c * MM;
    C[e] = t < m ? C64[(size_t)c * m + t] : 0.0;
  }
  if (threadIdx.x == 0) chg = 0;
  __syncthreads();
  for (int c = threadIdx.x; c < h.k; c += AS_THREADS)
    csq[c] = einsum_sq([&](int t) { return C[c * MM + t]; }, m);
  __syncthreads();
  const int64_t i0 = (int64_t)blockIdx.x * AS_THREADS * PPT + threadIdx.x;
  double x[PPT][MM], xs[PPT], bd[PPT];
  int bl[PPT];
  bool pos[PPT];   // bd > 0: while false (bd == 0) no later centroid can win (strict <)
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t i = i0 + (int64_t)j * AS_THREADS;
    const bool live = i < h.n;
#pragma unroll
    for (int t = 0; t < MM; ++t) x[j][t] = (t < m && live) ? (double)h.X[(size_t)t * h.n + i] : 0.0;
    xs[j] = live ? xsq[i] : 0.0;
    bd[j] = INFINITY;
    bl[j] = 0;
    pos[j] = true;
  }
  // AS_CU centroids at a time: AS_CU x PPT independent FMA chains per thread
  // (the latency of one dgemm-order chain is hidden by the others), compared
  // in ascending centroid order so the first argmin still wins
  auto visit = [&](int c, const double (&acc)[PPT]) {
    const double cs = csq[c];
#pragma unroll
    for (int j = 0; j < PPT; ++j) {
      // clustering._sq_dists: (xsq - 2 dot) + csq, clamped at 0; xsq - 2 dot is
      // one FMA (2 dot is exact), the clamp is applied only on an update:
      // max(v, 0) < bd  <=>  v < bd  whenever bd > 0
      const double v = __dadd_rn(__fma_rn(-2.0, acc[j], xs[j]), cs);
      if (v < bd[j] && pos[j]) {
        bd[j] = v > 0.0 ? v : 0.0;
        pos[j] = v > 0.0;
        bl[j] = c;
      }
    }
  };
  int c0 = 0;
  for (; c0 + AS_CU <= h.k; c0 += AS_CU) {
    double acc[AS_CU][PPT];
#pragma unroll
    for (int t2 = 0; t2 < MM / 2; ++t2) {
#pragma unroll
      for (int u = 0; u < AS_CU; ++u) {
        const double2 cv = reinterpret_cast<const double2*>(C + (c0 + u) * MM)[t2];
#pragma unroll
        for (int j = 0; j < PPT; ++j) {
          // dgemm order: one FMA chain over t from 0 (fma(x0, c0, 0) = x0 * c0)
          acc[u][j] = t2 == 0 ? __dmul_rn(x[j][0], cv.x) : __fma_rn(x[j][2 * t2], cv.x, acc[u][j]);
          acc[u][j] = __fma_rn(x[j][2 * t2 + 1], cv.y, acc[u][j]);
        }
      }
    }
#pragma unroll
    for (int u = 0; u < AS_CU; ++u) visit(c0 + u, acc[u]);
  }
  for (; c0 < h.k; ++c0) {
    double acc[PPT];
#pragma unroll
    for (int t2 = 0; t2 < MM / 2; ++t2) {
      const double2 cv = reinterpret_cast<const double2*>(C + c0 * MM)[t2];
#pragma unroll
      for (int j = 0; j < PPT; ++j) {
        acc[j] = t2 == 0 ? __dmul_rn(x[j][0], cv.x) : __fma_rn(x[j][2 * t2], cv.x, acc[j]);
        acc[j] = __fma_rn(x[j][2 * t2 + 1], cv.y, acc[j]);
      }
    }
    visit(c0, acc);
  }
  double my = 0.0;
  int changed = 0;
#pragma unroll
  for (int j = 0; j < PPT; ++j) {
    const int64_t i = i0 + (int64_t)j * AS_THREADS;
    if (i < h.n) {
      newlab[i] = bl[j];
      atomicAdd(&lhist[bl[j]], 1);
      pd[i] = bd[j];
      my = __dadd_rn(my, bd[j]);
      if (iter > 0 && lab[i] != bl[j]) changed = 1;
    }
  }
  if (__any_sync(0xffffffffu, changed) && (threadIdx.x & 31) == 0) atomicOr(&chg, 1);
  for (int o = 16; o > 0; o >>= 1) my = __dadd_rn(my, __shfl_xor_sync(0xffffffffu, my, o));
  if ((threadIdx.x & 31) == 0) red[threadIdx.x >> 5] = my;
  __syncthreads();
  for (int c = threadIdx.x; c < h.k; c += AS_THREADS)
    if (lhist[c]) atomicAdd(&cnt_cur[c], (unsigned long long)lhist[c]);
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

// A point's coordinates as one record of MP floats (the point-major copy);
// the label sort moves whole records, so every cluster ends up as one
// contiguous run of records in index order.
template <int MP>
struct __align__(16) PointRec {
  float v[MP];
};

// ---- Lloyd assignment on the tensor cores (m <= 8): the distance GEMM
// X[128 x 8] . C^T[8 x N] of each 128-point tile runs as three tcgen05 TF32
// MMAs (x_hi c_hi + x_hi c_lo + x_lo c_hi, hi = tf32(x), lo = tf32(x - hi):
// ~fp32-accurate products, fp32 accumulation in TMEM).  Thread r of the CTA
// owns TMEM lane r (point r): it reads the N approximate dot products, forms
// d2f = (xsq - 2 dot) + csq in fp32 and a bound e = 2^-14 (xsq + max csq) on
// |d2f - d2_ref| (TF32x3 products and accumulation <= 2^-17 A, A <= (xsq +
// csq)/2; fp32 formation <= 2^-22 (xsq + csq)), then re-evaluates in the
// reference's fp64 formula only the centroids whose interval can still hold
// the minimum -- the first exact argmin is the reference's label and point_d2.
constexpr int TC_THREADS = 128;
__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// K-major, no swizzle: 8-row x 16-byte core matrices; the K chunks (4 tf32)
// of an 8-row group 128 B apart (LBO), 8-row groups MP * 32 B apart (SBO)
template <int MP>
__device__ __forceinline__ int tc_off(int row, int k) {   // float index inside an operand tile
  return (row >> 3) * (MP * 8) + (k >> 2) * 32 + (row & 7) * 4 + (k & 3);
}
template <int MP>
__device__ __forceinline__ uint64_t tc_desc(const void* smem) {
  const uint64_t a = (uint64_t)((smem_u32(smem) >> 4) & 0x3FFF);
  const uint64_t lbo = 128 >> 4, sbo = (uint64_t)(MP * 32) >> 4;
  return a | (lbo << 16) | (sbo << 32) | (1ull << 46);   // version 1 (sm_100), SWIZZLE_NONE, base offset 0
}
__device__ __forceinline__ void tc_mma(uint32_t tmem_d, uint64_t da, uint64_t db, uint32_t idesc, uint32_t acc) {
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.b32 p, %4, 0;\n"
      " tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n}\n" ::"r"(tmem_d),
      "l"(da), "l"(db), "r"(idesc), "r"(acc));
}

template <int MP>
__global__ void __launch_bounds__(TC_THREADS) k_assign_tc(HalfView h, const float* __restrict__ xp,
                                                          const double* __restrict__ xsq,
                                                          const double* __restrict__ C64,
                                                          const int32_t* __restrict__ lab,
                                                          int32_t* __restrict__ newlab,
                                                          double* __restrict__ pd, int iter,
                                                          int64_t* __restrict__ status,
                                                          double* __restrict__ hsum,
                                                          unsigned long long* __restrict__ cnt_cur,
                                                          unsigned long long* __restrict__ cnt_next, int npad) {
  extern __shared__ __align__(128) float tsm[];
  float* Ahi = tsm;                       // 128 x MP
  float* Alo = Ahi + TC_THREADS * MP;
  float* Bhi = Alo + TC_THREADS * MP;     // npad x MP
  float* Blo = Bhi + npad * MP;
  double* C = reinterpret_cast<double*>(Blo + npad * MP);   // k x MP (fp64, zero padded)
  double* csq = C + (size_t)h.k * MP;
  float* ca = reinterpret_cast<float*>(csq + h.k + (h.k & 1));   // [npad] RU(csq (1 + K)) (+inf for pads), 16-B aligned
  float* cb_ = ca + npad;                              // [npad] RD(csq (1 - K))
  __shared__ __align__(8) uint64_t mbar;
  __shared__ uint32_t tmem_base;
  __shared__ int lhist[256];
  __shared__ double red[TC_THREADS / 32];
  __shared__ int chg;
  if (status[2]) return;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5, m = h.m, k = h.k;
  for (int c = tid; c < k; c += TC_THREADS) lhist[c] = 0;
  if (blockIdx.x == 0)
    for (int c = tid; c < k; c += TC_THREADS) cnt_next[c] = 0ull;
  for (int e = tid; e < npad * MP; e += TC_THREADS) {
    const int c = e / MP, t = e % MP;
    const double cv = (c < k && t < m) ? C64[(size_t)c * m + t] : 0.0;
    if (c < k) C[e] = cv;
    const float cf = __double2float_rn(cv);
    const float hi = tf32_rna(cf);
    Bhi[tc_off<MP>(c, t)] = hi;
    Blo[tc_off<MP>(c, t)] = tf32_rna(cf - hi);
  }
  if (tid == 0) {
    chg = 0;
    mbar_init(&mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (wid == 0) {
    uint32_t ncols = 32;
    while ((int)ncols < npad) ncols <<= 1;
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(&tmem_base)),
                 "r"(ncols));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n" ::);
  }
  __syncthreads();
  // |d2_fp32 - d2_ref| <= K (xsq + csq_c), K = 2^-14 (see above): the
  // centroid part is folded into per-centroid constants, the point part K xsq
  // is added to the threshold
  constexpr float KB = 6.103515625e-05f;
  for (int c = tid; c < npad; c += TC_THREADS) {
    if (c < k) {
      const double v = einsum_sq([&](int t) { return C[c * MP + t]; }, m);
      csq[c] = v;
      ca[c] = __double2float_ru(v * (1.0 + 6.103515625e-05));
      cb_[c] = __double2float_rd(v * (1.0 - 6.103515625e-05));
    } else {
      ca[c] = INFINITY;
      cb_[c] = INFINITY;
    }
  }
  __syncthreads();
  const uint32_t tmem = tmem_base;
  // tf32 . tf32 -> f32, both operands K-major, M = 128, N = npad
  const uint32_t idesc = (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(npad >> 3) << 17) | ((uint32_t)(128 >> 4) << 24);
  // k-block kb (8 tf32 = two 16-byte chunks) starts 256 B further into each operand
  const uint64_t dAhi = tc_desc<MP>(Ahi), dAlo = tc_desc<MP>(Alo), dBhi = tc_desc<MP>(Bhi), dBlo = tc_desc<MP>(Blo);
  const int64_t ntiles = (h.n + TC_THREADS - 1) / TC_THREADS;
  double my = 0.0;
  int changed = 0;
  uint32_t phase = 0;
  for (int64_t tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const int64_t i = tile * TC_THREADS + tid;
    const bool live = i < h.n;
    float x[MP];
    {
      const float4* src = reinterpret_cast<const float4*>(xp + (size_t)(live ? i : 0) * MP);
#pragma unroll
      for (int q4 = 0; q4 < MP / 4; ++q4) {
        const float4 a = live ? __ldg(src + q4) : make_float4(0.f, 0.f, 0.f, 0.f);
        x[4 * q4] = a.x; x[4 * q4 + 1] = a.y; x[4 * q4 + 2] = a.z; x[4 * q4 + 3] = a.w;
      }
    }
    const double xs = live ? xsq[i] : 0.0;
#pragma unroll
    for (int t = 0; t < MP; ++t) {
      const float hi = tf32_rna(x[t]);
      Ahi[tc_off<MP>(tid, t)] = hi;
      Alo[tc_off<MP>(tid, t)] = tf32_rna(x[t] - hi);
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");   // generic-proxy smem writes -> tensor core
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    __syncthreads();
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
#pragma unroll
      for (int kb = 0; kb < MP / 8; ++kb) {
        const uint64_t o = (uint64_t)(kb * 256) >> 4;   // descriptor start address is in 16 B units
        tc_mma(tmem, dAhi + o, dBhi + o, idesc, kb > 0 ? 1u : 0u);
        tc_mma(tmem, dAhi + o, dBlo + o, idesc, 1u);
        tc_mma(tmem, dAlo + o, dBhi + o, idesc, 1u);
      }
      asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(&mbar))
                   : "memory");
    }
    mbar_wait(&mbar, phase);
    phase ^= 1u;
    asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory");
    // this thread's row: TMEM lane tid, columns [0, npad).  With g = csq - 2 dot
    // (xsq is common to every centroid): pass 1 takes min_c RU(a_c - 2 dot),
    // pass 2 keeps the centroids with RD(b_c - 2 dot) <= that + 2 K xsq.
    const uint32_t trow = tmem + ((uint32_t)(wid * 32) << 16);
    auto tld = [&](int cb, float (&v)[16]) {
      uint32_t r[16];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
          : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]),
            "=r"(r[8]), "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
          : "r"(trow + (uint32_t)(cb * 16)));
      asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
      for (int u = 0; u < 16; ++u) v[u] = __uint_as_float(r[u]);
    };
    float gmin = INFINITY;
    for (int cb = 0; cb * 16 < npad; ++cb) {
      float v[16];
      tld(cb, v);
      const float4* a4 = reinterpret_cast<const float4*>(ca + cb * 16);
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const float4 a = a4[q];
        gmin = fminf(gmin, __fmaf_ru(-2.f, v[4 * q + 0], a.x));
        gmin = fminf(gmin, __fmaf_ru(-2.f, v[4 * q + 1], a.y));
        gmin = fminf(gmin, __fmaf_ru(-2.f, v[4 * q + 2], a.z));
        gmin = fminf(gmin, __fmaf_ru(-2.f, v[4 * q + 3], a.w));
      }
    }
    const float xsu = __double2float_ru(xs);
    const float thr = __fadd_ru(gmin, __fmul_ru(2.f * KB, xsu));
    // pass 2: candidate masks (16 centroids per block) and the least lower bound
    uint32_t cm[8];   // npad <= 256: 16 blocks of 16 bits
#pragma unroll
    for (int q = 0; q < 8; ++q) cm[q] = 0u;
    float lmin = INFINITY;
#pragma unroll
    for (int cb = 0; cb < 16; ++cb) {
      if (cb * 16 < npad) {
        float v[16];
        tld(cb, v);
        const float4* b4 = reinterpret_cast<const float4*>(cb_ + cb * 16);
        uint32_t mask = 0;
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const float4 bq = b4[q];
          const float l0 = __fmaf_rd(-2.f, v[4 * q + 0], bq.x), l1 = __fmaf_rd(-2.f, v[4 * q + 1], bq.y);
          const float l2 = __fmaf_rd(-2.f, v[4 * q + 2], bq.z), l3 = __fmaf_rd(-2.f, v[4 * q + 3], bq.w);
          mask |= ((uint32_t)(l0 <= thr) << (4 * q)) | ((uint32_t)(l1 <= thr) << (4 * q + 1)) |
                  ((uint32_t)(l2 <= thr) << (4 * q + 2)) | ((uint32_t)(l3 <= thr) << (4 * q + 3));
          lmin = fminf(lmin, fminf(fminf(l0, l1), fminf(l2, l3)));
        }
        cm[cb >> 1] |= mask << ((cb & 1) * 16);
      }
    }
    // every reference value provably > 0 unless xs (1 - K) + lmin <= 0: then the
    // clamp at 0 may tie several centroids and all of them are evaluated
    const bool clampy = !(__fadd_rd(__fmul_rd(__double2float_rd(xs), 1.f - KB), lmin) > 0.f);
    double bd = INFINITY;
    int bl = 0;
    bool pos = true;
#pragma unroll
    for (int q = 0; q < 8; ++q) {
      if (q * 32 < npad) {
        uint32_t mask = clampy ? 0xFFFFFFFFu : cm[q];
        while (mask) {
          const int u = __ffs(mask) - 1;
          mask &= mask - 1u;
          const int c = q * 32 + u;
          if (c >= k) break;
          const double* cr = C + c * MP;
          double acc = __dmul_rn((double)x[0], cr[0]);
#pragma unroll
          for (int t = 1; t < MP; ++t) acc = __fma_rn((double)x[t], cr[t], acc);   // padded t >= m add exact zeros
          const double dv = __dadd_rn(__fma_rn(-2.0, acc, xs), csq[c]);
          if (dv < bd && pos) {
            bd = dv > 0.0 ? dv : 0.0;
            pos = dv > 0.0;
            bl = c;
          }
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory");
    if (live) {
      newlab[i] = bl;
      atomicAdd(&lhist[bl], 1);
      pd[i] = bd;
      my = __dadd_rn(my, bd);
      if (iter > 0 && lab[i] != bl) changed = 1;
    }
    __syncthreads();   // A tiles and TMEM free for the next tile
  }
  if (__any_sync(0xffffffffu, changed) && lane == 0) atomicOr(&chg, 1);
  for (int o = 16; o > 0; o >>= 1) my = __dadd_rn(my, __shfl_xor_sync(0xffffffffu, my, o));
  if (lane == 0) red[wid] = my;
  __syncthreads();
  for (int c = tid; c < k; c += TC_THREADS)
    if (lhist[c]) atomicAdd(&cnt_cur[c], (unsigned long long)lhist[c]);
  if (tid == 0) {
    double t = 0.0;
    for (int w = 0; w < TC_THREADS / 32; ++w) t = __dadd_rn(t, red[w]);
    hsum[blockIdx.x] = t;
    if (chg) atomicAdd((unsigned long long*)&status[4], 1ull);
  }
  if (wid == 0) {
    uint32_t ncols = 32;
    while ((int)ncols < npad) ncols <<= 1;
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tmem), "r"(ncols));
  }
}

// centroid = (sequential fp64 sum over the cluster's points in index order) /
// count -- the np.add.at order (clustering.py:95-99).  The label sort leaves
// cluster c's records contiguous (index order inside the cluster), so one CTA
// per cluster streams its run with 1-D TMA bulk copies into a CS_ST-stage
// shared-memory ring (full/empty mbarriers), and the first m lanes of the
// consumer warp run the m dependent add chains at the DADD latency.  The
// producer warp's other lanes commit the new labels (lab = newlab).
constexpr int CS_R = 64, CS_ST = 8, CS_THREADS = 96;   // warp 0 chains, warp 1 (one lane) TMA, warp 2 labels
template <int MP>
__global__ void __launch_bounds__(CS_THREADS) k_cluster_sums(HalfView h, const PointRec<MP>* __restrict__ xs,
                                                             const int64_t* __restrict__ status,
                                                             const unsigned long long* __restrict__ counts,
                                                             const int32_t* __restrict__ newlab,
                                                             int32_t* __restrict__ lab,
                                                             double* __restrict__ C64) {
  if (status[2]) return;
  extern __shared__ __align__(128) float cs[];   // [CS_ST][CS_R][MP]
  __shared__ __align__(8) uint64_t full[CS_ST], empty[CS_ST];
  __shared__ int64_t s_start;
  const int c = blockIdx.x, m = h.m, tid = threadIdx.x, lane = tid & 31;
  const int64_t cnt = (int64_t)counts[c];
  if (tid < 32) {
    int64_t v = 0;
    for (int c2 = tid; c2 < c; c2 += 32) v += (int64_t)counts[c2];
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (tid == 0) {
      s_start = v;
      for (int st = 0; st < CS_ST; ++st) {
        mbar_init(&full[st], 1);
        mbar_init(&empty[st], 1);
      }
      asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
    }
  }
  __syncthreads();
  const PointRec<MP>* run = xs + s_start;
  const int64_t ntile = (cnt + CS_R - 1) / CS_R;
  if (tid >= 64) {
    // commit the labels of this iteration (lab = newlab) while the chains run
    // (own warp, so the TMA producer lane never waits behind it): CTA c copies
    // its slice with 16-byte accesses, 8 in flight per lane
    const int64_t per = ((h.n + gridDim.x - 1) / gridDim.x + 3) & ~(int64_t)3;
    const int64_t i0 = min(h.n, (int64_t)c * per), i1 = min(h.n, i0 + per);
    const bool al = ((reinterpret_cast<uintptr_t>(newlab) | reinterpret_cast<uintptr_t>(lab)) & 15) == 0;
    const int64_t v0 = i0 >> 2, v1 = al ? i1 >> 2 : v0;   // whole int4s (i0 is a multiple of 4)
    const int4* src = reinterpret_cast<const int4*>(newlab);
    int4* dst = reinterpret_cast<int4*>(lab);
    for (int64_t b = v0 + (tid - 64); b < v1; b += 32 * 8) {
      int4 t[8];
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b + u * 32 < v1) t[u] = __ldcs(src + b + u * 32);
#pragma unroll
      for (int u = 0; u < 8; ++u)
        if (b + u * 32 < v1) dst[b + u * 32] = t[u];
    }
    for (int64_t i = (al ? v1 << 2 : i0) + (tid - 64); i < i1; i += 32) lab[i] = newlab[i];
  } else if (tid == 32 && cnt > 0) {
    // producer: one elected thread streams the run
    for (int64_t tb = 0; tb < ntile; ++tb) {
      const int slot = (int)(tb % CS_ST);
      if (tb >= CS_ST) mbar_wait(&empty[slot], (unsigned)(((tb / CS_ST) - 1) & 1));
      const int rr = (int)min((int64_t)CS_R, cnt - tb * CS_R);
      const unsigned bytes = (unsigned)(rr * MP * sizeof(float));
      mbar_expect_tx(&full[slot], bytes);
      tma_g2s(cs + (size_t)slot * CS_R * MP, run + tb * CS_R, bytes, &full[slot]);
    }
  } else if (tid < 32 && cnt > 0) {
    double acc = 0.0;
    for (int64_t tb = 0; tb < ntile; ++tb) {
      const int slot = (int)(tb % CS_ST);
      mbar_wait(&full[slot], (unsigned)((tb / CS_ST) & 1));
      if (lane < m) {
        const int rr = (int)min((int64_t)CS_R, cnt - tb * CS_R);
        acc = chain_add(acc, cs + (size_t)slot * CS_R * MP + lane, rr, MP);
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[slot]);
    }
    if (lane < m) C64[(size_t)c * m + lane] = __ddiv_rn(acc, (double)cnt);
  }
}

// point-major copy of a half (xp[i][t], t padded to mp = 4*ceil(m/4)) so a
// point's coordinates are one contiguous 16-byte-aligned run for the gathers
__global__ void k_point_major(HalfView h, int mp, float* __restrict__ xp) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= h.n) return;
  for (int q = 0; q < mp; q += 4) {
    float4 v;
    v.x = q + 0 < h.m ? h.X[(size_t)(q + 0) * h.n + i] : 0.f;
    v.y = q + 1 < h.m ? h.X[(size_t)(q + 1) * h.n + i] : 0.f;
    v.z = q + 2 < h.m ? h.X[(size_t)(q + 2) * h.n + i] : 0.f;
    v.w = q + 3 < h.m ? h.X[(size_t)(q + 3) * h.n + i] : 0.f;
    *reinterpret_cast<float4*>(xp + (size_t)i * mp + q) = v;
  }
}


// empty clusters (ascending): farthest point (first argmax of point_d2 with
// already-taken points at -1) becomes the centroid and moves its label.
__global__ void k_reseed(HalfView h, const int64_t* __restrict__ status,
                         const unsigned long long* __restrict__ counts, double* __restrict__ far,
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
  status[5] = 0;
  status[6] = 0;
  status[7] = 0;
  status[8] = 0;   // sum xsq (double bits)
  status[9] = 0;   // max csq of the chosen centroids (double bits)
  status[10] = 0;  // k_ppx_total ticket
  status[11] = 0;  // k_ppx_quanta ticket
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
  int concurrent = 1;  // halves running at once: each k-means++ draw takes sms/concurrent CTAs
};

// ------------------------------------------------ stable counting sort
// Stable sort of n items by a small key (< B <= 256 buckets), segmented into
// independent segments of `seg` items (seg a multiple of the run length;
// one segment for the Lloyd label sort, one per id chunk for the CSR).  A
// warp owns a run of `run` consecutive items and handles them 32 at a time
// in index order: __match_any_sync groups the lanes with equal keys, a
// lane's rank among them is the popcount of the lower peers, the group's
// lowest lane advances the warp's per-bucket cursor -- stable without any
// cross-warp ordering.  Three launches per pass:
//   k_ls_hist     per-run bucket counts, bh[b][run]
//   k_ls_scan     one CTA per segment: bucket totals, bucket starts, and the
//                 exclusive scan of each bucket's run counts -> item offsets
//   k_ls_scatter  per-run cursors from bh, ranks by match_any, payload moves
// With 2 N_s k-means halves in flight on their own streams, the narrow grids
// (a warp per 2048 points) overlap across halves.
constexpr int LS_WARPS = 4;
constexpr int LS_SCAN_THREADS = 1024;

struct LsLabelKey {   // key = label[i] (items in index order)
  const int32_t* lab;
  __device__ __forceinline__ uint32_t operator()(int64_t i, uint32_t) const { return (uint32_t)lab[i]; }
};
struct LsIdKey {      // key = label[id] (items carry point ids)
  const int32_t* lab;
  __device__ __forceinline__ uint32_t operator()(int64_t, uint32_t id) const { return (uint32_t)lab[id]; }
};
struct LsIota {       // payload id of item i = i
  __device__ __forceinline__ uint32_t operator()(int64_t i) const { return (uint32_t)i; }
};
struct LsIds {        // payload id of item i = ids[i]
  const uint32_t* ids;
  __device__ __forceinline__ uint32_t operator()(int64_t i) const { return ids[i]; }
};
struct LsIdOut {      // out[pos] = id
  uint32_t* out;
  __device__ __forceinline__ void operator()(int64_t pos, int64_t, uint32_t id) const { out[pos] = id; }
};
template <int MP>
struct LsRecOut {     // out[pos] = record of point i
  const PointRec<MP>* in;
  PointRec<MP>* out;
  __device__ __forceinline__ void operator()(int64_t pos, int64_t i, uint32_t) const {
    const float4* s4 = reinterpret_cast<const float4*>(in + i);
    float4* d4 = reinterpret_cast<float4*>(out + pos);
#pragma unroll
    for (int q = 0; q < MP / 4; ++q) d4[q] = __ldg(s4 + q);
  }
};

template <class KeyF, class IdF>
__global__ void __launch_bounds__(32 * LS_WARPS) k_ls_hist(KeyF key, IdF idf, int64_t n, int run, int64_t nruns,
                                                           int B, uint32_t* __restrict__ bh,
                                                           const int64_t* __restrict__ status) {
  if (status && status[2]) return;   // k-means converged: nothing to sort
  __shared__ uint32_t cnt_s[LS_WARPS][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * LS_WARPS + w;
  if (r >= nruns) return;   // warp-private from here on
  uint32_t* cnt = cnt_s[w];
  for (int b = lane; b < B; b += 32) cnt[b] = 0;
  __syncwarp();
  const int64_t i0 = r * run, i1 = min(n, i0 + run);
  constexpr int U = 8;   // rounds whose keys are loaded together
  for (int64_t base = i0; base < i1; base += 32 * U) {
    uint32_t k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      k[u] = i < i1 ? key(i, idf(i)) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const unsigned peers = __match_any_sync(0xffffffffu, k[u]);
      if (k[u] != 0xFFFFFFFFu && lane == __ffs(peers) - 1) cnt[k[u]] += __popc(peers);
      __syncwarp();
    }
  }
  for (int b = lane; b < B; b += 32) bh[(size_t)b * nruns + r] = cnt[b];
}

// one CTA per segment s (runs [s*rps, min(nruns, (s+1)*rps)), items from s*seg)
__global__ void __launch_bounds__(LS_SCAN_THREADS) k_ls_scan(uint32_t* __restrict__ bh, int64_t nruns, int rps,
                                                             int B, int64_t seg, const int64_t* __restrict__ status) {
  if (status && status[2]) return;
  __shared__ uint32_t tot[256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31, nw = LS_SCAN_THREADS / 32;
  const int64_t s0 = blockIdx.x;
  const int64_t r0 = s0 * rps, r1 = min(nruns, r0 + rps);
  for (int b = w; b < B; b += nw) {
    uint32_t v = 0;
    for (int64_t r = r0 + lane; r < r1; r += 32) v += bh[(size_t)b * nruns + r];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) tot[b] = v;
  }
  __syncthreads();
  for (int b = w; b < B; b += nw) {
    uint32_t st = 0;   // items of this segment in buckets < b
    for (int b2 = lane; b2 < b; b2 += 32) st += tot[b2];
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) st += __shfl_xor_sync(0xffffffffu, st, o);
    int64_t carry = s0 * seg + st;
    for (int64_t rb = r0; rb < r1; rb += 32) {
      const int64_t r = rb + lane;
      const uint32_t v = r < r1 ? bh[(size_t)b * nruns + r] : 0u;
      uint32_t x = v;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (r < r1) bh[(size_t)b * nruns + r] = (uint32_t)(carry + x - v);
      carry += __shfl_sync(0xffffffffu, x, 31);
    }
  }
}

template <class KeyF, class IdF, class OutF>
__global__ void __launch_bounds__(32 * LS_WARPS) k_ls_scatter(KeyF key, IdF idf, OutF out, int64_t n, int run,
                                                              int64_t nruns, int B, const uint32_t* __restrict__ bh,
                                                              const int64_t* __restrict__ status) {
  if (status && status[2]) return;
  __shared__ uint32_t cur_s[LS_WARPS][256];
  const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t r = (int64_t)blockIdx.x * LS_WARPS + w;
  if (r >= nruns) return;
  uint32_t* cur = cur_s[w];
  for (int b = lane; b < B; b += 32) cur[b] = bh[(size_t)b * nruns + r];
  __syncwarp();
  const int64_t i0 = r * run, i1 = min(n, i0 + run);
  const unsigned lt = (1u << lane) - 1u;
  constexpr int U = 4;   // rounds whose keys (and ids) are loaded together
  for (int64_t base = i0; base < i1; base += 32 * U) {
    uint32_t id[U], k[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t i = base + u * 32 + lane;
      id[u] = i < i1 ? idf(i) : 0u;
      k[u] = i < i1 ? key(i, id[u]) : 0xFFFFFFFFu;
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const bool ok = k[u] != 0xFFFFFFFFu;
      const unsigned peers = __match_any_sync(0xffffffffu, k[u]);
      const uint32_t pos = ok ? cur[k[u]] + __popc(peers & lt) : 0u;
      __syncwarp();
      if (ok && lane == __ffs(peers) - 1) cur[k[u]] += __popc(peers);
      __syncwarp();
      if (ok) out((int64_t)pos, base + u * 32 + lane, id[u]);
    }
  }
}

// one stable counting-sort pass: hist, scan, scatter (bh: B * nruns u32)
template <class KeyF, class IdF, class OutF>
static int ls_pass(KeyF key, IdF idf, OutF out, int64_t n, int B, int run, int64_t seg, uint32_t* bh,
                   const int64_t* status, cudaStream_t st) {
  const int64_t nruns = ceil_div(n, run);
  const int rps = (int)(seg / run);
  const unsigned g = (unsigned)ceil_div(nruns, LS_WARPS);
  k_ls_hist<<<g, 32 * LS_WARPS, 0, st>>>(key, idf, n, run, nruns, B, bh, status);
  TACO_LAUNCHED();
  k_ls_scan<<<(unsigned)ceil_div(nruns, rps), LS_SCAN_THREADS, 0, st>>>(bh, nruns, rps, B, seg, status);
  TACO_LAUNCHED();
  k_ls_scatter<<<g, 32 * LS_WARPS, 0, st>>>(key, idf, out, n, run, nruns, B, bh, status);
  TACO_LAUNCHED();
  return TACO_OK;
}

constexpr int LS_LRUN = 2048;   // points per warp in the Lloyd label sort
static size_t label_sort_bytes(int64_t n, int k) { return sizeof(uint32_t) * (size_t)k * ceil_div(n, LS_LRUN); }

// Lloyd label sort: the point records (xp, index order) by new label into xs,
// stable, so every cluster is one contiguous run in index order
template <int MP>
static int label_sort(const int32_t* newlab, const void* rec_in, void* rec_out, int64_t n, int k, uint32_t* bh,
                      const int64_t* status, cudaStream_t st) {
  return ls_pass(LsLabelKey{newlab}, LsIota{},
                 LsRecOut<MP>{static_cast<const PointRec<MP>*>(rec_in), static_cast<PointRec<MP>*>(rec_out)}, n, k,
                 LS_LRUN, ceil_div(n, LS_LRUN) * LS_LRUN, bh, status, st);
}

// All allocations of one k-means run (no stream work): done for every half
// before any half is enqueued, so the enqueue loop never blocks in cudaMalloc.
static int kmeans_prepare(const KMeansRun& r, int64_t first, const double* uni_h, const int64_t* forced_h,
                          cudaStream_t st) {
  BuildScratch& s = *r.s;
  const HalfView h = r.h;
  const int64_t n = h.n;
  const int k = h.k;
  const int m = h.m;
  if (m > 32) TACO_FAIL(TACO_ERR_PARAMETER, "half width %d exceeds 32", m);
  if (k > 256) TACO_FAIL(TACO_ERR_PARAMETER, "codebook size %d exceeds 256", k);
  const int64_t nbx = ceil_div(n, 256);
  const int64_t nbp = ceil_div(n, PP_BLOCK);
  const int64_t nba = ceil_div(n, (int64_t)AS_THREADS);
  const int mp = m <= 8 ? 8 : m <= 16 ? 16 : 32;   // point-major stride (k_pp_step<MP> buckets)
  const size_t sort_bytes = label_sort_bytes(n, k);
  // host side of the exact replay: numpy's pairwise leaves and combine tree
  // for n -- the same for every half, computed once per n for the process
  // (it cost ~1 ms per half per build)
  if (s.leaves_n != n || s.leaf_blob.empty()) {
    static std::mutex blob_mu;
    static int64_t blob_n = -1, blob_leaves = 0;
    static std::vector<char> blob_cache;
    std::lock_guard<std::mutex> lk(blob_mu);
    if (blob_n != n) {
      std::vector<int64_t> lv;
      pairwise_leaves(0, n, lv);
      const PwTree tree = pairwise_tree(n);
      // layout: (off, len) per leaf as int64, then left[ni], right[ni], level_start[] as int32
      std::vector<char> blob(8 * lv.size() + 4 * (tree.left.size() + tree.right.size() + tree.level_start.size()));
      char* bp = blob.data();
      memcpy(bp, lv.data(), 8 * lv.size());
      bp += 8 * lv.size();
      memcpy(bp, tree.left.data(), 4 * tree.left.size());
      bp += 4 * tree.left.size();
      memcpy(bp, tree.right.data(), 4 * tree.right.size());
      bp += 4 * tree.right.size();
      memcpy(bp, tree.level_start.data(), 4 * tree.level_start.size());
      blob_cache.swap(blob);
      blob_leaves = (int64_t)lv.size() / 2;
      blob_n = n;
    }
    s.leaf_blob = blob_cache;
    s.nleaves = blob_leaves;
    s.leaves_n = n;
  }
  // One arena per half (a single pool allocation: the ~20 scratch buffers
  // used to cost ~20 allocations each, which dominated the warm build's
  // host time when the pool had to map memory)
  struct Cut { DevBuf* b; size_t bytes; };
  const Cut cuts[] = {
      {&s.xsq, 8 * (size_t)n}, {&s.best, 8 * (size_t)n}, {&s.bsum, 8 * (size_t)std::max(nbp, nbx)},
      {&s.picks, 8 * (size_t)k}, {&s.uni, 8 * (size_t)std::max(k, 1)}, {&s.forced, 8 * (size_t)std::max(k, 1)},
      {&s.status, 8 * 16}, {&s.C64, 8 * (size_t)k * m}, {&s.newlab, 4 * (size_t)n}, {&s.pd, 8 * (size_t)n},
      {&s.keys2, 4 * (size_t)n}, {&s.ctl, 8 * 2 * (size_t)k}, {&s.hsum, 8 * (size_t)std::max<int64_t>(nba, ceil_div(n, TC_THREADS))},   // fp64 or tensor-core assign partials
      {&s.xp, 4 * (size_t)n * mp}, {&s.xs, 4 * (size_t)n * mp}, {&s.sorttmp, std::max<size_t>(sort_bytes, 16)},
      {&s.leaves, s.leaf_blob.size()},
      {&s.pbuf, 8 * (size_t)std::max<int64_t>(std::max<int64_t>(n, s.nleaves), 3 * nbp)},
      {&s.cbuf, 8 * (size_t)std::max<int64_t>(std::max<int64_t>(n, 2 * s.nleaves), PP_BLOCK)}};
  size_t total = 0;
  for (const Cut& c : cuts) total += (c.bytes + 255) & ~(size_t)255;
  TACO_TRY(s.arena.ensure(total));
  {
    char* base = s.arena.as<char>();
    for (const Cut& c : cuts) {
      c.b->view_of(base, c.bytes);
      base += (c.bytes + 255) & ~(size_t)255;
    }
  }
  TACO_CHECK_CUDA(cudaMemcpyAsync(s.leaves.p, s.leaf_blob.data(), s.leaf_blob.size(), cudaMemcpyHostToDevice, st));
  const size_t ash = sizeof(double) * ((size_t)k * (m <= 8 ? 8 : m <= 16 ? 16 : 32) + k);
  auto* kas = m <= 8 ? k_assign<8, 1> : m <= 16 ? k_assign<16, 1> : k_assign<32, 1>;
  if (ash > 48 * 1024)
    TACO_CHECK_CUDA(cudaFuncSetAttribute(kas, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ash));
  TACO_CHECK_CUDA(cudaFuncSetAttribute(k_assign_tc<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  TACO_CHECK_CUDA(cudaFuncSetAttribute(k_assign_tc<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  TACO_CHECK_CUDA(cudaFuncSetAttribute(k_assign_tc<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024));
  const size_t css = sizeof(float) * CS_ST * CS_R * mp;
  if (css > 48 * 1024) {
    if (mp == 8) TACO_CHECK_CUDA(cudaFuncSetAttribute(k_cluster_sums<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)css));
    else if (mp == 16) TACO_CHECK_CUDA(cudaFuncSetAttribute(k_cluster_sums<16>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)css));
    else TACO_CHECK_CUDA(cudaFuncSetAttribute(k_cluster_sums<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)css));
  }
  // the draw plan (first pick, uniforms, forced draws) goes up before any
  // kernel of the run is enqueued (the enqueue may be a graph capture)
  TACO_CHECK_CUDA(cudaMemcpyAsync(s.picks.p, &first, 8, cudaMemcpyHostToDevice, st));
  if (k > 1) {
    TACO_CHECK_CUDA(cudaMemcpyAsync(s.uni.p, uni_h, 8 * (k - 1), cudaMemcpyHostToDevice, st));
    if (forced_h)
      TACO_CHECK_CUDA(cudaMemcpyAsync(s.forced.p, forced_h, 8 * (k - 1), cudaMemcpyHostToDevice, st));
  }
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  return TACO_OK;
}

// Lloyd assignment on the tensor cores (k_assign_tc) for half widths <= 8;
// TACO_TC_ASSIGN=0 keeps the all-fp64 k_assign (both give the same labels).
static bool use_tc_assign(int m, int k) {
  static int env = -1;
  if (env < 0) {
    const char* e = getenv("TACO_TC_ASSIGN");
    env = (e && e[0] == '0') ? 0 : 1;
  }
  return env && m <= 32 && k <= 256;
}

// The enqueue of one k-means run is cut into steps -- 0: xsq and the
// point-major copy; 1..k: one k-means++ draw each; then one Lloyd iteration
// each; last: the centroid export -- so the caller can interleave the steps of
// all concurrent halves (every half's first draw is queued before any half's
// second) and the GPU never waits for a host enqueue that is busy elsewhere.
static int kmeans_steps(const KMeansRun& r) { return 1 + r.h.k + r.iters + 1; }

static int kmeans_step(const KMeansRun& r, const int64_t* forced_h, cudaStream_t st, bool timing, int step) {
  BuildScratch& s = *r.s;
  const HalfView h = r.h;
  const int64_t n = h.n;
  const int k = h.k;
  const int m = h.m;
  const int64_t nbx = ceil_div(n, 256);
  const int64_t nbp = ceil_div(n, PP_BLOCK);
  const int64_t nba = ceil_div(n, (int64_t)AS_THREADS);
  const int mp = m <= 8 ? 8 : m <= 16 ? 16 : 32;   // point-major stride (k_pp_step<MP> buckets)
  unsigned long long* cnt = s.ctl.as<unsigned long long>();
  if (step == 0) {
    k_status_init<<<1, 1, 0, st>>>(s.status.as<int64_t>(), k);
    TACO_LAUNCHED();
    // xsq + its maximum (bound for the certified draw)
    k_xsq<<<(unsigned)nbx, 256, 0, st>>>(h, s.xsq.as<double>(), s.status.as<int64_t>());
    TACO_LAUNCHED();
    k_point_major<<<(unsigned)nbx, 256, 0, st>>>(h, mp, s.xp.as<float>());
    TACO_LAUNCHED();
    TACO_CHECK_CUDA(cudaMemsetAsync(cnt, 0, 8 * 2 * (size_t)k, st));
    if (timing) {
      for (auto& e : s.ev) cudaEventCreate(&e);
      cudaEventRecord(s.ev[0], st);
    }
    return TACO_OK;
  }
  if (step <= k) {
    const int ci = step - 1;
    auto* kpp = mp <= 8 ? k_pp_step<8> : mp <= 16 ? k_pp_step<16> : k_pp_step<32>;
    kpp<<<(unsigned)std::min<int64_t>(nbp, std::max(1, 4 * g_num_sms() / std::max(1, r.concurrent))), PP_THREADS,
          0, st>>>(h, s.xp.as<float>(), s.xsq.as<double>(), ci, s.best.as<double>(), s.C64.as<double>(),
                   s.bsum.as<double>(), nbp, s.uni.as<double>(), forced_h ? s.forced.as<int64_t>() : nullptr,
                   s.picks.as<int64_t>(), s.status.as<int64_t>(), s.leaves.as<int64_t>(), s.nleaves,
                   s.cbuf.as<double>(), s.pbuf.as<double>(), s.cbuf.as<double>(), g_force_replay);
    TACO_LAUNCHED();
    if (ci + 1 < k && g_force_replay >= 2) {
      // test hooks: the one-CTA replay (2: the sequential chain, 3: the binade scan)
      k_pp_replay<<<1, RP_THREADS, 0, st>>>(h, s.best.as<double>(), s.uni.as<double>(), ci, s.picks.as<int64_t>(),
                                            s.status.as<int64_t>(), s.leaves.as<int64_t>(), s.nleaves,
                                            s.cbuf.as<double>(), s.pbuf.as<double>(), s.cbuf.as<double>(),
                                            g_force_replay == 2 ? 2 : 1);
      TACO_LAUNCHED();
    } else if (ci + 1 < k) {
      long long* tbin = reinterpret_cast<long long*>(s.pbuf.as<double>());
      const int g1 = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(s.nleaves * 8, 256)), 2 * g_num_sms());
      k_ppx_total<<<g1, 256, 0, st>>>(h, s.best.as<double>(), ci, s.status.as<int64_t>(), s.leaves.as<int64_t>(),
                                      s.nleaves, s.cbuf.as<double>(), s.bsum.as<double>(), nbp, tbin);
      TACO_LAUNCHED();
      const int g2 = (int)std::min<int64_t>(std::max<int64_t>(1, ceil_div(nbp, PX_THREADS / 32)), 2 * g_num_sms());
      k_ppx_quanta<<<g2, PX_THREADS, 0, st>>>(h, s.best.as<double>(), s.uni.as<double>(), ci, s.picks.as<int64_t>(),
                                              s.status.as<int64_t>(), nbp, tbin, tbin + nbp,
                                              s.pbuf.as<double>() + 2 * nbp, s.cbuf.as<double>());
      TACO_LAUNCHED();
    }
    if (ci == k - 1 && timing) cudaEventRecord(s.ev[1], st);
    return TACO_OK;
  }
  if (step <= k + r.iters) {
    const int it = step - k - 1;
    const size_t ash = sizeof(double) * ((size_t)k * (m <= 8 ? 8 : m <= 16 ? 16 : 32) + k);
    auto* kas = m <= 8 ? k_assign<8, 1> : m <= 16 ? k_assign<16, 1> : k_assign<32, 1>;
    const size_t css = sizeof(float) * CS_ST * CS_R * mp;
    unsigned long long* cc = cnt + (size_t)(it & 1) * k;
    unsigned long long* cn = cnt + (size_t)((it + 1) & 1) * k;
    int64_t nb_h = nba;   // hsum entries written by the assignment
    if (use_tc_assign(m, k)) {
      const int npad = (k + 15) & ~15;
      const int64_t ntiles = ceil_div(n, TC_THREADS);
      const int G = (int)std::min<int64_t>(ntiles, 4 * g_num_sms());
      // at most 7 of these CTAs per SM (smem-limited), so their TMEM columns
      // (<= 64 each for K' <= 64) never exceed the SM's 512 and no CTA blocks in
      // tcgen05.alloc behind another half's kernel
      const size_t tsmem = sizeof(float) * (2 * TC_THREADS * (size_t)mp + 2 * (size_t)npad * mp) +
                           sizeof(double) * ((size_t)k * mp + k + 1) + sizeof(float) * 2 * npad;
      const int ncols = npad <= 32 ? 32 : npad <= 64 ? 64 : npad <= 128 ? 128 : 256;
      const size_t tsm_launch =
          std::min<size_t>(std::max(tsmem, (size_t)(228 * 1024) / (size_t)(512 / ncols) + 1024), 200 * 1024);
      auto* ktc = mp == 8 ? k_assign_tc<8> : mp == 16 ? k_assign_tc<16> : k_assign_tc<32>;
      ktc<<<G, TC_THREADS, tsm_launch, st>>>(h, s.xp.as<float>(), s.xsq.as<double>(), s.C64.as<double>(), r.labels,
                                             s.newlab.as<int32_t>(), s.pd.as<double>(), it, s.status.as<int64_t>(),
                                             s.hsum.as<double>(), cc, cn, npad);
      nb_h = G;
    } else {
      kas<<<(unsigned)nba, AS_THREADS, ash, st>>>(h, s.xsq.as<double>(), s.C64.as<double>(), r.labels,
                                                  s.newlab.as<int32_t>(), s.pd.as<double>(), it,
                                                  s.status.as<int64_t>(), s.hsum.as<double>(), cc, cn);
    }
    TACO_LAUNCHED();
    k_lloyd_ctl<<<1, 1024, 0, st>>>(s.hsum.as<double>(), nb_h, it, s.status.as<int64_t>(), r.history,
                                    r.n_iter);
    TACO_LAUNCHED();
    // stable counting sort of the point records by label (index order inside a label)
    const int32_t* nl = s.newlab.as<int32_t>();
    uint32_t* bh = s.sorttmp.as<uint32_t>();
    const int64_t* stt = s.status.as<int64_t>();
    if (mp == 8) {
      TACO_TRY(label_sort<8>(nl, s.xp.p, s.xs.p, n, k, bh, stt, st));
      k_cluster_sums<8><<<(unsigned)k, CS_THREADS, css, st>>>(h, s.xs.as<PointRec<8>>(), s.status.as<int64_t>(), cc,
                                                              s.newlab.as<int32_t>(), r.labels, s.C64.as<double>());
    } else if (mp == 16) {
      TACO_TRY(label_sort<16>(nl, s.xp.p, s.xs.p, n, k, bh, stt, st));
      k_cluster_sums<16><<<(unsigned)k, CS_THREADS, css, st>>>(h, s.xs.as<PointRec<16>>(), s.status.as<int64_t>(),
                                                               cc, s.newlab.as<int32_t>(), r.labels,
                                                               s.C64.as<double>());
    } else {
      TACO_TRY(label_sort<32>(nl, s.xp.p, s.xs.p, n, k, bh, stt, st));
      k_cluster_sums<32><<<(unsigned)k, CS_THREADS, css, st>>>(h, s.xs.as<PointRec<32>>(), s.status.as<int64_t>(),
                                                               cc, s.newlab.as<int32_t>(), r.labels,
                                                               s.C64.as<double>());
    }
    count_launch(1);
    TACO_CHECK_CUDA(cudaGetLastError());
    k_reseed<<<1, 1024, 0, st>>>(h, s.status.as<int64_t>(), cc, s.pd.as<double>(),
                                 r.labels, s.C64.as<double>());
    TACO_LAUNCHED();
    return TACO_OK;
  }
  k_centroids_out<<<(unsigned)ceil_div((int64_t)k * m, 256), 256, 0, st>>>(s.C64.as<double>(), k * m,
                                                                            r.cent_out);
  TACO_LAUNCHED();
  if (timing) cudaEventRecord(s.ev[2], st);
  return TACO_OK;
}

static int kmeans_enqueue(const KMeansRun& r, const int64_t* forced_h, cudaStream_t st, bool timing) {
  for (int i = 0; i < kmeans_steps(r); ++i) TACO_TRY(kmeans_step(r, forced_h, st, timing, i));
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

// sort keys for the CSR: (chunk, cell) of every local id; values = the id.
// A stable radix sort of ascending ids by this key is the (chunk, cell, id)
// order the counting kernels read (imi.py:72-81 lexsort((arange, l2, l1)),
// chunk-major).

}  // namespace taco

using namespace taco;

namespace {
int ensure_half_streams(taco_index* idx, int want) {
  while ((int)idx->half_streams.size() < want) {
    cudaStream_t s;
    TACO_CHECK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    idx->half_streams.push_back(s);
    cudaEvent_t e;
    TACO_CHECK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    idx->half_ev.push_back(e);
  }
  if (!idx->km_fork) TACO_CHECK_CUDA(cudaEventCreateWithFlags(&idx->km_fork, cudaEventDisableTiming));
  return TACO_OK;
}
}  // namespace

extern "C" {

static int covariance_impl(const float* Xd, int64_t n, int d, cudaStream_t st, double* mean_h,
                           double* gram_h, int64_t* bad_row, const double* mean_ready = nullptr) {
  DevBuf bad, mean, G, cstate;
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
    if (mean_ready) {   // the column mean was chained while X was being uploaded
      TACO_CHECK_CUDA(cudaMemcpyAsync(mean.p, mean_ready, 8 * (size_t)d, cudaMemcpyDeviceToDevice, st));
    } else {
      if ((rc = cstate.ensure(8 * (size_t)d))) break;
      if ((rc = launch_colmean(st, Xd, 0, n, n, d, cstate.as<double>(), mean.as<double>(), 0))) break;
    }
    const int64_t dd = (int64_t)d * d;
    TACO_CHECK_CUDA(cudaMemsetAsync(G.p, 0, 8 * (size_t)dd, st));
    if ((rc = gram_chain(Xd, n, d, mean.as<double>(), kGramBlock, G.as<double>(), st))) break;
    cudaMemcpyAsync(mean_h, mean.p, 8 * d, cudaMemcpyDeviceToHost, st);
    cudaMemcpyAsync(gram_h, G.p, 8 * dd, cudaMemcpyDeviceToHost, st);
    e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; }
  } while (0);
  bad.release(); mean.release(); G.release(); cstate.release();
  return rc;
}

int taco_fit_covariance(taco_index* idx, double* mean_h, double* gram_h, int64_t* bad_row) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "no data uploaded");
  const double* mr = nullptr;
  if (idx->mean_ready) {   // chained during the staged upload on the aux stream
    TACO_CHECK_CUDA(cudaStreamSynchronize(idx->aux));
    mr = idx->colmean.as<double>();
  }
  return covariance_impl(idx->X.as<float>(), idx->n, idx->d, idx->stream, mean_h, gram_h, bad_row, mr);
}

// ---------------------------------------------------- point-sharded build
// Column-sum chain of this shard's rows (numpy mean(axis=0)'s sequential
// per-column add, spectral.py:107): starts from carry_in (the running sums of
// all earlier shards) or, without one, from this shard's first row; the
// running sums after its last row go to carry_out.  *bad_row = the first
// local row holding a non-finite value (-1 if none; nothing else is done).
int taco_shard_colsum(taco_index* idx, const double* carry_in_h, double* carry_out_h, int64_t* bad_row) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "no data uploaded");
  const int64_t n = idx->n;
  const int d = idx->d;
  cudaStream_t st = idx->stream;
  if (idx->mean_ready) TACO_CHECK_CUDA(cudaStreamSynchronize(idx->aux));
  DevBuf bad, state;
  TACO_TRY(bad.ensure(8));
  TACO_TRY(state.ensure(8 * (size_t)d));
  unsigned long long init = ~0ull, b = 0;
  TACO_CHECK_CUDA(cudaMemcpyAsync(bad.p, &init, 8, cudaMemcpyHostToDevice, st));
  k_nonfinite<<<1184, 256, 0, st>>>(idx->X.as<float>(), n * d, d, bad.as<unsigned long long>());
  count_launch();
  TACO_CHECK_CUDA(cudaMemcpyAsync(&b, bad.p, 8, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  *bad_row = b == ~0ull ? -1 : (int64_t)b;
  if (b != ~0ull) return TACO_OK;
  if (carry_in_h) TACO_CHECK_CUDA(cudaMemcpyAsync(state.p, carry_in_h, 8 * (size_t)d, cudaMemcpyHostToDevice, st));
  TACO_TRY(launch_colmean(st, idx->X.as<float>(), 0, n, -1, d, state.as<double>(), nullptr, carry_in_h ? 1 : 0));
  TACO_CHECK_CUDA(cudaMemcpyAsync(carry_out_h, state.p, 8 * (size_t)d, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  return TACO_OK;
}

// Centred Gram chain of this shard's rows (spectral.py:108-109): gram_out =
// carry_in (or 0) + the kGramBlock-row block partials of its rows in order,
// the same sequence taco_fit_covariance runs over all rows, so shards that
// start on multiples of block_rows reproduce the single-GPU Gram exactly.
int taco_shard_gram(taco_index* idx, const double* mean_h, int64_t block_rows, const double* carry_in_h,
                    double* carry_out_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "no data uploaded");
  if (block_rows <= 0) block_rows = kGramBlock;
  const int d = idx->d;
  const int64_t dd = (int64_t)d * d;
  cudaStream_t st = idx->stream;
  DevBuf mean, G;
  TACO_TRY(mean.ensure(8 * (size_t)d));
  TACO_TRY(G.ensure(8 * (size_t)dd));
  TACO_CHECK_CUDA(cudaMemcpyAsync(mean.p, mean_h, 8 * (size_t)d, cudaMemcpyHostToDevice, st));
  if (carry_in_h) TACO_CHECK_CUDA(cudaMemcpyAsync(G.p, carry_in_h, 8 * (size_t)dd, cudaMemcpyHostToDevice, st));
  else TACO_CHECK_CUDA(cudaMemsetAsync(G.p, 0, 8 * (size_t)dd, st));
  TACO_TRY(gram_chain(idx->X.as<float>(), idx->n, d, mean.as<double>(), block_rows, G.as<double>(), st));
  TACO_CHECK_CUDA(cudaMemcpy(carry_out_h, G.p, 8 * (size_t)dd, cudaMemcpyDeviceToHost));
  return TACO_OK;
}

int taco_gram_block_rows(void) { return (int)kGramBlock; }

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
  // Halves in flight: up to 16, fewer when their scratch would not fit in the
  // free device memory (n = 1e8 needs ~15 GB per half).  Cached pool memory
  // is returned to the device first if that is what stands in the way.
  const int mpx = std::max(idx->m1, idx->m2) <= 8 ? 8 : std::max(idx->m1, idx->m2) <= 16 ? 16 : 32;
  const size_t per_half = (size_t)n * (64 + 12 * (size_t)mpx) + ((size_t)64 << 20);
  auto fit = [&]() {
    size_t fr = 0, tot = 0;
    cudaMemGetInfo(&fr, &tot);
    return (int)std::max<size_t>(1, (size_t)(0.85 * (double)fr) / per_half);
  };
  int NS = std::min({H, 16, fit()});
  if (NS < std::min(H, 16)) {
    cudaMemPool_t pool;
    if (cudaDeviceGetDefaultMemPool(&pool, idx->device) == cudaSuccess) {
      cudaDeviceSynchronize();
      cudaMemPoolTrimTo(pool, 0);
    }
    NS = std::min({H, 16, fit()});
  }
  if (const char* e = getenv("TACO_KM_HALVES")) NS = std::max(1, std::min(NS, atoi(e)));   // experiments
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
    std::vector<KMeansRun> runs;
    timespec tp0;
    clock_gettime(CLOCK_MONOTONIC, &tp0);
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
      r.concurrent = w1 - w0;
      TACO_TRY(kmeans_prepare(r, first_h[hh], uniforms_h + (size_t)hh * std::max(kp - 1, 0),
                              forced_h ? forced_h + (size_t)hh * std::max(kp - 1, 0) : nullptr,
                              idx->half_streams[hh - w0]));
      runs.push_back(r);
    }
    // All halves of the wave are independent.  Default: direct launches,
    // interleaved step by step across the halves (every half's draw i is
    // queued before any half's draw i+1), so the GPU starts on all halves at
    // once and the host enqueue (~2 us per launch) overlaps the execution.
    // TACO_KM_GRAPH=1 captures the same work into one graph instead (a branch
    // per half; instantiation costs more than it saves for a single build).
    const char* ge = getenv("TACO_KM_GRAPH");
    const bool timing = getenv("TACO_DEBUG_TIMING") != nullptr;
    const bool graph = ge && ge[0] == '1' && !timing;
    cudaStream_t origin = idx->stream;
    cudaGraph_t g = nullptr;
    const bool gdbg = getenv("TACO_DEBUG_GRAPH") != nullptr;
    auto now_ms = []() {
      timespec ts;
      clock_gettime(CLOCK_MONOTONIC, &ts);
      return ts.tv_sec * 1e3 + ts.tv_nsec * 1e-6;
    };
    const double tg0 = now_ms();
    if (gdbg)
      fprintf(stderr, "[taco] k-means prepare (allocations, draw-plan upload) %.2f ms\n",
              tg0 - (tp0.tv_sec * 1e3 + tp0.tv_nsec * 1e-6));
    int erc = TACO_OK;
    auto forced_of = [&](int hh) { return forced_h ? forced_h + (size_t)hh * std::max(kp - 1, 0) : nullptr; };
    if (graph) {
      TACO_CHECK_CUDA(cudaStreamBeginCapture(origin, cudaStreamCaptureModeThreadLocal));
      TACO_CHECK_CUDA(cudaEventRecord(idx->km_fork, origin));
      for (int hh = w0; hh < w1 && erc == TACO_OK; ++hh) {
        cudaStream_t hs = idx->half_streams[hh - w0];
        cudaStreamWaitEvent(hs, idx->km_fork, 0);
        erc = kmeans_enqueue(runs[hh - w0], forced_of(hh), hs, false);
        cudaEventRecord(idx->half_ev[hh - w0], hs);
        cudaStreamWaitEvent(origin, idx->half_ev[hh - w0], 0);
      }
      cudaError_t ce = cudaStreamEndCapture(origin, &g);
      if (erc != TACO_OK) { if (g) cudaGraphDestroy(g); return erc; }
      if (ce != cudaSuccess) TACO_FAIL(TACO_ERR_CUDA, "k-means graph capture: %s", cudaGetErrorString(ce));
      const double tg1 = now_ms();
      cudaGraphExec_t ex = nullptr;
      TACO_CHECK_CUDA(cudaGraphInstantiate(&ex, g, 0));
      cudaGraphDestroy(g);
      const double tg2 = now_ms();
      cudaError_t le = cudaGraphLaunch(ex, origin);
      const double tg3 = now_ms();
      cudaError_t se = cudaStreamSynchronize(origin);
      if (gdbg)
        fprintf(stderr, "[taco] k-means graph: prepare+capture %.2f ms, instantiate %.2f ms, launch %.2f ms, run %.2f ms\n",
                tg1 - tg0, tg2 - tg1, tg3 - tg2, now_ms() - tg3);
      cudaGraphExecDestroy(ex);
      if (le != cudaSuccess || se != cudaSuccess)
        TACO_FAIL(TACO_ERR_CUDA, "k-means graph: %s", cudaGetErrorString(le != cudaSuccess ? le : se));
    } else {
      int maxs = 0;
      for (auto& r : runs) maxs = std::max(maxs, kmeans_steps(r));
      for (int i = 0; i < maxs && erc == TACO_OK; ++i)
        for (int hh = w0; hh < w1 && erc == TACO_OK; ++hh)
          if (i < kmeans_steps(runs[hh - w0]))
            erc = kmeans_step(runs[hh - w0], forced_of(hh), idx->half_streams[hh - w0], timing, i);
      if (gdbg) fprintf(stderr, "[taco] k-means direct enqueue %.2f ms\n", now_ms() - tg0);
    }
    TACO_TRY(erc);
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
  // the scratch goes back to the device pool (a later build reuses it)
  for (auto& bs : idx->bs) {
    DevBuf* sb[] = {&bs.xsq, &bs.best, &bs.bsum, &bs.picks, &bs.uni, &bs.forced, &bs.status, &bs.C64, &bs.csq,
                    &bs.newlab, &bs.pd, &bs.changed, &bs.perm, &bs.lhist, &bs.loff, &bs.ctl, &bs.hsum, &bs.draws,
                    &bs.leaves, &bs.pbuf, &bs.cbuf, &bs.iota, &bs.keys2, &bs.sorttmp, &bs.xp, &bs.xs, &bs.arena};
    for (auto* b : sb) b->release();
    bs.leaves_n = -1;
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
  // (chunk, cell, id) order = inside every id chunk (a segment: chunk is a
  // multiple of the run), a stable sort by l2 then a stable sort by l1
  constexpr int CRUN = 1024;
  DevBuf chist, ids1, bh;
  TACO_TRY(chist.ensure(sizeof(uint32_t) * (size_t)nc * K2));
  TACO_TRY(ids1.ensure(sizeof(uint32_t) * (size_t)n));
  TACO_TRY(bh.ensure(sizeof(uint32_t) * (size_t)kp * ceil_div(n, CRUN)));
  if (idx->chunk % CRUN) TACO_FAIL(TACO_ERR_STATE, "id chunk %lld is not a multiple of %d", (long long)idx->chunk, CRUN);
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
    TACO_TRY(ls_pass(LsLabelKey{l2}, LsIota{}, LsIdOut{ids1.as<uint32_t>()}, n, kp, CRUN, idx->chunk,
                     bh.as<uint32_t>(), nullptr, st));
    TACO_TRY(ls_pass(LsIdKey{l1}, LsIds{ids1.as<uint32_t>()}, LsIdOut{idx->ids.as<uint32_t>() + (size_t)j * n}, n,
                     kp, CRUN, idx->chunk, bh.as<uint32_t>(), nullptr, st));
  }
  cudaError_t e = cudaStreamSynchronize(st);
  chist.release();
  ids1.release();
  bh.release();
  if (e != cudaSuccess) TACO_FAIL(TACO_ERR_CUDA, "%s", cudaGetErrorString(e));
  idx->has_cells = true;
  if (idx->n_global == idx->n) idx->has_gsize = true;
  TACO_TRY(build_count_csr(idx));
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
  g_force_replay = on;   // 1: every draw replays (k_ppx_*); 2: the one-CTA sequential chain; 3: the one-CTA binade scan
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
    if ((rc = kmeans_prepare(r, first, uniforms_h, forced_h, st)) || (rc = kmeans_enqueue(r, forced_h, st, false)))
      break;
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
                  &s.leaves, &s.pbuf, &s.cbuf, &s.iota, &s.keys2, &s.sorttmp, &s.xp, &s.xs, &s.arena};
  for (auto* b : sb) b->release();
  return rc;
}

}  // extern "C"
