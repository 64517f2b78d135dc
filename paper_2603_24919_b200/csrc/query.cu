// Batched TaCo query path on sm_100a.
//
//  per tile of Qt queries, all on one stream:
//   k_transform      qt = f32((q - mu) @ M)                spectral.py:301-316
//   k_csort          fp64 centroid distances + stable rank  imi.py:88-106
//   k_traverse       multi-sequence heap traversal          imi.py:130-166
//   k_count          uint8 collision counts, one 64 KiB id chunk per CTA in
//                    shared memory, + per-chunk level histograms   engine.py:201-219
//   k_hist_reduce    per-query histograms (all-reduced across shards here)
//   k_select         Alg. 5 threshold + candidate offsets   engine.py:239-251
//   k_compact        ordered candidate ids (score >= L)     engine.py:250
//   k_rerank         fp64 exact distances, rows staged through smem   engine.py:272-274
//   k_topk           radix select + bitonic sort on (d2, id)          engine.py:275-279
#include <algorithm>
#include <cmath>
#include <vector>

#include "index.cuh"

namespace taco {

// ------------------------------------------------------------- profiler
// Optional per-kernel timing with CUDA events recorded on the launching
// stream (bench.py's roofline), plus algorithmic-work counters.
enum KId { K_TRANSFORM, K_CSORT, K_TRAVERSE, K_COUNT, K_HIST, K_SELECT, K_COMPACT, K_RERANK, K_TOPK,
           K_FINAL, K_NKIDS };
static const char* kKNames[K_NKIDS] = {"k_transform", "k_csort", "k_traverse", "k_count", "k_hist_reduce",
                                       "k_select", "k_compact", "k_rerank", "k_topk", "k_finalize"};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct P { int kid; cudaEvent_t a, b; };
  std::vector<P> pend;
  double ms[K_NKIDS] = {};
  int64_t cnt[K_NKIDS] = {};
  int64_t sumR = 0, sumC = 0, sumPops = 0, queries = 0, tiles = 0, bytes_scores = 0;
};
static Prof g_prof;
static cudaEvent_t prof_event() {
  if (!g_prof.pool.empty()) { cudaEvent_t e = g_prof.pool.back(); g_prof.pool.pop_back(); return e; }
  cudaEvent_t e;
  cudaEventCreate(&e);
  return e;
}
struct ProfScope {
  int kid;
  cudaStream_t st;
  cudaEvent_t a = nullptr;
  ProfScope(int k, cudaStream_t s) : kid(k), st(s) {
    if (g_prof.on) { a = prof_event(); cudaEventRecord(a, st); }
  }
  ~ProfScope() {
    if (a) {
      cudaEvent_t b = prof_event();
      cudaEventRecord(b, st);
      g_prof.pend.push_back({kid, a, b});
    }
  }
};
static void prof_drain() {
  for (auto& p : g_prof.pend) {
    cudaEventSynchronize(p.b);
    float ms = 0.f;
    cudaEventElapsedTime(&ms, p.a, p.b);
    g_prof.ms[p.kid] += ms;
    g_prof.cnt[p.kid] += 1;
    g_prof.pool.push_back(p.a);
    g_prof.pool.push_back(p.b);
  }
  g_prof.pend.clear();
}

// ------------------------------------------------------------------ csort
// One warp per (query, subspace, half): fp64 direct-form distances to the K'
// centroids (einsum order) and their stable ascending rank (ties -> lower label).
__global__ void k_csort(const float* __restrict__ qt, int Q, int n_sub, int s, int m1, int m2,
                        int kp, const float* __restrict__ cb1, const float* __restrict__ cb2,
                        double* __restrict__ sd, uint16_t* __restrict__ sl) {
  extern __shared__ double csh[];
  const int wib = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t w = (int64_t)blockIdx.x * (blockDim.x >> 5) + wib;
  if (w >= (int64_t)Q * n_sub * 2) return;
  const int h = (int)(w & 1);
  const int64_t qj = w >> 1;
  const int j = (int)(qj % n_sub);
  const int64_t q = qj / n_sub;
  const int m = h ? m2 : m1;
  const float* C = h ? cb2 + (size_t)j * kp * m2 : cb1 + (size_t)j * kp * m1;
  const float* qv = qt + q * (int64_t)n_sub * s + (int64_t)j * s + (h ? m1 : 0);
  double* dd = csh + wib * kp;
  for (int c = lane; c < kp; c += 32) {
    const float* cr = C + (size_t)c * m;
    dd[c] = einsum_sq([&](int t) { return __dsub_rn((double)cr[t], (double)qv[t]); }, m);
  }
  __syncwarp();
  double* osd = sd + w * kp;
  uint16_t* osl = sl + w * kp;
  for (int c = lane; c < kp; c += 32) {
    const double v = dd[c];
    int rank = 0;
    for (int c2 = 0; c2 < kp; ++c2) {
      const double u = dd[c2];
      rank += (u < v) || (u == v && c2 < c);
    }
    osd[rank] = v;
    osl[rank] = (uint16_t)c;
  }
}

// --------------------------------------------------------------- traverse
// One thread per (query, subspace).  Min-heap of (key, row rank, col rank)
// with the frontier rule of imi.py:155-165; each row holds at most one heap
// entry, so KMAX >= K' suffices.  Cell sizes are the GLOBAL sizes so every
// shard derives the same popped set.
template <int KMAX>
__global__ void __launch_bounds__(128) k_traverse(const double* __restrict__ sd,
                                                  const uint16_t* __restrict__ sl,
                                                  const int64_t* __restrict__ gsize, int Q,
                                                  int n_sub, int kp, int64_t target,
                                                  uint16_t* __restrict__ pops, int cap,
                                                  double* __restrict__ keys_out,
                                                  int32_t* __restrict__ npop,
                                                  int64_t* __restrict__ ret) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (int64_t)Q * n_sub) return;
  const int j = (int)(t % n_sub);
  const double* d1 = sd + t * 2 * kp;
  const double* d2 = d1 + kp;
  const uint16_t* l1 = sl + t * 2 * kp;
  const uint16_t* l2 = l1 + kp;
  const int64_t* gs = gsize + (size_t)j * kp * kp;
  double hk[KMAX];
  uint32_t hp[KMAX];
  int hn = 0;
  auto less = [&](double ka, uint32_t pa, double kb, uint32_t pb) {
    return ka < kb || (ka == kb && pa < pb);
  };
  auto push = [&](double key, uint32_t pc) {
    int i = hn++;
    while (i > 0) {
      int par = (i - 1) >> 1;
      if (!less(key, pc, hk[par], hp[par])) break;
      hk[i] = hk[par];
      hp[i] = hp[par];
      i = par;
    }
    hk[i] = key;
    hp[i] = pc;
  };
  push(__dadd_rn(d1[0], d2[0]), 0u);
  int np = 0;
  int64_t got = 0;
  uint16_t* out = pops + t * cap;
  double* kout = keys_out ? keys_out + t * cap : nullptr;
  while (hn > 0) {
    const double key = hk[0];
    const uint32_t pc = hp[0];
    // pop: move last to root and sift down
    --hn;
    if (hn > 0) {
      const double lk = hk[hn];
      const uint32_t lp = hp[hn];
      int i = 0;
      while (true) {
        int a = 2 * i + 1;
        if (a >= hn) break;
        int b = a + 1;
        int m = (b < hn && less(hk[b], hp[b], hk[a], hp[a])) ? b : a;
        if (!less(hk[m], hp[m], lk, lp)) break;
        hk[i] = hk[m];
        hp[i] = hp[m];
        i = m;
      }
      hk[i] = lk;
      hp[i] = lp;
    }
    const int r = (int)(pc >> 16), c = (int)(pc & 0xFFFF);
    const int cell = (int)l1[r] * kp + (int)l2[c];
    out[np] = (uint16_t)cell;
    if (kout) kout[np] = key;
    ++np;
    got += gs[cell];
    if (got >= target) break;
    if (c == 0 && r + 1 < kp) push(__dadd_rn(d1[r + 1], d2[0]), (uint32_t)(r + 1) << 16);
    if (c + 1 < kp) push(__dadd_rn(d1[r], d2[c + 1]), ((uint32_t)r << 16) | (uint32_t)(c + 1));
  }
  npop[t] = np;
  ret[t] = got;
}

// ---------------------------------------------------------- level counting
// Histogram of levels 1..n_sub over `nbytes` score bytes (4-byte words),
// per-thread partial counts accumulated into cnt[] (shared, n_sub+1 ints).
__device__ __forceinline__ void count_levels_words(const uint32_t* words, int nwords, int n_sub,
                                                   int* cnt_sh) {
  if (n_sub <= 15) {
    int loc[16];
#pragma unroll
    for (int l = 0; l < 16; ++l) loc[l] = 0;
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
      const uint32_t w = words[i];
      if (w == 0) continue;
#pragma unroll
      for (int l = 1; l < 16; ++l) {
        if (l > n_sub) break;
        loc[l] += __popc(__vcmpeq4(w, 0x01010101u * (uint32_t)l) & 0x01010101u);
      }
    }
#pragma unroll
    for (int l = 1; l < 16; ++l) {
      if (l > n_sub) break;
      int v = loc[l];
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
      if ((threadIdx.x & 31) == 0 && v) atomicAdd(&cnt_sh[l], v);
    }
  } else {
    for (int i = threadIdx.x; i < nwords; i += blockDim.x) {
      uint32_t w = words[i];
      while (w) {
        int b = __ffs(w) - 1;
        int byte = b >> 3;
        int v = (int)((w >> (byte * 8)) & 0xFF);
        atomicAdd(&cnt_sh[v], 1);
        w &= ~(0xFFu << (byte * 8));
      }
    }
  }
}

// ------------------------------------------------------------------ count
constexpr int CNT_THREADS = 512;
constexpr int CNT_PB = 1024;   // popped cells staged per batch
constexpr int CNT_E = 8;       // ids gathered per thread before the byte RMWs

__global__ void __launch_bounds__(CNT_THREADS) k_count(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ ids, const uint32_t* __restrict__ offs, int n_sub, int K2,
    int64_t n, int64_t nchunks, uint8_t* __restrict__ scores, int32_t* __restrict__ part) {
  extern __shared__ __align__(16) uint8_t smem[];
  uint8_t* table = smem;
  uint32_t* st = reinterpret_cast<uint32_t*>(smem + kChunk);
  uint32_t* pref = st + CNT_PB;
  __shared__ int wtot[CNT_THREADS / 32];
  __shared__ int cnt_sh[256];
  const int c = blockIdx.x;
  const int64_t q = blockIdx.y;
  const int tid = threadIdx.x;
  const int64_t base = (int64_t)c << kChunkShift;
  const int valid = (int)min((int64_t)kChunk, n - base);
  uint4* t4 = reinterpret_cast<uint4*>(table);
  for (int i = tid; i < (int)(kChunk / 16); i += CNT_THREADS) t4[i] = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < 256; i += CNT_THREADS) cnt_sh[i] = 0;
  __syncthreads();
  const size_t offs_len = (size_t)nchunks * K2 + 1;
  for (int j = 0; j < n_sub; ++j) {
    const uint16_t* P = pops + ((size_t)q * n_sub + j) * cap;
    const int np = npop[q * n_sub + j];
    const uint32_t* O = offs + (size_t)j * offs_len + (size_t)c * K2;
    const uint32_t* I = ids + (size_t)j * n;
    for (int b0 = 0; b0 < np; b0 += CNT_PB) {
      const int nb = min(CNT_PB, np - b0);
      // phase A: slice [O[cell], O[cell+1]) of every popped cell in this chunk
      for (int t = tid; t < CNT_PB; t += CNT_THREADS) {
        uint32_t len = 0;
        if (t < nb) {
          const int cell = P[b0 + t];
          const uint32_t s0 = O[cell], s1 = O[cell + 1];
          st[t] = s0;
          len = s1 - s0;
        }
        pref[t + 1] = len;
      }
      __syncthreads();
      // inclusive scan of pref[1..CNT_PB]: 2 elements per thread
      {
        uint32_t a = pref[2 * tid + 1], b = pref[2 * tid + 2];
        uint32_t sum = a + b;
        uint32_t v = sum;
        const int lane = tid & 31, wid = tid >> 5;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          uint32_t x = __shfl_up_sync(0xffffffffu, v, o);
          if (lane >= o) v += x;
        }
        if (lane == 31) wtot[wid] = (int)v;
        __syncthreads();
        if (wid == 0) {
          uint32_t wv = lane < CNT_THREADS / 32 ? (uint32_t)wtot[lane] : 0u;
#pragma unroll
          for (int o = 1; o < 32; o <<= 1) {
            uint32_t x = __shfl_up_sync(0xffffffffu, wv, o);
            if (lane >= o) wv += x;
          }
          if (lane < CNT_THREADS / 32) wtot[lane] = (int)wv;
        }
        __syncthreads();
        const uint32_t off = (wid ? (uint32_t)wtot[wid - 1] : 0u) + v - sum;
        pref[2 * tid + 1] = off + a;
        pref[2 * tid + 2] = off + a + b;
        if (tid == 0) pref[0] = 0;
      }
      __syncthreads();
      const uint32_t total = pref[nb];
      // phase B: each thread owns a contiguous range of the flattened ids
      const uint32_t per = (total + CNT_THREADS - 1) / CNT_THREADS;
      uint32_t f = per * tid;
      const uint32_t f1 = min(total, f + per);
      if (f < f1) {
        int lo = 0, hi = nb;  // largest t with pref[t] <= f
        while (hi - lo > 1) {
          int mid = (lo + hi) >> 1;
          if (pref[mid] <= f) lo = mid; else hi = mid;
        }
        int t = lo;
        while (f < f1) {
          uint32_t idv[CNT_E];
          int cntv = 0;
#pragma unroll
          for (int e = 0; e < CNT_E; ++e) {
            if (f < f1) {
              while (f >= pref[t + 1]) ++t;
              idv[e] = __ldg(I + st[t] + (f - pref[t]));
              ++f;
              ++cntv;
            }
          }
#pragma unroll
          for (int e = 0; e < CNT_E; ++e)
            if (e < cntv) table[idv[e] - (uint32_t)base] += 1;
        }
      }
      __syncthreads();
    }
  }
  // store the chunk's table and its level histogram
  uint4* dst = reinterpret_cast<uint4*>(scores + ((size_t)q * nchunks + c) * kChunk);
  for (int i = tid; i < (int)(kChunk / 16); i += CNT_THREADS) dst[i] = t4[i];
  count_levels_words(reinterpret_cast<const uint32_t*>(table), (valid + 3) / 4, n_sub, cnt_sh);
  __syncthreads();
  int32_t* pp = part + ((size_t)q * nchunks + c) * (n_sub + 1);
  if (tid == 0) {
    int nz = 0;
    for (int l = 1; l <= n_sub; ++l) nz += cnt_sh[l];
    pp[0] = valid - nz;
  }
  for (int l = 1 + tid; l <= n_sub; l += CNT_THREADS) pp[l] = cnt_sh[l];
}

// Level histograms of externally provided score chunks (select_candidates tap).
__global__ void k_chunk_hist(const uint8_t* __restrict__ scores, int64_t n, int64_t nchunks,
                             int n_sub, int32_t* __restrict__ part) {
  __shared__ int cnt_sh[256];
  const int c = blockIdx.x;
  const int64_t q = blockIdx.y;
  for (int i = threadIdx.x; i < 256; i += blockDim.x) cnt_sh[i] = 0;
  __syncthreads();
  const int64_t base = (int64_t)c << kChunkShift;
  const int valid = (int)min((int64_t)kChunk, n - base);
  const uint32_t* w = reinterpret_cast<const uint32_t*>(scores + ((size_t)q * nchunks + c) * kChunk);
  count_levels_words(w, (valid + 3) / 4, n_sub, cnt_sh);
  __syncthreads();
  int32_t* pp = part + ((size_t)q * nchunks + c) * (n_sub + 1);
  if (threadIdx.x == 0) {
    int nz = 0;
    for (int l = 1; l <= n_sub; ++l) nz += cnt_sh[l];
    pp[0] = valid - nz;
  }
  for (int l = 1 + threadIdx.x; l <= n_sub; l += blockDim.x) pp[l] = cnt_sh[l];
}

__global__ void k_hist_reduce(const int32_t* __restrict__ part, int64_t nchunks, int n_sub,
                              int64_t* __restrict__ hist) {
  const int64_t q = blockIdx.x;
  for (int l = threadIdx.x; l <= n_sub; l += blockDim.x) {
    int64_t acc = 0;
    for (int64_t c = 0; c < nchunks; ++c) acc += part[((size_t)q * nchunks + c) * (n_sub + 1) + l];
    hist[q * (n_sub + 1) + l] = acc;
  }
}

// ----------------------------------------------------------------- select
// One thread per query: Alg. 5 on the (global) histogram exactly as
// engine.py:239-249 evaluates it in Python doubles, then the local candidate
// count per chunk and the block-wide query offsets.
__global__ void __launch_bounds__(1024) k_select(const int64_t* __restrict__ ghist,
                                                 const int32_t* __restrict__ part, int Q,
                                                 int64_t nchunks, int n_sub, double budget,
                                                 int32_t* __restrict__ lvl,
                                                 int64_t* __restrict__ cnum_global,
                                                 int64_t* __restrict__ coff,
                                                 int64_t* __restrict__ qbase,
                                                 int64_t* __restrict__ total) {
  __shared__ int64_t wsum[32];
  const int q = threadIdx.x;
  int64_t local = 0;
  if (q < Q) {
    const int64_t* h = ghist + (size_t)q * (n_sub + 1);
    int L = n_sub;
    int64_t cand = 0;
    for (int j = n_sub; j >= 0; --j) {
      cand += h[j];
      if ((double)h[j] <= __dsub_rn(budget, (double)cand)) L -= 1; else break;
    }
    if (L < 0) L = 0;
    lvl[q] = L;
    cnum_global[q] = cand;
    for (int64_t c = 0; c < nchunks; ++c) {
      const int32_t* pp = part + ((size_t)q * nchunks + c) * (n_sub + 1);
      int64_t cc = 0;
      for (int l = L; l <= n_sub; ++l) cc += pp[l];
      coff[(size_t)q * nchunks + c] = local;
      local += cc;
    }
  }
  // exclusive scan of `local` over the block
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  int64_t v = local;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t x = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o) v += x;
  }
  if (lane == 31) wsum[wid] = v;
  __syncthreads();
  if (wid == 0) {
    int64_t wv = lane < (int)(blockDim.x >> 5) ? wsum[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t x = __shfl_up_sync(0xffffffffu, wv, o);
      if (lane >= o) wv += x;
    }
    wsum[lane] = wv;
  }
  __syncthreads();
  const int64_t incl = (wid ? wsum[wid - 1] : 0) + v;
  if (q < Q) qbase[q] = incl - local;
  if (q == Q - 1) {
    qbase[Q] = incl;
    *total = incl;
  }
}

// ---------------------------------------------------------------- compact
constexpr int CMP_THREADS = 256;
__global__ void __launch_bounds__(CMP_THREADS) k_compact(const uint8_t* __restrict__ scores,
                                                          int64_t n, int64_t nchunks,
                                                          const int32_t* __restrict__ lvl,
                                                          const int64_t* __restrict__ coff,
                                                          const int64_t* __restrict__ qbase,
                                                          uint32_t* __restrict__ cand) {
  __shared__ int wtot[CMP_THREADS / 32];
  const int c = blockIdx.x;
  const int64_t q = blockIdx.y;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t base = (int64_t)c << kChunkShift;
  const int valid = (int)min((int64_t)kChunk, n - base);
  const uint32_t L = (uint32_t)lvl[q];
  const uint32_t Lrep = 0x01010101u * L;
  const uint4* sc = reinterpret_cast<const uint4*>(scores + ((size_t)q * nchunks + c) * kChunk);
  uint32_t* dst = cand + qbase[q] + coff[(size_t)q * nchunks + c];
  int64_t run = 0;
  for (int r0 = 0; r0 < valid; r0 += CMP_THREADS * 16) {
    const int p0 = r0 + tid * 16;
    uint32_t mask = 0;
    if (p0 < valid) {
      const uint4 v = sc[p0 >> 4];
      const uint32_t ws[4] = {v.x, v.y, v.z, v.w};
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const uint32_t ge = __vcmpgeu4(ws[u], Lrep);
#pragma unroll
        for (int b = 0; b < 4; ++b)
          if ((ge >> (8 * b)) & 1u) mask |= 1u << (u * 4 + b);
      }
      const int lim = valid - p0;
      if (lim < 16) mask &= (1u << lim) - 1u;
    }
    const int cnt = __popc(mask);
    int v = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += x;
    }
    if (lane == 31) wtot[wid] = v;
    __syncthreads();
    int woff = 0, btot = 0;
    for (int w = 0; w < CMP_THREADS / 32; ++w) {
      if (w < wid) woff += wtot[w];
      btot += wtot[w];
    }
    int pos = (int)run + woff + v - cnt;
    while (mask) {
      const int b = __ffs(mask) - 1;
      dst[pos++] = (uint32_t)(base + p0 + b);
      mask &= mask - 1u;
    }
    run += btot;
    __syncthreads();
  }
}

// ----------------------------------------------------------------- rerank
// Flattened over every candidate of the tile.  Each warp stages 32 candidate
// rows through shared memory 64 dims at a time (16-byte coalesced loads of
// whole row segments), then lane l folds row l into the two einsum lanes
// (engine.py:272-274) reading float4s conflict-free (row stride 68 floats).
constexpr int RR_WARPS = 4;
constexpr int RR_SEG = 64;
constexpr int RR_PITCH = RR_SEG + 4;

template <bool VEC>
__global__ void __launch_bounds__(RR_WARPS * 32) k_rerank(const float* __restrict__ X, int d,
                                                          const float* __restrict__ Qf, int Q,
                                                          const int64_t* __restrict__ qbase,
                                                          const uint32_t* __restrict__ cand,
                                                          double* __restrict__ d2out) {
  __shared__ __align__(16) float rows[RR_WARPS][32][RR_PITCH];
  __shared__ uint32_t wcid[RR_WARPS][32];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int64_t M = qbase[Q];
  const int64_t i = ((int64_t)blockIdx.x * RR_WARPS + wid) * 32 + lane;
  const bool live = i < M;
  const uint32_t cid = live ? cand[i] : 0u;
  int qi = 0;
  if (live) {
    int lo = 0, hi = Q;  // largest q with qbase[q] <= i
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (qbase[mid] <= i) lo = mid; else hi = mid;
    }
    qi = lo;
  }
  wcid[wid][lane] = cid;
  __syncwarp();
  const float* qrow = Qf + (size_t)qi * d;
  double a0 = 0.0, a1 = 0.0;
  float(*R)[RR_PITCH] = rows[wid];
  for (int seg = 0; seg < d; seg += RR_SEG) {
    const int len = min(RR_SEG, d - seg);
    if (VEC) {
      const int nv = len >> 2;  // float4 per row segment
      for (int e = lane; e < 32 * (RR_SEG / 4); e += 32) {
        const int r = e / (RR_SEG / 4), v = e % (RR_SEG / 4);
        if (v < nv) {
          const float4 x = __ldg(reinterpret_cast<const float4*>(X + (size_t)wcid[wid][r] * d + seg) + v);
          *reinterpret_cast<float4*>(&R[r][v * 4]) = x;
        }
      }
    } else {
      for (int e = lane; e < 32 * RR_SEG; e += 32) {
        const int r = e / RR_SEG, v = e % RR_SEG;
        if (v < len) R[r][v] = __ldg(X + (size_t)wcid[wid][r] * d + seg + v);
      }
    }
    __syncwarp();
    const bool last = seg + RR_SEG >= d;
    const int full = last ? (len & ~7) : len;
    for (int b = 0; b < full; b += 8) {
      float xv[8];
      if (VEC) {
        const float4 u = *reinterpret_cast<const float4*>(&R[lane][b]);
        const float4 w = *reinterpret_cast<const float4*>(&R[lane][b + 4]);
        xv[0] = u.x; xv[1] = u.y; xv[2] = u.z; xv[3] = u.w;
        xv[4] = w.x; xv[5] = w.y; xv[6] = w.z; xv[7] = w.w;
      } else {
#pragma unroll
        for (int t = 0; t < 8; ++t) xv[t] = R[lane][b + t];
      }
      double p[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double e = __dsub_rn((double)xv[t], (double)qrow[seg + b + t]);
        p[t] = __dmul_rn(e, e);
      }
      a0 = __dadd_rn(p[6], a0); a1 = __dadd_rn(p[7], a1);
      a0 = __dadd_rn(p[4], a0); a1 = __dadd_rn(p[5], a1);
      a0 = __dadd_rn(p[2], a0); a1 = __dadd_rn(p[3], a1);
      a0 = __dadd_rn(p[0], a0); a1 = __dadd_rn(p[1], a1);
    }
    if (last) {
      for (int b = full; b < len; b += 2) {
        const double e0 = __dsub_rn((double)R[lane][b], (double)qrow[seg + b]);
        a0 = __dadd_rn(__dmul_rn(e0, e0), a0);
        if (b + 1 < len) {
          const double e1 = __dsub_rn((double)R[lane][b + 1], (double)qrow[seg + b + 1]);
          a1 = __dadd_rn(__dmul_rn(e1, e1), a1);
        }
      }
    }
    __syncwarp();
  }
  if (live) {
    const double v = __dadd_rn(a0, a1);
    d2out[i] = v >= 0.0 ? v : 0.0;
  }
}

// ------------------------------------------------------------------- top-k
// One CTA per query: 8-bit-digit radix select of the k-th smallest d2 (fp64
// bits are order-preserving for d2 >= 0), ordered collection (ties -> earlier
// position == lower id, since candidates are ascending ids), bitonic sort.
constexpr int TK_THREADS = 256;
constexpr int TK_MAX = 2048;

__global__ void __launch_bounds__(TK_THREADS) k_topk(const double* __restrict__ d2,
                                                      const uint32_t* __restrict__ cand,
                                                      const int64_t* __restrict__ qbase, int k,
                                                      int64_t id_base,
                                                      double* __restrict__ out_d2,
                                                      int64_t* __restrict__ out_ids) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_prefix, s_mask;
  __shared__ int s_rem;
  __shared__ unsigned long long skey[TK_MAX];
  __shared__ int spos[TK_MAX];
  __shared__ int s_nless, s_ntie, wtmp[TK_THREADS / 32][2];
  const int64_t q = blockIdx.x;
  const int64_t lo = qbase[q];
  const int64_t m = qbase[q + 1] - lo;
  const int kk = (int)min((int64_t)k, m);
  const int tid = threadIdx.x;
  const unsigned long long* keys = reinterpret_cast<const unsigned long long*>(d2 + lo);
  if (tid == 0) {
    s_prefix = 0ull;
    s_mask = 0ull;
    s_rem = kk;
    s_nless = 0;
    s_ntie = 0;
  }
  __syncthreads();
  if (kk > 0) {
    for (int pass = 0; pass < 8; ++pass) {
      const int shift = 56 - 8 * pass;
      for (int i = tid; i < 256; i += TK_THREADS) hist[i] = 0;
      __syncthreads();
      const unsigned long long pre = s_prefix, msk = s_mask;
      for (int64_t i = tid; i < m; i += TK_THREADS) {
        const unsigned long long kv = keys[i];
        if ((kv & msk) == pre) atomicAdd(&hist[(kv >> shift) & 255ull], 1u);
      }
      __syncthreads();
      if (tid == 0) {
        int rem = s_rem;
        unsigned acc = 0;
        int dg = 0;
        for (; dg < 256; ++dg) {
          if (acc + hist[dg] >= (unsigned)rem) break;
          acc += hist[dg];
        }
        s_rem = rem - (int)acc;
        s_prefix = pre | ((unsigned long long)dg << shift);
        s_mask = msk | (255ull << shift);
      }
      __syncthreads();
    }
    const unsigned long long tau = s_prefix;
    const int take_ties = s_rem;
    // ordered collection in position order
    const int lane = tid & 31, wid = tid >> 5;
    int nl_run = 0, nt_run = 0;
    for (int64_t r0 = 0; r0 < m; r0 += TK_THREADS) {
      const int64_t i = r0 + tid;
      unsigned long long kv = 0;
      int isl = 0, ist = 0;
      if (i < m) {
        kv = keys[i];
        isl = kv < tau;
        ist = kv == tau;
      }
      int vl = isl, vt = ist;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        int a = __shfl_up_sync(0xffffffffu, vl, o);
        int b = __shfl_up_sync(0xffffffffu, vt, o);
        if (lane >= o) { vl += a; vt += b; }
      }
      if (lane == 31) { wtmp[wid][0] = vl; wtmp[wid][1] = vt; }
      __syncthreads();
      int ol = 0, ot = 0, tl = 0, tt = 0;
      for (int w = 0; w < TK_THREADS / 32; ++w) {
        if (w < wid) { ol += wtmp[w][0]; ot += wtmp[w][1]; }
        tl += wtmp[w][0];
        tt += wtmp[w][1];
      }
      const int rl = nl_run + ol + vl - isl;   // rank among "less"
      const int rt = nt_run + ot + vt - ist;   // rank among ties
      if (isl) { skey[rl] = kv; spos[rl] = (int)i; }
      if (ist && rt < take_ties) {
        const int slot = (kk - take_ties) + rt;
        skey[slot] = kv;
        spos[slot] = (int)i;
      }
      nl_run += tl;
      nt_run += tt;
      __syncthreads();
    }
  }
  // bitonic sort of kk items on (key, pos), padded to a power of two
  int P = 1;
  while (P < kk) P <<= 1;
  for (int i = kk + tid; i < P; i += TK_THREADS) {
    skey[i] = ~0ull;
    spos[i] = 0x7fffffff;
  }
  __syncthreads();
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < P; i += TK_THREADS) {
        const int jx = i ^ stride;
        if (jx > i) {
          const bool up = (i & size) == 0;
          const unsigned long long ka = skey[i], kb = skey[jx];
          const int pa = spos[i], pb = spos[jx];
          const bool gt = ka > kb || (ka == kb && pa > pb);
          if (gt == up) {
            skey[i] = kb; skey[jx] = ka;
            spos[i] = pb; spos[jx] = pa;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int r = tid; r < k; r += TK_THREADS) {
    if (r < kk) {
      out_d2[q * k + r] = __longlong_as_double((long long)skey[r]);
      out_ids[q * k + r] = (int64_t)cand[lo + spos[r]] + id_base;
    } else {
      out_d2[q * k + r] = __longlong_as_double(0x7ff0000000000000LL);
      out_ids[q * k + r] = -1;
    }
  }
}

// Final outputs: ids int32 (-1 padded), dists f32(sqrt(d2)) (+inf padded).
__global__ void k_finalize(const double* __restrict__ d2, const int64_t* __restrict__ ids, int64_t total,
                           int32_t* __restrict__ out_ids, float* __restrict__ out_d) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= total) return;
  const int64_t id = ids[i];
  out_ids[i] = (int32_t)id;
  out_d[i] = id < 0 ? __int_as_float(0x7f800000) : __double2float_rn(__dsqrt_rn(d2[i]));
}

// Merge R per-rank sorted top-k lists on (d2, id) (multi-GPU finish).
__global__ void k_merge(int R, int k, int64_t nq, const double* __restrict__ d2,
                        const int64_t* __restrict__ ids, int32_t* __restrict__ out_ids,
                        float* __restrict__ out_d) {
  const int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (q >= nq) return;
  int head[16];
  for (int r = 0; r < R; ++r) head[r] = 0;
  for (int o = 0; o < k; ++o) {
    int best = -1;
    double bd = 0.0;
    int64_t bi = 0;
    for (int r = 0; r < R; ++r) {
      if (head[r] >= k) continue;
      const size_t e = ((size_t)r * nq + q) * k + head[r];
      const int64_t id = ids[e];
      if (id < 0) continue;
      const double v = d2[e];
      if (best < 0 || v < bd || (v == bd && id < bi)) { best = r; bd = v; bi = id; }
    }
    if (best < 0) {
      out_ids[q * k + o] = -1;
      out_d[q * k + o] = __int_as_float(0x7f800000);
    } else {
      out_ids[q * k + o] = (int32_t)bi;
      out_d[q * k + o] = __double2float_rn(__dsqrt_rn(bd));
      head[best]++;
    }
  }
}

// ===================================================================== host
struct TileDims {
  int Q;
  int cap;
};

static int tile_queries(const taco_index* idx) {
  // keep the Q x n score tables within ~96 MiB (L2-resident) and Q <= 1024
  const int64_t per = idx->nchunks * kChunk;
  int64_t Q = (int64_t)(96ll << 20) / per;
  const int64_t popcap = (int64_t)idx->n_sub * idx->K * 2;
  Q = std::min<int64_t>(Q, (int64_t)(256ll << 20) / std::max<int64_t>(popcap, 1));
  Q = std::max<int64_t>(16, std::min<int64_t>(Q, 1024));
  return (int)Q;
}

static int ensure_tile(taco_index* idx, int Q, int k) {
  QueryTile& t = idx->qt;
  const size_t QS = (size_t)Q * idx->n_sub;
  TACO_TRY(t.Q.ensure(sizeof(float) * (size_t)Q * idx->d));
  TACO_TRY(t.qt.ensure(sizeof(float) * (size_t)Q * idx->D));
  TACO_TRY(t.sd.ensure(sizeof(double) * QS * 2 * idx->kp));
  TACO_TRY(t.sl.ensure(sizeof(uint16_t) * QS * 2 * idx->kp));
  TACO_TRY(t.pops.ensure(sizeof(uint16_t) * QS * idx->K));
  TACO_TRY(t.npop.ensure(sizeof(int32_t) * QS));
  TACO_TRY(t.ret.ensure(sizeof(int64_t) * QS));
  TACO_TRY(t.scores.ensure((size_t)Q * idx->nchunks * kChunk));
  TACO_TRY(t.part.ensure(sizeof(int32_t) * (size_t)Q * idx->nchunks * (idx->n_sub + 1)));
  TACO_TRY(t.hist.ensure(sizeof(int64_t) * (size_t)Q * (idx->n_sub + 1)));
  TACO_TRY(t.lvl.ensure(sizeof(int32_t) * Q));
  TACO_TRY(t.cnum.ensure(sizeof(int64_t) * Q));
  TACO_TRY(t.coff.ensure(sizeof(int64_t) * (size_t)Q * idx->nchunks));
  TACO_TRY(t.qbase.ensure(sizeof(int64_t) * (Q + 1)));
  TACO_TRY(t.total.ensure(sizeof(int64_t)));
  TACO_TRY(t.tk_d2.ensure(sizeof(double) * (size_t)Q * k));
  TACO_TRY(t.tk_ids.ensure(sizeof(int64_t) * (size_t)Q * k));
  return TACO_OK;
}

static int check_query_ready(taco_index* idx, double alpha, int k) {
  TACO_TRY(index_check(idx));
  if (!idx->has_model || !idx->has_cb || !idx->has_cells || !idx->has_gsize)
    TACO_FAIL(TACO_ERR_STATE, "index is not built (model %d codebooks %d cells %d sizes %d)",
              idx->has_model, idx->has_cb, idx->has_cells, idx->has_gsize);
  if (!(alpha > 0.0 && alpha <= 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "collision ratio %g outside (0, 1]", alpha);
  if (k < 0 || k > TK_MAX) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d outside [1, %d]", k, TK_MAX);
  return TACO_OK;
}

static int64_t retrieval_target(double alpha, int64_t n) {
  const double t = std::ceil(alpha * (double)n);   // imi.py:109-112 (Python float math)
  return std::min<int64_t>(n, (int64_t)t);
}

// Stages 1-5 for one tile already resident in idx->qt.Q: leaves part + hist.
static int run_count_stage(taco_index* idx, int Q, double alpha, cudaStream_t st,
                           double* keys_out) {
  QueryTile& t = idx->qt;
  const int kp = idx->kp;
  {
    ProfScope ps(K_TRANSFORM, st);
    TACO_TRY(launch_transform(st, t.Q.as<float>(), Q, idx->d, idx->D, idx->mean.as<float>(),
                              idx->M.as<float>(), t.qt.as<float>(), false));
  }
  {
    const int64_t warps = (int64_t)Q * idx->n_sub * 2;
    const int wpb = 8;
    ProfScope ps(K_CSORT, st);
    k_csort<<<(unsigned)ceil_div(warps, wpb), wpb * 32, sizeof(double) * kp * wpb, st>>>(
        t.qt.as<float>(), Q, idx->n_sub, idx->s, idx->m1, idx->m2, kp, idx->cb1.as<float>(),
        idx->cb2.as<float>(), t.sd.as<double>(), t.sl.as<uint16_t>());
    TACO_LAUNCHED();
  }
  {
    const int64_t th = (int64_t)Q * idx->n_sub;
    const int64_t target = retrieval_target(alpha, idx->n_global);
    const unsigned g = (unsigned)ceil_div(th, 128);
    ProfScope ps(K_TRAVERSE, st);
#define TRAV(KM)                                                                              \
  k_traverse<KM><<<g, 128, 0, st>>>(t.sd.as<double>(), t.sl.as<uint16_t>(),                   \
                                    idx->gsize.as<int64_t>(), Q, idx->n_sub, kp, target,        \
                                    t.pops.as<uint16_t>(), idx->K, keys_out, t.npop.as<int32_t>(), \
                                    t.ret.as<int64_t>())
    if (kp <= 32) TRAV(32);
    else if (kp <= 64) TRAV(64);
    else if (kp <= 128) TRAV(128);
    else TRAV(256);
#undef TRAV
    TACO_LAUNCHED();
  }
  {
    const size_t smem = kChunk + sizeof(uint32_t) * (2 * CNT_PB + 1);
    static bool attr = false;
    if (!attr) {
      TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      attr = true;
    }
    dim3 g((unsigned)idx->nchunks, (unsigned)Q);
    ProfScope ps(K_COUNT, st);
    k_count<<<g, CNT_THREADS, smem, st>>>(t.pops.as<uint16_t>(), t.npop.as<int32_t>(), idx->K,
                                          idx->ids.as<uint32_t>(), idx->offs.as<uint32_t>(),
                                          idx->n_sub, idx->K, idx->n, idx->nchunks,
                                          t.scores.as<uint8_t>(), t.part.as<int32_t>());
    TACO_LAUNCHED();
  }
  {
    ProfScope ps(K_HIST, st);
    k_hist_reduce<<<Q, 64, 0, st>>>(t.part.as<int32_t>(), idx->nchunks, idx->n_sub,
                                    t.hist.as<int64_t>());
    TACO_LAUNCHED();
  }
  return TACO_OK;
}

// Stages 6-9: select on `ghist`, compact, rerank, top-k into t.tk_d2/tk_ids.
static int run_finish_stage(taco_index* idx, int Q, const int64_t* ghist, double beta, int k,
                            cudaStream_t st) {
  QueryTile& t = idx->qt;
  const double budget = beta * (double)idx->n_global;   // engine.py:240
  {
    ProfScope ps_sel(K_SELECT, st);
    k_select<<<1, 1024, 0, st>>>(ghist, t.part.as<int32_t>(), Q, idx->nchunks, idx->n_sub, budget,
                                 t.lvl.as<int32_t>(), t.cnum.as<int64_t>(), t.coff.as<int64_t>(),
                                 t.qbase.as<int64_t>(), t.total.as<int64_t>());
    TACO_LAUNCHED();
  }
  int64_t total = 0;
  TACO_CHECK_CUDA(cudaMemcpyAsync(&total, t.total.p, sizeof(int64_t), cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  if (g_prof.on) {
    std::vector<int64_t> r((size_t)Q * idx->n_sub);
    std::vector<int32_t> np((size_t)Q * idx->n_sub);
    cudaMemcpy(r.data(), t.ret.p, 8 * r.size(), cudaMemcpyDeviceToHost);
    cudaMemcpy(np.data(), t.npop.p, 4 * np.size(), cudaMemcpyDeviceToHost);
    for (auto v : r) g_prof.sumR += v;
    for (auto v : np) g_prof.sumPops += v;
    g_prof.sumC += total;
    g_prof.queries += Q;
    g_prof.tiles += 1;
    g_prof.bytes_scores += (int64_t)Q * idx->nchunks * kChunk;
  }
  TACO_TRY(t.cand.ensure(sizeof(uint32_t) * (size_t)std::max<int64_t>(total, 1)));
  TACO_TRY(t.d2.ensure(sizeof(double) * (size_t)std::max<int64_t>(total, 1)));
  {
    dim3 g((unsigned)idx->nchunks, (unsigned)Q);
    ProfScope ps(K_COMPACT, st);
    k_compact<<<g, CMP_THREADS, 0, st>>>(t.scores.as<uint8_t>(), idx->n, idx->nchunks,
                                         t.lvl.as<int32_t>(), t.coff.as<int64_t>(),
                                         t.qbase.as<int64_t>(), t.cand.as<uint32_t>());
    TACO_LAUNCHED();
  }
  if (total > 0) {
    const unsigned g = (unsigned)ceil_div(total, RR_WARPS * 32);
    ProfScope ps(K_RERANK, st);
    if (idx->d % 4 == 0)
      k_rerank<true><<<g, RR_WARPS * 32, 0, st>>>(idx->X.as<float>(), idx->d, t.Q.as<float>(), Q,
                                                  t.qbase.as<int64_t>(), t.cand.as<uint32_t>(),
                                                  t.d2.as<double>());
    else
      k_rerank<false><<<g, RR_WARPS * 32, 0, st>>>(idx->X.as<float>(), idx->d, t.Q.as<float>(), Q,
                                                   t.qbase.as<int64_t>(), t.cand.as<uint32_t>(),
                                                   t.d2.as<double>());
    TACO_LAUNCHED();
  }
  if (k > 0) {
    ProfScope ps(K_TOPK, st);
    k_topk<<<Q, TK_THREADS, 0, st>>>(t.d2.as<double>(), t.cand.as<uint32_t>(), t.qbase.as<int64_t>(),
                                     k, idx->id_base, t.tk_d2.as<double>(), t.tk_ids.as<int64_t>());
    TACO_LAUNCHED();
  }
  return TACO_OK;
}

static int query_batch_impl(taco_index* idx, const float* Q_src, bool src_host, int64_t nq,
                            double alpha, double beta, int k, int32_t* ids_o, float* dists_o,
                            int64_t* cnum_o, int32_t* lvl_o, bool dst_host, cudaStream_t st) {
  TACO_TRY(check_query_ready(idx, alpha, k));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "base vectors are not resident");
  if (!(beta > 0.0 && beta < 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "re-rank ratio %g outside (0, 1)", beta);
  if (k < 1) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d is below 1", k);
  if (nq == 0) return TACO_OK;
  const int Qt = tile_queries(idx);
  TACO_TRY(ensure_tile(idx, Qt, k));
  QueryTile& t = idx->qt;
  TACO_TRY(t.out_ids.ensure(sizeof(int32_t) * (size_t)Qt * k));
  TACO_TRY(t.out_d.ensure(sizeof(float) * (size_t)Qt * k));
  for (int64_t q0 = 0; q0 < nq; q0 += Qt) {
    const int Q = (int)std::min<int64_t>(Qt, nq - q0);
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, Q_src + (size_t)q0 * idx->d, sizeof(float) * (size_t)Q * idx->d,
                                    src_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice, st));
    TACO_TRY(run_count_stage(idx, Q, alpha, st, nullptr));
    TACO_TRY(run_finish_stage(idx, Q, t.hist.as<int64_t>(), beta, k, st));
    const int64_t tot = (int64_t)Q * k;
    ProfScope ps(K_FINAL, st);
    k_finalize<<<(unsigned)ceil_div(tot, 256), 256, 0, st>>>(t.tk_d2.as<double>(), t.tk_ids.as<int64_t>(),
                                                             tot, t.out_ids.as<int32_t>(), t.out_d.as<float>());
    TACO_LAUNCHED();
    const cudaMemcpyKind kind = dst_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
    TACO_CHECK_CUDA(cudaMemcpyAsync(ids_o + q0 * k, t.out_ids.p, sizeof(int32_t) * tot, kind, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(dists_o + q0 * k, t.out_d.p, sizeof(float) * tot, kind, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(cnum_o + q0, t.cnum.p, sizeof(int64_t) * Q, kind, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(lvl_o + q0, t.lvl.p, sizeof(int32_t) * Q, kind, st));
  }
  if (dst_host) TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  return TACO_OK;
}

}  // namespace taco

using namespace taco;

extern "C" {

int taco_query_batch(taco_index* idx, const float* Q_h, int64_t nq, double alpha, double beta,
                     int32_t k, int32_t* ids_h, float* dists_h, int64_t* cand_num_h,
                     int32_t* last_coll_h) {
  if (!idx) TACO_FAIL(TACO_ERR_STATE, "null index handle");
  return query_batch_impl(idx, Q_h, true, nq, alpha, beta, k, ids_h, dists_h, cand_num_h,
                          last_coll_h, true, idx->stream);
}

int taco_query_batch_device(taco_index* idx, const float* Q_d, int64_t nq, double alpha,
                            double beta, int32_t k, int32_t* ids_d, float* dists_d,
                            int64_t* cand_num_d, int32_t* last_coll_d, void* stream) {
  if (!idx) TACO_FAIL(TACO_ERR_STATE, "null index handle");
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  return query_batch_impl(idx, Q_d, false, nq, alpha, beta, k, ids_d, dists_d, cand_num_d,
                          last_coll_d, false, st);
}

int taco_query_count_device(taco_index* idx, const float* Q_d, int64_t nq, double alpha,
                            int64_t* hist_d, void* stream) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  const int Qt = tile_queries(idx);
  if (nq > Qt) TACO_FAIL(TACO_ERR_PARAMETER, "split query batch %lld exceeds tile %d", (long long)nq, Qt);
  TACO_TRY(ensure_tile(idx, Qt, 1));
  QueryTile& t = idx->qt;
  TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, Q_d, sizeof(float) * (size_t)nq * idx->d,
                                  cudaMemcpyDeviceToDevice, st));
  TACO_TRY(run_count_stage(idx, (int)nq, alpha, st, nullptr));
  TACO_CHECK_CUDA(cudaMemcpyAsync(hist_d, t.hist.p, sizeof(int64_t) * (size_t)nq * (idx->n_sub + 1),
                                  cudaMemcpyDeviceToDevice, st));
  return TACO_OK;
}

int taco_query_finish_device(taco_index* idx, int64_t nq, const int64_t* ghist_d, double beta,
                               int32_t k, double* topk_d2_d, int64_t* topk_ids_d,
                               int64_t* cand_num_d, int32_t* last_coll_d, void* stream) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "base vectors are not resident");
  if (!(beta > 0.0 && beta < 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "re-rank ratio %g outside (0, 1)", beta);
  if (k < 1 || k > TK_MAX) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d outside [1, %d]", k, TK_MAX);
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  const int Qt = tile_queries(idx);
  if (nq > Qt) TACO_FAIL(TACO_ERR_PARAMETER, "split query batch %lld exceeds tile %d", (long long)nq, Qt);
  TACO_TRY(ensure_tile(idx, Qt, k));
  QueryTile& t = idx->qt;
  TACO_TRY(run_finish_stage(idx, (int)nq, ghist_d, beta, k, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(topk_d2_d, t.tk_d2.p, sizeof(double) * (size_t)nq * k, cudaMemcpyDeviceToDevice, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(topk_ids_d, t.tk_ids.p, sizeof(int64_t) * (size_t)nq * k, cudaMemcpyDeviceToDevice, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(cand_num_d, t.cnum.p, sizeof(int64_t) * nq, cudaMemcpyDeviceToDevice, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(last_coll_d, t.lvl.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToDevice, st));
  return TACO_OK;
}

int taco_query_tile_size(taco_index* idx) {
  if (!idx) return 0;
  return tile_queries(idx);
}

int taco_topk_merge_device(int32_t ranks, int64_t nq, int32_t k, const double* d2_d,
                           const int64_t* ids_d, int32_t* ids_out_d, float* dists_out_d,
                           void* stream) {
  if (ranks < 1 || ranks > 16) TACO_FAIL(TACO_ERR_PARAMETER, "rank count %d outside [1, 16]", ranks);
  if (nq == 0) return TACO_OK;
  k_merge<<<(unsigned)ceil_div(nq, 128), 128, 0, (cudaStream_t)stream>>>(ranks, k, nq, d2_d, ids_d,
                                                                        ids_out_d, dists_out_d);
  TACO_LAUNCHED();
  return TACO_OK;
}

// ------------------------------------------------------------ debug taps
int taco_count_scores(taco_index* idx, const float* q_h, double alpha, uint8_t* scores_h) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  const int Qt = tile_queries(idx);
  TACO_TRY(ensure_tile(idx, Qt, 1));
  QueryTile& t = idx->qt;
  cudaStream_t st = idx->stream;
  TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, q_h, sizeof(float) * idx->d, cudaMemcpyHostToDevice, st));
  TACO_TRY(run_count_stage(idx, 1, alpha, st, nullptr));
  TACO_CHECK_CUDA(cudaMemcpyAsync(scores_h, t.scores.p, idx->n, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  return TACO_OK;
}

int taco_activation_trace(taco_index* idx, const float* q_h, int32_t j, double alpha, int32_t cap,
                          int32_t* pops_h, double* keys_h, int32_t* npop_h, int64_t* retrieved_h) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  if (j < 0 || j >= idx->n_sub) TACO_FAIL(TACO_ERR_PARAMETER, "subspace %d out of range", j);
  const int Qt = tile_queries(idx);
  TACO_TRY(ensure_tile(idx, Qt, 1));
  QueryTile& t = idx->qt;
  cudaStream_t st = idx->stream;
  DevBuf keys;
  TACO_TRY(keys.ensure(sizeof(double) * (size_t)idx->n_sub * idx->K));
  TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, q_h, sizeof(float) * idx->d, cudaMemcpyHostToDevice, st));
  int rc = run_count_stage(idx, 1, alpha, st, keys.as<double>());
  if (rc != TACO_OK) { keys.release(); return rc; }
  int32_t np = 0;
  int64_t got = 0;
  std::vector<uint16_t> p16(idx->K);
  cudaMemcpyAsync(&np, t.npop.as<int32_t>() + j, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&got, t.ret.as<int64_t>() + j, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(p16.data(), t.pops.as<uint16_t>() + (size_t)j * idx->K, sizeof(uint16_t) * idx->K,
                  cudaMemcpyDeviceToHost, st);
  std::vector<double> kv(idx->K);
  cudaMemcpyAsync(kv.data(), keys.as<double>() + (size_t)j * idx->K, sizeof(double) * idx->K,
                  cudaMemcpyDeviceToHost, st);
  cudaError_t e = cudaStreamSynchronize(st);
  keys.release();
  if (e != cudaSuccess) TACO_FAIL(TACO_ERR_CUDA, "%s", cudaGetErrorString(e));
  for (int i = 0; i < np && i < cap; ++i) {
    pops_h[i] = p16[i];
    keys_h[i] = kv[i];
  }
  *npop_h = np;
  *retrieved_h = got;
  return TACO_OK;
}

int taco_select_candidates(int device, const uint8_t* scores_h, int64_t n, int32_t n_sub,
                           double beta, int64_t* ids_h, int64_t* cand_num_h, int32_t* last_coll_h) {
  TACO_TRY(with_device(device));
  if (n_sub < 0 || n_sub > 255) TACO_FAIL(TACO_ERR_PARAMETER, "subspace count %d outside [0, 255]", n_sub);
  if (n < 1) TACO_FAIL(TACO_ERR_PARAMETER, "empty score table");
  const int64_t nc = ceil_div(n, kChunk);
  DevBuf sc, part, hist, lvl, cnum, coff, qbase, total, cand;
  auto cleanup = [&]() {
    sc.release(); part.release(); hist.release(); lvl.release(); cnum.release(); coff.release();
    qbase.release(); total.release(); cand.release();
  };
  int rc = TACO_OK;
  do {
    if ((rc = sc.ensure(nc * kChunk)) != TACO_OK) break;
    if ((rc = part.ensure(sizeof(int32_t) * nc * (n_sub + 1))) != TACO_OK) break;
    if ((rc = hist.ensure(sizeof(int64_t) * (n_sub + 1))) != TACO_OK) break;
    if ((rc = lvl.ensure(4)) || (rc = cnum.ensure(8)) || (rc = coff.ensure(8 * nc)) ||
        (rc = qbase.ensure(16)) || (rc = total.ensure(8)) || (rc = cand.ensure(4 * n)))
      break;
    cudaMemset(sc.p, 0, nc * kChunk);
    cudaMemcpy(sc.p, scores_h, n, cudaMemcpyHostToDevice);
    // scores above n_sub would index past the histogram: reject like bincount would overflow minlength
    k_chunk_hist<<<dim3((unsigned)nc, 1), 256>>>(sc.as<uint8_t>(), n, nc, n_sub, part.as<int32_t>());
    count_launch();
    k_hist_reduce<<<1, 64>>>(part.as<int32_t>(), nc, n_sub, hist.as<int64_t>());
    count_launch();
    k_select<<<1, 1024>>>(hist.as<int64_t>(), part.as<int32_t>(), 1, nc, n_sub, beta * (double)n,
                          lvl.as<int32_t>(), cnum.as<int64_t>(), coff.as<int64_t>(),
                          qbase.as<int64_t>(), total.as<int64_t>());
    count_launch();
    k_compact<<<dim3((unsigned)nc, 1), CMP_THREADS>>>(sc.as<uint8_t>(), n, nc, lvl.as<int32_t>(),
                                                      coff.as<int64_t>(), qbase.as<int64_t>(),
                                                      cand.as<uint32_t>());
    count_launch();
    int64_t tot = 0;
    int32_t L = 0;
    cudaMemcpy(&tot, total.p, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&L, lvl.p, 4, cudaMemcpyDeviceToHost);
    int64_t cn = 0;
    cudaMemcpy(&cn, cnum.p, 8, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> ids(tot);
    cudaMemcpy(ids.data(), cand.p, 4 * tot, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    for (int64_t i = 0; i < tot; ++i) ids_h[i] = ids[i];
    *cand_num_h = cn;
    *last_coll_h = L;
    if (tot != cn) { set_error("candidate count %lld != histogram count %lld", (long long)tot, (long long)cn); rc = TACO_ERR_NUMERIC; }
  } while (0);
  cleanup();
  return rc;
}

int taco_rerank(int device, const float* X_h, int64_t n, int32_t d, const float* q_h,
                const int64_t* ids_h, int64_t m, int32_t k, int32_t* ids_out_h, float* dists_out_h,
                double* d2_out_h) {
  TACO_TRY(with_device(device));
  if (k < 1 || k > TK_MAX) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d outside [1, %d]", k, TK_MAX);
  if (m < 0) TACO_FAIL(TACO_ERR_PARAMETER, "negative candidate count");
  if (m == 0) return TACO_OK;
  for (int64_t i = 0; i < m; ++i)
    if (ids_h[i] < 0 || ids_h[i] >= n || ids_h[i] > 0xFFFFFFFFll)
      TACO_FAIL(TACO_ERR_PARAMETER, "candidate id %lld out of range", (long long)ids_h[i]);
  // candidates must be processed in ascending-id order for the position tie-break
  std::vector<uint32_t> c32(m);
  bool sorted = true;
  for (int64_t i = 0; i < m; ++i) {
    c32[i] = (uint32_t)ids_h[i];
    if (i && c32[i] < c32[i - 1]) sorted = false;
  }
  if (!sorted) std::sort(c32.begin(), c32.end());
  // gather the candidate rows on the host into a compact matrix (X may be huge)
  std::vector<float> rowsv((size_t)m * d);
  for (int64_t i = 0; i < m; ++i)
    std::copy(X_h + (size_t)c32[i] * d, X_h + (size_t)c32[i] * d + d, rowsv.begin() + (size_t)i * d);
  DevBuf Xd, Qd, qb, cd, d2, tkd, tki, oi, od;
  int rc = TACO_OK;
  do {
    if ((rc = Xd.ensure(sizeof(float) * rowsv.size())) || (rc = Qd.ensure(sizeof(float) * d)) ||
        (rc = qb.ensure(16)) || (rc = cd.ensure(4 * m)) || (rc = d2.ensure(8 * m)) ||
        (rc = tkd.ensure(8 * k)) || (rc = tki.ensure(8 * k)))
      break;
    std::vector<uint32_t> local(m);
    for (int64_t i = 0; i < m; ++i) local[i] = (uint32_t)i;
    int64_t qbh[2] = {0, m};
    cudaMemcpy(Xd.p, rowsv.data(), sizeof(float) * rowsv.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(Qd.p, q_h, sizeof(float) * d, cudaMemcpyHostToDevice);
    cudaMemcpy(qb.p, qbh, 16, cudaMemcpyHostToDevice);
    cudaMemcpy(cd.p, local.data(), 4 * m, cudaMemcpyHostToDevice);
    const unsigned g = (unsigned)ceil_div(m, RR_WARPS * 32);
    if (d % 4 == 0)
      k_rerank<true><<<g, RR_WARPS * 32>>>(Xd.as<float>(), d, Qd.as<float>(), 1, qb.as<int64_t>(),
                                           cd.as<uint32_t>(), d2.as<double>());
    else
      k_rerank<false><<<g, RR_WARPS * 32>>>(Xd.as<float>(), d, Qd.as<float>(), 1, qb.as<int64_t>(),
                                            cd.as<uint32_t>(), d2.as<double>());
    count_launch();
    k_topk<<<1, TK_THREADS>>>(d2.as<double>(), cd.as<uint32_t>(), qb.as<int64_t>(), k, 0,
                              tkd.as<double>(), tki.as<int64_t>());
    count_launch();
    std::vector<double> td(k);
    std::vector<int64_t> ti(k);
    cudaMemcpy(td.data(), tkd.p, 8 * k, cudaMemcpyDeviceToHost);
    cudaMemcpy(ti.data(), tki.p, 8 * k, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    const int kk = (int)std::min<int64_t>(k, m);
    for (int r = 0; r < kk; ++r) {
      ids_out_h[r] = (int32_t)c32[ti[r]];
      d2_out_h[r] = td[r];
      dists_out_h[r] = (float)std::sqrt(td[r]);
    }
  } while (0);
  Xd.release(); Qd.release(); qb.release(); cd.release(); d2.release(); tkd.release(); tki.release();
  return rc;
}

int taco_transform_points(int device, const float* mean_h, const float* matrix_h, int32_t d,
                          int32_t D, const float* P_h, int64_t np_, float* out_h) {
  TACO_TRY(with_device(device));
  if (np_ == 0) return TACO_OK;
  DevBuf mu, M, P, O;
  int rc = TACO_OK;
  do {
    if ((rc = mu.ensure(4 * d)) || (rc = M.ensure(4 * (size_t)d * D)) || (rc = P.ensure(4 * (size_t)np_ * d)) ||
        (rc = O.ensure(4 * (size_t)np_ * D)))
      break;
    cudaMemcpy(mu.p, mean_h, 4 * d, cudaMemcpyHostToDevice);
    cudaMemcpy(M.p, matrix_h, 4 * (size_t)d * D, cudaMemcpyHostToDevice);
    cudaMemcpy(P.p, P_h, 4 * (size_t)np_ * d, cudaMemcpyHostToDevice);
    if ((rc = launch_transform(0, P.as<float>(), np_, d, D, mu.as<float>(), M.as<float>(), O.as<float>(), false)))
      break;
    cudaError_t e = cudaMemcpy(out_h, O.p, 4 * (size_t)np_ * D, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; }
  } while (0);
  mu.release(); M.release(); P.release(); O.release();
  return rc;
}

int taco_centroid_order(int device, const float* c1_h, const float* c2_h, int32_t kp, int32_t m1,
                        int32_t m2, const float* q_h, double* d1s_h, int32_t* l1s_h, double* d2s_h,
                        int32_t* l2s_h) {
  TACO_TRY(with_device(device));
  if (kp < 1 || kp > 65535) TACO_FAIL(TACO_ERR_PARAMETER, "codebook size %d out of range", kp);
  DevBuf c1, c2, q, sd, sl;
  int rc = TACO_OK;
  do {
    if ((rc = c1.ensure(4 * (size_t)kp * std::max(m1, 1))) || (rc = c2.ensure(4 * (size_t)kp * std::max(m2, 1))) ||
        (rc = q.ensure(4 * (size_t)(m1 + m2))) || (rc = sd.ensure(8 * 2 * (size_t)kp)) ||
        (rc = sl.ensure(2 * 2 * (size_t)kp)))
      break;
    cudaMemcpy(c1.p, c1_h, 4 * (size_t)kp * m1, cudaMemcpyHostToDevice);
    if (m2 > 0) cudaMemcpy(c2.p, c2_h, 4 * (size_t)kp * m2, cudaMemcpyHostToDevice);
    cudaMemcpy(q.p, q_h, 4 * (size_t)(m1 + m2), cudaMemcpyHostToDevice);
    k_csort<<<1, 64, sizeof(double) * kp * 2>>>(q.as<float>(), 1, 1, m1 + m2, m1, m2, kp, c1.as<float>(),
                                                c2.as<float>(), sd.as<double>(), sl.as<uint16_t>());
    count_launch();
    std::vector<uint16_t> l(2 * kp);
    cudaMemcpy(d1s_h, sd.p, 8 * (size_t)kp, cudaMemcpyDeviceToHost);
    cudaMemcpy(d2s_h, sd.as<double>() + kp, 8 * (size_t)kp, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(l.data(), sl.p, 2 * 2 * (size_t)kp, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    for (int i = 0; i < kp; ++i) { l1s_h[i] = l[i]; l2s_h[i] = l[kp + i]; }
  } while (0);
  c1.release(); c2.release(); q.release(); sd.release(); sl.release();
  return rc;
}

int taco_traverse(int device, int32_t kp, const double* d1s_h, const int32_t* l1s_h,
                  const double* d2s_h, const int32_t* l2s_h, const int64_t* sizes_h, int64_t target,
                  int32_t* pops_h, double* keys_h, int32_t* npop_h, int64_t* retrieved_h) {
  TACO_TRY(with_device(device));
  if (kp < 1 || kp > 256) TACO_FAIL(TACO_ERR_PARAMETER, "codebook size %d out of range", kp);
  const int K2 = kp * kp;
  DevBuf sd, sl, gs, pops, keys, np, ret;
  int rc = TACO_OK;
  do {
    if ((rc = sd.ensure(16 * (size_t)kp)) || (rc = sl.ensure(4 * (size_t)kp)) || (rc = gs.ensure(8 * (size_t)K2)) ||
        (rc = pops.ensure(2 * (size_t)K2)) || (rc = keys.ensure(8 * (size_t)K2)) || (rc = np.ensure(4)) ||
        (rc = ret.ensure(8)))
      break;
    std::vector<uint16_t> l(2 * kp);
    for (int i = 0; i < kp; ++i) { l[i] = (uint16_t)l1s_h[i]; l[kp + i] = (uint16_t)l2s_h[i]; }
    cudaMemcpy(sd.p, d1s_h, 8 * (size_t)kp, cudaMemcpyHostToDevice);
    cudaMemcpy(sd.as<double>() + kp, d2s_h, 8 * (size_t)kp, cudaMemcpyHostToDevice);
    cudaMemcpy(sl.p, l.data(), 4 * (size_t)kp, cudaMemcpyHostToDevice);
    cudaMemcpy(gs.p, sizes_h, 8 * (size_t)K2, cudaMemcpyHostToDevice);
#define TRAV1(KM) k_traverse<KM><<<1, 128>>>(sd.as<double>(), sl.as<uint16_t>(), gs.as<int64_t>(), 1, 1, kp, \
                                            target, pops.as<uint16_t>(), K2, keys.as<double>(),        \
                                            np.as<int32_t>(), ret.as<int64_t>())
    if (kp <= 32) TRAV1(32);
    else if (kp <= 64) TRAV1(64);
    else if (kp <= 128) TRAV1(128);
    else TRAV1(256);
#undef TRAV1
    count_launch();
    int32_t n = 0;
    cudaMemcpy(&n, np.p, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(retrieved_h, ret.p, 8, cudaMemcpyDeviceToHost);
    std::vector<uint16_t> p16(K2);
    cudaMemcpy(p16.data(), pops.p, 2 * (size_t)K2, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaMemcpy(keys_h, keys.p, 8 * (size_t)n, cudaMemcpyDeviceToHost);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    for (int i = 0; i < n; ++i) pops_h[i] = p16[i];
    *npop_h = n;
  } while (0);
  sd.release(); sl.release(); gs.release(); pops.release(); keys.release(); np.release(); ret.release();
  return rc;
}

int taco_profile_enable(int on) {
  taco::prof_drain();
  taco::g_prof.on = on != 0;
  return TACO_OK;
}

// ms_out/cnt_out[K_NKIDS]; names via taco_profile_name; stats_out[6] =
// {sum retrieved ids, sum candidates, sum pops, queries, tiles, score-table bytes}
int taco_profile_read(double* ms_out, int64_t* cnt_out, int64_t* stats_out, int reset) {
  taco::prof_drain();
  for (int i = 0; i < taco::K_NKIDS; ++i) { ms_out[i] = taco::g_prof.ms[i]; cnt_out[i] = taco::g_prof.cnt[i]; }
  stats_out[0] = taco::g_prof.sumR; stats_out[1] = taco::g_prof.sumC; stats_out[2] = taco::g_prof.sumPops;
  stats_out[3] = taco::g_prof.queries; stats_out[4] = taco::g_prof.tiles; stats_out[5] = taco::g_prof.bytes_scores;
  if (reset) {
    for (int i = 0; i < taco::K_NKIDS; ++i) { taco::g_prof.ms[i] = 0; taco::g_prof.cnt[i] = 0; }
    taco::g_prof.sumR = taco::g_prof.sumC = taco::g_prof.sumPops = 0;
    taco::g_prof.queries = taco::g_prof.tiles = taco::g_prof.bytes_scores = 0;
  }
  return TACO_OK;
}

const char* taco_profile_name(int i) { return (i >= 0 && i < taco::K_NKIDS) ? taco::kKNames[i] : ""; }
int taco_profile_kernels(void) { return taco::K_NKIDS; }
void* taco_index_stream(taco_index* idx) { return idx ? (void*)idx->stream : nullptr; }

}  // extern "C"
