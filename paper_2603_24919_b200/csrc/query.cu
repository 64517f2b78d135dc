// Batched TaCo query path on sm_100a.
//
// Whole-batch stages (super-tiles of up to kSuperTile queries), one stream:
//   k_transform       qt = f32((q - mu) @ M)                     spectral.py:301-316
//   k_csort           fp64 centroid distances + stable rank       imi.py:88-106
//   k_traverse_pl     multi-sequence heap traversal, a thread per (query,
//                     subspace) walk, persistent lanes on a 4-ary
//                     shared-memory heap (k_traverse_sh / k_traverse for
//                     smaller batches)                            imi.py:130-166
//   cluster mode (single GPU, n <= 1.5M):
//   k_count_pg        persistent SOFTWARE groups of nchunks CTAs walk the
//                     queries; each CTA counts one id chunk into a 4-bit (8-bit
//                     at N_s = 16) shared-memory table from the encoded,
//                     unit-padded CSR, the group exchanges level histograms
//                     through global slots, Alg. 5 runs in every CTA and each
//                     compacts its candidates straight from shared memory
//                     (k_count_enc: the same as one hardware cluster per query;
//                     k_count_cluster: the round-1 kernel on the plain CSR,
//                     N_s > 16)                                   engine.py:201-251
//   global mode (large shards / multi-GPU, query tiles):
//   k_count_genc      per (query, id chunk) shared-memory counting -> per-chunk
//                     histograms + spilled score >= 2 records (k_count: the
//                     plain-CSR sweep);  k_hist_reduce -> (all-reduce across
//                     ranks) -> k_select (Alg. 5) -> k_emit_rec / recount
//   k_plan_*          32-candidate tiles per candidate segment (query-major
//                     output slots, chunk-major processing order)
//   k_rerank_i8       u8 rows + u8-exact queries: warp-private cp.async (LDGSTS)
//                     row pipelines, exact DP4A integer distances, running
//                     bound, per-tile partial top-k
//   k_rerank_async    other rows / queries: the same pipeline with fp64
//                     einsum-order distances                      engine.py:256-279
//   k_topk            final per-query top-k over the tile partials (radix select
//                     on d2 bits then id, bitonic sort on (d2, id))  engine.py:275-279
//   k_finalize        ids int32 / dists f32(sqrt(d2))              engine.py:276-279
#include <cooperative_groups.h>

#include <algorithm>
#include <cstring>
#include <cmath>
#include <type_traits>
#include <vector>

#include "index.cuh"

namespace cg = cooperative_groups;

namespace taco {

// ------------------------------------------------------------- profiler
// Optional per-kernel timing with CUDA events recorded on the launching
// stream (bench.py's roofline), plus algorithmic-work counters.
enum KId { K_TRANSFORM, K_CSORT, K_TRAVERSE, K_COUNT, K_HIST, K_SELECT, K_COMPACT, K_PLAN, K_RERANK,
           K_TOPK, K_FINAL, K_NKIDS };
static const char* kKNames[K_NKIDS] = {"k_transform", "k_csort", "k_traverse", "k_count", "k_hist_reduce",
                                       "k_select", "k_compact", "k_rr_plan", "k_rerank", "k_topk",
                                       "k_finalize"};
struct Prof {
  bool on = false;
  std::vector<cudaEvent_t> pool;
  struct P { int kid; cudaEvent_t a, b; };
  std::vector<P> pend;
  double ms[K_NKIDS] = {};
  int64_t cnt[K_NKIDS] = {};
  int64_t sumR = 0, sumC = 0, sumPops = 0, queries = 0, tiles = 0, bytes_scores = 0, maxPops = 0;
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
// shard derives the same popped set.  At most `cap` cells are
// stored; a longer traversal raises flags[0] and the host re-runs with cap=K'^2.
template <int KMAX>
__global__ void __launch_bounds__(128) k_traverse(const double* __restrict__ sd,
                                                  const uint16_t* __restrict__ sl,
                                                  const int64_t* __restrict__ gsize, int64_t Q,
                                                  int n_sub, int kp, int64_t target,
                                                  uint16_t* __restrict__ pops, int cap,
                                                  double* __restrict__ keys_out,
                                                  int32_t* __restrict__ npop,
                                                  int64_t* __restrict__ ret,
                                                  int64_t* __restrict__ flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Q * n_sub) return;
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
  // Software-pipelined: the top's successor distances and labels are loaded
  // before the pop's sift-down (which hides their latency), and a popped
  // cell's size is loaded when it is popped but added one pop later, so no
  // pop waits on the size load.  The pop made after the target was reached
  // is dropped (np does not count it): same pops, counts and sizes as the
  // reference loop.
  int64_t psz = 0;        // size of the last counted pop, not yet added
  bool pend = false;
  const double d20 = d2[0];
  while (true) {
    if (hn == 0) {
      if (pend) got += psz;
      break;
    }
    const double key = hk[0];
    const uint32_t pc = hp[0];
    const int r = (int)(pc >> 16), c = (int)(pc & 0xFFFF);
    const bool nr = c == 0 && r + 1 < kp, nc = c + 1 < kp;
    const double dr1 = nr ? d1[r + 1] : 0.0;
    const double dr = d1[r];
    const double dc1 = nc ? d2[c + 1] : 0.0;
    const int cell = (int)l1[r] * kp + (int)l2[c];
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
    if (np < cap) {
      out[np] = (uint16_t)cell;
      if (kout) kout[np] = key;
    }
    if (pend) {
      got += psz;
      if (got >= target) break;   // the previous pop reached the target: this one is not counted
    }
    psz = gs[cell];
    pend = true;
    ++np;
    if (nr) push(__dadd_rn(dr1, d20), (uint32_t)(r + 1) << 16);
    if (nc) push(__dadd_rn(dr, dc1), ((uint32_t)r << 16) | (uint32_t)(c + 1));
  }
  npop[t] = np;
  ret[t] = got;
  if (np > cap) atomicMax((unsigned long long*)&flags[0], (unsigned long long)np);
}

// Same walk with the heap in shared memory (TS_THREADS walks per CTA, the
// heap of walk x interleaved across threads): the thread-local heaps of
// k_traverse (768 B per walk at K' = 64, ~415 KB per SM) do not fit L1 and
// every sift step went to L2.  The walks' sorted distances and labels are
// read through L1.
template <int KMAX, int TS_THREADS>
__global__ void __launch_bounds__(TS_THREADS) k_traverse_sh(const double* __restrict__ sd,
                                                  const uint16_t* __restrict__ sl,
                                                  const int64_t* __restrict__ gsize, int64_t Q,
                                                  int n_sub, int kp, int64_t target,
                                                  uint16_t* __restrict__ pops, int cap,
                                                  double* __restrict__ keys_out,
                                                  int32_t* __restrict__ npop,
                                                  int64_t* __restrict__ ret,
                                                  int64_t* __restrict__ flags) {
  const int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= Q * n_sub) return;
  const int j = (int)(t % n_sub);
  const double* d1 = sd + t * 2 * kp;
  const double* d2 = d1 + kp;
  const uint16_t* l1 = sl + t * 2 * kp;
  const uint16_t* l2 = l1 + kp;
  const int64_t* gs = gsize + (size_t)j * kp * kp;
  // the heap lives in shared memory, element i of thread x at [i * TS_THREADS + x]
  extern __shared__ __align__(16) unsigned char tsh_sm[];
  double* const hkb = reinterpret_cast<double*>(tsh_sm) + threadIdx.x;
  // (row, col) as r << 8 | c (K' <= 256): the same (r, c) order as the heap's pc
  uint16_t* const hpb = reinterpret_cast<uint16_t*>(reinterpret_cast<double*>(tsh_sm) + KMAX * TS_THREADS) + threadIdx.x;
  struct HeapRef {
    double* k;
    uint16_t* p;
    __device__ double& key(int i) const { return k[i * TS_THREADS]; }
    __device__ uint16_t& pc(int i) const { return p[i * TS_THREADS]; }
  };
  const HeapRef H{hkb, hpb};
#define hk(i) H.key(i)
#define hp(i) H.pc(i)
  int hn = 0;
  auto less = [&](double ka, uint32_t pa, double kb, uint32_t pb) {
    return ka < kb || (ka == kb && pa < pb);
  };
  // Fixed-depth, predicated sift-up / sift-down (TS_BF): every lane runs
  // the same log2(KMAX) steps, so the 32 walks of a warp never diverge.
  constexpr int LOGK = KMAX <= 32 ? 5 : KMAX <= 64 ? 6 : KMAX <= 128 ? 7 : 8;
  auto push = [&](double key, uint32_t pc32, bool doit) {
    const uint16_t pc = (uint16_t)pc32;
    int i = hn;
    hn += doit ? 1 : 0;
    bool done = !doit || i == 0;
#pragma unroll
    for (int lev = 0; lev < LOGK; ++lev) {
      const int par = done ? 0 : (i - 1) >> 1;
      const double kp_ = hk(par);
      const uint16_t pp_ = hp(par);
      const bool go = !done && less(key, pc, kp_, pp_);
      if (go) {
        hk(i) = kp_;
        hp(i) = pp_;
        i = par;
      }
      done = done || !go || i == 0;
    }
    if (doit) {
      hk(i) = key;
      hp(i) = pc;
    }
  };
  push(__dadd_rn(d1[0], d2[0]), 0u, true);
  int np = 0;
  int64_t got = 0;
  uint16_t* out = pops + t * cap;
  double* kout = keys_out ? keys_out + t * cap : nullptr;
  // Software-pipelined: the top's successor distances and labels are loaded
  // before the pop's sift-down (which hides their latency), and a popped
  // cell's size is loaded when it is popped but added one pop later, so no
  // pop waits on the size load.  The pop made after the target was reached
  // is dropped (np does not count it): same pops, counts and sizes as the
  // reference loop.
  int64_t psz = 0;        // size of the last counted pop, not yet added
  bool pend = false;
  const double d20 = d2[0];
  while (true) {
    if (hn == 0) {
      if (pend) got += psz;
      break;
    }
    const double key = hk(0);
    const uint32_t pc = hp(0);
    const int r = (int)(pc >> 8), c = (int)(pc & 0xFF);
    const bool nr = c == 0 && r + 1 < kp, nc = c + 1 < kp;
    const double dr1 = nr ? d1[r + 1] : 0.0;
    const double dr = d1[r];
    const double dc1 = nc ? d2[c + 1] : 0.0;
    const int cell = (int)l1[r] * kp + (int)l2[c];
    --hn;
    {
      const double lk = hk(hn);
      const uint16_t lp = hp(hn);
      int i = 0;
      bool done = hn == 0;
#pragma unroll
      for (int lev = 0; lev < LOGK; ++lev) {
        const int a = 2 * i + 1, b = a + 1;
        const bool va = !done && a < hn, vb = !done && b < hn;
        const int ia = va ? a : 0, ib = vb ? b : 0;
        const double ka = hk(ia), kb = hk(ib);
        const uint16_t pa = hp(ia), pb = hp(ib);
        const bool useb = vb && less(kb, pb, ka, pa);
        const double km = useb ? kb : ka;
        const uint16_t pm = useb ? pb : pa;
        const bool go = va && less(km, pm, lk, lp);
        if (go) {
          hk(i) = km;
          hp(i) = pm;
          i = useb ? b : a;
        }
        done = done || !go;
      }
      if (hn > 0) {
        hk(i) = lk;
        hp(i) = lp;
      }
    }
    if (np < cap) {
      out[np] = (uint16_t)cell;
      if (kout) kout[np] = key;
    }
    if (pend) {
      got += psz;
      if (got >= target) break;   // the previous pop reached the target: this one is not counted
    }
    psz = gs[cell];
    pend = true;
    ++np;
    push(__dadd_rn(dr1, d20), (uint32_t)(r + 1) << 8, nr);
    push(__dadd_rn(dr, dc1), ((uint32_t)r << 8) | (uint32_t)(c + 1), nc);
  }
  npop[t] = np;
  ret[t] = got;
  if (np > cap) atomicMax((unsigned long long*)&flags[0], (unsigned long long)np);
}
#undef hk
#undef hp

// k_traverse_sh with PERSISTENT LANES: a lane that finishes its walk takes
// the next one from a global counter instead of idling until the longest of
// its warp's 32 walks ends (walk lengths at config 2: ~110 pops on average,
// 237 the longest), and the grid is one resident wave, so there is no second,
// partly filled wave either.  Same pops, counts and sizes.
template <int KMAX, int TS_THREADS>
__global__ void __launch_bounds__(TS_THREADS) k_traverse_pl(const double* __restrict__ sd,
                                                  const uint16_t* __restrict__ sl,
                                                  const int64_t* __restrict__ gsize, int64_t Q,
                                                  int n_sub, int kp, int64_t target,
                                                  uint16_t* __restrict__ pops, int cap,
                                                  double* __restrict__ keys_out,
                                                  int32_t* __restrict__ npop,
                                                  int64_t* __restrict__ ret,
                                                  int64_t* __restrict__ flags,
                                                  unsigned long long* __restrict__ next_walk) {
  const int64_t total = Q * n_sub;
  extern __shared__ __align__(16) unsigned char tsh_sm[];
  double* const hkb = reinterpret_cast<double*>(tsh_sm) + threadIdx.x;
  uint16_t* const hpb = reinterpret_cast<uint16_t*>(reinterpret_cast<double*>(tsh_sm) + KMAX * TS_THREADS) + threadIdx.x;
  struct HeapRef {
    double* k;
    uint16_t* p;
    __device__ double& key(int i) const { return k[i * TS_THREADS]; }
    __device__ uint16_t& pc(int i) const { return p[i * TS_THREADS]; }
  };
  const HeapRef H{hkb, hpb};
#define hk(i) H.key(i)
#define hp(i) H.pc(i)
  int hn = 0;
  auto less = [&](double ka, uint32_t pa, double kb, uint32_t pb) {
    return ka < kb || (ka == kb && pa < pb);
  };
  // 4-ary heap (depth 3 for K' <= 64): a sift level loads its 4 children at
  // once, so a pop's dependent chain is half a binary heap's; the pop and the
  // push of (r, c + 1) are ONE replace-top sift-down.  (key, r << 8 | c) is a
  // strict total order, so any correct priority queue pops the same sequence.
  constexpr int LOG4 = KMAX <= 21 ? 2 : KMAX <= 85 ? 3 : 4;
  auto sift_up = [&](double key, uint32_t pc32, bool doit) {   // insert at the end
    const uint16_t pc = (uint16_t)pc32;
    int i = hn;
    hn += doit ? 1 : 0;
    bool done = !doit || i == 0;
#pragma unroll
    for (int lev = 0; lev < LOG4; ++lev) {
      const int par = done ? 0 : (i - 1) >> 2;
      const double kp_ = hk(par);
      const uint16_t pp_ = hp(par);
      const bool go = !done && less(key, pc, kp_, pp_);
      if (go) {
        hk(i) = kp_;
        hp(i) = pp_;
        i = par;
      }
      done = done || !go || i == 0;
    }
    if (doit) {
      hk(i) = key;
      hp(i) = pc;
    }
  };
  auto sift_down_root = [&](double lk, uint32_t lp32, bool doit) {   // place (lk, lp) starting at the root
    const uint16_t lp = (uint16_t)lp32;
    int i = 0;
    bool done = !doit;
#pragma unroll
    for (int lev = 0; lev < LOG4; ++lev) {
      const int a = 4 * i + 1;
      const bool v0 = !done && a < hn, v1 = !done && a + 1 < hn, v2 = !done && a + 2 < hn, v3 = !done && a + 3 < hn;
      const int i0 = v0 ? a : 0, i1 = v1 ? a + 1 : 0, i2 = v2 ? a + 2 : 0, i3 = v3 ? a + 3 : 0;
      const double k0 = hk(i0), k1 = hk(i1), k2 = hk(i2), k3 = hk(i3);
      const uint16_t p0 = hp(i0), p1 = hp(i1), p2 = hp(i2), p3 = hp(i3);
      // tournament: (0 vs 1), (2 vs 3), then the winners; an invalid child never wins
      const bool b1 = v1 && less(k1, p1, k0, p0);
      const double ka = b1 ? k1 : k0;
      const uint16_t pa = b1 ? p1 : p0;
      const int ia = b1 ? a + 1 : a;
      const bool b3 = v3 && less(k3, p3, k2, p2);
      const double kb = b3 ? k3 : k2;
      const uint16_t pb = b3 ? p3 : p2;
      const int ib = b3 ? a + 3 : a + 2;
      const bool bb = v2 && less(kb, pb, ka, pa);
      const double km = bb ? kb : ka;
      const uint16_t pm = bb ? pb : pa;
      const int im = bb ? ib : ia;
      const bool go = v0 && less(km, pm, lk, lp);
      if (go) {
        hk(i) = km;
        hp(i) = pm;
        i = im;
      }
      done = done || !go;
    }
    if (doit) {
      hk(i) = lk;
      hp(i) = lp;
    }
  };
  // the walk in progress
  int64_t t = 0, got = 0, psz = 0;
  const double *d1 = nullptr, *d2 = nullptr;
  const uint16_t *l1 = nullptr, *l2 = nullptr;
  const int64_t* gs = nullptr;
  uint16_t* out = nullptr;
  double* kout = nullptr;
  double d20 = 0.0;
  int np = 0;
  bool pend = false, active = false;
  while (true) {
    if (!active) {
      t = (int64_t)atomicAdd(next_walk, 1ull);
      if (t >= total) break;
      const int j = (int)(t % n_sub);
      d1 = sd + t * 2 * kp;
      d2 = d1 + kp;
      l1 = sl + t * 2 * kp;
      l2 = l1 + kp;
      gs = gsize + (size_t)j * kp * kp;
      out = pops + t * cap;
      kout = keys_out ? keys_out + t * cap : nullptr;
      hn = 0;
      np = 0;
      got = 0;
      psz = 0;
      pend = false;
      d20 = d2[0];
      sift_up(__dadd_rn(d1[0], d20), 0u, true);
      active = true;
    }
    bool fin = false;
    if (hn == 0) {
      if (pend) got += psz;
      fin = true;
    } else {
      const double key = hk(0);
      const uint32_t pc = hp(0);
      const int r = (int)(pc >> 8), c = (int)(pc & 0xFF);
      const bool nr = c == 0 && r + 1 < kp, nc = c + 1 < kp;
      const double dr1 = nr ? d1[r + 1] : 0.0;
      const double dr = d1[r];
      const double dc1 = nc ? d2[c + 1] : 0.0;
      const int cell = (int)l1[r] * kp + (int)l2[c];
      if (np < cap) {
        out[np] = (uint16_t)cell;
        if (kout) kout[np] = key;
      }
      if (pend) {
        got += psz;
        fin = got >= target;   // the previous pop reached the target: this one is not counted
      }
      if (!fin) {
        psz = gs[cell];
        pend = true;
        ++np;
        // the top is replaced by its row successor (r, c + 1), or by the last entry when the row ends
        hn -= nc ? 0 : 1;
        const int li = nc ? 0 : hn;
        const double lk = nc ? __dadd_rn(dr, dc1) : hk(li);
        const uint32_t lp = nc ? (((uint32_t)r << 8) | (uint32_t)(c + 1)) : (uint32_t)hp(li);
        sift_down_root(lk, lp, hn > 0);
        sift_up(__dadd_rn(dr1, d20), (uint32_t)(r + 1) << 8, nr);
      }
    }
    if (fin) {
      npop[t] = np;
      ret[t] = got;
      if (np > cap) atomicMax((unsigned long long*)&flags[0], (unsigned long long)np);
      active = false;
    }
  }
}
#undef hk
#undef hp

static int num_sms();

// TACO_TRAVERSE=heap / =smem / =pl force the thread-local-heap / shared-memory
// / persistent-lane kernel (tests pin all three); default: by batch size
// (launch_traverse)
static int traverse_force() {
  const char* e = getenv("TACO_TRAVERSE");
  if (!e) return 0;
  return !strcmp(e, "heap") ? 1 : !strcmp(e, "smem") ? 2 : !strcmp(e, "pl") ? 3 : 0;
}

// launch the traversal of Q queries x n_sub subspaces
static int launch_traverse(const double* sd, const uint16_t* sl, const int64_t* gsize, int64_t Q, int n_sub, int kp,
                           int64_t target, uint16_t* pops, int cap, double* keys_out, int32_t* npop, int64_t* ret,
                           int64_t* flags, cudaStream_t st) {
  const int64_t th = Q * n_sub;
  // small batches (fewer than ~128 walks per SM): the thread-local heaps fit
  // L1 and the variable-depth sifts finish sooner (configs 1 / 3: 0.23 / 0.25
  // ms vs 0.29 / 0.27); large batches: the shared-memory fixed-depth heap
  const int force = traverse_force();
  if (force >= 2 || (force == 0 && th >= (int64_t)num_sms() * 128)) {
  // 64 walks per CTA; 32 when that would leave SMs idle
  static int narrow_env = -1;   // TACO_TRAVERSE_NARROW=1 / =0: force 32- / 64-walk CTAs (experiments)
  if (narrow_env < 0) {
    const char* e = getenv("TACO_TRAVERSE_NARROW");
    narrow_env = !e ? 2 : (e[0] == '1' ? 1 : 0);
  }
  const bool narrow = narrow_env == 2 ? th < (int64_t)num_sms() * 64 * 4 : narrow_env == 1;
#define TRAVP(KM)                                                                                           \
  {                                                                                                         \
    constexpr int TS = 32;                                                                                  \
    const size_t smem = (size_t)KM * TS * 10;                                                               \
    static int per_sm = 0;                                                                                  \
    if (!per_sm) {                                                                                          \
      TACO_CHECK_CUDA(cudaFuncSetAttribute(k_traverse_pl<KM, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           (int)smem));                                                     \
      TACO_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, k_traverse_pl<KM, TS>, TS, smem)); \
      if (per_sm < 1) per_sm = 1;                                                                           \
    }                                                                                                       \
    TACO_CHECK_CUDA(cudaMemsetAsync(flags + 5, 0, sizeof(int64_t), st));                                    \
    const int64_t ctas = std::min<int64_t>(ceil_div(th, TS), (int64_t)per_sm * num_sms());                  \
    k_traverse_pl<KM, TS><<<(unsigned)ctas, TS, smem, st>>>(sd, sl, gsize, Q, n_sub, kp, target, pops, cap, \
                                                            keys_out, npop, ret, flags,                    \
                                                            reinterpret_cast<unsigned long long*>(flags + 5)); \
  }
    // persistent lanes (flags[5] = the walk counter) once the batch exceeds one resident wave
    static int pl_env = -1;   // TACO_TRAVERSE_PL=0: one walk per thread (k_traverse_sh)
    if (pl_env < 0) {
      const char* e = getenv("TACO_TRAVERSE_PL");
      pl_env = (e && e[0] == '0') ? 0 : 1;
    }
    if (force == 3 || (pl_env && force == 0 && th >= (int64_t)num_sms() * 256)) {
      if (kp <= 32) TRAVP(32)
      else if (kp <= 64) TRAVP(64)
      else if (kp <= 128) TRAVP(128)
      else TRAVP(256)
      return TACO_OK;
    }
#undef TRAVP
#define TRAVS1(KM, TS)                                                                                      \
  {                                                                                                         \
    const size_t smem = (size_t)KM * TS * 10;                                                               \
    static bool attr = false;                                                                               \
    if (!attr) {                                                                                            \
      TACO_CHECK_CUDA(cudaFuncSetAttribute(k_traverse_sh<KM, TS>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                                           (int)smem));                                                     \
      attr = true;                                                                                          \
    }                                                                                                       \
    k_traverse_sh<KM, TS><<<(unsigned)ceil_div(th, TS), TS, smem, st>>>(sd, sl, gsize, Q, n_sub, kp, target, \
                                                                      pops, cap, keys_out, npop, ret, flags);  \
  }
#define TRAVS(KM) \
  if (narrow) TRAVS1(KM, 32) else TRAVS1(KM, 64)
    if (kp <= 32) TRAVS(32)
    else if (kp <= 64) TRAVS(64)
    else if (kp <= 128) TRAVS(128)
    else TRAVS(256)
#undef TRAVS
#undef TRAVS1
    return TACO_OK;
  }
  const unsigned g = (unsigned)ceil_div(th, 128);
#define TRAV(KM) \
  k_traverse<KM><<<g, 128, 0, st>>>(sd, sl, gsize, Q, n_sub, kp, target, pops, cap, keys_out, npop, ret, flags)
  if (kp <= 32) TRAV(32);
  else if (kp <= 64) TRAV(64);
  else if (kp <= 128) TRAV(128);
  else TRAV(256);
#undef TRAV
  return TACO_OK;
}

// ---------------------------------------------------------- block helpers
// Exclusive scan of one value per thread (uint32), returns the block total.
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan(uint32_t v, uint32_t* wtot, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtot[wid] = x;
  __syncthreads();
  if (wid == 0) {
    uint32_t w = lane < NT / 32 ? wtot[lane] : 0u;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      uint32_t y = __shfl_up_sync(0xffffffffu, w, o);
      if (lane >= o) w += y;
    }
    if (lane < NT / 32) wtot[lane] = w;
  }
  __syncthreads();
  total = wtot[NT / 32 - 1];
  const uint32_t excl = (wid ? wtot[wid - 1] : 0u) + x - v;
  __syncthreads();
  return excl;
}

// block_excl_scan with two barriers: every thread sums the warp totals below
// its warp itself (NT / 32 broadcast loads) instead of waiting for warp 0's scan
template <int NT>
__device__ __forceinline__ uint32_t block_excl_scan2(uint32_t v, uint32_t* wtot, uint32_t& total) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  uint32_t x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) wtot[wid] = x;
  __syncthreads();
  uint32_t below = 0, all = 0;
#pragma unroll
  for (int w = 0; w < NT / 32; ++w) {
    const uint32_t t = wtot[w];
    all += t;
    if (w < wid) below += t;
  }
  total = all;
  __syncthreads();   // wtot is free again
  return below + x - v;
}

// ------------------------------------------------------------ chunk counting
// Counts into `table` (ids [base, base+chunk)) every id of the cells popped for
// query q in subspaces 0..n_sub-1.  Phase A stages the slices of all popped
// cells (one round trip for their CSR bounds, one block scan).  Phase B walks
// subspace by subspace; each warp owns a contiguous part of the subspace's
// flattened id list and fetches it 32 consecutive ids per instruction
// (coalesced inside a slice), CT_E steps per round, the next round's ids in
// flight while the current round's byte increments are applied.  Ids are
// unique inside one subspace, so increments need no atomics; a barrier
// separates subspaces.  Every increment leaving level v is tallied (packed
// 16-bit counters), which gives the level histogram without rescanning:
// #(score >= l) = #(increments leaving level l-1).
constexpr int CT_THREADS = 256;
constexpr int CT_PB = 1024;   // slices staged per batch

constexpr int CT_UC = 2048;   // units (<= 8 consecutive ids of one slice) staged per round

struct CountSmem {
  uint32_t uidx[CT_UC];       // absolute index into ids[] of the unit's first id
  uint8_t ulen[CT_UC];        // ids in the unit (1..8)
  uint32_t wtot[CT_THREADS / 32];
  int jpref[257];             // pop prefix over subspaces
  int ge[257];                // ge[l] = #ids of the chunk with score >= l  (l >= 1)
  int lh[256];                // level histogram (lh[0] = ids at score 0)
  int batches;                // number of pop batches the query needed
};

// Per-thread tallies of "increment left level v": n_sub <= 8 packs levels
// 0..7 as 4-bit fields per unit, 8-bit fields per round and 16-bit fields per
// chunk; else 16-bit fields in four words.

__device__ __forceinline__ uint32_t smem_atomic_add(uint32_t addr, uint32_t v) {
  uint32_t old;
  asm volatile("atom.shared::cta.add.u32 %0, [%1], %2;" : "=r"(old) : "r"(addr), "r"(v) : "memory");
  return old;
}
struct Tally {
  uint64_t a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  // ev / od: 8-bit fields of levels 0,2,4,6 / 1,3,5,7 -> 16-bit fields
  __device__ __forceinline__ void add_round(uint32_t ev, uint32_t od) {
    a0 += ((uint64_t)__byte_perm(ev, 0, 0x4342) << 32) | __byte_perm(ev, 0, 0x4140);
    a1 += ((uint64_t)__byte_perm(od, 0, 0x4342) << 32) | __byte_perm(od, 0, 0x4140);
  }
  __device__ __forceinline__ void add_wide(uint32_t old) {
    const uint64_t inc = 1ull << ((old & 3u) << 4);
    if (old < 4) a0 += inc;
    else if (old < 8) a1 += inc;
    else if (old < 12) a2 += inc;
    else a3 += inc;
  }
  // levels 8..15 of the encoded kernels' wide tallies (a0 / a1 hold 0..7 as in add_round)
  __device__ __forceinline__ void add_round_hi(uint32_t ev, uint32_t od) {
    a2 += ((uint64_t)__byte_perm(ev, 0, 0x4342) << 32) | __byte_perm(ev, 0, 0x4140);
    a3 += ((uint64_t)__byte_perm(od, 0, 0x4342) << 32) | __byte_perm(od, 0, 0x4140);
  }
  __device__ __forceinline__ int level2(int l) const {   // add_round / add_round_hi layout, l <= 15
    const int b = l & 7;
    const uint64_t w = l < 8 ? ((b & 1) ? a1 : a0) : ((b & 1) ? a3 : a2);
    return (int)((w >> (16 * (b >> 1))) & 0xFFFFull);
  }
  __device__ __forceinline__ int level(int l, bool small) const {   // tally of level l
    if (small) {
      const uint64_t w = (l & 1) ? a1 : a0;
      return (int)((w >> (16 * (l >> 1))) & 0xFFFFull);
    }
    const uint64_t w = l < 4 ? a0 : l < 8 ? a1 : l < 12 ? a2 : a3;
    return (int)((w >> (16 * (l & 3))) & 0xFFFFull);
  }
};

// Phase A + B for one (query, chunk): the popped cells' slices of this chunk
// are cut into units of <= 8 consecutive ids (CSR order), units are staged
// CT_UC at a time and consumed round-robin by the threads: no per-id search
// or walk, 8 independent loads per unit, the next unit's loads in flight
// while the current one is applied with shared-memory byte-lane atomics
// (scores <= n_sub <= 255 never carry into the next byte).
template <bool NIB, bool SMALL>
__device__ void count_chunk_impl(const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
                            const uint32_t* __restrict__ ids, const uint32_t* __restrict__ offs,
                            size_t offs_len, int n_sub, int K2, int64_t n, int64_t c, int64_t q,
                            int64_t base, uint8_t* table, CountSmem& S) {
  const int tid = threadIdx.x;
  constexpr bool small = SMALL;   // n_sub <= 8
  static_assert(CT_UC / CT_THREADS * 8 <= 255, "per-round tally fields are 8-bit");
  // 32-bit smem address of the table, biased by the chunk base (mod 2^32 arithmetic)
  uint32_t tsg = (uint32_t)__cvta_generic_to_shared(table) - (NIB ? ((uint32_t)base >> 1) : (uint32_t)base);
  asm volatile("mov.u32 %0, %0;" : "+r"(tsg));   // keep it in a register (no per-atomic rematerialisation)
  Tally T;
  if (tid == 0) {
    int acc = 0;
    for (int j = 0; j < n_sub; ++j) {
      S.jpref[j] = acc;
      acc += min(npop[q * n_sub + j], cap);
    }
    S.jpref[n_sub] = acc;
    S.batches = (acc + CT_PB - 1) / CT_PB;
  }
  __syncthreads();
  const int P_all = S.jpref[n_sub];
  constexpr int PER = CT_PB / CT_THREADS;
  for (int b0 = 0; b0 < P_all; b0 += CT_PB) {
    const int nb = min(CT_PB, P_all - b0);
    uint32_t sa[PER], ln[PER], ub[PER];
    uint32_t myu = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int t = tid * PER + u;
      sa[u] = 0;
      ln[u] = 0;
      if (t < nb) {
        const int g = b0 + t;
        int lo = 0, hi = n_sub;  // largest j with jpref[j] <= g
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (S.jpref[mid] <= g) lo = mid; else hi = mid;
        }
        const int j = lo;
        const int cell = pops[((size_t)q * n_sub + j) * cap + (g - S.jpref[j])];
        const uint32_t* O = offs + (size_t)j * offs_len + (size_t)c * K2;
        const uint32_t s0 = __ldg(O + cell), s1 = __ldg(O + cell + 1);
        sa[u] = (uint32_t)((size_t)j * n + s0);
        ln[u] = s1 - s0;
      }
      myu += (ln[u] + 7u) >> 3;
    }
    uint32_t utot;
    uint32_t run = block_excl_scan<CT_THREADS>(myu, S.wtot, utot);
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      ub[u] = run;
      run += (ln[u] + 7u) >> 3;
    }
    for (uint32_t r0 = 0; r0 < utot; r0 += CT_UC) {
      const uint32_t r1 = min(utot, r0 + (uint32_t)CT_UC);
      // scatter my slices' units of this round into the table
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const uint32_t nu = (ln[u] + 7u) >> 3;
        const uint32_t k0 = max(ub[u], r0), k1 = min(ub[u] + nu, r1);
        for (uint32_t k = k0; k < k1; ++k) {
          const uint32_t off = (k - ub[u]) << 3;
          S.uidx[k - r0] = sa[u] + off;
          S.ulen[k - r0] = (uint8_t)min(8u, ln[u] - off);
        }
      }
      __syncthreads();
      // consume: units tid, tid + CT_THREADS, ... with one unit of lookahead
      const int nr = (int)(r1 - r0);
      uint32_t ev = 0, od = 0;   // per-round level tallies (small), 8-bit fields
      uint32_t va[8], vb[8];   // lanes past a unit's length keep a valid id of this chunk (+0 atomics)
#pragma unroll
      for (int e = 0; e < 8; ++e) va[e] = vb[e] = (uint32_t)base;
      int la = 0, lb = 0;
      auto fetch = [&](int k, uint32_t* v, int& l) {
        l = 0;
        if (k < nr) {
          const uint32_t* src = ids + S.uidx[k];
          l = S.ulen[k];
#pragma unroll
          for (int e = 0; e < 8; ++e)
            if (e < l) v[e] = __ldg(src + e);
        }
      };
      // All of a unit's atomics are issued before any returned word is used
      // (they are independent: the latencies overlap), lanes past the unit's
      // length add 0 to a word they already own (no branches, no effect).
      auto apply = [&](const uint32_t* v, int l) {
        uint32_t sh[8], ad[8], old[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          // table word of id x lives at tsg + (x >> 1 or x) & ~3: tsg absorbs the chunk base
          // (a multiple of 1024, so the lane position within the word is x's own low bits)
          const uint32_t x = v[e];
          sh[e] = NIB ? (x << 2) & 28u : (x << 3) & 24u;
          ad[e] = tsg + (NIB ? ((x >> 1) & ~3u) : (x & ~3u));
        }
#pragma unroll
        for (int e = 0; e < 8; ++e) old[e] = smem_atomic_add(ad[e], e < l ? 1u << sh[e] : 0u);
        uint32_t u4 = 0;   // small: 8 x 4-bit fields "left level v" (<= 8 ids per unit)
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const uint32_t r = old[e] >> sh[e];
          if (small) u4 += e < l ? 1u << ((r << 2) & 28u) : 0u;
          else if (e < l) T.add_wide(r & (NIB ? 0xFu : 0xFFu));
        }
        if (small) {   // <= CT_UC / CT_THREADS units per round: 8-bit fields cannot overflow
          ev += u4 & 0x0F0F0F0Fu;
          od += (u4 >> 4) & 0x0F0F0F0Fu;
        }
      };
      int k = tid;
      fetch(k, va, la);
      while (k < nr) {   // ping-pong buffers: no register moves between units
        fetch(k + CT_THREADS, vb, lb);
        apply(va, la);
        k += CT_THREADS;
        if (k >= nr) break;
        fetch(k + CT_THREADS, va, la);
        apply(vb, lb);
        k += CT_THREADS;
      }
      if (small) T.add_round(ev, od);
      __syncthreads();
    }
  }
  for (int i = tid; i < 257; i += CT_THREADS) S.ge[i] = 0;
  __syncthreads();
  if (n_sub <= 16) {
    for (int l = 1; l <= n_sub; ++l) {
      int x = T.level(l - 1, small);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if ((tid & 31) == 0 && x) atomicAdd(&S.ge[l], x);
    }
  }
  __syncthreads();
}

template <bool NIB>
__device__ __forceinline__ void count_chunk(const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop,
                                            int cap, const uint32_t* __restrict__ ids,
                                            const uint32_t* __restrict__ offs, size_t offs_len, int n_sub, int K2,
                                            int64_t n, int64_t c, int64_t q, int64_t base, uint8_t* table,
                                            CountSmem& S) {
  if (n_sub <= 8) count_chunk_impl<NIB, true>(pops, npop, cap, ids, offs, offs_len, n_sub, K2, n, c, q, base, table, S);
  else count_chunk_impl<NIB, false>(pops, npop, cap, ids, offs, offs_len, n_sub, K2, n, c, q, base, table, S);
}

// Level histogram of a chunk table.  n_sub <= 16: from the tallies; else by a
// scan of the table (atomics per nonzero byte).
template <typename SM>
__device__ void chunk_levels(const uint8_t* table, int valid, int n_sub, SM& S) {
  const int tid = threadIdx.x;
  constexpr bool kScan = sizeof(S.lh) / sizeof(int) >= 256;   // EncSmem holds 17 levels only
  if (n_sub <= 16 || !kScan) {
    for (int l = tid; l <= n_sub; l += blockDim.x) {
      const int gl = l == 0 ? valid : S.ge[l];
      const int gn = l == n_sub ? 0 : S.ge[l + 1];
      S.lh[l] = gl - gn;
    }
  } else {
    for (int l = tid; l < 256; l += blockDim.x) S.lh[l] = 0;
    __syncthreads();
    const uint32_t* w4 = reinterpret_cast<const uint32_t*>(table);
    for (int i = tid; i < (valid + 3) / 4; i += blockDim.x) {
      uint32_t w = w4[i];
      while (w) {
        const int b = __ffs(w) - 1;
        const int byte = b >> 3;
        atomicAdd(&S.lh[(w >> (byte * 8)) & 0xFF], 1);
        w &= ~(0xFFu << (byte * 8));
      }
    }
    __syncthreads();
    if (tid == 0) {
      int nz = 0;
      for (int l = 1; l <= n_sub; ++l) nz += S.lh[l];
      S.lh[0] = valid - nz;
    }
  }
  __syncthreads();
}

// Lanes (4-bit or 8-bit counters) of w that are >= L, as the lane's top bit:
// the carry out of lane + (2^W - L), computed without cross-lane carries
// (s holds each lane's carry into its top bit).  D = (2^W - L) per lane, L >= 1.
template <bool NIB>
__device__ __forceinline__ uint32_t lanes_ge(uint32_t w, uint32_t D) {
  constexpr uint32_t H = NIB ? 0x88888888u : 0x80808080u;
  const uint32_t s = (w & ~H) + (D & ~H);
  return ((w & D) | ((w | D) & s)) & H;
}

// Ordered compaction of ids (id0 + position) whose score >= L from a table of
// `valid` counters (4-bit or 8-bit, 16-byte aligned, zero padded): every
// thread owns a contiguous run of 16-byte vectors, one block scan places them.
template <int NT, bool NIB = false>
__device__ void compact_table(const uint8_t* tab, int valid, uint32_t L, int64_t id0, uint32_t* dst,
                              uint32_t* wtot) {
  constexpr int LW = NIB ? 4 : 8;                // lane width (bits)
  constexpr int LPW = 32 / LW;                   // lanes per word
  constexpr int IDS = 4 * LPW;                   // ids per 16-byte vector
  constexpr uint32_t H = NIB ? 0x88888888u : 0x80808080u;
  const uint32_t D = L == 0 ? 0u : (NIB ? (16u - L) * 0x11111111u : (256u - L) * 0x01010101u);
  const uint4* t4 = reinterpret_cast<const uint4*>(tab);
  const int nvec = (valid + IDS - 1) / IDS;
  const int per = (nvec + NT - 1) / NT;          // vectors per thread
  const int v0 = threadIdx.x * per, v1 = min(nvec, v0 + per);
  const int nv = max(v1 - v0, 0);
  // lane top bits of vector vi with score >= L, lanes past `valid` cleared
  auto vec_bits = [&](int vi, uint32_t (&g)[4]) {
    const uint4 v = t4[vi];
    if (L == 0) {
      g[0] = g[1] = g[2] = g[3] = H;
    } else {
      g[0] = lanes_ge<NIB>(v.x, D); g[1] = lanes_ge<NIB>(v.y, D);
      g[2] = lanes_ge<NIB>(v.z, D); g[3] = lanes_ge<NIB>(v.w, D);
    }
    const int lim = valid - vi * IDS;
    if (lim < IDS) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int al = min(max(lim - u * LPW, 0), LPW);
        g[u] &= al >= LPW ? 0xFFFFFFFFu : (1u << (al * LW)) - 1u;
      }
    }
  };
  uint32_t cnt = 0;
  uint32_t hit = 0;                              // which of my first 31 vectors hold matches
  for (int i = 0; i < nv; ++i) {
    const int vi = v0 + (i + threadIdx.x) % nv;  // rotated start: bank-conflict free
    uint32_t g[4];
    vec_bits(vi, g);
    if (g[0] | g[1] | g[2] | g[3]) {
      cnt += __popc(g[0]) + __popc(g[1]) + __popc(g[2]) + __popc(g[3]);
      hit |= vi - v0 < 31 ? 1u << (vi - v0) : 0x80000000u;
    }
  }
  uint32_t tot;
  uint32_t pos = block_excl_scan<NT>(cnt, wtot, tot);
  for (int i = 0; i < nv; ++i) {
    if (i < 31 ? !((hit >> i) & 1u) : !(hit >> 31)) continue;
    const int vi = v0 + i;
    uint32_t g[4];
    vec_bits(vi, g);
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int64_t idb = id0 + (int64_t)vi * IDS + u * LPW;
      uint32_t m = g[u];
      while (m) {
        const int bb = __ffs(m) - 1;
        dst[pos++] = (uint32_t)(idb + bb / LW);
        m &= m - 1u;
      }
    }
  }
}

// Unordered single-pass compaction (the batch paths: a segment's candidates
// are re-ranked as a set, ties are broken by id, so their order is free).
// A warp step covers CP_VPL x 32 consecutive 16-byte vectors: lane l tests
// vectors l, l + 32, ... (conflict-free 16-byte reads, CP_VPL independent
// load/compare chains in flight), one warp prefix of the lanes' hit counts
// and one shared-memory reservation place them, then each lane writes its
// own hits.  *fill ends = count.
constexpr int CP_VPL = 4;
template <bool NIB>
__device__ __forceinline__ uint32_t vec_hits(const uint4 v, uint32_t D, int lim) {
  constexpr int LW = NIB ? 4 : 8;
  constexpr int LPW = 32 / LW;
  constexpr int IDS = 4 * LPW;
  constexpr uint32_t H = NIB ? 0x88888888u : 0x80808080u;
  uint32_t g[4];
  if (D == 0u) {
    g[0] = g[1] = g[2] = g[3] = H;
  } else {
    g[0] = lanes_ge<NIB>(v.x, D); g[1] = lanes_ge<NIB>(v.y, D);
    g[2] = lanes_ge<NIB>(v.z, D); g[3] = lanes_ge<NIB>(v.w, D);
  }
  if (lim < IDS) {
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const int al = min(max(lim - u * LPW, 0), LPW);
      g[u] &= al >= LPW ? 0xFFFFFFFFu : (1u << (al * LW)) - 1u;
    }
  }
  // word u's hits sit at lane tops (bit LW*i + LW-1); shifted by u they are disjoint
  return g[0] | (g[1] >> 1) | (g[2] >> 2) | (g[3] >> 3);
}

// warp-inclusive prefix of c; lane 31 reserves the step's slots in *fill;
// returns the lane's first slot
__device__ __forceinline__ uint32_t warp_reserve(uint32_t c, int* fill) {
  const int lane = threadIdx.x & 31;
  uint32_t x = c;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  int base = 0;
  if (lane == 31) base = atomicAdd(fill, (int)x);
  return (uint32_t)__shfl_sync(0xffffffffu, base, 31) + x - c;
}

// SMALL (4-bit lanes holding scores <= 8, L >= 1): lane >= L <=> bit 3 of
// lane + (8 - L), which cannot carry into the next lane (<= 15).
__device__ __forceinline__ uint32_t vec_hits_small(const uint4 v, uint32_t K, int lim) {
  constexpr uint32_t H = 0x88888888u;
  uint32_t g0 = (v.x + K) & H, g1 = (v.y + K) & H, g2 = (v.z + K) & H, g3 = (v.w + K) & H;
  if (lim < 32) {
    const uint32_t m0 = lim >= 8 ? ~0u : (1u << (4 * lim)) - 1u;
    const uint32_t m1 = lim >= 16 ? ~0u : lim <= 8 ? 0u : (1u << (4 * (lim - 8))) - 1u;
    const uint32_t m2 = lim >= 24 ? ~0u : lim <= 16 ? 0u : (1u << (4 * (lim - 16))) - 1u;
    const uint32_t m3 = lim <= 24 ? 0u : (1u << (4 * (lim - 24))) - 1u;
    g0 &= m0; g1 &= m1; g2 &= m2; g3 &= m3;
  }
  return g0 | (g1 >> 1) | (g2 >> 2) | (g3 >> 3);
}

template <int NT, bool NIB, bool SMALL = false>
__device__ void compact_unordered(const uint8_t* tab, int valid, uint32_t L, int64_t id0, uint32_t* dst,
                                  int* fill) {
  constexpr int LW = NIB ? 4 : 8;
  constexpr int LPW = 32 / LW;
  constexpr int IDS = 4 * LPW;
  const uint32_t D = L == 0 ? 0u : (NIB ? (16u - L) * 0x11111111u : (256u - L) * 0x01010101u);
  const uint32_t K = (8u - L) * 0x11111111u;
  const uint4* t4 = reinterpret_cast<const uint4*>(tab);
  const int nvec = (valid + IDS - 1) / IDS;
  const int lane = threadIdx.x & 31;
  for (int v0 = (threadIdx.x - lane) * CP_VPL; v0 < nvec; v0 += NT * CP_VPL) {
    uint32_t m[CP_VPL];
    uint32_t c = 0;
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      const int vi = v0 + e * 32 + lane;
      if (SMALL && L >= 1)
        m[e] = vi < nvec ? vec_hits_small(t4[vi], K, valid - vi * IDS) : 0u;
      else
        m[e] = vi < nvec ? vec_hits<NIB>(t4[vi], D, valid - vi * IDS) : 0u;
      c += __popc(m[e]);
    }
    if (__ballot_sync(0xffffffffu, c != 0u) == 0u) continue;
    uint32_t pos = warp_reserve(c, fill);
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      const uint32_t idb = (uint32_t)(id0 + (int64_t)(v0 + e * 32 + lane) * IDS);
      uint32_t mm = m[e];
      while (mm) {
        const int b = 31 - __clz(mm);                  // highest hit first (order is free)
        mm ^= 1u << b;
        const int u = LW - 1 - (b & (LW - 1));          // word
        dst[pos++] = idb + (uint32_t)(u * LPW + b / LW);   // lane b / LW of word u
      }
    }
  }
}

// Two-phase unordered compaction for sparse hits (a query's candidates are
// ~0.3% of the ids).  Phase 1 only asks "does this 16-byte vector hold any
// lane >= L" (a few instructions per vector) and records the vector indices
// (ballot-ranked, one reservation per warp step) in `rec`; phase 2 gives
// every record to one thread, which recomputes the lane mask and writes the
// ids.  The single-pass scan spends most of its instructions on per-lane hit
// loops that run with one or two lanes active.  L >= 1; lanes past `valid`
// are zero, so they never hit.  Returns false (nothing written) when the
// records would not fit rcap.
#ifndef EC_TWOPHASE
#define EC_TWOPHASE 1
#endif
template <int NT, bool NIB, bool SMALL>
__device__ bool compact_two_phase(const uint8_t* tab, int valid, uint32_t L, int64_t id0, uint32_t* dst, int* fill,
                                  uint16_t* rec, int rcap, int* rfill) {
  constexpr int LW = NIB ? 4 : 8;
  constexpr int LPW = 32 / LW;
  constexpr int IDS = 4 * LPW;
  constexpr uint32_t H = NIB ? 0x88888888u : 0x80808080u;
  const uint32_t D = NIB ? (16u - L) * 0x11111111u : (256u - L) * 0x01010101u;
  const uint32_t K = (8u - L) * 0x11111111u;
  const uint4* t4 = reinterpret_cast<const uint4*>(tab);
  const int nvec = (valid + IDS - 1) / IDS;
  const int lane = threadIdx.x & 31;
  const uint32_t lt = (1u << lane) - 1u;
  auto any_hit = [&](const uint4 v) -> bool {
    if (SMALL) return ((((v.x + K) | (v.y + K)) | ((v.z + K) | (v.w + K))) & H) != 0u;
    return ((lanes_ge<NIB>(v.x, D) | lanes_ge<NIB>(v.y, D)) | (lanes_ge<NIB>(v.z, D) | lanes_ge<NIB>(v.w, D))) != 0u;
  };
  for (int v0 = (threadIdx.x - lane) * CP_VPL; v0 < nvec; v0 += NT * CP_VPL) {
    bool h[CP_VPL];
    uint32_t b[CP_VPL];
    int tot = 0;
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      const int vi = v0 + e * 32 + lane;
      h[e] = vi < nvec && any_hit(t4[vi]);
    }
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      b[e] = __ballot_sync(0xffffffffu, h[e]);
      tot += __popc(b[e]);
    }
    if (tot == 0) continue;
    int base = 0;
    if (lane == 0) base = atomicAdd(rfill, tot);
    base = __shfl_sync(0xffffffffu, base, 0);
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      const int at = base + __popc(b[e] & lt);
      if (h[e] && at < rcap) rec[at] = (uint16_t)(v0 + e * 32 + lane);
      base += __popc(b[e]);
    }
  }
  __syncthreads();
  const int R = *rfill;
  if (R > rcap) return false;
  for (int r = threadIdx.x; r < R; r += NT) {
    const int vi = rec[r];
    const uint4 v = t4[vi];
    uint32_t mm = SMALL ? vec_hits_small(v, K, IDS) : vec_hits<NIB>(v, D, IDS);
    uint32_t pos = (uint32_t)atomicAdd(fill, (int)__popc(mm));
    const uint32_t idb = (uint32_t)(id0 + (int64_t)vi * IDS);
    while (mm) {
      const int bb = 31 - __clz(mm);
      mm ^= 1u << bb;
      const int u = LW - 1 - (bb & (LW - 1));
      dst[pos++] = idb + (uint32_t)(u * LPW + bb / LW);
    }
  }
  return true;
}

// Global-mode spill: the ids of a chunk table with score >= 2 as packed
// records (chunk position << 8 | score), unordered, CP_VPL vectors per lane
// per warp step as above.  The emit sweep filters them at the query's level
// L >= 2 instead of re-reading the whole table (a query's candidates are a
// small fraction of the ids it touched).  *fill ends = record count.
template <int NT, bool NIB>
__device__ void compact_records(const uint8_t* tab, int valid, uint32_t* dst, int* fill) {
  constexpr int LW = NIB ? 4 : 8;
  constexpr int LPW = 32 / LW;
  constexpr int IDS = 4 * LPW;
  constexpr uint32_t MASK = (1u << LW) - 1u;
  const uint32_t D = NIB ? 14u * 0x11111111u : 254u * 0x01010101u;   // lanes >= 2
  const uint4* t4 = reinterpret_cast<const uint4*>(tab);
  const int nvec = (valid + IDS - 1) / IDS;
  const int lane = threadIdx.x & 31;
  for (int v0 = (threadIdx.x - lane) * CP_VPL; v0 < nvec; v0 += NT * CP_VPL) {
    uint4 w[CP_VPL];
    uint32_t m[CP_VPL];
    uint32_t c = 0;
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      const int vi = v0 + e * 32 + lane;
      w[e] = vi < nvec ? t4[vi] : make_uint4(0, 0, 0, 0);   // tables are zero past `valid`
      m[e] = vec_hits<NIB>(w[e], D, IDS);
      c += __popc(m[e]);
    }
    if (__ballot_sync(0xffffffffu, c != 0u) == 0u) continue;
    uint32_t pos = warp_reserve(c, fill);
#pragma unroll
    for (int e = 0; e < CP_VPL; ++e) {
      const uint32_t pos0 = (uint32_t)(v0 + e * 32 + lane) * IDS;
      uint32_t mm = m[e];
      while (mm) {
        const int b = 31 - __clz(mm);
        mm ^= 1u << b;
        const int u = LW - 1 - (b & (LW - 1));
        const int ln = b / LW;
        const uint32_t wu = u == 0 ? w[e].x : u == 1 ? w[e].y : u == 2 ? w[e].z : w[e].w;
        dst[pos++] = ((pos0 + (uint32_t)(u * LPW + ln)) << 8) | ((wu >> (ln * LW)) & MASK);
      }
    }
  }
}

// Alg. 5 (engine.py:239-249) on a histogram fetched through `get(level)`.
template <typename Get>
__device__ __forceinline__ int alg5(Get get, int n_sub, double budget, int64_t& cand) {
  int L = n_sub;
  cand = 0;
  for (int j = n_sub; j >= 0; --j) {
    const int64_t h = get(j);
    cand += h;
    if ((double)h <= __dsub_rn(budget, (double)cand)) L -= 1; else break;
  }
  return L < 0 ? 0 : L;
}

// ------------------------------------------------- cluster-fused count/select
// Candidates of a query live in per-CTA segments (segment q*S + rank); the
// final top-k breaks distance ties by id, so segment order is irrelevant.
__device__ int g_count_dbg = 0;   // timing experiments only (TACO_COUNT_DBG): 1 skip counting, 2 skip compaction, 4 skip the cluster exchange

template <bool NIB>
__global__ void __launch_bounds__(CT_THREADS, 3) k_count_cluster(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ ids, const uint32_t* __restrict__ offs, int n_sub, int K2, int64_t n,
    int64_t nchunks, int64_t chunk, double budget, uint32_t* __restrict__ cand, int64_t cand_cap,
    int64_t* __restrict__ flags, int64_t* __restrict__ sbase, int64_t* __restrict__ scnt,
    int64_t* __restrict__ cnum, int32_t* __restrict__ lvl) {
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ CountSmem S;
  __shared__ int s_L;
  __shared__ int64_t s_base, s_cnt;
  cg::cluster_group cluster = cg::this_cluster();
  const int rank = (int)cluster.block_rank();
  const int csz = (int)cluster.num_blocks();
  const int64_t q = blockIdx.y;
  const int64_t c = rank;
  const int tid = threadIdx.x;
  const int64_t base = c * chunk;
  const int valid = (int)max((int64_t)0, min(chunk, n - base));
  uint4* t4 = reinterpret_cast<uint4*>(table);
  const int tbytes = (int)(NIB ? chunk / 2 : chunk);
  const int dbg = g_count_dbg;
  for (int i = tid; i < tbytes / 16; i += CT_THREADS) t4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  if (!(dbg & 1))
    count_chunk<NIB>(pops, npop, cap, ids, offs, (size_t)nchunks * K2 + 1, n_sub, K2, n, c, q, base, table, S);
  else {
    for (int i = tid; i < 257; i += CT_THREADS) S.ge[i] = 0;
    __syncthreads();
  }
  chunk_levels(table, valid, n_sub, S);
  if (!(dbg & 4)) {
    cluster.sync();   // every CTA's level histogram is final
    // cluster-wide histogram: one level per thread, the csz remote reads in parallel
    for (int l = tid; l <= n_sub; l += CT_THREADS) {
      int h = 0;
      for (int r = 0; r < csz; ++r) h += cluster.map_shared_rank(S.lh, r)[l];
      S.ge[l] = h;
    }
  } else {
    for (int l = tid; l <= n_sub; l += CT_THREADS) S.ge[l] = S.lh[l] * csz;
  }
  // done reading remote shared memory: arrive now, wait only before exiting
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
  if (tid == 0) {
    int64_t cands = 0;
    const int L = alg5([&](int l) { return (int64_t)S.ge[l]; }, n_sub, budget, cands);
    int64_t mine = 0;
    for (int l = L; l <= n_sub; ++l) mine += S.lh[l];
    if (dbg & 3) mine = 0;   // timing experiment: no candidates
    const int64_t b = (int64_t)atomicAdd((unsigned long long*)&flags[3], (unsigned long long)mine);
    if (b + mine > cand_cap) flags[1] = 1;
    s_L = L;
    s_base = b;
    s_cnt = mine;
    S.batches = 0;   // fill counter of the compaction
    sbase[q * csz + rank] = b;
    scnt[q * csz + rank] = mine;
    if (rank == 0) {
      cnum[q] = cands;
      lvl[q] = L;
    }
  }
  __syncthreads();
  if (s_base + s_cnt <= cand_cap && !(dbg & 3))
    compact_unordered<CT_THREADS, NIB>(table, valid, (uint32_t)s_L, base, cand + s_base, &S.batches);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");   // nobody reads my histogram any more
}

// ------------------------------------------- encoded-CSR cluster count (N_s <= 16)
// Same contract as k_count_cluster (nchunks CTAs per query, one id chunk
// each), fed by the encoded CSR of build_count_csr: every (chunk, cell) slice
// is a run of 32-byte units of 8 entries (16-byte units of 4 in global mode),
// entry = table word byte offset << 6 | lane shift; padding entries have
// shift 32, so they add 0 (to a word of their own slice: EC_SPREAD) and read
// level 0.  Per entry: and (shift), lea (address), shl (increment), atom, shr
// (old lane), shl + funnel shift (tally field), add -- no predicates, no
// per-id address arithmetic.  Padding entries' level-0 tallies are subtracted
// (their count rides in the top 3 bits of the slice offsets).  Feeds:
//  - k_count_pg / k_count_enc: all threads stage the popped slices' unit
//    indices in shared memory (one store per unit), then consume them with
//    direct 16-byte loads -- lane pairs share a unit (EC_PAIR), a thread has
//    two groups of 4 entries in flight;
//  - k_count_tma: a producer warp streams each slice with one cp.async.bulk
//    into an mbarrier ring (TACO_COUNT_FEED=tma; measured slower: thousands
//    of 100-200 byte bulk copies per CTA).
#ifndef EC_PP
#define EC_PP 1      // ping-pong lookahead registers in the consume loop
#endif
#ifndef EC_SPREAD
#define EC_SPREAD 1  // padding entries point at a word of their own slice (not all at word 0)
#endif
#ifndef EC_SKIPHALF
#define EC_SKIPHALF 0   // (with EC_PAIR) a lane whose half unit is all padding applies nothing
#endif
#ifndef EC_SCAN2
#define EC_SCAN2 1      // the slice-unit scan with two barriers (block_excl_scan2)
#endif
#ifndef EC_STAGE_UNROLL
#define EC_STAGE_UNROLL 0
#endif
#ifndef EC_NPOP_AHEAD
#define EC_NPOP_AHEAD 0   // k_count_pg reads the next query's pop counts a query ahead (measured: 4.00 vs 3.98 ms without)
#endif
#ifndef EC_PREFETCH
#define EC_PREFETCH 0   // k_count_pg: the next query's slice lookups are issued under this query's epilogue
#endif
#ifndef EC_PAIR
#define EC_PAIR 1    // lane pairs split a 32-byte unit (16 sectors per warp load)
#endif
#ifndef EC_FASTGE
#define EC_FASTGE 1 // scores <= 8: lanes >= L as (w + (8 - L) * 0x11111111) & 0x88888888
#endif
#ifndef EC_RELAX
#define EC_RELAX 1   // relaxed cluster arrive after the histogram gather
#endif
constexpr uint32_t EC_SENT = 32u;
constexpr uint32_t EC_GMASK = 0x1FFFFFFFu;   // unit offset bits of coffs (top 3 bits: padding count)

__device__ __forceinline__ uint32_t shl_clamp(uint32_t v, uint32_t s) {
  uint32_t r;
  asm("shl.b32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
  return r;
}
__device__ __forceinline__ uint32_t shr_clamp(uint32_t v, uint32_t s) {
  uint32_t r;
  asm("shr.u32 %0, %1, %2;" : "=r"(r) : "r"(v), "r"(s));
  return r;
}
// one group of 4 encoded entries into the table at shared address tsg;
// ev/od collect "left level r" in 8-bit fields (levels 0,2,4,6 / 1,3,5,7)
#ifndef EC_PRED
#define EC_PRED 0    // padding entries skip their atomic (predicated) instead of adding 0
#endif
__device__ __forceinline__ uint32_t smem_atomic_add_unless_pad(uint32_t addr, uint32_t v, uint32_t s) {
  uint32_t old;
  asm volatile(
      "{\n .reg .pred p;\n setp.ne.u32 p, %3, 32;\n mov.u32 %0, 0;\n @p atom.shared::cta.add.u32 %0, [%1], %2;\n}"
      : "=r"(old) : "r"(addr), "r"(v), "r"(s) : "memory");
  return old;
}
__device__ __forceinline__ void apply_group(const uint4 e, uint32_t tsg, uint32_t& ev, uint32_t& od) {
  const uint32_t s0 = e.x & 63u, s1 = e.y & 63u, s2 = e.z & 63u, s3 = e.w & 63u;
#if EC_PRED
  const uint32_t o0 = smem_atomic_add_unless_pad(tsg + (e.x >> 6), shl_clamp(1u, s0), s0);
  const uint32_t o1 = smem_atomic_add_unless_pad(tsg + (e.y >> 6), shl_clamp(1u, s1), s1);
  const uint32_t o2 = smem_atomic_add_unless_pad(tsg + (e.z >> 6), shl_clamp(1u, s2), s2);
  const uint32_t o3 = smem_atomic_add_unless_pad(tsg + (e.w >> 6), shl_clamp(1u, s3), s3);
#else
  const uint32_t o0 = smem_atomic_add(tsg + (e.x >> 6), shl_clamp(1u, s0));
  const uint32_t o1 = smem_atomic_add(tsg + (e.y >> 6), shl_clamp(1u, s1));
  const uint32_t o2 = smem_atomic_add(tsg + (e.z >> 6), shl_clamp(1u, s2));
  const uint32_t o3 = smem_atomic_add(tsg + (e.w >> 6), shl_clamp(1u, s3));
#endif
  // 4-bit field r (r <= 7: the funnel shift wraps mod 32)
  const uint32_t u4 = __funnelshift_l(0u, 1u, shr_clamp(o0, s0) << 2) + __funnelshift_l(0u, 1u, shr_clamp(o1, s1) << 2) +
                      __funnelshift_l(0u, 1u, shr_clamp(o2, s2) << 2) + __funnelshift_l(0u, 1u, shr_clamp(o3, s3) << 2);
  ev += u4 & 0x0F0F0F0Fu;
  od += (u4 >> 4) & 0x0F0F0F0Fu;
}

// N_s 9..16: old values up to 15 -> 16 tally levels, 4-bit fields in two
// words (r < 8: lo, else hi; the clamped shifts drop the other word's share).
// Works for nibble and byte lanes (the lane value is < 16 either way).
__device__ __forceinline__ void apply_group_w(const uint4 e, uint32_t tsg, uint32_t& ev, uint32_t& od,
                                              uint32_t& evh, uint32_t& odh) {
  const uint32_t s0 = e.x & 63u, s1 = e.y & 63u, s2 = e.z & 63u, s3 = e.w & 63u;
  const uint32_t o0 = smem_atomic_add(tsg + (e.x >> 6), shl_clamp(1u, s0));
  const uint32_t o1 = smem_atomic_add(tsg + (e.y >> 6), shl_clamp(1u, s1));
  const uint32_t o2 = smem_atomic_add(tsg + (e.z >> 6), shl_clamp(1u, s2));
  const uint32_t o3 = smem_atomic_add(tsg + (e.w >> 6), shl_clamp(1u, s3));
  const uint32_t t0 = (shr_clamp(o0, s0) & 15u) << 2, t1 = (shr_clamp(o1, s1) & 15u) << 2,
                 t2 = (shr_clamp(o2, s2) & 15u) << 2, t3 = (shr_clamp(o3, s3) & 15u) << 2;
  const uint32_t lo = shl_clamp(1u, t0) + shl_clamp(1u, t1) + shl_clamp(1u, t2) + shl_clamp(1u, t3);
  const uint32_t hi = shl_clamp(1u, t0 - 32u) + shl_clamp(1u, t1 - 32u) + shl_clamp(1u, t2 - 32u) +
                      shl_clamp(1u, t3 - 32u);
  ev += lo & 0x0F0F0F0Fu;
  od += (lo >> 4) & 0x0F0F0F0Fu;
  evh += hi & 0x0F0F0F0Fu;
  odh += (hi >> 4) & 0x0F0F0F0Fu;
}

template <int NT>
struct EncSmem {
  uint64_t full[8], empty[8];   // k_count_tma ring
  int cnt[8];
  int pads, fill, L, ptot, rfill;
  int64_t sbase, scnt;
  uint32_t wtot[NT / 32];
  int jpref[17];
  int ge[33];   // the encoded kernels count N_s <= 16: 17 levels (the spare bytes went into the staging, EcCfg::GC)
  int lh[32];
};
constexpr int EC_LEVELS = 33;

template <int NT, bool WIDE>
__device__ __forceinline__ void enc_levels(Tally& T, const uint8_t* table, int valid, int n_sub, EncSmem<NT>& S);

// tallies -> level histogram, cluster exchange, Alg. 5, compaction (the
// k_count_cluster epilogue for NT threads).  Thread 0 reserves the CTA's
// candidate segment with one global atomic; while it is in flight the CTA
// compacts into `stage` (shared memory, scap ids) and copies the segment out
// coalesced once the base is known (direct global writes when it is larger).
// Alg. 5 on the group's level histogram S.ge, the CTA's candidate segment
// and its compaction (the common tail of the encoded kernels' epilogues).
// Thread 0 reserves the segment with one global atomic; while it is in
// flight the CTA compacts into `stage` (shared memory, scap ids) and copies
// the segment out coalesced once the base is known (direct global writes
// when it is larger).
template <int NT, bool NIB, bool WIDE>
__device__ __forceinline__ void enc_finish(const uint8_t* table, int valid, int n_sub, EncSmem<NT>& S, int rank, int csz,
                                           int64_t q, int64_t base, double budget, uint32_t* __restrict__ cand,
                                           int64_t cand_cap, int64_t* __restrict__ flags, int64_t* __restrict__ sbase,
                                           int64_t* __restrict__ scnt, int64_t* __restrict__ cnum,
                                           int32_t* __restrict__ lvl, uint32_t* stage, int scap) {
  const int tid = threadIdx.x;
  int64_t b = 0;
  if (tid == 0) {
    int64_t cands = 0;
    const int L = alg5([&](int l) { return (int64_t)S.ge[l]; }, n_sub, budget, cands);
    int64_t mine = 0;
    for (int l = L; l <= n_sub; ++l) mine += S.lh[l];
    b = (int64_t)atomicAdd((unsigned long long*)&flags[3], (unsigned long long)mine);   // used after the scan
    S.L = L;
    S.scnt = mine;
    S.fill = 0;
    S.rfill = 0;
    if (rank == 0) {
      cnum[q] = cands;
      lvl[q] = L;
    }
    if (mine > scap) S.sbase = b;   // direct path: the base is needed before the scan
  }
  __syncthreads();
  const int64_t mine = S.scnt;
  constexpr int IDSV = NIB ? 32 : 16;   // ids per 16-byte table vector
  if (EC_TWOPHASE && S.L >= 1 && mine <= scap / 2) {
    // candidates in stage[0, scap/2), vector records (u16) in the upper half; every record
    // holds at least one candidate, so there are at most `mine` of them
    compact_two_phase<NT, NIB, NIB && !WIDE && EC_FASTGE != 0>(table, valid, (uint32_t)S.L, base, stage, &S.fill,
                                                              reinterpret_cast<uint16_t*>(stage + scap / 2), scap,
                                                              &S.rfill);
    if (tid == 0) S.sbase = b;
    __syncthreads();
    const int64_t sb = S.sbase;
    if (sb + mine <= cand_cap)
      for (int i = tid; i < (int)mine; i += NT) cand[sb + i] = stage[i];
  } else if (EC_TWOPHASE && S.L >= 1 && (valid + IDSV - 1) / IDSV <= 2 * scap) {
    // a large segment: the records take the whole staging area (one per table vector at most) and
    // phase 2 writes the ids straight to the segment (its base is back long before phase 1 ends)
    if (tid == 0) S.sbase = b;
    __syncthreads();
    if (S.sbase + mine <= cand_cap)
      compact_two_phase<NT, NIB, NIB && !WIDE && EC_FASTGE != 0>(table, valid, (uint32_t)S.L, base, cand + S.sbase,
                                                                &S.fill, reinterpret_cast<uint16_t*>(stage), 2 * scap,
                                                                &S.rfill);
  } else if (mine <= scap) {
    compact_unordered<NT, NIB, NIB && !WIDE && EC_FASTGE != 0>(table, valid, (uint32_t)S.L, base, stage, &S.fill);
    if (tid == 0) S.sbase = b;
    __syncthreads();
    const int64_t sb = S.sbase;
    if (sb + mine <= cand_cap)
      for (int i = tid; i < (int)mine; i += NT) cand[sb + i] = stage[i];
  } else if (S.sbase + mine <= cand_cap) {
    compact_unordered<NT, NIB, NIB && !WIDE && EC_FASTGE != 0>(table, valid, (uint32_t)S.L, base, cand + S.sbase,
                                                              &S.fill);
  }
  if (tid == 0) {
    if (S.sbase + mine > cand_cap) flags[1] = 1;
    sbase[q * csz + rank] = S.sbase;
    scnt[q * csz + rank] = mine;
  }
}

// tallies -> level histogram, cluster exchange over DSMEM, then enc_finish
// (the k_count_cluster epilogue for NT threads).
template <int NT, bool NIB = true, bool WIDE = false>
__device__ __forceinline__ void enc_epilogue(Tally& T, const uint8_t* table, int valid, int n_sub, EncSmem<NT>& S,
                             cg::cluster_group& cluster, int64_t q, int64_t base, double budget,
                             uint32_t* __restrict__ cand, int64_t cand_cap, int64_t* __restrict__ flags,
                             int64_t* __restrict__ sbase, int64_t* __restrict__ scnt, int64_t* __restrict__ cnum,
                             int32_t* __restrict__ lvl, uint32_t* stage, int scap) {
  const int tid = threadIdx.x;
  const int rank = (int)cluster.block_rank();
  const int csz = (int)cluster.num_blocks();
  enc_levels<NT, WIDE>(T, table, valid, n_sub, S);
  cluster.sync();   // every CTA's level histogram is final
  for (int l = tid; l <= n_sub; l += NT) {
    int h = 0;
    for (int r = 0; r < csz; ++r) h += cluster.map_shared_rank(S.lh, r)[l];
    S.ge[l] = h;
  }
  if (EC_RELAX)   // publishes nothing: only "done reading the remote histograms"
    asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");
  else
    asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");
  __syncthreads();
  enc_finish<NT, NIB, WIDE>(table, valid, n_sub, S, rank, csz, q, base, budget, cand, cand_cap, flags, sbase, scnt, cnum,
                            lvl, stage, scap);
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// The same epilogue for a software group of csz CTAs (k_count_pg): every CTA
// publishes its level histogram as value + 1 in its own zero-initialised slots
// of xch[q][rank][level] and polls the group's slots until they are nonzero
// (each word validates itself: no fence, no counter, one store trip and one
// load trip).
__device__ __forceinline__ void st_relaxed_gpu(int32_t* p, int32_t v) {
  asm volatile("st.relaxed.gpu.global.s32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ int32_t ld_relaxed_gpu(const int32_t* p) {
  int32_t v;
  asm volatile("ld.relaxed.gpu.global.s32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
template <int NT, bool NIB = true, bool WIDE = false>
__device__ __forceinline__ void enc_epilogue_sw(const uint8_t* table, int valid, int n_sub, EncSmem<NT>& S,
                             int rank, int csz, int64_t q, int64_t base, double budget, int32_t* __restrict__ xch,
                             uint32_t* __restrict__ cand, int64_t cand_cap, int64_t* __restrict__ flags,
                             int64_t* __restrict__ sbase, int64_t* __restrict__ scnt, int64_t* __restrict__ cnum,
                             int32_t* __restrict__ lvl, uint32_t* stage, int scap) {
  const int tid = threadIdx.x;
  const int LV = n_sub + 1;   // S.lh is final (enc_levels, run by the caller, ends with a barrier)
  if (csz > 1 && (g_count_dbg & 4)) {   // timing experiment: no exchange (wrong levels)
    if (tid < LV) S.ge[tid] = S.lh[tid] * csz;
  } else if (csz > 1) {
    int32_t* X = xch + (size_t)q * csz * LV;
    if (tid < LV) {
      st_relaxed_gpu(&X[rank * LV + tid], S.lh[tid] + 1);
      S.ge[tid] = 0;
    }
    __syncthreads();
    for (int i = tid; i < csz * LV; i += NT) {
      int32_t v;
      while ((v = ld_relaxed_gpu(&X[i])) == 0) __nanosleep(20);
      atomicAdd(&S.ge[i % LV], v - 1);
    }
  } else if (tid < LV) {
    S.ge[tid] = S.lh[tid];
  }
  __syncthreads();
  enc_finish<NT, NIB, WIDE>(table, valid, n_sub, S, rank, csz, q, base, budget, cand, cand_cap, flags, sbase, scnt, cnum,
                            lvl, stage, scap);
}

// pop g of query q (flattened over subspaces; jpref = the subspaces' pop
// prefix, in registers): its slice's (first unit, unit count, padding) in
// chunk c and its subspace js
template <int JM>   // subspaces held in jpref (>= N_s)
__device__ __forceinline__ void enc_slice(const uint16_t* __restrict__ pops, const uint32_t* __restrict__ coffs,
                                          size_t offs_len, int cap, int n_sub, int K2, int64_t q, int64_t c,
                                          const int (&jpref)[JM], int g, uint32_t& g0, uint32_t& ng, uint32_t& pad,
                                          uint32_t& js) {
  int j = 0, jb = 0;
#pragma unroll
  for (int jj = 1; jj < JM; ++jj)
    if (jj < n_sub && g >= jpref[jj]) {
      j = jj;
      jb = jpref[jj];
    }
  const int cell = pops[((size_t)q * n_sub + j) * cap + (g - jb)];
  const uint32_t* O = coffs + (size_t)j * offs_len + (size_t)c * K2;
  const uint32_t a = __ldg(O + cell), b = __ldg(O + cell + 1);
  g0 = a & EC_GMASK;
  ng = (b & EC_GMASK) - g0;
  pad = b >> 29;
  js = (uint32_t)j;
}

// k_count_enc<NT, MINB>: NT threads, MINB CTAs per SM.  Per batch of NT *
// EC_PER popped slices: each thread looks up EC_PER slices (pops -> unit
// range), one block scan places their units, and rounds of EC_GC(NT) unit
// indices are staged in shared memory and consumed by all threads (unit t,
// t + NT, ...; one unit of load lookahead).
template <int NT>
struct EcCfg {
  static constexpr int PER = NT >= 512 ? 2 : 4;   // pops per thread per batch
  // staged units per round: 10 per thread at 256 threads (10 KiB next to the 64 KiB table: three
  // CTAs per SM; 80 entries per thread per round keep the tallies' 8-bit fields), else 8
  static constexpr int GC = (NT == 256 ? 10 : 8) * NT;
};

// k_count_pg looks the NEXT query's first batch of popped slices up while
// the current query is in its epilogue (the pops -> coffs chain is two
// dependent global loads): enc_pre_cells reads the pop prefix and the cells,
// enc_pre_offs the cells' unit offsets; the count phase then starts from
// registers.
template <int PER>
struct EncPre {
  uint32_t jc[PER];        // subspace << 16 | cell (0xFFFFFFFF: no slice)
  uint32_t a[PER], b[PER]; // coffs[cell], coffs[cell + 1]
};
template <int NT, bool WIDE>
__device__ __forceinline__ void enc_pre_cells(const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop,
                                              int cap, int n_sub, int64_t q, EncPre<EcCfg<NT>::PER>& P) {
  constexpr int JM = WIDE ? 16 : 8, PER = EcCfg<NT>::PER;
  int jp[JM];
  int acc = 0;
#pragma unroll
  for (int jj = 0; jj < JM; ++jj) {
    jp[jj] = acc;
    if (jj < n_sub) acc += min(__ldg(npop + q * n_sub + jj), cap);
  }
#pragma unroll
  for (int u = 0; u < PER; ++u) {
    const int g = u * NT + (int)threadIdx.x;
    P.jc[u] = 0xFFFFFFFFu;
    if (g < acc) {
      int j = 0, jb = 0;
#pragma unroll
      for (int jj = 1; jj < JM; ++jj)
        if (jj < n_sub && g >= jp[jj]) {
          j = jj;
          jb = jp[jj];
        }
      P.jc[u] = ((uint32_t)j << 16) | pops[((size_t)q * n_sub + j) * cap + (g - jb)];
    }
  }
}
template <int NT>
__device__ __forceinline__ void enc_pre_offs(const uint32_t* __restrict__ coffs, size_t offs_len, int K2, int64_t c,
                                             EncPre<EcCfg<NT>::PER>& P) {
#pragma unroll
  for (int u = 0; u < EcCfg<NT>::PER; ++u) {
    P.a[u] = P.b[u] = 0u;
    if (P.jc[u] != 0xFFFFFFFFu) {
      const uint32_t* O = coffs + (size_t)(P.jc[u] >> 16) * offs_len + (size_t)c * K2 + (P.jc[u] & 0xFFFFu);
      P.a[u] = __ldg(O);
      P.b[u] = __ldg(O + 1);
    }
  }
}

// The counting phase of the encoded kernels for (query q, chunk c): table
// zeroed and filled, tallies in T, padding entries counted in S.pads.  UW =
// 16-byte words per unit (2: cluster mode's 8-entry units, 1: global mode's
// 4-entry units).  Staging: gaddr[EcCfg<NT>::GC].
template <int NT, int UW, bool WIDE = false, bool PRE = false>
__device__ __forceinline__ void enc_count_phase(const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop,
                                                int cap, const uint32_t* __restrict__ cenc, size_t cstride,
                                                const uint32_t* __restrict__ coffs, int n_sub, int K2, int64_t nchunks,
                                                int64_t q, int64_t c, int tbytes, uint8_t* table, uint32_t* gaddr,
                                                EncSmem<NT>& S, Tally& T,
                                                const EncPre<EcCfg<NT>::PER>* pre = nullptr, int np_pre = -1) {
  constexpr int PER = EcCfg<NT>::PER, GC = EcCfg<NT>::GC, EU = 4 * UW;
  const int tid = threadIdx.x;
  const uint4* E4 = reinterpret_cast<const uint4*>(cenc);
  const uint32_t jstride = (uint32_t)(cstride / EU);                // units per subspace
  const size_t offs_len = (size_t)nchunks * K2 + 1;
  uint4* t4 = reinterpret_cast<uint4*>(table);
  // the subspaces' pop counts: read before the table is zeroed (the load is in flight
  // meanwhile), or handed over by k_count_pg, which reads them a query ahead (np_pre >= 0)
  int np_raw = np_pre;
  if (np_pre < 0 && tid < n_sub) np_raw = npop[q * n_sub + tid];
  for (int i = tid; i < tbytes / 16; i += NT) t4[i] = make_uint4(0, 0, 0, 0);
  for (int i = tid; i < EC_LEVELS; i += NT) S.ge[i] = 0;
  if (tid < 32) {
    const int np = tid < n_sub ? min(np_raw, cap) : 0;
    int x = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (tid >= o) x += y;
    }
    if (tid <= n_sub) S.jpref[tid] = x - np;   // jpref[n_sub] = total
    if (tid == 0) S.pads = 0;
  }
  __syncthreads();
  const int P_all = S.jpref[n_sub];
  constexpr int JM = WIDE ? 16 : 8;
  int jp[JM];
#pragma unroll
  for (int jj = 0; jj < JM; ++jj) jp[jj] = S.jpref[jj];
  const uint32_t tsg = smem_u32(table);
  uint32_t ev = 0, od = 0, evh = 0, odh = 0;
  int pads = 0;
  for (int b0 = 0; b0 < P_all; b0 += NT * PER) {
    uint32_t ga[PER], ng[PER];   // unit index of the slice start, unit count
    uint32_t my = 0;
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      const int g = b0 + u * NT + tid;
      ga[u] = 0;
      ng[u] = 0;
      if (PRE && b0 == 0) {   // looked up during the previous query's epilogue
        const uint32_t u0 = pre->a[u] & EC_GMASK;
        ng[u] = (pre->b[u] & EC_GMASK) - u0;
        ga[u] = (pre->jc[u] >> 16) * jstride + u0;   // no slice: a = b = 0, and ga is never used
        pads += (int)(pre->b[u] >> 29);
      } else if (g < P_all) {
        uint32_t u0, pad, j;
        enc_slice(pops, coffs, offs_len, cap, n_sub, K2, q, c, jp, g, u0, ng[u], pad, j);
        ga[u] = j * jstride + u0;
        pads += (int)((EC_PAIR && EC_SKIPHALF && UW == 2) ? pad & 3u : pad);
      }
      my += ng[u];
    }
    uint32_t tot;
    uint32_t run = EC_SCAN2 ? block_excl_scan2<NT>(my, S.wtot, tot) : block_excl_scan<NT>(my, S.wtot, tot);
    uint32_t gb[PER];
#pragma unroll
    for (int u = 0; u < PER; ++u) {
      gb[u] = run;
      run += ng[u];
    }
    for (uint32_t r0 = 0; r0 < tot; r0 += GC) {
      const uint32_t r1 = min(tot, r0 + (uint32_t)GC);
#pragma unroll
      for (int u = 0; u < PER; ++u) {
        const uint32_t k0 = max(gb[u], r0), k1 = min(gb[u] + ng[u], r1);
#if EC_STAGE_UNROLL == 2
#pragma unroll 2
#elif EC_STAGE_UNROLL == 4
#pragma unroll 4
#endif
        for (uint32_t k = k0; k < k1; ++k) gaddr[k - r0] = ga[u] + (k - gb[u]);
      }
      __syncthreads();
      const int nr = (int)(r1 - r0);
      // one unit of lookahead: unit k + NT loads while unit k is applied
      uint4 a0, a1, b0v, b1v;
      auto fetch = [&](int kk, uint4& x0, uint4& x1) {
        if (kk < nr) {
          const uint4* src = E4 + UW * (size_t)gaddr[kk];
          x0 = src[0];
          if (UW == 2) x1 = src[1];
        }
      };
      auto apply = [&](const uint4& x0, const uint4& x1) {
        if (WIDE) {
          apply_group_w(x0, tsg, ev, od, evh, odh);
          if (UW == 2) apply_group_w(x1, tsg, ev, od, evh, odh);
        } else {
          apply_group(x0, tsg, ev, od);
          if (UW == 2) apply_group(x1, tsg, ev, od);
        }
      };
      int k = tid;
      if (EC_PAIR && UW == 2) {
        // lane pairs share a 32-byte unit (one sector per pair: a warp load
        // touches 16 sectors instead of 32 half sectors); a thread's two
        // groups in flight are groups k and k + NT of the round
        const int G = 2 * nr;
        auto fetch2 = [&](int kk, uint4& x0, uint4& x1) {
          if (kk < G) x0 = E4[2 * (size_t)gaddr[kk >> 1] + (kk & 1)];
          if (kk + NT < G) x1 = E4[2 * (size_t)gaddr[(kk + NT) >> 1] + (kk & 1)];
        };
        auto apply1 = [&](const uint4& x) {
          if (EC_SKIPHALF && (x.x & 63u) == EC_SENT) return;   // an all-padding second half
          if (WIDE) apply_group_w(x, tsg, ev, od, evh, odh);
          else apply_group(x, tsg, ev, od);
        };
        fetch2(k, a0, a1);
        while (k < G) {
          fetch2(k + 2 * NT, b0v, b1v);
          apply1(a0);
          if (k + NT < G) apply1(a1);
          k += 2 * NT;
          if (k >= G) break;
          fetch2(k + 2 * NT, a0, a1);
          apply1(b0v);
          if (k + NT < G) apply1(b1v);
          k += 2 * NT;
        }
      } else if (EC_PP) {   // ping-pong registers: no moves between units
        fetch(k, a0, a1);
        while (k < nr) {
          fetch(k + NT, b0v, b1v);
          apply(a0, a1);
          k += NT;
          if (k >= nr) break;
          fetch(k + NT, a0, a1);
          apply(b0v, b1v);
          k += NT;
        }
      } else {
        fetch(k, a0, a1);
        for (; k < nr; k += NT) {
          fetch(k + NT, b0v, b1v);
          apply(a0, a1);
          a0 = b0v;
          a1 = b1v;
        }
      }
      T.add_round(ev, od);   // <= 4 UW per unit, <= 8 units per thread per round: 8-bit fields
      if (WIDE) T.add_round_hi(evh, odh);
      ev = od = evh = odh = 0;
      __syncthreads();
    }
  }
  if (pads) atomicAdd(&S.pads, pads);   // read after enc_levels' first barrier (every caller runs it next)
}

// tallies -> the chunk's level histogram S.ge / S.lh (packed reduction as in
// enc_epilogue; padding entries taken off level 0)
template <int NT, bool WIDE>
__device__ __forceinline__ void enc_levels(Tally& T, const uint8_t* table, int valid, int n_sub, EncSmem<NT>& S) {
  const int tid = threadIdx.x, lane = tid & 31;
  Tally P = T;
  constexpr uint64_t HI3 = 0xE000E000E000E000ull;
  const uint64_t any = P.a0 | P.a1 | (WIDE ? P.a2 | P.a3 : 0ull);
  if (!__any_sync(0xffffffffu, (any & HI3) != 0)) {
#pragma unroll
    for (int o = 4; o > 0; o >>= 1) {
      P.a0 += __shfl_xor_sync(0xffffffffu, P.a0, o);
      P.a1 += __shfl_xor_sync(0xffffffffu, P.a1, o);
      if (WIDE) {
        P.a2 += __shfl_xor_sync(0xffffffffu, P.a2, o);
        P.a3 += __shfl_xor_sync(0xffffffffu, P.a3, o);
      }
    }
    if ((lane & 7) == 0)
      for (int l = 1; l <= n_sub; ++l) {
        const int x = P.level2(l - 1);
        if (x) atomicAdd(&S.ge[l], x);
      }
  } else {
    for (int l = 1; l <= n_sub; ++l) {
      int x = T.level2(l - 1);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) x += __shfl_xor_sync(0xffffffffu, x, o);
      if (lane == 0 && x) atomicAdd(&S.ge[l], x);
    }
  }
  __syncthreads();
  // level histogram from the tallies: lh[l] = #(score >= l) - #(score >= l + 1); the padding
  // entries were tallied as leaving level 0, so they come off #(score >= 1)
  for (int l = tid; l <= n_sub; l += NT) {
    const int g1 = S.ge[1] - S.pads;
    const int gl = l == 0 ? valid : (l == 1 ? g1 : S.ge[l]);
    const int gn = l == n_sub ? 0 : (l == 0 ? g1 : S.ge[l + 1]);
    S.lh[l] = gl - gn;
  }
  __syncthreads();
}

// NSC: N_s at compile time (0 = runtime); NIB: 4-bit lanes (else 8-bit, N_s = 16);
// WIDE: N_s > 8 (16 tally levels)
template <int NT, int MINB, int NSC = 0, bool NIB = true, bool WIDE = false>
__global__ void __launch_bounds__(NT, MINB) k_count_enc(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ cenc, size_t cstride, const uint32_t* __restrict__ coffs, int n_sub_rt, int K2,
    int64_t n, int64_t nchunks, int64_t chunk, double budget, uint32_t* __restrict__ cand, int64_t cand_cap,
    int64_t* __restrict__ flags, int64_t* __restrict__ sbase, int64_t* __restrict__ scnt,
    int64_t* __restrict__ cnum, int32_t* __restrict__ lvl) {
  const int n_sub = NSC ? NSC : n_sub_rt;
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ EncSmem<NT> S;
  cg::cluster_group cluster = cg::this_cluster();
  const int64_t q = blockIdx.y;
  const int64_t c = cluster.block_rank();
  const int64_t base = c * chunk;
  const int valid = (int)max((int64_t)0, min(chunk, n - base));
  const int tbytes = (int)(NIB ? chunk / 2 : chunk);
  uint32_t* gaddr = reinterpret_cast<uint32_t*>(table + tbytes);   // [GC] unit indices
  Tally T;
  enc_count_phase<NT, 2, WIDE>(pops, npop, cap, cenc, cstride, coffs, n_sub, K2, nchunks, q, c, tbytes, table,
                               gaddr, S, T);
  enc_epilogue<NT, NIB, WIDE>(T, table, valid, n_sub, S, cluster, q, base, budget, cand, cand_cap, flags, sbase, scnt, cnum,
                   lvl, gaddr, EcCfg<NT>::GC);
}

// k_count_pg: k_count_enc as a persistent kernel over SOFTWARE groups of
// nchunks CTAs (group = blockIdx.x / nchunks walks queries grp, grp + ngrp,
// ...).  A hardware cluster cannot span GPCs, so clusters of 8 (16) reach
// only 384 (336) of the 444 co-resident CTA slots of this kernel's shape
// (tools/mb_clusters.cu); groups synchronise through global memory instead
// (enc_epilogue_sw) and use every slot.  The grid never exceeds the
// co-resident capacity (cooperative launch), so a polling CTA's siblings are
// always running.
template <int NT, int MINB, int NSC = 0, bool NIB = true, bool WIDE = false>
__global__ void __launch_bounds__(NT, MINB) k_count_pg(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ cenc, size_t cstride, const uint32_t* __restrict__ coffs, int n_sub_rt, int K2,
    int64_t n, int64_t nchunks, int64_t chunk, double budget, uint32_t* __restrict__ cand, int64_t cand_cap,
    int64_t* __restrict__ flags, int64_t* __restrict__ sbase, int64_t* __restrict__ scnt,
    int64_t* __restrict__ cnum, int32_t* __restrict__ lvl, int64_t Q, int32_t* __restrict__ xch) {
  const int n_sub = NSC ? NSC : n_sub_rt;
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ EncSmem<NT> S;
  const int csz = (int)nchunks;
  const int grp = (int)(blockIdx.x / csz), ngrp = (int)(gridDim.x / csz);
  const int rank = (int)(blockIdx.x % csz);
  if (grp >= ngrp) return;
  const int64_t c = rank;
  const int64_t base = c * chunk;
  const int valid = (int)max((int64_t)0, min(chunk, n - base));
  const int tbytes = (int)(NIB ? chunk / 2 : chunk);
  uint32_t* gaddr = reinterpret_cast<uint32_t*>(table + tbytes);   // [GC] unit indices
  const size_t offs_len = (size_t)nchunks * K2 + 1;
  EncPre<EcCfg<NT>::PER> pre;
  if (EC_PREFETCH && grp < Q) {
    enc_pre_cells<NT, WIDE>(pops, npop, cap, n_sub, grp, pre);
    enc_pre_offs<NT>(coffs, offs_len, K2, c, pre);
  }
  int np_next = (EC_NPOP_AHEAD && grp < Q && (int)threadIdx.x < n_sub) ? npop[(int64_t)grp * n_sub + threadIdx.x] : 0;
  for (int64_t q = grp; q < Q; q += ngrp) {
    Tally T;
    const int np_now = EC_NPOP_AHEAD ? np_next : -1;
    const int64_t qn = q + ngrp;
    if (EC_NPOP_AHEAD && qn < Q && (int)threadIdx.x < n_sub) np_next = npop[qn * n_sub + threadIdx.x];
    enc_count_phase<NT, 2, WIDE, EC_PREFETCH != 0>(pops, npop, cap, cenc, cstride, coffs, n_sub, K2, nchunks, q, c,
                                                   tbytes, table, gaddr, S, T, &pre, np_now);
    if (EC_PREFETCH && qn < Q) enc_pre_cells<NT, WIDE>(pops, npop, cap, n_sub, qn, pre);
    enc_levels<NT, WIDE>(T, table, valid, n_sub, S);   // S.lh final (ends with a barrier)
    if (EC_PREFETCH && qn < Q) enc_pre_offs<NT>(coffs, offs_len, K2, c, pre);
    enc_epilogue_sw<NT, NIB, WIDE>(table, valid, n_sub, S, rank, csz, q, base, budget, xch, cand, cand_cap, flags,
                                   sbase, scnt, cnum, lvl, gaddr, EcCfg<NT>::GC);
    __syncthreads();   // the table and the staging are free for the next query
  }
}

// Global mode, sweep 1 on the encoded CSR (4-entry units): per (chunk,
// query) CTA the chunk's level histogram -> part, and its score >= 2 ids as
// packed records (k_count CNT_HIST's contract; the emit sweep and the
// recount are unchanged).
template <int NT, int MINB>
__global__ void __launch_bounds__(NT, MINB) k_count_genc(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ cenc, size_t cstride, const uint32_t* __restrict__ coffs, int n_sub, int K2,
    int64_t n, int64_t nchunks, int64_t chunk, uint8_t* __restrict__ scores, int32_t* __restrict__ part) {
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ EncSmem<NT> S;
  const int64_t c = blockIdx.x, q = blockIdx.y;
  const int64_t base = c * chunk;
  const int valid = (int)min(chunk, n - base);
  const int tbytes = (int)(chunk / 2);
  const int rec_cap = tbytes / 4;   // records per spilled (query, chunk) slot
  uint32_t* gaddr = reinterpret_cast<uint32_t*>(table + tbytes);
  Tally T;
  enc_count_phase<NT, 1>(pops, npop, cap, cenc, cstride, coffs, n_sub, K2, nchunks, q, c, tbytes, table, gaddr, S, T);
  if (threadIdx.x == 0) S.fill = 0;
  enc_levels<NT, false>(T, table, valid, n_sub, S);   // ends with a barrier
  if (scores && n_sub >= 2 && valid - S.lh[0] - S.lh[1] <= rec_cap)
    compact_records<NT, true>(table, valid, reinterpret_cast<uint32_t*>(scores + ((size_t)q * nchunks + c) * tbytes),
                              &S.fill);
  int32_t* pp = part + ((size_t)q * nchunks + c) * (n_sub + 1);
  for (int l = threadIdx.x; l <= n_sub; l += NT) pp[l] = S.lh[l];
}

constexpr int TC_CW = 16;
constexpr int TC_THREADS = 32 * (TC_CW + 1);
constexpr int TC_SG = 32 * TC_CW;     // groups per stage: one per consumer thread
constexpr int TC_RS = 4;              // ring stages (32 KB)

__global__ void __launch_bounds__(TC_THREADS, 2) k_count_tma(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ cenc, size_t cstride, const uint32_t* __restrict__ coffs, int n_sub, int K2,
    int64_t n, int64_t nchunks, int64_t chunk, double budget, uint32_t* __restrict__ cand, int64_t cand_cap,
    int64_t* __restrict__ flags, int64_t* __restrict__ sbase, int64_t* __restrict__ scnt,
    int64_t* __restrict__ cnum, int32_t* __restrict__ lvl) {
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ EncSmem<TC_THREADS> S;
  cg::cluster_group cluster = cg::this_cluster();
  const int64_t q = blockIdx.y;
  const int64_t c = cluster.block_rank();
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t base = c * chunk;
  const int valid = (int)max((int64_t)0, min(chunk, n - base));
  const int tbytes = (int)(chunk / 2);
  uint4* ring = reinterpret_cast<uint4*>(table + tbytes);   // [TC_RS][TC_SG]
  if (tid == 0) {
    for (int k = 0; k < TC_RS; ++k) {
      mbar_init(&S.full[k], 1);
      mbar_init(&S.empty[k], TC_CW);
    }
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  for (int i = tid; i < EC_LEVELS; i += TC_THREADS) S.ge[i] = 0;
  if (tid < 32) {
    const int np = tid < n_sub ? min(npop[q * n_sub + tid], cap) : 0;
    int x = np;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int y = __shfl_up_sync(0xffffffffu, x, o);
      if (tid >= o) x += y;
    }
    if (tid <= n_sub) S.jpref[tid] = x - np;
  }
  __syncthreads();
  Tally T;
  if (wid == TC_CW) {
    // producer: slices of batch b + 1 are looked up while batch b is issued
    const int P_all = S.jpref[n_sub];
    const size_t offs_len = (size_t)nchunks * K2 + 1;
    const uint4* E4 = reinterpret_cast<const uint4*>(cenc);
    const uint32_t jstride = (uint32_t)(cstride / 4);   // groups per subspace
    int jp[8];
#pragma unroll
    for (int jj = 0; jj < 8; ++jj) jp[jj] = S.jpref[jj];
    uint32_t pos = 0;   // groups issued so far
    int opened = 0;     // ring stages [0, opened) are writable
    int pads = 0;
    auto open_until = [&](uint32_t end) {
      while ((uint32_t)opened * TC_SG < end) {
        if (opened >= TC_RS) mbar_wait(&S.empty[opened % TC_RS], (unsigned)((opened / TC_RS) - 1) & 1u);
        ++opened;
      }
    };
    auto lookup = [&](int b, uint32_t& ga, uint32_t& ng) {
      const int g = b * 32 + lane;
      ga = ng = 0;
      if (g < P_all) {
        uint32_t g0, pad, j;
        enc_slice(pops, coffs, offs_len, cap, n_sub, K2, q, c, jp, g, g0, ng, pad, j);
        ga = j * jstride + 2 * g0;   // units -> 16-byte groups
        ng *= 2;
        pads += (int)pad;
      }
    };
    const int nbat = (P_all + 31) / 32;
    uint32_t ga, ng, ga1, ng1;
    lookup(0, ga, ng);
    for (int b = 0; b < nbat; ++b) {
      lookup(b + 1, ga1, ng1);
      uint32_t x = ng;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const uint32_t y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const uint32_t end = pos + __shfl_sync(0xffffffffu, x, 31);
      const uint32_t my = pos + x - ng;
      for (uint32_t k = pos / TC_SG; k * TC_SG < end; ++k) {
        open_until(k * TC_SG + 1);
        const uint32_t lo = max(my, k * TC_SG), hi = min(my + ng, (k + 1) * TC_SG);
        if (lo < hi)
          tma_g2s(ring + (size_t)(k % TC_RS) * TC_SG + (lo - k * TC_SG), E4 + ga + (lo - my), (hi - lo) * 16u,
                  &S.full[k % TC_RS]);
        __syncwarp();
        if (lane == 0 && end >= (k + 1) * TC_SG) {
          S.cnt[k % TC_RS] = TC_SG;
          mbar_expect_tx(&S.full[k % TC_RS], TC_SG * 16u);
        }
      }
      pos = end;
      ga = ga1;
      ng = ng1;
    }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) pads += __shfl_xor_sync(0xffffffffu, pads, o);
    uint32_t kend = pos / TC_SG;
    if (pos % TC_SG) {   // last partial stage
      if (lane == 0) {
        S.cnt[kend % TC_RS] = (int)(pos % TC_SG);
        mbar_expect_tx(&S.full[kend % TC_RS], (pos % TC_SG) * 16u);
      }
      ++kend;
    }
    open_until(kend * TC_SG + 1);   // the end marker's stage
    if (lane == 0) {
      S.pads = pads;
      S.cnt[kend % TC_RS] = 0;
      mbar_arrive(&S.full[kend % TC_RS]);
    }
  } else {
    uint4* t4 = reinterpret_cast<uint4*>(table);
    for (int i = tid; i < tbytes / 16; i += TC_CW * 32) t4[i] = make_uint4(0, 0, 0, 0);
    asm volatile("bar.sync 1, %0;" ::"r"(TC_CW * 32) : "memory");
    const uint32_t tsg = smem_u32(table);
    uint32_t ev = 0, od = 0;
    for (int k = 0;; ++k) {
      const int slot = k % TC_RS;
      mbar_wait(&S.full[slot], (unsigned)(k / TC_RS) & 1u);
      const int cnt = *(volatile int*)&S.cnt[slot];
      if (cnt == 0) break;
      if (tid < cnt) apply_group(ring[(size_t)slot * TC_SG + tid], tsg, ev, od);
      __syncwarp();
      if (lane == 0) mbar_arrive(&S.empty[slot]);
      if ((k & 31) == 31) {   // <= 4 per stage in 8-bit fields: flush before they can carry
        T.add_round(ev, od);
        ev = od = 0;
      }
    }
    T.add_round(ev, od);
  }
  __syncthreads();
  enc_epilogue<TC_THREADS>(T, table, valid, n_sub, S, cluster, q, base, budget, cand, cand_cap, flags, sbase,
                           scnt, cnum, lvl, reinterpret_cast<uint32_t*>(ring), TC_RS * TC_SG * 4);
}

// Encoded CSR of the TMA count (cluster mode, 4-bit tables): per subspace,
// slices (chunk, cell) of the (chunk, cell, id) CSR padded to whole 16-byte
// groups; coffs = group offsets with the padding count of the slice ENDING
// there in the top 2 bits.  Three launches: per-1024-slice group sums, a scan
// of those sums, then per-slice offsets + the encoded fill.
constexpr int CC_NT = 1024;
__global__ void __launch_bounds__(CC_NT) k_ccsr_sums(const uint32_t* __restrict__ offs, size_t offs_len,
                                                    int64_t nsl, uint32_t* __restrict__ bsum, int U) {
  __shared__ uint32_t wtot[CC_NT / 32];
  const int j = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * CC_NT + threadIdx.x;
  const uint32_t* O = offs + (size_t)j * offs_len;
  const uint32_t g = i < nsl ? (O[i + 1] - O[i] + (U - 1)) / U : 0u;
  uint32_t tot;
  block_excl_scan<CC_NT>(g, wtot, tot);
  if (threadIdx.x == 0) bsum[(size_t)j * gridDim.x + blockIdx.x] = tot;
}
__global__ void __launch_bounds__(CC_NT) k_ccsr_scan(uint32_t* __restrict__ bsum, int nb) {
  __shared__ uint32_t wtot[CC_NT / 32];
  const int j = blockIdx.x;
  uint32_t carry = 0;
  for (int b0 = 0; b0 < nb; b0 += CC_NT) {
    const int b = b0 + threadIdx.x;
    const uint32_t v = b < nb ? bsum[(size_t)j * nb + b] : 0u;
    uint32_t tot;
    const uint32_t ex = block_excl_scan<CC_NT>(v, wtot, tot);
    if (b < nb) bsum[(size_t)j * nb + b] = carry + ex;
    carry += tot;
  }
}
__global__ void __launch_bounds__(CC_NT) k_ccsr_fill(const uint32_t* __restrict__ ids,
                                                    const uint32_t* __restrict__ offs, size_t offs_len,
                                                    int64_t nsl, int K2, int64_t n, int64_t chunk,
                                                    const uint32_t* __restrict__ bsum, uint32_t* __restrict__ coffs,
                                                    uint32_t* __restrict__ cenc, size_t cstride, int U, int nib) {
  __shared__ uint32_t wtot[CC_NT / 32];
  const int j = blockIdx.y;
  const int64_t i = (int64_t)blockIdx.x * CC_NT + threadIdx.x;
  const uint32_t* O = offs + (size_t)j * offs_len;
  uint32_t s0 = 0, len = 0;
  if (i < nsl) {
    s0 = O[i];
    len = O[i + 1] - s0;
  }
  const uint32_t g = (len + (U - 1)) / U;
  uint32_t tot;
  const uint32_t g0 = bsum[(size_t)j * gridDim.x + blockIdx.x] + block_excl_scan<CC_NT>(g, wtot, tot);
  uint32_t* C = coffs + (size_t)j * offs_len;
  if (i < nsl) {   // coffs is zeroed first: the padding bits of slice i land in C[i + 1]
    atomicOr(&C[i], g0);
    atomicOr(&C[i + 1], ((U * g - len) << 29) | (i + 1 == nsl ? g0 + g : 0u));
    const int64_t cbase = (i / K2) * chunk;
    const uint32_t* I = ids + (size_t)j * n + s0;
    uint32_t* E = cenc + (size_t)j * cstride + U * (size_t)g0;
    for (uint32_t e = 0; e < U * g; ++e) {
      // table word byte offset << 6 | lane shift (4-bit or 8-bit lanes); a
      // padding entry adds 0 (shift 32) to the word of one of the slice's own
      // ids: a warp's padding lanes then spread over the banks like real
      // entries instead of all hitting word 0
      const uint32_t p = (uint32_t)(I[e < len ? e : (EC_SPREAD ? e % len : 0u)] - cbase);
      uint32_t v = nib ? ((p >> 3) << 8) | ((p & 7u) << 2) : ((p >> 2) << 8) | ((p & 3u) << 3);
      if (e >= len) v = EC_SPREAD ? (v & ~63u) | EC_SENT : EC_SENT;
      E[e] = v;
    }
  }
}

// ------------------------------------------------------- global-mode count
// One CTA per (id chunk, query) over a whole super-tile.  Sweep 1 (CNT_HIST)
// writes the chunk's level histogram and spills its score >= 2 ids as packed
// records (not the 32-64 KB table); Alg. 5 runs on the (all-reduced)
// per-query histogram; sweep 2 is k_emit_rec (a warp per (query, chunk)
// filters the records at the level L straight into the query's candidate
// segment) plus, for the pairs it lists (L < 2, or records that overflowed
// their slot), this kernel in CNT_EMIT mode: persistent CTAs recount those
// chunks in shared memory and compact them.  CNT_TABLE stores the table
// itself (count_collisions tap).
enum { CNT_TABLE = 0, CNT_HIST = 1, CNT_EMIT = 2 };
template <bool NIB>
__global__ void __launch_bounds__(CT_THREADS, 4) k_count(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ ids, const uint32_t* __restrict__ offs, int n_sub, int K2, int64_t n,
    int64_t nchunks, int64_t chunk, int mode, uint8_t* __restrict__ scores, int32_t* __restrict__ part,
    const int32_t* __restrict__ lvl, const int64_t* __restrict__ sbase, const int64_t* __restrict__ coff,
    uint32_t* __restrict__ cand, const int64_t* __restrict__ rlist) {
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ CountSmem S;
  __shared__ int s_fill;
  const int tid = threadIdx.x;
  const int tbytes = (int)(NIB ? chunk / 2 : chunk);
  uint4* t4 = reinterpret_cast<uint4*>(table);
  if (mode == CNT_EMIT) {
    const int64_t cnt = rlist[0];
    for (int64_t i = blockIdx.x; i < cnt; i += gridDim.x) {
      const int64_t p = rlist[1 + i];
      const int64_t q = p / nchunks, c = p - q * nchunks;
      const int64_t base = c * chunk;
      const int valid = (int)min(chunk, n - base);
      for (int v = tid; v < tbytes / 16; v += CT_THREADS) t4[v] = make_uint4(0, 0, 0, 0);
      __syncthreads();
      count_chunk<NIB>(pops, npop, cap, ids, offs, (size_t)nchunks * K2 + 1, n_sub, K2, n, c, q, base, table, S);
      if (tid == 0) s_fill = 0;
      __syncthreads();
      compact_unordered<CT_THREADS, NIB>(table, valid, (uint32_t)lvl[q], base, cand + sbase[q] + coff[p], &s_fill);
      __syncthreads();   // table and S are reused by the next pair
    }
    return;
  }
  const int64_t c = blockIdx.x;
  const int64_t q = blockIdx.y;
  const int64_t base = c * chunk;
  const int valid = (int)min(chunk, n - base);
  const int rec_cap = tbytes / 4;                  // records per spilled (query, chunk) slot
  for (int i = tid; i < tbytes / 16; i += CT_THREADS) t4[i] = make_uint4(0, 0, 0, 0);
  __syncthreads();
  count_chunk<NIB>(pops, npop, cap, ids, offs, (size_t)nchunks * K2 + 1, n_sub, K2, n, c, q, base, table, S);
  if (mode == CNT_TABLE && !NIB) {
    uint4* dst = reinterpret_cast<uint4*>(scores + ((size_t)q * nchunks + c) * tbytes);
    for (int i = tid; i < tbytes / 16; i += CT_THREADS) dst[i] = t4[i];
  }
  if (tid == 0) s_fill = 0;
  chunk_levels(table, valid, n_sub, S);   // ends with a barrier
  if (mode == CNT_HIST && scores && n_sub >= 2 && valid - S.lh[0] - S.lh[1] <= rec_cap)
    compact_records<CT_THREADS, NIB>(table, valid,
                                     reinterpret_cast<uint32_t*>(scores + ((size_t)q * nchunks + c) * tbytes),
                                     &s_fill);
  int32_t* pp = part + ((size_t)q * nchunks + c) * (n_sub + 1);
  for (int l = tid; l <= n_sub; l += CT_THREADS) pp[l] = S.lh[l];
}

// Global-mode emit sweep: a warp per (query, chunk) pair filters the
// chunk's spilled score >= 2 records at the query's level L into its
// candidate slots; pairs without usable records (L < 2, overflowed slot) are
// appended to rlist (rlist[0] = count) for the CNT_EMIT recount.
constexpr int ER_WARPS = 8;
template <bool NIB>
__global__ void __launch_bounds__(32 * ER_WARPS) k_emit_rec(
    const uint8_t* __restrict__ recs, int64_t n, int64_t nchunks, int64_t chunk, int n_sub, int64_t QS,
    const int32_t* __restrict__ part, const int32_t* __restrict__ lvl, const int64_t* __restrict__ sbase,
    const int64_t* __restrict__ scnt, const int64_t* __restrict__ coff, int64_t cand_cap,
    uint32_t* __restrict__ cand, int64_t* __restrict__ rlist) {
  const int lane = threadIdx.x & 31;
  const int64_t p = (int64_t)blockIdx.x * ER_WARPS + (threadIdx.x >> 5);
  if (p >= QS * nchunks) return;
  const int64_t q = p / nchunks, c = p - q * nchunks;
  if (sbase[q] + scnt[q] > cand_cap) return;
  const int64_t lo = coff[p];
  const int64_t hi = c + 1 < nchunks ? coff[p + 1] : scnt[q];
  if (hi == lo) return;   // no candidate of this query in this chunk
  const int L = lvl[q];
  const int64_t base = c * chunk;
  const int valid = (int)min(chunk, n - base);
  const int64_t tbytes = NIB ? chunk / 2 : chunk;
  int rc = 0;
  if (L >= 2) {
    const int32_t* pp = part + (size_t)p * (n_sub + 1);
    rc = valid - pp[0] - pp[1];
  }
  if (L < 2 || rc > (int)(tbytes / 4)) {
    if (lane == 0) {
      const int64_t slot = (int64_t)atomicAdd((unsigned long long*)rlist, 1ull);
      rlist[1 + slot] = p;
    }
    return;
  }
  const uint32_t* rec = reinterpret_cast<const uint32_t*>(recs + (size_t)p * tbytes);
  uint32_t* dst = cand + sbase[q] + lo;
  const uint32_t lt = (1u << lane) - 1u;
  int w = 0;
#pragma unroll 4
  for (int i0 = 0; i0 < rc; i0 += 32) {
    const int i = i0 + lane;
    const uint32_t r = i < rc ? __ldg(rec + i) : 0u;
    const bool hit = (int)(r & 0xFFu) >= L;
    const uint32_t bal = __ballot_sync(0xffffffffu, hit);
    if (hit) dst[w + __popc(bal & lt)] = (uint32_t)base + (r >> 8);
    w += __popc(bal);
  }
}

// Level histograms of externally provided score chunks (select_candidates tap).
__global__ void __launch_bounds__(CT_THREADS) k_chunk_hist(const uint8_t* __restrict__ scores, int64_t n,
                                                           int64_t nchunks, int64_t chunk, int n_sub,
                                                           int32_t* __restrict__ part) {
  __shared__ CountSmem S;
  const int64_t c = blockIdx.x;
  const int64_t base = c * chunk;
  const int valid = (int)min(chunk, n - base);
  const uint8_t* tab = scores + (size_t)c * chunk;
  // force the scan path (no tallies here)
  for (int l = threadIdx.x; l < 256; l += blockDim.x) S.lh[l] = 0;
  __syncthreads();
  const uint32_t* w4 = reinterpret_cast<const uint32_t*>(tab);
  for (int i = threadIdx.x; i < (valid + 3) / 4; i += blockDim.x) {
    uint32_t w = w4[i];
    while (w) {
      const int b = __ffs(w) - 1;
      const int byte = b >> 3;
      atomicAdd(&S.lh[(w >> (byte * 8)) & 0xFF], 1);
      w &= ~(0xFFu << (byte * 8));
    }
  }
  __syncthreads();
  int32_t* pp = part + (size_t)c * (n_sub + 1);
  if (threadIdx.x == 0) {
    int nz = 0;
    for (int l = 1; l <= n_sub; ++l) nz += S.lh[l];
    pp[0] = valid - nz;
  }
  for (int l = 1 + threadIdx.x; l <= n_sub; l += blockDim.x) pp[l] = S.lh[l];
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

// Global mode: one warp per query.  Alg. 5 on the (global) histogram, local
// candidate offsets per chunk (warp scan), one candidate segment per query
// reserved in the super-tile candidate buffer through the cursor flags[3].
__global__ void k_select(const int64_t* __restrict__ ghist, const int32_t* __restrict__ part, int64_t Q,
                         int64_t nchunks, int n_sub, double budget, int64_t* __restrict__ coff,
                         int64_t cand_cap, int64_t* __restrict__ flags, int64_t* __restrict__ sbase,
                         int64_t* __restrict__ scnt, int64_t* __restrict__ cnum, int32_t* __restrict__ lvl,
                         int64_t* __restrict__ gsb = nullptr, int64_t* __restrict__ gsc = nullptr) {
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= Q) return;
  const int64_t* h = ghist + (size_t)q * (n_sub + 1);
  int64_t cands = 0;
  int L = 0;
  if (lane == 0) L = alg5([&](int l) { return h[l]; }, n_sub, budget, cands);
  L = __shfl_sync(0xffffffffu, L, 0);
  int64_t run = 0;
  for (int64_t c0 = 0; c0 < nchunks; c0 += 32) {
    const int64_t c = c0 + lane;
    int64_t cc = 0;
    if (c < nchunks) {
      const int32_t* pp = part + ((size_t)q * nchunks + c) * (n_sub + 1);
      for (int l = L; l <= n_sub; ++l) cc += pp[l];
    }
    int64_t v = cc;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t x = __shfl_up_sync(0xffffffffu, v, o);
      if (lane >= o) v += x;
    }
    if (c < nchunks) coff[q * nchunks + c] = run + v - cc;
    run += __shfl_sync(0xffffffffu, v, 31);
  }
  int64_t b = 0;
  if (lane == 0) {
    b = (int64_t)atomicAdd((unsigned long long*)&flags[3], (unsigned long long)run);
    if (b + run > cand_cap) flags[1] = 1;
    sbase[q] = b;
    scnt[q] = run;
    cnum[q] = cands;
    lvl[q] = L;
  }
  if (gsb) {   // per-(query, chunk) candidate segments: the re-rank's chunk-major plan
    b = __shfl_sync(0xffffffffu, b, 0);
    for (int64_t c = lane; c < nchunks; c += 32) {
      const int64_t o = coff[q * nchunks + c];
      gsb[q * nchunks + c] = b + o;
      gsc[q * nchunks + c] = (c + 1 < nchunks ? coff[q * nchunks + c + 1] : run) - o;
    }
  }
}

constexpr int CMP_THREADS = 256;
__global__ void __launch_bounds__(CMP_THREADS) k_compact(const uint8_t* __restrict__ scores, int64_t n,
                                                          int64_t nchunks, int64_t chunk, int64_t q0,
                                                          const int32_t* __restrict__ lvl,
                                                          const int64_t* __restrict__ coff,
                                                          const int64_t* __restrict__ sbase,
                                                          const int64_t* __restrict__ scnt,
                                                          int64_t cand_cap,
                                                          uint32_t* __restrict__ cand) {
  __shared__ uint32_t wtot[CMP_THREADS / 32];
  const int64_t c = blockIdx.x;
  const int64_t qt = blockIdx.y, q = q0 + qt;
  const int64_t b = sbase[q];
  if (b + scnt[q] > cand_cap) return;
  const int64_t base = c * chunk;
  const int valid = (int)min(chunk, n - base);
  compact_table<CMP_THREADS>(scores + ((size_t)qt * nchunks + c) * chunk, valid, (uint32_t)lvl[q], base,
                             cand + b + coff[(size_t)qt * nchunks + c], wtot);
}

// ------------------------------------------------------------ rerank plan
constexpr int GR = 32;    // candidate rows per rerank tile (one warp: lane = row)
// Tile plans: exclusive prefixes of the tiles per segment in two orders,
// query-major (segment p) and chunk-major (p = r * QS + q -> segment q * S + r);
// tq/tp[segment] = its first tile in that order, total in flags[2].  Two
// launches: per-1024-segment block sums, then block offsets + in-block scans.
constexpr int PLAN_NT = 1024;
__device__ __forceinline__ int64_t seg_cm(int64_t p, int64_t QS, int S) { return (p % QS) * S + p / QS; }
__device__ __forceinline__ int64_t seg_tiles(const int64_t* scnt, int64_t sg) { return (scnt[sg] + GR - 1) / GR; }

// inclusive block scan of two int64 values (PLAN_NT threads)
__device__ __forceinline__ void block_scan2(int64_t& a, int64_t& b, int64_t* ws /* [2][32] */) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    const int64_t x = __shfl_up_sync(0xffffffffu, a, o), y = __shfl_up_sync(0xffffffffu, b, o);
    if (lane >= o) { a += x; b += y; }
  }
  if (lane == 31) { ws[wid] = a; ws[32 + wid] = b; }
  __syncthreads();
  if (wid == 0) {
    int64_t x = ws[lane], y = ws[32 + lane];
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int64_t u = __shfl_up_sync(0xffffffffu, x, o), v = __shfl_up_sync(0xffffffffu, y, o);
      if (lane >= o) { x += u; y += v; }
    }
    ws[lane] = x;
    ws[32 + lane] = y;
  }
  __syncthreads();
  if (wid) { a += ws[wid - 1]; b += ws[32 + wid - 1]; }
}

__global__ void __launch_bounds__(PLAN_NT) k_plan_sums(const int64_t* __restrict__ scnt, int64_t nseg, int S,
                                                       int64_t QS, int64_t* __restrict__ bsum) {
  __shared__ int64_t ws[64];
  const int64_t p = (int64_t)blockIdx.x * PLAN_NT + threadIdx.x;
  int64_t a = p < nseg ? seg_tiles(scnt, p) : 0, b = p < nseg ? seg_tiles(scnt, seg_cm(p, QS, S)) : 0;
  block_scan2(a, b, ws);
  if (threadIdx.x == PLAN_NT - 1) {
    bsum[blockIdx.x] = a;
    bsum[gridDim.x + blockIdx.x] = b;
  }
}

__global__ void __launch_bounds__(PLAN_NT) k_plan_scan(const int64_t* __restrict__ scnt, int64_t nseg, int S,
                                                       int64_t QS, const int64_t* __restrict__ bsum,
                                                       int64_t* __restrict__ tq, int64_t* __restrict__ tp,
                                                       int64_t* __restrict__ flags) {
  __shared__ int64_t ws[64];
  __shared__ int64_t off[2];
  const int lane = threadIdx.x & 31;
  if (threadIdx.x < 32) {   // this block's offsets: sums of the earlier blocks
    int64_t x = 0, y = 0;
    for (int i = lane; i < (int)blockIdx.x; i += 32) { x += bsum[i]; y += bsum[gridDim.x + i]; }
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) { x += __shfl_xor_sync(0xffffffffu, x, o); y += __shfl_xor_sync(0xffffffffu, y, o); }
    if (lane == 0) { off[0] = x; off[1] = y; }
  }
  const int64_t p = (int64_t)blockIdx.x * PLAN_NT + threadIdx.x;
  const int64_t sq = p, sc = p < nseg ? seg_cm(p, QS, S) : 0;
  const int64_t ta = p < nseg ? seg_tiles(scnt, sq) : 0, tb = p < nseg ? seg_tiles(scnt, sc) : 0;
  int64_t a = ta, b = tb;
  block_scan2(a, b, ws);   // (syncs make off[] visible)
  if (p < nseg) {
    tq[sq] = off[0] + a - ta;
    if (tp) tp[sc] = off[1] + b - tb;
  }
  if (p == nseg - 1 && flags) flags[2] = off[0] + a;
}

// Tile descriptors in processing order (one warp per segment):
// {candidate offset lo, hi, query << 6 | rows, output tile (query-major)}.
__global__ void k_tile_map(const int64_t* __restrict__ scnt, const int64_t* __restrict__ tproc,
                           const int64_t* __restrict__ tout, const int64_t* __restrict__ sbase, int64_t nseg,
                           int S, int4* __restrict__ desc) {
  const int64_t sg = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  if (sg >= nseg) return;
  const int64_t cnt = scnt[sg], nt = (cnt + GR - 1) / GR, tp = tproc[sg], to = tout[sg], b = sbase[sg];
  for (int64_t i = threadIdx.x & 31; i < nt; i += 32) {
    const int64_t cb = b + i * GR;
    const int m = (int)min((int64_t)GR, cnt - i * GR);
    desc[tp + i] = make_int4((int)(uint32_t)cb, (int)(cb >> 32), (int)((sg / S) << 6) | m, (int)(to + i));
  }
}

// ---------------------------------------------------- warp top-k helpers
// warp-wide bitonic sort of one (key, id) pair per lane, ascending.
__device__ __forceinline__ void warp_sort_pairs(unsigned long long& key, uint32_t& id) {
  const int lane = threadIdx.x & 31;
#pragma unroll
  for (int size = 2; size <= 32; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      const unsigned long long ok = __shfl_xor_sync(0xffffffffu, key, stride);
      const uint32_t oi = __shfl_xor_sync(0xffffffffu, id, stride);
      const bool up = (lane & size) == 0;
      const bool lower = (lane & stride) == 0;
      const bool other_less = ok < key || (ok == key && oi < id);
      // lower lane keeps the min when sorting up
      const bool take = (lower == up) ? other_less : !other_less && !(ok == key && oi == id);
      if (take) { key = ok; id = oi; }
    }
  }
}

// fold 8 products of a block into numpy's two einsum lanes (engine.py:273)
__device__ __forceinline__ void einsum_block8(const float* xv, const float* qv8, double& a0, double& a1) {
  double p[8];
#pragma unroll
  for (int t = 0; t < 8; ++t) {
    const double e = __dsub_rn((double)xv[t], (double)qv8[t]);
    p[t] = __dmul_rn(e, e);
  }
  a0 = __dadd_rn(p[6], a0); a1 = __dadd_rn(p[7], a1);
  a0 = __dadd_rn(p[4], a0); a1 = __dadd_rn(p[5], a1);
  a0 = __dadd_rn(p[2], a0); a1 = __dadd_rn(p[3], a1);
  a0 = __dadd_rn(p[0], a0); a1 = __dadd_rn(p[1], a1);
}



struct TileRef {
  int64_t q;
  int m;
  int out;        // output tile (query-major)
  uint32_t cid;   // this lane's candidate id (valid if lane < m)
  int iq = 0;     // integer path: u8 rows and a u8-exact query
  int32_t xs = 0; // integer path: this lane's row sum of squares
  int32_t qs = 0; // integer path: the query's sum of squares
};

__device__ __forceinline__ TileRef tile_ref(const int4 dsc, int lane, const uint32_t* __restrict__ cand) {
  TileRef r;
  r.m = dsc.z & 63;
  r.q = dsc.z >> 6;
  r.out = dsc.w;
  const int64_t cb = (int64_t)(((uint64_t)(uint32_t)dsc.y << 32) | (uint32_t)dsc.x);
  r.cid = lane < r.m ? cand[cb + lane] : 0xFFFFFFFFu;
  return r;
}

// ----------------------------------------- rerank: cp.async warp pipelines
// Warp w of W takes tiles w, w + W, w + 2W, ... of the plan's processing
// order, so all warps sweep the (locality-ordered) queries together and rows
// shared by neighbouring queries are served from L2.  Each warp streams
// (tile, 64-dim segment) units through its own ring of AST shared-memory
// stages with cp.async (LDGSTS, 16 B per lane, L2-only; one instruction moves
// two 256-byte row segments): the next AST-1 units are in flight while lane r
// folds row r of the current unit into numpy's two einsum lanes against the
// query segment (pre-converted to fp64 in shared memory).  Warp top-k of the
// 32 (d2, id) pairs per tile.
// Rows are staged in the index's storage format (row_format.cuh): f32, or a
// lossless narrower copy (f16 / u8) when every value of X converts exactly,
// so the staged bytes per row shrink 2x / 4x and the fp64 arithmetic on the
// widened values is unchanged.
template <typename T> struct RowFmt;
template <> struct RowFmt<float> {    // 64 dims (256 B) per unit, 16 lanes per row segment
  static constexpr int UD = 64, LPR = 16, PITCH = 272, WARPS = 12, CTAS = 1;
};
template <> struct RowFmt<__half> {   // 128 dims (256 B) per unit
  static constexpr int UD = 128, LPR = 16, PITCH = 272, WARPS = 11, CTAS = 1;
};
template <> struct RowFmt<uint8_t> {  // 128 dims (128 B) per unit, 8 lanes per row segment
  static constexpr int UD = 128, LPR = 8, PITCH = 144, WARPS = 20, CTAS = 1;
};
constexpr int AST = 2;                 // stages per warp (the id lookahead assumes 2; a power of 2)
template <typename T>
struct AStage {
  uint8_t rows[GR][RowFmt<T>::PITCH];  // pitch = 16 B mod 128: 16-byte row reads are conflict free
  float q[RowFmt<T>::UD];
};
template <typename T>
struct AWarpSmem {
  AStage<T> st[AST];
  double qd[RowFmt<T>::UD];
};

// 8 consecutive row values (exact) widened to f64
__device__ __forceinline__ void load8(const uint8_t* rb, int b, double (&xv)[8], float) {
  const float4 x0 = *reinterpret_cast<const float4*>(rb + 4 * b);
  const float4 x1 = *reinterpret_cast<const float4*>(rb + 4 * b + 16);
  xv[0] = x0.x; xv[1] = x0.y; xv[2] = x0.z; xv[3] = x0.w;
  xv[4] = x1.x; xv[5] = x1.y; xv[6] = x1.z; xv[7] = x1.w;
}
__device__ __forceinline__ void load8(const uint8_t* rb, int b, double (&xv)[8], __half) {
  const uint4 w = *reinterpret_cast<const uint4*>(rb + 2 * b);
  const uint32_t ws[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
  for (int t = 0; t < 4; ++t) {
    const float2 f = __half22float2(*reinterpret_cast<const __half2*>(&ws[t]));
    xv[2 * t] = f.x;
    xv[2 * t + 1] = f.y;
  }
}
__device__ __forceinline__ void load8(const uint8_t* rb, int b, double (&xv)[8], uint8_t) {
  const uint2 w = *reinterpret_cast<const uint2*>(rb + b);
#pragma unroll
  for (int t = 0; t < 8; ++t) xv[t] = __uint2double_rn(__byte_perm(t < 4 ? w.x : w.y, 0, 0x4440u + (t & 3)));
}
__device__ __forceinline__ float elem(const uint8_t* rb, int b, float) { return reinterpret_cast<const float*>(rb)[b]; }
__device__ __forceinline__ float elem(const uint8_t* rb, int b, __half) {
  return __half2float(reinterpret_cast<const __half*>(rb)[b]);
}
__device__ __forceinline__ float elem(const uint8_t* rb, int b, uint8_t) { return (float)rb[b]; }

__device__ __forceinline__ void cp_async16(void* dst, const void* src) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(smem_u32(dst)), "l"(src) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() { asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory"); }

template <typename T>
__global__ void __launch_bounds__(32 * RowFmt<T>::WARPS, RowFmt<T>::CTAS) k_rerank_async(
    const T* __restrict__ X, int d, const float* __restrict__ Qf, const int4* __restrict__ desc,
    const uint32_t* __restrict__ cand, int64_t ntiles, int kk, unsigned long long* __restrict__ pkey,
    uint32_t* __restrict__ pid, unsigned long long* __restrict__ qthr, const uint8_t* __restrict__ Qb,
    const uint8_t* __restrict__ qok, const int32_t* __restrict__ qsq, const int32_t* __restrict__ xsq) {
  using F = RowFmt<T>;
  constexpr bool U8 = std::is_same<T, uint8_t>::value;
  constexpr int UD = F::UD, LPR = F::LPR, RPI = 32 / F::LPR;
  extern __shared__ __align__(128) unsigned char asm_[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  AWarpSmem<T>& W = reinterpret_cast<AWarpSmem<T>*>(asm_)[wid];
  // warps interleaved across CTAs: concurrently running warps hold adjacent tiles
  const int64_t gw = (int64_t)wid * gridDim.x + blockIdx.x, nw = (int64_t)gridDim.x * F::WARPS;
  if (gw >= ntiles) return;
  const int64_t t0 = gw;
  const int64_t nt = (ntiles - gw + nw - 1) / nw;        // my tiles: t0 + i * nw
  const int nsg = (d + UD - 1) / UD;
  const int64_t U = nt * nsg;
  // descriptors run two tiles ahead of the issue, candidate ids one tile ahead
  auto dsc = [&](int64_t i) { return i < nt ? __ldg(desc + t0 + i * nw) : make_int4(0, 0, 0, 0); };
  auto row_of = [&](const TileRef& r) {
    return reinterpret_cast<const uint8_t*>(X + (size_t)(lane < r.m ? r.cid : 0u) * d);
  };
  // integer path (U8 rows, qok[q]): d2 = sum x^2 - 2 sum x q + sum q^2 in
  // exact integers.  Loads are staged so none waits on another: descriptors
  // two tiles ahead, candidate ids (and qok) one tile ahead, the row / query
  // sums of squares when the tile starts issuing (its ids are resident then).
  auto ref_of = [&](const int4 dd) {
    TileRef r = tile_ref(dd, lane, cand);
    if (U8 && qok) r.iq = r.m > 0 ? qok[r.q] : 0;
    return r;
  };
  auto sums_of = [&](TileRef& r) {
    if (U8 && r.iq) {
      r.xs = lane < r.m ? __ldg(xsq + r.cid) : 0;
      r.qs = __ldg(qsq + r.q);
    }
  };
  TileRef tcur = ref_of(dsc(0));                         // tile being issued
  sums_of(tcur);
  TileRef tnext = ref_of(dsc(1));                        // its successor (ids in flight)
  int4 dpre = dsc(2);                                    // the one after
  int64_t tcur_i = 0;
  const uint8_t* rp = row_of(tcur);                      // my row of the issued tile
  TileRef tcomp = tcur;                                   // tile being computed
  const int r0 = lane / LPR, cl = lane % LPR;
  int64_t iss_i = 0;   // (tile, segment) of the next unit to issue: units are issued in order
  int iss_g = 0;
  auto issue = [&](int64_t u) {
    const int64_t i = iss_i;
    const int g = iss_g;
    if (++iss_g == nsg) {
      iss_g = 0;
      ++iss_i;
    }
    if (i != tcur_i) {
      tcur = tnext;
      tcur_i = i;
      sums_of(tcur);
      rp = row_of(tcur);
      tnext = ref_of(dpre);
      dpre = dsc(i + 2);
    }
    AStage<T>& st = W.st[(int)(u & (AST - 1))];
    const int s0 = g * UD;
    const int len = min(UD, d - s0);
    const int nch = (int)(len * sizeof(T)) / 16;          // 16-byte chunks per row segment (<= LPR)
    const int cofs = s0 * (int)sizeof(T) + cl * 16;
#pragma unroll
    for (int j = 0; j < GR / RPI; ++j) {                  // rows j * RPI + r0
      const int rr = j * RPI + r0;
      const uint8_t* src = reinterpret_cast<const uint8_t*>(
          __shfl_sync(0xffffffffu, reinterpret_cast<unsigned long long>(rp), rr));
      if (cl < nch && rr < tcur.m) cp_async16(&st.rows[rr][cl * 16], src + cofs);
    }
    if (U8 && tcur.iq) {   // the query's bytes (len is a multiple of 16 for u8 rows)
      if (lane < len / 16)
        cp_async16(reinterpret_cast<uint8_t*>(st.q) + lane * 16, Qb + (size_t)tcur.q * d + s0 + lane * 16);
    } else {
      for (int c = lane; c < len / 4; c += 32) cp_async16(&st.q[c * 4], Qf + (size_t)tcur.q * d + s0 + c * 4);
    }
  };
  for (int64_t u = 0; u < AST - 1; ++u) {
    if (u < U) issue(u);
    cp_async_commit();
  }
  double a0 = 0.0, a1 = 0.0;
  uint32_t iacc = 0;   // integer path: sum of x * q
  int64_t i = 0;       // (tile, segment) of unit u
  int g = 0;
  for (int64_t u = 0; u < U; ++u, (++g == nsg ? (g = 0, ++i) : 0)) {
    if (g == 0) tcomp = (i == tcur_i) ? tcur : tnext;     // ids of the tile computed now
    if (u + AST - 1 < U) issue(u + AST - 1);
    cp_async_commit();
    cp_async_wait<AST - 1>();
    __syncwarp();
    const AStage<T>& st = W.st[(int)(u & (AST - 1))];
    const int s0 = g * UD;
    const int len = min(UD, d - s0);
    const bool last = g == nsg - 1;
    if (U8 && tcomp.iq) {
      const uint8_t* row = st.rows[lane];
      const uint8_t* qb = reinterpret_cast<const uint8_t*>(st.q);
      for (int b = 0; b < len; b += 16) {
        const uint4 xw = *reinterpret_cast<const uint4*>(row + b);
        const uint4 qw = *reinterpret_cast<const uint4*>(qb + b);
        iacc = __dp4a(xw.x, qw.x, iacc);
        iacc = __dp4a(xw.y, qw.y, iacc);
        iacc = __dp4a(xw.z, qw.z, iacc);
        iacc = __dp4a(xw.w, qw.w, iacc);
      }
    } else {
    for (int t = lane; t < len; t += 32) W.qd[t] = (double)st.q[t];
    __syncwarp();
    const uint8_t* row = st.rows[lane];
    const double* qv = W.qd;
    const int full8 = last ? (len & ~7) : len;
    for (int b = 0; b < full8; b += 8) {
      double xv[8];
      load8(row, b, xv, T());
      double p[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) {
        const double e = __dsub_rn(xv[t], qv[b + t]);
        p[t] = __dmul_rn(e, e);
      }
      a0 = __dadd_rn(p[6], a0); a1 = __dadd_rn(p[7], a1);
      a0 = __dadd_rn(p[4], a0); a1 = __dadd_rn(p[5], a1);
      a0 = __dadd_rn(p[2], a0); a1 = __dadd_rn(p[3], a1);
      a0 = __dadd_rn(p[0], a0); a1 = __dadd_rn(p[1], a1);
    }
    if (last) {
      for (int b = full8; b < len; b += 2) {
        const double e0 = __dsub_rn((double)elem(row, b, T()), qv[b]);
        a0 = __dadd_rn(__dmul_rn(e0, e0), a0);
        if (b + 1 < len) {
          const double e1 = __dsub_rn((double)elem(row, b + 1, T()), qv[b + 1]);
          a1 = __dadd_rn(__dmul_rn(e1, e1), a1);
        }
      }
    }
    }   // fp64 path
    if (last) {
      double v;
      if (U8 && tcomp.iq) {   // every step of the reference's fp64 sum is exact on these integers
        v = (double)((int64_t)tcomp.xs - 2 * (int64_t)iacc + (int64_t)tcomp.qs);
        iacc = 0;
      } else {
        v = __dadd_rn(a0, a1);
        v = v >= 0.0 ? v : 0.0;
      }
      unsigned long long key = lane < tcomp.m ? (unsigned long long)__double_as_longlong(v) : ~0ull;
      uint32_t id = tcomp.cid;
      // qthr[q] bounds the query's final kk-th best from above (some earlier tile's kk-th
      // best), so rows above it cannot make the top-kk: when at most kk rows survive they
      // are written unsorted (k_topk selects), else the tile is sorted and tightens qthr.
      const unsigned long long thr = __ldcg(qthr + tcomp.q);
      const bool keep = key != ~0ull && key <= thr;
      const uint32_t bal = __ballot_sync(0xffffffffu, keep);
      const int ns = __popc(bal);
      unsigned long long* ok = pkey + (int64_t)tcomp.out * kk;
      uint32_t* oi = pid + (int64_t)tcomp.out * kk;
      if (ns <= kk) {
        if (keep) {
          const int slot = __popc(bal & ((1u << lane) - 1u));
          ok[slot] = key;
          oi[slot] = id;
        }
        if (lane >= ns && lane < kk) {
          ok[lane] = ~0ull;
          oi[lane] = 0xFFFFFFFFu;
        }
      } else {
        warp_sort_pairs(key, id);
        if (lane < kk) {
          ok[lane] = key;
          oi[lane] = id;
        }
        const unsigned long long kth = __shfl_sync(0xffffffffu, key, kk - 1);
        if (lane == 0 && kth != ~0ull) atomicMin(qthr + tcomp.q, kth);
      }
      a0 = 0.0;
      a1 = 0.0;
    }
    __syncwarp();   // the slot (and qd) are refilled next
  }
  cp_async_wait<0>();
}

// ------------------------------------- rerank: the integer fast path
// k_rerank_async's contract for the case config 2 runs: u8 rows, d <= 128
// (d % 16 == 0: one row segment per tile) and every query of the launch
// u8-exact, so every candidate takes the exact DP4A path.  Without the
// generic kernel's segment loop, fp64 path and per-unit bookkeeping a tile
// is: 8 row-copy instructions (8 lanes x 16 B per row, 4 rows each), 4
// DP4A per 16 bytes, the running bound and the partial top-k.  Tile state is
// staged so no load waits on another: descriptors three tiles ahead,
// candidate ids two ahead, row / query sums of squares one ahead.
#ifndef RI_WARPS_DEF
#define RI_WARPS_DEF 8
#endif
#ifndef RI_CTAS_DEF
#define RI_CTAS_DEF 2
#endif
constexpr int RI_WARPS = RI_WARPS_DEF, RI_CTAS = RI_CTAS_DEF, RI_PITCH = 144;
struct RiStage {
  uint8_t rows[GR][RI_PITCH];   // pitch = 16 B mod 128: conflict-free 16-byte row reads
  uint8_t q[128];
};
struct RiTile {
  int64_t q = 0;
  int m = 0, out = 0;
  uint32_t cid = 0;   // this lane's candidate (lane < m)
  int32_t xs = 0, qs = 0;
};

template <int NC>   // 16-byte chunks per row (d / 16); 0 = runtime d
__global__ void __launch_bounds__(32 * RI_WARPS, RI_CTAS) k_rerank_i8(
    const uint8_t* __restrict__ Xb, int d, const uint8_t* __restrict__ Qb, const int32_t* __restrict__ qsq,
    const int32_t* __restrict__ xsq, const int4* __restrict__ desc, const uint32_t* __restrict__ cand,
    int64_t ntiles, int kk, unsigned long long* __restrict__ pkey, uint32_t* __restrict__ pid,
    unsigned long long* __restrict__ qthr) {
  extern __shared__ __align__(128) unsigned char ri_sm[];
  const int wid = threadIdx.x >> 5, lane = threadIdx.x & 31;
  RiStage* st = reinterpret_cast<RiStage*>(ri_sm) + 2 * wid;
  const int64_t gw = (int64_t)wid * gridDim.x + blockIdx.x, nw = (int64_t)gridDim.x * RI_WARPS;
  if (gw >= ntiles) return;
  const int64_t nt = (ntiles - gw + nw - 1) / nw;   // my tiles: gw + i * nw
  const int nc = NC ? NC : d / 16;                   // 16-byte chunks per row
  auto dsc = [&](int64_t i) { return i < nt ? __ldg(desc + gw + i * nw) : make_int4(0, 0, 0, 0); };
  auto ids_of = [&](const int4 dd, RiTile& r) {   // tile fields + this lane's candidate id
    r.m = dd.z & 63;
    r.q = dd.z >> 6;
    r.out = dd.w;
    const int64_t cb = (int64_t)(((uint64_t)(uint32_t)dd.y << 32) | (uint32_t)dd.x);
    r.cid = lane < r.m ? cand[cb + lane] : 0u;
  };
  auto sums_of = [&](RiTile& r) {
    r.xs = lane < r.m ? __ldg(xsq + r.cid) : 0;
    r.qs = r.m > 0 ? __ldg(qsq + r.q) : 0;
  };
  const int r0 = lane >> 3, cl = lane & 7;
  // per-lane constants of the row copies: source column, destination offset inside a stage,
  // row pitch in bytes as an unsigned 32-bit factor (one IMAD.WIDE.U32 per address)
  const uint8_t* xcol = Xb + cl * 16;
  const uint32_t dst0 = (uint32_t)(r0 * RI_PITCH + cl * 16);
  const uint32_t rowb = NC ? (uint32_t)(NC * 16) : (uint32_t)d;
  const bool colok = NC == 8 ? true : cl < nc;
  auto issue = [&](const RiTile& r, RiStage& s) {
    uint8_t* dst = &s.rows[0][0] + dst0;
#pragma unroll
    for (int j = 0; j < GR / 4; ++j) {
      const int rr = j * 4 + r0;
      const uint32_t c = __shfl_sync(0xffffffffu, r.cid, rr);
      if (colok && rr < r.m) cp_async16(dst + j * 4 * RI_PITCH, xcol + (uint64_t)c * rowb);
    }
    if (lane < nc && r.m > 0) cp_async16(s.q + lane * 16, Qb + (uint64_t)r.q * rowb + lane * 16);
    cp_async_commit();
  };
  RiTile ta, tb, tc;              // computing i, issued i + 1, ids of i + 2
  ids_of(dsc(0), ta);
  sums_of(ta);
  ids_of(dsc(1), tb);
  int4 dn = dsc(2);
  issue(ta, st[0]);
  // the running bound of a tile is read one tile ahead (a bound read early is
  // only looser: qthr only decreases), so no compare waits on its L2 round trip
  unsigned long long thr_nx = __ldcg(qthr + ta.q);
  for (int64_t i = 0; i < nt; ++i) {
    ids_of(dn, tc);               // ids of tile i + 2
    dn = dsc(i + 3);
    sums_of(tb);                  // tile i + 1's ids arrived during tile i - 1
    if (i + 1 < nt) issue(tb, st[(i + 1) & 1]);
    else cp_async_commit();
    const unsigned long long thr = thr_nx;
    thr_nx = __ldcg(qthr + tb.q);   // tb.q = 0 past the last tile: a valid address
    cp_async_wait<1>();           // tile i's rows and query bytes have landed
    __syncwarp();
    const RiStage& s = st[i & 1];
    uint32_t acc = 0;
    for (int c = 0; c < nc; ++c) {
      const uint4 xw = *reinterpret_cast<const uint4*>(&s.rows[lane][c * 16]);
      const uint4 qw = *reinterpret_cast<const uint4*>(s.q + c * 16);
      acc = __dp4a(xw.x, qw.x, acc);
      acc = __dp4a(xw.y, qw.y, acc);
      acc = __dp4a(xw.z, qw.z, acc);
      acc = __dp4a(xw.w, qw.w, acc);
    }
    // every step of the reference's fp64 sum is exact on these integers
    const double v = (double)((int64_t)ta.xs - 2 * (int64_t)acc + (int64_t)ta.qs);
    unsigned long long key = lane < ta.m ? (unsigned long long)__double_as_longlong(v) : ~0ull;
    uint32_t id = ta.cid;
    const bool keep = key != ~0ull && key <= thr;
    const uint32_t bal = __ballot_sync(0xffffffffu, keep);
    const int ns = __popc(bal);
    unsigned long long* ok = pkey + (int64_t)ta.out * kk;
    uint32_t* oi = pid + (int64_t)ta.out * kk;
    if (ns <= kk) {
      if (keep) {
        const int slot = __popc(bal & ((1u << lane) - 1u));
        ok[slot] = key;
        oi[slot] = id;
      }
      if (lane >= ns && lane < kk) {
        ok[lane] = ~0ull;
        oi[lane] = 0xFFFFFFFFu;
      }
    } else {
      warp_sort_pairs(key, id);
      if (lane < kk) {
        ok[lane] = key;
        oi[lane] = id;
      }
      const unsigned long long kth = __shfl_sync(0xffffffffu, key, kk - 1);
      if (lane == 0 && kth != ~0ull) atomicMin(qthr + ta.q, kth);
    }
    __syncwarp();                 // stage i & 1 is refilled by tile i + 2
    ta = tb;
    tb = tc;
  }
  cp_async_wait<0>();
}

// ---------------------------------------------- fused count + re-rank
// Cluster mode, N_s <= 8, u8 rows with d <= 128, every query u8-exact, k <=
// 32 (config 2): k_count_enc's counting and Alg. 5, then, in the same CTA,
// the exact integer re-rank of the chunk's candidates and the top-k -- no
// candidate buffer round trip, no tile plan, no separate re-rank / top-k /
// finalize launches.  After the compaction the 64 KB score table is dead and
// becomes the warps' row staging; each warp re-ranks tiles of 32 candidates
// (one row per lane, DP4A) and keeps its best 32 (d2, id) sorted across its
// lanes (a tile is sorted and bitonic-merged in only when it beats the
// current k-th); the CTA merges its warps' lists, and rank 0 of the cluster
// merges the CTAs' lists over DSMEM and writes the query's answer.  Ties in
// d2 go to the lower id (engine.py:275).
__device__ __forceinline__ bool pair_less(unsigned long long ka, uint32_t ia, unsigned long long kb, uint32_t ib) {
  return ka < kb || (ka == kb && ia < ib);
}
// (key, id) ascending across the warp's lanes in A; B sorted ascending: A
// becomes the 32 smallest of A u B, sorted (bitonic merge)
__device__ __forceinline__ void warp_merge_sorted(unsigned long long& ak, uint32_t& ai, unsigned long long bk,
                                                  uint32_t bi) {
  const int lane = threadIdx.x & 31;
  const unsigned long long rk = __shfl_sync(0xffffffffu, bk, 31 - lane);   // B reversed: A ++ B^R is bitonic
  const uint32_t ri = __shfl_sync(0xffffffffu, bi, 31 - lane);
  if (pair_less(rk, ri, ak, ai)) {
    ak = rk;
    ai = ri;
  }
#pragma unroll
  for (int stride = 16; stride > 0; stride >>= 1) {   // half-cleaners: the bitonic 32 lowest, sorted
    const unsigned long long ok = __shfl_xor_sync(0xffffffffu, ak, stride);
    const uint32_t oi = __shfl_xor_sync(0xffffffffu, ai, stride);
    const bool lower = (lane & stride) == 0;
    const bool other_less = pair_less(ok, oi, ak, ai);
    if (lower ? other_less : (!other_less && !(ok == ak && oi == ai))) {
      ak = ok;
      ai = oi;
    }
  }
}

constexpr int FU_NT = 256;
constexpr int FU_PITCH = 144;   // row staging pitch: 16 B mod 128, conflict-free 16-byte row reads
// row staging + query bytes + warp lists, carved from the (then dead) table region
constexpr int FU_SCRATCH = ((FU_NT / 32) * 32 * FU_PITCH + 128 + 12 * FU_NT + 1023) / 1024 * 1024;

__global__ void __launch_bounds__(FU_NT, 3) k_count_fused(
    const uint16_t* __restrict__ pops, const int32_t* __restrict__ npop, int cap,
    const uint32_t* __restrict__ cenc, size_t cstride, const uint32_t* __restrict__ coffs, int n_sub, int K2,
    int64_t n, int64_t nchunks, int64_t chunk, double budget, uint32_t* __restrict__ cand, int64_t cand_cap,
    int64_t* __restrict__ flags, int64_t* __restrict__ cnum, int32_t* __restrict__ lvl,
    const uint8_t* __restrict__ Xb, int d, const uint8_t* __restrict__ Qb, const int32_t* __restrict__ qsq,
    const int32_t* __restrict__ xsq, int k, int32_t* __restrict__ out_ids, float* __restrict__ out_d) {
  constexpr int NT = FU_NT, GC = EcCfg<NT>::GC;
  extern __shared__ __align__(16) uint8_t table[];
  __shared__ EncSmem<NT> S;
  cg::cluster_group cluster = cg::this_cluster();
  const int64_t q = blockIdx.y;
  const int rank = (int)cluster.block_rank();
  const int csz = (int)cluster.num_blocks();
  const int64_t c = rank;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int64_t base = c * chunk;
  const int valid = (int)max((int64_t)0, min(chunk, n - base));
  const int tbytes = (int)(chunk / 2);
  uint32_t* gaddr = reinterpret_cast<uint32_t*>(table + max(tbytes, FU_SCRATCH));   // [GC]: staging, then the candidates
  // after the compaction the table region holds: the warps' row staging
  // (8 x 32 rows x FU_PITCH), the query bytes, the warp / CTA top lists
  uint8_t* s_q = table + (NT / 32) * 32 * FU_PITCH;
  unsigned long long (*s_key)[32] = reinterpret_cast<unsigned long long (*)[32]>(s_q + 128);
  uint32_t (*s_id)[32] = reinterpret_cast<uint32_t (*)[32]>(s_q + 128 + sizeof(unsigned long long) * NT);
  Tally T;
  enc_count_phase<NT, 2>(pops, npop, cap, cenc, cstride, coffs, n_sub, K2, nchunks, q, c, tbytes, table, gaddr, S,
                         T);
  enc_levels<NT, false>(T, table, valid, n_sub, S);
  cluster.sync();   // every CTA's level histogram is final
  for (int l = tid; l <= n_sub; l += NT) {
    int h = 0;
    for (int r = 0; r < csz; ++r) h += cluster.map_shared_rank(S.lh, r)[l];
    S.ge[l] = h;
  }
  asm volatile("barrier.cluster.arrive.relaxed.aligned;" ::: "memory");   // done reading remote histograms
  __syncthreads();
  int64_t b = 0;
  if (tid == 0) {
    int64_t cands = 0;
    const int L = alg5([&](int l) { return (int64_t)S.ge[l]; }, n_sub, budget, cands);
    int64_t mine = 0;
    for (int l = L; l <= n_sub; ++l) mine += S.lh[l];
    S.L = L;
    S.scnt = mine;
    S.fill = 0;
    if (rank == 0) {
      cnum[q] = cands;
      lvl[q] = L;
    }
    if (mine > GC) {   // more candidates than the staging holds: a global segment
      b = (int64_t)atomicAdd((unsigned long long*)&flags[3], (unsigned long long)mine);
      if (b + mine > cand_cap) flags[1] = 1;
      S.sbase = b;
    }
  }
  __syncthreads();
  const int64_t mine = S.scnt;
  const uint32_t* list = gaddr;
  if (mine <= GC) {
    compact_unordered<NT, true, true>(table, valid, (uint32_t)S.L, base, gaddr, &S.fill);
  } else if (S.sbase + mine <= cand_cap) {
    compact_unordered<NT, true, true>(table, valid, (uint32_t)S.L, base, cand + S.sbase, &S.fill);
    list = cand + S.sbase;
  }
  __syncthreads();   // the table is dead: row staging from here on
  if (tid < 32 && d >= 16 * (tid + 1))
    reinterpret_cast<uint4*>(s_q)[tid] = reinterpret_cast<const uint4*>(Qb + (size_t)q * d)[tid];
  __syncthreads();
  const bool ok_list = mine <= GC || S.sbase + mine <= cand_cap;
  // ---- re-rank: warp w takes tiles w, w + 8, ... of the chunk's candidates
  uint8_t* rows = table + (size_t)wid * 32 * FU_PITCH;
  const int nc = d / 16;
  const int32_t qs = qsq[q];
  unsigned long long bk = ~0ull;   // this warp's best 32, sorted across lanes
  uint32_t bi = 0xFFFFFFFFu;
  const int r0 = lane >> 3, cl = lane & 7;
  const int64_t ntile = ok_list ? (mine + 31) / 32 : 0;
  for (int64_t tt = wid; tt < ntile; tt += NT / 32) {
    const int64_t e = tt * 32 + lane;
    const bool have = e < mine;
    const uint32_t id = have ? list[e] : 0u;
#pragma unroll
    for (int j = 0; j < GR / 4; ++j) {   // rows j * 4 + r0, 8 lanes x 16 B per row
      const int rr = j * 4 + r0;
      const uint32_t rid = __shfl_sync(0xffffffffu, id, rr);
      if (cl < nc && tt * 32 + rr < mine) cp_async16(rows + rr * FU_PITCH + cl * 16, Xb + (size_t)rid * d + cl * 16);
    }
    cp_async_commit();
    const int32_t xs = have ? __ldg(xsq + id) : 0;
    cp_async_wait<0>();
    __syncwarp();
    uint32_t acc = 0;
    for (int cc = 0; cc < nc; ++cc) {
      const uint4 xw = *reinterpret_cast<const uint4*>(rows + lane * FU_PITCH + cc * 16);
      const uint4 qw = *reinterpret_cast<const uint4*>(s_q + cc * 16);
      acc = __dp4a(xw.x, qw.x, acc);
      acc = __dp4a(xw.y, qw.y, acc);
      acc = __dp4a(xw.z, qw.z, acc);
      acc = __dp4a(xw.w, qw.w, acc);
    }
    __syncwarp();   // the staging is refilled by the next tile
    // every step of the reference's fp64 sum is exact on these integers
    const double v = (double)((int64_t)xs - 2 * (int64_t)acc + (int64_t)qs);
    unsigned long long key = have ? (unsigned long long)__double_as_longlong(v) : ~0ull;
    uint32_t kid = have ? id : 0xFFFFFFFFu;
    const unsigned long long kth = __shfl_sync(0xffffffffu, bk, k - 1);
    const uint32_t kthi = __shfl_sync(0xffffffffu, bi, k - 1);
    if (__any_sync(0xffffffffu, pair_less(key, kid, kth, kthi))) {
      warp_sort_pairs(key, kid);
      warp_merge_sorted(bk, bi, key, kid);
    }
  }
  s_key[wid][lane] = bk;
  s_id[wid][lane] = bi;
  __syncthreads();
  if (wid == 0) {   // the CTA's best 32
    unsigned long long ak = s_key[0][lane];
    uint32_t ai = s_id[0][lane];
    for (int w = 1; w < NT / 32; ++w) warp_merge_sorted(ak, ai, s_key[w][lane], s_id[w][lane]);
    s_key[0][lane] = ak;
    s_id[0][lane] = ai;
  }
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");     // (histogram phase)
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");   // my list is written
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
  if (rank == 0 && wid == 0) {
    unsigned long long ak = s_key[0][lane];
    uint32_t ai = s_id[0][lane];
    for (int r = 1; r < csz; ++r)
      warp_merge_sorted(ak, ai, cluster.map_shared_rank(&s_key[0][0], r)[lane],
                        cluster.map_shared_rank(&s_id[0][0], r)[lane]);
    if (lane < k) {
      const bool real = ak != ~0ull;
      out_ids[q * k + lane] = real ? (int32_t)ai : -1;
      out_d[q * k + lane] = real ? __double2float_rn(__dsqrt_rn(__longlong_as_double((long long)ak)))
                                 : __int_as_float(0x7f800000);
    }
  }
  asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory");   // rank 0 is done reading
  asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory");
}

// Generic rerank for d % 4 != 0: lane = row, direct loads.
__global__ void __launch_bounds__(128) k_rerank_plain(const float* __restrict__ X, int d,
                                                      const float* __restrict__ Qf,
                                                      const int4* __restrict__ desc,
                                                      const uint32_t* __restrict__ cand, int64_t ntiles, int kk,
                                                      unsigned long long* __restrict__ pkey,
                                                      uint32_t* __restrict__ pid) {
  const int lane = threadIdx.x & 31;
  const int64_t tile = (int64_t)blockIdx.x * 4 + (threadIdx.x >> 5);
  if (tile >= ntiles) return;
  const TileRef tr = tile_ref(desc[tile], lane, cand);
  const int m = tr.m;
  const int64_t q = tr.q;
  const uint32_t cid = tr.cid;
  const float* row = X + (size_t)(lane < m ? cid : 0u) * d;
  const float* qv = Qf + (size_t)q * d;
  double a0 = 0.0, a1 = 0.0;
  const int full8 = d & ~7;
  for (int b = 0; b < full8; b += 8) {
    float xv[8], q8[8];
#pragma unroll
    for (int t = 0; t < 8; ++t) { xv[t] = row[b + t]; q8[t] = qv[b + t]; }
    einsum_block8(xv, q8, a0, a1);
  }
  for (int b = full8; b < d; b += 2) {
    const double e0 = __dsub_rn((double)row[b], (double)qv[b]);
    a0 = __dadd_rn(__dmul_rn(e0, e0), a0);
    if (b + 1 < d) {
      const double e1 = __dsub_rn((double)row[b + 1], (double)qv[b + 1]);
      a1 = __dadd_rn(__dmul_rn(e1, e1), a1);
    }
  }
  double v = __dadd_rn(a0, a1);
  v = v >= 0.0 ? v : 0.0;
  unsigned long long key = lane < m ? (unsigned long long)__double_as_longlong(v) : ~0ull;
  uint32_t id = cid;
  warp_sort_pairs(key, id);
  if (lane < kk) {
    pkey[(int64_t)tr.out * kk + lane] = key;
    pid[(int64_t)tr.out * kk + lane] = id;
  }
}

// ------------------------------------------------------------------- top-k
// One CTA per query over its tiles' partial lists: radix select of the k-th
// smallest d2 bits, then of the id among exact d2 ties (lower id wins,
// engine.py:275), bitonic sort of the kk survivors on (d2, id).
constexpr int TK_THREADS = 256;   // 512 when a query has many partial entries
constexpr int TK_MAX = 2048;

template <int NT>
__device__ void radix_select(const unsigned long long* keys, const uint32_t* ids, int64_t m, int kk,
                             bool by_id, unsigned long long key_eq, unsigned long long& out, int& remain,
                             unsigned* hist, unsigned long long* s_pre, int* s_rem) {
  const int tid = threadIdx.x;
  if (tid == 0) { *s_pre = 0ull; *s_rem = kk; }
  __syncthreads();
  unsigned long long msk = 0ull;
  const int passes = by_id ? 4 : 8;
  for (int p = 0; p < passes; ++p) {
    const int shift = (passes - 1 - p) * 8;
    for (int i = tid; i < 256; i += NT) hist[i] = 0;
    __syncthreads();
    const unsigned long long pre = *s_pre;
    // 4 keys per lane in flight; the keys of one query share their leading
    // digits, so a warp whose taken keys all fall in one bin adds once
    const int lane = tid & 31;
    for (int64_t b = tid - lane; b < m; b += 4 * NT) {
      unsigned long long v[4];
      bool in[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int64_t i = b + lane + (int64_t)u * NT;
        in[u] = i < m;
        v[u] = 0ull;
        if (in[u]) {
          if (by_id) {
            in[u] = keys[i] == key_eq;
            v[u] = (unsigned long long)ids[i];
          } else {
            v[u] = keys[i];
          }
        }
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const bool take = in[u] && (v[u] & msk) == pre;
        const unsigned dg = (unsigned)((v[u] >> shift) & 255ull);
        const unsigned tm = __ballot_sync(0xffffffffu, take);
        if (tm == 0u) continue;
        const unsigned d0 = __shfl_sync(0xffffffffu, dg, __ffs(tm) - 1);
        if (__all_sync(0xffffffffu, !take || dg == d0)) {
          if (lane == 0) atomicAdd(&hist[d0], (unsigned)__popc(tm));
        } else if (take) {
          atomicAdd(&hist[dg], 1u);   // (match.any aggregation per distinct digit measured slower: config 5 58 -> 78 ms)
        }
      }
    }
    __syncthreads();
    if (tid < 32) {   // the digit whose cumulative count reaches rem: warp 0, 8 bins per lane
      const unsigned rem = (unsigned)*s_rem;
      unsigned h[8], own = 0;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        h[u] = hist[tid * 8 + u];
        own += h[u];
      }
      unsigned inc = own;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const unsigned y = __shfl_up_sync(0xffffffffu, inc, o);
        if (tid >= o) inc += y;
      }
      // first lane whose inclusive count reaches rem (the last lane if none: digit 255)
      const unsigned bal = __ballot_sync(0xffffffffu, inc >= rem);
      const int ln = bal ? __ffs(bal) - 1 : 31;
      if (tid == ln) {
        unsigned acc = inc - own;
        int dg = tid * 8;
        for (int u = 0; u < 7; ++u, ++dg) {
          if (acc + h[u] >= rem) break;
          acc += h[u];
        }
        *s_rem = (int)(rem - acc);
        *s_pre = pre | ((unsigned long long)dg << shift);
      }
    }
    msk |= 255ull << shift;
    __syncthreads();
  }
  out = *s_pre;
  remain = *s_rem;
  __syncthreads();
}

__device__ __forceinline__ void bitonic_pairs(unsigned long long* key, uint32_t* id, int P) {
  for (int size = 2; size <= P; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = threadIdx.x; i < P; i += blockDim.x) {
        const int jx = i ^ stride;
        if (jx > i) {
          const bool up = (i & size) == 0;
          const unsigned long long ka = key[i], kb = key[jx];
          const uint32_t pa = id[i], pb = id[jx];
          const bool gt = ka > kb || (ka == kb && pa > pb);
          if (gt == up) {
            key[i] = kb; key[jx] = ka;
            id[i] = pb; id[jx] = pa;
          }
        }
      }
      __syncthreads();
    }
  }
}

// A query whose partial list is long (a level-1 query of config 5 re-ranks 4M
// candidates: one CTA's ten passes over them took 9 ms and set the kernel's
// time) is selected in two steps: the list is cut into `parts` ranges, CTA
// (q, y) of the first launch keeps range y's k best in xk / xi[(q * parts + y)
// * k ...], and a second launch (merge = 1) selects among those parts * k.
// Shorter lists are finished by CTA (q, 0) of the first launch as before.
template <int NT>
__global__ void __launch_bounds__(NT) k_topk(const unsigned long long* __restrict__ pkey,
                                                      const uint32_t* __restrict__ pid,
                                                      const int64_t* __restrict__ tstart, int S, int kk_part,
                                                      const int64_t* __restrict__ scnt, int k, int64_t id_base,
                                                      double* __restrict__ out_d2,
                                                      int64_t* __restrict__ out_ids, int parts, int64_t split_min,
                                                      unsigned long long* __restrict__ xk,
                                                      uint32_t* __restrict__ xi, int merge) {
  __shared__ unsigned hist[256];
  __shared__ unsigned long long s_pre;
  __shared__ int s_rem, s_fill;
  __shared__ int64_t s_ties, s_m, s_nt;
  __shared__ unsigned long long skey[TK_MAX];
  __shared__ uint32_t sid[TK_MAX];
  const int64_t q = blockIdx.x;
  const int tid = threadIdx.x;
  if (tid == 0) {
    s_m = 0;
    s_nt = 0;
    s_fill = 0;
    s_ties = 0;
  }
  __syncthreads();
  {   // candidates and tiles of the query's S segments (S = 763 at config 5: not one thread's loop)
    int64_t c = 0, nt = 0;
    for (int r = tid; r < S; r += NT) {
      const int64_t v = scnt[q * S + r];
      c += v;
      nt += (v + GR - 1) / GR;
    }
    for (int o = 16; o > 0; o >>= 1) {
      c += __shfl_xor_sync(0xffffffffu, c, o);
      nt += __shfl_xor_sync(0xffffffffu, nt, o);
    }
    if ((tid & 31) == 0 && nt) {
      atomicAdd((unsigned long long*)&s_m, (unsigned long long)c);
      atomicAdd((unsigned long long*)&s_nt, (unsigned long long)nt);
    }
  }
  __syncthreads();
  // the query's tiles are consecutive in the plan's processing order
  const int64_t lo = tstart[q * S] * kk_part;
  int64_t m = s_nt * kk_part;
  const bool split = parts > 1 && m > split_min;
  if (merge ? !split : (!split && blockIdx.y > 0)) return;   // (block-uniform)
  int kk = (int)min((int64_t)k, s_m);
  const unsigned long long* keys = pkey + lo;
  const uint32_t* ids = pid + lo;
  const bool part = split && !merge;
  if (part) {   // range y of the list; its real entries (padding slots hold all-ones keys)
    const int64_t per = (m + parts - 1) / parts;
    const int64_t b0 = min(m, (int64_t)blockIdx.y * per), b1 = min(m, b0 + per);
    keys += b0;
    ids += b0;
    m = b1 - b0;
    int64_t real = 0;
    for (int64_t i = tid; i < m; i += NT) real += keys[i] != ~0ull;
    for (int o = 16; o > 0; o >>= 1) real += __shfl_xor_sync(0xffffffffu, real, o);
    if ((tid & 31) == 0 && real) atomicAdd((unsigned long long*)&s_ties, (unsigned long long)real);
    __syncthreads();
    kk = (int)min((int64_t)k, s_ties);
    __syncthreads();
    if (tid == 0) s_ties = 0;
    __syncthreads();
  } else if (merge) {
    keys = xk + (size_t)q * parts * k;
    ids = xi + (size_t)q * parts * k;
    m = (int64_t)parts * k;
  }
  if (kk > 0) {
    unsigned long long tau;
    int take;
    radix_select<NT>(keys, ids, m, kk, false, 0ull, tau, take, hist, &s_pre, &s_rem);
    int64_t nties = 0;
    for (int64_t i = tid; i < m; i += NT) nties += keys[i] == tau;
    for (int o = 16; o > 0; o >>= 1) nties += __shfl_xor_sync(0xffffffffu, nties, o);
    if ((tid & 31) == 0 && nties) atomicAdd((unsigned long long*)&s_ties, (unsigned long long)nties);
    __syncthreads();
    unsigned long long pi = ~0ull;
    if (s_ties > take) {
      int dummy;
      radix_select<NT>(keys, ids, m, take, true, tau, pi, dummy, hist, &s_pre, &s_rem);
    }
    for (int64_t i = tid; i < m; i += NT) {
      const unsigned long long kv = keys[i];
      if (kv < tau || (kv == tau && (unsigned long long)ids[i] <= pi)) {
        const int slot = atomicAdd(&s_fill, 1);
        skey[slot] = kv;
        sid[slot] = ids[i];
      }
    }
    __syncthreads();
  }
  if (part) {   // the range's best kk (unsorted), all-ones padding to k
    unsigned long long* ok = xk + ((size_t)q * parts + blockIdx.y) * k;
    uint32_t* oi = xi + ((size_t)q * parts + blockIdx.y) * k;
    for (int r = tid; r < k; r += NT) {
      ok[r] = r < kk ? skey[r] : ~0ull;
      oi[r] = r < kk ? sid[r] : 0xFFFFFFFFu;
    }
    return;
  }
  int P = 1;
  while (P < kk) P <<= 1;
  for (int i = kk + tid; i < P; i += NT) {
    skey[i] = ~0ull;
    sid[i] = 0xFFFFFFFFu;
  }
  __syncthreads();
  bitonic_pairs(skey, sid, P);
  for (int r = tid; r < k; r += NT) {
    if (r < kk) {
      out_d2[q * k + r] = __longlong_as_double((long long)skey[r]);
      out_ids[q * k + r] = (int64_t)sid[r] + id_base;
    } else {
      out_d2[q * k + r] = __longlong_as_double(0x7ff0000000000000LL);
      out_ids[q * k + r] = -1;
    }
  }
}

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
constexpr int64_t kSuperTile = 16384;

// 4-bit score tables whenever a score (<= n_sub) fits a nibble: half the
// shared memory per CTA, so 4 CTAs of 256 threads share an SM.
static inline bool nib_tables(const taco_index* idx) { return idx->n_sub <= 15; }
static inline size_t table_bytes(const taco_index* idx) {
  return (size_t)(nib_tables(idx) ? idx->chunk / 2 : idx->chunk);
}

static int64_t super_tile(const taco_index* idx, int cap) {
  const int64_t per = (int64_t)idx->n_sub * (2LL * cap + 20LL * idx->kp + 16) + 8LL * (idx->d + idx->D) + 64;
  int64_t Q = (int64_t)(1ll << 30) / std::max<int64_t>(per, 1);
  if (!idx->cluster_mode) {   // + the spilled count tables: 8 GiB per tile
    const int64_t tb = (idx->n_sub <= 15 ? idx->chunk / 2 : idx->chunk) * idx->nchunks;
    Q = std::min<int64_t>(Q, (int64_t)(8ll << 30) / std::max<int64_t>(tb, 1));
  }
  return std::max<int64_t>(64, std::min<int64_t>(Q, kSuperTile));
}

static int ensure_front(taco_index* idx, QueryTile& t, int64_t QS, int k) {
  if (t.pop_cap == 0) t.pop_cap = std::min(idx->K, 1024);
  const size_t QN = (size_t)QS * idx->n_sub;
  TACO_TRY(t.Q.ensure(sizeof(float) * (size_t)QS * idx->d));
  TACO_TRY(t.qt.ensure(sizeof(float) * (size_t)QS * idx->D));
  TACO_TRY(t.sd.ensure(sizeof(double) * QN * 2 * idx->kp));
  TACO_TRY(t.sl.ensure(sizeof(uint16_t) * QN * 2 * idx->kp));
  TACO_TRY(t.pops.ensure(sizeof(uint16_t) * QN * t.pop_cap));
  TACO_TRY(t.npop.ensure(sizeof(int32_t) * QN));
  TACO_TRY(t.ret.ensure(sizeof(int64_t) * QN));
  TACO_TRY(t.flags.ensure(sizeof(int64_t) * 8));
  if (!t.flags_h) TACO_CHECK_CUDA(cudaMallocHost(&t.flags_h, sizeof(int64_t) * 8));
  TACO_TRY(t.lvl.ensure(sizeof(int32_t) * QS));
  TACO_TRY(t.cnum.ensure(sizeof(int64_t) * QS));
  const int64_t S = idx->nchunks;   // candidate segments per query (re-rank plan)
  const int64_t SC = idx->cluster_mode ? idx->nchunks : 1;   // count-side segments (clocal / qbase)
  TACO_TRY(t.clocal.ensure(sizeof(int64_t) * QS * SC));
  TACO_TRY(t.qbase.ensure(sizeof(int64_t) * QS * SC));
  TACO_TRY(t.bpref.ensure(sizeof(int64_t) * (QS * S + 1)));
  if (!idx->cluster_mode) {
    TACO_TRY(t.gsb.ensure(sizeof(int64_t) * QS * S));
    TACO_TRY(t.gsc.ensure(sizeof(int64_t) * QS * S));
  }
  TACO_TRY(t.tk_d2.ensure(sizeof(double) * (size_t)QS * std::max(k, 1)));
  TACO_TRY(t.tk_ids.ensure(sizeof(int64_t) * (size_t)QS * std::max(k, 1)));
  TACO_TRY(t.out_ids.ensure(sizeof(int32_t) * (size_t)QS * std::max(k, 1)));
  TACO_TRY(t.out_d.ensure(sizeof(float) * (size_t)QS * std::max(k, 1)));
  if (!idx->cluster_mode) {
    TACO_TRY(t.gtab.ensure(table_bytes(idx) * (size_t)QS * idx->nchunks));   // spilled count tables
    TACO_TRY(t.part.ensure(sizeof(int32_t) * (size_t)QS * idx->nchunks * (idx->n_sub + 1)));
    TACO_TRY(t.hist.ensure(sizeof(int64_t) * (size_t)QS * (idx->n_sub + 1)));
    TACO_TRY(t.coff.ensure(sizeof(int64_t) * (size_t)QS * idx->nchunks));
  }
  return TACO_OK;
}

static int ensure_cand(QueryTile& t, int64_t want) {
  if (want > t.cand_cap) {
    TACO_TRY(t.cand.ensure(sizeof(uint32_t) * (size_t)want));
    t.cand_cap = want;
  }
  return TACO_OK;
}

static int check_query_ready(taco_index* idx, double alpha, int k) {
  TACO_TRY(index_check(idx));
  if (!idx->has_model || !idx->has_cb || !idx->has_cells || !idx->has_gsize)
    TACO_FAIL(TACO_ERR_STATE, "index is not built (model %d codebooks %d cells %d sizes %d)",
              idx->has_model, idx->has_cb, idx->has_cells, idx->has_gsize);
  if (!(alpha > 0.0 && alpha <= 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "collision ratio %g outside (0, 1]", alpha);
  if (k < 1 || k > TK_MAX) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d outside [1, %d]", k, TK_MAX);
  if (idx->d > 4096) TACO_FAIL(TACO_ERR_PARAMETER, "dimension %d exceeds 4096", idx->d);
  return TACO_OK;
}

static int64_t retrieval_target(double alpha, int64_t n) {
  const double t = std::ceil(alpha * (double)n);   // imi.py:109-112 (Python float math)
  return std::min<int64_t>(n, (int64_t)t);
}

// transform + centroid ranks + traversal for QS queries resident in t.Q
// Queries [q0, q0 + QS) of the tile buffers (q0 > 0: one rank's slice of a
// split traversal, taco_query_front_device).
static int stage_front(taco_index* idx, QueryTile& t, int64_t QS, double alpha, cudaStream_t st,
                       double* keys_out, int64_t q0 = 0) {
  const int kp = idx->kp;
  if (QS == 0) return TACO_OK;
  const size_t qn0 = (size_t)q0 * idx->n_sub;
  float* qt = t.qt.as<float>() + (size_t)q0 * idx->D;
  double* sd = t.sd.as<double>() + qn0 * 2 * kp;
  uint16_t* sl = t.sl.as<uint16_t>() + qn0 * 2 * kp;
  {
    ProfScope ps(K_TRANSFORM, st);
    TACO_TRY(launch_transform(st, t.Q.as<float>() + (size_t)q0 * idx->d, QS, idx->d, idx->D,
                              idx->mean.as<float>(), idx->M.as<float>(), qt, false));
  }
  {
    const int64_t warps = QS * idx->n_sub * 2;
    const int wpb = 8;
    ProfScope ps(K_CSORT, st);
    k_csort<<<(unsigned)ceil_div(warps, wpb), wpb * 32, sizeof(double) * kp * wpb, st>>>(
        qt, (int)QS, idx->n_sub, idx->s, idx->m1, idx->m2, kp, idx->cb1.as<float>(),
        idx->cb2.as<float>(), sd, sl);
    TACO_LAUNCHED();
  }
  {
    const int64_t th = QS * idx->n_sub;
    const int64_t target = retrieval_target(alpha, idx->n_global);
    (void)th;
    ProfScope ps(K_TRAVERSE, st);
    TACO_TRY(launch_traverse(sd, sl, idx->gsize.as<int64_t>(), QS, idx->n_sub, kp, target,
                             t.pops.as<uint16_t>() + qn0 * t.pop_cap, t.pop_cap, keys_out, t.npop.as<int32_t>() + qn0,
                             t.ret.as<int64_t>() + qn0, t.flags.as<int64_t>(), st));
    TACO_LAUNCHED();
  }
  return TACO_OK;
}


// Entries per unit of the encoded count CSR, 0 = none (TACO_COUNT_TMA=0, or
// layouts it does not cover): cluster mode 8-entry units (k_count_enc /
// k_count_tma), global mode 4-entry units (k_count_genc); 4-bit tables with
// N_s <= 8, and padding to whole units below ~n entries per subspace (large
// K' with short slices keeps the unit-staged kernels).
static int enc_unit(const taco_index* idx) {
  const char* e = getenv("TACO_COUNT_TMA");   // read per index (tests pin both kernels)
  // cluster mode: N_s <= 16 (4-bit lanes to 15, 8-bit lanes at 16); global mode: N_s <= 8
  if ((e && e[0] == '0') || idx->n_sub > (idx->cluster_mode ? 16 : 8) || idx->chunk > kClusterWideChunk) return 0;
  const int U = idx->cluster_mode ? 8 : 4;
  const int64_t nsl = idx->nchunks * (int64_t)idx->kp * idx->kp;
  return (U - 1) * nsl <= idx->n ? U : 0;
}

int build_count_csr(taco_index* idx) {
  idx->has_ccsr = false;
  const int U = enc_unit(idx);
  if (!U) {
    idx->cenc.release();
    idx->coffs.release();
    return TACO_OK;
  }
  const int64_t K2 = (int64_t)idx->kp * idx->kp, nsl = idx->nchunks * K2;
  const size_t offs_len = (size_t)nsl + 1;
  idx->cunit = U;
  idx->cstride = (size_t)ceil_div(idx->n + (U - 1) * nsl, U) * U;
  TACO_TRY(idx->cenc.ensure(sizeof(uint32_t) * idx->cstride * idx->n_sub));
  TACO_TRY(idx->coffs.ensure(sizeof(uint32_t) * offs_len * idx->n_sub));
  const int nb = (int)ceil_div(nsl, CC_NT);
  DevBuf bsum;
  TACO_TRY(bsum.ensure(sizeof(uint32_t) * (size_t)nb * idx->n_sub));
  cudaStream_t st = idx->stream;
  TACO_CHECK_CUDA(cudaMemsetAsync(idx->coffs.p, 0, sizeof(uint32_t) * offs_len * idx->n_sub, st));
  k_ccsr_sums<<<dim3((unsigned)nb, (unsigned)idx->n_sub), CC_NT, 0, st>>>(idx->offs.as<uint32_t>(), offs_len, nsl,
                                                                       bsum.as<uint32_t>(), U);
  TACO_LAUNCHED();
  k_ccsr_scan<<<(unsigned)idx->n_sub, CC_NT, 0, st>>>(bsum.as<uint32_t>(), nb);
  TACO_LAUNCHED();
  k_ccsr_fill<<<dim3((unsigned)nb, (unsigned)idx->n_sub), CC_NT, 0, st>>>(
      idx->ids.as<uint32_t>(), idx->offs.as<uint32_t>(), offs_len, nsl, (int)K2, idx->n, idx->chunk,
      bsum.as<uint32_t>(), idx->coffs.as<uint32_t>(), idx->cenc.as<uint32_t>(), idx->cstride, U,
      nib_tables(idx) ? 1 : 0);
  TACO_LAUNCHED();
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  bsum.release();
  idx->has_ccsr = true;
  return TACO_OK;
}

static int set_count_attrs(taco_index*) {
  static bool done = false;
  if (!done) {
    const int mx = (int)kClusterMaxChunk;
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_cluster<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_cluster<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_cluster<true>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_cluster<false>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_tma, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint4) * TC_RS * TC_SG)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_tma, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint32_t) * EcCfg<256>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint32_t) * EcCfg<256>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3, 8>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3, 0, true, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint32_t) * EcCfg<256>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3, 0, true, true>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3, 16, false, true>,
                                         cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk8 + sizeof(uint32_t) * EcCfg<256>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<256, 3, 16, false, true>,
                                         cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<512, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint32_t) * EcCfg<512>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<512, 2>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<1024, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterWideChunk / 2 + sizeof(uint32_t) * EcCfg<1024>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_enc<1024, 1>, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_genc<256, 3>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint32_t) * EcCfg<256>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, mx));
    done = true;
  }
  return TACO_OK;
}

// global mode, sweep 1: level histograms of every (chunk, query) -> t.hist
static int global_count(taco_index* idx, QueryTile& t, int64_t QS, cudaStream_t st) {
  TACO_TRY(set_count_attrs(idx));
  if (idx->has_ccsr) {   // encoded CSR (4-entry units)
    dim3 g((unsigned)idx->nchunks, (unsigned)QS);
    ProfScope ps(K_COUNT, st);
    k_count_genc<256, 3><<<g, 256, table_bytes(idx) + sizeof(uint32_t) * EcCfg<256>::GC, st>>>(
        t.pops.as<uint16_t>(), t.npop.as<int32_t>(), t.pop_cap, idx->cenc.as<uint32_t>(), idx->cstride,
        idx->coffs.as<uint32_t>(), idx->n_sub, idx->K, idx->n, idx->nchunks, idx->chunk, t.gtab.as<uint8_t>(),
        t.part.as<int32_t>());
    TACO_LAUNCHED();
  } else {
    dim3 g((unsigned)idx->nchunks, (unsigned)QS);
    ProfScope ps(K_COUNT, st);
    auto kern = nib_tables(idx) ? k_count<true> : k_count<false>;
    kern<<<g, CT_THREADS, table_bytes(idx), st>>>(
        t.pops.as<uint16_t>(), t.npop.as<int32_t>(), t.pop_cap, idx->ids.as<uint32_t>(), idx->offs.as<uint32_t>(),
        idx->n_sub, idx->K, idx->n, idx->nchunks, idx->chunk, CNT_HIST, t.gtab.as<uint8_t>(), t.part.as<int32_t>(),
        nullptr, nullptr, nullptr, nullptr, nullptr);
    TACO_LAUNCHED();
  }
  {
    ProfScope ps(K_HIST, st);
    k_hist_reduce<<<(unsigned)QS, 64, 0, st>>>(t.part.as<int32_t>(), idx->nchunks, idx->n_sub, t.hist.as<int64_t>());
    TACO_LAUNCHED();
  }
  return TACO_OK;
}

static int num_sms();

// global mode: Alg. 5 on `ghist`, then sweep 2 emits (records, else recount)
static int global_select(taco_index* idx, QueryTile& t, int64_t QS, const int64_t* ghist, double beta,
                         cudaStream_t st) {
  const double budget = beta * (double)idx->n_global;   // engine.py:240
  {
    ProfScope ps(K_SELECT, st);
    k_select<<<(unsigned)ceil_div(QS * 32, 256), 256, 0, st>>>(
        ghist, t.part.as<int32_t>(), QS, idx->nchunks, idx->n_sub, budget, t.coff.as<int64_t>(), t.cand_cap,
        t.flags.as<int64_t>(), t.qbase.as<int64_t>(), t.clocal.as<int64_t>(), t.cnum.as<int64_t>(),
        t.lvl.as<int32_t>(), t.gsb.as<int64_t>(), t.gsc.as<int64_t>());
    TACO_LAUNCHED();
  }
  {
    ProfScope ps(K_COMPACT, st);
    const int64_t pairs = QS * idx->nchunks;
    TACO_TRY(t.rlist.ensure(sizeof(int64_t) * (size_t)(pairs + 1)));
    TACO_CHECK_CUDA(cudaMemsetAsync(t.rlist.p, 0, sizeof(int64_t), st));
    auto ek = nib_tables(idx) ? k_emit_rec<true> : k_emit_rec<false>;
    ek<<<(unsigned)ceil_div(pairs, ER_WARPS), 32 * ER_WARPS, 0, st>>>(
        t.gtab.as<uint8_t>(), idx->n, idx->nchunks, idx->chunk, idx->n_sub, QS, t.part.as<int32_t>(),
        t.lvl.as<int32_t>(), t.qbase.as<int64_t>(), t.clocal.as<int64_t>(), t.coff.as<int64_t>(), t.cand_cap,
        t.cand.as<uint32_t>(), t.rlist.as<int64_t>());
    TACO_LAUNCHED();
    // recount the listed pairs: persistent CTAs, as many as are co-resident
    auto kern = nib_tables(idx) ? k_count<true> : k_count<false>;
    const int64_t ctas = std::min<int64_t>(pairs, (int64_t)num_sms() * 4);
    kern<<<(unsigned)ctas, CT_THREADS, table_bytes(idx), st>>>(
        t.pops.as<uint16_t>(), t.npop.as<int32_t>(), t.pop_cap, idx->ids.as<uint32_t>(), idx->offs.as<uint32_t>(),
        idx->n_sub, idx->K, idx->n, idx->nchunks, idx->chunk, CNT_EMIT, nullptr, nullptr, t.lvl.as<int32_t>(),
        t.qbase.as<int64_t>(), t.coff.as<int64_t>(), t.cand.as<uint32_t>(), t.rlist.as<int64_t>());
    TACO_LAUNCHED();
  }
  return TACO_OK;
}

static int cluster_count(taco_index* idx, QueryTile& t, int64_t QS, double beta, cudaStream_t st) {
  TACO_TRY(set_count_attrs(idx));
  const double budget = beta * (double)idx->n_global;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)idx->nchunks, (unsigned)QS, 1);
  cfg.blockDim = dim3(CT_THREADS, 1, 1);
  cfg.dynamicSmemBytes = table_bytes(idx);
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = (unsigned)idx->nchunks;
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  ProfScope ps(K_COUNT, st);
  {
    static int dbg = -1;
    if (dbg < 0) {
      const char* e = getenv("TACO_COUNT_DBG");
      dbg = e ? atoi(e) : 0;
      if (dbg) TACO_CHECK_CUDA(cudaMemcpyToSymbol(g_count_dbg, &dbg, sizeof(int)));
    }
  }
  if (idx->has_ccsr) {
    const char* fe = getenv("TACO_COUNT_FEED");   // =tma: the cp.async.bulk ring feed
    const int feed = (fe && !strcmp(fe, "tma")) ? 1 : 0;
    const char* ne = getenv("TACO_COUNT_NT");   // 256 (3 CTAs per SM, default), 512 (2 per SM) or 1024 (1 per SM)
    const int nt = ne ? atoi(ne) : 256;
    const bool big = idx->n_sub > 8;   // 16 tally levels (4-bit lanes to N_s = 15, 8-bit at 16)
    const bool wide = !big && nt == 512, huge = !big && (nt == 1024 || idx->chunk > kClusterMaxChunk);
    const bool tfeed = feed && !big;
    cfg.blockDim = dim3(tfeed ? TC_THREADS : huge ? 1024 : wide ? 512 : 256, 1, 1);
    cfg.dynamicSmemBytes = table_bytes(idx) + (tfeed ? sizeof(uint4) * TC_RS * TC_SG
                                                     : sizeof(uint32_t) * (huge ? EcCfg<1024>::GC
                                                                           : wide ? EcCfg<512>::GC : EcCfg<256>::GC));
    // TACO_COUNT_PG=0 (read per batch): hardware clusters (k_count_enc) instead of persistent software groups
    const char* pe = getenv("TACO_COUNT_PG");
    const bool pg_on = !(pe && pe[0] == '0');
    // (a one-CTA query has no cluster to outgrow: the per-query launch balances better there)
    if (pg_on && idx->nchunks > 1 && !tfeed && !wide && !huge) {
      auto pk = big ? (nib_tables(idx) ? k_count_pg<256, 3, 0, true, true> : k_count_pg<256, 3, 16, false, true>)
                : idx->n_sub == 8 ? k_count_pg<256, 3, 8> : k_count_pg<256, 3>;
      static int slots[4] = {0, 0, 0, 0};   // co-resident CTAs of each instantiation ...
      static size_t slots_smem[4] = {0, 0, 0, 0};   // ... at this launch's shared-memory size
      static bool attr_set[4] = {false, false, false, false};
      const int which = big ? (nib_tables(idx) ? 0 : 1) : idx->n_sub == 8 ? 2 : 3;
      const size_t smem = table_bytes(idx) + sizeof(uint32_t) * EcCfg<256>::GC;
      if (!attr_set[which]) {
        const int smem_max =
            (int)((which == 1 ? kClusterMaxChunk8 : kClusterMaxChunk / 2) + sizeof(uint32_t) * EcCfg<256>::GC);
        TACO_CHECK_CUDA(cudaFuncSetAttribute(pk, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_max));
        attr_set[which] = true;
      }
      if (slots_smem[which] != smem) {
        int per_sm = 0;
        TACO_CHECK_CUDA(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, pk, 256, smem));
        slots[which] = per_sm * num_sms();
        slots_smem[which] = smem;
        if (slots[which] <= 0) TACO_FAIL(TACO_ERR_CUDA, "k_count_pg does not fit an SM");
      }
      const int64_t csz = idx->nchunks;
      const int64_t ngrp = std::min<int64_t>(QS, slots[which] / csz);
      if (ngrp >= 1) {
        const int LV = idx->n_sub + 1;
        const size_t xb = sizeof(int32_t) * (size_t)QS * (size_t)csz * LV;
        TACO_TRY(t.xch.ensure(xb));
        if (csz > 1) TACO_CHECK_CUDA(cudaMemsetAsync(t.xch.p, 0, xb, st));
        const uint16_t* a_pops = t.pops.as<uint16_t>();
        const int32_t* a_npop = t.npop.as<int32_t>();
        int a_cap = t.pop_cap;
        const uint32_t* a_cenc = idx->cenc.as<uint32_t>();
        size_t a_cstride = idx->cstride;
        const uint32_t* a_coffs = idx->coffs.as<uint32_t>();
        int a_nsub = idx->n_sub, a_K = idx->K;
        int64_t a_n = idx->n, a_nch = idx->nchunks, a_chunk = idx->chunk;
        double a_budget = budget;
        uint32_t* a_cand = t.cand.as<uint32_t>();
        int64_t a_ccap = t.cand_cap;
        int64_t *a_flags = t.flags.as<int64_t>(), *a_sb = t.qbase.as<int64_t>(), *a_sc = t.clocal.as<int64_t>(),
                *a_cnum = t.cnum.as<int64_t>();
        int32_t* a_lvl = t.lvl.as<int32_t>();
        int64_t a_Q = QS;
        int32_t* a_xch = t.xch.as<int32_t>();
        void* args[] = {&a_pops, &a_npop, &a_cap, &a_cenc, &a_cstride, &a_coffs, &a_nsub, &a_K, &a_n, &a_nch, &a_chunk,
                        &a_budget, &a_cand, &a_ccap, &a_flags, &a_sb, &a_sc, &a_cnum, &a_lvl, &a_Q, &a_xch};
        // cooperative: the whole grid is co-resident while it runs (the groups poll each other)
        TACO_CHECK_CUDA(cudaLaunchCooperativeKernel((const void*)pk, dim3((unsigned)(ngrp * csz)), dim3(256), args,
                                                    smem, st));
        TACO_LAUNCHED();
        return TACO_OK;
      }
    }
    auto kern = tfeed ? k_count_tma
                : big ? (nib_tables(idx) ? k_count_enc<256, 3, 0, true, true> : k_count_enc<256, 3, 16, false, true>)
                : huge ? k_count_enc<1024, 1>
                : wide ? k_count_enc<512, 2>
                : idx->n_sub == 8 ? k_count_enc<256, 3, 8> : k_count_enc<256, 3>;
    TACO_CHECK_CUDA(cudaLaunchKernelEx(&cfg, kern,
                                       (const uint16_t*)t.pops.as<uint16_t>(),
                                       (const int32_t*)t.npop.as<int32_t>(), t.pop_cap,
                                       (const uint32_t*)idx->cenc.as<uint32_t>(), idx->cstride,
                                       (const uint32_t*)idx->coffs.as<uint32_t>(), idx->n_sub, idx->K, idx->n,
                                       idx->nchunks, idx->chunk, budget, t.cand.as<uint32_t>(), t.cand_cap,
                                       t.flags.as<int64_t>(), t.qbase.as<int64_t>(), t.clocal.as<int64_t>(),
                                       t.cnum.as<int64_t>(), t.lvl.as<int32_t>()));
    TACO_LAUNCHED();
    return TACO_OK;
  }
  TACO_CHECK_CUDA(cudaLaunchKernelEx(&cfg, nib_tables(idx) ? k_count_cluster<true> : k_count_cluster<false>,
                                     (const uint16_t*)t.pops.as<uint16_t>(),
                                     (const int32_t*)t.npop.as<int32_t>(), t.pop_cap,
                                     (const uint32_t*)idx->ids.as<uint32_t>(),
                                     (const uint32_t*)idx->offs.as<uint32_t>(), idx->n_sub, idx->K, idx->n,
                                     idx->nchunks, idx->chunk, budget, t.cand.as<uint32_t>(), t.cand_cap,
                                     t.flags.as<int64_t>(), t.qbase.as<int64_t>(), t.clocal.as<int64_t>(),
                                     t.cnum.as<int64_t>(), t.lvl.as<int32_t>()));  // segment base/count per (q, rank)
  TACO_LAUNCHED();
  return TACO_OK;
}

// The fused count + re-rank (k_count_fused) applies to this tile?  Needs the
// encoded CSR in cluster mode, u8 rows with d <= 128 (d % 16 == 0), k <= 32
// and every query u8-exact (q_u8_prep's flags[4], read back by the caller).
// Opt-in (TACO_FUSED=1): measured slower at config 2 (10.9 ms against 5.6 +
// 1.75 + 0.38 for the separate kernels) -- re-ranking per query inside the
// count CTA loses the chunk-major order's L2 reuse of the candidate rows
// (each row serves ~100 queries of a batch), so the rows stream from HBM.
static bool fused_eligible(const taco_index* idx, int k) {
  const char* e = getenv("TACO_FUSED");
  return (e && e[0] == '1') && idx->cluster_mode && idx->n_sub <= 8 && idx->has_ccsr && idx->cunit == 8 &&
         idx->xfmt == TACO_ROWS_U8 && idx->d <= 128 && idx->d % 16 == 0 && k <= 32 && idx->Xsq.p;
}

static int cluster_count_fused(taco_index* idx, QueryTile& t, int64_t QS, double beta, int k, cudaStream_t st) {
  TACO_TRY(set_count_attrs(idx));
  static bool attr = false;
  const size_t smem = (size_t)std::max<int64_t>(table_bytes(idx), FU_SCRATCH) + sizeof(uint32_t) * EcCfg<FU_NT>::GC;
  if (!attr) {
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_fused, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)(kClusterMaxChunk / 2 + sizeof(uint32_t) * EcCfg<FU_NT>::GC)));
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_count_fused, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
    attr = true;
  }
  const double budget = beta * (double)idx->n_global;
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3((unsigned)idx->nchunks, (unsigned)QS, 1);
  cfg.blockDim = dim3(FU_NT, 1, 1);
  cfg.dynamicSmemBytes = smem;
  cfg.stream = st;
  cudaLaunchAttribute attr_c[1];
  attr_c[0].id = cudaLaunchAttributeClusterDimension;
  attr_c[0].val.clusterDim.x = (unsigned)idx->nchunks;
  attr_c[0].val.clusterDim.y = 1;
  attr_c[0].val.clusterDim.z = 1;
  cfg.attrs = attr_c;
  cfg.numAttrs = 1;
  ProfScope ps(K_COUNT, st);
  TACO_CHECK_CUDA(cudaLaunchKernelEx(&cfg, k_count_fused, (const uint16_t*)t.pops.as<uint16_t>(),
                                     (const int32_t*)t.npop.as<int32_t>(), t.pop_cap,
                                     (const uint32_t*)idx->cenc.as<uint32_t>(), idx->cstride,
                                     (const uint32_t*)idx->coffs.as<uint32_t>(), idx->n_sub, idx->K, idx->n,
                                     idx->nchunks, idx->chunk, budget, t.cand.as<uint32_t>(), t.cand_cap,
                                     t.flags.as<int64_t>(), t.cnum.as<int64_t>(), t.lvl.as<int32_t>(),
                                     (const uint8_t*)idx->Xn.as<uint8_t>(), idx->d,
                                     (const uint8_t*)t.qb.as<uint8_t>(), (const int32_t*)t.qsq.as<int32_t>(),
                                     (const int32_t*)idx->Xsq.as<int32_t>(), k, t.out_ids.as<int32_t>(),
                                     t.out_d.as<float>()));
  TACO_LAUNCHED();
  return TACO_OK;
}

// Tile plans: query-major output positions (t.bpref, for the top-k) and, in
// cluster mode, the chunk-major processing order (t.ppref): all queries'
// candidates in one id chunk are re-ranked before the next chunk, so the
// rows they share (each row is a candidate of ~beta*alpha-proportional many
// queries of a batch) are read from HBM about once and then served by L2.
// launches the plans and an async copy of flags[0..3] into t.flags_h (read after a stream sync)
// candidate segments per query: cluster mode (q, rank) in qbase/clocal; global
// mode (q, chunk) in gsb/gsc (k_select) -- both re-ranked chunk-major
static inline int64_t seg_per_query(const taco_index* idx) { return idx->nchunks; }
static inline const int64_t* seg_base(const taco_index* idx, const QueryTile& t) {
  return idx->cluster_mode ? t.qbase.as<int64_t>() : t.gsb.as<int64_t>();
}
static inline const int64_t* seg_cnt(const taco_index* idx, const QueryTile& t) {
  return idx->cluster_mode ? t.clocal.as<int64_t>() : t.gsc.as<int64_t>();
}

// flags[6] = the largest per-query candidate count of the tile (the top-k splits long lists)
__global__ void k_max_i64(const int64_t* __restrict__ v, int64_t n, int64_t* __restrict__ out) {
  const int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  long long x = i < n ? (long long)v[i] : 0;
  for (int o = 16; o > 0; o >>= 1) x = max(x, __shfl_xor_sync(0xffffffffu, x, o));
  if ((threadIdx.x & 31) == 0 && x > 0) atomicMax((long long*)out, x);
}
static int plan_async(taco_index* idx, QueryTile& t, int64_t QS, cudaStream_t st) {
  const int64_t S = seg_per_query(idx);
  {
    ProfScope ps(K_PLAN, st);
    const int64_t nseg = QS * S, nb = ceil_div(nseg, PLAN_NT);
    TACO_TRY(t.psum.ensure(sizeof(int64_t) * 2 * (size_t)nb));
    if (S > 1) TACO_TRY(t.ppref.ensure(sizeof(int64_t) * (size_t)(nseg + 1)));
    k_plan_sums<<<(unsigned)nb, PLAN_NT, 0, st>>>(seg_cnt(idx, t), nseg, (int)S, QS, t.psum.as<int64_t>());
    TACO_LAUNCHED();
    k_plan_scan<<<(unsigned)nb, PLAN_NT, 0, st>>>(seg_cnt(idx, t), nseg, (int)S, QS, t.psum.as<int64_t>(),
                                                  t.bpref.as<int64_t>(), S > 1 ? t.ppref.as<int64_t>() : nullptr,
                                                  t.flags.as<int64_t>());
    TACO_LAUNCHED();
  }
  k_max_i64<<<(unsigned)ceil_div(QS, 256), 256, 0, st>>>(t.cnum.as<int64_t>(), QS, t.flags.as<int64_t>() + 6);
  TACO_LAUNCHED();
  TACO_CHECK_CUDA(cudaMemcpyAsync(t.flags_h, t.flags.p, sizeof(int64_t) * 7, cudaMemcpyDeviceToHost, st));
  return TACO_OK;
}

static int plan_and_read(taco_index* idx, QueryTile& t, int64_t QS, cudaStream_t st, int64_t fl[4]) {
  TACO_TRY(plan_async(idx, t, QS, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  for (int i = 0; i < 4; ++i) fl[i] = t.flags_h[i];
  return TACO_OK;
}

static int g_num_sms = 0;
static int num_sms() {
  if (!g_num_sms) {
    int dev = 0;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&g_num_sms, cudaDevAttrMultiProcessorCount, dev);
  }
  return g_num_sms;
}

struct IntRerank {   // integer path inputs (u8 rows only); all null = off
  const uint8_t* Qb = nullptr;
  const uint8_t* qok = nullptr;
  const int32_t* qsq = nullptr;
  const int32_t* xsq = nullptr;
};

template <typename T>
static int launch_rerank_async(const void* X, int d, const float* Qf, const int4* desc, const uint32_t* cand,
                               int64_t ntiles, int kk, unsigned long long* pkey, uint32_t* pid,
                               unsigned long long* qthr, const IntRerank& ir, cudaStream_t st) {
  constexpr int WARPS = RowFmt<T>::WARPS;
  const size_t smem = sizeof(AWarpSmem<T>) * WARPS;
  static bool attr = false;
  if (!attr) {
    TACO_CHECK_CUDA(cudaFuncSetAttribute(k_rerank_async<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    attr = true;
  }
  const int64_t grid = std::min<int64_t>(ceil_div(ntiles, WARPS), (int64_t)num_sms() * RowFmt<T>::CTAS);
  k_rerank_async<T><<<(unsigned)grid, 32 * WARPS, smem, st>>>(static_cast<const T*>(X), d, Qf, desc, cand, ntiles,
                                                              kk, pkey, pid, qthr, ir.Qb, ir.qok, ir.qsq,
                                                              ir.xsq);
  return TACO_OK;
}

// Integer re-rank eligibility of each query (u8 rows only): every value an
// integer in [0, 255] (bit-exact f32 round trip; -0 counts as 0, which gives
// the same differences).  Then for rows and query in [0, 255] and d <= 4096,
// each step of the reference's fp64 einsum -- the difference, its square and
// every partial sum (< 2^31) -- is exact, so the fp64 d2 equals the integer
// sum x^2 - 2 sum x q + sum q^2, computed with DP4A.
__global__ void k_q_u8(const float* __restrict__ Q, int64_t nq, int d, uint8_t* __restrict__ Qb,
                       int32_t* __restrict__ qsq, uint8_t* __restrict__ qok, int64_t* __restrict__ any_fp) {
  const int64_t q = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  bool ok = true;
  uint32_t sq = 0;
  for (int t = lane; t < d; t += 32) {
    const float v = Q[q * d + t];
    const bool in = v >= 0.0f && v <= 255.0f && v == rintf(v);
    ok = ok && in;
    const uint32_t b = in ? (uint32_t)v : 0u;
    Qb[q * d + t] = (uint8_t)b;
    sq += b * b;
  }
  ok = __all_sync(0xffffffffu, ok);
  for (int o = 16; o > 0; o >>= 1) sq += __shfl_xor_sync(0xffffffffu, sq, o);
  if (lane == 0) {
    qsq[q] = (int32_t)sq;
    qok[q] = ok ? 1 : 0;
    if (!ok) any_fp[0] = 1;   // some query of the batch takes the fp64 path
  }
}

static bool int_rerank_enabled() {
  static int on = -1;
  if (on < 0) {
    const char* e = getenv("TACO_INT_RERANK");
    on = !(e && e[0] == '0');
  }
  return on;
}

// rows of candidates -> CTA partial top-k -> per-query top-k (t.tk_d2 / t.tk_ids)
static int rerank_core(const float* X, const void* Xn, int fmt, int d, const float* Qf, int64_t QS, int64_t S,
                       const int64_t* tstart,
                       const int64_t* tproc, const int64_t* sbase, const int64_t* scnt, const uint32_t* cand, int64_t ntiles, int k,
                       int64_t id_base, DevBuf& pkey, DevBuf& pid, DevBuf& tsegb, DevBuf& qthrb, double* out_d2,
                       int64_t* out_ids, cudaStream_t st, const IntRerank& ir = IntRerank(), bool all_int = false,
                       int64_t max_cand = 0, DevBuf* xbuf = nullptr) {
  const int kk = std::min(k, GR);
  TACO_TRY(qthrb.ensure(sizeof(unsigned long long) * (size_t)QS));
  TACO_CHECK_CUDA(cudaMemsetAsync(qthrb.p, 0xFF, sizeof(unsigned long long) * (size_t)QS, st));
  unsigned long long* qthr = qthrb.as<unsigned long long>();
  TACO_TRY(pkey.ensure(sizeof(unsigned long long) * (size_t)std::max<int64_t>(ntiles, 1) * kk));
  TACO_TRY(pid.ensure(sizeof(uint32_t) * (size_t)std::max<int64_t>(ntiles, 1) * kk));
  TACO_TRY(tsegb.ensure(sizeof(int4) * (size_t)std::max<int64_t>(ntiles, 1)));
  const int4* desc = tsegb.as<int4>();
  if (ntiles > 0) {
    ProfScope ps(K_PLAN, st);
    k_tile_map<<<(unsigned)ceil_div(QS * S * 32, 256), 256, 0, st>>>(scnt, tproc, tstart, sbase, QS * S,
                                                                    (int)S, tsegb.as<int4>());
    TACO_LAUNCHED();
  }
  if (ntiles > 0) {
    ProfScope ps(K_RERANK, st);
    unsigned long long* pk = pkey.as<unsigned long long>();
    static const bool fast = !(getenv("TACO_RERANK_I8") && getenv("TACO_RERANK_I8")[0] == '0');
    if (fmt == TACO_ROWS_U8 && all_int && ir.qok && fast && d <= 128 && d % 16 == 0) {
      // every query u8-exact: the integer fast path
      const size_t smem = sizeof(RiStage) * 2 * RI_WARPS;
      static bool attr = false;
      if (!attr) {
        TACO_CHECK_CUDA(cudaFuncSetAttribute(k_rerank_i8<8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        TACO_CHECK_CUDA(cudaFuncSetAttribute(k_rerank_i8<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
        attr = true;
      }
      const int64_t grid = std::min<int64_t>(ceil_div(ntiles, RI_WARPS), (int64_t)num_sms() * RI_CTAS);
      (d == 128 ? k_rerank_i8<8> : k_rerank_i8<0>)<<<(unsigned)grid, 32 * RI_WARPS, smem, st>>>(static_cast<const uint8_t*>(Xn), d, ir.Qb, ir.qsq,
                                                                ir.xsq, desc, cand, ntiles, kk, pk,
                                                                pid.as<uint32_t>(), qthr);
    } else if (fmt == TACO_ROWS_U8) {
      TACO_TRY(launch_rerank_async<uint8_t>(Xn, d, Qf, desc, cand, ntiles, kk, pk, pid.as<uint32_t>(), qthr, ir, st));
    } else if (fmt == TACO_ROWS_F16) {
      TACO_TRY(launch_rerank_async<__half>(Xn, d, Qf, desc, cand, ntiles, kk, pk, pid.as<uint32_t>(), qthr, ir, st));
    } else if (d % 4 == 0) {
      TACO_TRY(launch_rerank_async<float>(X, d, Qf, desc, cand, ntiles, kk, pk, pid.as<uint32_t>(), qthr, ir, st));
    } else {
      k_rerank_plain<<<(unsigned)ceil_div(ntiles, 4), 128, 0, st>>>(X, d, Qf, desc,
                                                                   cand, ntiles, kk, pkey.as<unsigned long long>(),
                                                                   pid.as<uint32_t>());
    }
    TACO_LAUNCHED();
  }
  {
    ProfScope ps(K_TOPK, st);
    // partial entries per query: many (k > 32 keeps every row) -> 512 threads
    const bool wide = ntiles * kk >= (int64_t)8192 * std::max<int64_t>(QS, 1);
    // long lists are cut into parts (k_topk): max_cand = the tile's largest candidate count when
    // the caller knows it (0: no split); scratch = QS x parts x k (key, id) pairs, capped at 1 GiB
    // TACO_TOPK_SPLIT=n (read per batch): lists above n entries are split (the tests force it)
    const char* se = getenv("TACO_TOPK_SPLIT");
    const int64_t split_min = se ? std::max<int64_t>(64, atoll(se)) : 65536;
    int parts = 1;
    if (max_cand > split_min && xbuf != nullptr) {
      parts = (int)std::min<int64_t>(32, ceil_div(max_cand, split_min / 2));
      while (parts > 1 && (size_t)QS * parts * k * 12 > ((size_t)1 << 30)) --parts;
    }
    unsigned long long* xk = nullptr;
    uint32_t* xi = nullptr;
    if (parts > 1) {
      const size_t nx = (size_t)QS * parts * k;
      TACO_TRY(xbuf->ensure(nx * 12));
      xk = xbuf->as<unsigned long long>();
      xi = reinterpret_cast<uint32_t*>(xk + nx);
    }
    const int nt = wide ? 2 * TK_THREADS : TK_THREADS;
    auto kern = wide ? k_topk<2 * TK_THREADS> : k_topk<TK_THREADS>;
    kern<<<dim3((unsigned)QS, (unsigned)parts), nt, 0, st>>>(pkey.as<unsigned long long>(), pid.as<uint32_t>(), tstart,
                                                             (int)S, kk, scnt, k, id_base, out_d2, out_ids, parts,
                                                             split_min, xk, xi, 0);
    TACO_LAUNCHED();
    if (parts > 1) {
      kern<<<dim3((unsigned)QS, 1), nt, 0, st>>>(pkey.as<unsigned long long>(), pid.as<uint32_t>(), tstart, (int)S, kk,
                                                 scnt, k, id_base, out_d2, out_ids, parts, split_min, xk, xi, 1);
      TACO_LAUNCHED();
    }
  }
  return TACO_OK;
}

static int q_u8_prep(taco_index* idx, QueryTile& t, int64_t QS, cudaStream_t st) {
  TACO_TRY(t.qb.ensure((size_t)QS * idx->d));
  TACO_TRY(t.qsq.ensure(sizeof(int32_t) * (size_t)QS));
  TACO_TRY(t.qok.ensure((size_t)QS));
  ProfScope ps(K_PLAN, st);
  k_q_u8<<<(unsigned)ceil_div(QS * 32, 256), 256, 0, st>>>(t.Q.as<float>(), QS, idx->d, t.qb.as<uint8_t>(),
                                                            t.qsq.as<int32_t>(), t.qok.as<uint8_t>(),
                                                            t.flags.as<int64_t>() + 4);
  TACO_LAUNCHED();
  return TACO_OK;
}

// prepped: tile_front already ran q_u8_prep (the split API has not)
static int rerank_stage(taco_index* idx, QueryTile& t, int64_t QS, int k, int64_t ntiles, cudaStream_t st,
                        bool prepped = false) {
  const int64_t S = seg_per_query(idx);
  IntRerank ir;
  const bool intp = idx->xfmt == TACO_ROWS_U8 && int_rerank_enabled();
  if (intp && !prepped) TACO_TRY(q_u8_prep(idx, t, QS, st));
  if (intp) {
    ir.Qb = t.qb.as<uint8_t>();
    ir.qok = t.qok.as<uint8_t>();
    ir.qsq = t.qsq.as<int32_t>();
    ir.xsq = idx->Xsq.as<int32_t>();
  }
  return rerank_core(idx->X.as<float>(), idx->Xn.p, idx->xfmt, idx->d, t.Q.as<float>(), QS, S, t.bpref.as<int64_t>(),
                     S > 1 ? t.ppref.as<int64_t>() : t.bpref.as<int64_t>(),
                     seg_base(idx, t), seg_cnt(idx, t), t.cand.as<uint32_t>(), ntiles, k, idx->id_base,
                     t.pd2, t.ppos, t.tseg, t.qthr, t.tk_d2.as<double>(), t.tk_ids.as<int64_t>(), st, ir,
                     intp && prepped && t.flags_h[4] == 0,   // flags[4]: some query is not u8-exact
                     t.flags_h ? t.flags_h[6] : 0, &t.tkx);   // flags[6]: the tile's largest candidate count
}

static void prof_stats(taco_index* idx, QueryTile& t, int64_t QS, int64_t total) {
  if (!g_prof.on) return;
  std::vector<int64_t> r((size_t)QS * idx->n_sub);
  std::vector<int32_t> np((size_t)QS * idx->n_sub);
  cudaMemcpy(r.data(), t.ret.p, 8 * r.size(), cudaMemcpyDeviceToHost);
  cudaMemcpy(np.data(), t.npop.p, 4 * np.size(), cudaMemcpyDeviceToHost);
  for (auto v : r) g_prof.sumR += v;
  for (auto v : np) {
    g_prof.sumPops += v;
    g_prof.maxPops = std::max<int64_t>(g_prof.maxPops, v);
  }
  if (t.fused) {   // the fused kernel keeps no global candidate count: |C| = candidate_num
    std::vector<int64_t> cn((size_t)QS);
    cudaMemcpy(cn.data(), t.cnum.p, 8 * cn.size(), cudaMemcpyDeviceToHost);
    total = 0;
    for (auto v : cn) total += v;
  }
  g_prof.sumC += total;
  g_prof.queries += QS;
  g_prof.tiles += 1;
  if (!idx->cluster_mode && idx->n_sub >= 2) {   // spilled score >= 2 records (k_count CNT_HIST)
    const size_t np1 = (size_t)idx->n_sub + 1;
    std::vector<int32_t> part((size_t)QS * idx->nchunks * np1);
    cudaMemcpy(part.data(), t.part.p, 4 * part.size(), cudaMemcpyDeviceToHost);
    const int64_t cap = table_bytes(idx) / 4;
    for (int64_t q = 0; q < QS; ++q)
      for (int64_t c = 0; c < idx->nchunks; ++c) {
        const int32_t* pp = part.data() + ((size_t)q * idx->nchunks + c) * np1;
        const int64_t valid = std::min<int64_t>(idx->chunk, idx->n - c * idx->chunk);
        const int64_t rc = valid - pp[0] - pp[1];
        if (rc <= cap) g_prof.bytes_scores += 4 * rc;
      }
  }
}

// Front half of a tile (queries already in t.Q): transform, ranks, traversal,
// counting, Alg. 5, plans; flags read back asynchronously.
static int tile_front(taco_index* idx, QueryTile& t, int64_t QS, double alpha, double beta, int k,
                      cudaStream_t st) {
  if (t.cand_cap == 0) {
    const int64_t est = QS * std::max<int64_t>(1024, (int64_t)(4.0 * beta * (double)idx->n_global)) + (1 << 20);
    TACO_TRY(ensure_cand(t, std::min<int64_t>(est, (int64_t)1 << 31)));
  }
  TACO_CHECK_CUDA(cudaMemsetAsync(t.flags.p, 0, sizeof(int64_t) * 8, st));
  const bool intp = idx->xfmt == TACO_ROWS_U8 && int_rerank_enabled();
  bool fuse = false;
  t.fused = false;
  if (intp && fused_eligible(idx, k)) {
    // u8-exactness first (flags[4]): it decides the count kernel; the host
    // waits only for this small kernel while the front runs on
    TACO_TRY(q_u8_prep(idx, t, QS, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.flags_h + 4, t.flags.as<int64_t>() + 4, sizeof(int64_t),
                                    cudaMemcpyDeviceToHost, st));
    if (!t.qev) TACO_CHECK_CUDA(cudaEventCreateWithFlags(&t.qev, cudaEventDisableTiming));
    TACO_CHECK_CUDA(cudaEventRecord(t.qev, st));
    TACO_TRY(stage_front(idx, t, QS, alpha, st, nullptr));
    TACO_CHECK_CUDA(cudaEventSynchronize(t.qev));
    fuse = t.flags_h[4] == 0;
  } else {
    TACO_TRY(stage_front(idx, t, QS, alpha, st, nullptr));
  }
  if (idx->cluster_mode) {
    if (fuse) TACO_TRY(cluster_count_fused(idx, t, QS, beta, k, st));
    else TACO_TRY(cluster_count(idx, t, QS, beta, st));
  } else {
    TACO_TRY(global_count(idx, t, QS, st));
    TACO_TRY(global_select(idx, t, QS, t.hist.as<int64_t>(), beta, st));
  }
  if (fuse) {   // answers written by the count kernel: only the flags come back
    t.fused = true;
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.flags_h, t.flags.p, sizeof(int64_t) * 5, cudaMemcpyDeviceToHost, st));
    return TACO_OK;
  }
  if (intp && !fused_eligible(idx, k))   // integer re-rank eligibility -> flags[4]
    TACO_TRY(q_u8_prep(idx, t, QS, st));
  return plan_async(idx, t, QS, st);
}

// Back half, after tile_front's stream work: re-run the front with larger
// scratch if a traversal or the candidate buffer overflowed, then re-rank.
static int tile_back(taco_index* idx, QueryTile& t, int64_t QS, double alpha, double beta, int k, cudaStream_t st) {
  for (int attempt = 0; attempt < 4; ++attempt) {
    TACO_CHECK_CUDA(cudaStreamSynchronize(st));
    const int64_t* fl = t.flags_h;
    if (fl[0] > t.pop_cap) {           // a traversal popped more cells than stored
      t.pop_cap = idx->K;
      TACO_TRY(t.pops.ensure(sizeof(uint16_t) * (size_t)QS * idx->n_sub * t.pop_cap));
      TACO_TRY(tile_front(idx, t, QS, alpha, beta, k, st));
      continue;
    }
    if (fl[1]) {                       // candidate buffer too small: grow to what was asked
      TACO_TRY(ensure_cand(t, fl[3] + fl[3] / 4 + 1024));
      TACO_TRY(tile_front(idx, t, QS, alpha, beta, k, st));
      continue;
    }
    prof_stats(idx, t, QS, fl[3]);
    if (t.fused) return TACO_OK;       // k_count_fused already wrote the answers
    return rerank_stage(idx, t, QS, k, fl[2], st, true);
  }
  TACO_FAIL(TACO_ERR_CUDA, "query scratch did not converge");
}

// Batches of >= 2 * kPipeMin queries run as tiles alternating between two
// buffers and two streams: tile i+1's front (transform .. count, issued
// before tile i's flags are read) overlaps tile i's re-rank on the other
// stream, and the latency-bound front kernels (ranks, traversal) overlap
// the other tile's counting.
constexpr int64_t kPipeMin = 2048;

static int query_batch_impl(taco_index* idx, const float* Q_src, bool src_host, int64_t nq, double alpha,
                            double beta, int k, int32_t* ids_o, float* dists_o, int64_t* cnum_o,
                            int32_t* lvl_o, bool dst_host, cudaStream_t st) {
  TACO_TRY(check_query_ready(idx, alpha, k));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "base vectors are not resident");
  if (!(beta > 0.0 && beta < 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "re-rank ratio %g outside (0, 1)", beta);
  if (nq == 0) return TACO_OK;
  QueryTile* tiles[2] = {&idx->qt, &idx->qt2};
  for (QueryTile* t : tiles)
    if (t->pop_cap == 0) t->pop_cap = std::min(idx->K, 1024);
  const int64_t QSmax = std::min<int64_t>(nq, super_tile(idx, idx->qt.pop_cap));
  // tiles a pipelined batch is cut into (TACO_PIPE_TILES; 1 = off).  Default:
  // off for u8 rows with d <= 128 (the integer re-rank is short enough that
  // overlapping it with the next tile's count no longer pays: config 2,
  // 1 tile 1.099 M QPS vs 2 tiles 1.060 M), else 2.
  static int ptiles_env = -2;
  if (ptiles_env == -2) {
    const char* e = getenv("TACO_PIPE_TILES");
    ptiles_env = e ? std::max(1, atoi(e)) : -1;
  }
  const int ptiles = ptiles_env > 0 ? ptiles_env : (idx->xfmt == TACO_ROWS_U8 && idx->d <= 128 ? 1 : 2);
  // profiled passes run unpipelined so per-kernel event times do not overlap
  const bool pipe = ptiles > 1 && nq >= 2 * kPipeMin && !g_prof.on;
  int64_t QT = QSmax;
  if (pipe) QT = std::min<int64_t>(QSmax, std::max<int64_t>(kPipeMin, ceil_div(nq, ptiles)));
  const int64_t ntile = ceil_div(nq, QT);
  cudaStream_t sts[2] = {st, st};
  if (pipe) {
    if (!idx->stream2) {
      TACO_CHECK_CUDA(cudaStreamCreateWithFlags(&idx->stream2, cudaStreamNonBlocking));
      TACO_CHECK_CUDA(cudaEventCreateWithFlags(&idx->ev_fork, cudaEventDisableTiming));
      TACO_CHECK_CUDA(cudaEventCreateWithFlags(&idx->ev_join, cudaEventDisableTiming));
    }
    sts[1] = idx->stream2;
    TACO_CHECK_CUDA(cudaEventRecord(idx->ev_fork, st));             // stream 2 starts after the caller's work
    TACO_CHECK_CUDA(cudaStreamWaitEvent(idx->stream2, idx->ev_fork, 0));
  }
  for (int b = 0; b < (pipe ? 2 : 1); ++b) TACO_TRY(ensure_front(idx, *tiles[b], QT, k));
  const cudaMemcpyKind kin = src_host ? cudaMemcpyHostToDevice : cudaMemcpyDeviceToDevice;
  const cudaMemcpyKind kout = dst_host ? cudaMemcpyDeviceToHost : cudaMemcpyDeviceToDevice;
  // host results land in pinned staging first: a D2H copy into pageable memory
  // blocks the host until the tile is done, which would stall the enqueue of
  // the next tiles (the pipeline); the caller's arrays are filled at the end
  int32_t* ids_u = ids_o;
  float* dists_u = dists_o;
  int64_t* cnum_u = cnum_o;
  int32_t* lvl_u = lvl_o;
  const size_t sb_ids = sizeof(int32_t) * (size_t)nq * k, sb_d = sizeof(float) * (size_t)nq * k;
  const size_t sb_c = sizeof(int64_t) * (size_t)nq, sb_l = sizeof(int32_t) * (size_t)nq;
  if (dst_host) {
    const size_t need = sb_ids + sb_d + sb_c + sb_l + 64;
    if (idx->hstage_bytes < need) {
      if (idx->hstage) TACO_CHECK_CUDA(cudaFreeHost(idx->hstage));
      idx->hstage = nullptr;
      idx->hstage_bytes = 0;
      TACO_CHECK_CUDA(cudaMallocHost(&idx->hstage, need));
      idx->hstage_bytes = need;
    }
    uint8_t* h = static_cast<uint8_t*>(idx->hstage);
    cnum_o = reinterpret_cast<int64_t*>(h);
    ids_o = reinterpret_cast<int32_t*>(h + sb_c);
    dists_o = reinterpret_cast<float*>(h + sb_c + sb_ids);
    lvl_o = reinterpret_cast<int32_t*>(h + sb_c + sb_ids + sb_d);
  }
  auto front = [&](int64_t i) -> int {
    QueryTile& t = *tiles[pipe ? i & 1 : 0];
    cudaStream_t s = sts[pipe ? i & 1 : 0];
    const int64_t q0 = i * QT, QS = std::min<int64_t>(QT, nq - q0);
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, Q_src + (size_t)q0 * idx->d, sizeof(float) * (size_t)QS * idx->d, kin, s));
    return tile_front(idx, t, QS, alpha, beta, k, s);
  };
  TACO_TRY(front(0));
  for (int64_t i = 0; i < ntile; ++i) {
    if (pipe && i + 1 < ntile) TACO_TRY(front(i + 1));
    QueryTile& t = *tiles[pipe ? i & 1 : 0];
    cudaStream_t s = sts[pipe ? i & 1 : 0];
    const int64_t q0 = i * QT, QS = std::min<int64_t>(QT, nq - q0);
    TACO_TRY(tile_back(idx, t, QS, alpha, beta, k, s));
    const int64_t tot = QS * k;
    if (!t.fused) {
      ProfScope ps(K_FINAL, s);
      k_finalize<<<(unsigned)ceil_div(tot, 256), 256, 0, s>>>(t.tk_d2.as<double>(), t.tk_ids.as<int64_t>(), tot,
                                                              t.out_ids.as<int32_t>(), t.out_d.as<float>());
      TACO_LAUNCHED();
    }
    TACO_CHECK_CUDA(cudaMemcpyAsync(ids_o + q0 * k, t.out_ids.p, sizeof(int32_t) * tot, kout, s));
    TACO_CHECK_CUDA(cudaMemcpyAsync(dists_o + q0 * k, t.out_d.p, sizeof(float) * tot, kout, s));
    TACO_CHECK_CUDA(cudaMemcpyAsync(cnum_o + q0, t.cnum.p, sizeof(int64_t) * QS, kout, s));
    TACO_CHECK_CUDA(cudaMemcpyAsync(lvl_o + q0, t.lvl.p, sizeof(int32_t) * QS, kout, s));
    if (!pipe && i + 1 < ntile) TACO_TRY(front(i + 1));
  }
  if (pipe) {   // the caller's stream resumes after both tiles' work
    TACO_CHECK_CUDA(cudaEventRecord(idx->ev_join, idx->stream2));
    TACO_CHECK_CUDA(cudaStreamWaitEvent(st, idx->ev_join, 0));
  }
  if (dst_host) {
    TACO_CHECK_CUDA(cudaStreamSynchronize(st));
    std::memcpy(ids_u, ids_o, sb_ids);
    std::memcpy(dists_u, dists_o, sb_d);
    std::memcpy(cnum_u, cnum_o, sb_c);
    std::memcpy(lvl_u, lvl_o, sb_l);
  }
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

int taco_query_tile_size(taco_index* idx) {
  if (!idx) return 0;
  return (int)super_tile(idx, idx->qt.pop_cap ? idx->qt.pop_cap : std::min(idx->K, 1024));
}

// Split query (multi-GPU): only global-mode (sharded) indexes.
int taco_query_count_device(taco_index* idx, const float* Q_d, int64_t nq, double alpha,
                            int64_t* hist_d, void* stream) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  if (idx->cluster_mode) TACO_FAIL(TACO_ERR_STATE, "split query needs a sharded (global-mode) index");
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  QueryTile& t = idx->qt;
  if (t.pop_cap == 0) t.pop_cap = std::min(idx->K, 1024);
  const int64_t Qt = super_tile(idx, t.pop_cap);
  if (nq > Qt) TACO_FAIL(TACO_ERR_PARAMETER, "split query batch %lld exceeds tile %lld", (long long)nq, (long long)Qt);
  TACO_TRY(ensure_front(idx, t, Qt, 1));
  TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, Q_d, sizeof(float) * (size_t)nq * idx->d, cudaMemcpyDeviceToDevice, st));
  for (int attempt = 0; attempt < 2; ++attempt) {
    TACO_CHECK_CUDA(cudaMemsetAsync(t.flags.p, 0, sizeof(int64_t) * 8, st));
    TACO_TRY(stage_front(idx, t, nq, alpha, st, nullptr));
    int64_t f0 = 0;
    TACO_CHECK_CUDA(cudaMemcpyAsync(&f0, t.flags.p, 8, cudaMemcpyDeviceToHost, st));
    TACO_CHECK_CUDA(cudaStreamSynchronize(st));
    if (f0 <= t.pop_cap) break;
    t.pop_cap = idx->K;
    TACO_TRY(t.pops.ensure(sizeof(uint16_t) * (size_t)Qt * idx->n_sub * t.pop_cap));
  }
  TACO_TRY(global_count(idx, t, nq, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(hist_d, t.hist.p, sizeof(int64_t) * (size_t)nq * (idx->n_sub + 1),
                                  cudaMemcpyDeviceToDevice, st));
  return TACO_OK;
}

// Split traversal (multi-GPU): this rank's slice [q_lo, q_hi) of a tile of nq
// queries (Q_d; rows >= nq is the all-gather's padded row count) -> popped
// cells in rows [q_lo, q_hi) of the tile buffers, which the caller
// all-gathers (taco_query_pop_buffers) before taco_query_count_popped_device.
// *need = the longest traversal when it exceeded pop_cap (every rank must then
// re-run with cap K'^2), else 0.
int taco_query_front_device(taco_index* idx, const float* Q_d, int64_t nq, int64_t q_lo, int64_t q_hi,
                            int64_t rows, double alpha, int32_t pop_cap, int64_t* need, void* stream) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  if (idx->cluster_mode) TACO_FAIL(TACO_ERR_STATE, "split query needs a sharded (global-mode) index");
  if (pop_cap < 1 || pop_cap > idx->K) TACO_FAIL(TACO_ERR_PARAMETER, "pop cap %d outside [1, %lld]", pop_cap, (long long)idx->K);
  if (!(q_lo >= 0 && q_lo <= q_hi && q_hi <= nq && nq <= rows))
    TACO_FAIL(TACO_ERR_PARAMETER, "query slice [%lld, %lld) of %lld outside [0, %lld)", (long long)q_lo,
              (long long)q_hi, (long long)nq, (long long)rows);
  const int64_t Qt = super_tile(idx, pop_cap);
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  QueryTile& t = idx->qt;
  t.pop_cap = pop_cap;
  TACO_TRY(ensure_front(idx, t, std::max(Qt, rows), 1));
  t.front_rows = std::max(t.front_rows, rows);
  // every query of the tile: the re-rank (taco_query_finish_device) reads them all
  if (nq > 0)
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, Q_d, sizeof(float) * (size_t)nq * idx->d, cudaMemcpyDeviceToDevice, st));
  TACO_CHECK_CUDA(cudaMemsetAsync(t.flags.p, 0, sizeof(int64_t) * 8, st));
  TACO_TRY(stage_front(idx, t, q_hi - q_lo, alpha, st, nullptr, q_lo));
  int64_t f0 = 0;
  TACO_CHECK_CUDA(cudaMemcpyAsync(&f0, t.flags.p, 8, cudaMemcpyDeviceToHost, st));
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  *need = f0 > pop_cap ? f0 : 0;
  return TACO_OK;
}

// As taco_query_front_device without the host round trip: the longest walk
// of the slice (pops, capped or not) is copied to need_d[0] on the stream, so
// a caller can all-reduce it and check all tiles of a batch with one sync.
int taco_query_front_async(taco_index* idx, const float* Q_d, int64_t nq, int64_t q_lo, int64_t q_hi,
                           int64_t rows, double alpha, int32_t pop_cap, int64_t* need_d, void* stream) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  if (idx->cluster_mode) TACO_FAIL(TACO_ERR_STATE, "split query needs a sharded (global-mode) index");
  if (pop_cap < 1 || pop_cap > idx->K) TACO_FAIL(TACO_ERR_PARAMETER, "pop cap %d outside [1, %lld]", pop_cap, (long long)idx->K);
  if (!(q_lo >= 0 && q_lo <= q_hi && q_hi <= nq && nq <= rows))
    TACO_FAIL(TACO_ERR_PARAMETER, "query slice [%lld, %lld) of %lld outside [0, %lld)", (long long)q_lo,
              (long long)q_hi, (long long)nq, (long long)rows);
  if (!need_d) TACO_FAIL(TACO_ERR_PARAMETER, "need_d is null");
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  QueryTile& t = idx->qt;
  t.pop_cap = pop_cap;
  TACO_TRY(ensure_front(idx, t, std::max(super_tile(idx, pop_cap), rows), 1));
  t.front_rows = std::max(t.front_rows, rows);
  if (nq > 0)
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, Q_d, sizeof(float) * (size_t)nq * idx->d, cudaMemcpyDeviceToDevice, st));
  TACO_CHECK_CUDA(cudaMemsetAsync(t.flags.p, 0, sizeof(int64_t) * 8, st));
  TACO_TRY(stage_front(idx, t, q_hi - q_lo, alpha, st, nullptr, q_lo));
  TACO_CHECK_CUDA(cudaMemcpyAsync(need_d, t.flags.p, 8, cudaMemcpyDeviceToDevice, st));
  return TACO_OK;
}

int taco_query_pop_buffers(taco_index* idx, void** pops, void** npop, void** ret, int32_t* pop_cap) {
  TACO_TRY(index_check(idx));
  QueryTile& t = idx->qt;
  if (!t.pops.p) TACO_FAIL(TACO_ERR_STATE, "no traversal buffers yet (call taco_query_front_device)");
  *pops = t.pops.p;
  *npop = t.npop.p;
  *ret = t.ret.p;
  *pop_cap = t.pop_cap;
  return TACO_OK;
}

// Counting sweep over the (gathered) popped cells of nq tile queries -> the
// local per-query level histograms, as taco_query_count_device.
int taco_query_count_popped_device(taco_index* idx, int64_t nq, int64_t* hist_d, void* stream) {
  TACO_TRY(index_check(idx));
  if (idx->cluster_mode) TACO_FAIL(TACO_ERR_STATE, "split query needs a sharded (global-mode) index");
  QueryTile& t = idx->qt;
  if (!t.pops.p) TACO_FAIL(TACO_ERR_STATE, "no traversal buffers yet (call taco_query_front_device)");
  if (nq > std::max(t.front_rows, super_tile(idx, t.pop_cap) + 16))
    TACO_FAIL(TACO_ERR_PARAMETER, "split query batch %lld exceeds tile", (long long)nq);
  if (nq == 0) return TACO_OK;
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  TACO_TRY(global_count(idx, t, nq, st));
  TACO_CHECK_CUDA(cudaMemcpyAsync(hist_d, t.hist.p, sizeof(int64_t) * (size_t)nq * (idx->n_sub + 1),
                                  cudaMemcpyDeviceToDevice, st));
  return TACO_OK;
}

int taco_query_finish_device(taco_index* idx, int64_t nq, const int64_t* ghist_d, double beta,
                             int32_t k, double* topk_d2_d, int64_t* topk_ids_d,
                             int64_t* cand_num_d, int32_t* last_coll_d, void* stream) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X) TACO_FAIL(TACO_ERR_STATE, "base vectors are not resident");
  if (idx->cluster_mode) TACO_FAIL(TACO_ERR_STATE, "split query needs a sharded (global-mode) index");
  if (!(beta > 0.0 && beta < 1.0)) TACO_FAIL(TACO_ERR_PARAMETER, "re-rank ratio %g outside (0, 1)", beta);
  if (k < 1 || k > TK_MAX) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d outside [1, %d]", k, TK_MAX);
  cudaStream_t st = stream ? (cudaStream_t)stream : idx->stream;
  QueryTile& t = idx->qt;
  if (t.pop_cap == 0) t.pop_cap = std::min(idx->K, 1024);
  const int64_t Qt = super_tile(idx, t.pop_cap);
  if (nq > Qt) TACO_FAIL(TACO_ERR_PARAMETER, "split query batch %lld exceeds tile %lld", (long long)nq, (long long)Qt);
  TACO_TRY(ensure_front(idx, t, Qt, k));
  if (t.cand_cap == 0)
    TACO_TRY(ensure_cand(t, Qt * std::max<int64_t>(1024, (int64_t)(4.0 * beta * (double)idx->n)) + (1 << 20)));
  for (int attempt = 0; attempt < 3; ++attempt) {
    int64_t zero = 0;
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.flags.as<int64_t>() + 1, &zero, 8, cudaMemcpyHostToDevice, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.flags.as<int64_t>() + 3, &zero, 8, cudaMemcpyHostToDevice, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(t.flags.as<int64_t>() + 4, &zero, 8, cudaMemcpyHostToDevice, st));
    TACO_TRY(global_select(idx, t, nq, ghist_d, beta, st));
    const bool intp = idx->xfmt == TACO_ROWS_U8 && int_rerank_enabled();
    if (intp) TACO_TRY(q_u8_prep(idx, t, nq, st));   // flags[4] is read back with the plan
    int64_t fl[4];
    TACO_TRY(plan_and_read(idx, t, nq, st, fl));
    if (fl[1]) {
      TACO_TRY(ensure_cand(t, fl[3] + fl[3] / 4 + 1024));
      continue;
    }
    prof_stats(idx, t, nq, fl[3]);
    TACO_TRY(rerank_stage(idx, t, nq, k, fl[2], st, intp));
    TACO_CHECK_CUDA(cudaMemcpyAsync(topk_d2_d, t.tk_d2.p, sizeof(double) * (size_t)nq * k, cudaMemcpyDeviceToDevice, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(topk_ids_d, t.tk_ids.p, sizeof(int64_t) * (size_t)nq * k, cudaMemcpyDeviceToDevice, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(cand_num_d, t.cnum.p, sizeof(int64_t) * nq, cudaMemcpyDeviceToDevice, st));
    TACO_CHECK_CUDA(cudaMemcpyAsync(last_coll_d, t.lvl.p, sizeof(int32_t) * nq, cudaMemcpyDeviceToDevice, st));
    return TACO_OK;
  }
  TACO_FAIL(TACO_ERR_CUDA, "candidate buffer did not converge");
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
  QueryTile& t = idx->qt;
  cudaStream_t st = idx->stream;
  TACO_TRY(ensure_front(idx, t, 1, 1));
  DevBuf sc, part, hist;
  TACO_TRY(sc.ensure((size_t)idx->nchunks * idx->chunk));
  TACO_TRY(part.ensure(sizeof(int32_t) * idx->nchunks * (idx->n_sub + 1)));
  int rc = TACO_OK;
  do {
    if (cudaMemcpyAsync(t.Q.p, q_h, sizeof(float) * idx->d, cudaMemcpyHostToDevice, st) != cudaSuccess) {
      rc = TACO_ERR_CUDA; break;
    }
    for (int attempt = 0; attempt < 2; ++attempt) {
      cudaMemsetAsync(t.flags.p, 0, sizeof(int64_t) * 8, st);
      if ((rc = stage_front(idx, t, 1, alpha, st, nullptr))) break;
      int64_t f0 = 0;
      cudaMemcpyAsync(&f0, t.flags.p, 8, cudaMemcpyDeviceToHost, st);
      cudaStreamSynchronize(st);
      if (f0 <= t.pop_cap) break;
      t.pop_cap = idx->K;
      if ((rc = t.pops.ensure(sizeof(uint16_t) * idx->n_sub * (size_t)t.pop_cap * super_tile(idx, t.pop_cap)))) break;
    }
    if (rc) break;
    if ((rc = set_count_attrs(idx))) break;
    k_count<false><<<dim3((unsigned)idx->nchunks, 1), CT_THREADS, (size_t)idx->chunk, st>>>(
        t.pops.as<uint16_t>(), t.npop.as<int32_t>(), t.pop_cap, idx->ids.as<uint32_t>(), idx->offs.as<uint32_t>(),
        idx->n_sub, idx->K, idx->n, idx->nchunks, idx->chunk, CNT_TABLE, sc.as<uint8_t>(), part.as<int32_t>(),
        nullptr, nullptr, nullptr, nullptr, nullptr);
    count_launch();
    cudaMemcpyAsync(scores_h, sc.p, idx->n, cudaMemcpyDeviceToHost, st);
    cudaError_t e = cudaStreamSynchronize(st);
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; }
  } while (0);
  sc.release(); part.release(); hist.release();
  return rc;
}

int taco_activation_trace(taco_index* idx, const float* q_h, int32_t j, double alpha, int32_t cap,
                          int32_t* pops_h, double* keys_h, int32_t* npop_h, int64_t* retrieved_h) {
  TACO_TRY(check_query_ready(idx, alpha, 1));
  if (j < 0 || j >= idx->n_sub) TACO_FAIL(TACO_ERR_PARAMETER, "subspace %d out of range", j);
  QueryTile& t = idx->qt;
  cudaStream_t st = idx->stream;
  const int saved = t.pop_cap;
  t.pop_cap = idx->K;
  TACO_TRY(ensure_front(idx, t, 1, 1));
  DevBuf keys;
  TACO_TRY(keys.ensure(sizeof(double) * (size_t)idx->n_sub * idx->K));
  TACO_CHECK_CUDA(cudaMemcpyAsync(t.Q.p, q_h, sizeof(float) * idx->d, cudaMemcpyHostToDevice, st));
  int rc = stage_front(idx, t, 1, alpha, st, keys.as<double>());
  t.pop_cap = saved;
  if (rc != TACO_OK) { keys.release(); return rc; }
  int32_t np = 0;
  int64_t got = 0;
  std::vector<uint16_t> p16(idx->K);
  std::vector<double> kv(idx->K);
  cudaMemcpyAsync(&np, t.npop.as<int32_t>() + j, sizeof(int32_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(&got, t.ret.as<int64_t>() + j, sizeof(int64_t), cudaMemcpyDeviceToHost, st);
  cudaMemcpyAsync(p16.data(), t.pops.as<uint16_t>() + (size_t)j * idx->K, sizeof(uint16_t) * idx->K,
                  cudaMemcpyDeviceToHost, st);
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
  const int64_t chunk = kGlobalChunk;
  const int64_t nc = ceil_div(n, chunk);
  DevBuf sc, part, hist, lvl, cnum, coff, qbase, clocal, flags, cand;
  int rc = TACO_OK;
  do {
    if ((rc = sc.ensure(nc * chunk)) || (rc = part.ensure(sizeof(int32_t) * nc * (n_sub + 1))) ||
        (rc = hist.ensure(sizeof(int64_t) * (n_sub + 1))) || (rc = lvl.ensure(4)) || (rc = cnum.ensure(8)) ||
        (rc = coff.ensure(8 * nc)) || (rc = qbase.ensure(8)) || (rc = clocal.ensure(8)) ||
        (rc = flags.ensure(64)) || (rc = cand.ensure(4 * n)))
      break;
    cudaMemset(sc.p, 0, nc * chunk);
    cudaMemset(flags.p, 0, 64);
    cudaMemcpy(sc.p, scores_h, n, cudaMemcpyHostToDevice);
    k_chunk_hist<<<(unsigned)nc, 256>>>(sc.as<uint8_t>(), n, nc, chunk, n_sub, part.as<int32_t>());
    count_launch();
    k_hist_reduce<<<1, 64>>>(part.as<int32_t>(), nc, n_sub, hist.as<int64_t>());
    count_launch();
    k_select<<<1, 32>>>(hist.as<int64_t>(), part.as<int32_t>(), 1, nc, n_sub, beta * (double)n,
                        coff.as<int64_t>(), n, flags.as<int64_t>(), qbase.as<int64_t>(), clocal.as<int64_t>(),
                        cnum.as<int64_t>(), lvl.as<int32_t>());
    count_launch();
    k_compact<<<dim3((unsigned)nc, 1), CMP_THREADS>>>(sc.as<uint8_t>(), n, nc, chunk, 0, lvl.as<int32_t>(),
                                                      coff.as<int64_t>(), qbase.as<int64_t>(), clocal.as<int64_t>(),
                                                      n, cand.as<uint32_t>());
    count_launch();
    int64_t tot = 0, cn = 0;
    int32_t L = 0;
    cudaMemcpy(&tot, clocal.p, 8, cudaMemcpyDeviceToHost);
    cudaMemcpy(&L, lvl.p, 4, cudaMemcpyDeviceToHost);
    cudaMemcpy(&cn, cnum.p, 8, cudaMemcpyDeviceToHost);
    std::vector<uint32_t> ids(std::max<int64_t>(tot, 1));
    cudaMemcpy(ids.data(), cand.p, 4 * tot, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    for (int64_t i = 0; i < tot; ++i) ids_h[i] = ids[i];
    *cand_num_h = cn;
    *last_coll_h = L;
    if (tot != cn) { set_error("candidate count %lld != histogram count %lld", (long long)tot, (long long)cn); rc = TACO_ERR_NUMERIC; }
  } while (0);
  sc.release(); part.release(); hist.release(); lvl.release(); cnum.release(); coff.release();
  qbase.release(); clocal.release(); flags.release(); cand.release();
  return rc;
}

int taco_rerank(int device, const float* X_h, int64_t n, int32_t d, const float* q_h,
                const int64_t* ids_h, int64_t m, int32_t k, int32_t* ids_out_h, float* dists_out_h,
                double* d2_out_h) {
  TACO_TRY(with_device(device));
  if (k < 1 || k > TK_MAX) TACO_FAIL(TACO_ERR_PARAMETER, "result count %d outside [1, %d]", k, TK_MAX);
  if (d > 4096) TACO_FAIL(TACO_ERR_PARAMETER, "dimension %d exceeds 4096", d);
  if (m < 0) TACO_FAIL(TACO_ERR_PARAMETER, "negative candidate count");
  if (m == 0) return TACO_OK;
  for (int64_t i = 0; i < m; ++i)
    if (ids_h[i] < 0 || ids_h[i] >= n || ids_h[i] > 0xFFFFFFFFll)
      TACO_FAIL(TACO_ERR_PARAMETER, "candidate id %lld out of range", (long long)ids_h[i]);
  std::vector<uint32_t> c32(m);
  bool sorted = true;
  for (int64_t i = 0; i < m; ++i) {
    c32[i] = (uint32_t)ids_h[i];
    if (i && c32[i] < c32[i - 1]) sorted = false;
  }
  if (!sorted) std::stable_sort(c32.begin(), c32.end());
  std::vector<float> rowsv((size_t)m * d);
  for (int64_t i = 0; i < m; ++i)
    std::copy(X_h + (size_t)c32[i] * d, X_h + (size_t)c32[i] * d + d, rowsv.begin() + (size_t)i * d);
  const int64_t ntiles = ceil_div(m, GR);
  DevBuf Xd, Qd, sb, sc, tp, ps, cd, pk, pi, ts, qh, tkd, tki, fl;
  int rc = TACO_OK;
  do {
    if ((rc = Xd.ensure(sizeof(float) * rowsv.size())) || (rc = Qd.ensure(sizeof(float) * d)) ||
        (rc = sb.ensure(8)) || (rc = sc.ensure(8)) || (rc = tp.ensure(16)) || (rc = ps.ensure(16)) ||
        (rc = cd.ensure(4 * m)) ||
        (rc = tkd.ensure(8 * k)) || (rc = tki.ensure(8 * k)) || (rc = fl.ensure(64)))
      break;
    std::vector<uint32_t> local(m);
    for (int64_t i = 0; i < m; ++i) local[i] = (uint32_t)i;
    const int64_t zero = 0;
    cudaMemcpy(Xd.p, rowsv.data(), sizeof(float) * rowsv.size(), cudaMemcpyHostToDevice);
    cudaMemcpy(Qd.p, q_h, sizeof(float) * d, cudaMemcpyHostToDevice);
    cudaMemcpy(sb.p, &zero, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(sc.p, &m, 8, cudaMemcpyHostToDevice);
    cudaMemcpy(cd.p, local.data(), 4 * m, cudaMemcpyHostToDevice);
    k_plan_sums<<<1, PLAN_NT>>>(sc.as<int64_t>(), 1, 1, 1, ps.as<int64_t>());
    k_plan_scan<<<1, PLAN_NT>>>(sc.as<int64_t>(), 1, 1, 1, ps.as<int64_t>(), tp.as<int64_t>(), nullptr,
                                fl.as<int64_t>());
    count_launch();
    count_launch();
    if ((rc = rerank_core(Xd.as<float>(), nullptr, TACO_ROWS_F32, d, Qd.as<float>(), 1, 1, tp.as<int64_t>(),
                          tp.as<int64_t>(),
                          sb.as<int64_t>(),
                          sc.as<int64_t>(), cd.as<uint32_t>(), ntiles, k, 0, pk, pi, ts, qh, tkd.as<double>(),
                          tki.as<int64_t>(), nullptr)))
      break;
    std::vector<double> td(k);
    std::vector<int64_t> ti(k);
    cudaMemcpy(td.data(), tkd.p, 8 * k, cudaMemcpyDeviceToHost);
    cudaMemcpy(ti.data(), tki.p, 8 * k, cudaMemcpyDeviceToHost);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) { set_error("%s", cudaGetErrorString(e)); rc = TACO_ERR_CUDA; break; }
    const int kr = (int)std::min<int64_t>(k, m);
    for (int r = 0; r < kr; ++r) {
      ids_out_h[r] = (int32_t)c32[ti[r]];
      d2_out_h[r] = td[r];
      dists_out_h[r] = (float)std::sqrt(td[r]);
    }
  } while (0);
  Xd.release(); Qd.release(); sb.release(); sc.release(); tp.release(); cd.release(); pk.release();
  pi.release(); ts.release(); qh.release(); ps.release(); tkd.release(); tki.release(); fl.release();
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
  DevBuf sd, sl, gs, pops, keys, np, ret, fl;
  int rc = TACO_OK;
  do {
    if ((rc = sd.ensure(16 * (size_t)kp)) || (rc = sl.ensure(4 * (size_t)kp)) || (rc = gs.ensure(8 * (size_t)K2)) ||
        (rc = pops.ensure(2 * (size_t)K2)) || (rc = keys.ensure(8 * (size_t)K2)) || (rc = np.ensure(4)) ||
        (rc = ret.ensure(8)) || (rc = fl.ensure(64)))
      break;
    std::vector<uint16_t> l(2 * kp);
    for (int i = 0; i < kp; ++i) { l[i] = (uint16_t)l1s_h[i]; l[kp + i] = (uint16_t)l2s_h[i]; }
    cudaMemcpy(sd.p, d1s_h, 8 * (size_t)kp, cudaMemcpyHostToDevice);
    cudaMemcpy(sd.as<double>() + kp, d2s_h, 8 * (size_t)kp, cudaMemcpyHostToDevice);
    cudaMemcpy(sl.p, l.data(), 4 * (size_t)kp, cudaMemcpyHostToDevice);
    cudaMemcpy(gs.p, sizes_h, 8 * (size_t)K2, cudaMemcpyHostToDevice);
    if ((rc = launch_traverse(sd.as<double>(), sl.as<uint16_t>(), gs.as<int64_t>(), 1, 1, kp, target,
                              pops.as<uint16_t>(), K2, keys.as<double>(), np.as<int32_t>(), ret.as<int64_t>(),
                              fl.as<int64_t>(), 0)))
      break;
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
  fl.release();
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
  stats_out[6] = taco::g_prof.maxPops;
  if (reset) {
    for (int i = 0; i < taco::K_NKIDS; ++i) { taco::g_prof.ms[i] = 0; taco::g_prof.cnt[i] = 0; }
    taco::g_prof.sumR = taco::g_prof.sumC = taco::g_prof.sumPops = 0;
    taco::g_prof.queries = taco::g_prof.tiles = taco::g_prof.bytes_scores = taco::g_prof.maxPops = 0;
  }
  return TACO_OK;
}

const char* taco_profile_name(int i) { return (i >= 0 && i < taco::K_NKIDS) ? taco::kKNames[i] : ""; }
int taco_profile_kernels(void) { return taco::K_NKIDS; }
void* taco_index_stream(taco_index* idx) { return idx ? (void*)idx->stream : nullptr; }

}  // extern "C"
