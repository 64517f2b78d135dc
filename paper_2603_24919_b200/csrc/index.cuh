// Device-resident TaCo index (one point shard per GPU) and its scratch.
//
// HBM layout:
//   X      f32 [n][d]            base vectors (row-major, rerank gathers rows)
//   T      f32 [D][n]            transformed points, dimension-major so each
//                                 k-means half is m contiguous n-vectors
//   cb1/2  f32 [Ns][K'][m1|m2]   codebooks (centroids), labels i32 [2Ns][n]
//   ids    u32 [Ns][n]           CSR ids, ordered (chunk, cell, id): chunk c
//                                 holds ids [c*CH, (c+1)*CH) so one CTA's
//                                 score table covers exactly one chunk
//   offs   u32 [Ns][nchunks*K'^2+1] start of (chunk, cell) inside ids
//   gsize  i64 [Ns][K'^2]        GLOBAL cell sizes (all shards) for traversal
#pragma once

#include <vector>

#include "common.cuh"

namespace taco {

// Score-table chunk: the id range one CTA counts in shared memory.
//  cluster mode (single GPU, n <= kClusterMaxN): n is split over <= 16 CTAs of
//    one thread-block cluster (~64 KiB each), chunk = ceil(n / ctas) rounded to 1 KiB;
//  global mode (larger shards / multi-GPU): chunk = 64 KiB, tables in HBM.
constexpr int64_t kGlobalChunk = 65536;
constexpr int64_t kClusterMaxChunk = 131072;   // 4-bit tables: 64 KiB; 8-bit tables are capped at 98304
constexpr int64_t kClusterMaxChunk8 = 98304;
constexpr int64_t kClusterWideChunk = 262144;   // TACO_CLUSTER_IDS up to this with the 1024-thread encoded count
constexpr int kClusterMaxCtas = 16;             // non-portable cluster size
constexpr int64_t kClusterMaxN = kClusterMaxChunk8 * kClusterMaxCtas;

struct DevBuf {
  void* p = nullptr;
  size_t bytes = 0;
  bool view = false;   // a window into another buffer (an arena): release() only forgets it
  int ensure(size_t want);
  void release();
  void view_of(void* base, size_t b) {
    release();
    p = b ? base : nullptr;
    bytes = b;
    view = b != 0;
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct QueryTile {
  DevBuf Q, qt, sd, sl, pops, npop, ret, flags, scores, part, hist, lvl, cnum, clocal, coff, qbase,
      cursor, cand, bpref, pd2, ppos, tseg, qthr, qb, qsq, qok, gsb, gsc, gtab, rlist, ppref, psum, tk_d2, tk_ids, out_ids, out_d;
  DevBuf xch;                   // k_count_pg: the groups' level-histogram exchange slots
  DevBuf tkx;                   // k_topk: the parts' best-k lists of split (long) queries
  int64_t cand_cap = 0;
  int pop_cap = 0;
  int64_t front_rows = 0;       // rows the split-traversal buffers were sized for
  bool fused = false;           // the tile ran k_count_fused: its answers are already in out_ids / out_d
  cudaEvent_t qev = nullptr;    // q_u8_prep done (the fused-count decision reads flags[4])
  int64_t* flags_h = nullptr;   // pinned copy of flags[0..3] (async read-back)
  void release();
};

struct BuildScratch {
  DevBuf xsq, best, bsum, picks, uni, forced, status, C64, csq, newlab, pd, changed, perm, lhist,
      loff, ctl, hsum, draws, leaves, pbuf, cbuf, iota, keys2, sorttmp, xp, xs, arena;
  std::vector<char> leaf_blob;   // host copy of the pairwise leaves + combine tree (exact replay)
  int64_t nleaves = 0, leaves_n = -1;
  cudaEvent_t ev[3] = {nullptr, nullptr, nullptr};   // TACO_DEBUG_TIMING
};

}  // namespace taco

struct taco_index {
  int device = 0;
  cudaStream_t stream = nullptr;
  int64_t n = 0, n_global = 0, id_base = 0, nchunks = 0, chunk = 0;
  bool cluster_mode = false;
  int d = 0, n_sub = 0, s = 0, K = 0, kp = 0, m1 = 0, m2 = 0, D = 0, iters = 0;
  taco::DevBuf X, mean, M, T, cb1, cb2, labels, hist, niter, ids, offs, gsize;
  taco::DevBuf cenc, coffs;   // encoded, group-padded CSR of the TMA count (build_count_csr)
  size_t cstride = 0;         // entries per subspace in cenc
  int cunit = 8;              // entries per cenc unit (8 cluster mode, 4 global mode)
  bool has_ccsr = false;
  taco::DevBuf Xn;            // lossless narrow copy of X for the rerank (xfmt != TACO_ROWS_F32)
  taco::DevBuf Xsq;           // u8 rows: int32 sum of squares per row (integer rerank path)
  int xfmt = 0;               // TACO_ROWS_*
  bool has_X = false, has_T = false, has_model = false, has_cb = false, has_labels = false,
       has_cells = false, has_gsize = false;
  std::vector<cudaStream_t> half_streams;
  std::vector<cudaEvent_t> half_ev;   // k-means graph join, one per half stream
  cudaEvent_t km_fork = nullptr;
  taco::QueryTile qt, qt2;      // two query tiles: the batch loop pipelines them on two streams
  cudaStream_t stream2 = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  void* hstage = nullptr;        // pinned host staging of host-API results (async per-tile D2H)
  size_t hstage_bytes = 0;
  std::vector<taco::BuildScratch> bs;
  cudaStream_t aux = nullptr;          // column-mean chain that runs behind the staged upload
  taco::DevBuf colstate, colmean;
  bool mean_ready = false;
};

namespace taco {
int with_device(int device);
int index_check(taco_index* idx);
// kernels shared between translation units
int launch_transform(cudaStream_t st, const float* P, int64_t np_, int d, int D,
                     const float* mean, const float* M, float* out, bool dim_major);
int build_count_csr(taco_index* idx);   // after the cells change (query.cu)
int launch_colmean(cudaStream_t st, const float* X, int64_t r0, int64_t r1, int64_t n, int d, double* state,
                   double* mean, int chained = 0);
}  // namespace taco
