// Index lifecycle, host<->device import/export, the fp64 transform GEMM.
#include <algorithm>
#include <atomic>
#include <cstring>
#include <chrono>
#include <emmintrin.h>
#include <mutex>
#include <condition_variable>
#include <functional>
#include <thread>
#include <vector>

#include "index.cuh"

namespace taco {

static thread_local std::string g_err;
static std::atomic<int64_t> g_launches{0};

void set_error(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
}

void count_launch(int n) { g_launches += n; }

// Device memory comes from the device's stream-ordered pool with an unbounded
// release threshold: freed blocks stay cached in the pool, so the scratch of a
// second build (or a resized query tile) is a pool hit instead of a
// cudaMalloc.  Allocation and free are issued on the legacy stream and
// completed before returning; release() first waits for all device work, which
// is the guarantee cudaFree gave the callers.
static void pool_setup() {
  static thread_local int done_dev = -1;
  int dev = 0;
  cudaGetDevice(&dev);
  if (done_dev == dev) return;
  cudaMemPool_t pool;
  if (cudaDeviceGetDefaultMemPool(&pool, dev) == cudaSuccess) {
    uint64_t thr = UINT64_MAX;
    cudaMemPoolSetAttribute(pool, cudaMemPoolAttrReleaseThreshold, &thr);
  }
  cudaGetLastError();
  done_dev = dev;
}

int DevBuf::ensure(size_t want) {
  if (want <= bytes && p) return TACO_OK;
  release();
  size_t b = want < 256 ? 256 : want;
  pool_setup();
  TACO_CHECK_CUDA(cudaMallocAsync(&p, b, cudaStreamLegacy));
  TACO_CHECK_CUDA(cudaStreamSynchronize(cudaStreamLegacy));
  bytes = b;
  return TACO_OK;
}

void QueryTile::release() {
  DevBuf* all[] = {&Q, &qt, &sd, &sl, &pops, &npop, &ret, &flags, &scores, &part, &hist, &lvl, &cnum, &clocal,
                  &coff, &qbase, &cursor, &cand, &bpref, &pd2, &ppos, &tseg, &qthr, &qb, &qsq, &qok, &gsb, &gsc, &gtab, &rlist, &ppref, &psum, &tk_d2, &tk_ids,
                  &out_ids, &out_d, &xch, &tkx};
  for (auto* b : all) b->release();
  if (flags_h) cudaFreeHost(flags_h);
  flags_h = nullptr;
  if (qev) cudaEventDestroy(qev);
  qev = nullptr;
  cand_cap = 0;
}

void DevBuf::release() {
  if (view) {
    p = nullptr;
    bytes = 0;
    view = false;
    return;
  }
  if (p) {
    cudaDeviceSynchronize();
    cudaFreeAsync(p, cudaStreamLegacy);
    cudaStreamSynchronize(cudaStreamLegacy);
  }
  p = nullptr;
  bytes = 0;
}

int with_device(int device) {
  TACO_CHECK_CUDA(cudaSetDevice(device));
  return TACO_OK;
}

int index_check(taco_index* idx) {
  if (!idx) TACO_FAIL(TACO_ERR_STATE, "null index handle");
  return with_device(idx->device);
}

// ------------------------------------------------------------ transform GEMM
// out = f32((f64 P - f64 mean) @ f64 M) (spectral.py:314-316).  Each output is
// one FMA chain over k = 0..d-1 starting from 0 -- the OpenBLAS dgemm order
// (DESIGN.md numerics).  64x64 output tile per 256-thread CTA, 4x4 per thread,
// k staged 16 at a time through shared memory in fp64.
constexpr int TM = 64, TN = 64, TK = 16;

__global__ void __launch_bounds__(256) k_transform(const float* __restrict__ P, int64_t np_, int d,
                                                   int D, const float* __restrict__ mean,
                                                   const float* __restrict__ M,
                                                   float* __restrict__ out, int dim_major) {
  __shared__ double As[TK][TM + 1];
  __shared__ double Bs[TK][TN + 1];
  const int tx = threadIdx.x & 15, ty = threadIdx.x >> 4;
  const int64_t r0 = int64_t(blockIdx.x) * TM;
  const int c0 = blockIdx.y * TN;
  double acc[4][4];
#pragma unroll
  for (int a = 0; a < 4; ++a)
#pragma unroll
    for (int b = 0; b < 4; ++b) acc[a][b] = 0.0;
  for (int k0 = 0; k0 < d; k0 += TK) {
    for (int e = threadIdx.x; e < TK * TM; e += 256) {
      int kk = e % TK, rr = e / TK;
      int64_t r = r0 + rr;
      int k = k0 + kk;
      double v = 0.0;
      if (r < np_ && k < d) v = __dsub_rn((double)P[r * d + k], (double)mean[k]);
      As[kk][rr] = v;
    }
    for (int e = threadIdx.x; e < TK * TN; e += 256) {
      int cc = e % TN, kk = e / TN;
      int c = c0 + cc, k = k0 + kk;
      Bs[kk][cc] = (c < D && k < d) ? (double)M[(int64_t)k * D + c] : 0.0;
    }
    __syncthreads();
    int kmax = min(TK, d - k0);
    for (int kk = 0; kk < kmax; ++kk) {
      double a[4], b[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) a[u] = As[kk][ty + 16 * u];
#pragma unroll
      for (int u = 0; u < 4; ++u) b[u] = Bs[kk][tx + 16 * u];
#pragma unroll
      for (int x = 0; x < 4; ++x)
#pragma unroll
        for (int y = 0; y < 4; ++y) acc[x][y] = __fma_rn(a[x], b[y], acc[x][y]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int x = 0; x < 4; ++x) {
    int64_t r = r0 + ty + 16 * x;
    if (r >= np_) continue;
#pragma unroll
    for (int y = 0; y < 4; ++y) {
      int c = c0 + tx + 16 * y;
      if (c >= D) continue;
      float v = __double2float_rn(acc[x][y]);
      if (dim_major)
        out[(int64_t)c * np_ + r] = v;
      else
        out[r * D + c] = v;
    }
  }
}

int launch_transform(cudaStream_t st, const float* P, int64_t np_, int d, int D, const float* mean,
                     const float* M, float* out, bool dim_major) {
  if (np_ == 0) return TACO_OK;
  dim3 grid((unsigned)ceil_div(np_, TM), (unsigned)ceil_div(D, TN));
  k_transform<<<grid, 256, 0, st>>>(P, np_, d, D, mean, M, out, dim_major ? 1 : 0);
  TACO_LAUNCHED();
  return TACO_OK;
}

}  // namespace taco

using namespace taco;

extern "C" {

const char* taco_last_error(void) { return g_err.c_str(); }
int taco_version(void) { return 1; }

int taco_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}
int64_t taco_launch_count(void) { return g_launches.load(); }

int taco_index_create(int device, int64_t n, int32_t d, int32_t n_subspaces, int32_t subspace_dim,
                      int32_t clusters, int32_t kmeans_iters, int64_t n_global, int64_t id_base,
                      taco_index** out) {
  if (!out) TACO_FAIL(TACO_ERR_PARAMETER, "null output handle");
  if (n < 1 || d < 1) TACO_FAIL(TACO_ERR_PARAMETER, "empty data (%lld x %d)", (long long)n, d);
  if (n_subspaces < 1 || n_subspaces > 255)
    TACO_FAIL(TACO_ERR_PARAMETER, "subspace count %d outside [1, 255]", n_subspaces);
  if (subspace_dim < 2) TACO_FAIL(TACO_ERR_PARAMETER, "subspace dimension %d is below 2", subspace_dim);
  int kp = 0;
  while ((int64_t)(kp + 1) * (kp + 1) <= clusters) ++kp;
  if (kp < 1 || kp * kp != clusters)
    TACO_FAIL(TACO_ERR_PARAMETER, "cluster count %d is not a perfect square", clusters);
  if (kp > 256) TACO_FAIL(TACO_ERR_PARAMETER, "per-codebook cluster count %d exceeds 256", kp);
  if ((int64_t)n_subspaces * subspace_dim > d)
    TACO_FAIL(TACO_ERR_PARAMETER, "subspace budget %d (%d x %d) exceeds data dimension %d",
              n_subspaces * subspace_dim, n_subspaces, subspace_dim, d);
  if (n > 0xFFFFFFFFLL) TACO_FAIL(TACO_ERR_PARAMETER, "shard of %lld points exceeds 2^32", (long long)n);
  if ((int64_t)n_subspaces * n > 0xFFFFFFFFLL)
    TACO_FAIL(TACO_ERR_PARAMETER, "shard of %lld points x %d subspaces exceeds the 2^32 CSR index range",
              (long long)n, n_subspaces);
  if (n_global < n) n_global = n;
  TACO_TRY(with_device(device));
  auto* idx = new taco_index();
  idx->device = device;
  idx->n = n;
  idx->n_global = n_global;
  idx->id_base = id_base;
  idx->d = d;
  idx->n_sub = n_subspaces;
  idx->s = subspace_dim;
  idx->K = clusters;
  idx->kp = kp;
  idx->m1 = (subspace_dim + 1) / 2;
  idx->m2 = subspace_dim - idx->m1;
  idx->D = n_subspaces * subspace_dim;
  idx->iters = kmeans_iters;
  const char* force_global = getenv("TACO_GLOBAL_MODE");   // =1: global mode at any size (sharded-path checks)
  if (n_global == n && n <= kClusterMaxN && !(force_global && force_global[0] == '1')) {
    // ids per CTA: 4-bit tables (n_sub <= 15) 128K = 64 KiB, 8-bit tables 64K (TACO_CLUSTER_IDS overrides)
    int64_t target = n_subspaces <= 15 ? 131072 : 65536;
    if (const char* e = getenv("TACO_CLUSTER_IDS")) target = std::max<int64_t>(1024, atoll(e));
    // 4-bit tables up to 128K ids per CTA (256K for N_s <= 8 with TACO_COUNT_NT=1024: one 1024-thread CTA per SM)
    const char* wnt = getenv("TACO_COUNT_NT");
    const int64_t cap4 = (n_subspaces <= 8 && wnt && atoi(wnt) == 1024) ? kClusterWideChunk : kClusterMaxChunk;
    target = std::min(target, n_subspaces <= 15 ? cap4 : kClusterMaxChunk8);
    const int ctas = (int)std::min<int64_t>(kClusterMaxCtas, std::max<int64_t>(1, ceil_div(n, target)));
    idx->chunk = ceil_div(ceil_div(n, ctas), 1024) * 1024;
    idx->cluster_mode = true;
  } else {
    // 4-bit tables: 64K-id chunks, 128K past 64 of them (every CTA looks up every
    // popped cell, so the slice lookups grow with the chunk count, and a cell's
    // slice of a chunk shrinks to a few ids: config 4 k_count 45.0 -> 42.5 ms per
    // 10,000 queries, config 5 152 -> 138 ms per 2,000; config 2 forced into
    // global mode measures the same either way); TACO_GLOBAL_CHUNK overrides
    idx->chunk = (n_subspaces <= 15 && n > 64 * kGlobalChunk) ? kClusterMaxChunk : kGlobalChunk;
    if (const char* e = getenv("TACO_GLOBAL_CHUNK"))
      idx->chunk = std::min<int64_t>(n_subspaces <= 15 ? kClusterMaxChunk : kClusterMaxChunk8,
                                     std::max<int64_t>(1024, atoll(e) / 1024 * 1024));
    idx->cluster_mode = false;
  }
  idx->nchunks = ceil_div(n, idx->chunk);
  cudaError_t e = cudaStreamCreateWithFlags(&idx->stream, cudaStreamNonBlocking);
  if (e != cudaSuccess) {
    delete idx;
    TACO_FAIL(TACO_ERR_CUDA, "stream create: %s", cudaGetErrorString(e));
  }
  *out = idx;
  return TACO_OK;
}

int taco_index_destroy(taco_index* idx) {
  if (!idx) return TACO_OK;
  cudaSetDevice(idx->device);
  cudaStreamSynchronize(idx->stream);
  DevBuf* bufs[] = {&idx->X, &idx->Xn, &idx->Xsq, &idx->mean, &idx->M, &idx->T, &idx->cb1, &idx->cb2, &idx->labels,
                    &idx->hist, &idx->niter, &idx->ids, &idx->offs, &idx->gsize, &idx->cenc, &idx->coffs};
  for (auto* b : bufs) b->release();
  idx->qt.release();
  idx->qt2.release();
  for (auto& s : idx->bs) {
    DevBuf* sb[] = {&s.xsq, &s.best, &s.bsum, &s.picks, &s.uni, &s.forced, &s.status, &s.C64,
                    &s.csq, &s.newlab, &s.pd, &s.changed, &s.perm, &s.lhist, &s.loff, &s.ctl,
                    &s.hsum, &s.draws, &s.leaves, &s.pbuf, &s.cbuf, &s.iota, &s.keys2, &s.sorttmp, &s.xp, &s.xs, &s.arena};
    for (auto* b : sb) b->release();
  }
  for (auto st : idx->half_streams) cudaStreamDestroy(st);
  for (auto e : idx->half_ev) cudaEventDestroy(e);
  if (idx->km_fork) cudaEventDestroy(idx->km_fork);
  if (idx->stream2) cudaStreamDestroy(idx->stream2);
  if (idx->aux) cudaStreamDestroy(idx->aux);
  idx->colstate.release();
  idx->colmean.release();
  if (idx->ev_fork) cudaEventDestroy(idx->ev_fork);
  if (idx->ev_join) cudaEventDestroy(idx->ev_join);
  if (idx->hstage) cudaFreeHost(idx->hstage);
  cudaStreamDestroy(idx->stream);
  delete idx;
  return TACO_OK;
}

namespace taco {
// ok[0] &= every value is an integer 0..255 (bit-exact round trip through u8),
// ok[1] &= every value round-trips exactly through f16
__global__ void k_row_formats(const float* __restrict__ X, size_t N, int* __restrict__ ok) {
  bool u8 = true, f16 = true;
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x) {
    const float x = X[i];
    const uint32_t b = __float_as_uint(x);
    const bool in = x >= 0.0f && x <= 255.0f;
    u8 = u8 && in && __float_as_uint((float)(uint32_t)x) == b;
    f16 = f16 && __float_as_uint(__half2float(__float2half_rn(x))) == b;
  }
  if (!__all_sync(0xffffffffu, u8) && (threadIdx.x & 31) == 0) atomicAnd(ok, 0);
  if (!__all_sync(0xffffffffu, f16) && (threadIdx.x & 31) == 0) atomicAnd(ok + 1, 0);
}
__global__ void k_rows_u8(const float* __restrict__ X, size_t N, uint8_t* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x)
    out[i] = (uint8_t)(uint32_t)X[i];
}
__global__ void k_rows_sq(const uint8_t* __restrict__ Xn, int64_t n, int d, int32_t* __restrict__ sq) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t* r = reinterpret_cast<const uint32_t*>(Xn + i * d);
    uint32_t acc = 0;
    for (int w = 0; w < d / 4; ++w) acc = __dp4a(r[w], r[w], acc);
    sq[i] = (int32_t)acc;
  }
}
__global__ void k_rows_f16(const float* __restrict__ X, size_t N, __half* __restrict__ out) {
  for (size_t i = (size_t)blockIdx.x * blockDim.x + threadIdx.x; i < N; i += (size_t)gridDim.x * blockDim.x)
    out[i] = __float2half_rn(X[i]);
}

// choose the rerank's row storage (lossless only) after X changed
static int narrow_rows(taco_index* idx) {
  idx->xfmt = TACO_ROWS_F32;
  idx->Xn.release();
  idx->Xsq.release();
  const char* env = getenv("TACO_ROWS");
  if (env && strcmp(env, "f32") == 0) return TACO_OK;
  const size_t N = (size_t)idx->n * idx->d;
  if (N == 0) return TACO_OK;
  DevBuf ok;
  TACO_TRY(ok.ensure(2 * sizeof(int)));
  const int ones[2] = {1, 1};
  int res[2] = {0, 0};
  TACO_CHECK_CUDA(cudaMemcpyAsync(ok.p, ones, sizeof(ones), cudaMemcpyHostToDevice, idx->stream));
  k_row_formats<<<1184, 256, 0, idx->stream>>>(idx->X.as<float>(), N, ok.as<int>());
  count_launch();
  TACO_CHECK_CUDA(cudaMemcpyAsync(res, ok.p, sizeof(res), cudaMemcpyDeviceToHost, idx->stream));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  ok.release();
  if (res[0] && idx->d % 16 == 0) {
    TACO_TRY(idx->Xn.ensure(N));
    k_rows_u8<<<1184, 256, 0, idx->stream>>>(idx->X.as<float>(), N, idx->Xn.as<uint8_t>());
    TACO_TRY(idx->Xsq.ensure(sizeof(int32_t) * (size_t)idx->n));
    k_rows_sq<<<1184, 256, 0, idx->stream>>>(idx->Xn.as<uint8_t>(), idx->n, idx->d, idx->Xsq.as<int32_t>());
    count_launch(2);
    idx->xfmt = TACO_ROWS_U8;
  } else if (res[1] && idx->d % 8 == 0) {
    TACO_TRY(idx->Xn.ensure(2 * N));
    k_rows_f16<<<1184, 256, 0, idx->stream>>>(idx->X.as<float>(), N, idx->Xn.as<__half>());
    count_launch();
    idx->xfmt = TACO_ROWS_F16;
  }
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  return TACO_OK;
}
}  // namespace taco

namespace taco {
// Host -> device upload of a pageable buffer (the numpy base vectors) through
// a ring of pinned staging buffers: the host threads copy chunk i+1 into one
// buffer while the DMA engine drains chunk i from another, so the upload runs
// at min(host memcpy, PCIe) instead of the driver's single-threaded pageable
// path.  Already-pinned sources go straight to cudaMemcpyAsync.
constexpr size_t kStageBytes = 32u << 20;
constexpr int kStages = 3;
static std::mutex g_stage_mu;
static char* g_stage[kStages] = {nullptr, nullptr, nullptr};
static cudaEvent_t g_stage_ev[kStages] = {nullptr, nullptr, nullptr};

// memcpy into the pinned staging with non-temporal 16-byte stores: the
// destination lines are not read for ownership first (the staging is written
// once and then read by the DMA engine), so the host memory traffic of the
// copy drops from ~3x to 2x the bytes moved.
static void stream_copy(char* dst, const char* src, size_t len) {
  size_t i = 0;
  const size_t head = (16 - (reinterpret_cast<uintptr_t>(dst) & 15)) & 15;
  if (head) {
    const size_t h = std::min(head, len);
    memcpy(dst, src, h);
    i = h;
  }
  for (; i + 64 <= len; i += 64) {
    const __m128i a = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i));
    const __m128i b = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 16));
    const __m128i c = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 32));
    const __m128i e = _mm_loadu_si128(reinterpret_cast<const __m128i*>(src + i + 48));
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i), a);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 16), b);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 32), c);
    _mm_stream_si128(reinterpret_cast<__m128i*>(dst + i + 48), e);
  }
  if (i < len) memcpy(dst + i, src + i, len - i);
  _mm_sfence();
}

// Host copy workers for the staged upload: plain threads that BLOCK between
// jobs (an OpenMP team would spin for ~100 ms after each region and starve
// the launch thread of the build that follows).
class CopyPool {
 public:
  static CopyPool& get() {
    // never destroyed: the workers block on cv_ for the life of the process, and
    // destroying a condition variable with waiters at exit can hang the exit
    static CopyPool* p = new CopyPool();
    return *p;
  }
  // dst[0, len) = src[0, len) split over the workers; returns when done
  void copy(char* dst, const char* src, size_t len) {
    std::unique_lock<std::mutex> lk(mu_);
    dst_ = dst;
    src_ = src;
    len_ = len;
    pending_ = (int)workers_.size();
    ++gen_;
    cv_.notify_all();
    done_.wait(lk, [&] { return pending_ == 0; });
  }

 private:
  CopyPool() {
    const int n = std::max(1, std::min(16, (int)std::thread::hardware_concurrency()));
    for (int t = 0; t < n; ++t) workers_.emplace_back([this, t, n] { run(t, n); });
    for (auto& w : workers_) w.detach();
  }
  void run(int t, int n) {
    uint64_t seen = 0;
    for (;;) {
      char* d;
      const char* s;
      size_t len;
      {
        std::unique_lock<std::mutex> lk(mu_);
        cv_.wait(lk, [&] { return gen_ != seen; });
        seen = gen_;
        d = dst_;
        s = src_;
        len = len_;
      }
      const size_t a0 = len * t / n, a1 = len * (t + 1) / n;
      stream_copy(d + a0, s + a0, a1 - a0);
      std::lock_guard<std::mutex> lk(mu_);
      if (--pending_ == 0) done_.notify_one();
    }
  }
  std::mutex mu_;
  std::condition_variable cv_, done_;
  std::vector<std::thread> workers_;
  char* dst_ = nullptr;
  const char* src_ = nullptr;
  size_t len_ = 0;
  int pending_ = 0;
  uint64_t gen_ = 0;
};

int upload_h2d(void* dst, const void* src, size_t bytes, cudaStream_t st,
               const std::function<int(size_t, cudaEvent_t)>& on_chunk) {
  cudaPointerAttributes pa;
  const bool pinned = cudaPointerGetAttributes(&pa, src) == cudaSuccess && pa.type == cudaMemoryTypeHost;
  cudaGetLastError();
  if (pinned || bytes <= 2 * kStageBytes) {
    TACO_CHECK_CUDA(cudaMemcpyAsync(dst, src, bytes, cudaMemcpyHostToDevice, st));
    TACO_CHECK_CUDA(cudaStreamSynchronize(st));
    return TACO_OK;
  }
  std::lock_guard<std::mutex> lk(g_stage_mu);
  for (int b = 0; b < kStages; ++b) {
    if (!g_stage[b]) {
      TACO_CHECK_CUDA(cudaHostAlloc((void**)&g_stage[b], kStageBytes, cudaHostAllocDefault));
      TACO_CHECK_CUDA(cudaEventCreateWithFlags(&g_stage_ev[b], cudaEventDisableTiming));
    }
  }
  const char* s = static_cast<const char*>(src);
  char* d = static_cast<char*>(dst);
  CopyPool& pool = CopyPool::get();
  static const bool dbg = getenv("TACO_DEBUG_UPLOAD") != nullptr;
  double t_wait = 0.0, t_copy = 0.0;
  for (size_t off = 0, i = 0; off < bytes; off += kStageBytes, ++i) {
    const int b = (int)(i % kStages);
    const size_t len = std::min(kStageBytes, bytes - off);
    const auto ta = std::chrono::steady_clock::now();
    TACO_CHECK_CUDA(cudaEventSynchronize(g_stage_ev[b]));   // buffer b drained
    const auto tb = std::chrono::steady_clock::now();
    char* stg = g_stage[b];
    pool.copy(stg, s + off, len);
    const auto tc = std::chrono::steady_clock::now();
    t_wait += std::chrono::duration<double, std::milli>(tb - ta).count();
    t_copy += std::chrono::duration<double, std::milli>(tc - tb).count();
    TACO_CHECK_CUDA(cudaMemcpyAsync(d + off, stg, len, cudaMemcpyHostToDevice, st));
    TACO_CHECK_CUDA(cudaEventRecord(g_stage_ev[b], st));
    if (on_chunk) TACO_TRY(on_chunk(off + len, g_stage_ev[b]));   // bytes [0, off + len) have landed once ev fires
  }
  TACO_CHECK_CUDA(cudaStreamSynchronize(st));
  if (dbg) fprintf(stderr, "[taco] upload: host copies %.2f ms, waits for a drained buffer %.2f ms\n", t_copy, t_wait);
  return TACO_OK;
}
}  // namespace taco

int taco_index_set_data(taco_index* idx, const float* X_h) {
  TACO_TRY(index_check(idx));
  size_t bytes = (size_t)idx->n * idx->d * sizeof(float);
  TACO_TRY(idx->X.ensure(bytes));
  // the sequential column-mean chain of fit_covariance follows the staged
  // upload chunk by chunk on the aux stream (it is bound by the DADD latency,
  // the upload by PCIe: run together they overlap)
  idx->mean_ready = false;
  if (!idx->aux) TACO_CHECK_CUDA(cudaStreamCreateWithFlags(&idx->aux, cudaStreamNonBlocking));
  TACO_TRY(idx->colstate.ensure(8 * (size_t)idx->d));
  TACO_TRY(idx->colmean.ensure(8 * (size_t)idx->d));
  int64_t rows_done = 0;
  const size_t row_bytes = sizeof(float) * (size_t)idx->d;
  auto on_chunk = [&](size_t landed, cudaEvent_t ev) -> int {
    const int64_t rows = (int64_t)(landed / row_bytes);
    if (rows <= rows_done) return TACO_OK;
    TACO_CHECK_CUDA(cudaStreamWaitEvent(idx->aux, ev, 0));
    TACO_TRY(launch_colmean(idx->aux, idx->X.as<float>(), rows_done, rows, idx->n, idx->d,
                            idx->colstate.as<double>(), idx->colmean.as<double>()));
    rows_done = rows;
    return TACO_OK;
  };
  static const bool dbg = getenv("TACO_DEBUG_UPLOAD") != nullptr;
  const auto t0 = std::chrono::steady_clock::now();
  TACO_TRY(upload_h2d(idx->X.p, X_h, bytes, idx->stream, on_chunk));
  const auto t1 = std::chrono::steady_clock::now();
  idx->mean_ready = rows_done == idx->n;
  idx->has_X = true;
  const int rc = narrow_rows(idx);
  if (dbg) {
    cudaStreamSynchronize(idx->aux);
    const auto t2 = std::chrono::steady_clock::now();
    fprintf(stderr, "[taco] set_data: upload %.2f ms, narrow rows %.2f ms (%zu MB)\n",
            std::chrono::duration<double, std::milli>(t1 - t0).count(),
            std::chrono::duration<double, std::milli>(t2 - t1).count(), bytes >> 20);
  }
  return rc;
}

int32_t taco_index_row_format(const taco_index* idx) {
  if (!idx || !idx->has_X) return -1;
  return idx->xfmt;
}

int taco_index_layout(const taco_index* idx, int64_t* chunk, int64_t* nchunks, int32_t* cluster_mode) {
  TACO_TRY(index_check(const_cast<taco_index*>(idx)));
  if (chunk) *chunk = idx->chunk;
  if (nchunks) *nchunks = idx->nchunks;
  if (cluster_mode) *cluster_mode = idx->cluster_mode ? 1 : 0;
  return TACO_OK;
}

int taco_index_set_data_device(taco_index* idx, const float* X_d) {
  TACO_TRY(index_check(idx));
  idx->mean_ready = false;
  size_t bytes = (size_t)idx->n * idx->d * sizeof(float);
  TACO_TRY(idx->X.ensure(bytes));
  TACO_CHECK_CUDA(cudaMemcpyAsync(idx->X.p, X_d, bytes, cudaMemcpyDeviceToDevice, idx->stream));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  idx->has_X = true;
  return narrow_rows(idx);
}

int taco_index_set_transform(taco_index* idx, const float* mean_h, const float* matrix_h) {
  TACO_TRY(index_check(idx));
  TACO_TRY(idx->mean.ensure(sizeof(float) * idx->d));
  TACO_TRY(idx->M.ensure(sizeof(float) * (size_t)idx->d * idx->D));
  TACO_CHECK_CUDA(cudaMemcpy(idx->mean.p, mean_h, sizeof(float) * idx->d, cudaMemcpyHostToDevice));
  TACO_CHECK_CUDA(cudaMemcpy(idx->M.p, matrix_h, sizeof(float) * (size_t)idx->d * idx->D,
                             cudaMemcpyHostToDevice));
  idx->has_model = true;
  return TACO_OK;
}

int taco_transform_data(taco_index* idx) {
  TACO_TRY(index_check(idx));
  if (!idx->has_X || !idx->has_model) TACO_FAIL(TACO_ERR_STATE, "transform needs data and model");
  TACO_TRY(idx->T.ensure(sizeof(float) * (size_t)idx->n * idx->D));
  TACO_TRY(launch_transform(idx->stream, idx->X.as<float>(), idx->n, idx->d, idx->D,
                            idx->mean.as<float>(), idx->M.as<float>(), idx->T.as<float>(), true));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  idx->has_T = true;
  return TACO_OK;
}

int taco_index_set_transformed(taco_index* idx, const float* T_h) {
  TACO_TRY(index_check(idx));
  const int64_t n = idx->n;
  const int D = idx->D;
  std::vector<float> tr((size_t)n * D);
  for (int64_t r = 0; r < n; ++r)
    for (int c = 0; c < D; ++c) tr[(size_t)c * n + r] = T_h[(size_t)r * D + c];
  TACO_TRY(idx->T.ensure(sizeof(float) * tr.size()));
  TACO_CHECK_CUDA(cudaMemcpy(idx->T.p, tr.data(), sizeof(float) * tr.size(), cudaMemcpyHostToDevice));
  idx->has_T = true;
  return TACO_OK;
}

// Device-resident exchange of the transformed matrix (point-sharded build):
// dimension-major [D][n] f32, the index's own layout.
int taco_index_set_transformed_device(taco_index* idx, const float* T_d) {
  TACO_TRY(index_check(idx));
  const size_t bytes = sizeof(float) * (size_t)idx->n * idx->D;
  TACO_TRY(idx->T.ensure(bytes));
  TACO_CHECK_CUDA(cudaMemcpyAsync(idx->T.p, T_d, bytes, cudaMemcpyDeviceToDevice, idx->stream));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  idx->has_T = true;
  return TACO_OK;
}

int taco_get_transformed_device(taco_index* idx, float* T_d) {
  TACO_TRY(index_check(idx));
  if (!idx->has_T) TACO_FAIL(TACO_ERR_STATE, "transformed matrix not available");
  TACO_CHECK_CUDA(cudaMemcpyAsync(T_d, idx->T.p, sizeof(float) * (size_t)idx->n * idx->D,
                                  cudaMemcpyDeviceToDevice, idx->stream));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  return TACO_OK;
}

// labels [2 N_s][n] i32, half 2j = codebook 1 of subspace j, 2j+1 = codebook 2
int taco_get_labels_device(taco_index* idx, int32_t* lab_d) {
  TACO_TRY(index_check(idx));
  if (!idx->has_labels) TACO_FAIL(TACO_ERR_STATE, "labels not available");
  for (auto s : idx->half_streams) TACO_CHECK_CUDA(cudaStreamSynchronize(s));
  TACO_CHECK_CUDA(cudaMemcpyAsync(lab_d, idx->labels.p, sizeof(int32_t) * (size_t)idx->n * 2 * idx->n_sub,
                                  cudaMemcpyDeviceToDevice, idx->stream));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  return TACO_OK;
}

int taco_index_set_labels_device(taco_index* idx, const int32_t* lab_d) {
  TACO_TRY(index_check(idx));
  const size_t bytes = sizeof(int32_t) * (size_t)idx->n * 2 * idx->n_sub;
  TACO_TRY(idx->labels.ensure(bytes));
  TACO_CHECK_CUDA(cudaMemcpyAsync(idx->labels.p, lab_d, bytes, cudaMemcpyDeviceToDevice, idx->stream));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  idx->has_labels = true;
  return TACO_OK;
}

int taco_get_transformed(taco_index* idx, float* T_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_T) TACO_FAIL(TACO_ERR_STATE, "transformed matrix not available");
  const int64_t n = idx->n;
  const int D = idx->D;
  std::vector<float> tr((size_t)n * D);
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  TACO_CHECK_CUDA(cudaMemcpy(tr.data(), idx->T.p, sizeof(float) * tr.size(), cudaMemcpyDeviceToHost));
  for (int64_t r = 0; r < n; ++r)
    for (int c = 0; c < D; ++c) T_h[(size_t)r * D + c] = tr[(size_t)c * n + r];
  return TACO_OK;
}

int taco_index_set_codebooks(taco_index* idx, const float* cb1_h, const float* cb2_h) {
  TACO_TRY(index_check(idx));
  size_t b1 = sizeof(float) * (size_t)idx->n_sub * idx->kp * idx->m1;
  size_t b2 = sizeof(float) * (size_t)idx->n_sub * idx->kp * idx->m2;
  TACO_TRY(idx->cb1.ensure(b1));
  TACO_TRY(idx->cb2.ensure(b2));
  TACO_CHECK_CUDA(cudaMemcpy(idx->cb1.p, cb1_h, b1, cudaMemcpyHostToDevice));
  TACO_CHECK_CUDA(cudaMemcpy(idx->cb2.p, cb2_h, b2, cudaMemcpyHostToDevice));
  idx->has_cb = true;
  return TACO_OK;
}

int taco_get_codebooks(taco_index* idx, float* cb1_h, float* cb2_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_cb) TACO_FAIL(TACO_ERR_STATE, "codebooks not built");
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  TACO_CHECK_CUDA(cudaMemcpy(cb1_h, idx->cb1.p, sizeof(float) * (size_t)idx->n_sub * idx->kp * idx->m1,
                             cudaMemcpyDeviceToHost));
  TACO_CHECK_CUDA(cudaMemcpy(cb2_h, idx->cb2.p, sizeof(float) * (size_t)idx->n_sub * idx->kp * idx->m2,
                             cudaMemcpyDeviceToHost));
  return TACO_OK;
}

int taco_index_set_labels(taco_index* idx, const int32_t* lab1_h, const int32_t* lab2_h) {
  TACO_TRY(index_check(idx));
  const int64_t n = idx->n;
  TACO_TRY(idx->labels.ensure(sizeof(int32_t) * (size_t)n * 2 * idx->n_sub));
  int32_t* L = idx->labels.as<int32_t>();
  for (int j = 0; j < idx->n_sub; ++j) {
    TACO_CHECK_CUDA(cudaMemcpy(L + (size_t)(2 * j) * n, lab1_h + (size_t)j * n, sizeof(int32_t) * n,
                               cudaMemcpyHostToDevice));
    TACO_CHECK_CUDA(cudaMemcpy(L + (size_t)(2 * j + 1) * n, lab2_h + (size_t)j * n,
                               sizeof(int32_t) * n, cudaMemcpyHostToDevice));
  }
  idx->has_labels = true;
  return TACO_OK;
}

int taco_get_labels(taco_index* idx, int32_t* lab1_h, int32_t* lab2_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_labels) TACO_FAIL(TACO_ERR_STATE, "labels not available");
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  const int64_t n = idx->n;
  const int32_t* L = idx->labels.as<int32_t>();
  for (int j = 0; j < idx->n_sub; ++j) {
    TACO_CHECK_CUDA(cudaMemcpy(lab1_h + (size_t)j * n, L + (size_t)(2 * j) * n, sizeof(int32_t) * n,
                               cudaMemcpyDeviceToHost));
    TACO_CHECK_CUDA(cudaMemcpy(lab2_h + (size_t)j * n, L + (size_t)(2 * j + 1) * n,
                               sizeof(int32_t) * n, cudaMemcpyDeviceToHost));
  }
  return TACO_OK;
}

int taco_get_history(taco_index* idx, double* hist_h, int32_t* n_iter_h) {
  TACO_TRY(index_check(idx));
  if (!idx->hist.p) TACO_FAIL(TACO_ERR_STATE, "no k-means history (index was imported)");
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  TACO_CHECK_CUDA(cudaMemcpy(hist_h, idx->hist.p, sizeof(double) * 2 * idx->n_sub * idx->iters,
                             cudaMemcpyDeviceToHost));
  TACO_CHECK_CUDA(cudaMemcpy(n_iter_h, idx->niter.p, sizeof(int32_t) * 2 * idx->n_sub,
                             cudaMemcpyDeviceToHost));
  return TACO_OK;
}

// Cell-major CSR import: rebuild the chunk-major layout on the host (import
// is not a hot path; it is the v1-file / oracle bridge).
int taco_index_set_cells(taco_index* idx, const int64_t* offsets_h, const uint32_t* ids_h) {
  TACO_TRY(index_check(idx));
  const int64_t n = idx->n, nc = idx->nchunks;
  const int K2 = idx->kp * idx->kp;
  const size_t offs_len = (size_t)nc * K2 + 1;
  TACO_TRY(idx->ids.ensure(sizeof(uint32_t) * (size_t)n * idx->n_sub));
  TACO_TRY(idx->offs.ensure(sizeof(uint32_t) * offs_len * idx->n_sub));
  TACO_TRY(idx->gsize.ensure(sizeof(int64_t) * (size_t)K2 * idx->n_sub));
  std::vector<uint32_t> ids(n), offs(offs_len);
  std::vector<int64_t> gs(K2);
  std::vector<int64_t> cnt((size_t)nc * K2);
  for (int j = 0; j < idx->n_sub; ++j) {
    const int64_t* O = offsets_h + (size_t)j * (K2 + 1);
    const uint32_t* I = ids_h + (size_t)j * n;
    if (O[0] != 0 || O[K2] != n)
      TACO_FAIL(TACO_ERR_FORMAT, "subspace %d cells hold %lld ids, expected %lld", j,
                (long long)(O[K2] - O[0]), (long long)n);
    std::fill(cnt.begin(), cnt.end(), 0);
    for (int c = 0; c < K2; ++c) {
      gs[c] = O[c + 1] - O[c];
      for (int64_t p = O[c]; p < O[c + 1]; ++p) {
        if (I[p] >= (uint64_t)n) TACO_FAIL(TACO_ERR_FORMAT, "cell id %u out of range", I[p]);
        cnt[(size_t)(I[p] / idx->chunk) * K2 + c]++;
      }
    }
    int64_t run = 0;
    for (size_t e = 0; e < (size_t)nc * K2; ++e) {
      offs[e] = (uint32_t)run;
      run += cnt[e];
    }
    offs[(size_t)nc * K2] = (uint32_t)run;
    std::vector<uint32_t> cur(offs.begin(), offs.end() - 1);
    for (int c = 0; c < K2; ++c)
      for (int64_t p = O[c]; p < O[c + 1]; ++p) {
        size_t slot = (size_t)(I[p] / idx->chunk) * K2 + c;
        ids[cur[slot]++] = I[p];
      }
    TACO_CHECK_CUDA(cudaMemcpy(idx->ids.as<uint32_t>() + (size_t)j * n, ids.data(),
                               sizeof(uint32_t) * n, cudaMemcpyHostToDevice));
    TACO_CHECK_CUDA(cudaMemcpy(idx->offs.as<uint32_t>() + (size_t)j * offs_len, offs.data(),
                               sizeof(uint32_t) * offs_len, cudaMemcpyHostToDevice));
    if (!idx->has_gsize || idx->n_global == idx->n)
      TACO_CHECK_CUDA(cudaMemcpy(idx->gsize.as<int64_t>() + (size_t)j * K2, gs.data(),
                                 sizeof(int64_t) * K2, cudaMemcpyHostToDevice));
  }
  idx->has_cells = true;
  if (idx->n_global == idx->n) idx->has_gsize = true;
  TACO_TRY(build_count_csr(idx));
  return TACO_OK;
}

int taco_index_set_global_sizes(taco_index* idx, const int64_t* sizes_h) {
  TACO_TRY(index_check(idx));
  const int K2 = idx->kp * idx->kp;
  TACO_TRY(idx->gsize.ensure(sizeof(int64_t) * (size_t)K2 * idx->n_sub));
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  TACO_CHECK_CUDA(cudaMemcpy(idx->gsize.p, sizes_h, sizeof(int64_t) * (size_t)K2 * idx->n_sub,
                             cudaMemcpyHostToDevice));
  idx->has_gsize = true;
  return TACO_OK;
}

int taco_get_global_sizes(taco_index* idx, int64_t* sizes_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_gsize) TACO_FAIL(TACO_ERR_STATE, "cell sizes not available");
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  const int K2 = idx->kp * idx->kp;
  TACO_CHECK_CUDA(cudaMemcpy(sizes_h, idx->gsize.p, sizeof(int64_t) * (size_t)K2 * idx->n_sub,
                             cudaMemcpyDeviceToHost));
  return TACO_OK;
}

int taco_get_cells(taco_index* idx, int32_t j, int64_t* offsets_h, uint32_t* ids_h) {
  TACO_TRY(index_check(idx));
  if (!idx->has_cells) TACO_FAIL(TACO_ERR_STATE, "cells not built");
  if (j < 0 || j >= idx->n_sub) TACO_FAIL(TACO_ERR_PARAMETER, "subspace %d out of range", j);
  const int64_t n = idx->n, nc = idx->nchunks;
  const int K2 = idx->kp * idx->kp;
  const size_t offs_len = (size_t)nc * K2 + 1;
  std::vector<uint32_t> ids(n), offs(offs_len);
  TACO_CHECK_CUDA(cudaStreamSynchronize(idx->stream));
  TACO_CHECK_CUDA(cudaMemcpy(ids.data(), idx->ids.as<uint32_t>() + (size_t)j * n,
                             sizeof(uint32_t) * n, cudaMemcpyDeviceToHost));
  TACO_CHECK_CUDA(cudaMemcpy(offs.data(), idx->offs.as<uint32_t>() + (size_t)j * offs_len,
                             sizeof(uint32_t) * offs_len, cudaMemcpyDeviceToHost));
  // cell-major = for each cell, its chunk slices in chunk order (ids ascending)
  int64_t w = 0;
  for (int c = 0; c < K2; ++c) {
    offsets_h[c] = w;
    for (int64_t ch = 0; ch < nc; ++ch) {
      size_t e = (size_t)ch * K2 + c;
      for (uint32_t p = offs[e]; p < offs[e + 1]; ++p) ids_h[w++] = ids[p];
    }
  }
  offsets_h[K2] = w;
  return TACO_OK;
}

}  // extern "C"
