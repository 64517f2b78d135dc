/*
 * taco_b200.h -- C ABI of the B200-native TaCo hot path (libtaco_b200.so).
 *
 * Plain pointers and sizes only.  Every entry point returns a status code
 * (TACO_OK == 0) and leaves a message in taco_last_error() (thread-local)
 * on failure; the Python host maps the codes onto the reference's
 * exception hierarchy (reference errors.py:4-45).
 *
 * The reference (pkg/src/taco) is pure Python/numpy and has no FFI; the
 * drop-in boundary is its Python engine API.  Each entry point below names
 * the reference function whose arithmetic it replaces; the Python mirror in
 * paper_2603_24919_b200/ binds them with ctypes.
 *
 * Pointers suffixed _h are host memory, _d device memory (cuda:device of
 * the index).  Stream arguments are cudaStream_t passed as void*; NULL is
 * the index's own (non-blocking) stream -- pass cudaStreamLegacy ((void*)1)
 * to order work with the legacy default stream.
 */
#ifndef TACO_B200_H
#define TACO_B200_H

#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  TACO_OK = 0,
  TACO_ERR_PARAMETER = 1,     /* ParameterError            errors.py:8   */
  TACO_ERR_DIMENSION = 2,     /* DimensionMismatchError    errors.py:12  */
  TACO_ERR_INSUFFICIENT = 3,  /* InsufficientDataError     errors.py:16  */
  TACO_ERR_NUMERIC = 4,       /* NumericError              errors.py:24  */
  TACO_ERR_CONVERGENCE = 5,   /* ConvergenceError          errors.py:28  */
  TACO_ERR_STATE = 6,         /* StateError                errors.py:44  */
  TACO_ERR_CUDA = 7,          /* CUDA runtime failure (no reference twin) */
  TACO_ERR_FORMAT = 8         /* FormatError               errors.py:32  */
};

typedef struct taco_index taco_index;

const char* taco_last_error(void);
/* Number of visible CUDA devices (0 when there is no usable GPU). */
int taco_device_count(void);
int taco_version(void);
/* Number of kernel launches issued by this process so far (bench evidence). */
int64_t taco_launch_count(void);

/* ------------------------------------------------------------- index life */
/* Creates an empty device index: IndexParams (engine.py:44-77) + n, d.
 * n_global/id_base describe the point shard this process owns (single GPU:
 * n_global = n, id_base = 0). */
int taco_index_create(int device, int64_t n, int32_t d, int32_t n_subspaces,
                      int32_t subspace_dim, int32_t clusters, int32_t kmeans_iters,
                      int64_t n_global, int64_t id_base, taco_index** out);
int taco_index_destroy(taco_index* idx);
/* Uploads the base vectors (owned device copy, used by build + rerank).
 * The rerank additionally keeps a lossless narrower copy of the rows when
 * EVERY value converts exactly (u8: integers 0..255, f16: exactly
 * representable halves; d a multiple of 16 / 8), so it reads 4x / 2x fewer
 * bytes per candidate with bit-identical distances.  TACO_ROWS=f32 in the
 * environment disables it. */
int taco_index_set_data(taco_index* idx, const float* X_h);
int taco_index_set_data_device(taco_index* idx, const float* X_d);
enum { TACO_ROWS_F32 = 0, TACO_ROWS_F16 = 1, TACO_ROWS_U8 = 2 };
/* Storage format the rerank reads rows in (TACO_ROWS_*), or -1 without data. */
int32_t taco_index_row_format(const taco_index* idx);
/* Id chunking of the count path: ids per chunk, the
 * number of chunks, and whether the index counts in cluster mode (one
 * thread-block cluster of nchunks CTAs per query) or global mode. */
int taco_index_layout(const taco_index* idx, int64_t* chunk, int64_t* nchunks, int32_t* cluster_mode);

/* ------------------------------------------------------------------ build */
/* spectral.fit_covariance (spectral.py:94-111): fp64 row mean (sequential,
 * bit-exact) and the centred Gram sum(x-mu)(x-mu)^T (fp64, unnormalised).
 * *bad_row = first row holding a non-finite value, or -1. */
int taco_fit_covariance(taco_index* idx, double* mean_h, double* gram_h, int64_t* bad_row);
/* spectral.jacobi_eigh sweeps (spectral.py:155-195), host, bit-exact restatement:
 * A (d x d, symmetric, row-major) is rotated in place, V receives the
 * eigenvectors (columns).  Returns TACO_ERR_CONVERGENCE past max_sweeps. */
int taco_jacobi_sweeps(double* A_h, double* V_h, int32_t d, double tol, int32_t max_sweeps,
                       int32_t* sweeps_out, double* residual_out);
/* The same sweeps on `device` (one cooperative kernel, eigen.cu); bit-identical
 * to taco_jacobi_sweeps (same IEEE operation sequence per element). */
int taco_jacobi_sweeps_device(int device, double* A_h, double* V_h, int32_t d, double tol, int32_t max_sweeps,
                              int32_t* sweeps_out, double* residual_out);
/* TransformModel (spectral.py:64-91): mean f32[d], matrix f32[d x D] row-major
 * (blocks concatenated column-wise). */
int taco_index_set_transform(taco_index* idx, const float* mean_h, const float* matrix_h);
/* spectral.transform_points on the owned data (spectral.py:301-316):
 * T = f32((f64 X - f64 mu) @ f64 M), stored dimension-major on device. */
int taco_transform_data(taco_index* idx);
/* Optional: replace T with a given host matrix (n x D row-major f32). */
int taco_index_set_transformed(taco_index* idx, const float* T_h);
/* clustering.kmeans for all 2*N_s halves (clustering.py:41-115, imi.py:67-69).
 * first_h[2Ns]: rng.integers(n) of each half; uniforms_h[2Ns*(K'-1)]: the
 * rng.random() draws; forced_h (nullable) [2Ns*(K'-1)]: >=0 forces a draw to
 * that point (the integers(n) branch taken when the D^2 total is 0).
 * degenerate_h[2Ns] receives the first draw whose D^2 total was 0 (K' if none). */
int taco_kmeans_all(taco_index* idx, const int64_t* first_h, const double* uniforms_h,
                    const int64_t* forced_h, int32_t* degenerate_h);
/* imi.build_subspace_index cells (imi.py:70-81): stable (l1,l2) sort into CSR. */
int taco_build_cells(taco_index* idx);
/* Replace the k-means state with given codebooks + labels (stage-wise parity). */
int taco_index_set_codebooks(taco_index* idx, const float* cb1_h, const float* cb2_h);
int taco_index_set_labels(taco_index* idx, const int32_t* lab1_h, const int32_t* lab2_h);
/* Import cells from a cell-major CSR per subspace (v1 file / oracle index):
 * offsets_h[j*(K'^2+1) ...] and ids_h[j*n ...]. */
int taco_index_set_cells(taco_index* idx, const int64_t* offsets_h, const uint32_t* ids_h);
/* Global cell sizes (u32[N_s*K'^2]) for a sharded index; single GPU derives them. */
int taco_index_set_global_sizes(taco_index* idx, const int64_t* sizes_h);

/* --------------------------------------------- point-sharded build (8(e)) */
/* Column-sum chain of this shard's rows (spectral.py:107, sequential fp64):
 * starts from carry_in_h[d] (the running sums after all earlier shards) or,
 * when NULL, from the shard's first row; carry_out_h[d] = the sums after its
 * last row.  *bad_row = first local row with a non-finite value, else -1
 * (spectral.py:102-105).  Ranks run it as a rank-ordered chain. */
int taco_shard_colsum(taco_index* idx, const double* carry_in_h, double* carry_out_h, int64_t* bad_row);
/* Centred Gram chain (spectral.py:108-109): carry_out_h[d*d] = carry_in_h (or
 * 0) + the Gram partials of this shard's rows in blocks of block_rows (<= 0:
 * taco_gram_block_rows(), the single-GPU decomposition), added in block
 * order.  Shards starting on multiples of block_rows, chained in rank order,
 * give exactly the single-GPU Gram. */
int taco_shard_gram(taco_index* idx, const double* mean_h, int64_t block_rows, const double* carry_in_h,
                    double* carry_out_h);
int taco_gram_block_rows(void);
/* Device copies of the transformed matrix (dimension-major [D][n] f32) and of
 * the k-means labels ([2 N_s][n] i32, half 2j / 2j+1 = codebook 1 / 2 of
 * subspace j): the all-to-all exchanges of the sharded k-means. */
int taco_index_set_transformed_device(taco_index* idx, const float* T_d);
int taco_get_transformed_device(taco_index* idx, float* T_d);
int taco_get_labels_device(taco_index* idx, int32_t* lab_d);
int taco_index_set_labels_device(taco_index* idx, const int32_t* lab_d);

/* ---------------------------------------------------------------- exports */
int taco_get_codebooks(taco_index* idx, float* cb1_h, float* cb2_h);
int taco_get_labels(taco_index* idx, int32_t* lab1_h, int32_t* lab2_h);
/* inertia history per half: hist_h[2Ns*iters], n_iter_h[2Ns] */
int taco_get_history(taco_index* idx, double* hist_h, int32_t* n_iter_h);
/* cell-major CSR of subspace j: offsets_h[K'^2+1], ids_h[n] (local ids) */
int taco_get_cells(taco_index* idx, int32_t j, int64_t* offsets_h, uint32_t* ids_h);
int taco_get_transformed(taco_index* idx, float* T_h);
int taco_get_global_sizes(taco_index* idx, int64_t* sizes_h);
/* Per-shard cell sizes i64[N_s*K'^2] (summed across ranks into the global table). */
int taco_get_local_sizes(taco_index* idx, int64_t* sizes_h);

/* ------------------------------------------------------------------ query */
/* Batched knn_query (engine.py:282-287 over a batch; padding of cli.py:155-164):
 * ids_h[nq*k] (-1 padded, global ids), dists_h[nq*k] (+inf padded),
 * cand_num_h[nq], last_coll_h[nq]. */
int taco_query_batch(taco_index* idx, const float* Q_h, int64_t nq, double alpha, double beta,
                     int32_t k, int32_t* ids_h, float* dists_h, int64_t* cand_num_h,
                     int32_t* last_coll_h);
/* Same with device buffers on `stream` (no host synchronisation except the
 * per-tile candidate-count readback). */
int taco_query_batch_device(taco_index* idx, const float* Q_d, int64_t nq, double alpha,
                            double beta, int32_t k, int32_t* ids_d, float* dists_d,
                            int64_t* cand_num_d, int32_t* last_coll_d, void* stream);
/* Split query for a point-sharded index.  Stage 1 counts the
 * local shard and leaves per-query score histograms hist_d[nq*(Ns+1)] (int64)
 * to be all-reduced across ranks; stage 2 applies Alg. 5 on the global
 * histograms and reranks locally: topk_d2_d[nq*k] (f64, +inf padded),
 * topk_ids_d[nq*k] (global ids, -1 padded), cand_num_d (global), last_coll_d. */
int taco_query_count_device(taco_index* idx, const float* Q_d, int64_t nq, double alpha,
                            int64_t* hist_d, void* stream);
int taco_query_finish_device(taco_index* idx, int64_t nq, const int64_t* ghist_d, double beta,
                             int32_t k, double* topk_d2_d, int64_t* topk_ids_d,
                             int64_t* cand_num_d, int32_t* last_coll_d, void* stream);
/* Split traversal: stage 1 as three calls so ranks can divide the replicated
 * per-query traversal.  taco_query_front_device computes rows [q_lo, q_hi)
 * of a tile of nq queries (Q_d; rows >= nq is the all-gather's padded row
 * count) into the index's tile
 * buffers; *need > 0 reports a traversal longer than pop_cap (all ranks then
 * repeat with pop_cap = K'^2).  taco_query_pop_buffers exposes those buffers
 * (pops u16 [rows][Ns][pop_cap], npop i32 [rows][Ns], ret i64 [rows][Ns]) for
 * an in-place all-gather; taco_query_count_popped_device then counts the
 * local shard for all nq queries.  Replaces the count half of
 * engine.py:201-220 (popped cells shared, ids counted per shard). */
int taco_query_front_device(taco_index* idx, const float* Q_d, int64_t nq, int64_t q_lo, int64_t q_hi,
                            int64_t rows, double alpha, int32_t pop_cap, int64_t* need, void* stream);
/* taco_query_front_async: the same walk without a host round trip; the
 * slice's longest walk (pops) is copied to need_d[0] (device int64) on the
 * stream, so a caller all-reduces it and checks every tile of a batch with one
 * sync (the batch is re-run with a raised cap in the rare overflow case). */
int taco_query_front_async(taco_index* idx, const float* Q_d, int64_t nq, int64_t q_lo, int64_t q_hi,
                           int64_t rows, double alpha, int32_t pop_cap, int64_t* need_d, void* stream);
int taco_query_pop_buffers(taco_index* idx, void** pops, void** npop, void** ret, int32_t* pop_cap);
int taco_query_count_popped_device(taco_index* idx, int64_t nq, int64_t* hist_d, void* stream);
/* Largest nq accepted by the split count/finish calls for this index. */
int taco_query_tile_size(taco_index* idx);
/* Merge R sorted per-rank top-k lists [R][nq][k] on (d2, id), write ids/dists. */
int taco_topk_merge_device(int32_t ranks, int64_t nq, int32_t k, const double* d2_d,
                           const int64_t* ids_d, int32_t* ids_out_d, float* dists_out_d,
                           void* stream);

/* Test hook: 1 forces every k-means++ draw through the exact numpy replay. */
int taco_debug_force_replay(int on);

/* --------------------------------------------------------- ground truth */
/* Exact k-NN (dataio.compute_ground_truth, dataio.py:142-172): fp64
 * d2 = max((xsq - 2 q.x) + qsq, 0) with numpy's einsum / dgemm orders, the k
 * smallest (d2, id), dists = f32(sqrt(d2)).  k <= 1024, d <= 25600.
 * ids_h int32 [nq][k], dists_h f32 [nq][k], host buffers. */
int taco_ground_truth(int device, const float* X_h, int64_t n, int32_t d, const float* Q_h, int64_t nq,
                      int32_t k, int32_t* ids_h, float* dists_h);
/* Same over the index's resident base vectors (whole dataset, not a shard). */
int taco_ground_truth_index(taco_index* idx, const float* Q_h, int64_t nq, int32_t k, int32_t* ids_h,
                            float* dists_h);

/* SC-Linear exact collision counting (engine.sc_linear_scores, engine.py:290-321):
 * per subspace, the ceil(alpha n) nearest points by (einsum fp64 d2, id) collide.
 * T_h row-major n x (n_sub*s) f32, qt_h the transformed query (n_sub*s f32),
 * scores_h uint8[n]. */
int taco_sc_linear_scores(int device, const float* T_h, int64_t n, int32_t n_sub, int32_t s, const float* qt_h,
                          double alpha, uint8_t* scores_h);
/* Same over the index's resident transformed matrix. */
int taco_sc_linear_scores_index(taco_index* idx, const float* qt_h, double alpha, uint8_t* scores_h);

/* --------------------------------------------------------------- profiling */
/* Per-kernel CUDA-event timing of the query path on its launching stream.
 * stats_out[7]: sum retrieved ids, sum candidates, sum pops, queries, tiles,
 * score-table bytes, max pops of one (query, subspace). */
int taco_profile_enable(int on);
int taco_profile_read(double* ms_out, int64_t* cnt_out, int64_t* stats_out, int reset);
const char* taco_profile_name(int i);
int taco_profile_kernels(void);
/* The index's own CUDA stream (cudaStream_t as void*). */
void* taco_index_stream(taco_index* idx);

/* -------------------------------------------------- fine-grained taps/API */
/* engine.count_collisions for one query (engine.py:188-220): scores_h[n] u8. */
int taco_count_scores(taco_index* idx, const float* q_h, double alpha, uint8_t* scores_h);
/* imi.sorted_centroid_distances + scalable_dynamic_activation trace for one
 * (query, subspace) (imi.py:88-166): pops_h[cap] cell ids (l1*K'+l2),
 * keys_h[cap] heap keys; returns counts through npop_h / retrieved_h. */
int taco_activation_trace(taco_index* idx, const float* q_h, int32_t j, double alpha,
                          int32_t cap, int32_t* pops_h, double* keys_h, int32_t* npop_h,
                          int64_t* retrieved_h);
/* engine.select_candidates on a host score table (engine.py:223-253). */
int taco_select_candidates(int device, const uint8_t* scores_h, int64_t n, int32_t n_sub,
                           double beta, int64_t* ids_h, int64_t* cand_num_h,
                           int32_t* last_coll_h);
/* engine.rerank on host data / ids (engine.py:256-279). */
int taco_rerank(int device, const float* X_h, int64_t n, int32_t d, const float* q_h,
                const int64_t* ids_h, int64_t m, int32_t k, int32_t* ids_out_h,
                float* dists_out_h, double* d2_out_h);
/* spectral.fit_covariance on host data (standalone). */
int taco_covariance(int device, const float* X_h, int64_t n, int32_t d, double* mean_h,
                    double* gram_h, int64_t* bad_row);
/* imi.sorted_centroid_distances (imi.py:88-106): sorted fp64 distances and the
 * stable argsort of both codebooks against one subspace query. */
int taco_centroid_order(int device, const float* c1_h, const float* c2_h, int32_t kp, int32_t m1,
                        int32_t m2, const float* q_h, double* d1s_h, int32_t* l1s_h,
                        double* d2s_h, int32_t* l2s_h);
/* imi.scalable_dynamic_activation (imi.py:130-166) on sorted inputs and a dense
 * K'^2 size table: pops_h / keys_h [K'^2], *npop_h, *retrieved_h. */
int taco_traverse(int device, int32_t kp, const double* d1s_h, const int32_t* l1s_h,
                  const double* d2s_h, const int32_t* l2s_h, const int64_t* sizes_h,
                  int64_t target, int32_t* pops_h, double* keys_h, int32_t* npop_h,
                  int64_t* retrieved_h);
/* spectral.transform_points for arbitrary points (spectral.py:301-316). */
int taco_transform_points(int device, const float* mean_h, const float* matrix_h, int32_t d,
                          int32_t D, const float* P_h, int64_t np_, float* out_h);
/* clustering.kmeans on one matrix (clustering.py:57-115), same RNG contract as
 * taco_kmeans_all.  history_h[max_iter]. */
int taco_kmeans(int device, const float* X_h, int64_t n, int32_t m, int32_t k, int32_t max_iter,
                int64_t first, const double* uniforms_h, const int64_t* forced_h,
                float* centroids_h, int32_t* labels_h, double* history_h, int32_t* n_iter_h,
                int32_t* degenerate_h);

#ifdef __cplusplus
}
#endif
#endif /* TACO_B200_H */
