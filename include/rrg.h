/*
 * rrg.h -- C ABI of the B200-native LoRANN query engine (librrg.so).
 *
 * The reference (`rrann`, pure Python/NumPy) has no native FFI; its drop-in
 * boundary is the Python function pair `query_batch` / `query`
 * (pkg/src/rrann/index.py:286-340, re-exported in __init__.py:11-21) plus the
 * index file loader `RrrIndex.load` -> `deserialize` (index.py:138-141,443-507).
 * SPEC.md:522-526 names the intended foreign binding
 * `bound_query_batch(BoundIndex, array2d, k, w, t) -> (ids, scores)` with
 * `bound_load`; the entry points below are exactly that binding, in C:
 *
 *   rrg_index_open        <- RrrIndex.load / deserialize        (index.py:138-141, 443-507)
 *   rrg_index_create      <- RrrIndex already in memory (the models of index.py:110-118)
 *   rrg_search            <- query_batch, device buffers        (index.py:338-340, 286-335)
 *   rrg_search_host       <- bound_query_batch, host buffers
 *   rrg_last_error        <- exception message text             (errors.py:8-39)
 *
 * Status codes mirror the error-category -> CLI exit-code map (cli.py:20,198-200):
 *   0 ok, 2 usage (ShapeError / ParameterError), 3 data (DataError / FormatError),
 *   4 internal (RrannError / CUDA failure).  rrg_last_error_kind() names the
 *   exception class so a binding can raise the reference's own type.
 *
 * All pointers are plain host or device pointers; no framework types cross
 * this boundary.  Index handles are immutable after creation and may be
 * searched concurrently from several host threads, each with its own stream
 * and workspace (index.py docstring "concurrent queries").
 */
#ifndef RRG_H_
#define RRG_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define RRG_OK 0
#define RRG_E_USAGE 2
#define RRG_E_DATA 3
#define RRG_E_INTERNAL 4

/* metric codes of the file header (index.py:48) */
#define RRG_METRIC_EUCLIDEAN 0
#define RRG_METRIC_IP 1
#define RRG_METRIC_COSINE 2

/* header flags (index.py:43-46) */
#define RRG_FLAG_QUANTIZED (1u << 0)
#define RRG_FLAG_CORPUS (1u << 1)
#define RRG_FLAG_BALANCED (1u << 2)
#define RRG_FLAG_EXACT_IVF (1u << 3)

typedef struct RrgIndex RrgIndex;

/* Host-side description of an in-memory index (the fields of RrrIndex and its
 * ClusterModels, index.py:110-118 / rrr.py:77-94).  Per-cluster payloads are
 * concatenated in cluster order.  Quantized factors are given exactly as the
 * file stores them (index.py:346-353): head_row[cols], col_scales[cols] and a
 * rows x cols int8 block whose row 0 is the zero pad row. */
typedef struct {
  int32_t metric;           /* RRG_METRIC_* */
  int32_t dim;              /* d */
  int32_t reduced_dim;      /* s (== d when reduction is off) */
  int32_t rank;             /* r */
  int32_t n_clusters;       /* L */
  int64_t n_points;         /* m */
  uint32_t flags;           /* RRG_FLAG_* */
  const float* projection;  /* d x s row-major */
  const float* centroids;   /* L x s row-major */
  const uint32_t* cluster_sizes;  /* L */
  const int64_t* point_ids;       /* m, cluster order */
  /* factor A of every cluster: s x cols_l (cols_l = m_l if exact else r) */
  const float* a_head;      /* sum cols_l */
  const float* a_scale;     /* sum cols_l */
  const int8_t* a_values;   /* sum s*cols_l */
  /* factor B of every non-exact cluster: r x m_l */
  const float* b_head;      /* sum m_l over non-exact clusters */
  const float* b_scale;
  const int8_t* b_values;   /* sum r*m_l */
  const float* norms;       /* m, cluster order; NULL unless euclidean */
  const float* corpus;      /* m x d in ORIGINAL id order; NULL if no corpus (host or device memory) */
  /* unquantized factors (RRG_FLAG_QUANTIZED clear, RrrConfig.quantize=False,
   * rrr.py:97-100): f32 blocks with the same shapes and concatenation as
   * a_values / b_values (no pad row, no head/scale); ignored when quantized */
  const float* a_values_f32; /* sum s*cols_l */
  const float* b_values_f32; /* sum r*m_l (non-NULL even if every cluster is exact) */
} RrgIndexDesc;

typedef struct {
  int32_t metric, dim, reduced_dim, rank, n_clusters;
  int64_t n_points;
  uint32_t flags;
  int32_t n_exact_clusters;
  int32_t max_cluster_size;
  int32_t device;
  uint64_t device_bytes;    /* HBM held by the index */
} RrgIndexInfo;

/* Parse an RRRANN01 file (streaming, CRC-checked, same FormatError texts as
 * deserialize) and upload it to `device`.  Returns RRG_E_DATA on a malformed
 * file. */
int rrg_index_open(const char* path, int device, RrgIndex** out);

/* Same, restricted to clusters [cluster_begin, cluster_end) -- the shard a
 * rank owns in cluster-sharded multi-GPU search; projection and centroids are
 * replicated. */
int rrg_index_open_shard(const char* path, int device, int32_t cluster_begin,
                         int32_t cluster_end, RrgIndex** out);

/* Build from host arrays (see RrgIndexDesc). */
int rrg_index_create(const RrgIndexDesc* desc, int device, RrgIndex** out);
/* Shard of an in-memory index: clusters [cluster_begin, cluster_end) keep their
 * factors and corpus rows, every cluster keeps its centroid (routing is replicated);
 * same layout as rrg_index_open_shard. */
int rrg_index_create_shard(const RrgIndexDesc* desc, int device, int32_t cluster_begin,
                           int32_t cluster_end, RrgIndex** out);

void rrg_index_destroy(RrgIndex* index);
/* Search-variant switches (RRG_GEMM, RRG_RERANK, RRG_SCREEN, ... -- A/B measurement
 * and test coverage of every kernel variant) are read from the environment once,
 * when the index is created; this re-reads them for an existing index. */
int rrg_index_reload_options(RrgIndex* index);
int rrg_index_info(const RrgIndex* index, RrgIndexInfo* out);
/* Points held per cluster (n_clusters entries; 0 for clusters outside a shard). */
int rrg_index_cluster_sizes(const RrgIndex* index, uint32_t* out);

/* Workspace bytes rrg_search needs for a batch of nq queries. */
size_t rrg_search_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t k,
                                  int32_t w, int32_t t, int32_t rerank);

/* Batched search, all buffers on the index's device, asynchronous on `stream`
 * (a cudaStream_t; NULL = legacy default stream).
 *   queries : nq x dim f32, finite (validated by the caller, index.py:339)
 *   ids     : nq x k int64, best first, -1 past count[i]
 *   scores  : nq x k f32 (squared distance for euclidean, inner product for
 *             ip/cosine, as QueryResult.scores, index.py:318-329), NaN past count[i]
 *   count   : nq int32 = len(QueryResult.ids); truncated = count < k
 * Parameter checks follow QueryParams.validate (index.py:92-100) and
 * index.py:290-295. */
int rrg_search(RrgIndex* index, const float* queries, int64_t nq, int32_t dim,
               int32_t k, int32_t w, int32_t t, int32_t rerank, int64_t* ids,
               float* scores, int32_t* count, void* workspace,
               size_t workspace_bytes, void* stream);

/* Host-buffer convenience form (the SPEC.md:522-526 binding): copies queries
 * in, searches, copies results out, synchronous.  Non-finite queries raise
 * DataError (index.py:144-150) ahead of parameter errors: the finiteness test
 * runs on the GPU inside the query-prep pass, and the batch is scanned on the
 * host only when the parameters are invalid, so the DataError still wins. */
int rrg_search_host(RrgIndex* index, const float* queries, int64_t nq,
                    int32_t dim, int32_t k, int32_t w, int32_t t,
                    int32_t rerank, int64_t* ids, float* scores,
                    int32_t* count);

/* A stream of `nbatch` host batches (queries[b]: nq[b] x dim; outputs as
 * rrg_search_host), software-pipelined over two device buffer sets so the
 * H2D copy of batch b+1 and the D2H copy of batch b-1 overlap the search of
 * batch b -- the serving loop over consecutive query_batch calls.  Results are
 * identical to nbatch rrg_search_host calls; pinned host buffers give full
 * copy bandwidth. */
int rrg_search_host_many(RrgIndex* index, int32_t nbatch, const float* const* queries,
                         const int64_t* nq, int32_t dim, int32_t k, int32_t w, int32_t t,
                         int32_t rerank, int64_t* const* ids, float* const* scores,
                         int32_t* const* count);

/* Stage entry points used by the stage-parity tests (device buffers). */
int rrg_stage_project(RrgIndex* index, const float* queries, int64_t nq,
                      float* xp, int8_t* qcodes, float* qscale, float* qhead,
                      void* stream);
int rrg_stage_route(RrgIndex* index, const float* xp, int64_t nq, int32_t w,
                    int32_t* selected, void* workspace, size_t workspace_bytes,
                    void* stream);

/* K4 of the search path (score_cluster, rrr.py:181-203 / quantize.py:109-156) for
 * caller-chosen probes sel [nq][w] (device int32), run by the production
 * cluster-major scoring kernel with its stage outputs switched on, so the int32
 * products and f32 scores can be compared bit for bit with the reference:
 *   raw1     [nq][w][rank] int32: stage-A products x_i8 . A_i8 of RRR clusters
 *   cand_off [nq + 1] int32: start of each query's candidates (probes in sel order)
 *   raw2     [cand_off[nq]] int32: last-stage product per point (stage B, or stage A
 *            of an exact model)
 *   scores   [cand_off[nq]] f32: score_cluster's output per point
 * Synchronous on `stream`. */
size_t rrg_stage_score_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t w);
int rrg_stage_score(RrgIndex* index, const float* queries, int64_t nq, int32_t w,
                    const int32_t* sel, int32_t* raw1, int32_t* raw2, float* scores,
                    int32_t* cand_off, void* workspace, size_t workspace_bytes, void* stream);

/* ---- cluster-sharded search; one index shard per rank
 * (rrg_index_open_shard), queries replicated.  Exact reference semantics need
 * two exchanges because index.py:314-322 re-ranks the GLOBAL top-t:
 *   1. rrg_shard_phase1 : local top-t (key, corpus id) over the shard's clusters
 *      -> all-gather -> rrg_merge_candidates : global top-t (identical on all ranks)
 *   2. rrg_shard_phase2 : re-rank the global candidates this shard holds, local top-k
 *      -> all-gather -> rrg_merge_results : final top-k == the unsharded result.
 * Merge inputs use the all-gather layout [G][nq][cap] with counts [G][nq]. */
size_t rrg_shard_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t k, int32_t w,
                                 int32_t t);

/* Data-parallel front stages: the per-query outputs of projection (index.py:298),
 * query quantization (quantize.py:61-77) and routing (cluster.py:254-264), row-major
 * over nq queries (device buffers).  Each rank computes a slice of the batch with
 * rrg_search_front; the slices are all-gathered and every rank continues from them
 * (rrg_search_from_front / rrg_shard_phase1_from_front), so projection and routing
 * are not replicated. */
typedef struct {
  float* xp;       /* nq x reduced_dim f32: f32(f64(x) @ f64(W)) */
  int8_t* qcodes;  /* nq x round_up(reduced_dim, 16) int8: mixed-precision codes (col 0 = 0) */
  float* qscale;   /* nq */
  float* qhead;    /* nq */
  double* pp;      /* nq: xp . xp (f64, NumPy pairwise order) */
  float* xx;       /* nq: x . x (f32) */
  int32_t* sel;    /* nq x w: routed clusters */
  int32_t* prim;   /* nq: the nearest routed cluster */
} RrgFront;
size_t rrg_front_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t w);
int rrg_search_front(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t w,
                     const RrgFront* out, void* workspace, size_t workspace_bytes, void* stream);
/* rrg_search with the front stages taken from `front` (rows of all nq queries).  On a
 * shard index (rrg_index_open_shard) a query whose probes are all held elsewhere
 * returns count 0; with w = 1 every query has exactly one owner, so each rank's
 * results are final for the queries it owns and one all-gather + rrg_merge_results
 * completes the batch -- no candidate exchange. */
int rrg_search_from_front(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                          int32_t w, int32_t t, int32_t rerank, const RrgFront* front, int64_t* ids,
                          float* scores, int32_t* count, void* workspace, size_t workspace_bytes,
                          void* stream);
int rrg_shard_phase1_from_front(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                                int32_t w, int32_t t, const RrgFront* front, uint32_t* keys, uint32_t* ids,
                                int32_t* count, void* workspace, size_t workspace_bytes, void* stream);
int rrg_shard_phase1(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                     int32_t w, int32_t t, uint32_t* keys, uint32_t* ids, int32_t* count,
                     void* workspace, size_t workspace_bytes, void* stream);
int rrg_merge_candidates(int64_t nq, int32_t G, int32_t cap, const uint32_t* keys,
                         const uint32_t* ids, const int32_t* counts, int32_t take,
                         uint32_t* out_keys, uint32_t* out_ids, int32_t* out_count, void* stream);
/* Sparse phase-1 exchange: a rank's [nq][cap] lists packed back to back
 * (offsets[nq + 1], offsets[nq] = total) before the all-gather, and the G gathered
 * packed lists (stride elements each) unpacked into the [G][nq][cap] layout
 * rrg_merge_candidates reads.  With w = 1 a query's candidates sit on one rank,
 * so the exchange shrinks about G-fold. */
int rrg_pack_candidates(int64_t nq, int32_t cap, const uint32_t* keys, const uint32_t* ids,
                        const int32_t* counts, uint32_t* packed_keys, uint32_t* packed_ids,
                        int32_t* offsets, void* stream);
int rrg_unpack_candidates(int64_t nq, int32_t G, int64_t stride, int32_t cap,
                          const uint32_t* packed_keys, const uint32_t* packed_ids,
                          const int32_t* offsets, uint32_t* keys, uint32_t* ids, int32_t* counts,
                          void* stream);
int rrg_shard_phase2(RrgIndex* index, const float* queries, int64_t nq, int32_t dim,
                     const uint32_t* cand_ids, const int32_t* cand_count, int32_t cap, int32_t k,
                     int64_t* ids, float* scores, int32_t* count, void* workspace,
                     size_t workspace_bytes, void* stream);
int rrg_merge_results(int64_t nq, int32_t G, int32_t k, int32_t metric, const float* scores,
                      const int64_t* ids, const int32_t* counts, float* out_scores,
                      int64_t* out_ids, int32_t* out_count, void* stream);

/* Exact k-NN ground truth, replacing rrann.bench.brute_force_knn
 * (pkg/src/rrann/bench.py:85-124): f64 distances (euclidean
 * (q.q - 2 q.c) + c.c, ip -(q.c), cosine -(q.c/||c||)), ids ordered by
 * (distance, id) like the stable argsort.  corpus m x dim and queries nq x dim
 * f32 on the current device; ids nq x k int64.  Synchronous on `stream`.
 * ParameterError when k is outside [1, m] (or > 2048). */
int rrg_ground_truth(const float* corpus, int64_t m, int32_t dim, const float* queries,
                     int64_t nq, int32_t k, int32_t metric, int64_t* ids, void* stream);

/* Number of CUDA kernel launches issued by the most recent rrg_search* call
 * on this thread (evidence for the bench's gpu_launches). */
int64_t rrg_last_launch_count(void);

/* Per-stage device timing (CUDA events recorded on the search stream around
 * every launch) for the calls made on this thread while enabled.  Stages:
 * 0 project, 1 prep/quantize, 2 route distances, 3 route select,
 * 4 top-t selection (query-major mode: scoring + top-t), 5 rerank+top-k,
 * 6 query bucketing, 7 cluster-major scoring (pair bucketing + scoring),
 * 8 ground truth (rrg_ground_truth launches), 9 re-rank screen (bounds + thresholds).
 * rrg_stage_times synchronizes the recorded events, writes the accumulated
 * milliseconds and launch counts per stage (arrays of RRG_N_STAGES) and resets
 * the accumulators. */
#define RRG_N_STAGES 10
void rrg_set_stage_timing(int enabled);
int rrg_stage_times(double* ms, int64_t* launches);

/* Critical-path spans recorded while stage timing is on, as events on the launching
 * stream only (side-stream work that overlaps them is not added in):
 *   RRG_PATH_RERANK  from the re-rank screen's launch (or the exact pass when there is
 *                    no screen) to the end of the final top-k;
 *   RRG_PATH_SEARCH  from a search's first launch to its last.
 * rrg_path_times synchronizes, writes the accumulated milliseconds and span counts
 * (arrays of RRG_N_PATHS) and resets them. */
#define RRG_PATH_RERANK 0
#define RRG_PATH_SEARCH 1
#define RRG_N_PATHS 2
int rrg_path_times(double* ms, int64_t* count);

/* Re-rank work counters accumulated by the searches of this thread while stage timing
 * is enabled (the roofline's algorithmic bytes come from these): returns and resets
 *   0 candidates entering the screen (sum over queries of the top-t size)
 *   1 candidates surviving the screen (re-ranked exactly)
 *   2 rows streamed by the screen (fp16 residual rows, 128-row blocks)
 *   3 corpus rows fetched by the cluster-major exact re-rank (f32 rows)
 *   4 distinct corpus rows the exact pass needs (union over each cluster's queries) */
#define RRG_N_COUNTERS 8
int rrg_search_counters(int64_t* out);

const char* rrg_last_error(void);
const char* rrg_last_error_kind(void); /* "ShapeError", "ParameterError", ... */
const char* rrg_version(void);

#ifdef __cplusplus
}
#endif
#endif /* RRG_H_ */
