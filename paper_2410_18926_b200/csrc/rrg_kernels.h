// rrg_kernels.h -- host-side launchers of the query-path kernels.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "rrg_common.cuh"

namespace rrg {

constexpr int EPI_PROJ = 0;
constexpr int EPI_L2 = 1;
constexpr int EPI_NEGIP = 2;
constexpr int EPI_GT_L2 = 3;   // (qq - 2 q.c) + cc, no clip (bench.py:110)
constexpr int EPI_GT_COS = 4;  // -(q.c / ||c||)           (bench.py:100-103,112)
constexpr int EPI_L2_ARGMIN = 5;     // routing w = 1: per-row nearest column per tile
constexpr int EPI_NEGIP_ARGMIN = 6;
constexpr int EPI_L2_TOP4 = 7;       // routing 1 < w <= 4: per-row 4 nearest columns per tile
constexpr int EPI_L2_TOP8 = 8;       //                w <= 8
constexpr int kMaxSmemPerCta = 227 * 1024;  // B200 opt-in limit per CTA
// cluster count bound: routing (w > 1) keeps 12 B per cluster in one CTA's shared memory
constexpr int kMaxClusters = (kMaxSmemPerCta - 4096) / 12;

struct ScoreArgsHost {
  DevIndexView ix;
  const int8_t* qcodes;
  const float* qscale;
  const float* qhead;
  const float* xx;
  const int* sel;
  int w, take_cap, rerank, k, smem_cap;
  uint32_t* gkeys;
  int* gpos;
  int64_t gcap;
  int* cand_pos;
  int* cand_n;
  int64_t* out_ids;
  float* out_scores;
  int* out_count;
  int q0;
  const int* order = nullptr;
  uint32_t* sel_keys = nullptr;
  uint32_t* sel_ids = nullptr;
  int* sel_count = nullptr;
};

struct RerankArgsHost {
  DevIndexView ix;
  const float* queries;
  const int* cand_pos;
  const int* cand_n;
  int take_cap, k;
  int64_t* out_ids;
  float* out_scores;
  int* out_count;
  int q0;
  const int* order = nullptr;
};

// small batches (a few queries): warp-per-output f64 GEMV (Wt = W^T, s x d)
void launch_project_small(const float* x, const float* Wt, int nq, int d, int s, float* xp,
                          cudaStream_t st);
void launch_route_dist_small(const float* xp, const float* cent, int nq, int L, int s, int metric,
                             const double* pp, const double* cnorm, double* diss, cudaStream_t st);
void launch_project(const float* x, const float* W, int nq, int d, int s, float* xp, int bk,
                    cudaStream_t st);
void launch_prep(const float* xp, const float* x, int nq, int s, int s_pad, int d, int8_t* qcodes,
                 float* qscale, float* qhead, double* pp, float* xx, cudaStream_t st,
                 int* nonfinite = nullptr);
void launch_route_dist(const float* xp, const float* cent, int nq, int L, int s, int metric,
                       const double* pp, const double* cnorm, double* diss, int bk, cudaStream_t st);
size_t route_select_smem(int L);
// w = 1 routing fused into the DMMA GEMM: per (row, 64-column tile) minima, then a
// warp argmin per query (part_v / part_i: nq x route_nearest_tiles(L))
int route_nearest_tiles(int L);
void launch_route_nearest_fused(const float* xp, const float* cent, int nq, int L, int s, int metric,
                                const double* pp, const double* cnorm, double* part_v, int* part_i,
                                cudaStream_t st);
void launch_route_topw_fused(const float* xp, const float* cent, int nq, int L, int s, int w, const double* pp,
                             const double* cnorm, double* part_v, int* part_i, cudaStream_t st);
void launch_route_topw_reduce(const double* part_v, const int* part_i, int nq, int L, int w, int* sel,
                              int* primary, cudaStream_t st);
void launch_route_nearest_reduce(const double* part_v, const int* part_i, int nq, int L, int* sel,
                                 int* primary, cudaStream_t st);
void launch_route_select(const double* diss, int nq, int L, int w, int* sel, int* primary,
                         cudaStream_t st);
void launch_bucket(const int* primary, int nq, int L, int* order, cudaStream_t st);
size_t score_select_smem(int smem_cap, int take_cap, int k);
void launch_score_select(const ScoreArgsHost& h, int nq, cudaStream_t st);
size_t rerank_smem(int d_stride, int take_cap, int k, bool tree);
bool rerank_uses_tree(const DevIndexView& ix);
void launch_rerank(const RerankArgsHost& h, int nq, cudaStream_t st);
// Cluster-major scoring (rrg_cluster_score.cu)
struct ClusterScoringHost {
  DevIndexView ix;
  const float* xp;  // [nq][s] projected queries (unquantized index)
  const int8_t* qcodes;
  const float* qscale;
  const float* qhead;
  const int* sel;
  int w;
  int* qoff;      // [nq][w+1]
  int* ncand;     // [nq]
  int* pair_off;  // [L+1]
  int* item_off;  // [L+1]
  int* pairs;     // [nq*w]
  int* kbase;     // [nq+1]
  uint32_t* keys; // [sum N]
  int* work_counter;
  int* dbg_raw1 = nullptr;     // rrg_stage_score only (see ClusterScoreArgs)
  int* dbg_raw2 = nullptr;
  float* dbg_score = nullptr;
};
// candidate offsets + pair bucketing (what the screen's side stream needs), then scoring
void launch_cluster_prep(const ClusterScoringHost& h, int nq, cudaStream_t st);
void launch_cluster_scoring(const ClusterScoringHost& h, int nq, cudaStream_t st, bool prep = true);

struct SelectTopTHost {
  DevIndexView ix;
  const int* sel;
  int w;
  const int* qoff;
  const int* kbase;
  const uint32_t* keys;
  int take_cap, rerank, k;
  const float* xx;
  int* cand_pos;
  int* cand_n;
  int64_t* out_ids;
  float* out_scores;
  int* out_count;
  int q0;
  const int* order;
  uint32_t* sel_keys;
  uint32_t* sel_ids;
  int* sel_count;
  int kcap;
  int* cand_idx = nullptr;    // cluster-major re-rank outputs
  uint32_t* marks = nullptr;
};
size_t select_topt_smem(int w, int take_cap, int k, int kcap);
void launch_select_topt(const SelectTopTHost& h, int nq, cudaStream_t st);

// Cluster-major re-rank (rrg_cluster_score.cu)
constexpr int kRrQ = 16;  // queries of one work item (x staged at once; the screen's MMA N)
// item_off[l] = ceil(pairs_l / kRrQ) * ceil(m_l / rows), exclusive scan, item_off[L] = total
void launch_rr_items(const int* pair_off, const int* cl_pos, int L, int rows, int* item_off,
                     cudaStream_t st);
// queries re-laid out like the corpus rows (interleaved for the pairwise plan), so the
// cluster re-rank stages a work item's x with plain vector loads
void launch_interleave_queries(const DevIndexView& ix, const float* queries, int nq, float* xint,
                               cudaStream_t st);
struct ClusterRerankHost {
  DevIndexView ix;
  const float* queries;
  const float* xint = nullptr;  // [nq][d_stride] interleaved queries
  const int* cand_idx = nullptr;  // screened: the survivors per query (membership source)
  const int* cand_n = nullptr;
  int take_cap = 0;
  int w;
  const int* qoff;
  const int* pair_off;
  int* rr_item_off;  // [L+1] scratch (filled by the launcher)
  const int* pairs;
  const int* kbase;
  const uint32_t* marks;
  uint32_t* diss;
  int* work_counter;
  bool skip;  // pass over row pairs no query of a work item selected (sparse selections)
  bool compact = false;  // list the selected rows first (after the screen: ~k of t survive)
  int64_t* counters = nullptr;  // rrg_search_counters[3]: rows fetched
  int mwords;
  int nq;  // queries of the chunk (work-item sizing)
};
bool cluster_rerank_ok(const DevIndexView& ix, int64_t max_cluster);
size_t cluster_rerank_smem(const DevIndexView& ix, int mwords);
void launch_cluster_rerank(const ClusterRerankHost& h, cudaStream_t st);

// Re-rank screen (rrg_screen.cu): tensor-core bounds of every (query, candidate row)
// of the cluster-major work items, then per query the k-th smallest upper bound T and
// the removal of the candidates whose lower bound exceeds it (see the file header).
int screen_max_dim();
size_t screen_smem(int kc);
size_t screen_group_bytes(int kc);
void launch_screen_build(const DevIndexView& v, float* mu, uint16_t* plane, size_t plane_bytes,
                         double* rr, float4* meta, cudaStream_t st);
struct ScreenHost {
  DevIndexView ix;
  const float* queries;  // chunk-local [nq][d]
  int w;
  const int* qoff;
  const int* pair_off;
  const int* pairs;
  const int* kbase;
  uint32_t* marks;       // membership bits of the top-t (cleared for non-survivors)
  int* item_off;         // [L+1] scratch
  int* grp_off;          // [L+1] scratch
  unsigned char* grec;   // n_groups_max x screen_group_bytes(scr_kc) scratch
  int n_groups_max;
  float* ub;             // per candidate bounds (key-array layout)
  float* lb;
  int* cand_idx;         // [nq][take_cap] top-t candidate indices -> the survivors
  int* cand_n;
  int take_cap, k;
  uint32_t* diss;        // key array re-used for distances
  int64_t* counters;     // rrg_search_counters (nullptr unless enabled)
};
struct ThreshArgs {
  const int* kbase;
  int* cand_idx;  // compacted in place to the survivors
  int* cand_n;
  int take_cap, k;
  const float* ub;
  const float* lb;
  uint32_t* marks;
  uint32_t* diss;
  int64_t* counters;
};
void launch_screen_prep(const ScreenHost& h, int nq, cudaStream_t st);  // items + group records
void launch_screen(const ScreenHost& h, int nq, cudaStream_t st);       // the bounds (k_rr_screen)
void launch_thresh(const ScreenHost& h, int nq, cudaStream_t st);       // T, survivors
// counter: distinct rows of every cluster marked by any of its queries
void launch_count_rows(const DevIndexView& ix, const int* pair_off, const int* pairs, const int* kbase,
                       const int* qoff, int w, const uint32_t* marks, const int* cand_idx, const int* cand_n,
                       int take_cap, int mwords, int64_t* out, cudaStream_t st);

// Routing screen (rrg_route_screen.cu): fp16 tensor-core bounds of every
// (query, centroid) d2, the centroids that can be among the w nearest, f64 recheck.
constexpr int kRtCap = 64;    // survivors rechecked per query (more: every centroid is rechecked)
constexpr int kRtMaxGroups = 32;  // centroid ranges (CTAs) per query block
size_t route_list_bytes(int nq, int L);  // scratch of the per-thread candidate lists
size_t route_cnt_bytes(int nq, int L);
constexpr int kRtMaxW = 8;    // w handled by the screen (larger w: the f64 GEMM path)
constexpr int kRtMaxKc = 24;  // s <= 384
int route_screen_max_dim();
size_t route_tile_bytes(int rows, int kc);
void launch_f16_tiles(const float* src, int rows, int K, int ld, int kc, uint16_t* tiles, float4* stats,
                      cudaStream_t st);
struct RouteScreenHost {
  DevIndexView ix;
  const float* xp;   // [nq][s] projected queries
  const double* pp;  // [nq] x.x (NumPy pairwise f64)
  int w;
  uint16_t* qt;      // route_tile_bytes(nq, rt_kc) scratch
  float4* qs;        // [nq padded to 128] scratch
  uint32_t* T;       // [nq] scratch
  int* cnt;          // route_cnt_bytes scratch
  int2* list;        // route_list_bytes scratch
  int* sel;          // [nq][w] out
  int* primary;      // [nq] out
};
void launch_route_screen(const RouteScreenHost& h, int nq, cudaStream_t st);

struct TopkFinalHost {
  DevIndexView ix;
  const int* sel;
  int w;
  const int* qoff;
  const int* kbase;
  const uint32_t* diss;
  const int* cand_idx;
  const int* cand_n;
  int take_cap, k;
  int64_t* out_ids;
  float* out_scores;
  int* out_count;
  int q0;
  const int* order;
};
size_t topk_final_smem(int w, int take_cap, int k);
void launch_topk_final(const TopkFinalHost& h, int nq, cudaStream_t st);

// Sharded search: merge G per-shard lists per query, laid out
// [G][nq][cap] (the all-gather layout) with counts [G][nq].
//   mode 0: (key u32, id u32) candidates -> global top-`take` by (key, id), sorted
//   mode 1: (score f32, id i64) results  -> global top-`take` by (diss, id), sorted,
//           diss = score (euclidean) | -score (ip/cosine)
void launch_merge(int mode, int metric, int nq, int G, int cap, const void* in_keys,
                  const void* in_ids, const int* in_counts, int take, void* out_keys,
                  void* out_ids, int* out_count, cudaStream_t st);
// ids -> positions held by this shard (others dropped): cand_pos [nq][cap], cand_n [nq]
void launch_pack_candidates(int nq, int cap, const uint32_t* keys, const uint32_t* ids,
                            const int* counts, uint32_t* pk, uint32_t* pi, int* off, cudaStream_t st);
void launch_unpack_candidates(int nq, int G, int64_t stride, int cap, const uint32_t* pk,
                              const uint32_t* pi, const int* off, uint32_t* keys, uint32_t* ids,
                              int* counts, cudaStream_t st);
void launch_ids_to_pos(const DevIndexView& ix, int nq, int cap, const uint32_t* ids,
                       const int* counts, int* cand_pos, int* cand_n, cudaStream_t st);

void launch_scatter_rows(const float* src, int64_t nrows, int d, int d_stride,
                         const int* pos_of_id, int64_t i0, const int* perm, float* dst,
                         cudaStream_t st);


// ---------------------------------------------------- ground truth (rrg_ground_truth.cu)
struct GtSelectHost {
  const double* diss;
  int64_t ld;
  int n;
  int64_t id0;
  const uint64_t* run_key;
  const int64_t* run_id;
  const int* run_n;
  uint64_t* out_key;
  int64_t* out_id;
  int* out_n;
  int k;
  int* err;
};
constexpr int kGtMaxK = 2048;
size_t gt_select_smem(int k);
void launch_gt_row_norms(const float* x, int64_t n, int d, int mode, double* out, cudaStream_t st);
void launch_gt_select(const GtSelectHost& h, int nq, cudaStream_t st);
// f64 distance block [M][ldo] of queries q (M x d) vs corpus rows c (N x d) (rrg_kernels.cu)
void launch_gt_dist(const float* q, int M, const float* c, int N, int d, int metric,
                    const double* qq, const double* cterm, double* out, int64_t ldo, cudaStream_t st);


// -------------------------------------- sliced int8 tensor-core GEMM (rrg_sliced_gemm.cu)
int sliced_kchunks(int K);
int sliced_rows_pad(int rows, bool a_operand);
size_t sliced_plane_bytes(int rows, int K, bool a_operand);
size_t sliced_block_bytes(int K, bool a_operand);  // one 128- (A) / 64-row (B) block
void launch_slice_rows(const float* x, int rows, int K, int ld, bool a_operand, int8_t* planes,
                       int* exps, cudaStream_t st);
void launch_gemm_sliced(const int8_t* a, const int* a_exp, int M, const int8_t* b, const int* b_exp,
                        int N, int K, int epi, float* outf, double* outd, int64_t ldo,
                        const double* rowterm, const double* colterm, cudaStream_t st,
                        int* outi = nullptr);  // EPI_*_ARGMIN: [M][ceil(N/64)] partials

}  // namespace rrg
