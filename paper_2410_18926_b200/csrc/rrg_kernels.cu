// rrg_kernels.cu -- sm_100a kernels of the LoRANN batched query path.
//
// Stage map (reference file:line -> kernel):
//   projection      index.py:298                 -> k_gemm_dmma<EPI_PROJ>
//   query quantize  quantize.py:61-77 (index.py:302) -> k_prep_queries
//   routing         cluster.py:46-58,254-264     -> k_gemm_dmma<EPI_L2|EPI_NEGIP> + k_route_select
//   bucketing       (none in the reference)      -> k_bucket_queries
//   scoring + top-t rrr.py:181-203, index.py:303-316 -> k_score_cluster + k_select_topt
//                                                   (rrg_cluster_score.cu; query-major
//                                                    k_score_select with RRG_SCORE_MODE=query)
//   rerank + top-k  index.py:278-283,318-335     -> k_rerank_tree (perfect pairwise plans,
//                                                   interleaved rows), k_rerank_topk (any d);
//                                                   opt-in: k_rerank_tma, k_rerank_cluster
//   sharded merges            -> k_merge, k_ids_to_pos
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

// =============================================================== f64 GEMM
// C[M x N] = A[M x K] * op(B), A f32 row-major (lda), B f32: !BT -> K x N (ldb),
// BT -> N x K (ldb).  Inputs are widened to f64 (exact), products and sums in
// f64 -- the reference's `x.astype(f64) @ W.astype(f64)` (index.py:298) and
// `p @ c.T` (cluster.py:50,58); the summation order differs from OpenBLAS only at
// the f64 rounding level (0/153,600 projection mismatches).
// FP64 tensor-core GEMM (DMMA, mma.sync.m8n8k4.f64): (32*WM)x64 CTA tile, WM x 2 warps of
// 32x32 (4x4 m8n8 tiles), K staged 8 at a time, double-buffered, in padded smem (pitch 12
// doubles: the four 32 B fragment rows of a half-warp fall in distinct banks).
// WM = 3 (96x64 tiles, 192 threads, 3 CTAs/SM): C2's projection is 105x4 = 420 tiles
// on 444 CTA slots (one wave, 94% balanced) where 128x64 tiles gave 316 tiles on 296
// slots (a 20-CTA second wave).
// f32 inputs are widened to f64 exactly (the reference's `x.astype(f64) @
// W.astype(f64)`, index.py:298, and `p @ c.T`, cluster.py:50,58); products and
// sums in f64, so only the f64 summation order differs from OpenBLAS.
constexpr int MBN = 64, MBK = 8, MPITCH = 12;
constexpr int kGemmWM = 3;

__device__ __forceinline__ void dmma_m8n8k4(double& d0, double& d1, double a, double b) {
  asm volatile("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
               : "+d"(d0), "+d"(d1)
               : "d"(a), "d"(b));
}

// BK: K depth of a stage (8 or 16; 16 halves the barriers per K), pitch BK + 4 doubles.
template <int WM, int BK>
constexpr size_t gemm_smem_bytes() { return (size_t)2 * (32 * WM + MBN) * (BK + 4) * 8; }

template <int EPI, bool BT, int WM = kGemmWM, int BK = MBK>
__global__ void __launch_bounds__(64 * WM, WM == 2 ? 4 : WM == 3 ? 3 : 2) k_gemm_dmma(const float* __restrict__ A, int lda,
                                                     const float* __restrict__ B, int ldb, int M,
                                                     int N, int K, float* __restrict__ outf,
                                                     double* __restrict__ outd, int ldo,
                                                     const double* __restrict__ rowterm,
                                                     const double* __restrict__ colterm,
                                                     int* __restrict__ outi = nullptr) {
  constexpr int MBM = 32 * WM, DMNT = 64 * WM, PITCH = BK + 4;
  constexpr int NA = (MBM * BK) / DMNT, NB = (MBN * BK + DMNT - 1) / DMNT;
  extern __shared__ __align__(16) double gemm_sm[];
  double (*As)[MBM][PITCH] = reinterpret_cast<double (*)[MBM][PITCH]>(gemm_sm);  // [buf][m][k]
  double (*Bs)[MBN][PITCH] = reinterpret_cast<double (*)[MBN][PITCH]>(gemm_sm + 2 * MBM * PITCH);
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wm = warp >> 1, wn = warp & 1;  // WM x 2 warps of 32x32
  const int m0 = blockIdx.y * MBM, n0 = blockIdx.x * MBN;
  double acc[4][4][2];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j][0] = acc[i][j][1] = 0.0;
  // global -> registers (next tile in flight while the current one is multiplied)
  float ra[NA], rb[NB];
  auto gload = [&](int k0) {
#pragma unroll
    for (int e = 0; e < NA; ++e) {  // A tile MBM x 8, k fastest
      const int idx = tid + e * DMNT, r = idx / BK, kk = idx % BK;
      const int gm = m0 + r, gk = k0 + kk;
      ra[e] = (gm < M && gk < K) ? __ldg(A + (size_t)gm * lda + gk) : 0.f;
    }
#pragma unroll
    for (int e = 0; e < NB; ++e) {  // B tile 64 (n) x 8 (k)
      const int idx = tid + e * DMNT;
      int c, kk;
      if (BT) { c = idx / BK; kk = idx % BK; } else { kk = idx / MBN; c = idx % MBN; }
      const int gn = n0 + c, gk = k0 + kk;
      float v = 0.f;
      if (idx < MBN * BK && gn < N && gk < K)
        v = BT ? __ldg(B + (size_t)gn * ldb + gk) : __ldg(B + (size_t)gk * ldb + gn);
      rb[e] = v;
    }
  };
  auto sstore = [&](int buf) {
#pragma unroll
    for (int e = 0; e < NA; ++e) {
      const int idx = tid + e * DMNT;
      As[buf][idx / BK][idx % BK] = (double)ra[e];
    }
#pragma unroll
    for (int e = 0; e < NB; ++e) {
      const int idx = tid + e * DMNT;
      if (idx >= MBN * BK) break;
      if (BT) Bs[buf][idx / BK][idx % BK] = (double)rb[e];
      else Bs[buf][idx % MBN][idx / MBN] = (double)rb[e];
    }
  };
  const int nk = (K + BK - 1) / BK;
  gload(0);
  sstore(0);
  __syncthreads();
  for (int kt = 0; kt < nk; ++kt) {
    const int buf = kt & 1;
    if (kt + 1 < nk) gload((kt + 1) * BK);
#pragma unroll
    for (int ks = 0; ks < BK; ks += 4) {
      double af[4], bf[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) af[i] = As[buf][wm * 32 + i * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int j = 0; j < 4; ++j) bf[j] = Bs[buf][wn * 32 + j * 8 + (lane >> 2)][ks + (lane & 3)];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) dmma_m8n8k4(acc[i][j][0], acc[i][j][1], af[i], bf[j]);
    }
    if (kt + 1 < nk) sstore(buf ^ 1);
    __syncthreads();
  }
  if constexpr (EPI == EPI_L2_TOP4 || EPI == EPI_L2_TOP8) {
    // routing with 1 < w <= TW: each row's TW nearest columns of this tile by
    // (dissimilarity, column), written as TW partials per (row, column tile); the
    // f64 row of dissimilarities is never stored (C3: 164 MB per batch)
    constexpr int TW = EPI == EPI_L2_TOP4 ? 4 : 8;
    double* red_v = gemm_sm;                                          // [MBM][2][TW]
    int* red_i = reinterpret_cast<int*>(gemm_sm + 2 * MBM * TW);      // [MBM][2][TW]
    constexpr double kInfD = __builtin_huge_val();
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = wm * 32 + i * 8 + (lane >> 2), gm = m0 + rl;
      // this lane's 8 columns, sorted by (value, column) with an insertion network
      double v[8];
      int c[8];
#pragma unroll
      for (int t = 0; t < 8; ++t) { v[t] = kInfD; c[t] = 0x7fffffff; }
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * 32 + j * 8 + (lane & 3) * 2 + h;
          double x = kInfD;
          int xi = 0x7fffffff;
          if (gn < N && gm < M) {
            x = __dadd_rn(__dsub_rn(rowterm[gm], __dmul_rn(2.0, acc[i][j][h])), colterm[gn]);
            x = x > 0.0 ? x : 0.0;
            xi = gn;
          }
          bool in = false;
#pragma unroll
          for (int t = 0; t < 8; ++t)
            if (in || x < v[t] || (x == v[t] && xi < c[t])) {
              const double tv = v[t]; const int tc = c[t];
              v[t] = x; c[t] = xi; x = tv; xi = tc; in = true;
            }
        }
      // TW rounds of an argmin over the row's 4 lanes (xor 1, 2): the row's TW smallest
      // of the warp's 32 columns
#pragma unroll
      for (int r = 0; r < TW; ++r) {
        double b = v[0];
        int bc = c[0];
#pragma unroll
        for (int o = 1; o <= 2; o <<= 1) {
          const double ob = __shfl_xor_sync(0xffffffffu, b, o);
          const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
          if (ob < b || (ob == b && oc < bc)) { b = ob; bc = oc; }
        }
        if (c[0] == bc && bc != 0x7fffffff) {
#pragma unroll
          for (int t = 0; t < 7; ++t) { v[t] = v[t + 1]; c[t] = c[t + 1]; }
          v[7] = kInfD; c[7] = 0x7fffffff;
        }
        if ((lane & 3) == 0) { red_v[(rl * 2 + wn) * TW + r] = b; red_i[(rl * 2 + wn) * TW + r] = bc; }
      }
    }
    __syncthreads();
    for (int r = tid; r < MBM; r += DMNT) {  // merge the two warp columns' sorted lists
      const int gm = m0 + r;
      if (gm >= M) continue;
      const double* va = red_v + (r * 2) * TW;
      const int* ia = red_i + (r * 2) * TW;
      int p0 = 0, p1 = 0;
      for (int k = 0; k < TW; ++k) {
        const double a0 = va[p0], a1 = va[TW + p1];
        const int i0 = ia[p0], i1 = ia[TW + p1];
        const bool first = a0 < a1 || (a0 == a1 && i0 < i1);
        const size_t o = ((size_t)gm * ldo + blockIdx.x) * TW + k;
        outd[o] = first ? a0 : a1;
        outi[o] = first ? i0 : i1;
        if (first) ++p0; else ++p1;
      }
    }
    return;
  }
  if constexpr (EPI == EPI_L2_ARGMIN || EPI == EPI_NEGIP_ARGMIN) {
    // routing with w = 1: only each row's nearest column is needed -- reduce this
    // tile's 64 columns to (dissimilarity, lowest column) per row and write one partial
    // per (row, column tile) instead of the row of f64 dissimilarities
    double* red_v = gemm_sm;                                   // [MBM][2]
    int* red_i = reinterpret_cast<int*>(gemm_sm + 2 * MBM);   // [MBM][2]
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const int rl = wm * 32 + i * 8 + (lane >> 2), gm = m0 + rl;
      double best = __longlong_as_double(0x7ff0000000000000ll);  // +inf
      int bcol = 0x7fffffff;
#pragma unroll
      for (int j = 0; j < 4; ++j)
#pragma unroll
        for (int h = 0; h < 2; ++h) {
          const int gn = n0 + wn * 32 + j * 8 + (lane & 3) * 2 + h;
          if (gn >= N || gm >= M) continue;
          double dv;
          if (EPI == EPI_L2_ARGMIN) {
            dv = __dadd_rn(__dsub_rn(rowterm[gm], __dmul_rn(2.0, acc[i][j][h])), colterm[gn]);
            dv = dv > 0.0 ? dv : 0.0;
          } else {
            dv = -acc[i][j][h];
            // a non-finite query (rejected with DataError after the search) must still
            // route to a valid cluster: NaN compares false, so rank it as +inf
            if (dv != dv) dv = __longlong_as_double(0x7ff0000000000000ll);
          }
          if (dv < best || (dv == best && gn < bcol)) { best = dv; bcol = gn; }
        }
#pragma unroll
      for (int o = 1; o <= 2; o <<= 1) {  // the 4 lanes holding this row's columns
        const double ob = __shfl_xor_sync(0xffffffffu, best, o);
        const int oc = __shfl_xor_sync(0xffffffffu, bcol, o);
        if (ob < best || (ob == best && oc < bcol)) { best = ob; bcol = oc; }
      }
      if ((lane & 3) == 0) { red_v[rl * 2 + wn] = best; red_i[rl * 2 + wn] = bcol; }
    }
    __syncthreads();
    for (int r = tid; r < MBM; r += DMNT) {
      const int gm = m0 + r;
      if (gm >= M) continue;
      double b0 = red_v[r * 2], b1 = red_v[r * 2 + 1];
      int c0 = red_i[r * 2], c1 = red_i[r * 2 + 1];
      if (b1 < b0 || (b1 == b0 && c1 < c0)) { b0 = b1; c0 = c1; }
      outd[(size_t)gm * ldo + blockIdx.x] = b0;
      outi[(size_t)gm * ldo + blockIdx.x] = c0;
    }
    return;
  }
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    const int gm = m0 + wm * 32 + i * 8 + (lane >> 2);
    if (gm >= M) continue;
#pragma unroll
    for (int j = 0; j < 4; ++j) {
#pragma unroll
      for (int h = 0; h < 2; ++h) {
        const int gn = n0 + wn * 32 + j * 8 + (lane & 3) * 2 + h;
        if (gn >= N) continue;
        const double v = acc[i][j][h];
        if (EPI == 0) {
          outf[(size_t)gm * ldo + gn] = (float)v;
        } else if (EPI == 1) {
          const double d2 = __dadd_rn(__dsub_rn(rowterm[gm], __dmul_rn(2.0, v)), colterm[gn]);
          outd[(size_t)gm * ldo + gn] = d2 > 0.0 ? d2 : 0.0;
        } else if (EPI == EPI_GT_L2) {
          outd[(size_t)gm * ldo + gn] = __dadd_rn(__dsub_rn(rowterm[gm], __dmul_rn(2.0, v)), colterm[gn]);
        } else if (EPI == EPI_GT_COS) {
          outd[(size_t)gm * ldo + gn] = -__ddiv_rn(v, colterm[gn]);
        } else {
          outd[(size_t)gm * ldo + gn] = -v;
        }
      }
    }
  }
}

// ======================================================= small-batch GEMV
// Batches of a few queries: one warp per output element, f64 accumulation of the
// exact f32 products in lane-strided order plus a shuffle tree (the same f64-level
// contract as k_gemm_dmma: only the f64 summation order differs from OpenBLAS), so
// the ~10 dependent K-steps of a 1-row GEMM tile do not set the latency.
// B is N x K row-major (W^T for the projection, the centroids for routing).
template <int EPI>
__global__ void k_gemv_f64(const float* __restrict__ A, int lda, const float* __restrict__ B,
                           int M, int N, int K, float* __restrict__ outf,
                           double* __restrict__ outd, int ldo, const double* __restrict__ rowterm,
                           const double* __restrict__ colterm) {
  const int64_t wid = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (wid >= (int64_t)M * N) return;
  const int q = (int)(wid / N), j = (int)(wid % N);
  const float* a = A + (size_t)q * lda;
  const float* b = B + (size_t)j * K;
  double acc = 0.0;
  for (int k = lane; k < K; k += 32) acc = fma((double)__ldg(a + k), (double)__ldg(b + k), acc);
  for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if (lane != 0) return;
  if (EPI == EPI_PROJ) {
    outf[(size_t)q * ldo + j] = (float)acc;
  } else if (EPI == EPI_L2) {
    const double d2 = __dadd_rn(__dsub_rn(rowterm[q], __dmul_rn(2.0, acc)), colterm[j]);
    outd[(size_t)q * ldo + j] = d2 > 0.0 ? d2 : 0.0;
  } else {
    outd[(size_t)q * ldo + j] = -acc;
  }
}

void launch_project_small(const float* x, const float* Wt, int nq, int d, int s, float* xp,
                          cudaStream_t st) {
  const int64_t warps = (int64_t)nq * s;
  (k_gemv_f64<EPI_PROJ><<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(x, d, Wt, nq, s, d, xp, nullptr,
                                                                     s, nullptr, nullptr), note_launch());
}

void launch_route_dist_small(const float* xp, const float* cent, int nq, int L, int s, int metric,
                             const double* pp, const double* cnorm, double* diss, cudaStream_t st) {
  const int64_t warps = (int64_t)nq * L;
  const unsigned grid = (unsigned)((warps + 7) / 8);
  if (metric == kMetricEuclidean)
    (k_gemv_f64<EPI_L2><<<grid, 256, 0, st>>>(xp, s, cent, nq, L, s, nullptr, diss, L, pp, cnorm), note_launch());
  else
    (k_gemv_f64<EPI_NEGIP><<<grid, 256, 0, st>>>(xp, s, cent, nq, L, s, nullptr, diss, L, nullptr,
                                                nullptr), note_launch());
}

// ========================================================== query prep
// One warp per query: quantize_vector(xp, mixed_precision=True) (quantize.py:61-77)
// -> qcodes[q][0..s_pad) with slot 0 = 0 (pairs with the file's zero pad row of A),
// qscale, qhead; pp = (p*p).sum() in f64 NumPy pairwise order for routing; and
// xx = f32(x.x) for the no-rerank euclidean score shift (index.py:327).
__global__ void k_prep_queries(const float* __restrict__ xp, const float* __restrict__ x, int nq,
                               int s, int s_pad, int d, int8_t* __restrict__ qcodes,
                               float* __restrict__ qscale, float* __restrict__ qhead,
                               double* __restrict__ pp, float* __restrict__ xx,
                               int* __restrict__ nonfinite) {
  int warp = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int lane = threadIdx.x & 31;
  if (warp >= nq) return;
  const float* row = xp + (size_t)warp * s;
  float amax = 0.0f;
  for (int i = 1 + lane; i < s; i += 32) amax = fmaxf(amax, fabsf(row[i]));
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  float sc = quant_scale(amax);
  int8_t* out = qcodes + (size_t)warp * s_pad;
  for (int i = lane; i < s_pad; i += 32) {
    int c = 0;
    if (i >= 1 && i < s && amax != 0.0f) c = quant_code(row[i], sc);
    out[i] = (int8_t)c;
  }
  double xsum = 0.0;
  const float* xr = x + (size_t)warp * d;
  bool bad = false;
  for (int i = lane; i < d; i += 32) {
    const float v = xr[i];
    bad |= !isfinite(v);
    xsum += (double)v * (double)v;
  }
  // _check_finite (index.py:144-150) for the host-buffer entry, folded into this pass
  if (nonfinite && __any_sync(0xffffffffu, bad) && lane == 0) atomicOr(nonfinite, 1);
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) xsum += __shfl_xor_sync(0xffffffffu, xsum, o);
  auto get = [&](int i) { double v = (double)row[i]; return v * v; };
  const int pwl = pw_warp_leaves(s);  // (s = 64, 256: one lane per accumulator chain)
  const double ppw = pwl ? pw_sum_warp<double>(get, s, pwl, lane) : 0.0;
  if (lane == 0) {
    qscale[warp] = sc;
    qhead[warp] = row[0];
    xx[warp] = (float)xsum;
    pp[warp] = pwl ? ppw : pw_sum_seq<double>(get, s);
  }
}

// ========================================================== routing select
// route(): stable argsort of the dissimilarities, first w (cluster.py:263-264):
// the w smallest by (diss, cluster id).  One CTA per query.
template <int NT>
__global__ void __launch_bounds__(NT) k_route_select(const double* __restrict__ diss, int L, int w,
                                                     int* __restrict__ sel,
                                                     int* __restrict__ primary) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  uint64_t* keys = reinterpret_cast<uint64_t*>(smem_raw);
  int* outidx = reinterpret_cast<int*>(keys + L);
  const double* row = diss + (size_t)blockIdx.x * L;
  for (int i = threadIdx.x; i < L; i += NT) keys[i] = mono64(row[i]);
  __syncthreads();
  auto key = [&](int i) { return keys[i]; };
  auto tie = [&](int i) { return (uint32_t)i; };
  auto val = [](uint64_t k) { return unmono64(k); };
  block_select_bucketed<NT, uint64_t, double>(L, w, key, tie, val, outidx, bs, sm);
  for (int i = threadIdx.x; i < w; i += NT) sel[(size_t)blockIdx.x * w + i] = outidx[i];
  // nearest cluster (route()[0]) -- the bucketing key that groups queries for locality
  if (threadIdx.x < 32) {
    uint64_t bk = ~0ull;
    int bi = 0x7fffffff;
    for (int i = threadIdx.x; i < w; i += 32) {
      int c = outidx[i];
      uint64_t kc = keys[c];
      if (kc < bk || (kc == bk && c < bi)) { bk = kc; bi = c; }
    }
    for (int o = 16; o > 0; o >>= 1) {
      uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
      int oi = __shfl_xor_sync(0xffffffffu, bi, o);
      if (ok < bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
    }
    if (threadIdx.x == 0) primary[blockIdx.x] = bi;
  }
}

// 1 < w <= 8: the w nearest by (dissimilarity, cluster id), one warp per query: each
// lane keeps the sorted w smallest of its strided share of the row (ascending ids per
// lane, so an equal key never displaces an earlier id), then w rounds of a warp argmin
// over the lanes' heads.  (A CTA per query with the bucketed block select spent ~10 us
// of barriers per query: C3, w = 4 over 2,048 clusters, 105 us per batch.)
template <int WM>
__global__ void k_route_select_warp(const double* __restrict__ diss, int nq, int L, int w,
                                    int* __restrict__ sel, int* __restrict__ primary) {
  const int q = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const double* row = diss + (size_t)q * L;
  uint64_t bk[WM];
  int bi[WM];
#pragma unroll
  for (int s = 0; s < WM; ++s) { bk[s] = ~0ull; bi[s] = 0x7fffffff; }
  auto insert = [&](uint64_t x, int xi) {
    if (!(x < bk[WM - 1])) return;
    bool in = false;  // once placed, every later slot shifts right by one
#pragma unroll
    for (int s = 0; s < WM; ++s)
      if (in || x < bk[s]) {
        const uint64_t tk = bk[s]; const int ti = bi[s];
        bk[s] = x; bi[s] = xi; x = tk; xi = ti;
        in = true;
      }
  };
  constexpr int U = 4;
  for (int c0 = lane; c0 < L; c0 += 32 * U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = c0 + 32 * u < L ? __ldg(row + c0 + 32 * u) : 0.0;
#pragma unroll
    for (int u = 0; u < U; ++u)
      if (c0 + 32 * u < L) insert(mono64(v[u]), c0 + 32 * u);
  }
  for (int r = 0; r < w; ++r) {
    uint64_t k = bk[0];
    int i = bi[0];
    for (int o = 16; o > 0; o >>= 1) {
      const uint64_t ok = __shfl_xor_sync(0xffffffffu, k, o);
      const int oi = __shfl_xor_sync(0xffffffffu, i, o);
      if (ok < k || (ok == k && oi < i)) { k = ok; i = oi; }
    }
    if (bi[0] == i) {  // the owner pops its head (ids are unique)
#pragma unroll
      for (int s = 0; s + 1 < WM; ++s) { bk[s] = bk[s + 1]; bi[s] = bi[s + 1]; }
      bk[WM - 1] = ~0ull; bi[WM - 1] = 0x7fffffff;
    }
    if (lane == 0) {
      sel[(size_t)q * w + r] = i;
      if (r == 0) primary[q] = i;
    }
  }
}

// w == 1: the nearest cluster by (dissimilarity, cluster id) -- argsort(stable)[0]
// (cluster.py:263-264) -- one warp per query, a coalesced sweep of the row and a
// shuffle argmin; no CTA barriers.
__global__ void k_route_nearest(const double* __restrict__ diss, int nq, int L,
                                int* __restrict__ sel, int* __restrict__ primary) {
  const int q = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  const double* row = diss + (size_t)q * L;
  uint64_t bk = ~0ull;
  int bi = 0x7fffffff;
  for (int i = lane; i < L; i += 32) {  // ascending ids per lane: strict < keeps the lowest
    const uint64_t k = mono64(__ldg(row + i));
    if (k < bk) { bk = k; bi = i; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const uint64_t ok = __shfl_xor_sync(0xffffffffu, bk, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ok < bk || (ok == bk && oi < bi)) { bk = ok; bi = oi; }
  }
  if (lane == 0) {
    sel[q] = bi;
    primary[q] = bi;
  }
}

// ======================================================== query bucketing
// Counting sort of the batch by nearest cluster (histogram, exclusive scan,
// scatter), one CTA.  The scoring and re-rank CTAs then visit queries in bucket
// order, so queries probing the same clusters -- and re-ranking overlapping
// corpus rows -- run concurrently and share L2.  Order only affects locality;
// every query's result is independent of it.
constexpr int BNT = 1024;
__global__ void __launch_bounds__(BNT) k_bucket_queries(const int* __restrict__ primary, int nq,
                                                        int L, int* __restrict__ order) {
  extern __shared__ int hist[];  // L + 1
  for (int i = threadIdx.x; i <= L; i += BNT) hist[i] = 0;
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += BNT) atomicAdd(&hist[primary[q]], 1);
  __syncthreads();
  if (threadIdx.x < 32) {  // exclusive scan by one warp
    int lane = threadIdx.x, carry = 0;
    for (int base = 0; base < L; base += 32) {
      int i = base + lane;
      int v = i < L ? hist[i] : 0, incl = v;
      for (int o = 1; o < 32; o <<= 1) {
        int t = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += t;
      }
      if (i < L) hist[i] = carry + incl - v;
      carry += __shfl_sync(0xffffffffu, incl, 31);
    }
  }
  __syncthreads();
  for (int q = threadIdx.x; q < nq; q += BNT) order[atomicAdd(&hist[primary[q]], 1)] = q;
}

// ====================================================== scoring + top-t select
// One CTA per query.  For every routed cluster:
//   rrr model   : raw1 = codes_x . A (int32, dp4a), inter = deq(raw1) (r values),
//                 re-quantize inter, raw2_p = codes_r . B[:,p], yhat_p = deq(raw2_p)
//   exact model : raw_p = codes_x . A[:,p], yhat_p = deq(raw_p)
//   key_p = -2 yhat_p + norm_p (euclidean) | -yhat_p (ip/cosine)   (rrr.py:198-202, index.py:310)
// then the take = min(t|k, ncand) smallest by (key, corpus id)  (index.py:314-316).
// Candidate keys/positions live in shared memory when they fit, else in a
// per-query global slice.
struct ScoreArgs {
  DevIndexView ix;
  const int8_t* qcodes;
  const float* qscale;
  const float* qhead;
  const float* xx;
  const int* sel;
  int w;
  int take_cap;   // t (rerank) or k (no rerank)
  int rerank;
  int k;
  int smem_cap;   // candidates that fit in dynamic smem
  uint32_t* gkeys;  // [nq][gcap] overflow
  int* gpos;
  int64_t gcap;
  int* cand_pos;  // [nq][take_cap] out (rerank)
  int* cand_n;    // [nq]
  int64_t* out_ids;  // no-rerank outputs [nq][k]
  float* out_scores;
  int* out_count;
  int q0;  // query offset of this chunk (outputs)
  const int* order;  // CTA -> chunk-local query (bucket order), or nullptr
  uint32_t* sel_keys;  // optional [nq][take_cap] keys of the local top-t (sharded phase 1)
  uint32_t* sel_ids;   // optional [nq][take_cap] corpus ids of the local top-t
  int* sel_count;      // optional [nq]
};

constexpr int SNT = 512;
constexpr int kMaxWChunk = 64;
constexpr int kMaxR = 64;

__global__ void __launch_bounds__(SNT) k_score_select(ScoreArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  __shared__ __align__(16) int8_t c2s[kMaxWChunk][kMaxR];
  __shared__ float s2s[kMaxWChunk], h2s[kMaxWChunk];
  __shared__ float inters[kMaxWChunk][kMaxR];
  __shared__ int cl_l[kMaxWChunk], cl_p0[kMaxWChunk], cl_m[kMaxWChunk], cl_off[kMaxWChunk + 1];
  __shared__ int total_n;
  __shared__ __align__(16) int8_t qs[1024 + 16];

  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = SNT / 32;
  const int s_pad = ix.s_pad, r = ix.r, r_pad = ix.r_pad;
  const float xscale = a.qscale[q], xhead = a.qhead[q];
  const int8_t* qc = a.qcodes + (size_t)q * s_pad;
  for (int i = tid; i < s_pad; i += SNT) qs[i] = qc[i];
  const int* selq = a.sel + (size_t)q * a.w;

  // total candidates
  if (tid == 0) total_n = 0;
  __syncthreads();
  {
    int local = 0;
    for (int c = tid; c < a.w; c += SNT) {
      int l = selq[c];
      local += ix.cl_pos[l + 1] - ix.cl_pos[l];
    }
    for (int o = 16; o > 0; o >>= 1) local += __shfl_xor_sync(0xffffffffu, local, o);
    if (lane == 0 && local) atomicAdd(&total_n, local);
  }
  __syncthreads();
  const int N = total_n;
  uint32_t* keys;
  int* pos;
  if (N <= a.smem_cap) {
    keys = reinterpret_cast<uint32_t*>(smem_raw);
    pos = reinterpret_cast<int*>(keys + a.smem_cap);
  } else {
    keys = a.gkeys + (size_t)q * a.gcap;
    pos = a.gpos + (size_t)q * a.gcap;
  }
  const bool euclid = ix.metric == kMetricEuclidean;

  int cand_base = 0;
  for (int c0 = 0; c0 < a.w; c0 += kMaxWChunk) {
    const int nc = min(kMaxWChunk, a.w - c0);
    if (warp == 0) {  // chunk's cluster table: parallel loads + warp prefix sum
      int carry = cand_base;
      for (int b0 = 0; b0 < nc; b0 += 32) {
        int c = b0 + lane, m = 0;
        if (c < nc) {
          int l = selq[c0 + c];
          int p0 = ix.cl_pos[l];
          m = ix.cl_pos[l + 1] - p0;
          cl_l[c] = l;
          cl_p0[c] = p0;
          cl_m[c] = m;
        }
        int incl = m;
        for (int o = 1; o < 32; o <<= 1) {
          int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        if (c < nc) cl_off[c] = carry + incl - m;
        carry += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) cl_off[nc] = carry;
    }
    __syncthreads();
    // ---- stage A (rrr clusters), all threads: raw1 = codes_x . A[:, j] for every
    // (cluster, j), the s_pad/16 int4 words split over `parts` consecutive lanes
    {
      const int pairs = nc * r;
      const int nvec = s_pad / 16;
      int parts = 1;
      while (parts < 32 && pairs * parts * 2 <= SNT && parts * 2 <= nvec) parts <<= 1;
      const int4* q4 = reinterpret_cast<const int4*>(qs);
      for (int base = 0; base < pairs * parts; base += SNT) {
        const int e = base + tid;
        const int pr = e / parts, part = e % parts;
        int raw = 0;
        int c = pr / r, j = pr % r;
        bool act = pr < pairs;
        int l = act ? cl_l[c] : 0;
        act = act && ix.cl_kind[l] == kKindRrr && cl_m[c] > 0;
        if (act) {
          const int4* aw =
              reinterpret_cast<const int4*>(ix.at + ((size_t)ix.cl_aidx[l] * r + j) * s_pad);
          for (int u = part; u < nvec; u += parts) {
            int4 b = __ldg(aw + u), cc = q4[u];
            raw = __dp4a(cc.x, b.x, raw);
            raw = __dp4a(cc.y, b.y, raw);
            raw = __dp4a(cc.z, b.z, raw);
            raw = __dp4a(cc.w, b.w, raw);
          }
        }
        for (int o = 1; o < parts; o <<= 1) raw += __shfl_xor_sync(0xffffffffu, raw, o);
        if (act && part == 0) {
          const size_t aj = (size_t)ix.cl_aidx[l] * r + j;
          inters[c][j] = deq(raw, xscale, ix.ascale[aj], xhead, ix.ahead[aj]);
        }
      }
    }
    __syncthreads();
    // re-quantize each cluster's intermediate vector (quantize.py:150): warp per cluster
    for (int c = warp; c < nc; c += nwarps) {
      int l = cl_l[c];
      if (ix.cl_kind[l] != kKindRrr || cl_m[c] == 0) continue;
      float amax = 0.0f;
      for (int j = 1 + lane; j < r; j += 32) amax = fmaxf(amax, fabsf(inters[c][j]));
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
      const float sc2 = quant_scale(amax);
      for (int j = lane; j < r_pad; j += 32) {
        int code = 0;
        if (j >= 1 && j < r && amax != 0.0f) code = quant_code(inters[c][j], sc2);
        c2s[c][j] = (int8_t)code;
      }
      if (lane == 0) { s2s[c] = sc2; h2s[c] = inters[c][0]; }
    }
    __syncthreads();
    // ---- stage B: one thread per candidate point; 16-byte code and metadata loads
    const int nloc = cl_off[nc] - cand_base;
    int c = 0;  // cluster of element e, advanced monotonically as e grows
    for (int e = tid; e < nloc; e += SNT) {
      while (cl_off[c + 1] - cand_base <= e) ++c;
      const int p = e - (cl_off[c] - cand_base);
      const int l = cl_l[c];
      const int gp = cl_p0[c] + p;
      const float4 meta = __ldg(ix.pmeta + gp);
      float yhat;
      if (ix.cl_kind[l] == kKindRrr) {
        const int4* bw = reinterpret_cast<const int4*>(ix.bt + (size_t)gp * r_pad);
        const int4* cw = reinterpret_cast<const int4*>(c2s[c]);
        int raw = 0;
        for (int u = 0; u < r_pad / 16; ++u) {
          int4 b = __ldg(bw + u), cc = cw[u];
          raw = __dp4a(cc.x, b.x, raw);
          raw = __dp4a(cc.y, b.y, raw);
          raw = __dp4a(cc.z, b.z, raw);
          raw = __dp4a(cc.w, b.w, raw);
        }
        yhat = deq(raw, s2s[c], meta.y, h2s[c], meta.x);
      } else {
        const int4* xw = reinterpret_cast<const int4*>(ix.xcodes + (size_t)(ix.cl_aidx[l] + p) * s_pad);
        const int4* q4 = reinterpret_cast<const int4*>(qs);
        int raw = 0;
        for (int u = 0; u < s_pad / 16; ++u) {
          int4 b = __ldg(xw + u), cc = q4[u];
          raw = __dp4a(cc.x, b.x, raw);
          raw = __dp4a(cc.y, b.y, raw);
          raw = __dp4a(cc.z, b.z, raw);
          raw = __dp4a(cc.w, b.w, raw);
        }
        yhat = deq(raw, xscale, meta.y, xhead, meta.x);
      }
      float keyf = euclid ? __fadd_rn(__fmul_rn(-2.0f, yhat), meta.z) : -yhat;
      keys[cl_off[c] + p] = mono32(keyf);
      pos[cl_off[c] + p] = gp;
    }
    cand_base = cl_off[nc];
    __syncthreads();
  }

  // ---- top-take by (key, corpus id)
  const int take = min(a.take_cap, N);
  int* selidx = reinterpret_cast<int*>(smem_raw + (size_t)a.smem_cap * 8);  // after keys+pos
  auto key = [&](int i) { return keys[i]; };
  auto tie = [&](int i) { return (uint32_t)ix.pid[pos[i]]; };
  auto val = [](uint32_t k) { return unmono32(k); };
  block_select_bucketed<SNT, uint32_t, float>(N, take, key, tie, val, selidx, bs, sm);

  const int gq = a.q0 + q;
  if (a.rerank) {
    int* outp = a.cand_pos + (size_t)q * a.take_cap;
    for (int i = tid; i < take; i += SNT) outp[i] = pos[selidx[i]];
    if (a.sel_keys) {  // sharded phase 1: (key, corpus id) of the local top-t
      uint32_t* ok = a.sel_keys + (size_t)(a.q0 + q) * a.take_cap;
      uint32_t* oi = a.sel_ids + (size_t)(a.q0 + q) * a.take_cap;
      for (int i = tid; i < take; i += SNT) {
        int ci = selidx[i];
        ok[i] = keys[ci];
        oi[i] = __float_as_uint(__ldg(ix.pmeta + pos[ci]).w);
      }
      if (tid == 0) a.sel_count[a.q0 + q] = take;
    }
    if (tid == 0) a.cand_n[q] = take;
    return;
  }
  // no rerank: order the take (<= k) winners by (key, id) and emit (index.py:323-329)
  uint64_t* srt = reinterpret_cast<uint64_t*>(selidx + a.take_cap + 2);
  srt = reinterpret_cast<uint64_t*>((reinterpret_cast<uintptr_t>(srt) + 15) & ~uintptr_t(15));
  int np2 = 1;
  while (np2 < take) np2 <<= 1;
  for (int i = tid; i < np2; i += SNT) {
    uint64_t v = ~0ull;
    if (i < take) {
      int ci = selidx[i];
      v = ((uint64_t)keys[ci] << 32) | (uint32_t)ix.pid[pos[ci]];
    }
    srt[i] = v;
  }
  block_bitonic_sort<SNT>(srt, np2);
  const float xxq = a.xx[q];
  for (int i = tid; i < a.k; i += SNT) {
    int64_t id = -1;
    float sc = __int_as_float(0x7fc00000);
    if (i < take) {
      uint64_t v = srt[i];
      id = (int64_t)(uint32_t)v;
      float kf = unmono32((uint32_t)(v >> 32));
      sc = euclid ? __fadd_rn(kf, xxq) : -kf;
    }
    a.out_ids[(size_t)gq * a.k + i] = id;
    a.out_scores[(size_t)gq * a.k + i] = sc;
  }
  if (tid == 0) a.out_count[gq] = take;
}

// ======================================================= rerank + top-k
// One CTA per query; one warp per candidate row.  Euclidean: the row's exact
// squared distance with NumPy's pairwise summation tree over the f32 squares
// rn(rn(c - x)^2) (index.py:281-282); ip/cosine: -(c . x) (index.py:283,
// BLAS-order dependent -> tolerance).  Then top-k by (diss, corpus id)
// (index.py:320-322), sorted, scores = diss | -diss.
struct RerankArgs {
  DevIndexView ix;
  const float* queries;  // [nq][d] (chunk-local)
  const int* cand_pos;
  const int* cand_n;
  int take_cap;
  int k;
  int64_t* out_ids;
  float* out_scores;
  int* out_count;
  int q0;
  const int* order;
};

constexpr int RNT = 256;

__global__ void __launch_bounds__(RNT) k_rerank_topk(RerankArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = RNT / 32;
  const int d = ix.d, ds = ix.d_stride;
  const int n = a.cand_n[q];
  // smem: x[ds] | per-warp row buffers [nwarps][ds] | diss keys[take_cap] | ids[take_cap] | sel[k] | sort[np2]
  float* xs = reinterpret_cast<float*>(smem_raw);
  float* rowbuf = xs + ds;
  uint32_t* dkeys = reinterpret_cast<uint32_t*>(rowbuf + (size_t)nwarps * ds);
  uint32_t* dids = dkeys + a.take_cap;
  int* selidx = reinterpret_cast<int*>(dids + a.take_cap);
  uintptr_t sp = reinterpret_cast<uintptr_t>(selidx + a.k);
  uint64_t* srt = reinterpret_cast<uint64_t*>((sp + 15) & ~uintptr_t(15));

  const float* xq = a.queries + (size_t)q * d;
  for (int i = tid; i < ds; i += RNT) xs[i] = i < d ? xq[i] : 0.0f;
  __syncthreads();
  const bool euclid = ix.metric == kMetricEuclidean;
  const int* cp = a.cand_pos + (size_t)q * a.take_cap;
  float* mybuf = rowbuf + (size_t)warp * ds;
  const int nv4 = ds / 4;
  for (int i = warp; i < n; i += nwarps) {
    int gp = cp[i];
    const float4* row = reinterpret_cast<const float4*>(ix.corpus + (size_t)gp * ds);
    const float4* x4 = reinterpret_cast<const float4*>(xs);
    float diss;
    if (euclid) {
      for (int v = lane; v < nv4; v += 32) {
        float4 c = __ldg(row + v);
        float4 xv = x4[v];
        float4 o;
        float t0 = __fsub_rn(c.x, xv.x), t1 = __fsub_rn(c.y, xv.y);
        float t2 = __fsub_rn(c.z, xv.z), t3 = __fsub_rn(c.w, xv.w);
        o.x = __fmul_rn(t0, t0); o.y = __fmul_rn(t1, t1);
        o.z = __fmul_rn(t2, t2); o.w = __fmul_rn(t3, t3);
        reinterpret_cast<float4*>(mybuf)[v] = o;
      }
      __syncwarp();
      if (lane == 0) {
        auto get = [&](int j) { return mybuf[j]; };
        diss = pw_sum_seq<float>(get, d);
      }
      __syncwarp();
    } else {
      float part = 0.0f;
      for (int v = lane; v < nv4; v += 32) {
        float4 c = __ldg(row + v);
        float4 xv = x4[v];
        part += c.x * xv.x + c.y * xv.y + c.z * xv.z + c.w * xv.w;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
      diss = -part;
    }
    if (lane == 0) {
      dkeys[i] = mono32(diss);
      dids[i] = (uint32_t)ix.pid[gp];
    }
  }
  __syncthreads();
  const int kk = min(a.k, n);
  auto key = [&](int i) { return dkeys[i]; };
  auto tie = [&](int i) { return dids[i]; };
  auto val = [](uint32_t k) { return unmono32(k); };
  block_select_bucketed<RNT, uint32_t, float>(n, kk, key, tie, val, selidx, bs, sm);
  int np2 = 1;
  while (np2 < kk) np2 <<= 1;
  for (int i = tid; i < np2; i += RNT) {
    uint64_t v = ~0ull;
    if (i < kk) {
      int ci = selidx[i];
      v = ((uint64_t)dkeys[ci] << 32) | dids[ci];
    }
    srt[i] = v;
  }
  block_bitonic_sort<RNT>(srt, np2);
  const int gq = a.q0 + q;
  for (int i = tid; i < a.k; i += RNT) {
    int64_t id = -1;
    float sc = __int_as_float(0x7fc00000);
    if (i < kk) {
      uint64_t v = srt[i];
      id = (int64_t)(uint32_t)v;
      float df = unmono32((uint32_t)(v >> 32));
      sc = euclid ? df : -df;
    }
    a.out_ids[(size_t)gq * a.k + i] = id;
    a.out_scores[(size_t)gq * a.k + i] = sc;
  }
  if (tid == 0) a.out_count[gq] = kk;
}

// ================================================= rerank (warp-parallel tree)
// Same contract as k_rerank_topk for a perfect pairwise plan (2^a equal leaves of
// nl = pw_leaf_n elements).  Lane layout: a row's 4*nleaves (leaf, pair) slots
// are spread over G lanes; lane (leaf b, pair h) owns NumPy's accumulators
// r[2h], r[2h+1] of leaf b and streams float2 elements b*nl + 8i + 2h.  Then
//   r[2h]+r[2h+1], xor-1, xor-2 shuffles  == ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//   + the nl%8 tail sequentially,
//   xor-4/8/16 shuffles (+ slot pairs)     == the perfect leaf tree,
// i.e. bit-identical to `(diff*diff).sum(axis=1)` (index.py:281-282).
// G = 4*nleaves lanes per row when <= 32 (so 32/G rows per warp pass), else
// SLOTS = 4*nleaves/32 slots per lane.
// NB = chain length nl/8 as a compile-time constant (loads use immediate
// offsets, no per-element predicates); NB = 0 is the runtime-length fallback.
// NLV = number of leaves as a compile-time constant too (step stride 8*NLV and
// the lane-group width G become immediates); 0 = runtime.
// UROWS row groups in flight per warp and MINB CTAs per SM: measured on C2 (d=768),
// U=1 at 4 CTAs/SM (64 regs, 32 warps/SM) beats U=2 at 2 CTAs/SM (1.66 vs 2.08 ms):
// more warps hide the L2 latency better than more rows per warp.
template <int SLOTS, int NB, int NLV, int UROWS = 1, int MINB = (SLOTS == 1 ? 4 : 1)>
__global__ void __launch_bounds__(RNT, MINB) k_rerank_tree(RerankArgs a) {
  constexpr int kMaxNb = NB > 0 ? NB : 16;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = RNT / 32;
  const int d = ix.d, ds = ix.d_stride, nl = ix.pw_leaf_n, tail = nl % 8;
  const int nb = NB > 0 ? NB : nl / 8;
  const int P = 4 * (NLV > 0 ? NLV : ix.pw_nleaves);
  const int G = SLOTS == 1 ? P : 32;
  const int R = 32 / G;
  const int g = lane / G, pl = lane % G;
  const int n = a.cand_n[q];
  uint32_t* dkeys = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* dids = dkeys + a.take_cap;
  int* selidx = reinterpret_cast<int*>(dids + a.take_cap);
  uintptr_t sp = reinterpret_cast<uintptr_t>(selidx + a.k);
  uint64_t* srt = reinterpret_cast<uint64_t*>((sp + 15) & ~uintptr_t(15));
  const bool euclid = ix.metric == kMetricEuclidean;
  const float* xq = a.queries + (size_t)q * d;

  // this lane's slice of the query, in registers
  float2 xv[SLOTS][kMaxNb];
  float xt[SLOTS][7];
  int off[SLOTS], coff[SLOTS], ctail[SLOTS];
  // corpus rows are interleaved step-major (DevIndexView::corpus_interleaved):
  // step i of (leaf b, pair h) sits at i*cstep + 8b + 2h
  const int cstep = 8 * (NLV > 0 ? NLV : ix.pw_nleaves);
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    int pair = pl + 32 * s;
    int b = pair >> 2, h = pair & 3;
    off[s] = b * nl + 2 * h;
    coff[s] = 8 * b + 2 * h;
    ctail[s] = nb * cstep + b * tail;
#pragma unroll
    for (int i = 0; i < kMaxNb; ++i)
      xv[s][i] = i < nb ? *reinterpret_cast<const float2*>(xq + off[s] + 8 * i) : make_float2(0.f, 0.f);
#pragma unroll
    for (int u = 0; u < 7; ++u) xt[s][u] = u < tail ? xq[b * nl + 8 * nb + u] : 0.f;
  }
  // candidate positions staged in smem (dids doubles as the position buffer: row i's
  // slot is read before it is overwritten with the row's corpus id)
  {
    const int* cp = a.cand_pos + (size_t)q * a.take_cap;
    for (int i = tid; i < n; i += RNT) dids[i] = (uint32_t)cp[i];
  }
  __syncthreads();
  // U row groups per warp pass: all U rows' loads are issued before any math
  constexpr int U = UROWS;
  for (int row0 = warp * R * U; row0 < n; row0 += nwarps * R * U) {
    int rows[U], gps[U];
    float2 cbuf[U][SLOTS][kMaxNb];
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
      rows[uu] = row0 + uu * R + g;
      gps[uu] = (int)dids[rows[uu] < n ? rows[uu] : row0];
      const float* crow = ix.corpus + (size_t)gps[uu] * ds;
#pragma unroll
      for (int s = 0; s < SLOTS; ++s)
#pragma unroll
        for (int i = 0; i < kMaxNb; ++i)
          if (i < nb && rows[uu] - g < n)
            cbuf[uu][s][i] = __ldg(reinterpret_cast<const float2*>(crow + coff[s] + cstep * i));
    }
#pragma unroll
    for (int uu = 0; uu < U; ++uu) {
    if (rows[uu] - g >= n) break;  // whole lane group past the end (warp-uniform)
    const int row = rows[uu];
    const bool valid = row < n;
    const int gp = gps[uu];
    const float* crow = ix.corpus + (size_t)gp * ds;
    float slot_sum[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      const float2* c = cbuf[uu][s];
      float v;
      if (euclid) {
        float r0 = 0.f, r1 = 0.f;
#pragma unroll
        for (int i = 0; i < kMaxNb; ++i) {
          if (i < nb) {
            // packed FADD2/FMUL2 (per-lane IEEE rn, == __fsub_rn/__fmul_rn); the
            // accumulation stays scalar __fadd_rn so ptxas cannot contract it
            // into an FFMA2 (it does contract __fmul2_rn + __fadd2_rn).
            float2 dd = __fadd2_rn(c[i], make_float2(-xv[s][i].x, -xv[s][i].y));
            float2 sq = __fmul2_rn(dd, dd);
            r0 = i == 0 ? sq.x : __fadd_rn(r0, sq.x);
            r1 = i == 0 ? sq.y : __fadd_rn(r1, sq.y);
          }
        }
        v = __fadd_rn(r0, r1);
        v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 1));
        v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 2));
        if (tail) {
          const float* tp = crow + ctail[s];
#pragma unroll
          for (int u = 0; u < 7; ++u)
            if (u < tail) {
              float dd = __fsub_rn(__ldg(tp + u), xt[s][u]);
              v = __fadd_rn(v, __fmul_rn(dd, dd));
            }
        }
      } else {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < kMaxNb; ++i)
          if (i < nb) acc += c[i].x * xv[s][i].x + c[i].y * xv[s][i].y;
        if ((pl & 3) == 0) {
          const float* tp = crow + ctail[s];
          for (int u = 0; u < tail; ++u) acc += __ldg(tp + u) * xt[s][u];
        }
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        v = acc;
      }
      // perfect leaf tree inside the slot (lane groups of 4 = one leaf)
      for (int o = 4; o < G; o <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      slot_sum[s] = v;
    }
    float tot = slot_sum[0];
    if (SLOTS == 2) tot = __fadd_rn(slot_sum[0], slot_sum[1]);
    if (SLOTS == 4)
      tot = __fadd_rn(__fadd_rn(slot_sum[0], slot_sum[1]), __fadd_rn(slot_sum[2], slot_sum[3]));
    if (valid && pl == 0) {
      float diss = euclid ? tot : -tot;
      dkeys[row] = mono32(diss);
      dids[row] = __float_as_uint(__ldg(ix.pmeta + gp).w);  // corpus id (low 32 bits)
    }
    }
  }
  __syncthreads();
  const int kk = min(a.k, n);
  auto key = [&](int i) { return dkeys[i]; };
  auto tie = [&](int i) { return dids[i]; };
  auto val = [](uint32_t k) { return unmono32(k); };
  block_select_bucketed<RNT, uint32_t, float>(n, kk, key, tie, val, selidx, bs, sm);
  int np2 = 1;
  while (np2 < kk) np2 <<= 1;
  for (int i = tid; i < np2; i += RNT) {
    uint64_t v = ~0ull;
    if (i < kk) {
      int ci = selidx[i];
      v = ((uint64_t)dkeys[ci] << 32) | dids[ci];
    }
    srt[i] = v;
  }
  block_bitonic_sort<RNT>(srt, np2);
  const int gq = a.q0 + q;
  for (int i = tid; i < a.k; i += RNT) {
    int64_t id = -1;
    float sc = __int_as_float(0x7fc00000);
    if (i < kk) {
      uint64_t v = srt[i];
      id = (int64_t)(uint32_t)v;
      float df = unmono32((uint32_t)(v >> 32));
      sc = euclid ? df : -df;
    }
    a.out_ids[(size_t)gq * a.k + i] = id;
    a.out_scores[(size_t)gq * a.k + i] = sc;
  }
  if (tid == 0) a.out_count[gq] = kk;
}

// ================================================ rerank, TMA-fed variant
// Same arithmetic and lane layout as k_rerank_tree, but the candidate rows are
// brought into shared memory by the TMA bulk-copy engine (cp.async.bulk,
// one instruction per interleaved row, completion on a per-slot mbarrier)
// through an NBUF-deep ring per warp.  The register file no longer bounds the
// bytes in flight (k_rerank_tree: 2 rows per warp), and the LSU only serves
// conflict-free 256 B shared-memory reads.
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "RRG_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RRG_WAIT_%=;\n\t}" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes,
                                         uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::
          "r"(smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar))
      : "memory");
}

constexpr int kRingDepth = 3;  // 3 x 3 KB per warp at d=768: two 256-thread CTAs per SM

template <int SLOTS, int NB>
__global__ void __launch_bounds__(RNT, 2) k_rerank_tma(RerankArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  __shared__ __align__(8) uint64_t bars[RNT / 32][kRingDepth];
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = RNT / 32;
  const int d = ix.d, ds = ix.d_stride, nl = ix.pw_leaf_n, tail = nl % 8;
  constexpr int nb = NB;
  const int P = 4 * ix.pw_nleaves;
  const int G = SLOTS == 1 ? P : 32;
  const int R = 32 / G;
  const int g = lane / G, pl = lane % G;
  const int n = a.cand_n[q];
  const bool euclid = ix.metric == kMetricEuclidean;
  // smem: ring (128 B aligned) | dkeys[t] | dids[t] | selidx[k] | srt[np2]
  const int rstride = R > 1 ? ds + 8 : ds;  // +8 floats: conflict-free row groups
  const int unit_floats = R * rstride;
  float* ring = reinterpret_cast<float*>(smem_raw);
  float* myring = ring + (size_t)warp * kRingDepth * unit_floats;
  uint32_t* dkeys = reinterpret_cast<uint32_t*>(ring + (size_t)nwarps * kRingDepth * unit_floats);
  uint32_t* dids = dkeys + a.take_cap;
  int* selidx = reinterpret_cast<int*>(dids + a.take_cap);
  uintptr_t sp = reinterpret_cast<uintptr_t>(selidx + a.k);
  uint64_t* srt = reinterpret_cast<uint64_t*>((sp + 15) & ~uintptr_t(15));
  const float* xq = a.queries + (size_t)q * d;
  const int cstep = 8 * ix.pw_nleaves;
  float2 xv[SLOTS][nb];
  float xt[SLOTS][7];
  int coff[SLOTS], ctail[SLOTS];
#pragma unroll
  for (int s = 0; s < SLOTS; ++s) {
    int pair = pl + 32 * s;
    int b = pair >> 2, h = pair & 3;
    coff[s] = 8 * b + 2 * h;
    ctail[s] = nb * cstep + b * tail;
#pragma unroll
    for (int i = 0; i < nb; ++i) xv[s][i] = *reinterpret_cast<const float2*>(xq + b * nl + 2 * h + 8 * i);
#pragma unroll
    for (int u = 0; u < 7; ++u) xt[s][u] = u < tail ? xq[b * nl + 8 * nb + u] : 0.f;
  }
  {
    const int* cp = a.cand_pos + (size_t)q * a.take_cap;
    for (int i = tid; i < n; i += RNT) dids[i] = (uint32_t)cp[i];
  }
  if (lane == 0) {
    for (int k = 0; k < kRingDepth; ++k) mbar_init(&bars[warp][k], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  const uint32_t row_bytes = (uint32_t)ds * 4u;
  const int units = (n + R - 1) / R;
  auto issue = [&](int k) {  // lane 0: unit (warp + k*nwarps) -> ring slot k % depth
    const int u = warp + k * nwarps;
    if (u >= units) return;
    const int slot = k % kRingDepth;
    const int r0 = u * R, nr = min(R, n - r0);
    mbar_expect_tx(&bars[warp][slot], (uint32_t)nr * row_bytes);
    for (int r = 0; r < nr; ++r)
      bulk_g2s(myring + (size_t)slot * unit_floats + r * rstride,
               ix.corpus + (size_t)dids[r0 + r] * ds, row_bytes, &bars[warp][slot]);
  };
  if (lane == 0)
    for (int k = 0; k < kRingDepth; ++k) issue(k);
  for (int k = 0;; ++k) {
    const int u = warp + k * nwarps;
    if (u >= units) break;
    const int slot = k % kRingDepth;
    mbar_wait(&bars[warp][slot], (uint32_t)((k / kRingDepth) & 1));
    const int row = u * R + g;
    const bool valid = row < n;
    const float* crow = myring + (size_t)slot * unit_floats + g * rstride;
    const int gp = valid ? (int)dids[row] : 0;
    float slot_sum[SLOTS];
#pragma unroll
    for (int s = 0; s < SLOTS; ++s) {
      float v;
      if (euclid) {
        float r0 = 0.f, r1 = 0.f;
#pragma unroll
        for (int i = 0; i < nb; ++i) {
          float2 c = *reinterpret_cast<const float2*>(crow + coff[s] + cstep * i);
          float2 dd = __fadd2_rn(c, make_float2(-xv[s][i].x, -xv[s][i].y));
          float2 sq = __fmul2_rn(dd, dd);
          r0 = i == 0 ? sq.x : __fadd_rn(r0, sq.x);
          r1 = i == 0 ? sq.y : __fadd_rn(r1, sq.y);
        }
        v = __fadd_rn(r0, r1);
        v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 1));
        v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, 2));
        if (tail) {
          const float* tp = crow + ctail[s];
#pragma unroll
          for (int t = 0; t < 7; ++t)
            if (t < tail) {
              float dd = __fsub_rn(tp[t], xt[s][t]);
              v = __fadd_rn(v, __fmul_rn(dd, dd));
            }
        }
      } else {
        float acc = 0.f;
#pragma unroll
        for (int i = 0; i < nb; ++i) {
          float2 c = *reinterpret_cast<const float2*>(crow + coff[s] + cstep * i);
          acc += c.x * xv[s][i].x + c.y * xv[s][i].y;
        }
        if ((pl & 3) == 0)
          for (int t = 0; t < tail; ++t) acc += crow[ctail[s] + t] * xt[s][t];
        acc += __shfl_xor_sync(0xffffffffu, acc, 1);
        acc += __shfl_xor_sync(0xffffffffu, acc, 2);
        v = acc;
      }
      for (int o = 4; o < G; o <<= 1) v = __fadd_rn(v, __shfl_xor_sync(0xffffffffu, v, o));
      slot_sum[s] = v;
    }
    float tot = slot_sum[0];
    if (SLOTS == 2) tot = __fadd_rn(slot_sum[0], slot_sum[1]);
    __syncwarp();  // every lane is done with this ring slot
    if (valid && pl == 0) {
      float diss = euclid ? tot : -tot;
      dkeys[row] = mono32(diss);
      dids[row] = __float_as_uint(__ldg(ix.pmeta + gp).w);
    }
    if (lane == 0) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(k + kRingDepth);
    }
  }
  __syncthreads();
  const int kk = min(a.k, n);
  auto key = [&](int i) { return dkeys[i]; };
  auto tie = [&](int i) { return dids[i]; };
  auto val = [](uint32_t kv) { return unmono32(kv); };
  block_select_bucketed<RNT, uint32_t, float>(n, kk, key, tie, val, selidx, bs, sm);
  int np2 = 1;
  while (np2 < kk) np2 <<= 1;
  for (int i = tid; i < np2; i += RNT) {
    uint64_t v = ~0ull;
    if (i < kk) {
      int ci = selidx[i];
      v = ((uint64_t)dkeys[ci] << 32) | dids[ci];
    }
    srt[i] = v;
  }
  block_bitonic_sort<RNT>(srt, np2);
  const int gq = a.q0 + q;
  for (int i = tid; i < a.k; i += RNT) {
    int64_t id = -1;
    float sc = __int_as_float(0x7fc00000);
    if (i < kk) {
      uint64_t v = srt[i];
      id = (int64_t)(uint32_t)v;
      float df = unmono32((uint32_t)(v >> 32));
      sc = euclid ? df : -df;
    }
    a.out_ids[(size_t)gq * a.k + i] = id;
    a.out_scores[(size_t)gq * a.k + i] = sc;
  }
  if (tid == 0) a.out_count[gq] = kk;
}

// ======================================================== sharded merges
// One CTA per query: compact the G sources' valid entries into shared memory,
// select the `take` smallest by (key, id) and emit them sorted (the reference's
// lexsort order, index.py:315,320).  Exact for any G: a global top-t / top-k is
// always contained in the union of the per-shard top-t / top-k lists.
constexpr int MNT = 256;
__global__ void __launch_bounds__(MNT) k_merge(int mode, int metric, int nq, int G, int cap,
                                               const void* __restrict__ in_keys,
                                               const void* __restrict__ in_ids,
                                               const int* __restrict__ in_counts, int take,
                                               void* __restrict__ out_keys,
                                               void* __restrict__ out_ids,
                                               int* __restrict__ out_count) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  __shared__ int base[65];
  const int q = blockIdx.x, tid = threadIdx.x;
  const int ncap = G * cap;
  uint32_t* keys = reinterpret_cast<uint32_t*>(smem_raw);
  uint32_t* ids = keys + ncap;
  int* selidx = reinterpret_cast<int*>(ids + ncap);
  uintptr_t sp = reinterpret_cast<uintptr_t>(selidx + take);
  uint64_t* srt = reinterpret_cast<uint64_t*>((sp + 15) & ~uintptr_t(15));
  if (tid == 0) {
    int acc = 0;
    for (int g = 0; g < G; ++g) { base[g] = acc; acc += in_counts[(size_t)g * nq + q]; }
    base[G] = acc;
  }
  __syncthreads();
  const int n = base[G];
  if (mode == 1) {  // one contributing shard (every row of the w = 1 owner-local search):
                    // its result list is already sorted by (distance, id), copied as is
    int g1 = -1, nz = 0;
    for (int g = 0; g < G; ++g)
      if (base[g + 1] > base[g]) { g1 = g; ++nz; }
    if (nz <= 1 && n <= take) {
      const size_t src = ((size_t)(g1 < 0 ? 0 : g1) * nq + q) * cap;
      for (int i = tid; i < take; i += MNT) {
        const size_t o = (size_t)q * take + i;
        static_cast<float*>(out_keys)[o] =
            i < n ? static_cast<const float*>(in_keys)[src + i] : __int_as_float(0x7fc00000);
        static_cast<int64_t*>(out_ids)[o] = i < n ? static_cast<const int64_t*>(in_ids)[src + i] : -1;
      }
      if (tid == 0) out_count[q] = n;
      return;
    }
  }
  for (int g = 0; g < G; ++g) {
    const int c = base[g + 1] - base[g];
    const size_t src = ((size_t)g * nq + q) * cap;
    for (int i = tid; i < c; i += MNT) {
      uint32_t k, id;
      if (mode == 0) {
        k = static_cast<const uint32_t*>(in_keys)[src + i];
        id = static_cast<const uint32_t*>(in_ids)[src + i];
      } else {
        float s = static_cast<const float*>(in_keys)[src + i];
        k = mono32(metric == kMetricEuclidean ? s : -s);
        id = (uint32_t) static_cast<const int64_t*>(in_ids)[src + i];
      }
      keys[base[g] + i] = k;
      ids[base[g] + i] = id;
    }
  }
  __syncthreads();
  const int kk = min(take, n);
  auto key = [&](int i) { return keys[i]; };
  auto tie = [&](int i) { return ids[i]; };
  auto val = [](uint32_t k) { return unmono32(k); };
  block_select_bucketed<MNT, uint32_t, float>(n, kk, key, tie, val, selidx, bs, sm);
  int np2 = 1;
  while (np2 < kk) np2 <<= 1;
  for (int i = tid; i < np2; i += MNT) {
    uint64_t v = ~0ull;
    if (i < kk) v = ((uint64_t)keys[selidx[i]] << 32) | ids[selidx[i]];
    srt[i] = v;
  }
  block_bitonic_sort<MNT>(srt, np2);
  for (int i = tid; i < take; i += MNT) {
    const size_t o = (size_t)q * take + i;
    if (mode == 0) {
      static_cast<uint32_t*>(out_keys)[o] = i < kk ? (uint32_t)(srt[i] >> 32) : ~0u;
      static_cast<uint32_t*>(out_ids)[o] = i < kk ? (uint32_t)srt[i] : ~0u;
    } else {
      float sc = __int_as_float(0x7fc00000);
      int64_t id = -1;
      if (i < kk) {
        float df = unmono32((uint32_t)(srt[i] >> 32));
        sc = metric == kMetricEuclidean ? df : -df;
        id = (int64_t)(uint32_t)srt[i];
      }
      static_cast<float*>(out_keys)[o] = sc;
      static_cast<int64_t*>(out_ids)[o] = id;
    }
  }
  if (tid == 0) out_count[q] = kk;
}

// Warp per query: keep the candidates this shard holds, as positions.
__global__ void k_ids_to_pos(DevIndexView ix, int nq, int cap, const uint32_t* __restrict__ ids,
                             const int* __restrict__ counts, int* __restrict__ cand_pos,
                             int* __restrict__ cand_n) {
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (q >= nq) return;
  const int c = counts[q];
  int outn = 0;
  for (int b = 0; b < c; b += 32) {
    int i = b + lane;
    int p = -1;
    if (i < c) {
      uint32_t id = ids[(size_t)q * cap + i];
      p = id < (uint64_t)ix.m ? ix.pos_of_id[id] : -1;
    }
    unsigned m = __ballot_sync(0xffffffffu, p >= 0);
    if (p >= 0) cand_pos[(size_t)q * cap + outn + __popc(m & ((1u << lane) - 1))] = p;
    outn += __popc(m);
  }
  if (lane == 0) cand_n[q] = outn;
}

void launch_merge(int mode, int metric, int nq, int G, int cap, const void* in_keys,
                  const void* in_ids, const int* in_counts, int take, void* out_keys,
                  void* out_ids, int* out_count, cudaStream_t st) {
  size_t np2 = 1;
  while (np2 < (size_t)take) np2 <<= 1;
  size_t sm = (size_t)G * cap * 8 + (size_t)take * 4 + 16 + np2 * 8 + 16;
  static int done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, (const void*)k_merge);
    cudaFuncSetAttribute((const void*)k_merge, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxSmemPerCta - (int)at.sharedSizeBytes);
    done[dev] = 1;
  }
  (k_merge<<<nq, MNT, sm, st>>>(mode, metric, nq, G, cap, in_keys, in_ids, in_counts, take,
                               out_keys, out_ids, out_count), note_launch());
}

void launch_ids_to_pos(const DevIndexView& ix, int nq, int cap, const uint32_t* ids,
                       const int* counts, int* cand_pos, int* cand_n, cudaStream_t st) {
  (k_ids_to_pos<<<(nq + 7) / 8, 256, 0, st>>>(ix, nq, cap, ids, counts, cand_pos, cand_n), note_launch());
}

// ======================================================= corpus scatter
// dst[pos_of_id[i0 + i]] = src[i] for a chunk of file rows (original id order
// -> cluster order), rows padded to d_stride.
__global__ void k_scatter_rows(const float* __restrict__ src, int64_t nrows, int d, int d_stride,
                               const int* __restrict__ pos_of_id, int64_t i0,
                               const int* __restrict__ perm, float* __restrict__ dst) {
  int64_t row = blockIdx.x;
  if (row >= nrows) return;
  int p = pos_of_id[i0 + row];
  if (p < 0) return;  // row not held by this shard
  const float* s = src + row * (int64_t)d;
  float* t = dst + (int64_t)p * d_stride;
  for (int j = threadIdx.x; j < d_stride; j += blockDim.x) {
    if (j >= d) t[j] = 0.0f;
    else t[perm ? perm[j] : j] = s[j];  // element j -> its (interleaved) slot
  }
}

// ===================================================================== launchers
// One launch of k_gemm_dmma<EPI, BT, WM, BK> with its dynamic shared memory (opt-in
// above 48 KB done once per instantiation and device).
template <int EPI, bool BT, int WM, int BK>
static void gemm_launch(dim3 grid, cudaStream_t st, const float* A, int lda, const float* B, int ldb,
                        int M, int N, int K, float* outf, double* outd, int ldo, const double* rt,
                        const double* ct, int* outi = nullptr) {
  constexpr size_t sm = gemm_smem_bytes<WM, BK>();
  static int done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncSetAttribute((const void*)k_gemm_dmma<EPI, BT, WM, BK>,
                         cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    done[dev] = 1;
  }
  (k_gemm_dmma<EPI, BT, WM, BK><<<grid, 64 * WM, sm, st>>>(A, lda, B, ldb, M, N, K, outf, outd, ldo,
                                                          rt, ct, outi), note_launch());
}

// K depth per stage: 8 (default) or 16 (RRG_GEMM_BK=16) -- measured equal on C2
// (projection 0.175 ms, routing 0.203 vs 0.207 ms): the DMMA pipe, not the barriers, bounds it
// (RrgOpts.gemm_bk, resolved once per index)

void launch_project(const float* x, const float* W, int nq, int d, int s, float* xp, int bk,
                    cudaStream_t st) {
  dim3 grid((s + MBN - 1) / MBN, (nq + 32 * kGemmWM - 1) / (32 * kGemmWM));
  if (bk == 16)
    gemm_launch<EPI_PROJ, false, kGemmWM, 16>(grid, st, x, d, W, s, nq, s, d, xp, nullptr, s, nullptr, nullptr);
  else
    gemm_launch<EPI_PROJ, false, kGemmWM, 8>(grid, st, x, d, W, s, nq, s, d, xp, nullptr, s, nullptr, nullptr);
}

void launch_prep(const float* xp, const float* x, int nq, int s, int s_pad, int d, int8_t* qcodes,
                 float* qscale, float* qhead, double* pp, float* xx, cudaStream_t st,
                 int* nonfinite) {
  int warps_per_block = 8;
  int blocks = (nq + warps_per_block - 1) / warps_per_block;
  (k_prep_queries<<<blocks, warps_per_block * 32, 0, st>>>(xp, x, nq, s, s_pad, d, qcodes, qscale,
                                                          qhead, pp, xx, nonfinite), note_launch());
}

void launch_route_dist(const float* xp, const float* cent, int nq, int L, int s, int metric,
                       const double* pp, const double* cnorm, double* diss, int bk, cudaStream_t st) {
  constexpr int WM = 4;  // C2: 128x64 tiles measured 0.214 ms vs 96x64 0.220 ms
  dim3 grid((L + MBN - 1) / MBN, (nq + 32 * WM - 1) / (32 * WM));
  const bool bk16 = bk == 16;
  if (metric == kMetricEuclidean) {
    if (bk16) gemm_launch<EPI_L2, true, WM, 16>(grid, st, xp, s, cent, s, nq, L, s, nullptr, diss, L, pp, cnorm);
    else gemm_launch<EPI_L2, true, WM, 8>(grid, st, xp, s, cent, s, nq, L, s, nullptr, diss, L, pp, cnorm);
  } else {
    if (bk16) gemm_launch<EPI_NEGIP, true, WM, 16>(grid, st, xp, s, cent, s, nq, L, s, nullptr, diss, L, nullptr, nullptr);
    else gemm_launch<EPI_NEGIP, true, WM, 8>(grid, st, xp, s, cent, s, nq, L, s, nullptr, diss, L, nullptr, nullptr);
  }
}

void launch_gt_dist(const float* q, int M, const float* c, int N, int d, int metric,
                    const double* qq, const double* cterm, double* out, int64_t ldo, cudaStream_t st) {
  constexpr int WM = 4;
  dim3 grid((N + MBN - 1) / MBN, (M + 32 * WM - 1) / (32 * WM));
  if (metric == kMetricEuclidean)
    gemm_launch<EPI_GT_L2, true, WM, 16>(grid, st, q, d, c, d, M, N, d, nullptr, out, (int)ldo, qq, cterm);
  else if (metric == kMetricIp)
    gemm_launch<EPI_NEGIP, true, WM, 16>(grid, st, q, d, c, d, M, N, d, nullptr, out, (int)ldo, nullptr, nullptr);
  else
    gemm_launch<EPI_GT_COS, true, WM, 16>(grid, st, q, d, c, d, M, N, d, nullptr, out, (int)ldo, nullptr, cterm);
}

// Opt in to the dynamic shared memory a launch may need (227 KB per CTA minus the
// kernel's static shared memory), once per kernel slot and device.
template <typename Kern>
static void allow_smem(Kern* kernel, int slot) {
  static int done[32][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[slot][dev]) return;
  cudaFuncAttributes at{};
  cudaFuncGetAttributes(&at, (const void*)kernel);
  cudaFuncSetAttribute((const void*)kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kMaxSmemPerCta - (int)at.sharedSizeBytes);
  done[slot][dev] = 1;
}

size_t route_select_smem(int L) { return (size_t)L * 8 + (size_t)L * 4 + 16; }

// w == 1 from the fused GEMM's per-tile partials: min over ntiles (dissimilarity,
// column) pairs per query; tiles ascend in column, so ties keep the lowest id.
__global__ void k_route_nearest_partials(const double* __restrict__ pv, const int* __restrict__ pi,
                                         int nq, int ntiles, int* __restrict__ sel,
                                         int* __restrict__ primary) {
  const int q = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  double bk = __longlong_as_double(0x7ff0000000000000ll);
  int bi = 0x7fffffff;
  for (int t = lane; t < ntiles; t += 32) {
    const double v = __ldg(pv + (size_t)q * ntiles + t);
    const int c = __ldg(pi + (size_t)q * ntiles + t);
    if (v < bk || (v == bk && c < bi)) { bk = v; bi = c; }
  }
  for (int o = 16; o > 0; o >>= 1) {
    const double ob = __shfl_xor_sync(0xffffffffu, bk, o);
    const int oi = __shfl_xor_sync(0xffffffffu, bi, o);
    if (ob < bk || (ob == bk && oi < bi)) { bk = ob; bi = oi; }
  }
  if (bi == 0x7fffffff) bi = 0;  // defensive: every partial was unordered
  if (lane == 0) { sel[q] = bi; primary[q] = bi; }
}

int route_nearest_tiles(int L) { return (L + MBN - 1) / MBN; }

// 1 < w <= 8: the w nearest of a query from its per-tile sorted top-TW partials (warp per
// query: each lane merges its tiles' lists into a sorted top-TW, then w rounds of a warp
// argmin by (dissimilarity, column) -- route()'s stable argsort order)
template <int TW>
__global__ void k_route_topw_partials(const double* __restrict__ part_v, const int* __restrict__ part_i, int nq,
                                      int nt, int w, int* __restrict__ sel, int* __restrict__ primary) {
  const int q = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  constexpr double kInfD = __builtin_huge_val();
  double v[TW];
  int c[TW];
#pragma unroll
  for (int t = 0; t < TW; ++t) { v[t] = kInfD; c[t] = 0x7fffffff; }
  for (int tile = lane; tile < nt; tile += 32) {
    const size_t b = ((size_t)q * nt + tile) * TW;
#pragma unroll
    for (int k = 0; k < TW; ++k) {
      double x = __ldg(part_v + b + k);
      int xi = __ldg(part_i + b + k);
      if (xi == 0x7fffffff) continue;
      bool in = false;
#pragma unroll
      for (int t = 0; t < TW; ++t)
        if (in || x < v[t] || (x == v[t] && xi < c[t])) {
          const double tv = v[t]; const int tc = c[t];
          v[t] = x; c[t] = xi; x = tv; xi = tc; in = true;
        }
    }
  }
  for (int r = 0; r < w; ++r) {
    double b = v[0];
    int bc = c[0];
    for (int o = 16; o > 0; o >>= 1) {
      const double ob = __shfl_xor_sync(0xffffffffu, b, o);
      const int oc = __shfl_xor_sync(0xffffffffu, bc, o);
      if (ob < b || (ob == b && oc < bc)) { b = ob; bc = oc; }
    }
    if (c[0] == bc) {
#pragma unroll
      for (int t = 0; t + 1 < TW; ++t) { v[t] = v[t + 1]; c[t] = c[t + 1]; }
      v[TW - 1] = kInfD; c[TW - 1] = 0x7fffffff;
    }
    if (lane == 0) {
      sel[(size_t)q * w + r] = bc == 0x7fffffff ? 0 : bc;
      if (r == 0) primary[q] = bc == 0x7fffffff ? 0 : bc;
    }
  }
}

void launch_route_topw_fused(const float* xp, const float* cent, int nq, int L, int s, int w, const double* pp,
                             const double* cnorm, double* part_v, int* part_i, cudaStream_t st) {
  constexpr int WM = 4;
  const int nt = route_nearest_tiles(L);
  dim3 grid(nt, (nq + 32 * WM - 1) / (32 * WM));
  if (w <= 4)
    gemm_launch<EPI_L2_TOP4, true, WM, 8>(grid, st, xp, s, cent, s, nq, L, s, nullptr, part_v, nt, pp, cnorm,
                                          part_i);
  else
    gemm_launch<EPI_L2_TOP8, true, WM, 8>(grid, st, xp, s, cent, s, nq, L, s, nullptr, part_v, nt, pp, cnorm,
                                          part_i);
}

void launch_route_topw_reduce(const double* part_v, const int* part_i, int nq, int L, int w, int* sel,
                              int* primary, cudaStream_t st) {
  const int nt = route_nearest_tiles(L);
  if (w <= 4)
    (k_route_topw_partials<4><<<(nq + 7) / 8, 256, 0, st>>>(part_v, part_i, nq, nt, w, sel, primary),
     note_launch());
  else
    (k_route_topw_partials<8><<<(nq + 7) / 8, 256, 0, st>>>(part_v, part_i, nq, nt, w, sel, primary),
     note_launch());
}

void launch_route_nearest_fused(const float* xp, const float* cent, int nq, int L, int s, int metric,
                                const double* pp, const double* cnorm, double* part_v, int* part_i,
                                cudaStream_t st) {
  constexpr int WM = 4;
  const int nt = route_nearest_tiles(L);
  dim3 grid(nt, (nq + 32 * WM - 1) / (32 * WM));
  if (metric == kMetricEuclidean)
    gemm_launch<EPI_L2_ARGMIN, true, WM, 8>(grid, st, xp, s, cent, s, nq, L, s, nullptr, part_v, nt,
                                            pp, cnorm, part_i);
  else
    gemm_launch<EPI_NEGIP_ARGMIN, true, WM, 8>(grid, st, xp, s, cent, s, nq, L, s, nullptr, part_v, nt,
                                               nullptr, nullptr, part_i);
}

void launch_route_nearest_reduce(const double* part_v, const int* part_i, int nq, int L, int* sel,
                                 int* primary, cudaStream_t st) {
  (k_route_nearest_partials<<<(nq + 7) / 8, 256, 0, st>>>(part_v, part_i, nq, route_nearest_tiles(L),
                                                         sel, primary), note_launch());
}

void launch_route_select(const double* diss, int nq, int L, int w, int* sel, int* primary,
                         cudaStream_t st) {
  if (w == 1) {
    (k_route_nearest<<<(nq + 7) / 8, 256, 0, st>>>(diss, nq, L, sel, primary), note_launch());
    return;
  }
  if (w <= 8 && L >= w) {
    (k_route_select_warp<8><<<(nq + 7) / 8, 256, 0, st>>>(diss, nq, L, w, sel, primary), note_launch());
    return;
  }
  allow_smem(k_route_select<256>, 0);
  (k_route_select<256><<<nq, 256, route_select_smem(L), st>>>(diss, L, w, sel, primary), note_launch());
}

void launch_bucket(const int* primary, int nq, int L, int* order, cudaStream_t st) {
  allow_smem(k_bucket_queries, 1);
  static int bdone[64] = {};
  int bdev = 0;
  cudaGetDevice(&bdev);
  if (bdev >= 0 && bdev < 64 && !bdone[bdev]) {  // (L + 1) * 4 bytes: past 48 KB above L = 12k
    cudaFuncSetAttribute((const void*)k_bucket_queries, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxSmemPerCta - 1024);
    bdone[bdev] = 1;
  }
  (k_bucket_queries<<<1, BNT, (size_t)(L + 1) * 4, st>>>(primary, nq, L, order), note_launch());
}

size_t score_select_smem(int smem_cap, int take_cap, int k) {
  size_t np2 = 1;
  while (np2 < (size_t)k) np2 <<= 1;
  return (size_t)smem_cap * 8 + (size_t)take_cap * 4 + 32 + np2 * 8 + 16;
}

void launch_score_select(const ScoreArgsHost& h, int nq, cudaStream_t st) {
  ScoreArgs a;
  a.ix = h.ix; a.qcodes = h.qcodes; a.qscale = h.qscale; a.qhead = h.qhead; a.xx = h.xx;
  a.sel = h.sel; a.w = h.w; a.take_cap = h.take_cap; a.rerank = h.rerank; a.k = h.k;
  a.smem_cap = h.smem_cap; a.gkeys = h.gkeys; a.gpos = h.gpos; a.gcap = h.gcap;
  a.cand_pos = h.cand_pos; a.cand_n = h.cand_n; a.out_ids = h.out_ids;
  a.out_scores = h.out_scores; a.out_count = h.out_count; a.q0 = h.q0;
  a.order = h.order;
  a.sel_keys = h.sel_keys; a.sel_ids = h.sel_ids; a.sel_count = h.sel_count;
  allow_smem(k_score_select, 2);
  (k_score_select<<<nq, SNT, score_select_smem(h.smem_cap, h.take_cap, h.k), st>>>(a), note_launch());
}

size_t rerank_smem(int d_stride, int take_cap, int k, bool tree) {
  size_t np2 = 1;
  while (np2 < (size_t)k) np2 <<= 1;
  size_t rows = tree ? 0 : (size_t)d_stride * 4 * (1 + RNT / 32);
  return rows + (size_t)take_cap * 8 + (size_t)k * 4 + 16 + np2 * 8 + 16;
}

bool rerank_uses_tree(const DevIndexView& ix) { return ix.corpus_interleaved != 0; }

void launch_rerank(const RerankArgsHost& h, int nq, cudaStream_t st) {
  RerankArgs a;
  a.ix = h.ix; a.queries = h.queries; a.cand_pos = h.cand_pos; a.cand_n = h.cand_n;
  a.take_cap = h.take_cap; a.k = h.k; a.out_ids = h.out_ids; a.out_scores = h.out_scores;
  a.out_count = h.out_count; a.q0 = h.q0; a.order = h.order;
  const bool tree = rerank_uses_tree(h.ix);
  const size_t sm = rerank_smem(h.ix.d_stride, h.take_cap, h.k, tree);

  // default: the register-pipelined k_rerank_tree (measured faster on C2 than the
  // TMA ring, whose mbarrier polling costs issue slots); RRG_RERANK=tma opts in
  const bool use_tma = h.ix.opt.rerank == 4;
  if (tree && use_tma) {
    const int nb = h.ix.pw_leaf_n / 8;
    const bool one = 4 * h.ix.pw_nleaves <= 32;
    const int G = one ? 4 * h.ix.pw_nleaves : 32, R = 32 / G;
    const int rstride = R > 1 ? h.ix.d_stride + 8 : h.ix.d_stride;
    const size_t ring = (size_t)(RNT / 32) * kRingDepth * R * rstride * 4;
    const size_t smt = ring + rerank_smem(h.ix.d_stride, h.take_cap, h.k, true);
#define RRG_TMA(S, NBV, SLOT)                           \
  do {                                                  \
    allow_smem(k_rerank_tma<S, NBV>, SLOT);             \
    (k_rerank_tma<S, NBV><<<nq, RNT, smt, st>>>(a), note_launch());      \
  } while (0)
    bool launched = true;
    if (one) {
      switch (nb) {
        case 8: RRG_TMA(1, 8, 12); break;
        case 12: RRG_TMA(1, 12, 13); break;
        case 15: RRG_TMA(1, 15, 14); break;
        case 16: RRG_TMA(1, 16, 15); break;
        default: launched = false;
      }
    } else {
      switch (nb) {
        case 12: RRG_TMA(2, 12, 16); break;
        case 16: RRG_TMA(2, 16, 17); break;
        default: launched = false;
      }
    }
#undef RRG_TMA
    if (launched) return;
  }
  if (tree) {
    const int nb = h.ix.pw_leaf_n / 8;
    const bool one = 4 * h.ix.pw_nleaves <= 32;
#define RRG_TREE(S, NBV, NLVV, SLOT)                    \
  do {                                                  \
    allow_smem(k_rerank_tree<S, NBV, NLVV>, SLOT);      \
    (k_rerank_tree<S, NBV, NLVV><<<nq, RNT, sm, st>>>(a), note_launch()); \
  } while (0)
    // specialised (chain length, leaf count) of the common dims:
    //   d=768 (8 leaves of 96), 960 (8 x 120), 1536 (16 x 96), 1024 (8 x 128),
    //   512/256/128 (4/2/1 x 128), 100 (1 x 100)
    const int key = nb * 100 + h.ix.pw_nleaves;
    switch (key) {
      case 1208: RRG_TREE(1, 12, 8, 18); break;
      case 1508: RRG_TREE(1, 15, 8, 19); break;
      case 1608: RRG_TREE(1, 16, 8, 20); break;
      case 1604: RRG_TREE(1, 16, 4, 21); break;
      case 1602: RRG_TREE(1, 16, 2, 22); break;
      case 1601: RRG_TREE(1, 16, 1, 23); break;
      case 1201: RRG_TREE(1, 12, 1, 24); break;
      case 1216: RRG_TREE(2, 12, 16, 25); break;
      case 1616: RRG_TREE(2, 16, 16, 26); break;
      default:
        if (one) {
          switch (nb) {
            case 8: RRG_TREE(1, 8, 0, 6); break;
            case 12: RRG_TREE(1, 12, 0, 7); break;
            case 15: RRG_TREE(1, 15, 0, 8); break;
            case 16: RRG_TREE(1, 16, 0, 9); break;
            default: RRG_TREE(1, 0, 0, 3); break;
          }
        } else {
          switch (nb) {
            case 12: RRG_TREE(2, 12, 0, 10); break;
            case 16: RRG_TREE(2, 16, 0, 11); break;
            default: RRG_TREE(2, 0, 0, 4); break;
          }
        }
    }
#undef RRG_TREE
    return;
  }
  allow_smem(k_rerank_topk, 5);
  (k_rerank_topk<<<nq, RNT, sm, st>>>(a), note_launch());
}

void launch_scatter_rows(const float* src, int64_t nrows, int d, int d_stride,
                         const int* pos_of_id, int64_t i0, const int* perm, float* dst,
                         cudaStream_t st) {
  if (nrows <= 0) return;
  (k_scatter_rows<<<(unsigned)nrows, 128, 0, st>>>(src, nrows, d, d_stride, pos_of_id, i0, perm,
                                                  dst), note_launch());
}

}  // namespace rrg
