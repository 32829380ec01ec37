// rrg_common.cuh -- shared device-side definitions of the B200 LoRANN query engine.
//
// Exact-arithmetic rules restated from the reference:
//  * quantize_vector (quantize.py:61-77): scale = rn_f32(127 / absmax) (f64 quotient
//    rounded once == __fdiv_rn for f32 operands), products in f64 (exact), round half
//    away from zero, clip to +-127;
//  * dequantize_product (quantize.py:129-136): rn(rn(f32(raw) / rn(scale*cs)) + rn(head*hr)),
//    never FMA-contracted (every op below is an explicit __f*_rn intrinsic);
//  * ordering keys: ascending (key, corpus id), -0.0 == +0.0 (np.lexsort, index.py:315,320).
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

namespace rrg {

constexpr int kMetricEuclidean = 0;
constexpr int kMetricIp = 1;
constexpr int kMetricCosine = 2;

constexpr int kKindRrr = 0;    // two-stage A/B model (rrr.py:181-203)
constexpr int kKindExact = 1;  // single-factor exact model (rrr.py:103-113, index.py:465-468)

// Search-variant switches (A/B measurement and test coverage of every kernel
// variant), read from the environment once per index -- at rrg_index_open /
// rrg_index_create and on rrg_index_reload_options -- never per search call.
struct RrgOpts {
  int proj_sliced;   // RRG_GEMM / RRG_PROJ = sliced|dmma (default sliced)
  int route_sliced;  // RRG_GEMM / RRG_ROUTE = sliced|dmma (default dmma)
  int route_fused;   // RRG_ROUTE_FUSED (default 1): w = 1 argmin fused into the GEMM
  int gemm_bk;       // RRG_GEMM_BK = 8|16: K depth per DMMA stage
  int score_query;   // RRG_SCORE_MODE=query: fused query-major scoring
  int rerank;        // RRG_RERANK: 0 auto, 1 cluster, 2 query, 3 regs, 4 tma
  int rr_skip;       // RRG_RR_SKIP: -1 auto, 0 off, 1 on
  int rr_async;      // RRG_RR_ASYNC: cp.async row staging in the cluster re-rank
  int warp_select;   // RRG_WARP_SELECT: -1 auto, 0 CTA per query, 1 warp per query
  int host_pieces;   // RRG_HOST_PIECES: 0 auto
  int graph;         // RRG_GRAPH: captured graphs for small host batches (default 1)
  int screen;        // RRG_SCREEN: -1 auto, 0 off, 1 on (tensor-core re-rank screen)
  int score_stage_a;  // RRG_SCORE_STAGE_A (default 1): K4 stage-A operands staged in shared memory
  int rr_order;       // RRG_RR_ORDER (default 1): sparse re-rank items largest cluster first
  int score_order;    // RRG_SCORE_ORDER (default 1): scoring items largest cluster first
  int route_screen;  // RRG_ROUTE_SCREEN: fp16 tensor-core routing bounds + f64 recheck (0 off, 1 at w = 1, 2 at any w <= 8)
  int screen_diag;   // RRG_SCREEN_DIAG: timing probes of k_rr_screen (1: no MMAs, 2: no MMAs or bounds)
  int score_tc;      // RRG_SCORE_TC: stage B of the cluster scoring on tcgen05 (kind::i8): -1 auto
  int sparse_variant;  // RRG_SPARSE_VARIANT: k_rerank_sparse 0 register prefetch / 1 more CTAs
  int screen_stages;   // RRG_SCREEN_STAGES: ring depth of k_rr_screen (0: as much as fits)
};

// POD view of a device-resident index, passed by value to kernels.
// Counts one kernel launch of this thread (rrg_last_launch_count; rrg_api.cu).
void note_launch();

struct DevIndexView {
  int metric, d, s, r, L;
  int s_pad;     // s rounded up to 16 (query / exact codes row pitch, bytes)
  int r_pad;     // r rounded up to 16 (B^T row pitch, bytes)
  int d_stride;  // corpus row pitch in floats (d rounded up to 4)
  int64_t P;     // points held (== m for an unsharded index)
  const float* W;        // d x s
  const float* cent;     // L x s
  const double* cnorm;   // L: (c*c).sum(axis=1) in f64, NumPy pairwise order
  const int* cl_pos;     // L+1: first global position of each cluster (cluster order)
  const int* cl_order;   // L: clusters by held size, largest first (sparse re-rank items)
  const int* cl_kind;    // L
  const int* cl_aidx;    // L: rrr -> model slot in at/ahead/ascale; exact -> row in xcodes
  const int8_t* at;      // [n_rrr][r][s_pad]: A^T codes, row 0 of A (pad) kept as column 0
  const float* ahead;    // [n_rrr][r]
  const float* ascale;   // [n_rrr][r]
  const int8_t* bt;      // [P][r_pad]: B^T codes per point, column 0 = pad row (zero)
  const int8_t* xcodes;  // [P_exact][s_pad]: exact-model codes per point
  // [P] per-point {head_row, col_scale} of the point's last factor (B, or A for an
  // exact model), ||c_p||^2 (euclidean, else 0) and the low 32 bits of its corpus id:
  // one 16-byte load per scored point.
  const float4* pmeta;
  const int64_t* pid;    // [P] original corpus ids
  const float* corpus;   // [P][d_stride] in cluster order, or nullptr
  const int* pos_of_id;  // [m] corpus id -> position held here, -1 if another shard's
  int64_t m;             // corpus size (all shards)
  // NumPy pairwise-summation plan for a row of d floats: when the recursion
  // tree is perfect (2^a equal leaves of pw_leaf_n <= 128 elements, e.g. d = 128,
  // 768, 960, 1536) the re-rank runs the warp-parallel kernel.
  int pw_nleaves, pw_leaf_n, pw_perfect;
  // corpus_interleaved: rows are stored step-major for the perfect pairwise plan
  // (element (leaf b, step i, accumulator j) at i*8*nleaves + 8*b + j, the nl%8
  // tails after all steps), so one warp instruction of the re-rank reads 256
  // contiguous bytes instead of eight 32-byte pieces of the natural layout.
  int corpus_interleaved;
  const int* elem_perm;  // [d] natural element -> interleaved slot (when interleaved)
  // unquantized index (quantize=False, rrr.py:97-100): f32 factors in the layouts of
  // at / bt / xcodes (pitches s_pad / r_pad elements); nullptr when quantized
  int quantized;
  const float* atf;  // [n_rrr][r][s_pad]
  const float* btf;  // [P][r_pad]
  const float* xf;   // [P_exact][s_pad]
  // W^T as 8 tiled int8 slice planes + per-row exponents (rrg_sliced_gemm.cu): the
  // tensor-core projection (RRG_PROJ=sliced)
  const float* Wt;  // W^T (s x d) f32, for the small-batch GEMV projection
  const int8_t* wt_planes;
  const int* wt_exps;
  const int8_t* cent_planes;  // centroids (L x s), same slicing, for the routing GEMM
  const int* cent_exps;
  // re-rank screen (rrg_screen.cu, euclidean indexes with a corpus; nullptr otherwise):
  // residual rows r = c - mu_l as fp16 (x 2^-e_row), pre-tiled per 128-row block in the
  // UMMA K-major layout, with the exact residual norms the error bound needs
  const uint16_t* scr_plane;  // [blocks][scr_kc][128 rows x 16 fp16]
  const int* scr_blk0;        // [L+1] first block of each cluster (clusters padded to 128 rows)
  const float* scr_mu;        // [L][d] per-cluster mean (natural element order)
  const double* scr_rr;       // [P] ||c - mu||^2 (f64)
  const float4* scr_rmeta;    // [P] {||r_hat||, ||r - r_hat||, 2^e_row, 0} (scaled units, rounded up)
  int scr_kc;                 // K chunks of 16 elements: ceil(d / 16)
  // routing screen (rrg_route_screen.cu): centroids as fp16 tiles (x 2^-e per row)
  const uint16_t* rt_cent_tiles;  // [ceil(L/128)][rt_kc][128 rows x 16 fp16]
  const float4* rt_cent_stats;    // [L_pad] {||c^||, ||c/2^e - c^||, e, 0}
  int rt_kc;                      // ceil(s / 16)
  RrgOpts opt;
};

// ---------------------------------------------------------------- numerics

__device__ __forceinline__ float deq(int raw, float xscale, float cs, float head, float hr) {
  // quantize.py:136 with head_contrib = F32(head) * head_row (quantize.py:153)
  float den = __fmul_rn(xscale, cs);
  float q = __fdiv_rn(__int2float_rn(raw), den);
  return __fadd_rn(q, __fmul_rn(head, hr));
}

__device__ __forceinline__ float quant_scale(float absmax) {
  return absmax == 0.0f ? 1.0f : __fdiv_rn(127.0f, absmax);
}

__device__ __forceinline__ int quant_code(float v, float scale) {
  // _round_half_away(f64(v) * f64(scale)), clip +-127 (quantize.py:28-29,75-76)
  double p = __dmul_rn((double)v, (double)scale);
  double a = floor(__dadd_rn(fabs(p), 0.5));
  int c = (int)a;
  c = c > 127 ? 127 : c;
  return p < 0.0 ? -c : c;
}

// Packed exact square rn(d*d) per half.  ptxas contracts mul.rn.f32x2 + add.rn.f32x2
// into FFMA2 (even with --fmad=false), which would break NumPy's square-then-add
// rounding; fma(d, d, -0) rounds d*d once and is bit-identical to the product, and
// with nz read from a kernel argument (opaque -0.0) ptxas has nothing to fold, so
// the following packed accumulation stays a separate FADD2.
__device__ __forceinline__ float2 sq2(float2 d, float2 nz) { return __ffma2_rn(d, d, nz); }

// Monotone maps so unsigned integer order == float order, with -0.0 == +0.0.
__device__ __forceinline__ uint32_t mono32(float f) {
  uint32_t u = __float_as_uint(f);
  if (u == 0x80000000u) u = 0u;
  return (u & 0x80000000u) ? ~u : (u | 0x80000000u);
}
__device__ __forceinline__ float unmono32(uint32_t k) {
  uint32_t u = (k & 0x80000000u) ? (k & 0x7fffffffu) : ~k;
  return __uint_as_float(u);
}
__device__ __forceinline__ double unmono64(uint64_t k) {
  uint64_t u = (k & 0x8000000000000000ull) ? (k & 0x7fffffffffffffffull) : ~k;
  return __longlong_as_double((long long)u);
}
__device__ __forceinline__ uint64_t mono64(double f) {
  uint64_t u = (uint64_t)__double_as_longlong(f);
  if (u == 0x8000000000000000ull) u = 0ull;
  return (u & 0x8000000000000000ull) ? ~u : (u | 0x8000000000000000ull);
}

// ---------------------------------------------------- NumPy pairwise summation
// NumPy's pairwise_sum (the loop behind `sum(axis=-1)` on a contiguous row):
//   n < 8     : sequential from 0
//   n <= 128  : 8 strided accumulators, tree ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)),
//               then the n%8 tail sequentially
//   else      : n2 = n/2 - (n/2)%8; pw(a[:n2]) + pw(a[n2:])
// Restated (and pinned against NumPy) in oracle/rrann_oracle.py:pairwise_sum_f32.
template <typename T, typename Get>
__device__ T pw_leaf(Get get, int start, int n) {
  if (n < 8) {
    T res = (T)0;
    for (int i = 0; i < n; ++i) res = res + get(start + i);
    return res;
  }
  T r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = get(start + j);
  int i = 8;
  for (; i < n - (n % 8); i += 8) {
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = r[j] + get(start + i + j);
  }
  T res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
  for (; i < n; ++i) res = res + get(start + i);
  return res;
}

// Warp evaluation of the same tree when it is perfect and narrow: n = m * 2^a with leaf
// size m <= 128, m % 8 == 0 (every split halves exactly) and 8 * 2^a <= 32 chains.
// Lane c runs chain c % 8 of leaf c / 8 in NumPy's order; xor-shuffles 1, 2, 4 then form
// ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) and 8, 16 the leaf tree (a+b == b+a exactly, so
// both lanes of a pair hold the same bits).  Every lane returns the sum.
__host__ __device__ inline int pw_warp_leaves(int n) {
  if (n < 8 || n % 8) return 0;
  int L = 1;
  while (n / L > 128) {
    if ((n / L) % 16) return 0;  // the halves must stay multiples of 8
    L *= 2;
  }
  return L <= 4 ? L : 0;
}
template <typename T, typename Get>
__device__ T pw_sum_warp(Get get, int n, int L, int lane) {
  const int m = n / L, c = lane & (8 * L - 1) , leaf = c >> 3, j = c & 7;
  T r = get(leaf * m + j);
  for (int i = 8; i < m; i += 8) r = r + get(leaf * m + i + j);
  for (int o = 1; o < 8 * L; o <<= 1) r = r + __shfl_xor_sync(0xffffffffu, r, o);
  return r;
}

// Single-thread iterative evaluation of the full tree (used for short rows and
// for ||p||^2 of the routing expansion).  The explicit stack mirrors the
// recursion; depth <= 32.
template <typename T, typename Get>
__device__ T pw_sum_seq(Get get, int n) {
  if (n <= 128) return pw_leaf<T>(get, 0, n);
  int st_start[32], st_n[32], st_state[32];
  T st_left[32];
  int sp = 0;
  st_start[0] = 0; st_n[0] = n; st_state[0] = 0;
  T ret = (T)0;
  while (sp >= 0) {
    int s0 = st_start[sp], nn = st_n[sp];
    if (nn <= 128) {
      ret = pw_leaf<T>(get, s0, nn);
      --sp;
      // deliver ret to parent
      while (sp >= 0) {
        if (st_state[sp] == 1) {  // left done -> start right
          st_left[sp] = ret;
          st_state[sp] = 2;
          int n2 = st_n[sp] / 2; n2 -= n2 % 8;
          ++sp;
          st_start[sp] = st_start[sp - 1] + n2; st_n[sp] = st_n[sp - 1] - n2; st_state[sp] = 0;
          break;
        } else {  // right done
          ret = st_left[sp] + ret;
          --sp;
        }
      }
      continue;
    }
    if (st_state[sp] == 0) {
      st_state[sp] = 1;
      int n2 = nn / 2; n2 -= n2 % 8;
      ++sp;
      st_start[sp] = s0; st_n[sp] = n2; st_state[sp] = 0;
    }
  }
  return ret;
}

// ---------------------------------------------------- block-wide selection
// Select the `take` smallest items of n by (key, tie) -- ties broken by the
// (unique) tie value -- and write their item indices (unordered) to out[].
// MSB-first radix select with 8-bit digits over the key, then, only when the
// boundary key value is shared by more items than remain to be taken, a second
// radix select over the tie values of the boundary-equal items.
struct SelectSmem {
  int hist[256];
  int count;
  int dg;
  int before;
  int eq;
};

template <typename K>
struct SelState {
  K prefix, mask;
  int rank;
};

__device__ __forceinline__ void warp_agg_add(int* hist, int bin, bool active) {
  unsigned am = __ballot_sync(0xffffffffu, active);
  if (!active) return;
  unsigned peers = __match_any_sync(am, bin);
  int leader = __ffs(peers) - 1;
  if ((threadIdx.x & 31) == leader) atomicAdd(&hist[bin], __popc(peers));
}

// One radix pass: find the digit holding the rank-th element among items whose
// masked key equals prefix.  Called by all threads.
template <int NT, typename K, typename KeyF, typename PredF>
__device__ void radix_pass(int n, KeyF key, PredF pred, SelState<K>& st, int shift,
                           SelectSmem& sm) {
  for (int i = threadIdx.x; i < 256; i += NT) sm.hist[i] = 0;
  __syncthreads();
  for (int base = 0; base < n; base += NT) {
    int i = base + threadIdx.x;
    bool act = false;
    int bin = 0;
    if (i < n && pred(i)) {
      K k = key(i);
      if ((k & st.mask) == st.prefix) {
        act = true;
        bin = (int)((k >> shift) & (K)255);
      }
    }
    warp_agg_add(sm.hist, bin, act);
  }
  __syncthreads();
  if (threadIdx.x < 32) {
    int lane = threadIdx.x;
    int h[8];
    int tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { h[j] = sm.hist[lane * 8 + j]; tot += h[j]; }
    int incl = tot;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    int excl = incl - tot;
    bool mine = excl < st.rank && st.rank <= incl;
    unsigned b = __ballot_sync(0xffffffffu, mine);
    if (mine) {
      int cum = excl;
      int j = 0;
      for (; j < 8; ++j) {
        if (cum + h[j] >= st.rank) break;
        cum += h[j];
      }
      sm.dg = lane * 8 + j;
      sm.before = cum;
      sm.eq = h[j];
    }
    (void)b;
  }
  __syncthreads();
  st.rank -= sm.before;
  st.prefix |= ((K)sm.dg) << shift;
  st.mask |= ((K)255) << shift;
  __syncthreads();
}

template <int NT, typename K, typename KeyF, typename TieF>
__device__ int block_select_smallest(int n, int take, KeyF key, TieF tie, int* out,
                                     SelectSmem& sm) {
  if (threadIdx.x == 0) sm.count = 0;
  __syncthreads();
  if (take >= n) {
    for (int i = threadIdx.x; i < n; i += NT) out[i] = i;
    __syncthreads();
    return n;
  }
  if (take <= 0) return 0;
  SelState<K> st{(K)0, (K)0, take};
  auto all = [](int) { return true; };
  int eq = 0;
  constexpr int kBits = (int)sizeof(K) * 8;
  int shift = kBits - 8;
  bool early = false;
  for (; shift >= 0; shift -= 8) {
    radix_pass<NT, K>(n, key, all, st, shift, sm);
    eq = sm.eq;
    if (eq == st.rank) { early = true; break; }
  }
  // Items with (key & mask) < prefix are strictly smaller than the boundary bucket.
  if (early || eq == st.rank) {
    K mask = st.mask, prefix = st.prefix;
    for (int base = 0; base < n; base += NT) {
      int i = base + threadIdx.x;
      bool sel = i < n && ((key(i) & mask) <= prefix);
      unsigned b = __ballot_sync(0xffffffffu, sel);
      int base_slot = 0;
      if ((threadIdx.x & 31) == 0 && b) base_slot = atomicAdd(&sm.count, __popc(b));
      base_slot = __shfl_sync(0xffffffffu, base_slot, 0);
      if (sel) out[base_slot + __popc(b & ((1u << (threadIdx.x & 31)) - 1))] = i;
    }
    __syncthreads();
    return take;
  }
  // Boundary key shared by more items than needed: select among equal-key items by tie.
  K kstar = st.prefix;
  int need = st.rank;
  SelState<uint32_t> st2{0u, 0u, need};
  auto eqpred = [&](int i) { return key(i) == kstar; };
  for (int sh = 24; sh >= 0; sh -= 8) radix_pass<NT, uint32_t>(n, tie, eqpred, st2, sh, sm);
  uint32_t tstar = st2.prefix;
  for (int base = 0; base < n; base += NT) {
    int i = base + threadIdx.x;
    bool sel = false;
    if (i < n) {
      K k = key(i);
      sel = k < kstar || (k == kstar && tie(i) <= tstar);
    }
    unsigned b = __ballot_sync(0xffffffffu, sel);
    int base_slot = 0;
    if ((threadIdx.x & 31) == 0 && b) base_slot = atomicAdd(&sm.count, __popc(b));
    base_slot = __shfl_sync(0xffffffffu, base_slot, 0);
    if (sel) out[base_slot + __popc(b & ((1u << (threadIdx.x & 31)) - 1))] = i;
  }
  __syncthreads();
  return take;
}

// ------------------------------------------------ bucketed block selection
// Same contract as block_select_smallest, cheaper in the common case: one pass
// for min/max of the keys, one histogram pass over 2^11 buckets of
// (key - min) >> shift (a monotone bucketing of the integer keys), a block
// scan to find the boundary bucket, and one collection pass.  Items of the
// boundary bucket are resolved exactly by (key, tie) rank counting in shared
// memory; a boundary bucket larger than the buffer (e.g. thousands of equal
// keys) falls back to the radix select above.
constexpr int kSelBins = 2048;
constexpr int kSelBuf = 512;
constexpr int kSelBigN = 16384;   // block selections: sampled range + 8 keys in flight from here
constexpr int kSelSamples = 512;  // (fits bs.buf_key before the boundary buffer is needed)

struct BucketSmem {
  int hist[kSelBins];
  unsigned long long buf_key[kSelBuf];
  uint32_t buf_tie[kSelBuf];
  int buf_idx[kSelBuf];
  int wsum[32];
  unsigned long long lo, hi;
  int bb, before, eq, nbuf, count;
};

__device__ __forceinline__ int bitlen64(unsigned long long v) { return v ? 64 - __clzll(v) : 0; }

// Bitonic sort (ascending) of n_pow2 u64 keys in shared memory; pad with ~0.
template <int NT>
__device__ void block_bitonic_sort(uint64_t* a, int n_pow2) {
  for (int size = 2; size <= n_pow2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      __syncthreads();
      for (int t = threadIdx.x; t < n_pow2 / 2; t += NT) {
        int lo = 2 * t - (t & (stride - 1));
        int hi = lo + stride;
        bool up = ((lo & size) == 0);
        uint64_t x = a[lo], y = a[hi];
        if ((x > y) == up) { a[lo] = y; a[hi] = x; }
      }
    }
  }
  __syncthreads();
}

// Bucketing is linear in the key's float value v: b = min(B-1, floor(rn(rn(v - vmin) *
// scale))), a monotone non-decreasing map (IEEE rounding is monotone), so every
// item of a lower bucket precedes every item of a higher one; ties and the order
// inside the boundary bucket are resolved on the exact (key, tie).
template <int NT, typename K, typename V, typename KeyF, typename TieF, typename ValF>
__device__ int block_select_bucketed(int n, int take, KeyF key, TieF tie, ValF val, int* out,
                                     BucketSmem& bs, SelectSmem& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (take >= n) {
    for (int i = tid; i < n; i += NT) out[i] = i;
    __syncthreads();
    return n;
  }
  if (take <= 0) return 0;
  // long lists with a small take (C5: 1,600 of ~62k keys): the bucket range comes from
  // kSelSamples spread samples -- [smallest sample, a sample well above rank take] --
  // instead of a min/max sweep, and the sweeps keep 8 keys per thread in flight.  Keys
  // are clamped to the range first (a monotone map: lower buckets still precede higher
  // ones, so the selection stays exact; an unlucky sample only overflows the boundary
  // buffer into block_select_smallest).
  const bool big = sizeof(K) == 4 && n >= kSelBigN && (long long)take * 8 <= n;
  if (tid == 0) { bs.lo = ~0ull; bs.hi = 0ull; bs.nbuf = 0; bs.count = 0; }
  if (big) {
    for (int sidx = tid; sidx < kSelSamples; sidx += NT) {
      const int i = (int)((((long long)sidx * 2 + 1) * n) / (2 * kSelSamples));
      bs.buf_key[sidx] = ((unsigned long long)key(i) << 32) | (unsigned)sidx;
    }
    block_bitonic_sort<NT>(reinterpret_cast<uint64_t*>(bs.buf_key), kSelSamples);  // (ends with a barrier)
    const int rh = min(kSelSamples - 1, (int)(((long long)take * kSelSamples * 3) / (2LL * n)) + 24);
    const unsigned long long slo = bs.buf_key[0] >> 32, shi = bs.buf_key[rh] >> 32;
    __syncthreads();
    if (tid == 0) { bs.lo = slo; bs.hi = shi; }
  } else {
    // 1. value range (keys are monotone in value, so the extreme keys give it)
    unsigned long long lo = ~0ull, hi = 0ull;
    for (int i = tid; i < n; i += NT) {
      unsigned long long k = (unsigned long long)key(i);
      lo = k < lo ? k : lo;
      hi = k > hi ? k : hi;
    }
    for (int o = 16; o > 0; o >>= 1) {
      unsigned long long a = __shfl_xor_sync(0xffffffffu, lo, o);
      unsigned long long b = __shfl_xor_sync(0xffffffffu, hi, o);
      lo = a < lo ? a : lo;
      hi = b > hi ? b : hi;
    }
    __syncthreads();
    if (lane == 0) { atomicMin(&bs.lo, lo); atomicMax(&bs.hi, hi); }
  }
  for (int i = tid; i < kSelBins; i += NT) bs.hist[i] = 0;
  __syncthreads();
  const K klo = (K)bs.lo, khi = (K)bs.hi;
  const V vmin = val(klo), vmax = val(khi);
  const V range = vmax - vmin;
  const V scale = range > (V)0 ? (V)(kSelBins - 1) / range : (V)0;
  auto bucket_k = [&](K kk) {
    kk = kk < klo ? klo : (kk > khi ? khi : kk);  // (no-op for the swept range)
    V f = (val(kk) - vmin) * scale;
    int b = (int)f;
    return b < kSelBins - 1 ? (b < 0 ? 0 : b) : kSelBins - 1;
  };
  auto bucket = [&](int i) { return bucket_k(key(i)); };
  // 2. histogram
  if (big) {
    // keys above the sampled range (most of them) are only counted, per warp: one
    // shared-memory counter hit by every thread would serialise the sweep
    int above = 0;
    for (int b0 = tid; b0 < n; b0 += NT * 8) {
      K kv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) kv[u] = b0 + u * NT < n ? key(b0 + u * NT) : khi;
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        if (b0 + u * NT >= n) continue;
        if (kv[u] > khi) ++above;
        else atomicAdd(&bs.hist[bucket_k(kv[u])], 1);
      }
    }
    for (int o = 16; o > 0; o >>= 1) above += __shfl_xor_sync(0xffffffffu, above, o);
    if (lane == 0 && above) atomicAdd(&bs.hist[kSelBins - 1], above);
  } else {
    for (int i = tid; i < n; i += NT) atomicAdd(&bs.hist[bucket(i)], 1);
  }
  __syncthreads();
  // 3. boundary bucket: block exclusive scan of per-thread bin ranges
  constexpr int per = kSelBins / NT;
  int loc = 0;
#pragma unroll
  for (int j = 0; j < per; ++j) loc += bs.hist[tid * per + j];
  int incl = loc;
  for (int o = 1; o < 32; o <<= 1) {
    int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  if (lane == 31) bs.wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int v = lane < NT / 32 ? bs.wsum[lane] : 0, iv = v;
    for (int o = 1; o < 32; o <<= 1) {
      int u = __shfl_up_sync(0xffffffffu, iv, o);
      if (lane >= o) iv += u;
    }
    if (lane < NT / 32) bs.wsum[lane] = iv - v;
  }
  __syncthreads();
  int cum = bs.wsum[warp] + incl - loc;
  if (cum < take && take <= cum + loc) {
#pragma unroll
    for (int j = 0; j < per; ++j) {
      int h = bs.hist[tid * per + j];
      if (cum + h >= take) {
        bs.bb = tid * per + j;
        bs.before = cum;
        bs.eq = h;
        break;
      }
      cum += h;
    }
  }
  __syncthreads();
  const int bb = bs.bb, need = take - bs.before, eq = bs.eq;
  const bool all_eq = eq == need;
  if (!all_eq && eq > kSelBuf) {
    __syncthreads();
    return block_select_smallest<NT, K>(n, take, key, tie, out, sm);
  }
  // 4. collect
  auto collect = [&](int i, bool valid, K kk) {
    bool sel = false;
    if (valid) {
      int b = bucket_k(kk);
      if (b < bb || (b == bb && all_eq)) {
        sel = true;
      } else if (b == bb) {
        int s = atomicAdd(&bs.nbuf, 1);
        bs.buf_key[s] = (unsigned long long)kk;
        bs.buf_tie[s] = tie(i);
        bs.buf_idx[s] = i;
      }
    }
    unsigned m = __ballot_sync(0xffffffffu, sel);
    int slot = 0;
    if (lane == 0 && m) slot = atomicAdd(&bs.count, __popc(m));
    slot = __shfl_sync(0xffffffffu, slot, 0);
    if (sel) out[slot + __popc(m & ((1u << lane) - 1))] = i;
  };
  if (big) {
    for (int base = 0; base < n; base += NT * 8) {
      K kv[8];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * NT + tid;
        kv[u] = i < n ? key(i) : khi;
      }
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        const int i = base + u * NT + tid;
        collect(i, i < n, kv[u]);
      }
    }
  } else {
    for (int base = 0; base < n; base += NT) {
      const int i = base + tid;
      collect(i, i < n, i < n ? key(i) : khi);
    }
  }
  __syncthreads();
  // 5. exact resolution of the boundary bucket by (key, tie) rank
  if (!all_eq) {
    const int nb = bs.nbuf;
    for (int e = tid; e < nb; e += NT) {
      unsigned long long ke = bs.buf_key[e];
      uint32_t te = bs.buf_tie[e];
      int rank = 0;
      for (int f = 0; f < nb; ++f) {
        unsigned long long kf = bs.buf_key[f];
        rank += (kf < ke) || (kf == ke && bs.buf_tie[f] < te);
      }
      if (rank < need) out[atomicAdd(&bs.count, 1)] = bs.buf_idx[e];
    }
    __syncthreads();
  }
  return take;
}

}  // namespace rrg
