// rrg_cluster_score.cu -- cluster-major ("bucketed") scoring of the LoRANN query path.
//
// The query-major k_score_select re-reads a probed cluster's factors once per
// query (C2: ~440 KB of A/B codes per query, from L2).  Here the batch's
// (query, cluster) pairs are bucketed by cluster (histogram, scan, scatter --
// the "bucketing pass" of the north star); one CTA then stages a cluster's
// A^T/B^T codes and metadata in shared memory once and scores every query of
// its bucket chunk against it:
//   stage A  raw1 = codes_x . A (per query, r outputs)  -> inter -> re-quantize
//   stage B  raw2 = codes_r . B[:,p] (8 dp4a per point at r=32) -> yhat -> key
// (rrr.py:181-203, quantize.py:109-156; identical arithmetic to k_score_select).
// Keys land in a per-query candidate array (query-major, exact offsets) that
// k_select_topt reduces to the top-t by (key, corpus id) (index.py:314-316).
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>
#include <cstdlib>

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

// ---------------------------------------------------------- per-query offsets
// Warp per query: qoff[q][c] = sum of the sizes of sel[q][0..c) (selection
// order = candidate order), qoff[q][w] = N[q].
__global__ void k_cand_offsets(DevIndexView ix, const int* __restrict__ sel, int nq, int w,
                               int* __restrict__ qoff, int* __restrict__ ncand) {
  const int q = (blockIdx.x * blockDim.x + threadIdx.x) >> 5, lane = threadIdx.x & 31;
  if (q >= nq) return;
  int carry = 0;
  for (int b = 0; b < w; b += 32) {
    int c = b + lane, m = 0;
    if (c < w) {
      int l = sel[(size_t)q * w + c];
      m = ix.cl_pos[l + 1] - ix.cl_pos[l];
    }
    int incl = m;
    for (int o = 1; o < 32; o <<= 1) {
      int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    if (c < w) qoff[(size_t)q * (w + 1) + c] = carry + incl - m;
    carry += __shfl_sync(0xffffffffu, incl, 31);
  }
  if (lane == 0) {
    qoff[(size_t)q * (w + 1) + w] = carry;
    ncand[q] = carry;
  }
}

// ----------------------------------------------------------- pair bucketing
// One CTA: histogram of the Q*w (query, slot) pairs by cluster, exclusive scans
// (pair offsets per cluster, work items of <= kPairsPerItem pairs per cluster,
// key-array base per query), scatter of the pairs into cluster order.
constexpr int PNT = 1024;
constexpr int kPairsPerItem = 32;

// In-place exclusive scan of a[0..n) by the whole block (a contiguous run per
// thread, a shuffle scan of the run sums); *total = sum (all threads call it).
__device__ void block_exclusive_scan_inplace(int* a, int n, int* total) {
  __shared__ int wsum[33];
  const int tid = threadIdx.x, nt = blockDim.x, lane = tid & 31, warp = tid >> 5;
  const int per = (n + nt - 1) / nt;
  const int b0 = min(n, tid * per), b1 = min(n, b0 + per);
  int sum = 0;
  for (int i = b0; i < b1; ++i) sum += a[i];
  int incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) wsum[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    const int v = lane < nt / 32 ? wsum[lane] : 0;
    int iv = v;
    for (int o = 1; o < 32; o <<= 1) {
      const int t = __shfl_up_sync(0xffffffffu, iv, o);
      if (lane >= o) iv += t;
    }
    wsum[lane] = iv - v;
    if (lane == 31) wsum[32] = iv;
  }
  __syncthreads();
  int run = wsum[warp] + incl - sum;
  for (int i = b0; i < b1; ++i) {
    const int v = a[i];
    a[i] = run;
    run += v;
  }
  if (tid == 0) *total = wsum[32];
  __syncthreads();
}

// Scoring work items split a cluster's points into chunks of kScorePts (the largest
// clusters would otherwise set the tail of the persistent grid).
#ifndef RRG_SCORE_PTS
#define RRG_SCORE_PTS 1024  // C2 scoring: 256 -> 0.188, 512 -> 0.142, 1024 -> 0.126, 1536 -> 0.132, 2048 -> 0.143 ms
#endif
#ifndef RRG_SCORE_CTAS
#define RRG_SCORE_CTAS 4
#endif
constexpr int kScorePts = RRG_SCORE_PTS;

__global__ void __launch_bounds__(PNT) k_pairs_build(const int* __restrict__ sel, int nq, int w,
                                                     int L, const int* __restrict__ cl_pos,
                                                     const int* __restrict__ ncand,
                                                     int* __restrict__ pair_off,   // L+1
                                                     int* __restrict__ item_off,   // L+1
                                                     int* __restrict__ pairs,      // nq*w
                                                     int* __restrict__ kbase,      // nq+1
                                                     int stage_kbase, const int* __restrict__ order) {
  extern __shared__ int sh[];  // cnt[L], cur[L]
  int* cnt = sh;
  int* cur = sh + L;
  __shared__ int tot;
  for (int i = threadIdx.x; i < L; i += PNT) cnt[i] = 0;
  __syncthreads();
  const int np = nq * w;
  for (int i = threadIdx.x; i < np; i += PNT) atomicAdd(&cnt[sel[i]], 1);
  __syncthreads();
  for (int i = threadIdx.x; i < L; i += PNT) {
    cur[i] = cnt[i];
    // the scoring items run largest cluster first when `order` is given (entry i counts
    // the items of cluster order[i]; the kernel maps back through it)
    const int l = order ? order[i] : i;
    const int m = cl_pos[l + 1] - cl_pos[l];
    item_off[i] = ((cnt[l] + kPairsPerItem - 1) / kPairsPerItem) * ((m + kScorePts - 1) / kScorePts);
  }
  __syncthreads();
  block_exclusive_scan_inplace(cur, L, &tot);
  if (threadIdx.x == 0) pair_off[L] = tot;
  for (int i = threadIdx.x; i < L; i += PNT) pair_off[i] = cur[i];
  __syncthreads();
  block_exclusive_scan_inplace(item_off, L, &tot);
  if (threadIdx.x == 0) item_off[L] = tot;
  // scatter (order inside a cluster's bucket is irrelevant to results)
  for (int i = threadIdx.x; i < np; i += PNT) pairs[atomicAdd(&cur[sel[i]], 1)] = i;
  // key-array base per query: scanned in shared memory when the launch gave room for
  // it (coalesced in and out; the in-place scan of global memory was a chain of
  // dependent loads per thread)
  int* kb = stage_kbase ? sh + 2 * L : kbase;
  for (int q = threadIdx.x; q < nq; q += PNT) kb[q] = ncand[q];
  __syncthreads();
  block_exclusive_scan_inplace(kb, nq, &tot);
  if (stage_kbase) {
    __syncthreads();
    for (int q = threadIdx.x; q < nq; q += PNT) kbase[q] = kb[q];
  }
  if (threadIdx.x == 0) kbase[nq] = tot;
}

// ------------------------------------------------------------ cluster scoring
constexpr int CNT = 256;
constexpr int kMaxRc = 64;

struct ClusterScoreArgs {
  DevIndexView ix;
  const int8_t* qcodes;  // [nq][s_pad]
  const float* qscale;
  const float* qhead;
  const int* sel;        // [nq][w]
  int w;
  const int* qoff;       // [nq][w+1]
  const int* pair_off;   // [L+1]
  const int* item_off;   // [L+1]
  const int* pairs;      // [nq*w] pair ids (q*w + c) in cluster order
  const int* kbase;      // [nq+1]
  uint32_t* keys;        // [kbase[nq]]
  int* work_counter;     // zeroed before launch
  const float* xp;       // [nq][s] projected queries (f32-factor scoring)
  // stage outputs for the bit-parity tests (rrg_stage_score; nullptr on the search
  // path): stage-A int32 products per (pair, j < r) of RRR clusters, and per scored
  // point (key-array layout) the last stage's int32 product and the f32 score of
  // score_cluster (rrr.py:181-203: -2 yhat + ||c||^2 for euclidean, yhat otherwise)
  int* dbg_raw1;
  int* dbg_raw2;
  float* dbg_score;
  int stage_a_bytes;     // > 0: stage A operands staged in shared memory ((r + 32) * s_pad)
};

// TC: stage B on the 5th-gen tensor cores.  A work item's (<= 32) queries form the
// N = 32 operand (their re-quantized stage-A codes, K = r_pad = 32 bytes, one
// kind::i8 MMA per 128 points: M = 128 points of the cluster), the int32 products
// land in TMEM and the dequant / key epilogue reads them with tcgen05.ld -- warps w and
// w + 4 share TMEM lane quarter w % 4 and take 16 queries each.  Exact int8 x int8 ->
// int32 like the dp4a loop it replaces (rrr.py:196-197, quantize.py:109-126).
__device__ __forceinline__ uint32_t sc_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// kind::i8: D s32, A/B signed, K-major, N = 32, M = 128
constexpr uint32_t kScIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kPairsPerItem >> 3) << 17) |
                              ((uint32_t)(128 >> 4) << 24);

template <bool TC>
__global__ void __launch_bounds__(CNT) k_score_cluster(ClusterScoreArgs a) {
  const DevIndexView& ix = a.ix;
  extern __shared__ __align__(16) int8_t sc_dyn[];  // stage A operands (a.stage_a_bytes)
  __shared__ int item_s;
  // TC: A tile (128 points x 32 B), B tile (32 queries x 32 B), canonical K-major layout
  __shared__ __align__(128) int8_t tc_a[TC ? 128 * 32 : 16];
  __shared__ __align__(128) int8_t tc_b[TC ? kPairsPerItem * 32 : 16];
  __shared__ uint64_t tc_bar;
  __shared__ uint32_t tc_tmem;
  __shared__ __align__(16) int8_t c2s[kPairsPerItem][kMaxRc];
  __shared__ float s2s[kPairsPerItem], h2s[kPairsPerItem];
  __shared__ float inters[kPairsPerItem][kMaxRc];
  __shared__ int pq[kPairsPerItem], pkey[kPairsPerItem];
  __shared__ float pxs[kPairsPerItem], pxh[kPairsPerItem];
  const int L = ix.L, r = ix.r, r_pad = ix.r_pad, s_pad = ix.s_pad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total_items = a.item_off[L];
  const bool euclid = ix.metric == kMetricEuclidean;
  uint32_t tc_phase = 0;
  if (TC) {
    if (warp == 0) {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(sc_smem(&tc_tmem))
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
    if (tid == 32) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sc_smem(&tc_bar)));
      asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  }
  while (true) {
    if (tid == 0) item_s = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int item = item_s;
    __syncthreads();
    if (item >= total_items) break;
    // cluster of this item: upper_bound over item_off
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (a.item_off[mid] <= item) lo = mid; else hi = mid;
    }
    const int l = ix.opt.score_order ? __ldg(ix.cl_order + lo) : lo;  // (largest clusters first)
    const int p0 = ix.cl_pos[l], mcl = ix.cl_pos[l + 1] - p0;
    const int npc = (mcl + kScorePts - 1) / kScorePts;
    const int local = item - a.item_off[lo];
    const int j0 = a.pair_off[l] + (local / npc) * kPairsPerItem;
    const int np = min(kPairsPerItem, a.pair_off[l + 1] - j0);
    const int pbeg = (local % npc) * kScorePts, pend = min(mcl, pbeg + kScorePts);
    const int m = pend - pbeg;
    const bool rrr = ix.cl_kind[l] == kKindRrr;
    if (tid < np) {
      const int pr = a.pairs[j0 + tid];
      const int q = pr / a.w, c = pr % a.w;
      pq[tid] = q;
      pkey[tid] = a.kbase[q] + a.qoff[(size_t)q * (a.w + 1) + c];
      pxs[tid] = a.qscale[q];
      pxh[tid] = a.qhead[q];
    }
    __syncthreads();
    if (m == 0) continue;
    if (rrr) {
      // stage A: np x r dot products over s_pad bytes, `parts` lanes per product
      const int slot = ix.cl_aidx[l];
      const int nvec = s_pad / 16;
      const int prs = np * r;
      int parts = 1;
      while (parts < 32 && prs * parts * 2 <= CNT && parts * 2 <= nvec) parts <<= 1;
      // the cluster's A^T codes and the item's query codes staged once (all loads in
      // flight together): reading them per product from L2 was a chain of dependent
      // round trips per item (C2: the kernel's top stall)
      const bool staged = a.stage_a_bytes > 0;
      int8_t* s_at = sc_dyn;
      int8_t* s_qc = sc_dyn + (size_t)r * s_pad;
      if (staged) {
        const int4* ga = reinterpret_cast<const int4*>(ix.at + (size_t)slot * r * s_pad);
        for (int e = tid; e < r * nvec; e += CNT) reinterpret_cast<int4*>(s_at)[e] = __ldg(ga + e);
        for (int e = tid; e < np * nvec; e += CNT) {
          const int pi = e / nvec, u = e - pi * nvec;
          reinterpret_cast<int4*>(s_qc)[e] = __ldg(reinterpret_cast<const int4*>(a.qcodes + (size_t)pq[pi] * s_pad) + u);
        }
        __syncthreads();
      }
      for (int base = 0; base < prs * parts; base += CNT) {
        const int e = base + tid;
        const int pr = e / parts, part = e % parts;
        const bool act = pr < prs;
        const int pi = act ? pr / r : 0, jj = act ? pr % r : 0;
        int raw = 0;
        if (act) {
          const int4* aw = staged ? reinterpret_cast<const int4*>(s_at + (size_t)jj * s_pad)
                                  : reinterpret_cast<const int4*>(ix.at + ((size_t)slot * r + jj) * s_pad);
          const int4* q4 = staged ? reinterpret_cast<const int4*>(s_qc + (size_t)pi * s_pad)
                                  : reinterpret_cast<const int4*>(a.qcodes + (size_t)pq[pi] * s_pad);
          for (int u = part; u < nvec; u += parts) {
            int4 b = staged ? aw[u] : __ldg(aw + u), cc = staged ? q4[u] : __ldg(q4 + u);
            raw = __dp4a(cc.x, b.x, raw);
            raw = __dp4a(cc.y, b.y, raw);
            raw = __dp4a(cc.z, b.z, raw);
            raw = __dp4a(cc.w, b.w, raw);
          }
        }
        for (int o = 1; o < parts; o <<= 1) raw += __shfl_xor_sync(0xffffffffu, raw, o);
        if (act && part == 0) {
          const size_t aj = (size_t)slot * r + jj;
          inters[pi][jj] = deq(raw, pxs[pi], ix.ascale[aj], pxh[pi], ix.ahead[aj]);
          if (a.dbg_raw1) a.dbg_raw1[(size_t)a.pairs[j0 + pi] * r + jj] = raw;
        }
      }
      __syncthreads();
      for (int pi = warp; pi < np; pi += CNT / 32) {  // re-quantize (quantize.py:150)
        float amax = 0.0f;
        for (int j = 1 + lane; j < r; j += 32) amax = fmaxf(amax, fabsf(inters[pi][j]));
        for (int o = 16; o > 0; o >>= 1) amax = fmaxf(amax, __shfl_xor_sync(0xffffffffu, amax, o));
        const float sc2 = quant_scale(amax);
        for (int j = lane; j < r_pad; j += 32) {
          int code = 0;
          if (j >= 1 && j < r && amax != 0.0f) code = quant_code(inters[pi][j], sc2);
          c2s[pi][j] = (int8_t)code;
        }
        if (lane == 0) { s2s[pi] = sc2; h2s[pi] = inters[pi][0]; }
      }
      __syncthreads();
      if (TC) {
        // B operand: the item's stage-B query codes, row n = query slot, 32 code bytes
        for (int e = tid; e < kPairsPerItem * 2; e += CNT) {
          const int n = e >> 1, half = e & 1;
          int4 v = make_int4(0, 0, 0, 0);
          if (n < np) v = *reinterpret_cast<const int4*>(&c2s[n][half * 16]);
          *reinterpret_cast<int4*>(tc_b + (n >> 3) * 256 + half * 128 + (n & 7) * 16) = v;
        }
        for (int pb = pbeg; pb < pend; pb += 128) {
          // A operand: B^T codes of 128 points (32 bytes each), zero past the item's end
          for (int e = tid; e < 128 * 2; e += CNT) {
            const int row = e >> 1, half = e & 1, p = pb + row;
            int4 v = make_int4(0, 0, 0, 0);
            if (p < pend) v = __ldg(reinterpret_cast<const int4*>(ix.bt + (size_t)(p0 + p) * 32) + half);
            *reinterpret_cast<int4*>(tc_a + (row >> 3) * 256 + half * 128 + (row & 7) * 16) = v;
          }
          asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
          __syncthreads();
          if (tid == 0) {
            asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
            const uint64_t ad = (uint64_t)((sc_smem(tc_a) >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
                                ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
            const uint64_t bd = (uint64_t)((sc_smem(tc_b) >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
                                ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
            asm volatile(
                "{\n\t.reg .pred p;\n\t"
                "setp.ne.b32 p, 0, 0;\n\t"
                "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tc_tmem),
                "l"(ad), "l"(bd), "r"(kScIdesc)
                : "memory");
            asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                             sc_smem(&tc_bar))
                         : "memory");
          }
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "SC_WAIT_%=:\n\t"
              "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
              "@!p bra SC_WAIT_%=;\n\t}" ::"r"(sc_smem(&tc_bar)),
              "r"(tc_phase)
              : "memory");
          tc_phase ^= 1;
          asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
          const int row = (warp & 3) * 32 + lane, c0 = (warp >> 2) * 16, p = pb + row;
          uint32_t v[16];
          asm volatile(
              "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
              : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
                "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
              : "r"(tc_tmem + ((uint32_t)((warp & 3) * 32) << 16) + (uint32_t)c0));
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
          if (p < pend) {
            const int gp = p0 + p;
            const float4 meta = __ldg(ix.pmeta + gp);
#pragma unroll
            for (int j = 0; j < 16; ++j) {
              const int pi = c0 + j;
              if (pi < np) {
                const int raw = (int)v[j];
                const float yhat = deq(raw, s2s[pi], meta.y, h2s[pi], meta.x);
                const float keyf = euclid ? __fadd_rn(__fmul_rn(-2.0f, yhat), meta.z) : -yhat;
                a.keys[pkey[pi] + p] = mono32(keyf);
                if (a.dbg_raw2) {
                  a.dbg_raw2[pkey[pi] + p] = raw;
                  a.dbg_score[pkey[pi] + p] = euclid ? keyf : yhat;
                }
              }
            }
          }
          asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
          __syncthreads();  // the tiles and the accumulator are reused by the next block
        }
      }
      // stage B: thread per point, codes/meta loaded once, all np queries scored
      for (int p = pbeg + tid; p < (TC ? pbeg : pend); p += CNT) {
        const int gp = p0 + p;
        const float4 meta = __ldg(ix.pmeta + gp);
        int4 b[4];
        const int4* bw = reinterpret_cast<const int4*>(ix.bt + (size_t)gp * r_pad);
        const int nb4 = r_pad / 16;
#pragma unroll
        for (int u = 0; u < 4; ++u)
          if (u < nb4) b[u] = __ldg(bw + u);
        for (int pi = 0; pi < np; ++pi) {
          const int4* cw = reinterpret_cast<const int4*>(c2s[pi]);
          int raw = 0;
#pragma unroll
          for (int u = 0; u < 4; ++u)
            if (u < nb4) {
              int4 cc = cw[u];
              raw = __dp4a(cc.x, b[u].x, raw);
              raw = __dp4a(cc.y, b[u].y, raw);
              raw = __dp4a(cc.z, b[u].z, raw);
              raw = __dp4a(cc.w, b[u].w, raw);
            }
          const float yhat = deq(raw, s2s[pi], meta.y, h2s[pi], meta.x);
          const float keyf = euclid ? __fadd_rn(__fmul_rn(-2.0f, yhat), meta.z) : -yhat;
          a.keys[pkey[pi] + p] = mono32(keyf);
          if (a.dbg_raw2) {
            a.dbg_raw2[pkey[pi] + p] = raw;
            a.dbg_score[pkey[pi] + p] = euclid ? keyf : yhat;
          }
        }
      }
    } else {
      // exact model: raw_p = codes_x . A[:, p] over s_pad bytes (rrr.py:103-113)
      const int x0 = ix.cl_aidx[l];
      const int nvec = s_pad / 16;
      for (int p = pbeg + tid; p < pend; p += CNT) {
        const int gp = p0 + p;
        const float4 meta = __ldg(ix.pmeta + gp);
        const int4* xw = reinterpret_cast<const int4*>(ix.xcodes + (size_t)(x0 + p) * s_pad);
        for (int pi = 0; pi < np; ++pi) {
          const int4* q4 = reinterpret_cast<const int4*>(a.qcodes + (size_t)pq[pi] * s_pad);
          int raw = 0;
          for (int u = 0; u < nvec; ++u) {
            int4 bb = __ldg(xw + u), cc = __ldg(q4 + u);
            raw = __dp4a(cc.x, bb.x, raw);
            raw = __dp4a(cc.y, bb.y, raw);
            raw = __dp4a(cc.z, bb.z, raw);
            raw = __dp4a(cc.w, bb.w, raw);
          }
          const float yhat = deq(raw, pxs[pi], meta.y, pxh[pi], meta.x);
          const float keyf = euclid ? __fadd_rn(__fmul_rn(-2.0f, yhat), meta.z) : -yhat;
          a.keys[pkey[pi] + p] = mono32(keyf);
          if (a.dbg_raw2) {
            a.dbg_raw2[pkey[pi] + p] = raw;
            a.dbg_score[pkey[pi] + p] = euclid ? keyf : yhat;
          }
        }
      }
    }
    __syncthreads();
  }
  if (TC) {
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tc_tmem) : "memory");
  }
}

// ------------------------------------------------- cluster scoring, f32 factors
// Unquantized index (RrrConfig.quantize=False): score = x @ A (@ B) in f32
// (rrr.py:97-100, 196-202).  NumPy runs these as OpenBLAS sgemv, whose f32 FMA
// order is not reproducible, so parity is tolerance-level; the
// dot products here accumulate exact f32 products in f64 and round once, i.e.
// they return (nearly) the correctly rounded value, which OpenBLAS approximates.
// Same work items and key layout as k_score_cluster.
__global__ void __launch_bounds__(CNT) k_score_cluster_f32(ClusterScoreArgs a) {
  const DevIndexView& ix = a.ix;
  __shared__ int item_s;
  __shared__ float inters[kPairsPerItem][kMaxRc];
  __shared__ int pq[kPairsPerItem], pkey[kPairsPerItem];
  const int L = ix.L, r = ix.r, r_pad = ix.r_pad, s = ix.s, s_pad = ix.s_pad;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total_items = a.item_off[L];
  const bool euclid = ix.metric == kMetricEuclidean;
  while (true) {
    if (tid == 0) item_s = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int item = item_s;
    __syncthreads();
    if (item >= total_items) break;
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (a.item_off[mid] <= item) lo = mid; else hi = mid;
    }
    const int l = ix.opt.score_order ? __ldg(ix.cl_order + lo) : lo;  // (largest clusters first)
    const int p0 = ix.cl_pos[l], mcl = ix.cl_pos[l + 1] - p0;
    const int npc = (mcl + kScorePts - 1) / kScorePts;
    const int local = item - a.item_off[lo];
    const int j0 = a.pair_off[l] + (local / npc) * kPairsPerItem;
    const int np = min(kPairsPerItem, a.pair_off[l + 1] - j0);
    const int pbeg = (local % npc) * kScorePts, pend = min(mcl, pbeg + kScorePts);
    const int m = pend - pbeg;
    if (tid < np) {
      const int pr = a.pairs[j0 + tid];
      const int q = pr / a.w, c = pr % a.w;
      pq[tid] = q;
      pkey[tid] = a.kbase[q] + a.qoff[(size_t)q * (a.w + 1) + c];
    }
    __syncthreads();
    if (m == 0) continue;
    if (ix.cl_kind[l] == kKindRrr) {
      // inter = x @ A: warp per (pair, column), lanes over the s inputs
      const int slot = ix.cl_aidx[l];
      for (int o = warp; o < np * r; o += CNT / 32) {
        const int pi = o / r, j = o % r;
        const float* av = ix.atf + ((size_t)slot * r + j) * s_pad;
        const float* xv = a.xp + (size_t)pq[pi] * s;
        double acc = 0.0;
        for (int i = lane; i < s; i += 32) acc = fma((double)__ldg(xv + i), (double)__ldg(av + i), acc);
        for (int d = 16; d > 0; d >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, d);
        if (lane == 0) inters[pi][j] = (float)acc;
      }
      __syncthreads();
      // yhat = inter @ B: thread per point, B^T row held in registers
      for (int p = pbeg + tid; p < pend; p += CNT) {
        const int gp = p0 + p;
        const float4 meta = __ldg(ix.pmeta + gp);
        float b[kMaxRc];
        const float4* bw = reinterpret_cast<const float4*>(ix.btf + (size_t)gp * r_pad);
#pragma unroll
        for (int u = 0; u < kMaxRc / 4; ++u) {
          float4 v = u < r_pad / 4 ? __ldg(bw + u) : make_float4(0.f, 0.f, 0.f, 0.f);
          b[4 * u] = v.x; b[4 * u + 1] = v.y; b[4 * u + 2] = v.z; b[4 * u + 3] = v.w;
        }
        for (int pi = 0; pi < np; ++pi) {
          double acc = 0.0;
#pragma unroll
          for (int j = 0; j < kMaxRc; ++j)
            if (j < r) acc = fma((double)inters[pi][j], (double)b[j], acc);
          const float yhat = (float)acc;
          const float keyf = euclid ? __fadd_rn(__fmul_rn(-2.0f, yhat), meta.z) : -yhat;
          a.keys[pkey[pi] + p] = mono32(keyf);
          if (a.dbg_score) a.dbg_score[pkey[pi] + p] = euclid ? keyf : yhat;
        }
      }
    } else {
      // exact model: yhat = x @ A[:, p] over s (rrr.py:103-113)
      const int x0 = ix.cl_aidx[l];
      const int n4 = s / 4;
      for (int p = pbeg + tid; p < pend; p += CNT) {
        const int gp = p0 + p;
        const float4 meta = __ldg(ix.pmeta + gp);
        const float* xr = ix.xf + (size_t)(x0 + p) * s_pad;
        for (int pi = 0; pi < np; ++pi) {
          const float* xv = a.xp + (size_t)pq[pi] * s;
          double acc = 0.0;
          if ((s & 3) == 0) {
            const float4* x4 = reinterpret_cast<const float4*>(xv);
            const float4* r4 = reinterpret_cast<const float4*>(xr);
            for (int u = 0; u < n4; ++u) {
              const float4 xa = __ldg(x4 + u), ra = __ldg(r4 + u);
              acc = fma((double)xa.x, (double)ra.x, acc);
              acc = fma((double)xa.y, (double)ra.y, acc);
              acc = fma((double)xa.z, (double)ra.z, acc);
              acc = fma((double)xa.w, (double)ra.w, acc);
            }
          } else {
            for (int i = 0; i < s; ++i) acc = fma((double)__ldg(xv + i), (double)__ldg(xr + i), acc);
          }
          const float yhat = (float)acc;
          const float keyf = euclid ? __fadd_rn(__fmul_rn(-2.0f, yhat), meta.z) : -yhat;
          a.keys[pkey[pi] + p] = mono32(keyf);
          if (a.dbg_score) a.dbg_score[pkey[pi] + p] = euclid ? keyf : yhat;
        }
      }
    }
    __syncthreads();
  }
}

// ------------------------------------------------------------- top-t select
// One CTA per query: the take = min(t|k, N) smallest of the query's keys by
// (key, corpus id); positions recovered from (slot, offset) via the query's
// candidate offsets.
constexpr int TNT = 256;

struct SelectArgs {
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
  int kcap;      // keys staged in smem when N <= kcap
  int sort_cap;  // power of two >= k (no-rerank ordering)
  // cluster-major re-rank: selected candidate indices (into the query's key array)
  // and a membership bitmap over all keys (bit kbase[q] + i)
  int* cand_idx;
  uint32_t* marks;
};

__global__ void __launch_bounds__(TNT) k_select_topt(SelectArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x;
  const int w = a.w;
  int* offs = reinterpret_cast<int*>(smem_raw);      // w+1
  int* pbase = offs + (w + 1);                        // w: cl_pos of each slot
  int* selidx = pbase + w;                            // take_cap
  uintptr_t sp = reinterpret_cast<uintptr_t>(selidx + a.take_cap);
  uint64_t* srt = reinterpret_cast<uint64_t*>((sp + 15) & ~uintptr_t(15));
  uint32_t* kst = reinterpret_cast<uint32_t*>(srt + a.sort_cap);  // kcap staged keys
  for (int c = tid; c <= w; c += TNT) offs[c] = a.qoff[(size_t)q * (w + 1) + c];
  for (int c = tid; c < w; c += TNT) pbase[c] = ix.cl_pos[a.sel[(size_t)q * w + c]];
  __syncthreads();
  const int N = offs[w];
  const uint32_t* kq = a.keys + a.kbase[q];
  if (N <= a.kcap) {  // stage the query's keys once; the select makes ~3 passes
    const uint4* src = reinterpret_cast<const uint4*>(kq);
    const bool al = (reinterpret_cast<uintptr_t>(kq) & 15) == 0;
    if (al) {
      for (int i = tid; i < N / 4; i += TNT) reinterpret_cast<uint4*>(kst)[i] = __ldg(src + i);
      for (int i = (N / 4) * 4 + tid; i < N; i += TNT) kst[i] = __ldg(kq + i);
    } else {
      for (int i = tid; i < N; i += TNT) kst[i] = __ldg(kq + i);
    }
    __syncthreads();
    kq = kst;
  }
  auto pos_of = [&](int i) {
    int lo = 0, hi = w;  // largest c with offs[c] <= i
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (offs[mid] <= i) lo = mid; else hi = mid;
    }
    return pbase[lo] + (i - offs[lo]);
  };
  const int take = min(a.take_cap, N);
  auto key = [&](int i) { return kq[i]; };
  auto tie = [&](int i) { return __float_as_uint(__ldg(ix.pmeta + pos_of(i)).w); };
  auto val = [](uint32_t k) { return unmono32(k); };
  block_select_bucketed<TNT, uint32_t, float>(N, take, key, tie, val, selidx, bs, sm);
  const int gq = a.q0 + q;
  if (a.rerank && a.marks) {  // cluster-major re-rank consumes (index, membership bit)
    int* oi = a.cand_idx + (size_t)q * a.take_cap;
    const size_t kb = (size_t)a.kbase[q];
    const int sh = (int)(kb & 31), nw = (sh + N + 31) / 32;
    if (N <= a.kcap && nw <= a.kcap) {
      // the query's bits are one contiguous run: build its words in shared memory
      // (the staged keys are dead now) and OR whole words into the global bitmap
      uint32_t* bm = kst;
      __syncthreads();
      for (int i = tid; i < nw; i += TNT) bm[i] = 0u;
      __syncthreads();
      for (int i = tid; i < take; i += TNT) {
        const int ci = selidx[i];
        oi[i] = ci;
        atomicOr(&bm[(sh + ci) >> 5], 1u << ((sh + ci) & 31));
      }
      __syncthreads();
      uint32_t* gm = a.marks + (kb >> 5);
      for (int i = tid; i < nw; i += TNT) {
        const uint32_t v = bm[i];
        if (v) atomicOr(gm + i, v);  // edge words are shared with the neighbouring queries
      }
    } else {
      for (int i = tid; i < take; i += TNT) {
        const int ci = selidx[i];
        oi[i] = ci;
        const size_t bit = kb + (size_t)ci;
        atomicOr(a.marks + (bit >> 5), 1u << (bit & 31));
      }
    }
    if (tid == 0) a.cand_n[q] = take;
    return;
  }
  if (a.rerank) {
    int* outp = a.cand_pos + (size_t)q * a.take_cap;
    for (int i = tid; i < take; i += TNT) outp[i] = pos_of(selidx[i]);
    if (a.sel_keys) {
      uint32_t* ok = a.sel_keys + (size_t)gq * a.take_cap;
      uint32_t* oi = a.sel_ids + (size_t)gq * a.take_cap;
      for (int i = tid; i < take; i += TNT) {
        ok[i] = key(selidx[i]);
        oi[i] = tie(selidx[i]);
      }
      if (tid == 0) a.sel_count[gq] = take;
    }
    if (tid == 0) a.cand_n[q] = take;
    return;
  }
  int np2 = 1;
  while (np2 < take) np2 <<= 1;
  for (int i = tid; i < np2; i += TNT) {
    uint64_t v = ~0ull;
    if (i < take) v = ((uint64_t)key(selidx[i]) << 32) | tie(selidx[i]);
    srt[i] = v;
  }
  block_bitonic_sort<TNT>(srt, np2);
  const bool euclid = ix.metric == kMetricEuclidean;
  const float xxq = a.xx[q];
  for (int i = tid; i < a.k; i += TNT) {
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

// ---------------------------------------------- warp-per-query selection
// The per-query selections (top-t of the scores, top-k of the re-ranked
// distances) have ~1k candidates: a 256-thread CTA spends them on barriers
// (47% barrier stalls in ncu).  Here one warp owns a query: its keys are
// staged in the warp's shared-memory slice, a 4-pass 8-bit radix select finds
// the take-th smallest key K* (lanes with equal digits aggregated by
// __match_any_sync before one shared atomic), keys < K* are compacted by
// ballot, and the ties at K* are resolved by (key, corpus id) like the block
// select -- the same exact result, no CTA barrier.
constexpr int kWarpTieCap = 64;  // boundary elements resolved by rank on-chip

struct WarpSel {
  const uint32_t* keys;  // the query's keys (staged in the warp's smem slice, or global)
  int* hist;             // 256
  int* bidx;             // kWarpTieCap boundary candidates
  uint32_t* bkey;        // kWarpTieCap
  uint32_t* selbits;     // ceil(n/32) words marking the selected candidates (optional)
};

// Selects the `take` smallest of keys[0..n) by (key, tie(i)) -- tie(i) the corpus
// id, as the reference's lexsort((ids, keys)) (index.py:315,321); n > take >= 1.
// Indices go out through emit(slot, i), slot in [0, take), arbitrary order; when
// ws.selbits is set, bit i of it marks the selected candidates.
//  1. value range of the keys (warp min/max), 256 float-linear buckets (monotone
//     in the key, so equal keys share a bucket), histogram, boundary bucket bb;
//  2. buckets < bb are selected (ballot compaction); the boundary bucket's members
//     are ranked exactly by (key, tie) when they fit kWarpTieCap;
//  3. otherwise (a dense boundary bucket, e.g. many equal keys) an exact 8-bit
//     radix select over the keys, equal keys at the take-th ranked by tie.
template <typename KeyF, typename TieF, typename EmitF>
__device__ void warp_select_smallest(const WarpSel& ws, KeyF key, int n, int take, TieF tie,
                                     EmitF emit) {
  const int lane = threadIdx.x & 31;
  const unsigned lt_mask = (1u << lane) - 1u;
  // in-order sweep over 32-key chunks with four chunks' loads in flight:
  // body(chunk base, i, valid, key) for every chunk (warp-uniform)
  auto sweep = [&](auto&& body) {
    for (int base = 0; base < n; base += 128) {
      uint32_t kv[4];
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int i = base + 32 * u + lane;
        kv[u] = i < n ? key(i) : 0xFFFFFFFFu;
      }
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int b0 = base + 32 * u;
        if (b0 < n) body(b0, b0 + lane, b0 + lane < n, kv[u]);
      }
    }
  };
  auto mark = [&](int i) {
    if (ws.selbits) atomicOr(&ws.selbits[i >> 5], 1u << (i & 31));
  };
  // locate the bucket (of a 256-bin histogram of bucket_of) holding rank `take`
  auto boundary = [&](int& bb, int& before, int& cnt) {
    int c[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { c[j] = ws.hist[lane * 8 + j]; tot += c[j]; }
    int incl = tot;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const bool own = incl - tot < take && take <= incl;
    bb = 0; before = 0; cnt = 0;
    if (own) {
      int run = incl - tot;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (run + c[j] >= take) { bb = lane * 8 + j; before = run; cnt = c[j]; break; }
        run += c[j];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, own)) - 1;
    bb = __shfl_sync(0xffffffffu, bb, src);
    before = __shfl_sync(0xffffffffu, before, src);
    cnt = __shfl_sync(0xffffffffu, cnt, src);
    __syncwarp();
  };
  // ---- 1. range and float-linear histogram (two levels: the boundary bucket of the
  // first is re-bucketed over its own value span, which absorbs outliers that
  // stretch the first range)
  uint32_t lo = 0xFFFFFFFFu, hi = 0u;
  sweep([&](int, int, bool valid, uint32_t k) {
    if (valid) { lo = min(lo, k); hi = max(hi, k); }
  });
  for (int o = 16; o > 0; o >>= 1) {
    lo = min(lo, __shfl_xor_sync(0xffffffffu, lo, o));
    hi = max(hi, __shfl_xor_sync(0xffffffffu, hi, o));
  }
  const float vmin = unmono32(lo), vmax = unmono32(hi);
  const float range = vmax - vmin;
  const float scale = (range > 0.f && range < 3.0e38f) ? 256.f / range : 0.f;
  auto bucket = [&](uint32_t k) {
    const int b = (int)((unmono32(k) - vmin) * scale);
    return b < 0 ? 0 : (b > 255 ? 255 : b);
  };
  for (int b = lane; b < 256; b += 32) ws.hist[b] = 0;
  __syncwarp();
  sweep([&](int, int, bool valid, uint32_t k) {
    if (valid) atomicAdd(&ws.hist[bucket(k)], 1);
  });
  __syncwarp();
  int bb, before, cnt;
  boundary(bb, before, cnt);
  // level 2 over the boundary bucket's value span [vmin + bb/scale, vmin + (bb+1)/scale)
  const float v2lo = scale > 0.f ? vmin + (float)bb / scale : vmin;
  const float v2hi = scale > 0.f ? vmin + (float)(bb + 1) / scale : vmax;
  const float r2 = v2hi - v2lo;
  const float scale2 = (r2 > 0.f && r2 < 3.0e38f) ? 256.f / r2 : 0.f;
  auto bucket2 = [&](uint32_t k) {
    const int b = (int)((unmono32(k) - v2lo) * scale2);
    return b < 0 ? 0 : (b > 255 ? 255 : b);
  };
  int bb2 = -1;
  if (cnt > kWarpTieCap) {
    const int take1 = take - before;
    for (int b = lane; b < 256; b += 32) ws.hist[b] = 0;
    __syncwarp();
    sweep([&](int, int, bool valid, uint32_t k) {
      if (valid && bucket(k) == bb) atomicAdd(&ws.hist[bucket2(k)], 1);
    });
    __syncwarp();
    int before2, cnt2;
    {
      // boundary() searches rank `take`; shift by the elements below bucket bb
      int c[8], tot = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) { c[j] = ws.hist[lane * 8 + j]; tot += c[j]; }
      int incl = tot;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const bool own = incl - tot < take1 && take1 <= incl;
      int b2 = 0, bf = 0, cn = 0;
      if (own) {
        int run = incl - tot;
#pragma unroll
        for (int j = 0; j < 8; ++j) {
          if (run + c[j] >= take1) { b2 = lane * 8 + j; bf = run; cn = c[j]; break; }
          run += c[j];
        }
      }
      const int src = __ffs(__ballot_sync(0xffffffffu, own)) - 1;
      bb2 = __shfl_sync(0xffffffffu, b2, src);
      before2 = __shfl_sync(0xffffffffu, bf, src);
      cnt2 = __shfl_sync(0xffffffffu, cn, src);
      __syncwarp();
    }
    before += before2;
    cnt = cnt2;
  }
  if (cnt <= kWarpTieCap) {
    // ---- 2. buckets below the boundary selected; the boundary bucket ranked exactly
    auto cls = [&](uint32_t k) {  // -1 below, 0 boundary, 1 above
      const int b = bucket(k);
      if (b != bb) return b < bb ? -1 : 1;
      if (bb2 < 0) return 0;
      const int b2 = bucket2(k);
      return b2 < bb2 ? -1 : (b2 == bb2 ? 0 : 1);
    };
    int nlt = 0, nb = 0;
    sweep([&](int base, int i, bool valid, uint32_t k) {
      const int c = valid ? cls(k) : 1;
      const bool lt = c < 0, eq = c == 0;
      const unsigned bl = __ballot_sync(0xffffffffu, lt), be = __ballot_sync(0xffffffffu, eq);
      if (lt) emit(nlt + __popc(bl & lt_mask), i);
      if (eq) {
        const int slot = nb + __popc(be & lt_mask);
        ws.bidx[slot] = i;
        ws.bkey[slot] = k;
      }
      if (ws.selbits && lane == 0) ws.selbits[base >> 5] = bl;
      nlt += __popc(bl);
      nb += __popc(be);
    });
    __syncwarp();
    const int need = take - before;
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int e = lane + 32 * u;
      if (e < nb) {
        const uint32_t ke = ws.bkey[e];
        int r = 0;
        bool dup = false;
        for (int f = 0; f < nb; ++f) {
          const uint32_t kf = ws.bkey[f];
          r += kf < ke;
          dup |= kf == ke && f != e;
        }
        if (dup) {  // equal keys: corpus id order
          const uint32_t te = tie(ws.bidx[e]);
          for (int f = 0; f < nb; ++f)
            if (f != e && ws.bkey[f] == ke) r += tie(ws.bidx[f]) < te;
        }
        if (r < need) {
          emit(before + r, ws.bidx[e]);
          mark(ws.bidx[e]);
        }
      }
    }
    __syncwarp();
    return;
  }
  // ---- 3. exact radix select over the key bits
  uint32_t prefix = 0;
  int kk = take;
#pragma unroll 1
  for (int pass = 0; pass < 4; ++pass) {
    const int shift = 24 - 8 * pass;
    const uint32_t hmask = pass == 0 ? 0u : (0xFFFFFFFFu << (shift + 8));
    for (int b = lane; b < 256; b += 32) ws.hist[b] = 0;
    __syncwarp();
    sweep([&](int, int, bool valid, uint32_t k) {
      const bool m = valid && (k & hmask) == prefix;
      const unsigned dig = (k >> shift) & 255u;
      const unsigned peers = __match_any_sync(0xffffffffu, m ? dig : 256u + lane);
      if (m && (peers & lt_mask) == 0) atomicAdd(&ws.hist[dig], __popc(peers));
    });
    __syncwarp();
    int c[8], tot = 0;
#pragma unroll
    for (int j = 0; j < 8; ++j) { c[j] = ws.hist[lane * 8 + j]; tot += c[j]; }
    int incl = tot;
    for (int o = 1; o < 32; o <<= 1) {
      const int v = __shfl_up_sync(0xffffffffu, incl, o);
      if (lane >= o) incl += v;
    }
    const bool own = incl - tot < kk && kk <= incl;
    int bin = 0, bef = 0;
    if (own) {
      int run = incl - tot;
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        if (run + c[j] >= kk) { bin = lane * 8 + j; bef = run; break; }
        run += c[j];
      }
    }
    const int src = __ffs(__ballot_sync(0xffffffffu, own)) - 1;
    bin = __shfl_sync(0xffffffffu, bin, src);
    bef = __shfl_sync(0xffffffffu, bef, src);
    kk -= bef;
    prefix |= (uint32_t)bin << shift;
    __syncwarp();
  }
  // prefix == K*: keys below it are selected; kk of the keys equal to it, by tie
  int nlt = 0, nt = 0;
  sweep([&](int base, int i, bool valid, uint32_t k) {
    const bool lt = valid && k < prefix, eq = valid && k == prefix;
    const unsigned bl = __ballot_sync(0xffffffffu, lt), be = __ballot_sync(0xffffffffu, eq);
    if (lt) emit(nlt + __popc(bl & lt_mask), i);
    if (eq) {
      const int slot = nt + __popc(be & lt_mask);
      if (slot < kWarpTieCap) ws.bidx[slot] = i;
    }
    if (ws.selbits && lane == 0) ws.selbits[base >> 5] = bl;
    nlt += __popc(bl);
    nt += __popc(be);
  });
  __syncwarp();
  if (nt == kk) {  // every key equal to K* is selected
    int cidx = 0;
    sweep([&](int base, int i, bool valid, uint32_t k) {
      const bool eq = valid && k == prefix;
      const unsigned be = __ballot_sync(0xffffffffu, eq);
      if (eq) emit(nlt + cidx + __popc(be & lt_mask), i);
      if (ws.selbits && lane == 0 && be) atomicOr(&ws.selbits[base >> 5], be);
      cidx += __popc(be);
    });
  } else if (nt <= kWarpTieCap) {
    uint32_t* tv = ws.bkey;
    for (int j = lane; j < nt; j += 32) tv[j] = tie(ws.bidx[j]);
    __syncwarp();
#pragma unroll
    for (int u = 0; u < 2; ++u) {
      const int j = lane + 32 * u;
      if (j < nt) {
        int r = 0;
        for (int f = 0; f < nt; ++f) r += tv[f] < tv[j];
        if (r < kk) {
          emit(nlt + r, ws.bidx[j]);
          mark(ws.bidx[j]);
        }
      }
    }
  } else {  // more than kWarpTieCap equal keys at K*: rank by streaming (rare)
    for (int base = 0; base < n; base += 32) {
      const int i = base + lane;
      const bool eq = i < n && key(i) == prefix;
      if (eq) {
        const uint32_t tv = tie(i);
        int r = 0;
        for (int f = 0; f < n; ++f) r += key(f) == prefix && tie(f) < tv;
        if (r < kk) {
          emit(nlt + r, i);
          mark(i);
        }
      }
    }
  }
  __syncwarp();
}

// Per-warp slice of the dynamic shared memory of the warp kernels: staged keys
// (stage_cap, may be 0), histogram, boundary buffers, selection bits.
__host__ __device__ inline size_t warp_sel_bytes(int stage_cap, int bits_cap) {
  return ((size_t)stage_cap * 4 + 256 * 4 + kWarpTieCap * 8 + (size_t)((bits_cap + 31) / 32) * 4 +
          15) / 16 * 16;
}
__device__ inline WarpSel warp_sel_slice(unsigned char* base, int stage_cap, int bits_cap,
                                         uint32_t*& stage) {
  unsigned char* p = base + (size_t)(threadIdx.x >> 5) * warp_sel_bytes(stage_cap, bits_cap);
  WarpSel ws;
  stage = reinterpret_cast<uint32_t*>(p);
  ws.keys = stage;
  ws.hist = reinterpret_cast<int*>(stage + stage_cap);
  ws.bidx = ws.hist + 256;
  ws.bkey = reinterpret_cast<uint32_t*>(ws.bidx + kWarpTieCap);
  ws.selbits = bits_cap > 0 ? ws.bkey + kWarpTieCap : nullptr;
  return ws;
}

// Candidate index -> held position: largest c with offs[c] <= i (w+1 offsets, global).
__device__ __forceinline__ int cand_pos(const DevIndexView& ix, const int* qoffq, const int* selq,
                                        int w, int i) {
  int lo = 0, hi = w;
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(qoffq + mid) <= i) lo = mid; else hi = mid;
  }
  return __ldg(ix.cl_pos + __ldg(selq + lo)) + (i - __ldg(qoffq + lo));
}

// top-t of the scores (index.py:314-316), warp per query, for the re-ranking
// searches: cluster-major (cand_idx + membership bits) or per-query (cand_pos,
// plus the sharded phase-1 (key, id) lists).  Keys are staged on-chip when the
// largest candidate list fits stage_cap, else read through L1.
__global__ void k_select_topt_warp(SelectArgs a, int stage_cap, int bits_cap, int nq) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wq = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wq >= nq) return;
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[wq] : wq;
  const int w = a.w;
  const int* qoffq = a.qoff + (size_t)q * (w + 1);
  const int* selq = a.sel + (size_t)q * w;
  const int N = __ldg(qoffq + w);
  const int take = min(a.take_cap, N);
  uint32_t* stage;
  WarpSel ws = warp_sel_slice(smem_raw, stage_cap, bits_cap, stage);
  const uint32_t* kq = a.keys + a.kbase[q];
  auto key = [&](int i) { return __ldg(kq + i); };  // read through L1 (4 chunks in flight)
  (void)stage;
  auto tie = [&](int i) { return __float_as_uint(__ldg(ix.pmeta + cand_pos(ix, qoffq, selq, w, i)).w); };
  const int gq = a.q0 + q;
  if (a.marks) {  // cluster-major re-rank: candidate indices + membership bits
    int* oi = a.cand_idx + (size_t)q * a.take_cap;
    if (take >= N) {
      for (int i = lane; i < N; i += 32) oi[i] = i;
      for (int j = lane; j < (N + 31) / 32; j += 32)
        ws.selbits[j] = (j + 1) * 32 <= N ? 0xFFFFFFFFu : ((1u << (N & 31)) - 1u);
    } else {
      warp_select_smallest(ws, key, N, take, tie, [&](int slot, int i) { oi[slot] = i; });
    }
    __syncwarp();
    // OR the bits into the query's (unaligned) run of the global bitmap; the edge
    // words are shared with the neighbouring queries
    const size_t kb = (size_t)a.kbase[q];
    const unsigned sh = (unsigned)(kb & 31);
    uint32_t* gm = a.marks + (kb >> 5);
    for (int j = lane; j < (N + 31) / 32; j += 32) {
      const uint32_t word = ws.selbits[j];
      if (word) {
        atomicOr(gm + j, word << sh);
        if (sh) atomicOr(gm + j + 1, word >> (32 - sh));
      }
    }
  } else {
    int* outp = a.cand_pos + (size_t)q * a.take_cap;
    uint32_t* ok = a.sel_keys ? a.sel_keys + (size_t)gq * a.take_cap : nullptr;
    uint32_t* oid = a.sel_keys ? a.sel_ids + (size_t)gq * a.take_cap : nullptr;
    auto emit = [&](int slot, int i) {
      const int pos = cand_pos(ix, qoffq, selq, w, i);
      outp[slot] = pos;
      if (ok) { ok[slot] = key(i); oid[slot] = __float_as_uint(__ldg(ix.pmeta + pos).w); }
    };
    if (take >= N) for (int i = lane; i < N; i += 32) emit(i, i);
    else warp_select_smallest(ws, key, N, take, tie, emit);
    if (ok && lane == 0) a.sel_count[gq] = take;
  }
  if (lane == 0) a.cand_n[q] = take;
}

// Warp bitonic sort (ascending) of 32*E u64 values, element e = lane + 32*j in v[j].
template <int E>
__device__ __forceinline__ void warp_bitonic_sort(uint64_t (&v)[E]) {
  const int lane = threadIdx.x & 31;
  constexpr int P = 32 * E;
#pragma unroll
  for (int size = 2; size <= P; size <<= 1) {
#pragma unroll
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      if (stride >= 32) {  // partner in the same lane, register j ^ (stride/32)
        const int js = stride >> 5;
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int jp = j ^ js;
          if (jp > j) {
            const int e = lane + 32 * j;
            const bool up = (e & size) == 0;
            const uint64_t x = v[j], y = v[jp];
            const bool sw = (x > y) == up;
            v[j] = sw ? y : x;
            v[jp] = sw ? x : y;
          }
        }
      } else {
#pragma unroll
        for (int j = 0; j < E; ++j) {
          const int e = lane + 32 * j;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[j], stride);
          const bool up = (e & size) == 0;
          const bool lower = (lane & stride) == 0;
          // the lower element of a pair keeps the min when ascending
          const bool keep_min = lower == up;
          v[j] = keep_min ? (o < v[j] ? o : v[j]) : (o > v[j] ? o : v[j]);
        }
      }
    }
  }
}

// ---------------------------------------------------- cluster-major re-rank
// Re-ranking is a (query x candidate-row) distance matrix restricted to each
// query's top-t; rows of one cluster are shared by every query of its bucket
// (C2: ~10 queries re-rank ~800 of the same ~1000 rows).  One CTA takes a
// (cluster, <=32 queries) work item of the scoring pass, stages the queries'
// x (interleaved like the rows) and top-t membership bits in shared memory,
// and streams the cluster's rows through registers once: each row pair is
// loaded by one warp and scored against every query of the item that selected
// either row.  The per-(query, row) arithmetic is k_rerank_tree's -- NumPy's
// pairwise tree, bit-exact -- with lane (leaf b, pair h) of a 32-lane row
// group (8 leaves; leaf size a multiple of 8).  Distances land as mono32 keys
// over the query's candidate-key array; k_topk_final orders them.
constexpr int XNT = 256;
#ifndef RRG_CM_CTAS
#define RRG_CM_CTAS 2  // C2 with next-pair prefetch: 2 CTAs/SM (123 regs) 1.20 ms vs 3 CTAs (80 regs + spill) 1.31 ms
#endif
constexpr int kCmCtas = RRG_CM_CTAS;  // resident CTAs per SM
#ifndef RRG_RR_ROWS
#define RRG_RR_ROWS 512  // C2 re-rank: 128 -> 1.240, 256 -> 1.122, 384 -> 1.106, 512 -> 1.095, 768 -> 1.134, 1024 -> 1.149 ms
#endif
constexpr int kRrRows = RRG_RR_ROWS;  // rows of the cluster per work item (large batches)

struct ClusterRerankArgs {
  DevIndexView ix;
  const float* queries;  // chunk-local [nq][d]
  const float* xint;     // the same queries interleaved like the corpus rows [nq][d_stride]
  int ordered;           // rr_item_off runs over ix.cl_order (sparse kernels)
  const int* cand_idx;   // k_rerank_sparse: the screen's survivors per query
  const int* cand_n;
  int take_cap;
  int w;
  const int* qoff;
  const int* pair_off;
  const int* rr_item_off;  // [L+1] prefix of ceil(pairs_l/kRrQ) * ceil(m_l/rr_rows)
  int rr_rows;             // rows per work item: kRrRows, fewer for small batches
  const int* pairs;
  const int* kbase;
  const uint32_t* marks;
  uint32_t* diss;
  int* work_counter;
  int mwords;  // bitmap words staged per query (>= ceil(max m_l / 32) + 1)
  float neg_zero;  // -0.0f at run time: see sq2()
  int64_t* counters;  // rrg_search_counters (nullptr unless enabled): [3] += rows fetched
};

// rr_item_off for the re-rank work items (one CTA)
__global__ void __launch_bounds__(PNT) k_rr_items(const int* __restrict__ pair_off,
                                                  const int* __restrict__ cl_pos, int L, int rows,
                                                  int* __restrict__ rr_item_off,
                                                  const int* __restrict__ order = nullptr) {
  // entry j counts the items of cluster order[j] (or j): the kernels map an item back
  // through the same order
  __shared__ int tot;
  for (int j = threadIdx.x; j < L; j += PNT) {
    const int l = order ? order[j] : j;
    const int cnt = pair_off[l + 1] - pair_off[l], m = cl_pos[l + 1] - cl_pos[l];
    rr_item_off[j] = ((cnt + kRrQ - 1) / kRrQ) * ((m + rows - 1) / rows);
  }
  __syncthreads();
  block_exclusive_scan_inplace(rr_item_off, L, &tot);
  if (threadIdx.x == 0) rr_item_off[L] = tot;
}

__global__ void k_interleave_queries(DevIndexView ix, const float* __restrict__ x, int nq,
                                     float* __restrict__ xint) {
  // block per query: its row is staged in shared memory, then written out in slot
  // order (coalesced), slot = elem_perm[j]; the d_stride - d pad slots are zero
  extern __shared__ float xrow[];
  const int q = blockIdx.x;
  for (int j = threadIdx.x; j < ix.d_stride; j += blockDim.x) xrow[j] = 0.f;
  __syncthreads();
  for (int j = threadIdx.x; j < ix.d; j += blockDim.x)
    xrow[ix.elem_perm ? __ldg(ix.elem_perm + j) : j] = __ldg(x + (size_t)q * ix.d + j);
  __syncthreads();
  float4* dst = reinterpret_cast<float4*>(xint + (size_t)q * ix.d_stride);
  for (int j = threadIdx.x; j < ix.d_stride / 4; j += blockDim.x) dst[j] = reinterpret_cast<float4*>(xrow)[j];
}

void launch_interleave_queries(const DevIndexView& ix, const float* queries, int nq, float* xint,
                               cudaStream_t st) {
  (k_interleave_queries<<<nq, 256, (size_t)ix.d_stride * 4, st>>>(ix, queries, nq, xint), note_launch());
}

void launch_rr_items(const int* pair_off, const int* cl_pos, int L, int rows, int* item_off,
                     cudaStream_t st) {
  (k_rr_items<<<1, PNT, 0, st>>>(pair_off, cl_pos, L, rows, item_off), note_launch());
}

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  const unsigned sa = (unsigned)__cvta_generic_to_shared(smem);
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(sa), "l"(gmem) : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_all;" ::: "memory"); }

// ASYNC: the next row pair is copied global -> shared (cp.async, no registers) while
// the current pair is scored, so the copy has a whole pair's arithmetic to land;
// without it the next pair is loaded into registers after the scoring, with only
// the reduction to hide its latency.
// NH = 2: rows of 16 equal leaves (d = 1536): NumPy's tree is pw(first half) +
// pw(second half), each half a perfect 8-leaf tree over the same lanes -- the pair is
// scored half by half (leaves 0-7 sit at [0, 64) of every interleaved 128-float step,
// leaves 8-15 at [64, 128)) and the two reduced halves are added.
// RM (row mode) 0: every row pair of the item's range is loaded (balanced clusters: a
// C2 query keeps 82% of its rows; measured 1.10 vs 1.26 ms for RM 1).  RM 1 (SKIP): row
// pairs no query of the work item selected are passed over before any load is issued
// (unbalanced clusters, C4: up to 11x the mean size).  RM 2 (COMPACT): the rows any
// query of the item selected are listed first (a block-wide compaction of the OR of
// the item's membership words) and the warps take pairs of listed rows -- for the
// sparse selections the re-rank screen leaves (~k of t rows per query survive), where
// pairs of adjacent rows would load many unselected rows.
template <int NB, bool ASYNC, int NH = 1, int RM = 0>
__global__ void __launch_bounds__(XNT, kCmCtas) k_rerank_cluster(ClusterRerankArgs a) {
  constexpr bool SKIP = RM == 1;
  static_assert(!(ASYNC && RM == 2), "the cp.async variant streams adjacent row pairs");
  constexpr int NLV = 8 * NH, cstep = 8 * NLV;
  static_assert(NH == 1 || !ASYNC, "the cp.async variant handles 8-leaf rows");
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const DevIndexView& ix = a.ix;
  const int ds = ix.d_stride, d = ix.d;
  float* xs = reinterpret_cast<float*>(smem_raw);                       // [kRrQ][ds]
  uint32_t* mb = reinterpret_cast<uint32_t*>(xs + (size_t)kRrQ * ds);  // [kRrQ][mwords]
  // ASYNC: per-warp staging of one row pair [warp][2][ds] after the bitmaps
  float* rowbuf = reinterpret_cast<float*>(mb + (size_t)kRrQ * a.mwords) +
                  (size_t)(threadIdx.x >> 5) * 2 * ds;
  __shared__ int item_s;
  __shared__ int pq[kPairsPerItem], pkey[kPairsPerItem];
  __shared__ int slotq[XNT / 32][kRrQ];
  __shared__ int rowlist[RM == 2 ? kRrRows : 1], nrows_s;
  const int L = ix.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = XNT / 32;
  const int b = lane >> 2, h = lane & 3;
  const int coff = 8 * b + 2 * h;
  const bool euclid = ix.metric == kMetricEuclidean;
  const float2 nz2 = make_float2(a.neg_zero, a.neg_zero);
  // work item = (cluster, <= kRrQ queries, <= kRrRows rows): bounded size, so the
  // largest clusters with the most queries do not serialise the tail
  const int total_items = a.rr_item_off[L];
  while (true) {
    if (tid == 0) item_s = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int item = item_s;
    __syncthreads();
    if (item >= total_items) break;
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (a.rr_item_off[mid] <= item) lo = mid; else hi = mid;
    }
    const int l = lo;
    const int p0 = ix.cl_pos[l], m = ix.cl_pos[l + 1] - p0;
    const int nrc = (m + a.rr_rows - 1) / a.rr_rows;
    const int local = item - a.rr_item_off[l];
    const int qc = nrc > 0 ? local / nrc : 0, rc = nrc > 0 ? local % nrc : 0;
    const int j0 = a.pair_off[l] + qc * kRrQ;
    const int np = min(kRrQ, a.pair_off[l + 1] - j0);
    const int r0 = rc * a.rr_rows, r1 = min(m, r0 + a.rr_rows);
    if (tid < np) {
      const int pr = a.pairs[j0 + tid];
      const int q = pr / a.w, c = pr % a.w;
      pq[tid] = q;
      pkey[tid] = a.kbase[q] + a.qoff[(size_t)q * (a.w + 1) + c];
    }
    __syncthreads();
    if (m == 0) continue;
    const int mw = (m + 31) / 32;
    for (int g0 = 0; g0 < np; g0 += kRrQ) {
      const int ng = min(kRrQ, np - g0);
      if (a.xint) {  // stage x: pre-interleaved rows, 16-byte loads, 4 in flight per thread
        constexpr int SU = 4;
        const int n4 = ds / 4, tot = ng * n4;
        float4* xs4 = reinterpret_cast<float4*>(xs);
        for (int e0 = tid; e0 < tot; e0 += XNT * SU) {
          float4 xv[SU];
#pragma unroll
          for (int u = 0; u < SU; ++u) {
            const int e = e0 + u * XNT;
            if (e < tot) {
              const int g = e / n4, j = e - g * n4;
              xv[u] = __ldg(reinterpret_cast<const float4*>(a.xint + (size_t)pq[g0 + g] * ds) + j);
            }
          }
#pragma unroll
          for (int u = 0; u < SU; ++u)
            if (e0 + u * XNT < tot) xs4[e0 + u * XNT] = xv[u];
        }
      } else {  // stage x (interleaved): SU independent loads in flight per thread
        constexpr int SU = 4;
        const int tot = ng * d;
        for (int e0 = tid; e0 < tot; e0 += XNT * SU) {
          float xv[SU];
          int dst[SU];
#pragma unroll
          for (int u = 0; u < SU; ++u) {
            const int e = e0 + u * XNT;
            if (e < tot) {
              const int g = e / d, j = e - g * d;
              xv[u] = __ldg(a.queries + (size_t)pq[g0 + g] * d + j);
              dst[u] = g * ds + __ldg(ix.elem_perm + j);
            }
          }
#pragma unroll
          for (int u = 0; u < SU; ++u)
            if (e0 + u * XNT < tot) xs[dst[u]] = xv[u];
        }
      }
      for (int e = tid; e < ng * mw; e += XNT) {
        const int g = e / mw, k = e - g * mw;
        const size_t bit = (size_t)pkey[g0 + g] + 32 * (size_t)k;
        const uint32_t lo32 = a.marks[bit >> 5];
        const uint32_t hi32 = a.marks[(bit >> 5) + 1];  // bitmap carries one pad word
        mb[g * a.mwords + k] = __funnelshift_r(lo32, hi32, (unsigned)(bit & 31));
      }
      __syncthreads();
      auto marked = [&](int g, int p) {
        return p < r1 && ((mb[g * a.mwords + (p >> 5)] >> (p & 31)) & 1u);
      };
      if (RM == 2) {  // list the rows of [r0, r1) any query of the item selected
        if (warp == 0) {
          int base_n = 0;
          for (int k0 = r0 >> 5; k0 <= (r1 - 1) >> 5; k0 += 32) {
            const int k = k0 + lane;
            uint32_t u = 0;
            if (k <= (r1 - 1) >> 5) {
              for (int g = 0; g < ng; ++g) u |= mb[g * a.mwords + k];
              if (k == r0 >> 5) u &= 0xffffffffu << (r0 & 31);
              if (k == (r1 - 1) >> 5) u &= 0xffffffffu >> (31 - ((r1 - 1) & 31));
            }
            const int cnt = __popc(u);
            int incl = cnt;
            for (int o = 1; o < 32; o <<= 1) {
              const int v = __shfl_up_sync(0xffffffffu, incl, o);
              if (lane >= o) incl += v;
            }
            int at = base_n + incl - cnt;
            while (u) {
              const int b = __ffs(u) - 1;
              u &= u - 1;
              rowlist[at++] = 32 * k + b;
            }
            base_n += __shfl_sync(0xffffffffu, incl, 31);
          }
          if (lane == 0) nrows_s = base_n;
        }
        __syncthreads();
      }
      // work runs over indices ia of the item's rows: r0 + ia, or the listed rows (RM 2)
      const int n_idx = RM == 2 ? nrows_s : r1 - r0;
      auto row_of = [&](int ia) { return RM == 2 ? rowlist[ia] : r0 + ia; };
      // this lane's 2-element slice of each step of rows pa and pa+1 (register
      // double use: the next pair's loads are issued before this pair's reduction)
      float2 ca[NB], cb[NB];
      int hoff = 0;  // NH = 2: the half (0 or 64 floats into each step) being scored
      auto load_pair = [&](int ia) {
        const int pa = row_of(ia);
        const int pb = ia + 1 < n_idx ? row_of(ia + 1) : pa;
        if (ASYNC) {  // issue the copy of both rows into this warp's staging slot
          const float4* ra = reinterpret_cast<const float4*>(ix.corpus + (size_t)(p0 + pa) * ds);
          const float4* rb = reinterpret_cast<const float4*>(ix.corpus + (size_t)(p0 + pb) * ds);
          float4* sa = reinterpret_cast<float4*>(rowbuf);
          float4* sb = reinterpret_cast<float4*>(rowbuf + ds);
          const int n16 = ds / 4;
          for (int c = lane; c < n16; c += 32) {
            cp_async16(sa + c, ra + c);
            cp_async16(sb + c, rb + c);
          }
          cp_async_commit();
          return;
        }
        const float* ra = ix.corpus + (size_t)(p0 + pa) * ds + coff + hoff;
        const float* rb = ix.corpus + (size_t)(p0 + pb) * ds + coff + hoff;
#pragma unroll
        for (int i = 0; i < NB; ++i) ca[i] = __ldg(reinterpret_cast<const float2*>(ra + cstep * i));
#pragma unroll
        for (int i = 0; i < NB; ++i) cb[i] = __ldg(reinterpret_cast<const float2*>(rb + cstep * i));
      };
      // ASYNC: wait for the staged pair and move this lane's slices to registers
      auto take_pair = [&]() {
        cp_async_wait_all();
        __syncwarp();
        const float* sa = rowbuf + coff;
        const float* sb = rowbuf + ds + coff;
#pragma unroll
        for (int i = 0; i < NB; ++i) ca[i] = *reinterpret_cast<const float2*>(sa + cstep * i);
#pragma unroll
        for (int i = 0; i < NB; ++i) cb[i] = *reinterpret_cast<const float2*>(sb + cstep * i);
        __syncwarp();
      };
      // per (query, row pair): this lane's r[2h]+r[2h+1] of both rows
      auto lane_sums = [&](int g, float& va, float& vb) {
        const float* xg = xs + (size_t)g * ds + coff + hoff;
        if (euclid) {
          float2 acca = make_float2(0.f, 0.f), accb = acca;
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            const float2 xv = *reinterpret_cast<const float2*>(xg + cstep * i);
            const float2 nx = make_float2(-xv.x, -xv.y);
            const float2 da = __fadd2_rn(ca[i], nx), db = __fadd2_rn(cb[i], nx);
            const float2 sa = sq2(da, nz2), sb = sq2(db, nz2);
            acca = i == 0 ? sa : __fadd2_rn(acca, sa);
            accb = i == 0 ? sb : __fadd2_rn(accb, sb);
          }
          va = __fadd_rn(acca.x, acca.y);
          vb = __fadd_rn(accb.x, accb.y);
        } else {
          float acc_a = 0.f, acc_b = 0.f;
#pragma unroll
          for (int i = 0; i < NB; ++i) {
            const float2 xv = *reinterpret_cast<const float2*>(xg + cstep * i);
            acc_a += ca[i].x * xv.x + ca[i].y * xv.y;
            acc_b += cb[i].x * xv.x + cb[i].y * xv.y;
          }
          va = acc_a;
          vb = acc_b;
        }
      };
      auto next_marked = [&](int ia) {
        if (!(SKIP || ASYNC)) return ia;
        while (ia < n_idx && !__ballot_sync(0xffffffffu, lane < ng && (marked(lane, r0 + ia) ||
                                                                         marked(lane, r0 + ia + 1))))
          ia += nwarps * 2;
        return ia;
      };
      int ia = next_marked(warp * 2);
      if (ia < n_idx) load_pair(ia);
      int nfetch = 0;
      for (; ia < n_idx;) {
        const int pa = row_of(ia);
        const int pb = ia + 1 < n_idx ? row_of(ia + 1) : pa;
        nfetch += pb != pa ? 2 : 1;
        const int pn = next_marked(ia + nwarps * 2);
        // the queries that selected either row (one lane per query, ballot)
        const bool mine = lane < ng && (marked(lane, pa) || marked(lane, pb));
        const unsigned act0 = __ballot_sync(0xffffffffu, mine);
        if (ASYNC) {
          take_pair();
          if (pn < n_idx) load_pair(pn);
        } else if (!act0) {
          if (pn < n_idx) load_pair(pn);
          ia = pn;
          continue;
        }
        float res = 0.f;  // NH = 2: the first half's reduced value
#pragma unroll
        for (int h2 = 0; h2 < NH; ++h2) {
        // per-lane partials of every active (query, row) pair: value 2*slot + row
        float v[2 * kRrQ];
        unsigned act = act0;
#pragma unroll
        for (int slot = 0; slot < kRrQ; ++slot) {
          if (act) {  // warp-uniform
            const int g = __ffs(act) - 1;
            act &= act - 1;
            lane_sums(g, v[2 * slot], v[2 * slot + 1]);
          } else {
            v[2 * slot] = 0.f;
            v[2 * slot + 1] = 0.f;
          }
        }
        if (h2 + 1 < NH) {  // the pair's next half
          hoff = 64 * (h2 + 1);
          load_pair(ia);
        } else if (!ASYNC && pn < n_idx) {
          hoff = 0;
          load_pair(pn);
        }
        // Transposing butterfly: five xor-steps (1, 2, 4, 8, 16 -- NumPy's
        // ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7)) per leaf, then the perfect 8-leaf tree)
        // that halve the values held per lane, so lane j ends with value j fully
        // reduced.  Each add combines the same two partial sums as the plain
        // butterfly (a+b == b+a exactly), at 31 shuffles per 32 values instead of 160.
#pragma unroll
        for (int s = 0; s < 5; ++s) {
          const int o = 1 << s;
          const bool hi = (lane >> s) & 1;
#pragma unroll
          for (int i = 0; i < (16 >> s); ++i) {
            const float keep = hi ? v[2 * i + 1] : v[2 * i];
            const float send = hi ? v[2 * i] : v[2 * i + 1];
            v[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
          }
        }
        res = h2 == 0 ? v[0] : __fadd_rn(res, v[0]);  // pw(half 0) + pw(half 1)
        }
        // lane j holds (slot j/2, row j%2); slot s is the s-th set bit of act0
        if (mine) slotq[warp][__popc(act0 & ((1u << lane) - 1u))] = lane;
        __syncwarp();
        const int slot = lane >> 1;
        if (slot < __popc(act0)) {
          const int g = slotq[warp][slot];
          const int p = (lane & 1) ? pb : pa;
          if (marked(g, p)) a.diss[pkey[g0 + g] + p] = mono32(euclid ? res : -res);
        }
        __syncwarp();
        ia = pn;
      }
      if (a.counters && lane == 0 && nfetch)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 3), (unsigned long long)nfetch);
      __syncthreads();
    }
  }
}

// ------------------------------------------------- sparse exact re-rank (screened)
// After the tensor-core screen about k of a query's t candidates survive (C2: 114 of
// 800), so a work item's rows are each wanted by one or a few of its queries.  Here a
// warp takes ONE listed row at a time (the next row's loads in flight meanwhile),
// forms this lane's pairwise partial for every query that kept the row, and reduces
// the P (next power of two of the active count) values with a P-way transposing
// butterfly: (P - 1) + (5 - log2 P) shuffles instead of 31 for a full 16-slot pair,
// and no arithmetic for queries that did not keep the row.  Same summation tree as
// k_rerank_cluster (NumPy's, bit-exact).
template <int P, int N>
__device__ __forceinline__ float reduce_p(float (&v)[N], int lane) {
  // transposing levels: lane bits 0..log2(P)-1 end up indexing the value they hold
#pragma unroll
  for (int s = 0; (1 << s) < P; ++s) {
    const int o = 1 << s;
    const bool hi = (lane >> s) & 1;
#pragma unroll
    for (int i = 0; i < (P >> (s + 1)); ++i) {
      const float keep = hi ? v[2 * i + 1] : v[2 * i];
      const float send = hi ? v[2 * i] : v[2 * i + 1];
      v[i] = __fadd_rn(keep, __shfl_xor_sync(0xffffffffu, send, o));
    }
  }
  float r = v[0];
#pragma unroll
  for (int o = P; o < 32; o <<= 1) r = __fadd_rn(r, __shfl_xor_sync(0xffffffffu, r, o));
  return r;
}
template <int N>
__device__ __forceinline__ float reduce_any(float (&v)[N], int nval, int lane) {
  if (nval <= 1) return reduce_p<1>(v, lane);
  if constexpr (N >= 2) if (nval <= 2) return reduce_p<2>(v, lane);
  if constexpr (N >= 4) if (nval <= 4) return reduce_p<4>(v, lane);
  if constexpr (N >= 8) if (nval <= 8) return reduce_p<8>(v, lane);
  if constexpr (N >= 32) if (nval > 16) return reduce_p<32>(v, lane);
  if constexpr (N >= 16) return reduce_p<16>(v, lane);
  return reduce_p<N>(v, lane);  // (nval <= N here)
}

// One listed row against the S first active queries (act: their slot bits, nact <= S):
// this lane's pairwise partial per (query, half), then the P-way reduction.  S is the
// next power of two of nact, so a row only one or two queries kept costs no unrolled
// work for the other 14 slots (C2: 2.2 queries per fetched row).
template <int S, int NB, int NH>
__device__ __forceinline__ float sparse_row_dist(unsigned act, int nact, const float* __restrict__ xs, int ds,
                                                 int coff, const float2 (&c)[NH][NB], float2 nz2, int lane) {
  constexpr int cstep = 64 * NH;
  float v[NH * S];
  unsigned rem = act;
#pragma unroll
  for (int s = 0; s < S; ++s) {
#pragma unroll
    for (int hh = 0; hh < NH; ++hh) v[NH * s + hh] = 0.f;
    if (rem) {  // warp-uniform
      const int g = __ffs(rem) - 1;
      rem &= rem - 1;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh) {
        const float* xg = xs + (size_t)g * ds + coff + 64 * hh;
        float2 acc = make_float2(0.f, 0.f);
#pragma unroll
        for (int i = 0; i < NB; ++i) {
          const float2 xv = *reinterpret_cast<const float2*>(xg + cstep * i);
          const float2 dd = __fadd2_rn(c[hh][i], make_float2(-xv.x, -xv.y));
          const float2 sq = sq2(dd, nz2);
          acc = i == 0 ? sq : __fadd2_rn(acc, sq);
        }
        v[NH * s + hh] = __fadd_rn(acc.x, acc.y);  // r[2h] + r[2h+1] of this lane
      }
    }
  }
  return reduce_any<NH * S>(v, NH * nact, lane);
}
template <int NB, int NH>
__device__ __forceinline__ float sparse_row(unsigned act, int nact, const float* __restrict__ xs, int ds, int coff,
                                            const float2 (&c)[NH][NB], float2 nz2, int lane) {
  if (nact <= 1) return sparse_row_dist<1, NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
  if (nact <= 2) return sparse_row_dist<2, NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
  if (nact <= 4) return sparse_row_dist<4, NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
  if (nact <= 8) return sparse_row_dist<8, NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
  return sparse_row_dist<kRrQ, NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
}

constexpr int SNT = 256;
#ifndef RRG_SP_ROWS
#define RRG_SP_ROWS 2048  // rows per sparse item: C2 512 -> 1.248, 1024 -> 1.237, 2048 -> 1.224, 4096 -> 1.353 ms (smem)
#endif
constexpr int kSpRows = RRG_SP_ROWS;
// PF: the next row's loads are issued before this row's arithmetic (register double
// buffer); CT: resident CTAs per SM the register budget targets
template <int NB, int NH, bool PF = true, int CT = (NH == 1 ? 2 : 1)>
__global__ void __launch_bounds__(SNT, CT) k_rerank_sparse(ClusterRerankArgs a) {
  constexpr int NLV = 8 * NH, cstep = 8 * NLV;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const DevIndexView& ix = a.ix;
  const int ds = ix.d_stride;
  float* xs = reinterpret_cast<float*>(smem_raw);                       // [kRrQ][ds]
  uint32_t* mb = reinterpret_cast<uint32_t*>(xs + (size_t)kRrQ * ds);  // [kRrQ][mwords]
  __shared__ int item_s, nrows_s;
  __shared__ int pq[kRrQ], pkey[kRrQ], pofs[kRrQ];
  __shared__ int rowlist[kSpRows];
  __shared__ int slotg[SNT / 32][kRrQ];
  const int L = ix.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int nwarps = SNT / 32;
  const int b = lane >> 2, h = lane & 3;
  const int coff = 8 * b + 2 * h;
  const float2 nz2 = make_float2(a.neg_zero, a.neg_zero);
  const int total_items = a.rr_item_off[L];
  while (true) {
    if (tid == 0) item_s = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int item = item_s;
    __syncthreads();
    if (item >= total_items) break;
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (a.rr_item_off[mid] <= item) lo = mid; else hi = mid;
    }
    const int l = a.ordered ? __ldg(ix.cl_order + lo) : lo;  // (largest clusters first)
    const int p0 = ix.cl_pos[l], m = ix.cl_pos[l + 1] - p0;
    const int nrc = (m + a.rr_rows - 1) / a.rr_rows;
    const int local = item - a.rr_item_off[lo];
    const int qc = nrc > 0 ? local / nrc : 0, rc = nrc > 0 ? local % nrc : 0;
    const int j0 = a.pair_off[l] + qc * kRrQ;
    const int ng = min(kRrQ, a.pair_off[l + 1] - j0);
    const int r0 = rc * a.rr_rows, r1 = min(m, r0 + a.rr_rows);
    if (tid < ng) {
      const int pr = a.pairs[j0 + tid];
      const int q = pr / a.w, c = pr % a.w;
      pq[tid] = q;
      pofs[tid] = a.qoff[(size_t)q * (a.w + 1) + c];
      pkey[tid] = a.kbase[q] + pofs[tid];
    }
    __syncthreads();
    if (m == 0) continue;
    {  // x of the item's queries (pre-interleaved): 16-byte loads, 4 in flight per thread
      constexpr int SU = 4;
      const int n4 = ds / 4, tot = ng * n4;
      float4* xs4 = reinterpret_cast<float4*>(xs);
      for (int e0 = tid; e0 < tot; e0 += SNT * SU) {
        float4 xv[SU];
#pragma unroll
        for (int u = 0; u < SU; ++u) {
          const int e = e0 + u * SNT;
          if (e < tot) {
            const int g = e / n4, j = e - g * n4;
            xv[u] = __ldg(reinterpret_cast<const float4*>(a.xint + (size_t)pq[g] * ds) + j);
          }
        }
#pragma unroll
        for (int u = 0; u < SU; ++u)
          if (e0 + u * SNT < tot) xs4[e0 + u * SNT] = xv[u];
      }
    }
    // membership bits of the item's rows [r0, r1) (word k covers rows 32k..32k+31): the
    // screen's survivors of each slot's query that fall in this probe's rows
    const int k0 = r0 >> 5, k1 = (r1 - 1) >> 5, nwd = k1 - k0 + 1;
    for (int e = tid; e < ng * nwd; e += SNT) {
      const int g = e / nwd, k = k0 + e - g * nwd;
      mb[g * a.mwords + k] = 0;
    }
    __syncthreads();
    for (int g = warp; g < ng; g += nwarps) {
      const int q = pq[g], off = pofs[g], n = a.cand_n[q];
      const int* list = a.cand_idx + (size_t)q * a.take_cap;
      for (int i = lane; i < n; i += 32) {
        const int row = __ldg(list + i) - off;
        if (row >= r0 && row < r1) atomicOr(mb + g * a.mwords + (row >> 5), 1u << (row & 31));
      }
    }
    __syncthreads();
    if (warp == 0) {  // list the rows any query of the item kept
      int base_n = 0;
      for (int kk = k0; kk <= k1; kk += 32) {
        const int k = kk + lane;
        uint32_t u = 0;
        if (k <= k1) {
          for (int g = 0; g < ng; ++g) u |= mb[g * a.mwords + k];
          if (k == k0) u &= 0xffffffffu << (r0 & 31);
          if (k == k1) u &= 0xffffffffu >> (31 - ((r1 - 1) & 31));
        }
        const int cnt = __popc(u);
        int incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        int at = base_n + incl - cnt;
        while (u) {
          const int bb = __ffs(u) - 1;
          u &= u - 1;
          rowlist[at++] = 32 * k + bb;
        }
        base_n += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) nrows_s = base_n;
    }
    __syncthreads();
    const int nrows = nrows_s;
    float2 c[NH][NB], cn[NH][PF ? NB : 1];
    auto load_row = [&](int ia, float2 (&dst)[NH][NB]) {
      const float* ra = ix.corpus + (size_t)(p0 + rowlist[ia]) * ds + coff;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
#pragma unroll
        for (int i = 0; i < NB; ++i) dst[hh][i] = __ldg(reinterpret_cast<const float2*>(ra + 64 * hh + cstep * i));
    };
    auto load_next = [&](int ib) {
      const float* ra = ix.corpus + (size_t)(p0 + rowlist[ib]) * ds + coff;
#pragma unroll
      for (int hh = 0; hh < NH; ++hh)
#pragma unroll
        for (int i = 0; i < (PF ? NB : 1); ++i)
          cn[hh][i] = __ldg(reinterpret_cast<const float2*>(ra + 64 * hh + cstep * i));
    };
    int ia = warp;
    if (ia < nrows) load_row(ia, c);
    int nfetch = 0;
    for (; ia < nrows; ia += nwarps) {
      const int row = rowlist[ia];
      if (PF && ia + nwarps < nrows) load_next(ia + nwarps);
      ++nfetch;
      // queries that kept this row, in slot order
      const bool mine = lane < ng && ((mb[lane * a.mwords + (row >> 5)] >> (row & 31)) & 1u);
      const unsigned act = __ballot_sync(0xffffffffu, mine);
      const int nact = __popc(act);
      if (mine) slotg[warp][__popc(act & ((1u << lane) - 1u))] = lane;
      __syncwarp();
      // lane j holds value j fully reduced; NH = 2: dist = pw(half 0) + pw(half 1)
      float r = sparse_row<NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
      if (NH == 2) r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));
      if (lane < NH * nact && lane % NH == 0) {
        const int g = slotg[warp][lane / NH];
        a.diss[pkey[g] + row] = mono32(r);
      }
      __syncwarp();
      if (PF) {
#pragma unroll
        for (int hh = 0; hh < NH; ++hh)
#pragma unroll
          for (int i = 0; i < (PF ? NB : 1); ++i) c[hh][i] = cn[hh][i];
      } else if (ia + nwarps < nrows) {
        load_row(ia + nwarps, c);
      }
    }
    if (a.counters && lane == 0 && nfetch)
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 3), (unsigned long long)nfetch);
    __syncthreads();
  }
}

// Same computation as k_rerank_sparse, with the listed rows streamed into a shared-
// memory ring by a producer warp (cp.async.bulk, one row per copy, an mbarrier per
// slot) instead of register loads by the computing warps: the rows in flight per SM
// are set by the ring depth (16-32 rows) rather than by what the warps have issued
// while they compute.  RRG_SPARSE_VARIANT=2.
constexpr int RNT = SNT + 32;  // 8 computing warps + the producer warp
__device__ __forceinline__ void rr_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "RR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RR_WAIT_%=;\n\t}" ::"r"(sc_smem(bar)),
      "r"(parity)
      : "memory");
}
template <int NB, int NH>
__global__ void __launch_bounds__(RNT, NH == 1 ? 2 : 1) k_rerank_sparse_ring(ClusterRerankArgs a, int nslots) {
  constexpr int NLV = 8 * NH, cstep = 8 * NLV;
  constexpr int kMaxSlots = 32;
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const DevIndexView& ix = a.ix;
  const int ds = ix.d_stride;
  const int row_bytes = ds * 4;
  float* xs = reinterpret_cast<float*>(smem_raw);                       // [kRrQ][ds]
  uint32_t* mb = reinterpret_cast<uint32_t*>(xs + (size_t)kRrQ * ds);  // [kRrQ][mwords]
  unsigned char* ring = smem_raw + (((size_t)kRrQ * ds * 4 + (size_t)kRrQ * a.mwords * 4 + 127) & ~(size_t)127);
  __shared__ uint64_t full[kMaxSlots], empty[kMaxSlots];
  __shared__ int item_s, nrows_s;
  __shared__ int pq[kRrQ], pkey[kRrQ], pofs[kRrQ];
  __shared__ int rowlist[kSpRows];
  __shared__ int slotg[SNT / 32][kRrQ];
  const int L = ix.L;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int ncw = SNT / 32;  // computing warps
  const int b = lane >> 2, h = lane & 3;
  const int coff = 8 * b + 2 * h;
  const float2 nz2 = make_float2(a.neg_zero, a.neg_zero);
  const int total_items = a.rr_item_off[L];
  if (tid == 0) {
    for (int i = 0; i < nslots; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sc_smem(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sc_smem(&empty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  int gbase = 0;  // rows this CTA has streamed before the current item (ring position)
  while (true) {
    if (tid == 0) item_s = atomicAdd(a.work_counter, 1);
    __syncthreads();
    const int item = item_s;
    __syncthreads();
    if (item >= total_items) break;
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (a.rr_item_off[mid] <= item) lo = mid; else hi = mid;
    }
    const int l = a.ordered ? __ldg(ix.cl_order + lo) : lo;  // (largest clusters first)
    const int p0 = ix.cl_pos[l], m = ix.cl_pos[l + 1] - p0;
    const int nrc = (m + a.rr_rows - 1) / a.rr_rows;
    const int local = item - a.rr_item_off[lo];
    const int qc = nrc > 0 ? local / nrc : 0, rc = nrc > 0 ? local % nrc : 0;
    const int j0 = a.pair_off[l] + qc * kRrQ;
    const int ng = min(kRrQ, a.pair_off[l + 1] - j0);
    const int r0 = rc * a.rr_rows, r1 = min(m, r0 + a.rr_rows);
    if (tid < ng) {
      const int pr = a.pairs[j0 + tid];
      const int q = pr / a.w, c = pr % a.w;
      pq[tid] = q;
      pofs[tid] = a.qoff[(size_t)q * (a.w + 1) + c];
      pkey[tid] = a.kbase[q] + pofs[tid];
    }
    __syncthreads();
    if (m == 0) continue;
    const int k0 = r0 >> 5, k1 = (r1 - 1) >> 5, nwd = k1 - k0 + 1;
    for (int e = tid; e < ng * nwd; e += RNT) {
      const int g = e / nwd, k = k0 + e - g * nwd;
      mb[g * a.mwords + k] = 0;
    }
    __syncthreads();
    for (int g = warp; g < ng; g += RNT / 32) {
      const int q = pq[g], off = pofs[g], n = a.cand_n[q];
      const int* list = a.cand_idx + (size_t)q * a.take_cap;
      for (int i = lane; i < n; i += 32) {
        const int row = __ldg(list + i) - off;
        if (row >= r0 && row < r1) atomicOr(mb + g * a.mwords + (row >> 5), 1u << (row & 31));
      }
    }
    __syncthreads();
    if (warp == 0) {  // list the rows any query of the item kept
      int base_n = 0;
      for (int kk = k0; kk <= k1; kk += 32) {
        const int k = kk + lane;
        uint32_t u = 0;
        if (k <= k1) {
          for (int g = 0; g < ng; ++g) u |= mb[g * a.mwords + k];
          if (k == k0) u &= 0xffffffffu << (r0 & 31);
          if (k == k1) u &= 0xffffffffu >> (31 - ((r1 - 1) & 31));
        }
        const int cnt = __popc(u);
        int incl = cnt;
        for (int o = 1; o < 32; o <<= 1) {
          const int v = __shfl_up_sync(0xffffffffu, incl, o);
          if (lane >= o) incl += v;
        }
        int at = base_n + incl - cnt;
        while (u) {
          const int bb = __ffs(u) - 1;
          u &= u - 1;
          rowlist[at++] = 32 * k + bb;
        }
        base_n += __shfl_sync(0xffffffffu, incl, 31);
      }
      if (lane == 0) nrows_s = base_n;
    }
    __syncthreads();
    const int nrows = nrows_s;
    if (warp == ncw) {
      if (lane == 0) {  // producer: the listed rows, in order, through the ring
        for (int i = 0; i < nrows; ++i) {
          const int gi = gbase + i, slot = gi % nslots, ph = gi / nslots;
          if (ph > 0) rr_wait(&empty[slot], (ph - 1) & 1);
          asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sc_smem(&full[slot])),
                       "r"(row_bytes)
                       : "memory");
          asm volatile(
              "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                  sc_smem(ring + (size_t)slot * row_bytes)),
              "l"(ix.corpus + (size_t)(p0 + rowlist[i]) * ds), "r"(row_bytes), "r"(sc_smem(&full[slot]))
              : "memory");
        }
      }
    } else {
      // x of the item's queries (pre-interleaved) while the first rows land
      {
        constexpr int SU = 4;
        const int n4 = ds / 4, tot = ng * n4;
        float4* xs4 = reinterpret_cast<float4*>(xs);
        for (int e0 = tid; e0 < tot; e0 += SNT * SU) {
          float4 xv[SU];
#pragma unroll
          for (int u = 0; u < SU; ++u) {
            const int e = e0 + u * SNT;
            if (e < tot) {
              const int g = e / n4, j = e - g * n4;
              xv[u] = __ldg(reinterpret_cast<const float4*>(a.xint + (size_t)pq[g] * ds) + j);
            }
          }
#pragma unroll
          for (int u = 0; u < SU; ++u)
            if (e0 + u * SNT < tot) xs4[e0 + u * SNT] = xv[u];
        }
      }
      asm volatile("bar.sync 1, %0;" ::"n"(SNT) : "memory");  // the computing warps only
      int nfetch = 0;
      for (int ia = warp; ia < nrows; ia += ncw) {
        const int row = rowlist[ia];
        const int gi = gbase + ia, slot = gi % nslots;
        ++nfetch;
        const bool mine = lane < ng && ((mb[lane * a.mwords + (row >> 5)] >> (row & 31)) & 1u);
        const unsigned act = __ballot_sync(0xffffffffu, mine);
        const int nact = __popc(act);
        if (mine) slotg[warp][__popc(act & ((1u << lane) - 1u))] = lane;
        rr_wait(&full[slot], (gi / nslots) & 1);
        const float* rs = reinterpret_cast<const float*>(ring + (size_t)slot * row_bytes) + coff;
        float2 c[NH][NB];
#pragma unroll
        for (int hh = 0; hh < NH; ++hh)
#pragma unroll
          for (int i = 0; i < NB; ++i) c[hh][i] = *reinterpret_cast<const float2*>(rs + 64 * hh + cstep * i);
        __syncwarp();
        if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sc_smem(&empty[slot])) : "memory");
        float r = sparse_row<NB, NH>(act, nact, xs, ds, coff, c, nz2, lane);
        if (NH == 2) r = __fadd_rn(r, __shfl_down_sync(0xffffffffu, r, 1));
        if (lane < NH * nact && lane % NH == 0) {
          const int g = slotg[warp][lane / NH];
          a.diss[pkey[g] + row] = mono32(r);
        }
        __syncwarp();
      }
      if (a.counters && lane == 0 && nfetch)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 3), (unsigned long long)nfetch);
    }
    gbase += nrows;
    __syncthreads();
  }
}

// Final per-query top-k over the re-ranked candidates (index.py:320-322).
constexpr int FNT = 256;  // (128 measured slower on C2)

struct TopkFinalArgs {
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

__global__ void __launch_bounds__(FNT) k_topk_final(TopkFinalArgs a) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  __shared__ SelectSmem sm;
  __shared__ BucketSmem bs;
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[blockIdx.x] : (int)blockIdx.x;
  const int tid = threadIdx.x, w = a.w;
  const int n = a.cand_n[q];
  int* offs = reinterpret_cast<int*>(smem_raw);  // w+1
  int* pbase = offs + (w + 1);                    // w
  uint32_t* dk = reinterpret_cast<uint32_t*>(pbase + w);  // take_cap
  uint32_t* di = dk + a.take_cap;                          // take_cap
  int* selidx = reinterpret_cast<int*>(di + a.take_cap);   // k
  uintptr_t sp = reinterpret_cast<uintptr_t>(selidx + a.k);
  uint64_t* srt = reinterpret_cast<uint64_t*>((sp + 15) & ~uintptr_t(15));
  for (int c = tid; c <= w; c += FNT) offs[c] = a.qoff[(size_t)q * (w + 1) + c];
  for (int c = tid; c < w; c += FNT) pbase[c] = ix.cl_pos[a.sel[(size_t)q * w + c]];
  __syncthreads();
  const uint32_t* dq = a.diss + a.kbase[q];
  const int* ci = a.cand_idx + (size_t)q * a.take_cap;
  for (int i = tid; i < n; i += FNT) dk[i] = dq[ci[i]];
  __syncthreads();
  const int kk = min(a.k, n);
  auto key = [&](int i) { return dk[i]; };
  // corpus ids are gathered lazily: only the boundary bucket and the k winners need them
  auto tie = [&](int i) {
    const int c = ci[i];
    int lo = 0, hi = w;
    while (hi - lo > 1) {
      int mid = (lo + hi) >> 1;
      if (offs[mid] <= c) lo = mid; else hi = mid;
    }
    return __float_as_uint(__ldg(ix.pmeta + pbase[lo] + (c - offs[lo])).w);
  };
  auto val = [](uint32_t kv) { return unmono32(kv); };
  block_select_bucketed<FNT, uint32_t, float>(n, kk, key, tie, val, selidx, bs, sm);
  int np2 = 1;
  while (np2 < kk) np2 <<= 1;
  for (int i = tid; i < np2; i += FNT) {
    uint64_t v = ~0ull;
    if (i < kk) v = ((uint64_t)dk[selidx[i]] << 32) | tie(selidx[i]);
    srt[i] = v;
  }
  block_bitonic_sort<FNT>(srt, np2);
  const bool euclid = ix.metric == kMetricEuclidean;
  const int gq = a.q0 + q;
  for (int i = tid; i < a.k; i += FNT) {
    int64_t id = -1;
    float sc = __int_as_float(0x7fc00000);
    if (i < kk) {
      const uint64_t v = srt[i];
      id = (int64_t)(uint32_t)v;
      const float df = unmono32((uint32_t)(v >> 32));
      sc = euclid ? df : -df;
    }
    a.out_ids[(size_t)gq * a.k + i] = id;
    a.out_scores[(size_t)gq * a.k + i] = sc;
  }
  if (tid == 0) a.out_count[gq] = kk;
}

// Final top-k (index.py:320-322), warp per query: radix select of the k smallest
// re-ranked distances, then a warp bitonic sort of their (distance, corpus id).
template <int E>
__global__ void k_topk_final_warp(TopkFinalArgs a, int cap, int nq) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int lane = threadIdx.x & 31;
  const int wq = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  if (wq >= nq) return;
  const DevIndexView& ix = a.ix;
  const int q = a.order ? a.order[wq] : wq;
  const int w = a.w;
  const int* qoffq = a.qoff + (size_t)q * (w + 1);
  const int* selq = a.sel + (size_t)q * w;
  const int n = a.cand_n[q];
  const int kk = min(a.k, n);
  uint32_t* stage;
  const WarpSel ws = warp_sel_slice(smem_raw, cap, 0, stage);
  const uint32_t* dq = a.diss + a.kbase[q];
  const int* ci = a.cand_idx + (size_t)q * a.take_cap;
  for (int i = lane; i < n; i += 32) stage[i] = __ldg(dq + __ldg(ci + i));
  __syncwarp();
  auto tie = [&](int i) {
    return __float_as_uint(__ldg(ix.pmeta + cand_pos(ix, qoffq, selq, w, __ldg(ci + i))).w);
  };
  uint64_t v[E];
  if (kk >= n || n <= 32 * E) {
    // every candidate fits the sort: (key, id) bitonic order, the first kk are the top-k
    // (C2: ~115 survivors for k = 100 -- no radix passes)
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int i = lane + 32 * j;
      v[j] = i < n ? ((uint64_t)stage[i] << 32) | tie(i) : ~0ull;
    }
  } else {
    // the selected indices are emitted after the radix passes, when the 256-entry
    // histogram is dead: it holds them (kk <= 32*E <= 256)
    int* out = ws.hist;
    warp_select_smallest(ws, [&](int i) { return stage[i]; }, n, kk, tie,
                         [&](int slot, int i) { out[slot] = i; });
    __syncwarp();
#pragma unroll
    for (int j = 0; j < E; ++j) {
      const int sl = lane + 32 * j;
      v[j] = ~0ull;
      if (sl < kk) {
        const int i = out[sl];
        v[j] = ((uint64_t)stage[i] << 32) | tie(i);
      }
    }
  }
  warp_bitonic_sort<E>(v);
  const bool euclid = ix.metric == kMetricEuclidean;
  const int gq = a.q0 + q;
#pragma unroll
  for (int j = 0; j < E; ++j) {
    const int i = lane + 32 * j;
    if (i < a.k) {
      int64_t id = -1;
      float sc = __int_as_float(0x7fc00000);
      if (i < kk) {
        id = (int64_t)(uint32_t)v[j];
        const float df = unmono32((uint32_t)(v[j] >> 32));
        sc = euclid ? df : -df;
      }
      a.out_ids[(size_t)gq * a.k + i] = id;
      a.out_scores[(size_t)gq * a.k + i] = sc;
    }
  }
  for (int i = 32 * E + lane; i < a.k; i += 32) {  // k beyond the sorted width: padding
    a.out_ids[(size_t)gq * a.k + i] = -1;
    a.out_scores[(size_t)gq * a.k + i] = __int_as_float(0x7fc00000);
  }
  if (lane == 0) a.out_count[gq] = kk;
}

// ---------------------------------------------------------------- launchers

// RRG_WARP_SELECT=0 selects the CTA-per-query selections (k_select_topt, k_topk_final)
// RRG_WARP_SELECT: 1 forces the warp-per-query selections, 0 the CTA-per-query ones;
// unset: warp per query once the batch fills the GPU (>= 1184 queries = 8 per SM)
static bool warp_select_ok(const DevIndexView& ix, int nq) {
  if (ix.opt.warp_select >= 0) return ix.opt.warp_select != 0;
  if (ix.P < ix.m) {
    // a cluster shard: about P/m of the batch's queries have candidates here (w = 1
    // owner-local search); with few of them per SM a CTA per query has the more
    // parallelism -- C4 at G = 8 (~1,250 active queries): 0.08 vs 0.20 ms; unsharded
    // 10k queries: warp 0.26 vs CTA 0.37 ms
    const double active = (double)nq * (double)ix.P / (double)std::max<int64_t>(ix.m, 1);
    return active >= 4736;
  }
  return nq >= 1184;
}


template <typename Kern>
static void opt_in_smem(Kern* kern, int slot) {
  static int done[64][64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev < 0 || dev >= 64 || done[slot][dev]) return;
  cudaFuncAttributes at{};
  cudaFuncGetAttributes(&at, (const void*)kern);
  cudaFuncSetAttribute((const void*)kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                       kMaxSmemPerCta - (int)at.sharedSizeBytes);
  done[slot][dev] = 1;
}

void launch_cluster_prep(const ClusterScoringHost& h, int nq, cudaStream_t st) {
  const DevIndexView& ix = h.ix;
  (k_cand_offsets<<<(nq + 7) / 8, 256, 0, st>>>(ix, h.sel, nq, h.w, h.qoff, h.ncand), note_launch());
  opt_in_smem(k_pairs_build, 15);  // L * 8 bytes: 64 KB at L = 8192 (C4)
  const size_t pb_stage = ((size_t)ix.L * 2 + nq + 1) * 4;
  const int stage_kb = pb_stage <= 160 * 1024;
  (k_pairs_build<<<1, PNT, stage_kb ? pb_stage : (size_t)ix.L * 8, st>>>(
       h.sel, nq, h.w, ix.L, ix.cl_pos, h.ncand, h.pair_off, h.item_off, h.pairs, h.kbase, stage_kb,
       ix.opt.score_order ? ix.cl_order : nullptr),
   note_launch());
  cudaMemsetAsync(h.work_counter, 0, sizeof(int), st);
}

void launch_cluster_scoring(const ClusterScoringHost& h, int nq, cudaStream_t st, bool prep) {
  const DevIndexView& ix = h.ix;
  if (prep) launch_cluster_prep(h, nq, st);
  ClusterScoreArgs a;
  a.ix = ix; a.qcodes = h.qcodes; a.qscale = h.qscale; a.qhead = h.qhead; a.sel = h.sel;
  a.w = h.w; a.qoff = h.qoff; a.pair_off = h.pair_off; a.item_off = h.item_off;
  a.pairs = h.pairs; a.kbase = h.kbase; a.keys = h.keys; a.work_counter = h.work_counter;
  a.dbg_raw1 = h.dbg_raw1; a.dbg_raw2 = h.dbg_raw2; a.dbg_score = h.dbg_score;
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  a.xp = h.xp;
  // tensor-core stage B (r_pad = 32): the int8 products of a work item's 32 queries x 128
  // points in one MMA.  Auto: dense buckets (>= 64 queries per probed cluster on average)
  // -- measured C5 w=64 4.51 -> 4.14 ms, w=16 1.54 -> 1.40 ms; C2 (10 per cluster) 0.13 ->
  // 0.14 ms, where the items hold few queries and the dp4a loop is cheaper
  const bool tc = ix.opt.score_tc >= 0 ? ix.opt.score_tc != 0 : (double)nq * h.w >= 64.0 * ix.L;
  // stage A operands in shared memory while they fit beside 4 CTAs per SM
  const size_t sa = (size_t)(ix.r + kPairsPerItem) * ix.s_pad;
  a.stage_a_bytes = ix.opt.score_stage_a && sa <= 32 * 1024 ? (int)sa : 0;
  const size_t dyn = (size_t)a.stage_a_bytes;
  if (ix.quantized && ix.r_pad == 32 && tc)
    (k_score_cluster<true><<<sms * RRG_SCORE_CTAS, CNT, dyn, st>>>(a), note_launch());
  else if (ix.quantized)
    (k_score_cluster<false><<<sms * RRG_SCORE_CTAS, CNT, dyn, st>>>(a), note_launch());
  else
    (k_score_cluster_f32<<<sms * 4, CNT, 0, st>>>(a), note_launch());
}

static int pow2_at_least(int v) {
  int p = 1;
  while (p < v) p <<= 1;
  return p;
}

size_t select_topt_smem(int w, int take_cap, int k, int kcap) {
  return (size_t)(2 * w + 1) * 4 + (size_t)take_cap * 4 + 32 + (size_t)pow2_at_least(k) * 8 +
         (size_t)kcap * 4 + 16;
}

void launch_select_topt(const SelectTopTHost& h, int nq, cudaStream_t st) {
  SelectArgs a;
  a.ix = h.ix; a.sel = h.sel; a.w = h.w; a.qoff = h.qoff; a.kbase = h.kbase; a.keys = h.keys;
  a.take_cap = h.take_cap; a.rerank = h.rerank; a.k = h.k; a.xx = h.xx; a.cand_pos = h.cand_pos;
  a.cand_n = h.cand_n; a.out_ids = h.out_ids; a.out_scores = h.out_scores;
  a.out_count = h.out_count; a.q0 = h.q0; a.order = h.order; a.sel_keys = h.sel_keys;
  a.sel_ids = h.sel_ids; a.sel_count = h.sel_count;
  a.kcap = h.kcap; a.sort_cap = pow2_at_least(h.k);
  a.cand_idx = h.cand_idx; a.marks = h.marks;
  static int done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, (const void*)k_select_topt);
    cudaFuncSetAttribute((const void*)k_select_topt, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxSmemPerCta - (int)at.sharedSizeBytes);
    done[dev] = 1;
  }
  // warp per query once the batch fills the GPU, for lists up to kSelBigN keys
  // (the membership bits are sized by kcap = min(largest list, 24k): a capped kcap
  // cannot hold every candidate's bit, so the CTA select handles that case)
  // long lists without membership bits (C5's per-query re-rank) take the CTA select
  // with its sampled range: w=64 (~62k keys) 14.5 -> 9.9 ms per batch, w=16 5.5 -> 4.3
  const bool long_lists = !h.marks && h.kcap >= kSelBigN && h.ix.opt.warp_select < 0;
  if (warp_select_ok(h.ix, nq) && h.rerank && !(h.marks && h.kcap >= 24 * 1024) && !long_lists) {
    // 8 warps per CTA; keys staged on-chip only while that keeps >= 32 warps per SM
    const int bits_cap = h.marks ? h.kcap : 0;
    const int stage_cap = 0;  // keys are read through L1
    const size_t per = warp_sel_bytes(stage_cap, bits_cap);
    constexpr int wpc = 8;
    static int wdone[64] = {};
    if (dev >= 0 && dev < 64 && !wdone[dev]) {
      cudaFuncSetAttribute((const void*)k_select_topt_warp,
                           cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemPerCta);
      wdone[dev] = 1;
    }
    (k_select_topt_warp<<<(nq + wpc - 1) / wpc, 32 * wpc, per * wpc, st>>>(a, stage_cap, bits_cap, nq), note_launch());
    return;
  }
  // long lists without membership bits: no key staging (the sampled two-sweep select
  // reads each key twice from HBM anyway), so the CTA's shared memory stays small and
  // 8 CTAs fit per SM (staging 24k keys left 2)
  if (!h.marks && h.kcap >= kSelBigN) a.kcap = 0;
  (k_select_topt<<<nq, TNT, select_topt_smem(h.w, h.take_cap, h.k, a.kcap), st>>>(a), note_launch());
}

// RRG_RR_ASYNC=1 (ix.opt.rr_async): cp.async row staging -- measured on C2 (w=1,
// t=800): register loads 1.134 ms vs cp.async staging 1.249 ms
size_t cluster_rerank_smem(const DevIndexView& ix, int mwords) {
  return (size_t)kRrQ * ix.d_stride * 4 + (size_t)kRrQ * mwords * 4 +
         (ix.opt.rr_async ? (size_t)(XNT / 32) * 2 * ix.d_stride * 4 : 0);
}

// the row plan fits k_rerank_cluster and a query group's x + membership bits of the
// largest cluster fit in shared memory (otherwise the per-query re-rank serves)
bool cluster_rerank_ok(const DevIndexView& ix, int64_t max_cluster) {
  const int nb = ix.pw_leaf_n / 8;
  if (!(ix.corpus_interleaved && (ix.pw_nleaves == 8 || ix.pw_nleaves == 16) &&
        ix.pw_leaf_n % 8 == 0 && (nb == 12 || nb == 15 || nb == 16)))
    return false;
  const int mwords = (int)((max_cluster + 31) / 32) + 1;
  return cluster_rerank_smem(ix, mwords) + 8 * 1024 <= (size_t)kMaxSmemPerCta;
}


void launch_cluster_rerank(const ClusterRerankHost& h, cudaStream_t st) {
  ClusterRerankArgs a;
  a.ix = h.ix; a.queries = h.queries; a.xint = h.xint; a.w = h.w; a.qoff = h.qoff; a.pair_off = h.pair_off;
  a.cand_idx = h.cand_idx; a.cand_n = h.cand_n; a.take_cap = h.take_cap;
  a.rr_item_off = h.rr_item_off; a.pairs = h.pairs; a.kbase = h.kbase; a.marks = h.marks;
  // rows per work item: 256 (few, long items) once the batch's (query, cluster) probes
  // give enough items to fill the GPU; 128 / 32 for small batches (one query's rows
  // spread over many CTAs: C2 batch 1, 4 -> 31 items)
  const int64_t probes = (int64_t)h.nq * h.w;
  a.rr_rows = probes >= 512 ? kRrRows : (probes >= 64 ? 128 : 32);
  // sparse (screened) items: whole clusters (up to kSpRows rows) amortise the item
  // staging; small batches keep the short items that spread one query over CTAs
  if (h.compact) a.rr_rows = probes >= 512 ? kSpRows : std::min(a.rr_rows, kSpRows);
  // the sparse kernels take the items largest cluster first (their work is about
  // proportional to the cluster's rows): in cluster order the long items formed the
  // grid's tail (C2: SMs active 83% of the kernel on average)
  a.ordered = h.compact && h.ix.metric == kMetricEuclidean && h.ix.opt.rr_order;
  (k_rr_items<<<1, PNT, 0, st>>>(h.pair_off, h.ix.cl_pos, h.ix.L, a.rr_rows, h.rr_item_off,
                                 a.ordered ? h.ix.cl_order : nullptr), note_launch());
  a.diss = h.diss; a.work_counter = h.work_counter; a.mwords = h.mwords;
  a.neg_zero = -0.0f;
  a.counters = h.counters;
  cudaMemsetAsync(h.work_counter, 0, sizeof(int), st);
  const size_t sm = cluster_rerank_smem(h.ix, h.mwords);
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (h.compact && h.ix.metric == kMetricEuclidean) {  // screened: sparse per-row kernel
    const size_t ssm = (size_t)kRrQ * h.ix.d_stride * 4 + (size_t)kRrQ * h.mwords * 4;
#define RRG_SP(NB, NH, PF, CT, SLOT)                                                         \
  do {                                                                                       \
    opt_in_smem(k_rerank_sparse<NB, NH, PF, CT>, SLOT);                                      \
    (k_rerank_sparse<NB, NH, PF, CT><<<sms * (CT), SNT, ssm, st>>>(a), note_launch());       \
  } while (0)
    const int nb = h.ix.pw_leaf_n / 8;
    // 1 (default): no register prefetch, 3 CTAs/SM (C2 1.49 -> 1.46 ms, C3 3.36 -> 3.18 ms);
    // 0: the next row prefetched into registers, 2 CTAs/SM
    const int var = h.ix.opt.sparse_variant;
    if (var == 2) {  // ring-staged rows: as many 16 KB-aligned slots as shared memory allows
      const size_t fixed = (ssm + 127) / 128 * 128;
      const size_t rowb = (size_t)h.ix.d_stride * 4;
      // 2 CTAs per SM (one's item staging hidden behind the other's stream) when both
      // fit with >= 12 slots each, else one CTA with the deepest ring
      const int ns2 = ((228 * 1024) / 2 - 8 * 1024 - (int)fixed) / (int)rowb;
      const int ns1 = (kMaxSmemPerCta - 8 * 1024 - (int)fixed) / (int)rowb;
      const int cta = ns2 >= 12 ? 2 : 1;
      const int ns = std::min(32, cta == 2 ? ns2 : ns1);
      if (ns >= 8) {
        const size_t rsm = fixed + (size_t)ns * rowb;
#define RRG_SPR(NB, NH, SLOT)                                                                \
  do {                                                                                       \
    opt_in_smem(k_rerank_sparse_ring<NB, NH>, SLOT);                                         \
    (k_rerank_sparse_ring<NB, NH><<<sms * cta, RNT, rsm, st>>>(a, ns), note_launch());       \
  } while (0)
        const int nb = h.ix.pw_leaf_n / 8;
        if (h.ix.pw_nleaves == 16) {
          if (nb == 12) RRG_SPR(12, 2, 48); else if (nb == 15) RRG_SPR(15, 2, 49); else RRG_SPR(16, 2, 50);
        } else {
          if (nb == 12) RRG_SPR(12, 1, 51); else if (nb == 15) RRG_SPR(15, 1, 52); else RRG_SPR(16, 1, 53);
        }
#undef RRG_SPR
        return;
      }
    }
    if (h.ix.pw_nleaves == 16) {
      if (var == 1) {
        if (nb == 12) RRG_SP(12, 2, false, 2, 42); else if (nb == 15) RRG_SP(15, 2, false, 2, 43);
        else RRG_SP(16, 2, false, 2, 44);
      } else {
        if (nb == 12) RRG_SP(12, 2, true, 1, 36); else if (nb == 15) RRG_SP(15, 2, true, 1, 37);
        else RRG_SP(16, 2, true, 1, 38);
      }
    } else if (var == 1) {
      if (nb == 12) RRG_SP(12, 1, false, 3, 45); else if (nb == 15) RRG_SP(15, 1, false, 3, 46);
      else RRG_SP(16, 1, false, 3, 47);
    } else {
      if (nb == 12) RRG_SP(12, 1, true, 2, 39); else if (nb == 15) RRG_SP(15, 1, true, 2, 40);
      else RRG_SP(16, 1, true, 2, 41);
    }
#undef RRG_SP
    return;
  }
#define RRG_RR_LAUNCH(NB, AS, NH, RM, SLOT)                                      \
  do {                                                                           \
    opt_in_smem(k_rerank_cluster<NB, AS, NH, RM>, SLOT);                         \
    (k_rerank_cluster<NB, AS, NH, RM><<<sms * kCmCtas, XNT, sm, st>>>(a), note_launch()); \
  } while (0)
#define RRG_RR_SK(NB, NH, SLOT)                                                  \
  do {                                                                           \
    if (h.compact) RRG_RR_LAUNCH(NB, false, NH, 2, SLOT + 20);                   \
    else if (h.skip) RRG_RR_LAUNCH(NB, false, NH, 1, SLOT + 16);                 \
    else RRG_RR_LAUNCH(NB, false, NH, 0, SLOT);                                  \
  } while (0)
  const bool as = h.ix.opt.rr_async && h.ix.pw_nleaves == 8 && !h.compact;
  if (h.ix.pw_nleaves == 16) {  // d = 16 leaves (e.g. 1536): scored as two 8-leaf halves
    switch (h.ix.pw_leaf_n / 8) {
      case 12: RRG_RR_SK(12, 2, 12); break;
      case 15: RRG_RR_SK(15, 2, 13); break;
      default: RRG_RR_SK(16, 2, 14); break;
    }
    return;
  }
  // persistent grid: kCmCtas CTAs per SM
  switch (h.ix.pw_leaf_n / 8) {
    case 12: if (as) RRG_RR_LAUNCH(12, true, 1, 0, 4); else RRG_RR_SK(12, 1, 0); break;
    case 15: if (as) RRG_RR_LAUNCH(15, true, 1, 0, 5); else RRG_RR_SK(15, 1, 1); break;
    default: if (as) RRG_RR_LAUNCH(16, true, 1, 0, 6); else RRG_RR_SK(16, 1, 2); break;
  }
#undef RRG_RR_SK
#undef RRG_RR_LAUNCH
}

size_t topk_final_smem(int w, int take_cap, int k) {
  return (size_t)(2 * w + 1) * 4 + (size_t)take_cap * 8 + (size_t)k * 4 + 32 +
         (size_t)pow2_at_least(k) * 8 + 16;
}

void launch_topk_final(const TopkFinalHost& h, int nq, cudaStream_t st) {
  TopkFinalArgs a;
  a.ix = h.ix; a.sel = h.sel; a.w = h.w; a.qoff = h.qoff; a.kbase = h.kbase; a.diss = h.diss;
  a.cand_idx = h.cand_idx; a.cand_n = h.cand_n; a.take_cap = h.take_cap; a.k = h.k;
  a.out_ids = h.out_ids; a.out_scores = h.out_scores; a.out_count = h.out_count; a.q0 = h.q0;
  a.order = h.order;
  const size_t per = warp_sel_bytes(h.take_cap, 0);
  // warp per query once the batch fills the GPU; tiny batches get a CTA per query
  if (warp_select_ok(h.ix, nq) && h.k <= 256 && per <= 24 * 1024) {
    const int wpc = (int)std::max<size_t>(1, std::min<size_t>(8, (56 * 1024) / per));
    const unsigned grid = (unsigned)((nq + wpc - 1) / wpc);
    const size_t sm = per * wpc;
#define RRG_TKW(E, SLOT)                                                          \
  do {                                                                            \
    opt_in_smem(k_topk_final_warp<E>, SLOT);                                      \
    (k_topk_final_warp<E><<<grid, 32 * wpc, sm, st>>>(a, h.take_cap, nq), note_launch());          \
  } while (0)
    if (h.k <= 32) RRG_TKW(1, 8);
    else if (h.k <= 64) RRG_TKW(2, 9);
    else if (h.k <= 128) RRG_TKW(4, 10);
    else RRG_TKW(8, 11);
#undef RRG_TKW
    return;
  }
  opt_in_smem(k_topk_final, 3);
  (k_topk_final<<<nq, FNT, topk_final_smem(h.w, h.take_cap, h.k), st>>>(a), note_launch());
}

// ======================================================= sparse phase-1 exchange
// A rank's local top-t lists are mostly short or empty when its clusters hold few
// of a query's probes (w = 1: one rank holds all of them), so they travel packed:
// counts -> offsets (one CTA scan), then one warp per query copies its list.
__global__ void __launch_bounds__(PNT) k_pack_offsets(const int* __restrict__ counts, int nq,
                                                      int* __restrict__ off) {
  __shared__ int tot;
  for (int i = threadIdx.x; i < nq; i += PNT) off[i] = counts[i];
  __syncthreads();
  block_exclusive_scan_inplace(off, nq, &tot);
  if (threadIdx.x == 0) off[nq] = tot;
}

__global__ void k_pack_lists(const uint32_t* __restrict__ keys, const uint32_t* __restrict__ ids,
                             int nq, int cap, const int* __restrict__ off,
                             uint32_t* __restrict__ pk, uint32_t* __restrict__ pi) {
  const int q = blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5), lane = threadIdx.x & 31;
  if (q >= nq) return;
  const int o = off[q], n = off[q + 1] - o;
  for (int j = lane; j < n; j += 32) {
    pk[o + j] = keys[(size_t)q * cap + j];
    pi[o + j] = ids[(size_t)q * cap + j];
  }
}

// G packed lists (stride elements each, offsets [G][nq+1]) -> the [G][nq][cap] layout k_merge reads
__global__ void k_unpack_lists(const uint32_t* __restrict__ pk, const uint32_t* __restrict__ pi,
                               const int* __restrict__ off, int G, int nq, int64_t stride, int cap,
                               uint32_t* __restrict__ keys, uint32_t* __restrict__ ids,
                               int* __restrict__ counts) {
  const int64_t gq = (int64_t)blockIdx.x * (blockDim.x >> 5) + (threadIdx.x >> 5);
  const int lane = threadIdx.x & 31;
  if (gq >= (int64_t)G * nq) return;
  const int g = (int)(gq / nq), q = (int)(gq % nq);
  const int* og = off + (size_t)g * (nq + 1);
  const int o = og[q], n = min(og[q + 1] - o, cap);
  const uint32_t* sk = pk + g * stride + o;
  const uint32_t* si = pi + g * stride + o;
  uint32_t* dk = keys + (size_t)gq * cap;
  uint32_t* di = ids + (size_t)gq * cap;
  for (int j = lane; j < n; j += 32) {
    dk[j] = sk[j];
    di[j] = si[j];
  }
  if (lane == 0) counts[gq] = n;
}

void launch_pack_candidates(int nq, int cap, const uint32_t* keys, const uint32_t* ids,
                            const int* counts, uint32_t* pk, uint32_t* pi, int* off, cudaStream_t st) {
  (k_pack_offsets<<<1, PNT, 0, st>>>(counts, nq, off), note_launch());
  (k_pack_lists<<<(nq + 7) / 8, 256, 0, st>>>(keys, ids, nq, cap, off, pk, pi), note_launch());
}

void launch_unpack_candidates(int nq, int G, int64_t stride, int cap, const uint32_t* pk,
                              const uint32_t* pi, const int* off, uint32_t* keys, uint32_t* ids,
                              int* counts, cudaStream_t st) {
  const int64_t n = (int64_t)G * nq;
  (k_unpack_lists<<<(unsigned)((n + 7) / 8), 256, 0, st>>>(pk, pi, off, G, nq, stride, cap, keys, ids,
                                                          counts), note_launch());
}

}  // namespace rrg
