// rrg_screen.cu -- exact-by-construction screen of the re-rank on the tensor cores.
//
// The reference re-ranks the top-t candidates of a query with the exact f32 distance
// in NumPy's pairwise order (index.py:278-283,318-322) and keeps the k smallest by
// (distance, id).  Evaluating that order costs 3 unfusable FP32 ops per element for
// all t candidates, which bounds the re-rank at C2 by the FP32 pipe.  Most of those
// candidates cannot reach the top k, and a bound proves which:
//
//   with any per-cluster vector mu (the cluster mean here), x' = x - mu, r = c - mu,
//   D = ||x - c||^2 = ||x'||^2 + ||r||^2 - 2 x'.r   (exact in real arithmetic).
//   The tensor cores compute G = x^'.r^ from fp16 roundings x^' ~ x'/2^eq and
//   r^ ~ r/2^er (power-of-two scales), and
//     |x'.r - 2^(eq+er) x^'.r^| <= 2^(eq+er) (|x^'| |e_r| + |e_x| |r^| + |e_x| |e_r|)
//   (Cauchy-Schwarz on the exact rounding residuals e, whose norms are computed in
//   f64 from the stored values), |G - x^'.r^| <= eps_acc |x^'| |r^| for the f32
//   accumulation (eps_acc = (d + 32) 2^-21, four times the truncating-sum bound).
//   So D lies in [S - E, S + E] with S = ||x'||^2 + ||r||^2 - 2^(1+eq+er) G.  The
//   exact f32 pairwise distance (positive terms, depth <= d) lies within
//   eta = (d + 4) 2^-24 of D relatively, giving per candidate
//     LB = max(S - E, 0) (1 - eta)  <=  dist_f32  <=  UB = (S + E)(1 + eta).
//   With T = the k-th smallest UB of the query's t candidates, k candidates have
//   dist <= T, so the k-th smallest dist is <= T; a candidate with LB > T has
//   dist > T and can never be in the top k -- not even by an id tie.  Only the
//   candidates with LB <= T ("survivors") are re-ranked exactly; the result is the
//   reference's, bit for bit, with the FP32 work cut from t to ~k per query.
//
// k_rr_screen is a warp-specialised persistent kernel: warp 0 streams the fp16
// residual blocks (128 rows x d, pre-tiled in the UMMA canonical K-major layout) with
// cp.async.bulk into a 6-stage ring, warp 1 issues tcgen05.mma kind::f16
// (M = 128 rows, N = 16 queries of a work item, K = 16 per instruction) into a
// double-buffered TMEM accumulator, warps 2-5 build the queries' fp16 tiles and turn
// the accumulators (tcgen05.ld) into (LB, UB) for the marked (query, row) pairs.
// k_rr_thresh then finds T per query and clears the non-survivors' bits.
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

constexpr int kScrRows = 128;                   // rows per block = MMA M = TMEM lanes
constexpr int kScrChunk = kScrRows * 32;        // bytes of one K = 16 chunk of a block
constexpr int kScrStageChunks = 4;              // 16 KB per ring stage
constexpr int kScrStagesMax = 12;              // ring depth: as many stages as shared memory allows
constexpr int kScrStageBytes = kScrStageChunks * kScrChunk;
constexpr int kScrRingMin = 6 * kScrStageBytes;
constexpr int kScrThreads = 192;                // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
// Measured on C2 (per-stage probes, RRG_SCREEN_DIAG): the stream alone runs at ~93% of
// HBM peak; the MMAs add ~60 us per batch whatever the operand swizzle (none / 128 B),
// the number of accumulators the K chunks rotate over (1 / 4), the TMEM item buffers
// (2 / 4) -- and an L2 prefetch two items ahead made it slower (0.66 vs 0.51 ms).
constexpr int kScrAcc = 1;   // accumulators per item (K chunks rotate over them)
constexpr int kScrTBuf = 4;  // item accumulators in TMEM: the MMAs run up to 3 items ahead
constexpr int kScrTmemCols = kScrTBuf * kScrAcc * kRrQ;  // 64
constexpr int kScrMaxKc = 120;                  // d <= 1920: two group records + the ring fit

// Group record (one per (cluster, <= kRrQ queries) work group, built by k_rr_groups and
// bulk-copied by the screen's producer): the queries' fp16 residual tile in the UMMA
// K-major layout (N = kRrQ rows, 512 B per K chunk), then per slot the bound terms.
struct GroupSlot {
  double xx;   // ||x - mu_l||^2
  double sc;   // 2^e_q
  float nxh;   // ||x^'|| (scaled units, rounded up)
  float nex;   // ||x'/2^e_q - x^'||
  int pkey;    // key-array offset of the (query, probe) pair
  int pad;
};
static_assert(sizeof(GroupSlot) == 32, "group slot layout");
__host__ __device__ constexpr size_t grp_rec_bytes(int kc) {
  return ((size_t)kc * 512 + kRrQ * sizeof(GroupSlot) + 16 + 127) / 128 * 128;
}

int screen_max_dim() { return kScrMaxKc * 16; }
// ring stages for a d: the two group records first, the rest of the CTA's shared memory
// for the ring (d = 768: 10 stages = 160 KB in flight per SM; d = 1536: 8)
int screen_stages(int kc) {
  const int avail = (kMaxSmemPerCta - 4096 - 1024 - 2 * (int)grp_rec_bytes(kc)) / kScrStageBytes;
  return std::max(1, std::min(kScrStagesMax, avail));
}
size_t screen_smem(int kc) { return (size_t)screen_stages(kc) * kScrStageBytes + 2 * grp_rec_bytes(kc) + 1024; }
size_t screen_group_bytes(int kc) { return grp_rec_bytes(kc); }

// halves offset of element e of row rr inside a block.  The residual rows are laid out
// for UMMA's 128-byte-swizzled K-major operand: K in 64-element (128 B) chunks of
// 128 rows x 128 B = 16 KB (one ring stage), 8-row atoms of 1 KB, and the 16-byte
// piece j of row r stored at piece j ^ (r % 8) -- the tensor core reads it at full
// shared-memory bandwidth (the no-swizzle layout measured ~1 us of MMA time per 128-row
// block on C2, not hidden by the stream)
__device__ __forceinline__ size_t scr_half_off(int rr, int e) {
  return (size_t)(e >> 6) * (kScrStageBytes / 2) + (rr >> 3) * 512 + (rr & 7) * 64 +
         ((((e & 63) >> 3) ^ (rr & 7)) << 3) + (e & 7);
}

// ------------------------------------------------------------------ build
// Per-cluster mean of the held rows (natural element order), f64 sums rounded to f32.
__global__ void k_scr_mean(DevIndexView ix, float* __restrict__ mu) {
  const int l = blockIdx.x;
  const int p0 = ix.cl_pos[l], m = ix.cl_pos[l + 1] - p0;
  for (int j = threadIdx.x; j < ix.d; j += blockDim.x) {
    const int col = ix.elem_perm ? __ldg(ix.elem_perm + j) : j;
    double acc = 0.0;
    for (int p = 0; p < m; ++p) acc += (double)__ldg(ix.corpus + (size_t)(p0 + p) * ix.d_stride + col);
    mu[(size_t)l * ix.d + j] = m > 0 ? (float)(acc / m) : 0.f;
  }
}

__device__ __forceinline__ double warp_sum_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  return v;
}
__device__ __forceinline__ double warp_max_d(double v) {
  for (int o = 16; o > 0; o >>= 1) v = fmax(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

// Warp per held row: r = c - mu_l in f64 (exact for f32 operands of nearby exponents),
// e_row with max|r| / 2^e_row in [2^14, 2^15), the fp16 rounding r^ of r / 2^e_row
// into the tiled plane, and ||r||^2, ||r^||, ||r/2^e - r^|| from the stored values.
__global__ void k_scr_rows(DevIndexView ix, uint16_t* __restrict__ plane, double* __restrict__ rr_out,
                           float4* __restrict__ meta) {
  const int64_t p = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (p >= ix.P) return;
  int lo = 0, hi = ix.L;  // last cluster whose first position is <= p (skips empty clusters)
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (__ldg(ix.cl_pos + mid) <= p) lo = mid; else hi = mid;
  }
  const int l = lo;
  const int j = (int)(p - ix.cl_pos[l]);
  uint16_t* blk = plane + ((size_t)ix.scr_blk0[l] + j / kScrRows) * ix.scr_kc * (kScrChunk / 2);
  const int rr = j % kScrRows;
  const float* row = ix.corpus + (size_t)p * ix.d_stride;
  const float* mu = ix.scr_mu + (size_t)l * ix.d;
  auto resid = [&](int e) {
    const int col = ix.elem_perm ? __ldg(ix.elem_perm + e) : e;
    return (double)__ldg(row + col) - (double)__ldg(mu + e);
  };
  double amax = 0.0;
  for (int e = lane; e < ix.d; e += 32) amax = fmax(amax, fabs(resid(e)));
  amax = warp_max_d(amax);
  const int ex = amax > 0.0 ? ilogb(amax) - 14 : 0;
  const double inv = ldexp(1.0, -ex);
  double s_r = 0.0, s_h = 0.0, s_e = 0.0;
  for (int e = lane; e < ix.scr_kc * 16; e += 32) {
    uint16_t hb = 0;
    if (e < ix.d) {
      const double r = resid(e);
      const __half h = __double2half(r * inv);
      const double hd = (double)__half2float(h);
      const double er = r * inv - hd;
      s_r += r * r;
      s_h += hd * hd;
      s_e += er * er;
      hb = __half_as_ushort(h);
    }
    blk[scr_half_off(rr, e)] = hb;
  }
  s_r = warp_sum_d(s_r);
  s_h = warp_sum_d(s_h);
  s_e = warp_sum_d(s_e);
  if (lane == 0) {
    rr_out[p] = s_r;
    meta[p] = make_float4(__double2float_ru(sqrt(s_h)), __double2float_ru(sqrt(s_e)), (float)ex, 0.f);
  }
}

void launch_screen_build(const DevIndexView& v, float* mu, uint16_t* plane, size_t plane_bytes,
                         double* rr, float4* meta, cudaStream_t st) {
  cudaMemsetAsync(plane, 0, plane_bytes, st);  // pad rows of every cluster's last block
  (k_scr_mean<<<v.L, 256, 0, st>>>(v, mu), note_launch());
  DevIndexView w = v;
  w.scr_mu = mu;
  const int64_t warps = v.P;
  (k_scr_rows<<<(unsigned)((warps + 7) / 8), 256, 0, st>>>(w, plane, rr, meta), note_launch());
}

// ------------------------------------------------------------------ tcgen05 helpers
__device__ __forceinline__ uint32_t s_addr(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, 128-byte swizzle (A: the residual rows): SBO 1024 B between 8-row atoms,
// LBO unused (1), version 1, layout type 2; a K = 16 step inside the 128-byte row
// advances the start address by 32 B
__device__ __forceinline__ uint64_t scr_desc_sw128(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | (1ull << 16) | ((uint64_t)(1024 >> 4) << 32) | (1ull << 46) |
         (2ull << 61);
}
// K-major, no swizzle (B: the group's query tile): start >> 4, LBO (K direction) 128 B,
// SBO (8-row groups) 256 B, version 1
__device__ __forceinline__ uint64_t scr_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}
// kind::f16 instruction descriptor: D f32, A f16, B f16, both K-major, N = 16, M = 128
constexpr uint32_t kScrIdesc = (1u << 4) | ((uint32_t)(kRrQ >> 3) << 17) | ((uint32_t)(kScrRows >> 4) << 24);

__device__ __forceinline__ void scr_mma(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(kScrIdesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void scr_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(s_addr(bar))
               : "memory");
}
__device__ __forceinline__ void scr_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "SCR_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SCR_WAIT_%=;\n\t}" ::"r"(s_addr(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void scr_arrive(uint64_t* bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(s_addr(bar)) : "memory");
}
__device__ __forceinline__ void scr_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(s_addr(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void scr_bulk(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(s_addr(bar))
      : "memory");
}
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory"); }
__device__ __forceinline__ void epi_sync() { asm volatile("bar.sync 1, 128;" ::: "memory"); }

// Group records: block per (cluster, query group); warp per slot.  x' = x - mu_l in
// f64, e_q with max|x'| / 2^e_q in [2^14, 2^15), x^' = fp16(x' / 2^e_q) into the tile,
// and the norms the bound needs, from the stored values.
__global__ void __launch_bounds__(512) k_rr_groups(DevIndexView ix, const float* __restrict__ queries, int w,
                                                   const int* __restrict__ qoff, const int* __restrict__ pair_off,
                                                   const int* __restrict__ pairs, const int* __restrict__ kbase,
                                                   const int* __restrict__ grp_off, unsigned char* __restrict__ grec) {
  const int gid = blockIdx.x;
  const int L = ix.L, d = ix.d, KC = ix.scr_kc;
  if (gid >= grp_off[L]) return;  // the grid is sized by an upper bound
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  // the group's cluster: the largest l with grp_off[l] <= gid, by a 32-way search per
  // warp (3 dependent loads at L = 2048 instead of 11 for a binary search)
  int lo = 0, hi = L;  // grp_off[lo] <= gid < grp_off[hi]
  while (hi - lo > 1) {
    const int step = (hi - lo + 31) >> 5;
    const int idx = lo + lane * step;
    const bool le = idx < hi && __ldg(grp_off + idx) <= gid;
    const int last = 31 - __clz(__ballot_sync(0xffffffffu, le));  // lane 0 always holds
    lo += last * step;
    hi = min(hi, lo + step);
  }
  const int l = lo, gi = gid - grp_off[l];
  const int j0 = pair_off[l] + gi * kRrQ;
  const int ng = min(kRrQ, pair_off[l + 1] - j0);
  unsigned char* rec = grec + (size_t)gid * grp_rec_bytes(KC);
  uint16_t* bt = reinterpret_cast<uint16_t*>(rec);
  GroupSlot* slots = reinterpret_cast<GroupSlot*>(rec + (size_t)KC * 512);
  const float* mu = ix.scr_mu + (size_t)l * d;
  for (int g = warp; g < kRrQ; g += blockDim.x >> 5) {
    if (g >= ng) {  // unused slot: zero tile rows (their columns are never read)
      for (int e = lane; e < KC * 16; e += 32)
        bt[(size_t)(e >> 4) * 256 + (g >> 3) * 128 + ((e & 15) >> 3) * 64 + (g & 7) * 8 + (e & 7)] = 0;
      continue;
    }
    const int pr = pairs[j0 + g];
    const int q = pr / w, c = pr % w;
    const float* x = queries + (size_t)q * d;
    // x' = x - mu (exact in f64): each lane owns runs of 8 consecutive elements, so a run
    // is two 16-byte loads of x and of mu and one 16-byte store of 8 fp16 into the tile
    // (8 consecutive K elements of one row are one 16-byte core-matrix row)
    const int KE = KC * 16;
    const bool vec = (d & 7) == 0;
    auto load8 = [&](int e0, double (&xr)[8]) {
      if (vec && e0 + 8 <= d) {
        const float4 xa = __ldg(reinterpret_cast<const float4*>(x + e0));
        const float4 xb = __ldg(reinterpret_cast<const float4*>(x + e0 + 4));
        const float4 ma = __ldg(reinterpret_cast<const float4*>(mu + e0));
        const float4 mb = __ldg(reinterpret_cast<const float4*>(mu + e0 + 4));
        xr[0] = (double)xa.x - ma.x; xr[1] = (double)xa.y - ma.y; xr[2] = (double)xa.z - ma.z;
        xr[3] = (double)xa.w - ma.w; xr[4] = (double)xb.x - mb.x; xr[5] = (double)xb.y - mb.y;
        xr[6] = (double)xb.z - mb.z; xr[7] = (double)xb.w - mb.w;
      } else {
#pragma unroll
        for (int u = 0; u < 8; ++u)
          xr[u] = e0 + u < d ? (double)__ldg(x + e0 + u) - (double)__ldg(mu + e0 + u) : 0.0;
      }
    };
    double amax = 0.0;
#pragma unroll 3
    for (int e0 = lane * 8; e0 < KE; e0 += 256) {
      double xr[8];
      load8(e0, xr);
#pragma unroll
      for (int u = 0; u < 8; ++u) amax = fmax(amax, fabs(xr[u]));
    }
    amax = warp_max_d(amax);
    const int ex = amax > 0.0 ? ilogb(amax) - 14 : 0;
    const double inv = ldexp(1.0, -ex);
    double s_x = 0.0, s_h = 0.0, s_e = 0.0;
#pragma unroll 3
    for (int e0 = lane * 8; e0 < KE; e0 += 256) {
      double xr[8];
      load8(e0, xr);
      uint32_t packed[4];
#pragma unroll
      for (int u = 0; u < 8; ++u) {
        // any fp16 near x'/2^e will do: the bound uses the exact residual of the stored value
        const __half hv = __float2half_rn((float)(xr[u] * inv));
        const double hd = (double)__half2float(hv);
        const double er = xr[u] * inv - hd;
        s_x += xr[u] * xr[u];
        s_h += hd * hd;
        s_e += er * er;
        const uint32_t hb = __half_as_ushort(hv);
        packed[u >> 1] = (u & 1) ? (packed[u >> 1] | (hb << 16)) : hb;
      }
      *reinterpret_cast<uint4*>(bt + (size_t)(e0 >> 4) * 256 + (g >> 3) * 128 + ((e0 & 15) >> 3) * 64 + (g & 7) * 8) =
          make_uint4(packed[0], packed[1], packed[2], packed[3]);
    }
    s_x = warp_sum_d(s_x);
    s_h = warp_sum_d(s_h);
    s_e = warp_sum_d(s_e);
    if (lane == 0) {
      GroupSlot gs;
      gs.xx = s_x;
      gs.sc = ldexp(1.0, ex);
      gs.nxh = __double2float_ru(sqrt(s_h));
      gs.nex = __double2float_ru(sqrt(s_e));
      gs.pkey = kbase[q] + qoff[(size_t)q * (w + 1) + c];
      gs.pad = 0;
      slots[g] = gs;
    }
  }
  if (threadIdx.x == 0) *reinterpret_cast<int*>(rec + (size_t)KC * 512 + kRrQ * sizeof(GroupSlot)) = ng;
}

struct ScreenArgs {
  DevIndexView ix;
  const int* pair_off;
  const uint32_t* marks;
  const int* item_off;   // [L+1]: ceil(pairs_l / kRrQ) * blocks_l, scanned
  const int* grp_off;    // [L+1]: ceil(pairs_l / kRrQ), scanned
  const unsigned char* grec;  // group records
  float* ub;             // per candidate bounds (key-array layout)
  float* lb;
  double eta, eps_acc;
  int nst;               // ring stages
  int64_t* counters;     // rrg_search_counters (nullptr unless enabled): [2] += rows streamed
};

__global__ void __launch_bounds__(kScrThreads, 1) k_rr_screen(ScreenArgs a) {
  extern __shared__ __align__(1024) unsigned char scr_sm[];
  __shared__ uint64_t full[kScrStagesMax], empty[kScrStagesMax], bfull[2], bempty[2], tfull[kScrTBuf],
      tempty[kScrTBuf], sfull[kScrTBuf], sempty[kScrTBuf];
  // per item (indexed like the TMEM buffers) the group's slot terms + slot count, copied
  // by the producer: the epilogue never holds a group tile buffer, so the producer may
  // refill one as soon as its MMAs are done (with the epilogue gating the tile buffers,
  // the stream stalled behind it: C3 screen 1.21 ms, MMA-only or epilogue-only ~0.7)
  constexpr int kSlotBytes = kRrQ * (int)sizeof(GroupSlot) + 16;
  __shared__ __align__(128) unsigned char sslot[kScrTBuf][kSlotBytes];
  __shared__ uint32_t tmem_base;
  const DevIndexView& ix = a.ix;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(scr_sm) + 1023) & ~uintptr_t(1023));
  unsigned char* ring = base;
  const int nst = a.nst;
  unsigned char* gbuf = base + (size_t)nst * kScrStageBytes;
  const int KC = ix.scr_kc, L = ix.L;
  const int rec_bytes = (int)grp_rec_bytes(KC);
  const int total = a.item_off[L];
  const int i0 = (int)((int64_t)total * blockIdx.x / gridDim.x);
  const int i1 = (int)((int64_t)total * (blockIdx.x + 1) / gridDim.x);
  if (i0 >= i1) return;  // uniform over the CTA, before any barrier or TMEM use

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 64;" ::"r"(s_addr(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < nst; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&empty[i])));
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&bfull[i])));
      // freed by the MMAs of the group (commit) and by the 4 epilogue warps
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&bempty[i])));
    }
    for (int i = 0; i < kScrTBuf; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&tfull[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(s_addr(&tempty[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&sfull[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(s_addr(&sempty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;

  // item -> (cluster, 128-row block, query group).  A CTA's items are a contiguous
  // range; within a cluster the query groups of one block are adjacent, so a block that
  // several groups screen is re-read from L2 right after its first (HBM) read -- group-
  // major order re-streamed it from HBM (C3: 1.92 M rows streamed for 1 M rows).  After
  // one binary search the roles step through their items (a search per item costs ~10
  // dependent L2 loads, which throttled the producer).
  struct ItemIt {
    int l, gi, b, nb, ng;  // ng = query groups of cluster l
  };
  auto it_begin = [&](int i) {
    ItemIt t;
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.item_off + mid) <= i) lo = mid; else hi = mid;
    }
    t.l = lo;
    t.nb = __ldg(ix.scr_blk0 + lo + 1) - __ldg(ix.scr_blk0 + lo);
    const int local = i - __ldg(a.item_off + lo);
    t.ng = (__ldg(a.item_off + lo + 1) - __ldg(a.item_off + lo)) / t.nb;
    t.b = local / t.ng;
    t.gi = local % t.ng;
    return t;
  };
  auto it_next = [&](ItemIt& t) {  // only called while items remain
    if (++t.gi < t.ng) return;
    t.gi = 0;
    if (++t.b < t.nb) return;
    t.b = 0;
    do {  // next cluster with items
      ++t.l;
      t.nb = __ldg(ix.scr_blk0 + t.l + 1) - __ldg(ix.scr_blk0 + t.l);
    } while (__ldg(a.item_off + t.l + 1) == __ldg(a.item_off + t.l));
    t.ng = (__ldg(a.item_off + t.l + 1) - __ldg(a.item_off + t.l)) / t.nb;
  };
  if (warp == 0) {
    if (lane == 0) {  // producer: group records and the CTA's blocks through the ring
      int slot = 0, pass = 0, j = -1, pl = -1, pg = -1;
      long long rows_streamed = 0;  // rrg_search_counters[2] (whole 8-row atoms)
      ItemIt t = it_begin(i0);
      for (int i = i0, it = 0; i < i1; ++i, ++it, i < i1 ? it_next(t) : void()) {
        const int l = t.l, gi = t.gi, b = t.b;
        const unsigned char* grec = a.grec + (size_t)(a.grp_off[l] + gi) * rec_bytes;
        const int ab = it % kScrTBuf, u = it / kScrTBuf;
        if (u > 0) scr_wait(&sempty[ab], (u - 1) & 1);
        scr_expect_tx(&sfull[ab], kSlotBytes);
        scr_bulk(s_addr(sslot[ab]), grec + (size_t)KC * 512, kSlotBytes, &sfull[ab]);
        if (l != pl || gi != pg) {
          ++j; pl = l; pg = gi;
          const int buf = j & 1;
          if (j >= 2) scr_wait(&bempty[buf], ((j >> 1) - 1) & 1);
          scr_expect_tx(&bfull[buf], KC * 512);
          scr_bulk(s_addr(gbuf + buf * rec_bytes), grec, KC * 512, &bfull[buf]);
        }
        const unsigned char* src = reinterpret_cast<const unsigned char*>(ix.scr_plane) +
                                   ((size_t)(ix.scr_blk0[l] + b) * KC) * kScrChunk;
        // a stage is 16 row atoms of 1 KB (8 rows x 128 B): a cluster's last block
        // copies only the atoms holding its rows (the padding rows' products land in
        // accumulator rows the epilogue never reads)
        const int mrows = min(kScrRows, (ix.cl_pos[l + 1] - ix.cl_pos[l]) - b * kScrRows);
        const uint32_t sbytes = (uint32_t)((mrows + 7) >> 3) * (kScrStageBytes / (kScrRows / 8));
        rows_streamed += (mrows + 7) & ~7;
        for (int c0 = 0; c0 < KC; c0 += kScrStageChunks) {
          if (pass > 0) scr_wait(&empty[slot], (pass - 1) & 1);
          scr_expect_tx(&full[slot], sbytes);
          scr_bulk(s_addr(ring + slot * kScrStageBytes), src + (size_t)c0 * kScrChunk, sbytes, &full[slot]);
          if (++slot == nst) { slot = 0; ++pass; }
        }
      }
      if (a.counters)
        atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 2), (unsigned long long)rows_streamed);
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      // descriptors advance by plain adds (start address field = addr >> 4, no carry for
      // shared-memory addresses): the issue loop was ~42 instructions per MMA and, sharing
      // its SM sub-partition with an epilogue warp, paced the whole kernel (C3: 1.20 ms,
      // vs 0.65 with the epilogue's arithmetic off and 0.71 with the MMAs off)
      static_assert(kScrAcc == 1 && kScrStageBytes % 16 == 0, "one accumulator per item");
      const uint64_t ring_desc = scr_desc_sw128(s_addr(ring));
      int slot = 0, pass = 0, j = -1, pl = -1, pg = -1;
      const bool mma_on = ix.opt.screen_diag == 0;
      ItemIt t = it_begin(i0);
      for (int i = i0, it = 0; i < i1; ++i, ++it, i < i1 ? it_next(t) : void()) {
        const int l = t.l, gi = t.gi, b = t.b, nb = t.nb;
        if (l != pl || gi != pg) {
          ++j; pl = l; pg = gi;
          scr_wait(&bfull[j & 1], (j >> 1) & 1);
          fence_after();
        }
        const int ab = it % kScrTBuf, u = it / kScrTBuf;
        if (u > 0) {
          scr_wait(&tempty[ab], (u - 1) & 1);
          fence_after();
        }
        uint64_t bd = scr_desc(s_addr(gbuf + (j & 1) * rec_bytes));
        const uint32_t dt = tmem + (uint32_t)(ab * kRrQ);
        for (int c0 = 0; c0 < KC; c0 += kScrStageChunks) {
          scr_wait(&full[slot], pass & 1);
          fence_after();
          const uint64_t ad = ring_desc + (uint64_t)(slot * (kScrStageBytes >> 4));
          if (mma_on) {
            // a K16 step is 32 B inside the 128-byte swizzle atom (A) and one 512-byte
            // K chunk of the group tile (B)
            scr_mma(dt, ad, bd, c0 > 0 ? 1u : 0u);
#pragma unroll
            for (int c = 1; c < kScrStageChunks; ++c) scr_mma(dt, ad + 2 * c, bd + 32 * c, 1u);
          }
          bd += 32 * kScrStageChunks;
          scr_commit(&empty[slot]);
          if (++slot == nst) { slot = 0; ++pass; }
        }
        scr_commit(&tfull[ab]);
        if (t.ng > 1 || b + 1 == nb || i + 1 == i1) scr_commit(&bempty[j & 1]);  // the group's tile is read
      }
    }
  } else {
    // epilogue warps: TMEM lane quarter = warp % 4, one block row per thread
    const int q4 = warp & 3, row = q4 * 32 + lane;
    const double eta = a.eta, eps = a.eps_acc;
    ItemIt t = it_begin(i0);
    for (int i = i0, it = 0; i < i1; ++i, ++it, i < i1 ? it_next(t) : void()) {
      const int l = t.l, b = t.b;
      const int ab = it % kScrTBuf, u = it / kScrTBuf;
      const GroupSlot* slots = reinterpret_cast<const GroupSlot*>(sslot[ab]);
      const int p0 = ix.cl_pos[l], m = ix.cl_pos[l + 1] - p0;
      const int jr = b * kScrRows + row;
      // bounds for every (row, slot) of the item: the candidate range of a (query, probe)
      // pair covers all m rows of the cluster, and entries outside the query's top t are
      // never read -- cheaper than loading the membership bits first
      const bool live = jr < m;
      double rr = 0.0;
      float4 rm = make_float4(0.f, 0.f, 0.f, 0.f);
      if (live) {
        rr = __ldg(ix.scr_rr + p0 + jr);
        rm = __ldg(ix.scr_rmeta + p0 + jr);
      }
      scr_wait(&tfull[ab], u & 1);  // (the slot copy was issued before the item's stream)
      fence_after();
      scr_wait(&sfull[ab], u & 1);
      const int ng = *reinterpret_cast<const int*>(sslot[ab] + kRrQ * sizeof(GroupSlot));
      float gsum[kRrQ];
#pragma unroll
      for (int g = 0; g < kRrQ; ++g) gsum[g] = 0.f;
      const int nacc = min(kScrAcc, KC);  // accumulators the item's chunks wrote
#pragma unroll
      for (int ac = 0; ac < kScrAcc; ++ac) {
        uint32_t v[kRrQ];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
            : "r"(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)((ab * kScrAcc + ac) * kRrQ)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (ac < nacc)
#pragma unroll
          for (int g = 0; g < kRrQ; ++g) gsum[g] += __uint_as_float(v[g]);
      }
      fence_before();
      __syncwarp();
      if (lane == 0) scr_arrive(&tempty[ab]);
      if (live && ix.opt.screen_diag < 2) {
        // f32 arithmetic; its own rounding (a handful of ops on magnitudes <= xx + rr +
        // 2|x'.r|) is covered by the 2^-18 slack and the (1 +- 2^-20) factors
        const float rsc = ldexpf(1.f, (int)rm.z), nrh = rm.x, ner = rm.y, rrf = (float)rr;
        const float etap = (float)eta * (1.f + 0x1p-20f), epsf = (float)eps;
#pragma unroll
        for (int g = 0; g < kRrQ; ++g) {
          if (g >= ng) break;
          const GroupSlot gs = slots[g];
          const float sc = (float)gs.sc * rsc;
          const float nxh = gs.nxh, nex = gs.nex, xx = (float)gs.xx;
          const float cross = 2.f * sc * gsum[g];
          const float S = (xx + rrf) - cross;
          const float F = sc * (nxh * ner + nex * nrh + nex * ner + epsf * nxh * nrh);
          const float E = 2.f * F * 1.0001f + 0x1p-18f * (xx + rrf + fabsf(cross));
          const int bit = gs.pkey + jr;
          a.ub[bit] = fmaxf((S + E) * (1.f + etap), 0.f);
          a.lb[bit] = fmaxf(S - E, 0.f) * (1.f - etap);
        }
      }
      __syncwarp();
      if (lane == 0) scr_arrive(&sempty[ab]);
    }
  }
  __syncwarp();
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 64;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ threshold
// Warp per query.  The bounds of its top-t candidates are gathered into shared memory;
// T is any value >= the k-th smallest UB: here the largest UB of the float-linear
// buckets (256 over [min UB, max UB]) up to the one holding the k-th smallest -- at
// least k candidates lie in those buckets, so at least k have UB <= T -- which costs
// one histogram pass and adds at most one bucket of extra survivors.  The survivors
// (LB <= T) are compacted in place into the query's candidate list (cand_idx, cand_n),
// which the sparse exact re-rank and the final top-k then read.
__device__ __forceinline__ float warp_min_f(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fminf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}
__device__ __forceinline__ float warp_max_f(float v) {
  for (int o = 16; o > 0; o >>= 1) v = fmaxf(v, __shfl_xor_sync(0xffffffffu, v, o));
  return v;
}

__global__ void k_rr_thresh(ThreshArgs a, int nq) {
  extern __shared__ __align__(16) unsigned char thr_sm[];
  __shared__ int hist[8][256];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5, wpb = blockDim.x >> 5;
  const int q = blockIdx.x * wpb + wl;
  if (q >= nq) return;
  const size_t per = (size_t)a.take_cap * 4;  // only the marked UBs are staged (occupancy)
  float* uu = reinterpret_cast<float*>(thr_sm + per * wl);
  int* h = hist[wl];
  const int n = a.cand_n[q];
  const int kb = a.kbase[q], nc = a.kbase[q + 1] - kb;
  int* ci = a.cand_idx + (size_t)q * a.take_cap;
  if (n <= a.k) {  // nothing can be pruned
    if (a.counters && lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 0), (unsigned long long)n);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 1), (unsigned long long)n);
    }
    return;
  }
  // the top-t candidates are the marked ones of the query's range [kb, kb + nc): stream the
  // range (coalesced bounds, no index gathers) and stage the marked (UB, LB, index)
  float umin = __int_as_float(0x7f800000), umax = 0.f;
  int got = 0;
  constexpr int SU = 8;  // 8 x (membership word, UB, LB) loads in flight per lane, none dependent
  for (int j0 = 0; j0 < nc; j0 += 32 * SU) {
    uint32_t mw[SU];
    float u[SU];
#pragma unroll
    for (int t = 0; t < SU; ++t) {
      const int j = j0 + 32 * t + lane;
      const int bit = kb + min(j, nc - 1);
      mw[t] = __ldg(a.marks + (bit >> 5));
      u[t] = __ldg(a.ub + bit);
    }
#pragma unroll
    for (int t = 0; t < SU; ++t) {
      const int j = j0 + 32 * t + lane;
      const int bit = kb + j;
      const bool mk = j < nc && ((mw[t] >> (bit & 31)) & 1u);
      const unsigned bal = __ballot_sync(0xffffffffu, mk);
      if (mk) {
        uu[got + __popc(bal & ((1u << lane) - 1u))] = u[t];
        umin = fminf(umin, u[t]);
        umax = fmaxf(umax, u[t]);
      }
      got += __popc(bal);
    }
  }
  umin = warp_min_f(umin);
  umax = warp_max_f(umax);
  for (int i = lane; i < 256; i += 32) h[i] = 0;
  __syncwarp();
  const float scale = umax > umin ? 256.f / (umax - umin) : 0.f;
  auto bucket = [&](float u) {
    const int bk = (int)((u - umin) * scale);
    return bk < 0 ? 0 : (bk > 255 ? 255 : bk);
  };
  for (int i = lane; i < got; i += 32) atomicAdd(&h[bucket(uu[i])], 1);
  __syncwarp();
  // bucket holding the k-th smallest: warp scan over 8 buckets per lane
  int loc[8], sum = 0;
#pragma unroll
  for (int t = 0; t < 8; ++t) { loc[t] = h[lane * 8 + t]; sum += loc[t]; }
  int incl = sum;
  for (int o = 1; o < 32; o <<= 1) {
    const int v = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += v;
  }
  int found = 256;
  if (incl - sum < a.k && a.k <= incl) {
    int run = incl - sum;
#pragma unroll
    for (int t = 0; t < 8; ++t) {
      if (found == 256 && run + loc[t] >= a.k) found = lane * 8 + t;
      run += loc[t];
    }
  }
  for (int o = 16; o > 0; o >>= 1) found = min(found, __shfl_xor_sync(0xffffffffu, found, o));
  float T = 0.f;
  for (int i = lane; i < got; i += 32)
    if (bucket(uu[i]) <= found) T = fmaxf(T, uu[i]);
  T = warp_max_f(T);
  if (found == 256) T = __int_as_float(0x7f800000);  // (fewer marked than k: keep all)
  // survivors (marked, LB <= T) replace the query's candidate list: a second coalesced
  // stream over the range (membership words and LBs, L2-resident)
  int ns = 0;
  for (int j0 = 0; j0 < nc; j0 += 32 * SU) {
    uint32_t mw[SU];
    float lv[SU];
#pragma unroll
    for (int t = 0; t < SU; ++t) {
      const int bit = kb + min(j0 + 32 * t + lane, nc - 1);
      mw[t] = __ldg(a.marks + (bit >> 5));
      lv[t] = __ldg(a.lb + bit);
    }
#pragma unroll
    for (int t = 0; t < SU; ++t) {
      const int j = j0 + 32 * t + lane;
      const int bit = kb + j;
      const bool keep = j < nc && ((mw[t] >> (bit & 31)) & 1u) && !(lv[t] > T);
      const unsigned bal = __ballot_sync(0xffffffffu, keep);
      if (keep) ci[ns + __popc(bal & ((1u << lane) - 1u))] = j;
      ns += __popc(bal);
    }
  }
  if (lane == 0) a.cand_n[q] = ns;
  if (a.counters && lane == 0) {
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 0), (unsigned long long)n);
    atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 1), (unsigned long long)ns);
  }
}

// ------------------------------------------------------------------ launchers
// Work items and group records: needs only the pair bucketing, so it runs on a side
// stream while the top-t selection (which makes the membership bits) runs.
void launch_screen_prep(const ScreenHost& h, int nq, cudaStream_t st) {
  (void)nq;
  const DevIndexView& ix = h.ix;
  // groups (cluster, <= kRrQ queries): one record each, built in parallel up front
  launch_rr_items(h.pair_off, ix.cl_pos, ix.L, 1 << 30, h.grp_off, st);
  launch_rr_items(h.pair_off, ix.cl_pos, ix.L, kScrRows, h.item_off, st);
  (k_rr_groups<<<h.n_groups_max, 32 * kRrQ, 0, st>>>(ix, h.queries, h.w, h.qoff, h.pair_off, h.pairs, h.kbase,
                                              h.grp_off, h.grec), note_launch());
}

void launch_screen(const ScreenHost& h, int nq, cudaStream_t st) {
  const DevIndexView& ix = h.ix;
  ScreenArgs a;
  a.ix = ix; a.pair_off = h.pair_off; a.marks = h.marks; a.item_off = h.item_off; a.grp_off = h.grp_off;
  a.grec = h.grec; a.ub = h.ub; a.lb = h.lb; a.counters = h.counters;
  a.nst = ix.opt.screen_stages > 0 ? std::min(ix.opt.screen_stages, screen_stages(ix.scr_kc))
                                    : screen_stages(ix.scr_kc);
  a.eta = (double)(ix.d + 4) * 0x1p-24 * 1.001;
  a.eps_acc = (double)(ix.d + 32) * 0x1p-21;
  const size_t sm = (size_t)a.nst * kScrStageBytes + 2 * grp_rec_bytes(ix.scr_kc) + 1024;
  static int done[64] = {};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {  // the largest tile any index may need
    cudaFuncAttributes at{};
    cudaFuncGetAttributes(&at, (const void*)k_rr_screen);
    cudaFuncSetAttribute((const void*)k_rr_screen, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         kMaxSmemPerCta - (int)at.sharedSizeBytes);
    done[dev] = 1;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  (k_rr_screen<<<sms, kScrThreads, sm, st>>>(a), note_launch());
}

void launch_thresh(const ScreenHost& h, int nq, cudaStream_t st) {
  int dev = 0;
  cudaGetDevice(&dev);
  ThreshArgs t;
  t.kbase = h.kbase; t.cand_idx = h.cand_idx; t.cand_n = h.cand_n; t.take_cap = h.take_cap; t.k = h.k;
  t.ub = h.ub; t.lb = h.lb; t.marks = h.marks; t.diss = h.diss; t.counters = h.counters;
  static int tdone[64] = {};
  if (dev >= 0 && dev < 64 && !tdone[dev]) {
    cudaFuncSetAttribute((const void*)k_rr_thresh, cudaFuncAttributeMaxDynamicSharedMemorySize, 192 * 1024);
    tdone[dev] = 1;
  }
  const size_t per = (size_t)h.take_cap * 4;
  const int wpb = (int)std::max<size_t>(1, std::min<size_t>(8, (160 * 1024) / per));
  (k_rr_thresh<<<(nq + wpb - 1) / wpb, 32 * wpb, per * wpb, st>>>(t, nq), note_launch());
}

// Counter only (rrg_search_counters[4]): block per cluster, the union over its queries
// of the rows they keep (membership words, or the screen's survivor lists), popcounted.
__global__ void k_count_rows(DevIndexView ix, const int* __restrict__ pair_off, const int* __restrict__ pairs,
                             const int* __restrict__ kbase, const int* __restrict__ qoff, int w,
                             const uint32_t* __restrict__ marks, const int* __restrict__ cand_idx,
                             const int* __restrict__ cand_n, int take_cap, int64_t* out) {
  extern __shared__ uint32_t u[];
  const int l = blockIdx.x;
  const int m = ix.cl_pos[l + 1] - ix.cl_pos[l], mw = (m + 31) / 32;
  const int j0 = pair_off[l], j1 = pair_off[l + 1];
  if (m == 0 || j1 == j0) return;
  for (int k = threadIdx.x; k < mw; k += blockDim.x) u[k] = 0;
  __syncthreads();
  for (int j = j0; j < j1; ++j) {
    const int pr = pairs[j], q = pr / w, c = pr % w;
    const int off = qoff[(size_t)q * (w + 1) + c];
    if (cand_idx) {
      for (int i = threadIdx.x; i < cand_n[q]; i += blockDim.x) {
        const int row = cand_idx[(size_t)q * take_cap + i] - off;
        if (row >= 0 && row < m) atomicOr(u + (row >> 5), 1u << (row & 31));
      }
      continue;
    }
    const size_t key = (size_t)kbase[q] + off;
    for (int k = threadIdx.x; k < mw; k += blockDim.x) {
      const size_t bit = key + 32 * (size_t)k;
      uint32_t v = __funnelshift_r(marks[bit >> 5], marks[(bit >> 5) + 1], (unsigned)(bit & 31));
      if (k == mw - 1 && (m & 31)) v &= (1u << (m & 31)) - 1u;
      u[k] |= v;  // one thread per word: no race
    }
  }
  __syncthreads();
  int cnt = 0;
  for (int k = threadIdx.x; k < mw; k += blockDim.x) cnt += __popc(u[k]);
  for (int o = 16; o > 0; o >>= 1) cnt += __shfl_xor_sync(0xffffffffu, cnt, o);
  if ((threadIdx.x & 31) == 0 && cnt) atomicAdd(reinterpret_cast<unsigned long long*>(out), (unsigned long long)cnt);
}

void launch_count_rows(const DevIndexView& ix, const int* pair_off, const int* pairs, const int* kbase,
                       const int* qoff, int w, const uint32_t* marks, const int* cand_idx, const int* cand_n,
                       int take_cap, int mwords, int64_t* out, cudaStream_t st) {
  (k_count_rows<<<ix.L, 256, (size_t)mwords * 4, st>>>(ix, pair_off, pairs, kbase, qoff, w, marks, cand_idx,
                                                      cand_n, take_cap, out),
   note_launch());
}

}  // namespace rrg
