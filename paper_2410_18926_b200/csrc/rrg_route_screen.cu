// rrg_route_screen.cu -- routing on the tensor cores, exact by construction.
//
// route() (cluster.py:46-58,254-264) needs the w smallest f64 dissimilarities
//   d2(x, c) = max((x.x - 2 x.c) + c.c, 0)
// of every query against all L centroids: an f64 GEMM (DMMA: 0.21 ms of a C2 batch).
// Almost all of those L values are far from the w-th smallest, so bounds decide:
// with fp16 roundings x^ ~ x / 2^ex and c^ ~ c / 2^ec (power-of-two row scales) the
// tensor cores compute G = x^.c^ and
//   |x.c - 2^(ex+ec) G| <= 2^(ex+ec) (|x^| |e_c| + |e_x| |c^| + |e_x| |e_c| + eps |x^| |c^|)
// (Cauchy-Schwarz on the exact rounding residuals, eps for the f32 accumulation), so
// d2 lies in [LB, UB].  With T = the w-th smallest UB (any T above it is also valid:
// each CTA's own w-th smallest, minimised over CTAs), a centroid with LB > T has
// d2 > T >= the w-th smallest d2 and cannot be selected -- not even by an id tie.
// The survivors (typically 1-2 per query) are then evaluated in f64 (the same
// f64-grade contract as the DMMA path: f32 products, f64 sums) and the w smallest
// by (d2, id) are taken, like the stable argsort.
//
// k_route_screen: per (128-query block, centroid range) CTA, tcgen05.mma kind::f16
// (M = 128 queries, N = 128 centroids, K = 16) into double-buffered TMEM; each epilogue
// thread (one query, half of every tile's columns) keeps its w smallest UB (-> atomicMin
// into T[q]) and lists the centroids whose LB is <= its running w-th smallest UB -- a
// superset of the survivors it saw, since the final T[q] is below every running bound.
// k_route_recheck: warp per query, keeps the listed centroids with LB <= T[q], exact f64
// d2 for those (every centroid when a list overflowed), top w by (d2, id).
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

#include <algorithm>

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

constexpr int kRtRows = 128;              // queries per CTA (M) = centroids per tile (N)
constexpr int kRtChunk = kRtRows * 32;    // one K = 16 chunk of a 128-row tile: 4 KB
// warps 0-7 epilogue (TMEM lane quarter = warp % 4, column half = warp / 4), warp 8 TMA + MMA
constexpr int kRtThreads = 288;
constexpr int kRtIssuer = 8;

int route_screen_max_dim() { return kRtMaxKc * 16; }
size_t route_tile_bytes(int rows, int kc) { return (size_t)((rows + kRtRows - 1) / kRtRows) * kc * kRtChunk; }

__device__ __forceinline__ uint32_t rt_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ uint64_t rt_desc(uint32_t addr) {  // K-major, no swizzle, LBO 128, SBO 256
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46);
}
// kind::f16: D f32, A/B f16, K-major, N = 128, M = 128
constexpr uint32_t kRtIdesc = (1u << 4) | ((uint32_t)(kRtRows >> 3) << 17) | ((uint32_t)(kRtRows >> 4) << 24);
__device__ __forceinline__ void rt_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "RT_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra RT_WAIT_%=;\n\t}" ::"r"(rt_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void rt_bulk(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(rt_smem(bar)), "r"(bytes) : "memory");
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(rt_smem(bar))
      : "memory");
}
__device__ __forceinline__ void rt_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(rt_smem(bar))
               : "memory");
}

// ------------------------------------------------------------------ fp16 tiles
// Warp per row of src (rows x K f32, leading dimension ld): e with max|x| / 2^e in
// [2^14, 2^15), x^ = fp16(x / 2^e) into the tiled layout, stats = {|x^|, |x/2^e - x^|
// (both rounded up), e, 0}.  Rows past `rows` up to the tile boundary are zero.
__global__ void k_f16_tiles(const float* __restrict__ src, int rows, int K, int ld, int kc,
                            uint16_t* __restrict__ tiles, float4* __restrict__ stats) {
  const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int rows_pad = (rows + kRtRows - 1) / kRtRows * kRtRows;
  if (row >= rows_pad) return;
  const bool valid = row < rows;
  const float* r = src + (size_t)(valid ? row : 0) * ld;
  double amax = 0.0;
  if (valid)
    for (int e = lane; e < K; e += 32) amax = fmax(amax, fabs((double)__ldg(r + e)));
  for (int o = 16; o > 0; o >>= 1) amax = fmax(amax, __shfl_xor_sync(0xffffffffu, amax, o));
  const int ex = amax > 0.0 ? ilogb(amax) - 14 : 0;
  const double inv = ldexp(1.0, -ex);
  uint16_t* blk = tiles + (size_t)(row / kRtRows) * kc * (kRtChunk / 2);
  const int rr = row % kRtRows;
  double s_h = 0.0, s_e = 0.0;
  for (int e = lane; e < kc * 16; e += 32) {
    uint16_t hb = 0;
    if (valid && e < K) {
      const double v = (double)__ldg(r + e) * inv;
      const __half h = __double2half(v);
      const double hd = (double)__half2float(h);
      s_h += hd * hd;
      s_e += (v - hd) * (v - hd);
      hb = __half_as_ushort(h);
    }
    blk[(size_t)(e >> 4) * (kRtChunk / 2) + (rr >> 3) * 128 + ((e & 15) >> 3) * 64 + (rr & 7) * 8 + (e & 7)] = hb;
  }
  for (int o = 16; o > 0; o >>= 1) {
    s_h += __shfl_xor_sync(0xffffffffu, s_h, o);
    s_e += __shfl_xor_sync(0xffffffffu, s_e, o);
  }
  if (lane == 0)
    stats[row] = make_float4(__double2float_ru(sqrt(s_h)), __double2float_ru(sqrt(s_e)), (float)ex, 0.f);
}

void launch_f16_tiles(const float* src, int rows, int K, int ld, int kc, uint16_t* tiles, float4* stats,
                      cudaStream_t st) {
  const int64_t rp = (rows + kRtRows - 1) / kRtRows * kRtRows;
  (k_f16_tiles<<<(unsigned)((rp * 32 + 255) / 256), 256, 0, st>>>(src, rows, K, ld, kc, tiles, stats),
   note_launch());
}

// ------------------------------------------------------------------ screen
constexpr int kRtLoc = 12;  // list slots per thread and (CTA, half): 4 at w = 1, 12 for w <= 8
// (kept in registers while the thread sweeps its columns: an entry whose LB rises above
// the running bound is dropped, so only the near-ties of the running best accumulate)

struct RouteScreenArgs {
  const uint16_t* qt;   // query tiles
  const float4* qs;     // query stats [nq]
  const double* pp;     // x.x (NumPy pairwise f64) [nq]
  const uint16_t* ct;   // centroid tiles
  const float4* cs;     // centroid stats [L]
  const double* cc;     // c.c [L]
  int nq, L, kc, w, tiles_per_cta, nslot;
  float eps;
  uint32_t* T;          // [nq] f32 bits; min over CTAs of their w-th smallest UB
  int* cnt;             // [nq][nslot] listed per (CTA, column half); kRtLoc + 1 = overflow
  int2* list;           // [nq][nslot][kRtLoc] (centroid, LB bits)
};

__device__ __forceinline__ void rt_bounds(float G, float sc, float ppq, float ccc, float nhq, float neq,
                                          float nhc, float nec, float eps, float& lb, float& ub) {
  // f32 arithmetic with a generous slack for its own rounding (a few ops on values of
  // magnitude <= pp + cc + 2|x.c|): the bound stays valid and only ~1e-6 looser
  const float cross = 2.f * sc * G;
  const float S = (ppq + ccc) - cross;
  const float F = sc * (nhq * nec + neq * nhc + neq * nec + eps * nhq * nhc);
  const float E = 2.f * F * 1.0001f + 0x1p-18f * (ppq + ccc + fabsf(cross));
  ub = fmaxf(S + E, 0.f);
  lb = fmaxf(S - E, 0.f);
}

// WM: the w the running-bound list is sized for (1, or kRtMaxW for any w <= 8 -- the
// general form's insertion and w-th selection were ~half the epilogue's instructions)
template <int LOC, int WM>
__global__ void __launch_bounds__(kRtThreads, 1) k_route_screen(RouteScreenArgs a) {
  extern __shared__ __align__(1024) unsigned char rt_sm[];
  __shared__ uint64_t afull, bfull[2], bempty[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ float4 cst[kRtRows];  // per centroid of the tile: {|c^|, |e_c|, 2^e_c, c.c}
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int qb = blockIdx.x;
  const int t0 = blockIdx.y * a.tiles_per_cta;
  const int ntile = (a.L + kRtRows - 1) / kRtRows;
  const int t1 = min(ntile, t0 + a.tiles_per_cta);
  if (t0 >= t1) return;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(rt_sm) + 1023) & ~uintptr_t(1023));
  const int tile_bytes = a.kc * kRtChunk;
  unsigned char* sa = base;
  unsigned char* sb = base + tile_bytes;
  if (warp == kRtIssuer) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 256;" ::"r"(rt_smem(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&afull)));
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&bfull[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&bempty[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(rt_smem(&tfull[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 8;" ::"r"(rt_smem(&tempty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  if (warp == kRtIssuer) {
    if (lane == 0) {  // TMA + MMA issue
      rt_bulk(rt_smem(sa), a.qt + (size_t)qb * a.kc * (kRtChunk / 2), tile_bytes, &afull);
      for (int t = t0; t < min(t1, t0 + 2); ++t)
        rt_bulk(rt_smem(sb + (t - t0) * tile_bytes), a.ct + (size_t)t * a.kc * (kRtChunk / 2), tile_bytes,
                &bfull[t - t0]);
      rt_wait(&afull, 0);
      for (int t = t0; t < t1; ++t) {
        const int i = t - t0, buf = i & 1, u = i >> 1;
        rt_wait(&bfull[buf], u & 1);
        if (u > 0) rt_wait(&tempty[buf], (u - 1) & 1);
        asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
        // descriptors advance by adds to the start-address field (addr >> 4): fewer issue
        // instructions per MMA (see k_rr_screen)
        const uint64_t ad = rt_desc(rt_smem(sa)), bd = rt_desc(rt_smem(sb + buf * tile_bytes));
        const uint32_t dt = tmem + (uint32_t)(buf * kRtRows);
        for (int c = 0; c < a.kc; ++c) {
          asm volatile(
              "{\n\t.reg .pred p;\n\t"
              "setp.ne.b32 p, %4, 0;\n\t"
              "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t}" ::"r"(dt),
              "l"(ad + (uint64_t)(c * (kRtChunk >> 4))), "l"(bd + (uint64_t)(c * (kRtChunk >> 4))), "r"(kRtIdesc),
              "r"(c > 0 ? 1u : 0u)
              : "memory");
        }
        rt_commit(&bempty[buf]);
        rt_commit(&tfull[buf]);
        if (t + 2 < t1) {  // refill this buffer once its MMAs have read it
          rt_wait(&bempty[buf], u & 1);
          rt_bulk(rt_smem(sb + buf * tile_bytes), a.ct + (size_t)(t + 2) * a.kc * (kRtChunk / 2), tile_bytes,
                  &bfull[buf]);
        }
      }
    }
  } else {
    const int q4 = warp & 3, half = warp >> 2;  // lane quarter (queries), column half
    const int q = qb * kRtRows + q4 * 32 + lane;
    const bool valid = q < a.nq;
    float ppq = 0.f, nhq = 0.f, neq = 0.f, scq = 0.f;
    if (valid) {
      const float4 s4 = a.qs[q];
      nhq = s4.x; neq = s4.y; scq = ldexpf(1.f, (int)s4.z);
      ppq = (float)a.pp[q];
    }
    const int slot = blockIdx.y * 2 + half;
    int lid[LOC];
    float llb[LOC];
#pragma unroll
    for (int i = 0; i < LOC; ++i) { lid[i] = -1; llb[i] = 0.f; }  // lid < 0: empty
    bool over = false;
    float best[WM];
#pragma unroll
    for (int i = 0; i < WM; ++i) best[i] = __int_as_float(0x7f800000);
    for (int t = t0; t < t1; ++t) {
      const int i = t - t0, buf = i & 1, u = i >> 1;
      {  // the tile's centroid terms, one per epilogue thread, while the MMAs run
        asm volatile("bar.sync 1, 256;" ::: "memory");  // previous tile's readers are done
        if (warp < 4) {
          const int c = t * kRtRows + warp * 32 + lane;
          float4 v4 = make_float4(0.f, 0.f, 0.f, __int_as_float(0x7f800000));
          if (c < a.L) {
            const float4 cs = __ldg(a.cs + c);
            v4 = make_float4(cs.x, cs.y, ldexpf(1.f, (int)cs.z), (float)__ldg(a.cc + c));
          }
          cst[warp * 32 + lane] = v4;
        }
        asm volatile("bar.sync 1, 256;" ::: "memory");
      }
      rt_wait(&tfull[buf], u & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
#pragma unroll 1
      for (int c0 = half * (kRtRows / 2); c0 < (half + 1) * (kRtRows / 2); c0 += 32) {
        uint32_t v[32];
        asm volatile(
            "tcgen05.ld.sync.aligned.32x32b.x32.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
            "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
            : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
              "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]),
              "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
              "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]), "=r"(v[27]), "=r"(v[28]),
              "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
            : "r"(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(buf * kRtRows + c0)));
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        if (valid) {
#pragma unroll
          for (int j = 0; j < 32; ++j) {
            const int c = t * kRtRows + c0 + j;
            const float4 cs = cst[c0 + j];  // (c >= L: c.c = +inf, never a survivor)
            float lb, ub;
            rt_bounds(__uint_as_float(v[j]), scq * cs.z, ppq, cs.w, nhq, neq, cs.x, cs.y, a.eps, lb, ub);
            if (ub < best[WM - 1]) {  // insertion into the sorted w smallest
              float x = ub;
#pragma unroll
              for (int s = 0; s < WM; ++s) {
                const float lo = fminf(best[s], x);
                x = fmaxf(best[s], x);
                best[s] = lo;
              }
            }
            float bw = best[0];  // the running w-th smallest UB
#pragma unroll
            for (int s = 1; s < WM; ++s)
              if (s == a.w - 1) bw = best[s];
            if (!(lb > bw) && c < a.L) {  // (NaN bounds are listed too)
              bool placed = false;  // into an empty slot or one no longer within the bound
#pragma unroll
              for (int i = 0; i < LOC; ++i)
                if (!placed && (lid[i] < 0 || llb[i] > bw)) { llb[i] = lb; lid[i] = c; placed = true; }
              over |= !placed;
            }
          }
        }
      }
      asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
      __syncwarp();
      if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(rt_smem(&tempty[buf])) : "memory");
    }
    if (valid) {
      // this thread's w-th smallest UB bounds the query's w-th smallest d2 (if it saw w)
      float tw = best[0];
#pragma unroll
      for (int s = 0; s < WM; ++s)
        if (s == a.w - 1) tw = best[s];
      if (tw == tw && tw < __int_as_float(0x7f800000)) atomicMin(a.T + q, __float_as_uint(tw));
      int2* lst = a.list + ((size_t)q * a.nslot + slot) * kRtLoc;
      int nl = 0;
#pragma unroll
      for (int i = 0; i < LOC; ++i)
        if (lid[i] >= 0 && !(llb[i] > tw)) lst[nl++] = make_int2(lid[i], __float_as_int(llb[i]));
      a.cnt[(size_t)q * a.nslot + slot] = over ? kRtLoc + 1 : nl;
    }
  }
  __syncwarp();
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  if (warp == kRtIssuer)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 256;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ recheck
// Warp per query: f64 d2 of the survivors (every centroid when the list overflowed or
// came out shorter than w), the w smallest by (d2, id) -> sel, primary = the nearest.
__global__ void k_route_recheck(const float* __restrict__ xp, int nq, int s, const float* __restrict__ cent,
                                int L, int w, const double* __restrict__ pp, const double* __restrict__ cc,
                                const uint32_t* __restrict__ Tq, const int* __restrict__ cnt,
                                const int2* __restrict__ list, int nslot, int* __restrict__ sel,
                                int* __restrict__ primary) {
  const int q = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  if (q >= nq) return;
  // the survivors: listed centroids with LB <= T (a warp-wide compaction of the slots)
  __shared__ int surv_s[8][kRtCap];
  int* surv = surv_s[(threadIdx.x >> 5) & 7];
  const float T = __uint_as_float(Tq[q]);
  bool over = false;
  int n = 0;
  for (int e0 = 0; e0 < nslot * kRtLoc; e0 += 32) {
    const int e = e0 + lane, sl = e / kRtLoc, j = e % kRtLoc;
    bool keep = false;
    int c = 0;
    if (e < nslot * kRtLoc) {
      const int nc = cnt[(size_t)q * nslot + sl];
      over |= nc > kRtLoc;
      if (j < min(nc, kRtLoc)) {
        const int2 v = list[((size_t)q * nslot + sl) * kRtLoc + j];
        c = v.x;
        keep = !(__int_as_float(v.y) > T);
      }
    }
    const unsigned bal = __ballot_sync(0xffffffffu, keep);
    const int at = n + __popc(bal & ((1u << lane) - 1u));
    if (keep && at < kRtCap) surv[at] = c;
    n += __popc(bal);
  }
  over = __any_sync(0xffffffffu, over);
  __syncwarp();
  const bool full = over || n > kRtCap || n < w;
  const int m = full ? L : n;
  const float* x = xp + (size_t)q * s;
  // each lane keeps its own w smallest (d2, id) over the centroids it evaluated
  double bd[kRtMaxW];
  int bi[kRtMaxW];
#pragma unroll
  for (int i = 0; i < kRtMaxW; ++i) { bd[i] = __longlong_as_double(0x7ff0000000000000ll); bi[i] = 0x7fffffff; }
  for (int j = 0; j < m; ++j) {
    const int c = full ? j : surv[j];
    const float* cr = cent + (size_t)c * s;
    double acc = 0.0;
    for (int k = lane; k < s; k += 32) acc = fma((double)__ldg(x + k), (double)__ldg(cr + k), acc);
    for (int o = 16; o > 0; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
    double d2 = __dadd_rn(__dsub_rn(pp[q], __dmul_rn(2.0, acc)), cc[c]);
    d2 = d2 > 0.0 ? d2 : 0.0;  // (NaN -> 0: a non-finite query is rejected after the search)
    if ((j & 31) == lane) {  // lane j % 32 keeps candidate j
      double xd = d2;
      int xi = c;
#pragma unroll
      for (int i = 0; i < kRtMaxW; ++i) {
        const bool lt = xd < bd[i] || (xd == bd[i] && xi < bi[i]);
        const double td = lt ? bd[i] : xd;
        const int ti = lt ? bi[i] : xi;
        if (lt) { bd[i] = xd; bi[i] = xi; }
        xd = td; xi = ti;
      }
    }
  }
  // merge: w rounds of a warp argmin over the lanes' heads
  int head = 0;
  for (int r = 0; r < w; ++r) {
    double hd = head < kRtMaxW ? bd[0] : __longlong_as_double(0x7ff0000000000000ll);
    int hi = head < kRtMaxW ? bi[0] : 0x7fffffff;
#pragma unroll
    for (int i = 1; i < kRtMaxW; ++i)
      if (i == head) { hd = bd[i]; hi = bi[i]; }
    double md = hd;
    int mi = hi;
    for (int o = 16; o > 0; o >>= 1) {
      const double od = __shfl_xor_sync(0xffffffffu, md, o);
      const int oi = __shfl_xor_sync(0xffffffffu, mi, o);
      if (od < md || (od == md && oi < mi)) { md = od; mi = oi; }
    }
    if (mi == 0x7fffffff) mi = r;  // defensive: fewer evaluated than w
    if (lane == 0) {
      sel[(size_t)q * w + r] = mi;
      if (r == 0) primary[q] = mi;
    }
    if (hi == mi) ++head;  // the lane whose head was taken advances
  }
}

// (CTA, column half) list slots per query: the launch's centroid ranges x 2
static int route_groups(int nq, int L, int& tiles_per_cta) {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const int qblocks = (nq + kRtRows - 1) / kRtRows;
  const int ntile = (L + kRtRows - 1) / kRtRows;
  // enough CTAs for ~2 per SM, each with >= 2 centroid tiles when there are several
  int groups = std::max(1, std::min(std::min(ntile, kRtMaxGroups), (2 * sms + qblocks - 1) / qblocks));
  tiles_per_cta = (ntile + groups - 1) / groups;
  return (ntile + tiles_per_cta - 1) / tiles_per_cta;
}
size_t route_list_bytes(int nq, int L) {
  int tpc = 0;
  return (size_t)nq * 2 * route_groups(nq, L, tpc) * kRtLoc * 8;
}
size_t route_cnt_bytes(int nq, int L) {
  int tpc = 0;
  return (size_t)nq * 2 * route_groups(nq, L, tpc) * 4;
}

void launch_route_screen(const RouteScreenHost& h, int nq, cudaStream_t st) {
  const DevIndexView& v = h.ix;
  launch_f16_tiles(h.xp, nq, v.s, v.s, v.rt_kc, h.qt, h.qs, st);
  cudaMemsetAsync(h.T, 0x7f, (size_t)nq * 4, st);  // 0x7f7f7f7f: a huge finite bound
  RouteScreenArgs a;
  a.qt = h.qt; a.qs = h.qs; a.pp = h.pp; a.ct = v.rt_cent_tiles; a.cs = v.rt_cent_stats; a.cc = v.cnorm;
  a.nq = nq; a.L = v.L; a.kc = v.rt_kc; a.w = h.w;
  a.eps = (float)((double)(v.s + 32) * 0x1p-21);
  a.T = h.T; a.cnt = h.cnt; a.list = h.list;
  int dev = 0;
  cudaGetDevice(&dev);
  const int qblocks = (nq + kRtRows - 1) / kRtRows;
  const int groups = route_groups(nq, v.L, a.tiles_per_cta);
  a.nslot = 2 * groups;
  const size_t sm = (size_t)3 * v.rt_kc * kRtChunk + 1024;
  static int done[64] = {};
  if (dev >= 0 && dev < 64 && !done[dev]) {
    for (const void* f : {(const void*)k_route_screen<4, 1>, (const void*)k_route_screen<kRtLoc, kRtMaxW>}) {
      cudaFuncAttributes at{};
      cudaFuncGetAttributes(&at, f);
      cudaFuncSetAttribute(f, cudaFuncAttributeMaxDynamicSharedMemorySize, kMaxSmemPerCta - (int)at.sharedSizeBytes);
    }
    done[dev] = 1;
  }
  dim3 grid(qblocks, groups);
  // w = 1: the near-ties of the running minimum (4 slots, fewer registers); w <= 8: 12
  if (h.w == 1)
    (k_route_screen<4, 1><<<grid, kRtThreads, sm, st>>>(a), note_launch());
  else
    (k_route_screen<kRtLoc, kRtMaxW><<<grid, kRtThreads, sm, st>>>(a), note_launch());
  (k_route_recheck<<<(nq + 7) / 8, 256, 0, st>>>(h.xp, nq, v.s, v.cent, v.L, h.w, h.pp, v.cnorm, h.T, h.cnt,
                                                 h.list, a.nslot, h.sel, h.primary),
   note_launch());
}

}  // namespace rrg
