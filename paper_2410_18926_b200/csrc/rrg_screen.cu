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

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

constexpr int kScrRows = 128;                   // rows per block = MMA M = TMEM lanes
constexpr int kScrChunk = kScrRows * 32;        // bytes of one K = 16 chunk of a block
constexpr int kScrStageChunks = 4;              // 16 KB per ring stage
constexpr int kScrStages = 6;
constexpr int kScrStageBytes = kScrStageChunks * kScrChunk;
constexpr int kScrRing = kScrStages * kScrStageBytes;  // 96 KB
constexpr int kScrThreads = 192;                // warp 0 TMA, warp 1 MMA, warps 2-5 epilogue
constexpr int kScrMaxKc = 128;                  // d <= 2048: two B tiles + the ring fit

int screen_max_dim() { return kScrMaxKc * 16; }
size_t screen_smem(int kc) { return (size_t)kScrRing + 2 * (size_t)kc * 512 + 1024; }

// halves offset of element e of row rr inside a block: chunk e/16, then the canonical
// K-major no-swizzle core matrices (8 rows x 16 B; +128 B per K half, +256 B per 8 rows)
__device__ __forceinline__ size_t scr_half_off(int rr, int e) {
  return (size_t)(e >> 4) * (kScrChunk / 2) + (rr >> 3) * 128 + ((e & 15) >> 3) * 64 + (rr & 7) * 8 + (e & 7);
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
// K-major, no swizzle: start >> 4, LBO (K direction) 128 B, SBO (8-row groups) 256 B, version 1
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

struct ScreenArgs {
  DevIndexView ix;
  const float* queries;  // chunk-local [nq][d]
  int w;
  const int* qoff;
  const int* pair_off;
  const int* pairs;
  const int* kbase;
  const uint32_t* marks;
  const int* item_off;   // [L+1]: ceil(pairs_l / kRrQ) * blocks_l, scanned
  float* ub;             // per candidate (key-array layout)
  float* lb;
  double eta, eps_acc;
};

__global__ void __launch_bounds__(kScrThreads, 1) k_rr_screen(ScreenArgs a) {
  extern __shared__ __align__(1024) unsigned char scr_sm[];
  __shared__ uint64_t full[kScrStages], empty[kScrStages], bfull[2], tfull[2], tempty[2];
  __shared__ uint32_t tmem_base;
  __shared__ double s_xx[2][kRrQ], s_sc[2][kRrQ];
  __shared__ float s_nxh[2][kRrQ], s_nex[2][kRrQ];
  __shared__ int s_pkey[2][kRrQ], s_ng[2];
  const DevIndexView& ix = a.ix;
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  unsigned char* base = reinterpret_cast<unsigned char*>((reinterpret_cast<uintptr_t>(scr_sm) + 1023) & ~uintptr_t(1023));
  unsigned char* ring = base;
  unsigned char* btile = base + kScrRing;
  const int KC = ix.scr_kc, d = ix.d, L = ix.L;
  const int bt_bytes = KC * 512;
  const int total = a.item_off[L];
  const int i0 = (int)((int64_t)total * blockIdx.x / gridDim.x);
  const int i1 = (int)((int64_t)total * (blockIdx.x + 1) / gridDim.x);
  if (i0 >= i1) return;  // uniform over the CTA, before any barrier or TMEM use

  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 32;" ::"r"(s_addr(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 0) {
    for (int i = 0; i < kScrStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&empty[i])));
    }
    for (int i = 0; i < 2; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&bfull[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(s_addr(&tfull[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 4;" ::"r"(s_addr(&tempty[i])));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tmem = tmem_base;

  // item -> (cluster, query group, 128-row block); a CTA's items are a contiguous range,
  // a group's items are its cluster's blocks in order
  auto decode = [&](int i, int& l, int& gi, int& b, int& nb) {
    int lo = 0, hi = L;
    while (hi - lo > 1) {
      const int mid = (lo + hi) >> 1;
      if (__ldg(a.item_off + mid) <= i) lo = mid; else hi = mid;
    }
    l = lo;
    nb = __ldg(ix.scr_blk0 + l + 1) - __ldg(ix.scr_blk0 + l);
    const int local = i - __ldg(a.item_off + l);
    gi = local / nb;
    b = local % nb;
  };

  if (warp == 0) {
    if (lane == 0) {  // producer: the CTA's blocks, chunk by chunk, through the ring
      int sc = 0;
      for (int i = i0; i < i1; ++i) {
        int l, gi, b, nb;
        decode(i, l, gi, b, nb);
        const unsigned char* src = reinterpret_cast<const unsigned char*>(ix.scr_plane) +
                                   ((size_t)(ix.scr_blk0[l] + b) * KC) * kScrChunk;
        for (int c0 = 0; c0 < KC; c0 += kScrStageChunks, ++sc) {
          const int slot = sc % kScrStages, pass = sc / kScrStages;
          if (pass > 0) scr_wait(&empty[slot], (pass - 1) & 1);
          const int bytes = min(kScrStageChunks, KC - c0) * kScrChunk;
          scr_expect_tx(&full[slot], bytes);
          scr_bulk(s_addr(ring + slot * kScrStageBytes), src + (size_t)c0 * kScrChunk, bytes, &full[slot]);
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // MMA issuer
      int sc = 0, j = -1, pl = -1, pg = -1;
      for (int i = i0, it = 0; i < i1; ++i, ++it) {
        int l, gi, b, nb;
        decode(i, l, gi, b, nb);
        if (l != pl || gi != pg) {
          ++j; pl = l; pg = gi;
          scr_wait(&bfull[j & 1], (j >> 1) & 1);
          fence_after();
        }
        const int ab = it & 1, u = it >> 1;
        if (u > 0) {
          scr_wait(&tempty[ab], (u - 1) & 1);
          fence_after();
        }
        const uint32_t sb = s_addr(btile + (j & 1) * bt_bytes);
        const uint32_t dt = tmem + (uint32_t)(ab * kRrQ);
        for (int c0 = 0; c0 < KC; c0 += kScrStageChunks, ++sc) {
          const int slot = sc % kScrStages, pass = sc / kScrStages;
          scr_wait(&full[slot], pass & 1);
          fence_after();
          const uint32_t sa = s_addr(ring + slot * kScrStageBytes);
          const int nch = min(kScrStageChunks, KC - c0);
          for (int c = 0; c < nch; ++c)
            scr_mma(dt, scr_desc(sa + c * kScrChunk), scr_desc(sb + (c0 + c) * 512), (c0 + c) > 0 ? 1u : 0u);
          scr_commit(&empty[slot]);
        }
        scr_commit(&tfull[ab]);
      }
    }
  } else {
    // epilogue warps: TMEM lane quarter = warp % 4, one block row per thread
    const int ew = warp - 2, q4 = warp & 3, row = q4 * 32 + lane;
    // the queries of item i's group -> fp16 tile `buf` + per-slot bound terms
    auto build = [&](int i, int buf) {
      int l, gi, b, nb;
      decode(i, l, gi, b, nb);
      const int j0 = a.pair_off[l] + gi * kRrQ;
      const int ng = min(kRrQ, a.pair_off[l + 1] - j0);
      epi_sync();  // every epilogue warp is done with the buffer's previous group
      uint16_t* bt = reinterpret_cast<uint16_t*>(btile + buf * bt_bytes);
      const float* mu = ix.scr_mu + (size_t)l * d;
      for (int g = ew; g < ng; g += 4) {
        const int pr = a.pairs[j0 + g];
        const int q = pr / a.w, c = pr % a.w;
        const float* x = a.queries + (size_t)q * d;
        double amax = 0.0;
        for (int e = lane; e < d; e += 32) amax = fmax(amax, fabs((double)__ldg(x + e) - (double)__ldg(mu + e)));
        amax = warp_max_d(amax);
        const int ex = amax > 0.0 ? ilogb(amax) - 14 : 0;
        const double inv = ldexp(1.0, -ex);
        double s_x = 0.0, s_h = 0.0, s_e = 0.0;
        for (int e = lane; e < KC * 16; e += 32) {
          uint16_t hb = 0;
          if (e < d) {
            const double xr = (double)__ldg(x + e) - (double)__ldg(mu + e);
            const __half h = __double2half(xr * inv);
            const double hd = (double)__half2float(h);
            const double er = xr * inv - hd;
            s_x += xr * xr;
            s_h += hd * hd;
            s_e += er * er;
            hb = __half_as_ushort(h);
          }
          // B tile: N = kRrQ rows (slots), same core-matrix layout, 512 B per K chunk
          bt[(size_t)(e >> 4) * 256 + (g >> 3) * 128 + ((e & 15) >> 3) * 64 + (g & 7) * 8 + (e & 7)] = hb;
        }
        s_x = warp_sum_d(s_x);
        s_h = warp_sum_d(s_h);
        s_e = warp_sum_d(s_e);
        if (lane == 0) {
          s_xx[buf][g] = s_x;
          s_sc[buf][g] = ldexp(1.0, ex);
          s_nxh[buf][g] = __double2float_ru(sqrt(s_h));
          s_nex[buf][g] = __double2float_ru(sqrt(s_e));
          s_pkey[buf][g] = a.kbase[q] + a.qoff[(size_t)q * (a.w + 1) + c];
        }
      }
      if (ew == 0 && lane == 0) s_ng[buf] = ng;
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // tile -> tensor core (async proxy)
      epi_sync();
      if (ew == 0 && lane == 0) scr_arrive(&bfull[buf]);
    };
    {
      int l, gi, b, nb;
      decode(i0, l, gi, b, nb);
      build(i0, 0);
      const int s1 = i0 + (nb - b);
      if (s1 < i1) build(s1, 1);
    }
    const double eta = a.eta, eps = a.eps_acc;
    int j = -1, pl = -1, pg = -1;
    for (int i = i0, it = 0; i < i1; ++i, ++it) {
      int l, gi, b, nb;
      decode(i, l, gi, b, nb);
      if (l != pl || gi != pg) { ++j; pl = l; pg = gi; }
      const int buf = j & 1, ab = it & 1, u = it >> 1;
      scr_wait(&tfull[ab], u & 1);
      fence_after();
      uint32_t v[kRrQ];
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];"
          : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]), "=r"(v[7]),
            "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15])
          : "r"(tmem + ((uint32_t)(q4 * 32) << 16) + (uint32_t)(ab * kRrQ)));
      asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
      fence_before();
      __syncwarp();
      if (lane == 0) scr_arrive(&tempty[ab]);
      const int p0 = ix.cl_pos[l], m = ix.cl_pos[l + 1] - p0;
      const int jr = b * kScrRows + row;
      if (jr < m) {
        const int gp = p0 + jr;
        const double rr = __ldg(ix.scr_rr + gp);
        const float4 rm = __ldg(ix.scr_rmeta + gp);
        const double rsc = ldexp(1.0, (int)rm.z), nrh = rm.x, ner = rm.y;
        const int ng = s_ng[buf];
#pragma unroll
        for (int g = 0; g < kRrQ; ++g) {
          if (g >= ng) break;
          const int bit = s_pkey[buf][g] + jr;
          if (!((__ldg(a.marks + (bit >> 5)) >> (bit & 31)) & 1u)) continue;
          const double G = (double)__uint_as_float(v[g]);
          const double sc = s_sc[buf][g] * rsc;
          const double xx = s_xx[buf][g], nxh = s_nxh[buf][g], nex = s_nex[buf][g];
          const double S = xx + rr - 2.0 * sc * G;
          const double F = sc * (nxh * ner + nex * nrh + nex * ner + eps * nxh * nrh);
          const double E = 2.0 * F * (1.0 + 0x1p-20) + 0x1p-40 * (xx + rr + 2.0 * sc * fabs(G));
          const double ubv = fmax((S + E) * (1.0 + eta), 0.0);
          const double lbv = fmax(S - E, 0.0) * (1.0 - eta);
          a.ub[bit] = __double2float_ru(ubv);
          a.lb[bit] = __double2float_rd(lbv);
        }
      }
      // after the group's last item: its tile buffer is free, build the group after next
      if (b + 1 == nb && i + 1 < i1) {
        int l1, g1, b1, nb1;
        decode(i + 1, l1, g1, b1, nb1);
        const int s2 = i + 1 + (nb1 - b1);
        if (s2 < i1) build(s2, buf);
      }
    }
  }
  __syncwarp();
  fence_before();
  __syncthreads();
  fence_after();
  if (warp == 1)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 32;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ threshold
// Warp per query: T = k-th smallest UB of its top-t candidates (radix select on the
// bits of the non-negative f32 bounds), then every non-survivor (LB > T) loses its
// membership bit (the cluster re-rank skips it) and gets the +inf key (k_topk_final
// never selects it).  Survivor and candidate counts feed rrg_search_counters.
constexpr int kThrWarps = 8;

__global__ void __launch_bounds__(32 * kThrWarps) k_rr_thresh(ThreshArgs a, int nq) {
  __shared__ int hist[kThrWarps][256];
  const int lane = threadIdx.x & 31, wl = threadIdx.x >> 5;
  const int q = blockIdx.x * kThrWarps + wl;
  if (q >= nq) return;
  int* h = hist[wl];
  const int n = a.cand_n[q];
  const int kb = a.kbase[q], nc = a.kbase[q + 1] - kb;
  const int* ci = a.cand_idx + (size_t)q * a.take_cap;
  uint32_t T = 0x7f800000u;  // +inf: fewer than k candidates keep everything
  if (n > a.k) {
    uint32_t prefix = 0, pmask = 0;
    int want = a.k;  // rank (1-based) of the k-th smallest inside the current prefix
    for (int shift = 24; shift >= 0; shift -= 8) {
      for (int i = lane; i < 256; i += 32) h[i] = 0;
      __syncwarp();
      for (int i = lane; i < n; i += 32) {
        const uint32_t u = __float_as_uint(__ldg(a.ub + kb + __ldg(ci + i)));
        if ((u & pmask) == prefix) atomicAdd(&h[(u >> shift) & 255], 1);
      }
      __syncwarp();
      // bucket holding the want-th value: warp scan over 8 buckets per lane
      int loc[8], s = 0;
#pragma unroll
      for (int t = 0; t < 8; ++t) { loc[t] = h[lane * 8 + t]; s += loc[t]; }
      int incl = s;
      for (int o = 1; o < 32; o <<= 1) {
        const int v = __shfl_up_sync(0xffffffffu, incl, o);
        if (lane >= o) incl += v;
      }
      const int excl = incl - s;
      int found = -1, before = 0;
      if (excl < want && want <= incl) {
        int run = excl;
#pragma unroll
        for (int t = 0; t < 8; ++t) {
          if (found < 0 && run + loc[t] >= want) { found = lane * 8 + t; before = run; }
          run += loc[t];
        }
      }
      const unsigned who = __ballot_sync(0xffffffffu, found >= 0);
      const int src = __ffs(who) - 1;
      found = __shfl_sync(0xffffffffu, found, src);
      before = __shfl_sync(0xffffffffu, before, src);
      want -= before;
      prefix |= (uint32_t)found << shift;
      pmask |= 255u << shift;
      __syncwarp();
    }
    T = prefix;
  }
  const float Tf = __uint_as_float(T);
  // membership bits of the query's candidate range [kb, kb + nc): clear non-survivors
  int surv = 0;
  if (n > a.k) {
    const int w0 = kb >> 5, w1 = (kb + nc - 1) >> 5;
    for (int wi = w0 + lane; wi <= w1; wi += 32) {
      uint32_t in = 0xffffffffu;  // bits of this query inside the word
      if (wi == w0) in &= 0xffffffffu << (kb & 31);
      if (wi == w1) in &= 0xffffffffu >> (31 - ((kb + nc - 1) & 31));
      const uint32_t m = a.marks[wi] & in;
      uint32_t drop = 0, bits = m;
      while (bits) {
        const int bb = __ffs(bits) - 1;
        bits &= bits - 1;
        if (__ldg(a.lb + 32 * (size_t)wi + bb) > Tf) drop |= 1u << bb;
      }
      surv += __popc(m & ~drop);
      if (drop) atomicAnd(a.marks + wi, ~drop);
    }
    for (int i = lane; i < n; i += 32) {
      const int c = __ldg(ci + i);
      if (__ldg(a.lb + kb + c) > Tf) a.diss[kb + c] = 0xffffffffu;
    }
  } else {
    surv = lane == 0 ? n : 0;
  }
  if (a.counters) {
    for (int o = 16; o > 0; o >>= 1) surv += __shfl_xor_sync(0xffffffffu, surv, o);
    if (lane == 0) {
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 0), (unsigned long long)n);
      atomicAdd(reinterpret_cast<unsigned long long*>(a.counters + 1), (unsigned long long)surv);
    }
  }
}

// ------------------------------------------------------------------ launchers
void launch_screen(const ScreenHost& h, int nq, cudaStream_t st) {
  const DevIndexView& ix = h.ix;
  launch_rr_items(h.pair_off, ix.cl_pos, ix.L, kScrRows, h.item_off, st);
  ScreenArgs a;
  a.ix = ix; a.queries = h.queries; a.w = h.w; a.qoff = h.qoff; a.pair_off = h.pair_off;
  a.pairs = h.pairs; a.kbase = h.kbase; a.marks = h.marks; a.item_off = h.item_off;
  a.ub = h.ub; a.lb = h.lb;
  a.eta = (double)(ix.d + 4) * 0x1p-24 * 1.001;
  a.eps_acc = (double)(ix.d + 32) * 0x1p-21;
  const size_t sm = screen_smem(ix.scr_kc);
  static int done[64] = {};
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncSetAttribute((const void*)k_rr_screen, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    done[dev] = 1;
  }
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  (k_rr_screen<<<sms, kScrThreads, sm, st>>>(a), note_launch());
  ThreshArgs t;
  t.kbase = h.kbase; t.cand_idx = h.cand_idx; t.cand_n = h.cand_n; t.take_cap = h.take_cap; t.k = h.k;
  t.ub = h.ub; t.lb = h.lb; t.marks = h.marks; t.diss = h.diss; t.counters = h.counters;
  (k_rr_thresh<<<(nq + kThrWarps - 1) / kThrWarps, 32 * kThrWarps, 0, st>>>(t, nq), note_launch());
}

}  // namespace rrg
