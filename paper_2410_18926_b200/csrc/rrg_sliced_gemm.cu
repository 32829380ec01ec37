// rrg_sliced_gemm.cu -- f64-exact GEMMs of the projection and routing on the 5th-gen
// tensor cores (tcgen05.mma kind::i8, accumulators in TMEM).
//
// The reference computes  f32(f64(x) @ f64(W))  (index.py:298) and the routing
// dissimilarities  (p.p) - 2 p.c + (c.c)  in f64 (cluster.py:46-58).  Every f32
// operand row is split into S = 8 signed 7-bit slices against a power-of-two row
// scale (x = 2^e * sum_s a_s 2^-7(s+1), exact down to 2^-56 of the row maximum),
// the slice products are exact int8 x int8 -> int32 tensor-core MMAs, and the
// S(S+1)/2 slice pairs with i + j <= S-1 are summed per "level" l = i + j into
// one int32 TMEM accumulator (|level| <= 8 * K * 127^2 < 2^31 for K <= 16384).
// The epilogue combines the levels in f64 by Horner's rule (multiplications by
// 2^-7 are exact) and scales by 2^(ea + eb - 14): the result carries f64
// rounding error only, like the DMMA path (k_gemm_dmma), at int8 tensor-core rate.
//
// Tile: 128 rows (A) x 64 columns (B) per CTA, K in 64-byte chunks, two shared-
// memory stages filled by cp.async in the UMMA canonical K-major no-swizzle layout
// (8-row x 16-byte core matrices: LBO = 128 B along K, SBO = 512 B along rows).
// One elected thread issues the 72 MMAs of a chunk; tcgen05.commit arrives on the
// stage's mbarrier when they have read it.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

constexpr int kSl = 8;            // slices per operand
constexpr int kSlBM = 128;        // rows of A per CTA (TMEM lanes)
constexpr int kSlBN = 64;         // columns (rows of B) per CTA
constexpr int kSlBK = 32;         // K bytes per stage (one K=32 MMA per slice pair)
constexpr int kSlStages = 4;
constexpr int kSlThreads = 128;
constexpr int kSlRegK = 2048;  // k_slice_rows keeps rows up to this length in registers
constexpr int kSlATile = kSlBM * kSlBK;  // 4 KB per slice plane
constexpr int kSlBTile = kSlBN * kSlBK;  // 2 KB
constexpr int kSlAStage = kSl * kSlATile;  // 32 KB
constexpr int kSlBStage = kSl * kSlBTile;  // 16 KB
constexpr int kSlStage = kSlAStage + kSlBStage;
constexpr size_t kSlSmem = (size_t)kSlStages * kSlStage + 1024;

// ------------------------------------------------------------------ slicing
// Planes are stored pre-tiled for the MMA: for row block rb (tile_rows rows) and K
// chunk kc (32 bytes), the 8 slice tiles are one contiguous block
// [rb][kc][s][tile_rows x 32 B], each tile in the UMMA canonical K-major no-swizzle
// layout (8-row x 16-byte core matrices: +16 B per row, +128 B per K half, +256 B
// per 8-row group), so a pipeline stage is two bulk copies.
__device__ __forceinline__ size_t sl_tiled_off(int r, int k, int s, int tile_rows, int kchunks) {
  const int rb = r / tile_rows, rr = r % tile_rows, kc = k >> 5, kb = k & 31;
  return (((size_t)rb * kchunks + kc) * kSl + s) * (size_t)(tile_rows * kSlBK) + (rr >> 3) * 256 +
         (kb >> 4) * 128 + (rr & 7) * 16 + (kb & 15);
}

// Warp per row: e = exponent with max|x| < 2^e, then 8 truncated 7-bit digits of
// x * 2^-e (each step u*128 and u - trunc(u) is exact in f32); rows >= rows_valid
// (tile padding) and k >= K are zero.  Lane handles 4 consecutive k per step.
__global__ void __launch_bounds__(256, 3) k_slice_rows16(const float* __restrict__ x, int rows_valid, int rows_pad, int K,
                             int ld, int kchunks, int tile_rows, int8_t* __restrict__ planes,
                             int* __restrict__ exps) {
  const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int Kp = kchunks * kSlBK;
  if (row >= rows_pad) return;
  const bool valid = row < rows_valid;
  const float* r = x + (size_t)(valid ? row : 0) * ld;
  // the row is read once: up to kSlRegK elements stay in registers (16 consecutive per
  // lane per 512-element step) between the max pass and the slicing (two passes over
  // global memory were latency-bound: C2 41 us for 7.7 M elements), and each lane's 16
  // digits of one slice are one 16-byte store (4-byte stores kept the LSU busy: C3 97 us)
  constexpr int kV = kSlRegK / 512;
  const bool vec = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  auto load4 = [&](int k0) {
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!valid || k0 >= K) return u;
    if (vec && k0 + 4 <= K) return __ldg(reinterpret_cast<const float4*>(r + k0));
    u.x = __ldg(r + k0);
    if (k0 + 1 < K) u.y = __ldg(r + k0 + 1);
    if (k0 + 2 < K) u.z = __ldg(r + k0 + 2);
    if (k0 + 3 < K) u.w = __ldg(r + k0 + 3);
    return u;
  };
  float4 xv[kV][4];
  float mx = 0.f;
  if (Kp <= kSlRegK) {
#pragma unroll
    for (int i = 0; i < kV; ++i)
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        xv[i][v] = load4(lane * 16 + 512 * i + 4 * v);
        mx = fmaxf(mx, fmaxf(fmaxf(fabsf(xv[i][v].x), fabsf(xv[i][v].y)),
                             fmaxf(fabsf(xv[i][v].z), fabsf(xv[i][v].w))));
      }
  } else if (valid) {
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(__ldg(r + k)));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = mx > 0.f ? ilogbf(mx) + 1 : 0;
  if (lane == 0) exps[row] = e;
  // |x| * 2^(56 - e) truncated to an integer (exact: x = m 2^x_e with a 24-bit m), whose
  // base-128 digits, signed like x, are the slices -- the same digits as peeling
  // trunc(u * 128) off u = x / 2^e eight times in f32 (each step exact; values below
  // 2^-56 of the row max have all-zero slices either way), in integer instructions
  auto fixed56 = [&](float xf) -> unsigned long long {
    const uint32_t bits = __float_as_uint(xf);
    const int be = (int)((bits >> 23) & 0xFFu);
    if (be == 0xFF) return 0ull;  // non-finite rows are rejected before the projection
    const unsigned long long m = be ? ((bits & 0x7FFFFFu) | 0x800000u) : (bits & 0x7FFFFFu);
    const int sh = (be ? be : 1) - 150 - e + 56;  // x = m 2^(be - 150)
    if (sh >= 0) return m << sh;                  // (< 2^56: |x| < 2^e)
    return sh > -64 ? m >> -sh : 0ull;
  };
  // k0 % 16 == 0: the 16 bytes of one slice are contiguous in the tiled layout
  auto slice16 = [&](int k0, const float4 (&xq)[4]) {
    unsigned long long f[16];
    uint32_t neg = 0;
#pragma unroll
    for (int v = 0; v < 4; ++v) {
      const float xs4[4] = {xq[v].x, xq[v].y, xq[v].z, xq[v].w};
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        f[4 * v + t] = fixed56(xs4[t]);
        neg |= (__float_as_uint(xs4[t]) >> 31) << (4 * v + t);
      }
    }
#pragma unroll
    for (int s = 0; s < kSl; ++s) {
      uint32_t word[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) {
        word[v] = 0;
#pragma unroll
        for (int t = 0; t < 4; ++t) {
          const int dg = (int)((f[4 * v + t] >> (7 * (kSl - 1 - s))) & 127u);
          word[v] |= (uint32_t)(uint8_t)(int8_t)(((neg >> (4 * v + t)) & 1u) ? -dg : dg) << (8 * t);
        }
      }
      *reinterpret_cast<uint4*>(planes + sl_tiled_off(row, k0, s, tile_rows, kchunks)) =
          make_uint4(word[0], word[1], word[2], word[3]);
    }
  };
  if (Kp <= kSlRegK) {
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int k0 = lane * 16 + 512 * i;
      if (k0 < Kp) slice16(k0, xv[i]);
    }
  } else {
    for (int k0 = lane * 16; k0 < Kp; k0 += 512) {
      float4 xq[4];
#pragma unroll
      for (int v = 0; v < 4; ++v) xq[v] = load4(k0 + 4 * v);
      slice16(k0, xq);
    }
  }
}

// (K <= 1024: 4 elements per lane per step -- fewer registers, more warps per SM;
// C2 37 us vs 45 us for k_slice_rows16, which wins from K = 1536: 71 vs 97 us)
__global__ void k_slice_rows(const float* __restrict__ x, int rows_valid, int rows_pad, int K,
                             int ld, int kchunks, int tile_rows, int8_t* __restrict__ planes,
                             int* __restrict__ exps) {
  const int row = (int)(((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5);
  const int lane = threadIdx.x & 31;
  const int Kp = kchunks * kSlBK;
  if (row >= rows_pad) return;
  const bool valid = row < rows_valid;
  const float* r = x + (size_t)(valid ? row : 0) * ld;
  // the row is read once: up to kSlRegK elements stay in registers (4 per lane per
  // 128-element step) between the max pass and the slicing (two passes over global
  // memory were latency-bound: C2 41 us for 7.7 M elements)
  constexpr int kV = kSlRegK / 128;
  const bool vec = ((ld & 3) == 0) && ((reinterpret_cast<uintptr_t>(x) & 15) == 0);
  auto load4 = [&](int k0) {
    float4 u = make_float4(0.f, 0.f, 0.f, 0.f);
    if (!valid || k0 >= K) return u;
    if (vec && k0 + 4 <= K) return __ldg(reinterpret_cast<const float4*>(r + k0));
    u.x = __ldg(r + k0);
    if (k0 + 1 < K) u.y = __ldg(r + k0 + 1);
    if (k0 + 2 < K) u.z = __ldg(r + k0 + 2);
    if (k0 + 3 < K) u.w = __ldg(r + k0 + 3);
    return u;
  };
  float4 xv[kV];
  float mx = 0.f;
  if (Kp <= kSlRegK) {
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      xv[i] = load4(lane * 4 + 128 * i);
      mx = fmaxf(mx, fmaxf(fmaxf(fabsf(xv[i].x), fabsf(xv[i].y)), fmaxf(fabsf(xv[i].z), fabsf(xv[i].w))));
    }
  } else if (valid) {
    for (int k = lane; k < K; k += 32) mx = fmaxf(mx, fabsf(__ldg(r + k)));
  }
  for (int o = 16; o > 0; o >>= 1) mx = fmaxf(mx, __shfl_xor_sync(0xffffffffu, mx, o));
  const int e = mx > 0.f ? ilogbf(mx) + 1 : 0;
  if (lane == 0) exps[row] = e;
  // |x| * 2^(56 - e) truncated to an integer (exact: x = m 2^x_e with a 24-bit m), whose
  // base-128 digits, signed like x, are the slices -- the same digits as peeling
  // trunc(u * 128) off u = x / 2^e eight times in f32 (each step exact; values below
  // 2^-56 of the row max have all-zero slices either way), in integer instructions
  auto fixed56 = [&](float xf) -> unsigned long long {
    const uint32_t bits = __float_as_uint(xf);
    const int be = (int)((bits >> 23) & 0xFFu);
    if (be == 0xFF) return 0ull;  // non-finite rows are rejected before the projection
    const unsigned long long m = be ? ((bits & 0x7FFFFFu) | 0x800000u) : (bits & 0x7FFFFFu);
    const int sh = (be ? be : 1) - 150 - e + 56;  // x = m 2^(be - 150)
    if (sh >= 0) return m << sh;                  // (< 2^56: |x| < 2^e)
    return sh > -64 ? m >> -sh : 0ull;
  };
  auto slice4 = [&](int k0, float4 xq) {
    const float xs4[4] = {xq.x, xq.y, xq.z, xq.w};
    unsigned long long f[4];
    uint32_t neg = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      f[t] = fixed56(xs4[t]);
      neg |= (__float_as_uint(xs4[t]) >> 31) << t;
    }
#pragma unroll
    for (int s = 0; s < kSl; ++s) {
      uint32_t word = 0;
#pragma unroll
      for (int t = 0; t < 4; ++t) {
        const int dg = (int)((f[t] >> (7 * (kSl - 1 - s))) & 127u);
        word |= (uint32_t)(uint8_t)(int8_t)(((neg >> t) & 1u) ? -dg : dg) << (8 * t);
      }
      *reinterpret_cast<uint32_t*>(planes + sl_tiled_off(row, k0, s, tile_rows, kchunks)) = word;
    }
  };
  if (Kp <= kSlRegK) {
#pragma unroll
    for (int i = 0; i < kV; ++i) {
      const int k0 = lane * 4 + 128 * i;
      if (k0 < Kp) slice4(k0, xv[i]);
    }
  } else {
    for (int k0 = lane * 4; k0 < Kp; k0 += 128) slice4(k0, load4(k0));
  }
}

// ------------------------------------------------------------------ helpers
__device__ __forceinline__ uint32_t sl_smem(const void* p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
// K-major, no swizzle: start >> 4, LBO (K direction) 128 B, SBO (8-row groups) 256 B,
// descriptor version 1 (sm_100), layout type 0.
__device__ __forceinline__ uint64_t sl_desc(uint32_t addr) {
  return (uint64_t)((addr >> 4) & 0x3FFFu) | ((uint64_t)(128 >> 4) << 16) |
         ((uint64_t)(256 >> 4) << 32) | (1ull << 46);
}
// kind::i8 instruction descriptor: D s32, A/B signed int8, K-major, N = 64, M = 128
constexpr uint32_t kSlIdesc = (2u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(kSlBN >> 3) << 17) |
                              ((uint32_t)(kSlBM >> 4) << 24);

__device__ __forceinline__ void sl_mma(uint32_t tmem, uint64_t ad, uint64_t bd, uint32_t acc) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::i8 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem),
      "l"(ad), "l"(bd), "r"(kSlIdesc), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void sl_commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   sl_smem(bar))
               : "memory");
}
__device__ __forceinline__ void sl_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "SL_WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra SL_WAIT_%=;\n\t}" ::"r"(sl_smem(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void sl_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(sl_smem(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void sl_bulk(uint32_t dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(dst),
      "l"(src), "r"(bytes), "r"(sl_smem(bar))
      : "memory");
}

struct SlicedGemmArgs {
  const int8_t* a;   // tiled planes of A (row blocks of kSlBM)
  const int* a_exp;  // [M padded]
  const int8_t* b;   // tiled planes of B (row blocks of kSlBN)
  const int* b_exp;  // [N padded]
  int M, N, kchunks;
  int epi;           // EPI_PROJ (f32 store) | EPI_L2 (clipped f64 distance) | EPI_NEGIP
  float* outf;
  double* outd;
  int64_t ldo;
  const double* rowterm;
  const double* colterm;
  int* outi;  // EPI_*_ARGMIN: per (row, column tile) nearest column
};

// Warp 0 (one lane): bulk-copy producer over a kSlStages ring; warp 1 (one lane):
// MMA issuer; all four warps: epilogue (warp w owns TMEM lanes 32w..32w+31).
__global__ void __launch_bounds__(kSlThreads, 1) k_gemm_sliced(SlicedGemmArgs g) {
  extern __shared__ __align__(1024) unsigned char sl_sm[];
  __shared__ uint64_t full[kSlStages], empty[kSlStages], done;
  __shared__ uint32_t tmem_base;
  // the tile's per-column terms, staged once: the epilogue read them per output from
  // global memory, a dependent load ahead of every column's arithmetic (it was ~2/3 of
  // the kernel's time at C2)
  __shared__ double col_sc[kSlBN], col_t[kSlBN];
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  const int mb = blockIdx.y, nb = blockIdx.x;
  const int m0 = mb * kSlBM, n0 = nb * kSlBN;
  // 2^e as an exact f64 power of two (|e| stays far inside the range)
  auto pow2 = [](int e) { return __longlong_as_double((long long)(1023 + e) << 52); };
  if (tid >= 64 && tid < 64 + kSlBN) {
    const int j = tid - 64, gn = n0 + j;
    col_sc[j] = gn < g.N ? pow2(g.b_exp[gn]) : 0.0;
    col_t[j] = gn < g.N && g.colterm ? g.colterm[gn] : 0.0;
  }
  unsigned char* base = reinterpret_cast<unsigned char*>(
      (reinterpret_cast<uintptr_t>(sl_sm) + 1023) & ~uintptr_t(1023));
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 512;" ::"r"(
                     sl_smem(&tmem_base))
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  if (tid == 32) {
    for (int i = 0; i < kSlStages; ++i) {
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sl_smem(&full[i])));
      asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sl_smem(&empty[i])));
    }
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(sl_smem(&done)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = tmem_base;
  const int nk = g.kchunks;
  if (tid == 0) {  // producer
    const int8_t* ga = g.a + (size_t)mb * nk * kSlAStage;
    const int8_t* gb = g.b + (size_t)nb * nk * kSlBStage;
    for (int kc = 0; kc < nk; ++kc) {
      const int st = kc % kSlStages;
      if (kc >= kSlStages) sl_wait(&empty[st], ((kc / kSlStages) - 1) & 1);
      const uint32_t sa = sl_smem(base + (size_t)st * kSlStage);
#ifdef SL_NO_RELOAD  // probe: MMA throughput with the operands already on-chip
      if (kc >= kSlStages) {
        asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(sl_smem(&full[st])) : "memory");
        continue;
      }
#endif
      sl_expect_tx(&full[st], kSlStage);
      sl_bulk(sa, ga + (size_t)kc * kSlAStage, kSlAStage, &full[st]);
      sl_bulk(sa + kSlAStage, gb + (size_t)kc * kSlBStage, kSlBStage, &full[st]);
    }
  } else if (tid == 32) {  // MMA issuer
    for (int kc = 0; kc < nk; ++kc) {
      const int st = kc % kSlStages;
      sl_wait(&full[st], (kc / kSlStages) & 1);
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      // descriptors advance by adds to the start-address field (addr >> 4)
      const uint64_t ad = sl_desc(sl_smem(base + (size_t)st * kSlStage));
      const uint64_t bd = ad + (uint64_t)(kSlAStage >> 4);
#pragma unroll
      for (int i = 0; i < kSl; ++i)
#pragma unroll
        for (int j = 0; j < kSl - i; ++j) {
          const uint32_t first = kc == 0 && i == 0;  // first product into level i+j
          sl_mma(tmem + (uint32_t)((i + j) * kSlBN), ad + (uint64_t)((i * kSlATile) >> 4),
                 bd + (uint64_t)((j * kSlBTile) >> 4), first ? 0u : 1u);
        }
      sl_commit(&empty[st]);
    }
    sl_commit(&done);
  }
  __syncwarp();
  sl_wait(&done, 0);
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  // epilogue
  const int gm = m0 + warp * 32 + lane;
  const uint32_t lane_addr = tmem + ((uint32_t)(warp * 32) << 16);
  const double sa = pow2(g.a_exp[gm] - 14);  // 2^(ea - 14); padded rows have exponent 0
  const double rterm = (g.epi == EPI_L2 || g.epi == EPI_L2_ARGMIN) && gm < g.M ? g.rowterm[gm] : 0.0;
  constexpr double kInf = __builtin_huge_val();
  double best = kInf;  // EPI_*_ARGMIN: this row's (value, lowest column) over the tile
  int bcol = 0x7fffffff;
#pragma unroll 1
  for (int c0 = 0; c0 < kSlBN; c0 += 16) {
    uint32_t v[kSl][16];
#pragma unroll
    for (int l = 0; l < kSl; ++l)
      asm volatile(
          "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,"
          "%14,%15}, [%16];"
          : "=r"(v[l][0]), "=r"(v[l][1]), "=r"(v[l][2]), "=r"(v[l][3]), "=r"(v[l][4]),
            "=r"(v[l][5]), "=r"(v[l][6]), "=r"(v[l][7]), "=r"(v[l][8]), "=r"(v[l][9]),
            "=r"(v[l][10]), "=r"(v[l][11]), "=r"(v[l][12]), "=r"(v[l][13]), "=r"(v[l][14]),
            "=r"(v[l][15])
          : "r"(lane_addr + (uint32_t)(l * kSlBN + c0)));
    asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
    if (gm < g.M && g.epi == EPI_PROJ && (g.ldo & 3) == 0 && (reinterpret_cast<uintptr_t>(g.outf) & 15) == 0 &&
        n0 + c0 + 16 <= g.N) {
      // 16 consecutive columns of this thread's row as four 16-byte stores (a store per
      // column wrote 4 bytes into 32 different rows' sectors per warp instruction)
      float f[16];
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        double acc = 0.0;
#pragma unroll
        for (int l = kSl - 1; l >= 0; --l) acc = fma(acc, 0.0078125, (double)(int)v[l][j]);
        f[j] = (float)((acc * sa) * col_sc[c0 + j]);
      }
      float4* o = reinterpret_cast<float4*>(g.outf + (size_t)gm * g.ldo + n0 + c0);
#pragma unroll
      for (int j = 0; j < 4; ++j) o[j] = make_float4(f[4 * j], f[4 * j + 1], f[4 * j + 2], f[4 * j + 3]);
    } else if (gm < g.M) {
#pragma unroll
      for (int j = 0; j < 16; ++j) {
        const int gn = n0 + c0 + j;
        double acc = 0.0;
#pragma unroll
        for (int l = kSl - 1; l >= 0; --l) acc = fma(acc, 0.0078125, (double)(int)v[l][j]);
        if (gn >= g.N) continue;
        const double val = (acc * sa) * col_sc[c0 + j];
        if (g.epi == EPI_PROJ) {
          g.outf[(size_t)gm * g.ldo + gn] = (float)val;
        } else if (g.epi == EPI_L2 || g.epi == EPI_L2_ARGMIN) {
          double d2 = __dadd_rn(__dsub_rn(rterm, __dmul_rn(2.0, val)), col_t[c0 + j]);
          d2 = d2 > 0.0 ? d2 : 0.0;
          if (g.epi == EPI_L2) g.outd[(size_t)gm * g.ldo + gn] = d2;
          else if (d2 < best) { best = d2; bcol = gn; }  // columns ascend: ties keep the lowest
        } else if (g.epi == EPI_NEGIP_ARGMIN) {
          const double dv = -val == -val ? -val : kInf;  // NaN (non-finite query) ranks as +inf
          if (dv < best || (dv == best && gn < bcol)) { best = dv; bcol = gn; }
        } else {
          g.outd[(size_t)gm * g.ldo + gn] = -val;
        }
      }
    }
  }
  if ((g.epi == EPI_L2_ARGMIN || g.epi == EPI_NEGIP_ARGMIN) && gm < g.M) {
    g.outd[(size_t)gm * g.ldo + nb] = best;
    g.outi[(size_t)gm * g.ldo + nb] = bcol;
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  if (warp == 0)
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 512;" ::"r"(tmem) : "memory");
}

// ------------------------------------------------------------------ launchers
int sliced_kchunks(int K) { return (K + kSlBK - 1) / kSlBK; }
int sliced_rows_pad(int rows, bool a_operand) {
  const int t = a_operand ? kSlBM : kSlBN;
  return (rows + t - 1) / t * t;
}
size_t sliced_block_bytes(int K, bool a_operand) {
  return (size_t)sliced_kchunks(K) * kSl * (a_operand ? kSlBM : kSlBN) * kSlBK;
}
size_t sliced_plane_bytes(int rows, int K, bool a_operand) {
  return (size_t)kSl * sliced_rows_pad(rows, a_operand) * (size_t)sliced_kchunks(K) * kSlBK;
}

void launch_slice_rows(const float* x, int rows, int K, int ld, bool a_operand, int8_t* planes,
                       int* exps, cudaStream_t st) {
  const int rp = sliced_rows_pad(rows, a_operand);
  const int64_t blocks = ((int64_t)rp * 32 + 255) / 256;
  if (K > 1024)
    (k_slice_rows16<<<(unsigned)blocks, 256, 0, st>>>(x, rows, rp, K, ld, sliced_kchunks(K),
                                                     a_operand ? kSlBM : kSlBN, planes, exps), note_launch());
  else
    (k_slice_rows<<<(unsigned)blocks, 256, 0, st>>>(x, rows, rp, K, ld, sliced_kchunks(K),
                                                   a_operand ? kSlBM : kSlBN, planes, exps), note_launch());
}

void launch_gemm_sliced(const int8_t* a, const int* a_exp, int M, const int8_t* b, const int* b_exp,
                        int N, int K, int epi, float* outf, double* outd, int64_t ldo,
                        const double* rowterm, const double* colterm, cudaStream_t st, int* outi) {
  static int done[64] = {};
  int dev = 0;
  cudaGetDevice(&dev);
  if (dev >= 0 && dev < 64 && !done[dev]) {
    cudaFuncSetAttribute((const void*)k_gemm_sliced, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)kSlSmem);
    done[dev] = 1;
  }
  SlicedGemmArgs g;
  g.a = a; g.a_exp = a_exp; g.b = b; g.b_exp = b_exp; g.M = M; g.N = N;
  g.kchunks = sliced_kchunks(K);
  g.epi = epi; g.outf = outf; g.outd = outd; g.ldo = ldo; g.rowterm = rowterm; g.colterm = colterm;
  g.outi = outi;
  dim3 grid((N + kSlBN - 1) / kSlBN, (M + kSlBM - 1) / kSlBM);
  (k_gemm_sliced<<<grid, kSlThreads, kSlSmem, st>>>(g), note_launch());
}

}  // namespace rrg
