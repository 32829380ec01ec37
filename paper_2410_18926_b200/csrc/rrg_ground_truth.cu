// rrg_ground_truth.cu -- exact k-NN ground truth on the GPU.
//
// Restates the reference's `brute_force_knn` (pkg/src/rrann/bench.py:85-124):
//   euclidean  diss = (q*q).sum(1)[:,None] - 2*(q @ c.T) + (c*c).sum(1)[None,:]   (f64)
//   ip         diss = -(q @ c.T)                                                   (f64)
//   cosine     diss = -(q @ (c / ||c||).T), ||c|| = 0 -> 1                         (f64)
//   ids        argsort(diss, kind="stable")[:, :k]  -> ties toward the lower id
// Recall@k of the 1M / 10M workloads needs this: the CPU reference takes minutes
// to hours at those sizes.
//
// Pipeline per (query chunk, corpus chunk): the f64 distance block comes from the
// FP64 tensor-core GEMM (k_gemm_dmma, EPI_GT_*; rrg_kernels.cu), then
// k_gt_select merges it with the running top-k of each query.  k_gt_select is a
// CTA-per-query radix select on order-preserving 64-bit keys of the f64
// distances (11-bit digits): passes stream the distance row from HBM until the
// rows still matching the selected prefix fit in shared memory, are compacted
// there, and the remaining passes run on-chip.  The k selected (key, id) pairs
// are then sorted by (key, id) -- the stable argsort's order.
#include <cuda_runtime.h>
#include <stdint.h>

#include "rrg_common.cuh"
#include "rrg_kernels.h"

namespace rrg {

constexpr int GT_T = 512;        // threads per select CTA
constexpr int GT_BINS = 2048;    // 11-bit digits: 64 = 5 x 11 + 9
constexpr int GT_CAP = 4096;     // on-chip candidate capacity

__global__ void k_gt_row_norms(const float* __restrict__ x, int64_t n, int d, int mode,
                               double* __restrict__ out) {
  // warp per row: mode 0 -> sum of squares (f64), 1 -> sqrt of it with 0 -> 1
  const int64_t row = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= n) return;
  const float* r = x + row * d;
  double s = 0.0;
  for (int i = lane; i < d; i += 32) {
    const double v = (double)__ldg(r + i);
    s = fma(v, v, s);
  }
  for (int o = 16; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if (lane == 0) {
    if (mode == 1) {
      s = sqrt(s);
      if (s == 0.0) s = 1.0;
    }
    out[row] = s;
  }
}

struct GtSelectArgs {
  const double* diss;     // [nq][ld] distance block of this corpus chunk
  int64_t ld;
  int n;                  // valid columns
  int64_t id0;            // corpus id of column 0
  const uint64_t* run_key;  // [nq][k] running top-k (or nullptr)
  const int64_t* run_id;
  const int* run_n;
  uint64_t* out_key;      // [nq][k]
  int64_t* out_id;
  int* out_n;
  int k;
  int* err;               // set when the boundary ties exceed the on-chip capacity
};

__device__ __forceinline__ void gt_item(const GtSelectArgs& a, const double* row, int kc, int i,
                                        uint64_t& key, int64_t& id, int q) {
  if (i < a.n) {
    key = mono64(row[i]);  // order-preserving, -0.0 -> +0.0 (rrg_common.cuh)
    id = a.id0 + i;
  } else {
    key = a.run_key[(size_t)q * a.k + (i - a.n)];
    id = a.run_id[(size_t)q * a.k + (i - a.n)];
  }
  (void)kc;
}

// Block-wide exclusive scan of one int per thread (GT_T threads); returns the total.
__device__ int gt_block_scan(int v, int* excl, int* warp_tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int incl = v;
  for (int o = 1; o < 32; o <<= 1) {
    int t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) warp_tot[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int w = lane < GT_T / 32 ? warp_tot[lane] : 0, wi = w;
    for (int o = 1; o < 32; o <<= 1) {
      int t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < GT_T / 32) warp_tot[lane] = wi - w;  // exclusive warp offsets
    if (lane == 31) warp_tot[GT_T / 32] = wi;
  }
  __syncthreads();
  *excl = warp_tot[warp] + incl - v;
  const int total = warp_tot[GT_T / 32];
  __syncthreads();
  return total;
}

__global__ void __launch_bounds__(GT_T) k_gt_select(GtSelectArgs a) {
  extern __shared__ __align__(16) unsigned char gsm[];
  uint64_t* ckey = reinterpret_cast<uint64_t*>(gsm);            // GT_CAP
  int64_t* cid = reinterpret_cast<int64_t*>(ckey + GT_CAP);     // GT_CAP
  uint64_t* skey = reinterpret_cast<uint64_t*>(cid + GT_CAP);   // k (selected)
  int64_t* sid = reinterpret_cast<int64_t*>(skey + a.k);        // k
  int* hist = reinterpret_cast<int*>(sid + a.k);                // GT_BINS
  __shared__ int warp_tot[GT_T / 32 + 1];
  __shared__ int s_nsel, s_ncand, s_bin, s_before, s_ntie;
  const int q = blockIdx.x, tid = threadIdx.x;
  const double* row = a.diss + (size_t)q * a.ld;
  const int kc = a.run_n ? a.run_n[q] : 0;
  const int N = a.n + kc;
  const int k = a.k;
  if (tid == 0) { s_nsel = 0; s_ncand = 0; s_ntie = 0; }
  __syncthreads();
  int take = min(k, N);
  if (N <= k) {  // everything is selected
    for (int i = tid; i < N; i += GT_T) {
      uint64_t key; int64_t id;
      gt_item(a, row, kc, i, key, id, q);
      skey[i] = key; sid[i] = id;
    }
  } else {
    // radix select on the 128-bit composite (key, id): passes 0-5 fix the key's
    // digits, passes 6-11 (only reached with more than GT_CAP exact ties at the
    // k-th key) the id's
    uint64_t pk = 0, mk = 0, pi = 0, mi = 0;  // prefix / mask of key and id
    int kk = k;               // rank (1-based) of the k-th smallest among matching items
    bool local = false;       // candidates compacted on-chip
    int m = N;                // items matching the prefix
    int ncand = 0;            // compacted candidates (local)
    auto matches = [&](uint64_t key, int64_t id) {
      return (key & mk) == pk && ((uint64_t)id & mi) == pi;
    };
    auto below = [&](uint64_t key, int64_t id, uint64_t npk, uint64_t nmk, uint64_t npi,
                     uint64_t nmi) {
      const uint64_t a = key & nmk;
      return a < npk || (a == npk && ((uint64_t)id & nmi) < npi);
    };
    for (int pass = 0; pass < 12; ++pass) {
      if (pass >= 6 && local) break;  // key fixed, ties on-chip: ranked by id below
      const int pp = pass % 6;
      const int width = pp < 5 ? 11 : 9;
      const int shift = pp < 5 ? 64 - 11 * (pp + 1) : 0;
      const uint64_t dmask = ((1ull << width) - 1ull) << shift;
      const bool on_id = pass >= 6;
      for (int b = tid; b < GT_BINS; b += GT_T) hist[b] = 0;
      __syncthreads();
      if (!local) {
        for (int i = tid; i < N; i += GT_T) {
          uint64_t key; int64_t id;
          gt_item(a, row, kc, i, key, id, q);
          if (matches(key, id))
            atomicAdd(&hist[((on_id ? (uint64_t)id : key) & dmask) >> shift], 1);
        }
      } else {
        for (int i = tid; i < ncand; i += GT_T) {
          const uint64_t key = ckey[i];
          atomicAdd(&hist[(key & dmask) >> shift], 1);  // all match (compacted)
        }
      }
      __syncthreads();
      // find the digit holding rank kk: 4 bins per thread, block scan
      int c4 = 0;
      for (int j = 0; j < GT_BINS / GT_T; ++j) c4 += hist[tid * (GT_BINS / GT_T) + j];
      int excl;
      gt_block_scan(c4, &excl, warp_tot);
      if (excl < kk && kk <= excl + c4) {
        int run = excl;
        for (int j = 0; j < GT_BINS / GT_T; ++j) {
          const int b = tid * (GT_BINS / GT_T) + j;
          if (run + hist[b] >= kk) { s_bin = b; s_before = run; break; }
          run += hist[b];
        }
      }
      __syncthreads();
      const int bin = s_bin;
      kk -= s_before;
      m = hist[bin];
      uint64_t npk = pk, nmk = mk, npi = pi, nmi = mi;
      if (on_id) { npi |= (uint64_t)bin << shift; nmi |= dmask; }
      else { npk |= (uint64_t)bin << shift; nmk |= dmask; }
      __syncthreads();
      if (!local && m <= GT_CAP) {
        // compact: items below the prefix are selected outright, matching ones kept
        for (int i = tid; i < N; i += GT_T) {
          uint64_t key; int64_t id;
          gt_item(a, row, kc, i, key, id, q);
          if (below(key, id, npk, nmk, npi, nmi)) {
            const int slot = atomicAdd(&s_nsel, 1);
            skey[slot] = key; sid[slot] = id;
          } else if ((key & nmk) == npk && ((uint64_t)id & nmi) == npi) {
            const int slot = atomicAdd(&s_ncand, 1);
            ckey[slot] = key; cid[slot] = id;
          }
        }
        __syncthreads();
        local = true;
        m = ncand = s_ncand;
      } else if (local) {
        // move candidates below the new prefix to the selection; keep matching ones
        uint64_t rk[GT_CAP / GT_T];
        int64_t ri[GT_CAP / GT_T];
        int cnt = 0;
        for (int i = tid; i < ncand; i += GT_T) { rk[cnt] = ckey[i]; ri[cnt] = cid[i]; ++cnt; }
        __syncthreads();
        if (tid == 0) s_ncand = 0;
        __syncthreads();
        for (int j = 0; j < cnt; ++j) {
          if (below(rk[j], ri[j], npk, nmk, npi, nmi)) {
            const int slot = atomicAdd(&s_nsel, 1);
            skey[slot] = rk[j]; sid[slot] = ri[j];
          } else if ((rk[j] & nmk) == npk) {
            const int slot = atomicAdd(&s_ncand, 1);
            ckey[slot] = rk[j]; cid[slot] = ri[j];
          }
        }
        __syncthreads();
        m = ncand = s_ncand;
      }
      pk = npk; mk = nmk; pi = npi; mi = nmi;
    }
    // all 64 bits fixed: the m candidates are exact ties at the k-th key; take the kk
    // with the smallest ids (stable argsort order)
    for (int i = tid; i < m; i += GT_T) {
      const int64_t id = cid[i];
      int rank = 0;
      for (int j = 0; j < m; ++j) rank += cid[j] < id;
      if (rank < kk) {
        const int slot = atomicAdd(&s_nsel, 1);
        skey[slot] = ckey[i]; sid[slot] = id;
      }
    }
    __syncthreads();
  }
  __syncthreads();
  // bitonic sort of the take selected pairs by (key, id), padded to a power of two
  int np2 = 1;
  while (np2 < take) np2 <<= 1;
  uint64_t* tk = ckey;  // reuse the candidate region (np2 <= 2048 <= GT_CAP)
  int64_t* ti = cid;
  for (int i = tid; i < np2; i += GT_T) {
    if (i < take) { tk[i] = skey[i]; ti[i] = sid[i]; }
    else { tk[i] = ~0ull; ti[i] = INT64_MAX; }
  }
  __syncthreads();
  for (int size = 2; size <= np2; size <<= 1) {
    for (int stride = size >> 1; stride > 0; stride >>= 1) {
      for (int i = tid; i < np2; i += GT_T) {
        const int j = i ^ stride;
        if (j > i) {
          const bool up = (i & size) == 0;
          const bool gt = tk[i] > tk[j] || (tk[i] == tk[j] && ti[i] > ti[j]);
          if (gt == up) {
            uint64_t t0 = tk[i]; tk[i] = tk[j]; tk[j] = t0;
            int64_t t1 = ti[i]; ti[i] = ti[j]; ti[j] = t1;
          }
        }
      }
      __syncthreads();
    }
  }
  for (int i = tid; i < take; i += GT_T) {
    a.out_key[(size_t)q * k + i] = tk[i];
    a.out_id[(size_t)q * k + i] = ti[i];
  }
  if (tid == 0) a.out_n[q] = take;
}

size_t gt_select_smem(int k) {
  return (size_t)GT_CAP * 16 + (size_t)k * 16 + GT_BINS * 4;
}

void launch_gt_row_norms(const float* x, int64_t n, int d, int mode, double* out, cudaStream_t st) {
  const int64_t blocks = (n * 32 + 255) / 256;
  (k_gt_row_norms<<<(unsigned)blocks, 256, 0, st>>>(x, n, d, mode, out), note_launch());
}

void launch_gt_select(const GtSelectHost& h, int nq, cudaStream_t st) {
  GtSelectArgs a;
  a.diss = h.diss; a.ld = h.ld; a.n = h.n; a.id0 = h.id0; a.run_key = h.run_key;
  a.run_id = h.run_id; a.run_n = h.run_n; a.out_key = h.out_key; a.out_id = h.out_id;
  a.out_n = h.out_n; a.k = h.k; a.err = h.err;
  const size_t smem = gt_select_smem(h.k);
  cudaFuncSetAttribute(k_gt_select, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  (k_gt_select<<<nq, GT_T, smem, st>>>(a), note_launch());
}

}  // namespace rrg
