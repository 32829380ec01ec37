// rrg_api.cu -- C ABI of librrg.so: index loading/upload and batched search orchestration.
//
// Reference boundary replaced (see include/rrg.h):
//   RrrIndex.load / deserialize   pkg/src/rrann/index.py:138-141, 405-507
//   query_batch / query           pkg/src/rrann/index.py:286-340
//   QueryParams.validate          pkg/src/rrann/index.py:92-100
#include <cuda_runtime.h>
#include <zlib.h>

#include <algorithm>
#include <atomic>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <map>
#include <tuple>
#include <vector>

#include "../../include/rrg.h"
#include "rrg_common.cuh"
#include "rrg_kernels.h"

using namespace rrg;

// ------------------------------------------------------------------ errors

namespace {

thread_local std::string g_err;
thread_local std::string g_kind;
thread_local int64_t g_launches = 0;  // kernels launched by this thread (note_launch)

// per-stage event timing (rrg_set_stage_timing / rrg_stage_times)
struct StageTimer {
  bool on = false;
  struct Rec { int stage; cudaEvent_t a, b; };
  std::vector<Rec> pending;
  double ms[RRG_N_STAGES] = {0};
  int64_t n[RRG_N_STAGES] = {0};
  std::vector<cudaEvent_t> pool;
  int64_t* dcounters = nullptr;  // device counters (rrg_search_counters), while timing is on
  int cdev = -1;
  // critical-path spans on the launching stream (rrg_path_times)
  cudaEvent_t path_open[RRG_N_PATHS] = {};
  std::vector<Rec> path_pending;
  double pms[RRG_N_PATHS] = {0};
  int64_t pn[RRG_N_PATHS] = {0};
  cudaEvent_t get() {
    if (!pool.empty()) { cudaEvent_t e = pool.back(); pool.pop_back(); return e; }
    cudaEvent_t e;
    cudaEventCreate(&e);
    return e;
  }
};
thread_local StageTimer g_timer;

// A second stream per host thread and device: work that depends only on the pair
// bucketing (query interleave, the screen's group records) overlaps the top-t selection.
struct AuxStream {
  int device = -1;
  cudaStream_t s = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr, cfork = nullptr, cjoin = nullptr;
  ~AuxStream() {
    if (s) cudaStreamDestroy(s);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    if (cfork) cudaEventDestroy(cfork);
    if (cjoin) cudaEventDestroy(cjoin);
  }
};
thread_local AuxStream g_aux;
AuxStream& aux_stream() {
  int dev = 0;
  cudaGetDevice(&dev);
  AuxStream& a = g_aux;
  if (a.device != dev) {
    if (a.s) cudaStreamDestroy(a.s);
    if (a.fork) cudaEventDestroy(a.fork);
    if (a.join) cudaEventDestroy(a.join);
    if (a.cfork) cudaEventDestroy(a.cfork);
    if (a.cjoin) cudaEventDestroy(a.cjoin);
    cudaStreamCreateWithFlags(&a.s, cudaStreamNonBlocking);
    cudaEventCreateWithFlags(&a.fork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&a.join, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&a.cfork, cudaEventDisableTiming);
    cudaEventCreateWithFlags(&a.cjoin, cudaEventDisableTiming);
    a.device = dev;
  }
  return a;
}

[[noreturn]] void launch_failed(int stage, cudaError_t e);

// Work counters of the re-rank (rrg_search_counters), collected while stage timing is
// enabled; nullptr otherwise, so the search path never touches them.
int64_t* counters_ptr(cudaStream_t st) {
  StageTimer& t = g_timer;
  if (!t.on) return nullptr;
  int dev = 0;
  cudaGetDevice(&dev);
  if (t.dcounters == nullptr || t.cdev != dev) {
    if (cudaMalloc(&t.dcounters, RRG_N_COUNTERS * 8) != cudaSuccess) return t.dcounters = nullptr;
    cudaMemsetAsync(t.dcounters, 0, RRG_N_COUNTERS * 8, st);
    t.cdev = dev;
  }
  return t.dcounters;
}

// Runs one launch, counting it and (when enabled) bracketing it with events; a launch
// rejected at submission (bad grid / shared-memory size) fails here, naming its stage.
void path_begin(int p, cudaStream_t st) {
  StageTimer& t = g_timer;
  if (!t.on) return;
  if (t.path_open[p]) t.pool.push_back(t.path_open[p]);
  t.path_open[p] = t.get();
  cudaEventRecord(t.path_open[p], st);
}
void path_end(int p, cudaStream_t st) {
  StageTimer& t = g_timer;
  if (!t.on || !t.path_open[p]) return;
  StageTimer::Rec r{p, t.path_open[p], t.get()};
  cudaEventRecord(r.b, st);
  t.path_pending.push_back(r);
  t.path_open[p] = nullptr;
}

template <typename F>
void staged(int stage, cudaStream_t st, F&& launch) {
  StageTimer& t = g_timer;
  if (t.on) {
    StageTimer::Rec r{stage, t.get(), t.get()};
    cudaEventRecord(r.a, st);
    launch();
    cudaEventRecord(r.b, st);
    t.pending.push_back(r);
  } else {
    launch();
  }
  cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) launch_failed(stage, e);
}

int fail(int code, const char* kind, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  g_kind = kind;
  return code;
}

struct RrgFail {
  int code;
};

void launch_failed(int stage, cudaError_t e) {
  cudaGetLastError();
  fail(RRG_E_INTERNAL, "RrannError", "CUDA error %s at launch %lld (stage %d): %s", cudaGetErrorName(e),
       (long long)g_launches, stage, cudaGetErrorString(e));
  throw RrgFail{RRG_E_INTERNAL};
}

#define CUDA_TRY(expr)                                                                        \
  do {                                                                                        \
    cudaError_t e_ = (expr);                                                                  \
    if (e_ != cudaSuccess) {                                                                  \
      fail(RRG_E_INTERNAL, "RrannError", "CUDA error %s at %s:%d: %s", cudaGetErrorName(e_), \
           __FILE__, __LINE__, cudaGetErrorString(e_));                                       \
      throw RrgFail{RRG_E_INTERNAL};                                                          \
    }                                                                                         \
  } while (0)

[[noreturn]] void raise_format(const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  g_kind = "FormatError";
  throw RrgFail{RRG_E_DATA};
}

[[noreturn]] void raise_usage(const char* kind, const char* fmt, ...) {
  char buf[1024];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof buf, fmt, ap);
  va_end(ap);
  g_err = buf;
  g_kind = kind;
  throw RrgFail{RRG_E_USAGE};
}

// Python-style repr of a bytes object (for the "bad magic" message, index.py:447).
std::string py_bytes_repr(const unsigned char* b, size_t n) {
  std::string s = "b'";
  for (size_t i = 0; i < n; ++i) {
    unsigned c = b[i];
    char tmp[8];
    if (c == '\\') s += "\\\\";
    else if (c == '\'') s += "\\'";
    else if (c == '\t') s += "\\t";
    else if (c == '\n') s += "\\n";
    else if (c == '\r') s += "\\r";
    else if (c >= 32 && c < 127) s += (char)c;
    else { snprintf(tmp, sizeof tmp, "\\x%02x", c); s += tmp; }
  }
  return s + "'";
}

// NumPy float64 pairwise sum (same tree as rrg_common.cuh pw_sum_seq).
double pw_sum_host(const double* a, int64_t n) {
  if (n < 8) {
    double r = 0.0;
    for (int64_t i = 0; i < n; ++i) r += a[i];
    return r;
  }
  if (n <= 128) {
    double r[8];
    for (int j = 0; j < 8; ++j) r[j] = a[j];
    int64_t i = 8;
    for (; i < n - (n % 8); i += 8)
      for (int j = 0; j < 8; ++j) r[j] += a[i + j];
    double res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]));
    for (; i < n; ++i) res += a[i];
    return res;
  }
  int64_t n2 = n / 2;
  n2 -= n2 % 8;
  return pw_sum_host(a, n2) + pw_sum_host(a + n2, n - n2);
}

int64_t round_up(int64_t v, int64_t a) { return (v + a - 1) / a * a; }

// ---------------------------------------------------------- host staging

struct HostCluster {
  uint32_t m = 0;
  bool exact = false;
  bool owned = true;
  std::vector<int64_t> ids;
  std::vector<float> a_head, a_scale;
  std::vector<int8_t> a_vals;  // s x cols (row 0 = pad)
  std::vector<float> b_head, b_scale;
  std::vector<int8_t> b_vals;  // r x m
  std::vector<float> a_f, b_f;  // unquantized factors (quantize=False): s x cols, r x m
  std::vector<float> norms;
};

struct HostModel {
  int metric = 0, d = 0, s = 0, r = 0, L = 0;
  int64_t m = 0;
  uint32_t flags = 0;
  std::vector<float> projection, centroids;
  std::vector<HostCluster> clusters;
};

}  // namespace

void rrg::note_launch() { ++g_launches; }

// ------------------------------------------------------------------ index

struct RrgIndex {
  // process-unique id: keys cached per-thread state (captured graphs) so a later
  // index allocated at a freed one's address never reuses it
  uint64_t serial = next_serial();
  static uint64_t next_serial() {
    static std::atomic<uint64_t> n{0};
    return ++n;
  }
  int device = 0;
  HostModel meta;  // header fields only (vectors released after upload)
  DevIndexView view{};
  std::vector<void*> allocs;
  RrgIndexInfo info{};
  int64_t max_cluster = 0;
  double m_biased = 0.0;  // size-biased mean cluster size: sum m_l^2 / sum m_l
  std::vector<int> sizes_sorted_desc;  // cluster sizes (held), descending
  std::vector<uint32_t> held_sizes;    // per cluster
  int n_exact = 0;

  void* dalloc(size_t bytes) {
    void* p = nullptr;
    if (bytes == 0) bytes = 16;
    CUDA_TRY(cudaMalloc(&p, bytes));
    allocs.push_back(p);
    info.device_bytes += bytes;
    return p;
  }
  template <typename T>
  T* upload(const std::vector<T>& v) {
    T* p = static_cast<T*>(dalloc(v.size() * sizeof(T)));
    if (!v.empty()) CUDA_TRY(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
    return p;
  }
  ~RrgIndex() {
    int prev = 0;
    cudaGetDevice(&prev);
    cudaSetDevice(device);
    for (void* p : allocs) cudaFree(p);
    cudaSetDevice(prev);
  }
};

namespace {

RrgOpts read_opts();

// Build the device layout from the staged host model.  `corpus_rows` fills the
// reordered corpus (cluster order) given pos_of_id on the device.
template <typename CorpusFill>
void build_device_index(RrgIndex* ix, HostModel& hm, bool has_corpus, CorpusFill fill_corpus) {
  const int d = hm.d, s = hm.s, r = hm.r, L = hm.L;
  const bool quant = hm.flags & RRG_FLAG_QUANTIZED;
  if (s > 1024) raise_usage("ParameterError", "reduced dimension %d > 1024 not supported", s);
  if (r > 64) raise_usage("ParameterError", "rank %d > 64 not supported", r);
  // per-batch cluster tables (pair offsets, query buckets) live in one CTA's shared memory
  if (L > kMaxClusters) raise_usage("ParameterError", "%d clusters > %d not supported", L, kMaxClusters);
  if (hm.m >= (int64_t)1 << 31) raise_usage("ParameterError", "more than 2^31 points");
  DevIndexView& v = ix->view;
  v.opt = read_opts();
  v.metric = hm.metric; v.d = d; v.s = s; v.r = r; v.L = L;
  v.s_pad = (int)round_up(s, 16);
  v.r_pad = (int)round_up(r, 16);
  v.d_stride = (int)round_up(d, 4);
  {  // pairwise-sum leaves of a d-element row (NumPy recursion, see rrg_common.cuh)
    std::vector<int> leaves;
    std::vector<std::pair<int, int>> stack{{0, d}};
    while (!stack.empty()) {
      auto [st0, n] = stack.back();
      stack.pop_back();
      if (n <= 128) { leaves.push_back(n); continue; }
      int n2 = n / 2; n2 -= n2 % 8;
      stack.push_back({st0 + n2, n - n2});  // right after left (LIFO)
      stack.push_back({st0, n2});
    }
    bool equal = true;
    for (int n : leaves) equal = equal && n == leaves[0];
    int nl = (int)leaves.size();
    v.pw_nleaves = nl;
    v.pw_leaf_n = leaves[0];
    v.pw_perfect = equal && (nl & (nl - 1)) == 0 && leaves[0] >= 8 && nl <= 16;
  }

  // cluster order positions
  std::vector<int> cl_pos(L + 1), cl_kind(L), cl_aidx(L);
  int64_t P = 0, P_exact = 0;
  int n_rrr = 0;
  for (int l = 0; l < L; ++l) {
    HostCluster& c = hm.clusters[l];
    cl_pos[l] = (int)P;
    uint32_t held = c.owned ? c.m : 0;
    cl_kind[l] = c.exact ? kKindExact : kKindRrr;
    if (c.exact) {
      cl_aidx[l] = (int)P_exact;
      P_exact += held;
    } else {
      cl_aidx[l] = c.owned && held ? n_rrr++ : -1;
    }
    P += held;
    ix->held_sizes.push_back(held);
    if (held) ix->sizes_sorted_desc.push_back((int)held);
    ix->max_cluster = std::max<int64_t>(ix->max_cluster, held);
    if (c.exact) ix->n_exact++;
  }
  cl_pos[L] = (int)P;
  v.P = P;
  {
    double s1 = 0.0, s2 = 0.0;
    for (uint32_t hsz : ix->held_sizes) { s1 += hsz; s2 += (double)hsz * hsz; }
    ix->m_biased = s1 > 0 ? s2 / s1 : 0.0;
  }
  std::sort(ix->sizes_sorted_desc.begin(), ix->sizes_sorted_desc.end(), std::greater<int>());

  // quantized: int8 codes (+ head/scale); unquantized: f32 factors, same layouts
  // (A^T per model slot, B^T per point, exact-model rows per point; rrr.py:97-100)
  const size_t n_at = (size_t)n_rrr * r * v.s_pad, n_bt = (size_t)P * v.r_pad,
               n_xc = (size_t)P_exact * v.s_pad;
  std::vector<int8_t> at(quant ? n_at : 0, 0);
  std::vector<float> atf(quant ? 0 : n_at, 0.f), btf(quant ? 0 : n_bt, 0.f),
      xcf(quant ? 0 : n_xc, 0.f);
  std::vector<float> ahead((size_t)n_rrr * r), ascale((size_t)n_rrr * r);
  std::vector<int8_t> bt(quant ? n_bt : 0, 0), xc(quant ? n_xc : 0, 0);
  std::vector<float4> pmeta(P, make_float4(0.f, 0.f, 0.f, 0.f));
  std::vector<int64_t> pid(P);
  std::vector<int> pos_of_id(hm.m, -1);
  for (int l = 0; l < L; ++l) {
    HostCluster& c = hm.clusters[l];
    if (!c.owned || c.m == 0) continue;
    const int64_t p0 = cl_pos[l];
    const int m = (int)c.m;
    for (int p = 0; p < m; ++p) {
      int64_t id = c.ids[p];
      if (id < 0 || id >= hm.m) raise_format("cluster %d ids: id %lld out of range", l, (long long)id);
      pid[p0 + p] = id;
      pos_of_id[id] = (int)(p0 + p);
      if (hm.metric == kMetricEuclidean) pmeta[p0 + p].z = c.norms[p];
      uint32_t id32 = (uint32_t)id;
      memcpy(&pmeta[p0 + p].w, &id32, 4);
    }
    if (!quant) {
      if (c.exact) {
        const int64_t x0 = cl_aidx[l];
        for (int i = 0; i < s; ++i)
          for (int p = 0; p < m; ++p) xcf[(size_t)(x0 + p) * v.s_pad + i] = c.a_f[(size_t)i * m + p];
      } else {
        const int slot = cl_aidx[l];
        for (int i = 0; i < s; ++i)
          for (int j = 0; j < r; ++j) atf[((size_t)slot * r + j) * v.s_pad + i] = c.a_f[(size_t)i * r + j];
        for (int j = 0; j < r; ++j)
          for (int p = 0; p < m; ++p) btf[(size_t)(p0 + p) * v.r_pad + j] = c.b_f[(size_t)j * m + p];
      }
    } else if (c.exact) {
      // A: s x m (cols = points)
      const int64_t x0 = cl_aidx[l];
      for (int i = 0; i < s; ++i)
        for (int p = 0; p < m; ++p) xc[(size_t)(x0 + p) * v.s_pad + i] = c.a_vals[(size_t)i * m + p];
      for (int p = 0; p < m; ++p) { pmeta[p0 + p].x = c.a_head[p]; pmeta[p0 + p].y = c.a_scale[p]; }
    } else {
      const int slot = cl_aidx[l];
      for (int i = 0; i < s; ++i)
        for (int j = 0; j < r; ++j)
          at[((size_t)slot * r + j) * v.s_pad + i] = c.a_vals[(size_t)i * r + j];
      for (int j = 0; j < r; ++j) {
        ahead[(size_t)slot * r + j] = c.a_head[j];
        ascale[(size_t)slot * r + j] = c.a_scale[j];
      }
      for (int j = 0; j < r; ++j)
        for (int p = 0; p < m; ++p) bt[(size_t)(p0 + p) * v.r_pad + j] = c.b_vals[(size_t)j * m + p];
      for (int p = 0; p < m; ++p) { pmeta[p0 + p].x = c.b_head[p]; pmeta[p0 + p].y = c.b_scale[p]; }
    }
  }
  // centroid squared norms in f64, NumPy order: (c*c).sum(axis=1) (cluster.py:50)
  std::vector<double> cnorm(L), tmp(s);
  for (int l = 0; l < L; ++l) {
    for (int i = 0; i < s; ++i) {
      double x = hm.centroids[(size_t)l * s + i];
      tmp[i] = x * x;
    }
    cnorm[l] = pw_sum_host(tmp.data(), s);
  }
  v.W = ix->upload(hm.projection);
  v.cent = ix->upload(hm.centroids);
  v.cnorm = ix->upload(cnorm);
  v.cl_pos = ix->upload(cl_pos);
  {  // clusters by held size, largest first (ties by id): the order the sparse exact
     // pass hands out its work items, so the longest items do not form the grid's tail
    std::vector<int> ord(L);
    for (int l = 0; l < L; ++l) ord[l] = l;
    std::stable_sort(ord.begin(), ord.end(), [&](int a, int b) {
      return cl_pos[a + 1] - cl_pos[a] > cl_pos[b + 1] - cl_pos[b];
    });
    v.cl_order = ix->upload(ord);
  }
  v.cl_kind = ix->upload(cl_kind);
  v.cl_aidx = ix->upload(cl_aidx);
  v.at = ix->upload(at);
  v.ahead = ix->upload(ahead);
  v.ascale = ix->upload(ascale);
  v.bt = ix->upload(bt);
  v.xcodes = ix->upload(xc);
  {  // W^T slice planes for the tensor-core projection (s x d, rows = columns of W)
    std::vector<float> wt((size_t)s * d);
    for (int i = 0; i < d; ++i)
      for (int j = 0; j < s; ++j) wt[(size_t)j * d + i] = hm.projection[(size_t)i * s + j];
    float* dwt = ix->upload(wt);
    v.Wt = dwt;
    int8_t* planes = static_cast<int8_t*>(ix->dalloc(sliced_plane_bytes(s, d, false)));
    int* exps = static_cast<int*>(ix->dalloc((size_t)sliced_rows_pad(s, false) * 4));
    launch_slice_rows(dwt, s, d, d, false, planes, exps, 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    v.wt_planes = planes;
    v.wt_exps = exps;
    // centroid slice planes (L x s) for the tensor-core routing
    int8_t* cpl = static_cast<int8_t*>(ix->dalloc(sliced_plane_bytes(L, s, false)));
    int* cex = static_cast<int*>(ix->dalloc((size_t)sliced_rows_pad(L, false) * 4));
    launch_slice_rows(v.cent, L, s, s, false, cpl, cex, 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    v.cent_planes = cpl;
    v.cent_exps = cex;
  }
  v.quantized = quant ? 1 : 0;
  v.atf = quant ? nullptr : ix->upload(atf);
  v.btf = quant ? nullptr : ix->upload(btf);
  v.xf = quant ? nullptr : ix->upload(xcf);
  v.pmeta = ix->upload(pmeta);
  v.pid = ix->upload(pid);
  v.corpus = nullptr;
  int* d_pos = ix->upload(pos_of_id);
  v.pos_of_id = d_pos;
  v.m = hm.m;
  v.corpus_interleaved = 0;
  v.elem_perm = nullptr;
  if (has_corpus) {
    float* corp = static_cast<float*>(ix->dalloc((size_t)std::max<int64_t>(P, 1) * v.d_stride * 4));
    const int* d_perm = nullptr;
    if (v.pw_perfect && d % 2 == 0) {  // step-major interleaved rows (see DevIndexView)
      const int nl = v.pw_leaf_n, NL = v.pw_nleaves, nb = nl / 8, tail = nl % 8;
      std::vector<int> perm(d);
      for (int b = 0; b < NL; ++b)
        for (int p = 0; p < nl; ++p) {
          const int e = b * nl + p;
          perm[e] = p < 8 * nb ? (p / 8) * 8 * NL + 8 * b + (p % 8)
                               : nb * 8 * NL + b * tail + (p - 8 * nb);
        }
      d_perm = ix->upload(perm);
      v.corpus_interleaved = 1;
      v.elem_perm = d_perm;
    }
    fill_corpus(corp, d_pos, (int)v.d_stride, d_perm);
    v.corpus = corp;
  }
  v.rt_cent_tiles = nullptr; v.rt_cent_stats = nullptr; v.rt_kc = 0;
  if (s <= route_screen_max_dim() && L >= 512) {  // routing screen: centroids as fp16 tiles
    v.rt_kc = (s + 15) / 16;
    uint16_t* ct = static_cast<uint16_t*>(ix->dalloc(route_tile_bytes(L, v.rt_kc)));
    float4* cst = static_cast<float4*>(ix->dalloc((size_t)((L + 127) / 128 * 128) * 16));
    launch_f16_tiles(v.cent, L, s, s, v.rt_kc, ct, cst, 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    v.rt_cent_tiles = ct;
    v.rt_cent_stats = cst;
  }
  v.scr_plane = nullptr; v.scr_blk0 = nullptr; v.scr_mu = nullptr; v.scr_rr = nullptr;
  v.scr_rmeta = nullptr; v.scr_kc = 0;
  if (has_corpus && hm.metric == kMetricEuclidean && d <= screen_max_dim() && v.opt.screen != 0 && P > 0) {
    // re-rank screen data (rrg_screen.cu): clusters padded to 128-row blocks
    std::vector<int> blk0(L + 1, 0);
    for (int l = 0; l < L; ++l) blk0[l + 1] = blk0[l] + (int)((ix->held_sizes[l] + 127) / 128);
    v.scr_kc = (d + 63) / 64 * 4;  // K16 chunks, a multiple of 4: the plane's K64 swizzle atoms
    const size_t plane_bytes = (size_t)blk0[L] * v.scr_kc * 128 * 32;
    uint16_t* plane = static_cast<uint16_t*>(ix->dalloc(plane_bytes));
    float* mu = static_cast<float*>(ix->dalloc((size_t)L * d * 4));
    double* rr = static_cast<double*>(ix->dalloc((size_t)P * 8));
    float4* meta = static_cast<float4*>(ix->dalloc((size_t)P * 16));
    v.scr_blk0 = ix->upload(blk0);
    launch_screen_build(v, mu, plane, plane_bytes, rr, meta, 0);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaDeviceSynchronize());
    v.scr_plane = plane; v.scr_mu = mu; v.scr_rr = rr; v.scr_rmeta = meta;
  }
  ix->info.metric = hm.metric; ix->info.dim = d; ix->info.reduced_dim = s; ix->info.rank = r;
  ix->info.n_clusters = L; ix->info.n_points = hm.m; ix->info.flags = hm.flags;
  ix->info.n_exact_clusters = ix->n_exact;
  ix->info.max_cluster_size = (int)ix->max_cluster;
  ix->info.device = ix->device;
  ix->meta.metric = hm.metric; ix->meta.d = d; ix->meta.s = s; ix->meta.r = r; ix->meta.L = L;
  ix->meta.m = hm.m; ix->meta.flags = hm.flags;
}

// Streaming reader with incremental CRC32 (index.py:401,481-485) and the
// reference's section/offset error messages (index.py:410-412).
struct FileReader {
  FILE* f = nullptr;
  uint64_t off = 0, size = 0;
  uLong crc = 0;
  explicit FileReader(const char* path) {
    f = fopen(path, "rb");
    if (!f) {
      g_err = std::string("cannot open index file: ") + path;
      g_kind = "FormatError";
      throw RrgFail{RRG_E_DATA};
    }
    fseeko(f, 0, SEEK_END);
    size = (uint64_t)ftello(f);
    fseeko(f, 0, SEEK_SET);
    crc = crc32(0L, Z_NULL, 0);
  }
  ~FileReader() { if (f) fclose(f); }
  void take(void* dst, uint64_t n, const std::string& section, bool update_crc = true) {
    if (off + n > size) raise_format("truncated file: %s at offset %llu", section.c_str(), (unsigned long long)off);
    if (n && fread(dst, 1, n, f) != n) raise_format("read error: %s at offset %llu", section.c_str(), (unsigned long long)off);
    if (update_crc) {
      const unsigned char* p = static_cast<const unsigned char*>(dst);
      uint64_t left = n;
      while (left) {
        uInt chunk = (uInt)std::min<uint64_t>(left, 1u << 30);
        crc = crc32(crc, p, chunk);
        p += chunk;
        left -= chunk;
      }
    }
    off += n;
  }
  template <typename T>
  void vec(std::vector<T>& v, uint64_t count, const std::string& section) {
    v.resize(count);
    take(v.data(), count * sizeof(T), section);
  }
};

int open_impl(const char* path, int device, int32_t cb, int32_t ce, RrgIndex** out) {
  FileReader fr(path);
  unsigned char magic[8];
  fr.take(magic, 8, "magic");
  if (memcmp(magic, "RRRANN01", 8) != 0)
    raise_format("bad magic %s; expected b'RRRANN01'", py_bytes_repr(magic, 8).c_str());
  unsigned char hdr[29];  // struct "<BIIIIQI"
  fr.take(hdr, 29, "header");
  HostModel hm;
  uint8_t mc = hdr[0];
  uint32_t d, s, r, L, flags;
  uint64_t m;
  memcpy(&d, hdr + 1, 4); memcpy(&s, hdr + 5, 4); memcpy(&r, hdr + 9, 4); memcpy(&L, hdr + 13, 4);
  memcpy(&m, hdr + 17, 8); memcpy(&flags, hdr + 25, 4);
  if (mc > 2) raise_format("unknown metric code %u", (unsigned)mc);
  hm.metric = mc; hm.d = (int)d; hm.s = (int)s; hm.r = (int)r; hm.L = (int)L; hm.m = (int64_t)m;
  hm.flags = flags;
  const bool quantized = flags & RRG_FLAG_QUANTIZED;
  const bool has_corpus = flags & RRG_FLAG_CORPUS;
  const bool exact_ivf = flags & RRG_FLAG_EXACT_IVF;
  if (ce < 0) ce = (int32_t)L;
  if (cb < 0 || cb > ce || (int64_t)ce > (int64_t)L)
    raise_usage("ParameterError", "shard cluster range [%d, %d) outside [0, %lld]", cb, ce, (long long)L);
  fr.vec(hm.projection, (uint64_t)d * s, "projection");
  fr.vec(hm.centroids, (uint64_t)L * s, "centroids");
  hm.clusters.resize(L);
  uint64_t total = 0;
  for (uint32_t l = 0; l < L; ++l) {
    HostCluster& c = hm.clusters[l];
    std::string sec = "cluster " + std::to_string(l);
    uint32_t ml;
    fr.take(&ml, 4, sec + " size");
    c.m = ml;
    c.owned = (int32_t)l >= cb && (int32_t)l < ce;
    std::vector<uint64_t> ids;
    fr.vec(ids, ml, sec + " ids");
    c.ids.assign(ids.begin(), ids.end());
    c.exact = exact_ivf || ml < r;
    const uint64_t acols = c.exact ? ml : r;
    auto read_factor = [&](uint64_t rows, uint64_t cols, const std::string& fsec,
                           std::vector<float>& head, std::vector<float>& scale,
                           std::vector<int8_t>& vals, std::vector<float>& fvals) {
      if (quantized) {
        fr.vec(head, cols, fsec + " head row");
        fr.vec(scale, cols, fsec + " scales");
        fr.vec(vals, rows * cols, fsec + " values");
      } else {
        fr.vec(fvals, rows * cols, fsec);  // f32 rows x cols (index.py:500-502)
      }
    };
    read_factor(s, acols, sec + " factor A", c.a_head, c.a_scale, c.a_vals, c.a_f);
    if (!c.exact) read_factor(r, ml, sec + " factor B", c.b_head, c.b_scale, c.b_vals, c.b_f);
    if (mc == kMetricEuclidean) fr.vec(c.norms, ml, sec + " norms");
    if (!c.owned) {  // keep only metadata for routing; release payloads
      std::vector<float>().swap(c.a_head); std::vector<float>().swap(c.a_scale);
      std::vector<int8_t>().swap(c.a_vals); std::vector<float>().swap(c.b_head);
      std::vector<float>().swap(c.b_scale); std::vector<int8_t>().swap(c.b_vals);
      std::vector<float>().swap(c.norms);
      std::vector<float>().swap(c.a_f); std::vector<float>().swap(c.b_f);
    }
    total += ml;
  }
  if (total != m)
    raise_format("cluster records cover %llu points, header says %llu", (unsigned long long)total,
                 (unsigned long long)m);
  CUDA_TRY(cudaSetDevice(device));
  std::unique_ptr<RrgIndex> ix(new RrgIndex());
  ix->device = device;
  bool corpus_done = false;
  auto fill = [&](float* dst, const int* d_pos, int d_stride, const int* perm) {
    // stream the corpus (original id order) through pinned chunks, scatter into cluster order
    const uint64_t row_bytes = (uint64_t)d * 4;
    const uint64_t rows_per_chunk = std::max<uint64_t>(1, (64ull << 20) / std::max<uint64_t>(row_bytes, 1));
    float* pinned[2] = {nullptr, nullptr};
    float* staging[2] = {nullptr, nullptr};
    cudaEvent_t ev[2];
    cudaStream_t st;
    CUDA_TRY(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(cudaMallocHost(&pinned[b], rows_per_chunk * row_bytes));
      CUDA_TRY(cudaMalloc(&staging[b], rows_per_chunk * row_bytes));
      CUDA_TRY(cudaEventCreate(&ev[b]));
    }
    uint64_t done = 0;
    int b = 0;
    try {
      while (done < m) {
        uint64_t n = std::min<uint64_t>(rows_per_chunk, m - done);
        CUDA_TRY(cudaEventSynchronize(ev[b]));
        if (done == 0 && fr.off + m * row_bytes > fr.size)
          raise_format("truncated file: corpus at offset %llu", (unsigned long long)fr.off);
        fr.take(pinned[b], n * row_bytes, "corpus");
        CUDA_TRY(cudaMemcpyAsync(staging[b], pinned[b], n * row_bytes, cudaMemcpyHostToDevice, st));
        launch_scatter_rows(staging[b], (int64_t)n, (int)d, d_stride, d_pos, (int64_t)done, perm,
                            dst, st);
        CUDA_TRY(cudaGetLastError());
        CUDA_TRY(cudaEventRecord(ev[b], st));
        done += n;
        b ^= 1;
      }
      CUDA_TRY(cudaStreamSynchronize(st));
    } catch (...) {
      cudaStreamSynchronize(st);
      for (int q = 0; q < 2; ++q) { cudaFreeHost(pinned[q]); cudaFree(staging[q]); cudaEventDestroy(ev[q]); }
      cudaStreamDestroy(st);
      throw;
    }
    for (int q = 0; q < 2; ++q) { cudaFreeHost(pinned[q]); cudaFree(staging[q]); cudaEventDestroy(ev[q]); }
    cudaStreamDestroy(st);
    corpus_done = true;
  };
  build_device_index(ix.get(), hm, has_corpus, fill);
  (void)corpus_done;
  (void)quantized;
  uint64_t crc_off = fr.off;
  uint32_t stored;
  uLong actual = fr.crc;
  fr.take(&stored, 4, "crc32", false);
  if ((uint32_t)actual != stored)
    raise_format("crc mismatch at offset %llu: %#x != %#x", (unsigned long long)crc_off, stored,
                 (unsigned)actual);
  if (fr.off != fr.size)
    raise_format("unknown trailing section at offset %llu: %llu extra bytes",
                 (unsigned long long)fr.off, (unsigned long long)(fr.size - fr.off));
  *out = ix.release();
  return RRG_OK;
}

int create_impl(const RrgIndexDesc* dsc, int device, int32_t cb, int32_t ce, RrgIndex** out) {
  CUDA_TRY(cudaSetDevice(device));
  HostModel hm;
  hm.metric = dsc->metric; hm.d = dsc->dim; hm.s = dsc->reduced_dim; hm.r = dsc->rank;
  hm.L = dsc->n_clusters; hm.m = dsc->n_points; hm.flags = dsc->flags;
  if (hm.metric < 0 || hm.metric > 2) raise_usage("ParameterError", "unknown metric code %d", hm.metric);
  const int d = hm.d, s = hm.s, r = hm.r, L = hm.L;
  hm.projection.assign(dsc->projection, dsc->projection + (size_t)d * s);
  hm.centroids.assign(dsc->centroids, dsc->centroids + (size_t)L * s);
  hm.clusters.resize(L);
  const bool exact_ivf = hm.flags & RRG_FLAG_EXACT_IVF;
  const bool quant = hm.flags & RRG_FLAG_QUANTIZED;
  if (ce < 0) ce = L;
  if (cb < 0 || cb > ce || ce > L)
    raise_usage("ParameterError", "shard cluster range [%d, %d) outside [0, %d]", cb, ce, L);
  if (!quant && (!dsc->a_values_f32 || !dsc->b_values_f32))
    raise_usage("ParameterError", "unquantized index description needs a_values_f32/b_values_f32");
  int64_t po = 0, ao = 0, aoff = 0, bo = 0, boff = 0;
  for (int l = 0; l < L; ++l) {
    HostCluster& c = hm.clusters[l];
    c.m = dsc->cluster_sizes[l];
    c.exact = exact_ivf || (int)c.m < r;
    c.owned = l >= cb && l < ce;  // a shard keeps only the payloads of its own clusters
    const int64_t m = c.m;
    c.ids.assign(dsc->point_ids + po, dsc->point_ids + po + m);
    if (dsc->norms && c.owned) c.norms.assign(dsc->norms + po, dsc->norms + po + m);
    const int64_t acols = c.exact ? m : r;
    if (!c.owned) {
    } else if (quant) {
      c.a_head.assign(dsc->a_head + ao, dsc->a_head + ao + acols);
      c.a_scale.assign(dsc->a_scale + ao, dsc->a_scale + ao + acols);
      c.a_vals.assign(dsc->a_values + aoff, dsc->a_values + aoff + (size_t)s * acols);
    } else {
      c.a_f.assign(dsc->a_values_f32 + aoff, dsc->a_values_f32 + aoff + (size_t)s * acols);
    }
    ao += acols;
    aoff += (int64_t)s * acols;
    if (!c.exact) {
      if (!c.owned) {
      } else if (quant) {
        c.b_head.assign(dsc->b_head + bo, dsc->b_head + bo + m);
        c.b_scale.assign(dsc->b_scale + bo, dsc->b_scale + bo + m);
        c.b_vals.assign(dsc->b_values + boff, dsc->b_values + boff + (size_t)r * m);
      } else {
        c.b_f.assign(dsc->b_values_f32 + boff, dsc->b_values_f32 + boff + (size_t)r * m);
      }
      bo += m;
      boff += (int64_t)r * m;
    }
    po += m;
  }
  if (po != hm.m) raise_usage("ShapeError", "cluster sizes cover %lld points, n_points is %lld",
                             (long long)po, (long long)hm.m);
  std::unique_ptr<RrgIndex> ix(new RrgIndex());
  ix->device = device;
  const bool has_corpus = dsc->corpus != nullptr;
  auto fill = [&](float* dst, const int* d_pos, int d_stride, const int* perm) {
    const uint64_t row_bytes = (uint64_t)d * 4;
    const uint64_t rows_per_chunk = std::max<uint64_t>(1, (64ull << 20) / std::max<uint64_t>(row_bytes, 1));
    float* staging = nullptr;
    CUDA_TRY(cudaMalloc(&staging, rows_per_chunk * row_bytes));
    for (uint64_t done = 0; done < (uint64_t)hm.m;) {
      uint64_t n = std::min<uint64_t>(rows_per_chunk, hm.m - done);
      // host or device corpus (unified addressing): a GPU-built index hands its corpus over
      // without a host copy
      CUDA_TRY(cudaMemcpy(staging, dsc->corpus + done * d, n * row_bytes, cudaMemcpyDefault));
      launch_scatter_rows(staging, (int64_t)n, d, d_stride, d_pos, (int64_t)done, perm, dst, 0);
      CUDA_TRY(cudaGetLastError());
      done += n;
    }
    CUDA_TRY(cudaDeviceSynchronize());
    cudaFree(staging);
  };
  if (has_corpus) hm.flags |= RRG_FLAG_CORPUS; else hm.flags &= ~RRG_FLAG_CORPUS;
  build_device_index(ix.get(), hm, has_corpus, fill);
  *out = ix.release();
  return RRG_OK;
}

// ------------------------------------------------------------------ search

// Projection / routing GEMM engines: the int8 tensor cores (k_gemm_sliced: f64-exact
// 7-bit slices, tcgen05 + TMEM) or the FP64 DMMA GEMM (k_gemm_dmma).  Measured on C2
// (10k queries): projection 0.162 ms sliced vs 0.175 ms DMMA, routing 0.220 ms sliced
// vs 0.203 ms DMMA -- so the defaults are sliced projection, DMMA routing.
// RRG_PROJ / RRG_ROUTE = sliced|dmma choose each; RRG_GEMM = sliced|dmma sets both.
// Every switch is read here, once per index (RrgOpts), not per search call.
RrgOpts read_opts() {
  auto env = [](const char* v) -> const char* { return getenv(v); };
  auto gemm = [&](const char* var, bool dflt) {
    const char* e = env("RRG_GEMM");
    if (!e) e = env(var);
    return e ? (strcmp(e, "sliced") == 0 ? 1 : 0) : (dflt ? 1 : 0);
  };
  auto flag = [&](const char* var, int dflt) {
    const char* e = env(var);
    return e ? atoi(e) : dflt;
  };
  RrgOpts o{};
  o.proj_sliced = gemm("RRG_PROJ", true);
  o.route_sliced = gemm("RRG_ROUTE", false);
  o.route_fused = flag("RRG_ROUTE_FUSED", 1) != 0;
  o.gemm_bk = flag("RRG_GEMM_BK", 8) == 16 ? 16 : 8;
  {
    const char* e = env("RRG_SCORE_MODE");
    o.score_query = e && strcmp(e, "query") == 0;
  }
  {
    const char* e = env("RRG_RERANK");
    o.rerank = !e ? 0 : strcmp(e, "cluster") == 0 ? 1 : strcmp(e, "query") == 0 ? 2
             : strcmp(e, "regs") == 0 ? 3 : strcmp(e, "tma") == 0 ? 4 : 0;
  }
  o.rr_skip = env("RRG_RR_SKIP") ? (flag("RRG_RR_SKIP", 0) != 0) : -1;
  o.rr_async = flag("RRG_RR_ASYNC", 0) == 1;
  o.warp_select = env("RRG_WARP_SELECT") ? (flag("RRG_WARP_SELECT", 0) != 0) : -1;
  o.host_pieces = std::max(0, std::min(8, flag("RRG_HOST_PIECES", 0)));
  o.graph = flag("RRG_GRAPH", 1) != 0;
  o.screen = env("RRG_SCREEN") ? (flag("RRG_SCREEN", 0) != 0) : -1;
  o.score_stage_a = flag("RRG_SCORE_STAGE_A", 1);
  o.rr_order = flag("RRG_RR_ORDER", 1);
  o.score_order = flag("RRG_SCORE_ORDER", 1);
  o.route_screen = flag("RRG_ROUTE_SCREEN", 1);  // 0 off, 1 w = 1, 2 any w <= kRtMaxW
  o.screen_diag = flag("RRG_SCREEN_DIAG", 0);
  o.score_tc = env("RRG_SCORE_TC") ? (flag("RRG_SCORE_TC", 0) != 0) : -1;
  o.sparse_variant = flag("RRG_SPARSE_VARIANT", 1);
  o.screen_stages = flag("RRG_SCREEN_STAGES", 0);
  return o;
}
// up to this many queries the projection / routing run as warp-per-output GEMVs
// (a GEMM tile of one row is ~10 dependent K-steps: 30-37 us at C2 batch 1)
constexpr int kSmallBatch = 32;

// Query sub-range bounds of the front stages (and the host entry's copy pieces):
// multiples of the sliced GEMM's 128-row blocks, so a piece's slice planes are a
// contiguous run of blocks.
int64_t piece_bound(int64_t n, int j, int nsub) {
  if (j >= nsub) return n;
  return (n * j / nsub) / 128 * 128;
}

// Routing dissimilarities of n projected queries: sliced tensor-core GEMM (xp slices in
// qpl/qex) or the DMMA GEMM.
void route_dist(const DevIndexView& v, const float* xp, int n, const double* pp, double* diss,
                int8_t* qpl, int* qex, cudaStream_t st) {
  if (n <= kSmallBatch) {
    launch_route_dist_small(xp, v.cent, n, v.L, v.s, v.metric, pp, v.cnorm, diss, st);
  } else if (qpl && v.opt.route_sliced) {
    launch_slice_rows(xp, n, v.s, v.s, true, qpl, qex, st);
    launch_gemm_sliced(qpl, qex, n, v.cent_planes, v.cent_exps, v.L, v.s,
                       v.metric == kMetricEuclidean ? EPI_L2 : EPI_NEGIP, nullptr, diss, v.L, pp,
                       v.cnorm, st);
  } else {
    launch_route_dist(xp, v.cent, n, v.L, v.s, v.metric, pp, v.cnorm, diss, v.opt.gemm_bk, st);
  }
}

struct Plan {
  int64_t qc;      // queries per chunk
  bool sliced_proj;
  size_t off_qpl, off_qex;
  int take_cap;
  int smem_cap;
  int64_t gcap;    // global overflow capacity per query (0 if none)
  size_t off_xp, off_qc, off_qs, off_qh, off_xx, off_pp, off_diss, off_sel, off_cpos, off_cn,
      off_gk, off_gp, off_prim, off_order, total;
  // cluster-major scoring (score_mode == 1)
  int score_mode;
  int kcap;
  size_t off_qoff, off_ncand, off_pairoff, off_itemoff, off_pairs, off_kbase, off_keys, off_ctr;
  // cluster-major re-rank (rr_mode == 1)
  int rr_mode;
  int mwords;
  size_t off_cidx, off_marks, marks_bytes, off_rritem;
  // re-rank screen (rr_mode == 1, euclidean)
  size_t off_xint;
  bool screen;
  int n_groups_max;
  size_t off_ub, off_lb, off_scritem, off_grpoff, off_grec;
};

Plan make_plan(const RrgIndex* ix, int64_t nq, int k, int w, int t, int rerank,
               bool exact_take = false) {
  Plan p{};
  const DevIndexView& v = ix->view;
  const int64_t L = v.L;
  // query chunk: the f64 routing rows (Q x L x 8 B) stay within 1 GB.  Chunks cost
  // row re-reads in the cluster-major re-rank (each chunk's query groups fetch their
  // rows again): C4 (L = 8192) at 256 MB ran 3 chunks of 4096 queries, 5.0 ms of
  // re-rank for 10k queries
  int64_t qc = std::max<int64_t>(256, (1ll << 30) / (L * 8));
  qc = std::min<int64_t>(qc, 16384);
  // max candidates of any query: sum of the w largest held clusters
  int64_t nmax = 0;
  for (int i = 0; i < (int)ix->sizes_sorted_desc.size() && i < w; ++i) nmax += ix->sizes_sorted_desc[i];
  // the chunk's key array (and its membership bits) is indexed with int32 offsets:
  // keep a chunk's candidates below 2^29 (2 GB of keys)
  if (nmax > 0) qc = std::min<int64_t>(qc, std::max<int64_t>(1, ((int64_t)1 << 29) / nmax));
  p.qc = std::max<int64_t>(1, std::min<int64_t>(nq, qc));
  p.take_cap = rerank ? t : k;
  if (!exact_take) p.take_cap = (int)std::min<int64_t>(p.take_cap, std::max<int64_t>(nmax, 1));
  // dynamic smem per scoring CTA: with ~40 KB static this keeps 2 CTAs (2 x 512
  // threads) resident per SM; queries with more candidates spill to global
  const size_t budget = 64 * 1024;
  int64_t np2 = 1;
  while (np2 < k) np2 <<= 1;
  int64_t fixed = (int64_t)p.take_cap * 4 + 64 + np2 * 8;
  int64_t cap = ((int64_t)budget - fixed) / 8;
  cap = std::max<int64_t>(cap, 256);
  p.smem_cap = (int)std::min<int64_t>(cap, std::max<int64_t>(nmax, 1));
  p.gcap = nmax > p.smem_cap ? nmax : 0;
  size_t o = 0;
  auto carve = [&](size_t bytes) { size_t r = o; o += (bytes + 255) / 256 * 256; return r; };
  const int64_t Q = p.qc;
  p.off_xp = carve(Q * v.s * 4);
  p.off_qc = carve(Q * v.s_pad);
  p.off_qs = carve(Q * 4);
  p.off_qh = carve(Q * 4);
  p.off_xx = carve(Q * 4);
  p.off_pp = carve(Q * 8);
  p.off_diss = carve(Q * L * 8);
  p.off_sel = carve(Q * (int64_t)w * 4);
  p.off_cpos = carve(Q * (int64_t)p.take_cap * 4);
  p.off_cn = carve(Q * 4);
  p.off_gk = carve(Q * p.gcap * 4);
  p.off_gp = carve(Q * p.gcap * 4);
  p.off_prim = carve(Q * 4);
  p.off_order = carve(Q * 4);
  p.sliced_proj = v.opt.proj_sliced || v.opt.route_sliced;  // slice-plane workspace needed
  if (p.sliced_proj) {
    p.off_qpl = carve(sliced_plane_bytes((int)Q, v.d, true));
    p.off_qex = carve((size_t)sliced_rows_pad((int)Q, true) * 4);
  }
  // scoring strategy: cluster-major (bucketed pairs, factors staged once per
  // cluster) unless RRG_SCORE_MODE=query selects the fused query-major kernel
  // the fused query-major kernel scores int8 factors only
  p.score_mode = (v.opt.score_query && v.quantized) ? 0 : 1;
  if (p.score_mode == 1) {
    p.kcap = (int)std::min<int64_t>(std::max<int64_t>(nmax, 1), 24 * 1024);
    p.off_qoff = carve(Q * (int64_t)(w + 1) * 4);
    p.off_ncand = carve(Q * 4);
    p.off_pairoff = carve((L + 1) * 4);
    p.off_itemoff = carve((L + 1) * 4);
    p.off_pairs = carve(Q * (int64_t)w * 4);
    p.off_kbase = carve((Q + 1) * 4);
    p.off_keys = carve(Q * std::max<int64_t>(nmax, 1) * 4);
    p.off_ctr = carve(16);
  }
  p.screen = false;
  // re-rank strategy: cluster-major (rows of a cluster shared by its queries) when
  // the scoring is cluster-major and the row plan fits k_rerank_cluster;
  // RRG_RERANK=query|regs|tma forces a per-query kernel
  {
    // measured on C2 (w=1, t=800): cluster-major 1.41 ms (+0.14 ms final top-k) vs
    // per-query k_rerank_tree 1.66 ms; RRG_RERANK=query|regs|tma selects a per-query kernel
    const bool want = v.opt.rerank <= 1;  // query / regs / tma force a per-query kernel
    // the cluster-major re-rank streams every row of a probed cluster for its query
    // group: worth it while a query keeps a large share of its probed rows (C2, w=1:
    // t / (w m) = 0.82); with many probes per query (C5, w=8: 0.10) the rows a query
    // keeps are sparse and the per-query kernel is 3-10x faster (measured)
    // The share is taken with cluster sizes as a random query sees them (the
    // size-biased mean sum m_l^2 / sum m_l: C2 1,037, C3 613, C4 1,622 against a
    // plain mean of 1,221).  That is what moves C4 w = 2 to the per-query kernel
    // (800 < 0.3 * 2 * 1,622; measured 5.72 vs 7.46 ms per 10k), while C4 w = 1 stays
    // cluster-major (800 >= 0.3 * 1,622).
    const double mbar = ix->m_biased;
    // small batches: the cluster-major items ((cluster, row chunk) per probe) spread one
    // query's rows over many CTAs, where the per-query kernel has one CTA per query
    const bool small = p.qc * w < 2 * 148;
    const bool dense = (double)t >= 0.3 * w * mbar || small ||
                       v.opt.rerank == 1;
    p.rr_mode = (want && dense && p.score_mode == 1 && rerank && !exact_take &&
                 cluster_rerank_ok(v, ix->max_cluster)) ? 1 : 0;
  }
  if (p.rr_mode == 1) {
    p.mwords = (int)((ix->max_cluster + 31) / 32) + 1;
    p.off_cidx = carve(Q * (int64_t)p.take_cap * 4);
    p.marks_bytes = ((size_t)Q * std::max<int64_t>(nmax, 1) / 32 + 2) * 4;
    p.off_marks = carve(p.marks_bytes);
    p.off_rritem = carve((L + 1) * 4);
    // tensor-core screen of the re-rank (rrg_screen.cu): worth it once most of a query's
    // t candidates cannot reach its top k (t >= 2k) and a cluster's rows serve several
    // queries -- the screen streams every row of a probed cluster (fp16) once per query
    // group, the exact pass only the survivors' f32 rows; with ~1 query per cluster
    // (C4: 10k queries over 8192 clusters) the dense exact pass reads fewer bytes.
    // RRG_SCREEN=1 forces, 0 disables.
    const double per_cluster = v.L > 0 ? (double)nq * w / v.L : 0.0;
    p.screen = v.scr_plane != nullptr && v.metric == kMetricEuclidean &&
               (v.opt.screen == 1 || (v.opt.screen < 0 && t >= 2 * k && per_cluster >= 4.0));
    p.off_xint = carve(Q * (int64_t)v.d_stride * 4);
    if (p.screen) {
      p.off_ub = carve(Q * std::max<int64_t>(nmax, 1) * 4);
      p.off_lb = carve(Q * std::max<int64_t>(nmax, 1) * 4);
      p.off_scritem = carve((L + 1) * 4);
      p.off_grpoff = carve((L + 1) * 4);
      const int64_t pairs = Q * (int64_t)w;
      p.n_groups_max = (int)std::max<int64_t>(1, (pairs + 15 * std::min<int64_t>(L, pairs)) / kRrQ);
      p.off_grec = carve((size_t)p.n_groups_max * screen_group_bytes(v.scr_kc));
    }
  }
  p.total = o;
  return p;
}

void validate_search(const RrgIndex* ix, int32_t dim, int32_t k, int32_t w, int32_t t,
                     int32_t rerank) {
  // QueryParams.validate (index.py:92-100), then index.py:290-295
  const int L = ix->meta.L;
  if (k < 1) raise_usage("ParameterError", "k must be >= 1");
  if (!(1 <= w && w <= L)) raise_usage("ParameterError", "w=%d out of range [1, %d]", w, L);
  if (t < 1) raise_usage("ParameterError", "t must be >= 1");
  if (rerank && k > t) raise_usage("ParameterError", "k=%d must be <= t=%d when re-ranking", k, t);
  if (dim != ix->meta.d)
    raise_usage("ShapeError", "query dimension %d != index dimension %d", dim, ix->meta.d);
  if (rerank && ix->view.corpus == nullptr)
    raise_usage("ParameterError", "index was built without the corpus; re-ranking unavailable");
}

// Sharded phase 1 outputs: the shard's local top-t (key, corpus id) per query.
struct Phase1Out {
  uint32_t* keys;
  uint32_t* ids;
  int32_t* count;
};

// front: per-query outputs of projection .. routing.  With `fin` the search skips
// those stages and takes them from the caller (data-parallel front stages of the
// sharded search: each rank computes a slice, the slices are all-gathered); with
// `fout` it stops after them and hands them out.
void search_impl(RrgIndex* ix, const float* queries, int64_t nq, int32_t k, int32_t w, int32_t t,
                 int32_t rerank, int64_t* ids, float* scores, int32_t* count, void* ws,
                 size_t ws_bytes, cudaStream_t st, const Phase1Out* ph1 = nullptr,
                 int* nonfinite = nullptr,
                 const std::vector<cudaEvent_t>* in_ready = nullptr,
                 const RrgFront* fin = nullptr, const RrgFront* fout = nullptr) {
  Plan p = make_plan(ix, nq, k, w, t, rerank, ph1 != nullptr);
  {  // shared-memory budgets of the per-query CTAs (static parts bounded by 48 KB)
    const size_t lim = kMaxSmemPerCta - 48 * 1024;
    if ((p.score_mode == 0 ? score_select_smem(p.smem_cap, p.take_cap, k)
                           : select_topt_smem(w, p.take_cap, k, p.kcap)) > lim ||
        (rerank && rerank_smem(ix->view.d_stride, p.take_cap, k, rerank_uses_tree(ix->view)) > lim))
      raise_usage("ParameterError", "t=%d / k=%d exceed the device search limits", t, k);
  }
  if (ws_bytes < p.total)
    raise_usage("ParameterError", "workspace too small: %zu < %zu bytes", ws_bytes, p.total);
  char* base = static_cast<char*>(ws);
  const DevIndexView& v = ix->view;
  float* xp = reinterpret_cast<float*>(base + p.off_xp);
  int8_t* qcodes = reinterpret_cast<int8_t*>(base + p.off_qc);
  float* qscale = reinterpret_cast<float*>(base + p.off_qs);
  float* qhead = reinterpret_cast<float*>(base + p.off_qh);
  float* xx = reinterpret_cast<float*>(base + p.off_xx);
  double* pp = reinterpret_cast<double*>(base + p.off_pp);
  double* diss = reinterpret_cast<double*>(base + p.off_diss);
  int* sel = reinterpret_cast<int*>(base + p.off_sel);
  int* cpos = reinterpret_cast<int*>(base + p.off_cpos);
  int* cn = reinterpret_cast<int*>(base + p.off_cn);
  uint32_t* gk = reinterpret_cast<uint32_t*>(base + p.off_gk);
  int* gp = reinterpret_cast<int*>(base + p.off_gp);
  int* prim = reinterpret_cast<int*>(base + p.off_prim);
  int* order_buf = reinterpret_cast<int*>(base + p.off_order);
  path_begin(RRG_PATH_SEARCH, st);
  for (int64_t q0 = 0; q0 < nq; q0 += p.qc) {
    const int n = (int)std::min<int64_t>(p.qc, nq - q0);
    const float* x = queries + q0 * v.d;
    // front stages (projection .. routing) are independent per query: with host input
    // events they run per arriving sub-range, overlapping the remaining H2D copies
    const int nsub = (in_ready && n == nq) ? (int)in_ready->size() : 1;
    if (fin) {  // front outputs supplied: copy this chunk's rows into the workspace
      auto cp = [&](void* dst, const void* src, size_t row_bytes) {
        CUDA_TRY(cudaMemcpyAsync(dst, static_cast<const char*>(src) + q0 * row_bytes, n * row_bytes,
                                 cudaMemcpyDeviceToDevice, st));
      };
      cp(xp, fin->xp, (size_t)v.s * 4);
      cp(qcodes, fin->qcodes, (size_t)v.s_pad);
      cp(qscale, fin->qscale, 4);
      cp(qhead, fin->qhead, 4);
      cp(pp, fin->pp, 8);
      cp(xx, fin->xx, 4);
      cp(sel, fin->sel, (size_t)w * 4);
      cp(prim, fin->prim, 4);
    }
    for (int j = 0; j < (fin ? 0 : nsub); ++j) {
      const int s0 = (int)piece_bound(n, j, nsub), s1 = (int)piece_bound(n, j + 1, nsub);
      const int ns = s1 - s0;
      if (ns <= 0) continue;
      if (in_ready)  // copies are in order on one stream: the last event covers them all
        CUDA_TRY(cudaStreamWaitEvent(st, (*in_ready)[nsub > 1 ? j : in_ready->size() - 1], 0));
      const float* xs = x + (int64_t)s0 * v.d;
      float* xps = xp + (int64_t)s0 * v.s;
      // this piece's run of 128-row slice-plane blocks (s0 is a multiple of 128)
      int8_t* qpl_d = p.sliced_proj ? reinterpret_cast<int8_t*>(base + p.off_qpl) +
                                          (s0 / 128) * sliced_block_bytes(v.d, true) : nullptr;
      int8_t* qpl_s = p.sliced_proj ? reinterpret_cast<int8_t*>(base + p.off_qpl) +
                                          (s0 / 128) * sliced_block_bytes(v.s, true) : nullptr;
      int* qex = p.sliced_proj ? reinterpret_cast<int*>(base + p.off_qex) + s0 : nullptr;
      if (ns <= kSmallBatch) {
        staged(0, st, [&] { launch_project_small(xs, v.Wt, ns, v.d, v.s, xps, st); });
      } else if (v.opt.proj_sliced) {
        int8_t* qpl = qpl_d;
        staged(0, st, [&] { launch_slice_rows(xs, ns, v.d, v.d, true, qpl, qex, st); });
        staged(0, st, [&] {
          launch_gemm_sliced(qpl, qex, ns, v.wt_planes, v.wt_exps, v.s, v.d, EPI_PROJ, xps, nullptr,
                             v.s, nullptr, nullptr, st);
        });
      } else {
        staged(0, st, [&] { launch_project(xs, v.W, ns, v.d, v.s, xps, v.opt.gemm_bk, st); });
      }
      staged(1, st, [&] {
        launch_prep(xps, xs, ns, v.s, v.s_pad, v.d, qcodes + (int64_t)s0 * v.s_pad, qscale + s0,
                    qhead + s0, pp + s0, xx + s0, st, nonfinite);
      });
      auto al256 = [](size_t b) { return (b + 255) / 256 * 256; };
      const size_t rt_need = v.rt_cent_tiles == nullptr ? 0 :
          al256(route_tile_bytes(ns, v.rt_kc)) + al256((size_t)(ns + 127) / 128 * 128 * 16) +
          al256((size_t)ns * 4) + al256(route_cnt_bytes(ns, v.L)) + al256(route_list_bytes(ns, v.L));
      // (w = 1 only: at C3, w = 4, the per-thread candidate lists cost more than the f64
      // GEMM they replace -- 0.43 vs 0.25 ms)
      if (ns > kSmallBatch && (w == 1 || (v.opt.route_screen == 2 && w <= kRtMaxW)) && v.rt_cent_tiles &&
          v.opt.route_screen &&
          rt_need <= (size_t)ns * v.L * 8) {
        // bounds on the fp16 tensor cores, f64 recheck of the few candidates that can be
        // among the w nearest (rrg_route_screen.cu); scratch inside this piece's rows of
        // the routing buffer (>= 4 KB per query for L >= 512; this needs ~2.8 KB + the tile)
        char* rb = reinterpret_cast<char*>(diss + (int64_t)s0 * v.L);
        auto al = [](size_t b) { return (b + 255) / 256 * 256; };
        RouteScreenHost rh{};
        rh.ix = v; rh.xp = xps; rh.pp = pp + s0; rh.w = w;
        size_t o = 0;
        rh.qt = reinterpret_cast<uint16_t*>(rb + o); o += al(route_tile_bytes(ns, v.rt_kc));
        rh.qs = reinterpret_cast<float4*>(rb + o); o += al((size_t)(ns + 127) / 128 * 128 * 16);
        rh.T = reinterpret_cast<uint32_t*>(rb + o); o += al((size_t)ns * 4);
        rh.cnt = reinterpret_cast<int*>(rb + o); o += al(route_cnt_bytes(ns, v.L));
        rh.list = reinterpret_cast<int2*>(rb + o); o += al(route_list_bytes(ns, v.L));
        rh.sel = sel + (int64_t)s0 * w; rh.primary = prim + s0;
        staged(2, st, [&] { launch_route_screen(rh, ns, st); });
      } else if (w == 1 && ns > kSmallBatch && v.opt.route_fused) {
        // nearest cluster straight from the GEMM: per (query, 64-centroid tile) minima
        const int nt = route_nearest_tiles(v.L);
        double* part_v = diss + (int64_t)s0 * nt;
        int* part_i = reinterpret_cast<int*>(diss + p.qc * nt) + (int64_t)s0 * nt;
        if (v.opt.route_sliced && qpl_s) {
          staged(2, st, [&] { launch_slice_rows(xps, ns, v.s, v.s, true, qpl_s, qex, st); });
          staged(2, st, [&] {
            launch_gemm_sliced(qpl_s, qex, ns, v.cent_planes, v.cent_exps, v.L, v.s,
                               v.metric == kMetricEuclidean ? EPI_L2_ARGMIN : EPI_NEGIP_ARGMIN,
                               nullptr, part_v, nt, pp + s0, v.cnorm, st, part_i);
          });
        } else {
          staged(2, st, [&] {
            launch_route_nearest_fused(xps, v.cent, ns, v.L, v.s, v.metric, pp + s0, v.cnorm, part_v,
                                       part_i, st);
          });
        }
        staged(3, st, [&] {
          launch_route_nearest_reduce(part_v, part_i, ns, v.L, sel + s0, prim + s0, st);
        });
      } else if (w > 1 && w <= 8 && ns > kSmallBatch && v.opt.route_fused && v.metric == kMetricEuclidean) {
        // the w nearest straight from the GEMM: per (query, 64-centroid tile) sorted top-4 / -8
        // (C3, w = 4: the 164 MB f64 distance rows and their CTA-per-query select, 0.25 ms)
        const int nt = route_nearest_tiles(v.L), tw = w <= 4 ? 4 : 8;
        double* part_v = diss + (int64_t)s0 * nt * tw;
        int* part_i = reinterpret_cast<int*>(diss + (int64_t)p.qc * nt * tw) + (int64_t)s0 * nt * tw;
        staged(2, st, [&] {
          launch_route_topw_fused(xps, v.cent, ns, v.L, v.s, w, pp + s0, v.cnorm, part_v, part_i, st);
        });
        staged(3, st, [&] {
          launch_route_topw_reduce(part_v, part_i, ns, v.L, w, sel + (int64_t)s0 * w, prim + s0, st);
        });
      } else {
        staged(2, st, [&] {
          route_dist(v, xps, ns, pp + s0, diss + (int64_t)s0 * v.L, qpl_s, qex, st);
        });
        staged(3, st, [&] {
          launch_route_select(diss + (int64_t)s0 * v.L, ns, v.L, w, sel + (int64_t)s0 * w, prim + s0, st);
        });
      }
    }
    if (fout) {  // front only: hand this chunk's rows out
      auto cp = [&](void* dst, const void* src, size_t row_bytes) {
        CUDA_TRY(cudaMemcpyAsync(static_cast<char*>(dst) + q0 * row_bytes, src, n * row_bytes,
                                 cudaMemcpyDeviceToDevice, st));
      };
      cp(fout->xp, xp, (size_t)v.s * 4);
      cp(fout->qcodes, qcodes, (size_t)v.s_pad);
      cp(fout->qscale, qscale, 4);
      cp(fout->qhead, qhead, 4);
      cp(fout->pp, pp, 8);
      cp(fout->xx, xx, 4);
      cp(fout->sel, sel, (size_t)w * 4);
      cp(fout->prim, prim, 4);
      continue;
    }
    // queries bucketed by nearest cluster: the per-query kernels then visit the queries
    // cluster by cluster (L2 locality of the per-query re-rank's rows); the cluster-major
    // path reads per-query key ranges only, so it keeps the batch order
    int* order = p.score_mode != 0 && p.rr_mode == 1 && v.opt.rr_order ? nullptr : order_buf;
    if (order) staged(6, st, [&] { launch_bucket(prim, n, v.L, order, st); });
    ScoreArgsHost sa{};
    sa.ix = v; sa.qcodes = qcodes; sa.qscale = qscale; sa.qhead = qhead; sa.xx = xx; sa.sel = sel;
    sa.w = w; sa.take_cap = p.take_cap; sa.rerank = rerank; sa.k = k; sa.smem_cap = p.smem_cap;
    sa.gkeys = gk; sa.gpos = gp; sa.gcap = p.gcap; sa.cand_pos = cpos; sa.cand_n = cn;
    sa.out_ids = ids; sa.out_scores = scores; sa.out_count = count; sa.q0 = (int)q0;
    sa.order = order;
    if (ph1) { sa.sel_keys = ph1->keys; sa.sel_ids = ph1->ids; sa.sel_count = ph1->count; }
    if (p.score_mode == 0) {
      staged(4, st, [&] { launch_score_select(sa, n, st); });
    } else {
      ClusterScoringHost ch{};
      ch.ix = v; ch.xp = xp; ch.qcodes = qcodes; ch.qscale = qscale; ch.qhead = qhead; ch.sel = sel; ch.w = w;
      ch.qoff = reinterpret_cast<int*>(base + p.off_qoff);
      ch.ncand = reinterpret_cast<int*>(base + p.off_ncand);
      ch.pair_off = reinterpret_cast<int*>(base + p.off_pairoff);
      ch.item_off = reinterpret_cast<int*>(base + p.off_itemoff);
      ch.pairs = reinterpret_cast<int*>(base + p.off_pairs);
      ch.kbase = reinterpret_cast<int*>(base + p.off_kbase);
      ch.keys = reinterpret_cast<uint32_t*>(base + p.off_keys);
      ch.work_counter = reinterpret_cast<int*>(base + p.off_ctr);
      // the screen path's side stream needs the pair bucketing only: bucket first, then the
      // scoring and the top-t selection run on this stream while the side stream builds
      // the group records and streams the screen (the bounds of every (row, query slot))
      staged(7, st, [&] { launch_cluster_prep(ch, n, st); });
      AuxStream& ax = aux_stream();
      const bool side = p.rr_mode == 1;
      if (side) {
        CUDA_TRY(cudaEventRecord(ax.fork, st));
        CUDA_TRY(cudaStreamWaitEvent(ax.s, ax.fork, 0));
      }
      staged(7, st, [&] { launch_cluster_scoring(ch, n, st, false); });
      SelectTopTHost th{};
      th.ix = v; th.sel = sel; th.w = w; th.qoff = ch.qoff; th.kbase = ch.kbase; th.keys = ch.keys;
      th.take_cap = p.take_cap; th.rerank = rerank; th.k = k; th.xx = xx; th.cand_pos = cpos;
      th.cand_n = cn; th.out_ids = ids; th.out_scores = scores; th.out_count = count;
      th.q0 = (int)q0; th.order = order; th.kcap = p.kcap;
      if (ph1) { th.sel_keys = ph1->keys; th.sel_ids = ph1->ids; th.sel_count = ph1->count; }
      uint32_t* marks = reinterpret_cast<uint32_t*>(base + p.off_marks);
      int* cidx = reinterpret_cast<int*>(base + p.off_cidx);
      if (p.rr_mode == 1) {
        CUDA_TRY(cudaMemsetAsync(marks, 0, p.marks_bytes, st));
        th.cand_idx = cidx;
        th.marks = marks;
      }
      if (side)
        staged(5, ax.s, [&] {
          launch_interleave_queries(v, x, n, reinterpret_cast<float*>(base + p.off_xint), ax.s);
        });
      ScreenHost sh{};
      if (p.screen) {
        sh.ix = v; sh.queries = x; sh.w = w; sh.qoff = ch.qoff; sh.pair_off = ch.pair_off;
        sh.pairs = ch.pairs; sh.kbase = ch.kbase; sh.marks = marks;
        sh.item_off = reinterpret_cast<int*>(base + p.off_scritem);
        sh.grp_off = reinterpret_cast<int*>(base + p.off_grpoff);
        sh.grec = reinterpret_cast<unsigned char*>(base + p.off_grec);
        sh.n_groups_max = p.n_groups_max;
        sh.ub = reinterpret_cast<float*>(base + p.off_ub);
        sh.lb = reinterpret_cast<float*>(base + p.off_lb);
        sh.cand_idx = cidx; sh.cand_n = cn; sh.take_cap = p.take_cap; sh.k = k; sh.diss = ch.keys;
        sh.counters = counters_ptr(st);
        staged(9, ax.s, [&] { launch_screen_prep(sh, n, ax.s); });
      }
      if (side) CUDA_TRY(cudaEventRecord(ax.join, ax.s));
      staged(4, st, [&] { launch_select_topt(th, n, st); });
      if (side) CUDA_TRY(cudaStreamWaitEvent(st, ax.join, 0));
      // the screen (every SM, HBM-bound) runs after the selection: launched on the side
      // stream next to the scoring it measured no faster (C2 1.45 vs 1.44 ms), its
      // persistent CTAs leave no room for the scoring and selection CTAs
      if (p.rr_mode == 1) path_begin(RRG_PATH_RERANK, st);
      if (p.screen) staged(9, st, [&] { launch_screen(sh, n, st); });
      if (p.screen) staged(9, st, [&] { launch_thresh(sh, n, st); });
      if (p.rr_mode == 1) {
        // scores are consumed: the key array is reused for the re-ranked distances
        ClusterRerankHost rh{};
        rh.ix = v; rh.queries = x; rh.w = w; rh.qoff = ch.qoff; rh.pair_off = ch.pair_off;
        rh.rr_item_off = reinterpret_cast<int*>(base + p.off_rritem); rh.pairs = ch.pairs;
        rh.kbase = ch.kbase; rh.marks = marks;
        rh.diss = ch.keys; rh.work_counter = ch.work_counter + 1; rh.mwords = p.mwords; rh.nq = n;
        // sparse selections (a query keeps < half of the rows its probes cover, taking
        // cluster sizes as a random query sees them): skip unselected row pairs
        rh.skip = v.opt.rr_skip >= 0 ? v.opt.rr_skip != 0 : (double)t < 0.5 * w * ix->m_biased;
        rh.compact = p.screen;
        if (p.screen) { rh.cand_idx = cidx; rh.cand_n = cn; rh.take_cap = p.take_cap; }
        rh.xint = reinterpret_cast<float*>(base + p.off_xint);
        rh.counters = counters_ptr(st);
        if (rh.counters) {  // rows the exact pass needs: union over each cluster's queries
          // (measurement only; on the side stream, outside the stage's span)
          CUDA_TRY(cudaEventRecord(ax.cfork, st));
          CUDA_TRY(cudaStreamWaitEvent(ax.s, ax.cfork, 0));
          launch_count_rows(v, ch.pair_off, ch.pairs, ch.kbase, ch.qoff, w, marks,
                            p.screen ? cidx : nullptr, cn, p.take_cap, p.mwords, rh.counters + 4, ax.s);
          CUDA_TRY(cudaEventRecord(ax.cjoin, ax.s));
        }
        staged(5, st, [&] { launch_cluster_rerank(rh, st); });
        TopkFinalHost fh{};
        fh.ix = v; fh.sel = sel; fh.w = w; fh.qoff = ch.qoff; fh.kbase = ch.kbase; fh.diss = ch.keys;
        fh.cand_idx = cidx; fh.cand_n = cn; fh.take_cap = p.take_cap; fh.k = k;
        fh.out_ids = ids; fh.out_scores = scores; fh.out_count = count; fh.q0 = (int)q0;
        fh.order = order;
        staged(5, st, [&] { launch_topk_final(fh, n, st); });
        path_end(RRG_PATH_RERANK, st);
        if (rh.counters) CUDA_TRY(cudaStreamWaitEvent(st, ax.cjoin, 0));
      }
    }
    if (rerank && !ph1 && p.rr_mode == 0) {
      RerankArgsHost ra{};
      ra.ix = v; ra.queries = x; ra.cand_pos = cpos; ra.cand_n = cn; ra.take_cap = p.take_cap;
      ra.k = k; ra.out_ids = ids; ra.out_scores = scores; ra.out_count = count; ra.q0 = (int)q0;
      ra.order = order;
      path_begin(RRG_PATH_RERANK, st);
      staged(5, st, [&] { launch_rerank(ra, n, st); });
      path_end(RRG_PATH_RERANK, st);
    }
    CUDA_TRY(cudaGetLastError());
  }
  path_end(RRG_PATH_SEARCH, st);
}

template <typename F>
int guarded(F&& f) {
  try {
    return f();
  } catch (const RrgFail& e) {
    return e.code;
  } catch (const std::bad_alloc&) {
    return fail(RRG_E_INTERNAL, "RrannError", "host out of memory");
  } catch (const std::exception& e) {
    return fail(RRG_E_INTERNAL, "RrannError", "%s", e.what());
  }
}

// Exact k-NN ground truth (brute_force_knn, bench.py:85-124): f64 distance blocks
// from the FP64 tensor-core GEMM, merged per query by the radix select of
// rrg_ground_truth.cu.  Chunked so the distance block stays near 4 GB.
void ground_truth_impl(const float* corpus, int64_t m, int32_t d, const float* queries,
                       int64_t nq, int32_t k, int32_t metric, int64_t* out_ids, cudaStream_t st) {
  if (k < 1 || k > m) raise_usage("ParameterError", "k=%d out of range [1, %lld]", k, (long long)m);
  if (metric < 0 || metric > 2) raise_usage("ParameterError", "unknown metric code %d", metric);
  if (k > kGtMaxK) raise_usage("ParameterError", "k=%d > %d not supported by the device ground truth", k, kGtMaxK);
  if (d < 1) raise_usage("ShapeError", "dimension %d", d);
  if (nq == 0) return;
  int64_t Pc = std::min<int64_t>(m, 1 << 20);
  if (const char* e = getenv("RRG_GT_CHUNK")) Pc = std::max<int64_t>(1, std::min<int64_t>(Pc, atoll(e)));
  int64_t Qc = std::max<int64_t>(128, ((int64_t)4 << 30) / (Pc * 8));
  Qc = std::min<int64_t>(Qc, std::max<int64_t>(nq, 1));
  const int64_t Ql = Qc;
  char* base = nullptr;
  size_t off = 0;
  auto carve = [&](size_t bytes) { size_t r = off; off += (bytes + 255) / 256 * 256; return r; };
  const size_t o_cc = carve(m * 8), o_qq = carve(Ql * 8), o_diss = carve(Ql * Pc * 8),
               o_rk0 = carve(Ql * k * 8), o_ri0 = carve(Ql * k * 8), o_rn0 = carve(Ql * 4),
               o_rk1 = carve(Ql * k * 8), o_ri1 = carve(Ql * k * 8), o_rn1 = carve(Ql * 4),
               o_err = carve(4);
  CUDA_TRY(cudaMallocAsync((void**)&base, off, st));
  struct Free { char* p; cudaStream_t s; ~Free() { cudaFreeAsync(p, s); } } guard{base, st};
  double* cc = reinterpret_cast<double*>(base + o_cc);
  double* qq = reinterpret_cast<double*>(base + o_qq);
  double* diss = reinterpret_cast<double*>(base + o_diss);
  uint64_t* rk[2] = {reinterpret_cast<uint64_t*>(base + o_rk0), reinterpret_cast<uint64_t*>(base + o_rk1)};
  int64_t* ri[2] = {reinterpret_cast<int64_t*>(base + o_ri0), reinterpret_cast<int64_t*>(base + o_ri1)};
  int* rn[2] = {reinterpret_cast<int*>(base + o_rn0), reinterpret_cast<int*>(base + o_rn1)};
  int* err = reinterpret_cast<int*>(base + o_err);
  CUDA_TRY(cudaMemsetAsync(err, 0, 4, st));
  if (metric != kMetricIp)  // euclidean: (c*c).sum(1); cosine: ||c|| with 0 -> 1
    staged(8, st, [&] { launch_gt_row_norms(corpus, m, d, metric == kMetricCosine ? 1 : 0, cc, st); });
  for (int64_t q0 = 0; q0 < nq; q0 += Qc) {
    const int n = (int)std::min<int64_t>(Qc, nq - q0);
    const float* qx = queries + q0 * d;
    if (metric == kMetricEuclidean) staged(8, st, [&] { launch_gt_row_norms(qx, n, d, 0, qq, st); });
    int cur = 0;
    bool first = true;
    for (int64_t p0 = 0; p0 < m; p0 += Pc) {
      const int np = (int)std::min<int64_t>(Pc, m - p0);
      staged(8, st, [&] {
        launch_gt_dist(qx, n, corpus + p0 * d, np, d, metric, qq, cc + p0, diss, Pc, st);
      });
      GtSelectHost h{};
      h.diss = diss; h.ld = Pc; h.n = np; h.id0 = p0;
      h.run_key = first ? nullptr : rk[cur]; h.run_id = first ? nullptr : ri[cur];
      h.run_n = first ? nullptr : rn[cur];
      h.out_key = rk[cur ^ 1]; h.out_id = ri[cur ^ 1]; h.out_n = rn[cur ^ 1];
      h.k = k; h.err = err;
      staged(8, st, [&] { launch_gt_select(h, n, st); });
      cur ^= 1;
      first = false;
    }
    CUDA_TRY(cudaMemcpy2DAsync(out_ids + q0 * k, (size_t)k * 8, ri[cur], (size_t)k * 8, (size_t)k * 8,
                               n, cudaMemcpyDeviceToDevice, st));
    CUDA_TRY(cudaGetLastError());
  }
  int herr = 0;
  CUDA_TRY(cudaMemcpyAsync(&herr, err, 4, cudaMemcpyDeviceToHost, st));
  CUDA_TRY(cudaStreamSynchronize(st));
  if (herr) raise_usage("RrannError", "more than 4096 exact ties at a k-th distance");
}

// A captured small-batch host search (rrg_search_host): H2D of the pinned staged
// queries, every kernel of the search and the D2H of the results replay as one
// CUDA graph -- one launch instead of ~15 stream operations per call.
struct GraphKey {
  uint64_t ix;  // RrgIndex::serial
  int64_t nq;
  int k, w, t, rerank, dim;
  bool operator<(const GraphKey& o) const {
    return std::tie(ix, nq, k, w, t, rerank, dim) < std::tie(o.ix, o.nq, o.k, o.w, o.t, o.rerank, o.dim);
  }
};
struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int64_t launches = 0;
};

struct HostCtx {
  int device = -1;
  cudaStream_t st = nullptr;  // compute
  cudaStream_t cs = nullptr;  // copies
  void* dbuf = nullptr;
  size_t dcap = 0;
  std::vector<cudaEvent_t> ev;
  // graph path: pinned staging (queries in; ids, scores, count, flag out)
  void* pin = nullptr;
  size_t pcap = 0;
  std::map<GraphKey, GraphEntry> graphs;
  void drop_graphs() {
    for (auto& kv : graphs) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
  ~HostCtx() {
    drop_graphs();
    if (pin) cudaFreeHost(pin);
    if (dbuf) cudaFree(dbuf);
    if (st) cudaStreamDestroy(st);
    if (cs) cudaStreamDestroy(cs);
    for (auto e : ev) cudaEventDestroy(e);
  }
};
thread_local HostCtx g_host;

}  // namespace

// ================================================================= C ABI

extern "C" {

int rrg_index_open(const char* path, int device, RrgIndex** out) {
  return guarded([&] { return open_impl(path, device, 0, -1, out); });
}

int rrg_index_open_shard(const char* path, int device, int32_t cb, int32_t ce, RrgIndex** out) {
  return guarded([&] { return open_impl(path, device, cb, ce, out); });
}

int rrg_index_create(const RrgIndexDesc* desc, int device, RrgIndex** out) {
  return guarded([&] { return create_impl(desc, device, 0, -1, out); });
}

int rrg_index_create_shard(const RrgIndexDesc* desc, int device, int32_t cb, int32_t ce,
                           RrgIndex** out) {
  return guarded([&] { return create_impl(desc, device, cb, ce, out); });
}

void rrg_index_destroy(RrgIndex* index) { delete index; }

int rrg_index_reload_options(RrgIndex* index) {
  if (!index) return fail(RRG_E_USAGE, "ParameterError", "null argument");
  index->view.opt = read_opts();
  index->serial = RrgIndex::next_serial();  // captured graphs embed the old variant choices
  return RRG_OK;
}

int rrg_index_info(const RrgIndex* index, RrgIndexInfo* out) {
  if (!index || !out) return fail(RRG_E_USAGE, "ParameterError", "null argument");
  *out = index->info;
  return RRG_OK;
}

int rrg_index_cluster_sizes(const RrgIndex* index, uint32_t* out) {
  if (!index || !out) return fail(RRG_E_USAGE, "ParameterError", "null argument");
  std::copy(index->held_sizes.begin(), index->held_sizes.end(), out);
  return RRG_OK;
}

size_t rrg_search_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t k, int32_t w,
                                  int32_t t, int32_t rerank) {
  if (!index || nq <= 0 || k < 1 || w < 1 || t < 1) return 0;
  return make_plan(index, nq, k, w, t, rerank).total;
}

int rrg_search(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
               int32_t w, int32_t t, int32_t rerank, int64_t* ids, float* scores, int32_t* count,
               void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  return guarded([&] {
    if (!index) return fail(RRG_E_USAGE, "ParameterError", "null index");
    if (nq == 0) return RRG_OK;  // query_batch on an empty batch returns [] (index.py:340)
    validate_search(index, dim, k, w, t, rerank);
    CUDA_TRY(cudaSetDevice(index->device));
    search_impl(index, queries, nq, k, w, t, rerank, ids, scores, count, workspace,
                workspace_bytes, static_cast<cudaStream_t>(stream));
    return RRG_OK;
  });
}

int rrg_search_host(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                    int32_t w, int32_t t, int32_t rerank, int64_t* ids, float* scores,
                    int32_t* count) {
  g_launches = 0;
  return guarded([&] {
    if (!index) return fail(RRG_E_USAGE, "ParameterError", "null index");
    if (nq == 0) return RRG_OK;
    // Validation order of query_batch: _check_finite (DataError, index.py:144-150)
    // before QueryParams.validate.  The finiteness test runs on the GPU inside the
    // query-prep pass; only when the parameters are invalid is the batch scanned on
    // the host first, so that a non-finite batch still reports DataError.
    try {
      validate_search(index, dim, k, w, t, rerank);
    } catch (const RrgFail&) {
      const std::string msg = g_err, kind = g_kind;
      for (int64_t i = 0; i < nq * (int64_t)dim; ++i)
        if (!std::isfinite(queries[i]))
          return fail(RRG_E_DATA, "DataError", "queries: contains non-finite values");
      g_err = msg;
      g_kind = kind;
      throw;
    }
    CUDA_TRY(cudaSetDevice(index->device));
    HostCtx& h = g_host;
    if (h.device != index->device) {
      h.drop_graphs();
      if (h.dbuf) cudaFree(h.dbuf);
      if (h.st) cudaStreamDestroy(h.st);
      if (h.cs) cudaStreamDestroy(h.cs);
      h.dbuf = nullptr; h.dcap = 0; h.st = nullptr; h.cs = nullptr;
      CUDA_TRY(cudaStreamCreateWithFlags(&h.st, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&h.cs, cudaStreamNonBlocking));
      h.device = index->device;
    }
    // Pipeline: the whole batch is one search (scoring and re-rank gain from seeing
    // every query), but the queries are copied in NSUB pieces on a copy stream and the
    // per-query front stages (projection .. routing) of piece j start as soon as it
    // has landed, overlapping the copies of pieces j+1..; results come back after.
    int nsub = nq >= 4096 ? 2 : 1;  // measured on C2: 2 pieces 3.17 ms, 4: 3.20, 1: 3.32
    if (index->view.opt.host_pieces > 0) nsub = index->view.opt.host_pieces;
    Plan p = make_plan(index, nq, k, w, t, rerank);
    const size_t qbytes = (size_t)nq * dim * 4, ibytes = (size_t)nq * k * 8,
                 sbytes = (size_t)nq * k * 4, cbytes = (size_t)nq * 4;
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    size_t need = al(qbytes) + al(ibytes) + al(sbytes) + al(cbytes) + 256 + p.total;
    if (need > h.dcap) {
      h.drop_graphs();  // captured pointers die with the buffer
      if (h.dbuf) cudaFree(h.dbuf);
      h.dbuf = nullptr;
      CUDA_TRY(cudaMalloc(&h.dbuf, need));
      h.dcap = need;
    }
    char* b = static_cast<char*>(h.dbuf);
    float* dq = reinterpret_cast<float*>(b);
    int64_t* di = reinterpret_cast<int64_t*>(b + al(qbytes));
    float* dsc = reinterpret_cast<float*>(b + al(qbytes) + al(ibytes));
    int32_t* dc = reinterpret_cast<int32_t*>(b + al(qbytes) + al(ibytes) + al(sbytes));
    int* dflag = reinterpret_cast<int*>(b + al(qbytes) + al(ibytes) + al(sbytes) + al(cbytes));
    void* ws = b + al(qbytes) + al(ibytes) + al(sbytes) + al(cbytes) + 256;
    if (h.ev.empty()) {
      h.ev.resize(9);
      for (auto& e : h.ev) CUDA_TRY(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
    }
    // small batches: replay a captured graph (launch latency dominates there)
    const bool use_graph = nq <= 2048 && !g_timer.on && index->view.opt.graph;
    if (use_graph) {
      const size_t pneed = al(qbytes) + al(ibytes) + al(sbytes) + al(cbytes) + 256;
      if (pneed > h.pcap) {
        h.drop_graphs();
        if (h.pin) cudaFreeHost(h.pin);
        h.pin = nullptr;
        CUDA_TRY(cudaMallocHost(&h.pin, pneed));
        h.pcap = pneed;
      }
      char* hp = static_cast<char*>(h.pin);
      float* hq = reinterpret_cast<float*>(hp);
      int64_t* hi = reinterpret_cast<int64_t*>(hp + al(qbytes));
      float* hs = reinterpret_cast<float*>(hp + al(qbytes) + al(ibytes));
      int32_t* hc = reinterpret_cast<int32_t*>(hp + al(qbytes) + al(ibytes) + al(sbytes));
      int* hf = reinterpret_cast<int*>(hp + al(qbytes) + al(ibytes) + al(sbytes) + al(cbytes));
      const GraphKey key{index->serial, nq, k, w, t, rerank, dim};
      auto it = h.graphs.find(key);
      if (it == h.graphs.end()) {
        if (h.graphs.size() >= 64) h.drop_graphs();  // bound the cache
        cudaGraph_t graph = nullptr;
        CUDA_TRY(cudaStreamBeginCapture(h.st, cudaStreamCaptureModeRelaxed));
        const int64_t before = g_launches;
        try {
          CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int), h.st));
          CUDA_TRY(cudaMemcpyAsync(dq, hq, qbytes, cudaMemcpyHostToDevice, h.st));
          search_impl(index, dq, nq, k, w, t, rerank, di, dsc, dc, ws, p.total, h.st, nullptr, dflag);
          CUDA_TRY(cudaMemcpyAsync(hi, di, ibytes, cudaMemcpyDeviceToHost, h.st));
          CUDA_TRY(cudaMemcpyAsync(hs, dsc, sbytes, cudaMemcpyDeviceToHost, h.st));
          CUDA_TRY(cudaMemcpyAsync(hc, dc, cbytes, cudaMemcpyDeviceToHost, h.st));
          CUDA_TRY(cudaMemcpyAsync(hf, dflag, sizeof(int), cudaMemcpyDeviceToHost, h.st));
        } catch (...) {
          cudaStreamEndCapture(h.st, &graph);
          if (graph) cudaGraphDestroy(graph);
          throw;
        }
        CUDA_TRY(cudaStreamEndCapture(h.st, &graph));
        GraphEntry ge2;
        ge2.launches = g_launches - before;
        const cudaError_t ie = cudaGraphInstantiate(&ge2.exec, graph, 0);
        cudaGraphDestroy(graph);
        CUDA_TRY(ie);
        it = h.graphs.emplace(key, ge2).first;
      }
      memcpy(hq, queries, qbytes);
      CUDA_TRY(cudaGraphLaunch(it->second.exec, h.st));
      CUDA_TRY(cudaStreamSynchronize(h.st));
      g_launches = it->second.launches;
      if (*hf) return fail(RRG_E_DATA, "DataError", "queries: contains non-finite values");
      memcpy(ids, hi, ibytes);
      memcpy(scores, hs, sbytes);
      memcpy(count, hc, cbytes);
      return RRG_OK;
    }
    CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int), h.st));
    std::vector<cudaEvent_t> in_ready;
    for (int j = 0; j < nsub; ++j) {
      const int64_t s0 = piece_bound(nq, j, nsub), s1 = piece_bound(nq, j + 1, nsub);
      CUDA_TRY(cudaMemcpyAsync(dq + s0 * dim, queries + s0 * dim, (size_t)(s1 - s0) * dim * 4,
                               cudaMemcpyHostToDevice, h.cs));
      CUDA_TRY(cudaEventRecord(h.ev[j], h.cs));
      in_ready.push_back(h.ev[j]);
    }
    search_impl(index, dq, nq, k, w, t, rerank, di, dsc, dc, ws, p.total, h.st, nullptr, dflag,
                &in_ready);
    CUDA_TRY(cudaEventRecord(h.ev[8], h.st));
    CUDA_TRY(cudaStreamWaitEvent(h.cs, h.ev[8], 0));
    CUDA_TRY(cudaMemcpyAsync(ids, di, (size_t)nq * k * 8, cudaMemcpyDeviceToHost, h.cs));
    CUDA_TRY(cudaMemcpyAsync(scores, dsc, (size_t)nq * k * 4, cudaMemcpyDeviceToHost, h.cs));
    CUDA_TRY(cudaMemcpyAsync(count, dc, (size_t)nq * 4, cudaMemcpyDeviceToHost, h.cs));
    int flag = 0;
    CUDA_TRY(cudaStreamSynchronize(h.st));
    CUDA_TRY(cudaMemcpyAsync(&flag, dflag, sizeof(int), cudaMemcpyDeviceToHost, h.cs));
    CUDA_TRY(cudaStreamSynchronize(h.cs));
    if (flag) return fail(RRG_E_DATA, "DataError", "queries: contains non-finite values");
    return RRG_OK;
  });
}

// Several host batches in one call, software-pipelined over two device buffer sets:
// the H2D copy of batch b+1 (copy-in stream) and the D2H copy of batch b-1
// (copy-out stream) overlap the search of batch b (compute stream).  Each batch
// is validated and searched exactly like rrg_search_host.
struct PipeSlot {
  void* buf = nullptr;
  size_t cap = 0;
  cudaEvent_t in_ready = nullptr, comp_done = nullptr, out_done = nullptr;
};
struct PipeCtx {
  int device = -1;
  cudaStream_t cs = nullptr, ci = nullptr, co = nullptr;
  PipeSlot slot[2];
  int* hflags = nullptr;  // pinned, one per batch
  int64_t nflags = 0;
  void reset() {
    for (auto& sl : slot) {
      if (sl.buf) cudaFree(sl.buf);
      if (sl.in_ready) cudaEventDestroy(sl.in_ready);
      if (sl.comp_done) cudaEventDestroy(sl.comp_done);
      if (sl.out_done) cudaEventDestroy(sl.out_done);
      sl = PipeSlot{};
    }
    if (hflags) cudaFreeHost(hflags);
    hflags = nullptr;
    nflags = 0;
    if (cs) cudaStreamDestroy(cs);
    if (ci) cudaStreamDestroy(ci);
    if (co) cudaStreamDestroy(co);
    cs = ci = co = nullptr;
    device = -1;
  }
  ~PipeCtx() { reset(); }
};
thread_local PipeCtx g_pipe;

int rrg_search_host_many(RrgIndex* index, int32_t nbatch, const float* const* queries,
                         const int64_t* nq, int32_t dim, int32_t k, int32_t w, int32_t t,
                         int32_t rerank, int64_t* const* ids, float* const* scores,
                         int32_t* const* count) {
  g_launches = 0;
  return guarded([&] {
    if (!index) return fail(RRG_E_USAGE, "ParameterError", "null index");
    if (nbatch < 0) return fail(RRG_E_USAGE, "ParameterError", "nbatch < 0");
    int64_t qmax = 0;
    for (int b = 0; b < nbatch; ++b) qmax = std::max<int64_t>(qmax, nq[b]);
    if (qmax == 0) return RRG_OK;
    try {
      validate_search(index, dim, k, w, t, rerank);
    } catch (const RrgFail&) {  // DataError first for a non-finite batch (index.py:339)
      const std::string msg = g_err, kind = g_kind;
      for (int b = 0; b < nbatch; ++b)
        for (int64_t i = 0; i < nq[b] * (int64_t)dim; ++i)
          if (!std::isfinite(queries[b][i]))
            return fail(RRG_E_DATA, "DataError", "queries: contains non-finite values");
      g_err = msg;
      g_kind = kind;
      throw;
    }
    CUDA_TRY(cudaSetDevice(index->device));
    PipeCtx& pc = g_pipe;
    if (pc.device != index->device) {
      pc.reset();
      CUDA_TRY(cudaStreamCreateWithFlags(&pc.cs, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&pc.ci, cudaStreamNonBlocking));
      CUDA_TRY(cudaStreamCreateWithFlags(&pc.co, cudaStreamNonBlocking));
      for (auto& sl : pc.slot) {
        CUDA_TRY(cudaEventCreateWithFlags(&sl.in_ready, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.comp_done, cudaEventDisableTiming));
        CUDA_TRY(cudaEventCreateWithFlags(&sl.out_done, cudaEventDisableTiming));
      }
      pc.device = index->device;
    }
    if (pc.nflags < nbatch) {
      if (pc.hflags) cudaFreeHost(pc.hflags);
      pc.hflags = nullptr;
      CUDA_TRY(cudaMallocHost(&pc.hflags, (size_t)nbatch * sizeof(int)));
      pc.nflags = nbatch;
    }
    auto al = [](size_t b) { return (b + 255) / 256 * 256; };
    Plan pmax = make_plan(index, qmax, k, w, t, rerank);
    const size_t qb = al((size_t)qmax * dim * 4), ib = al((size_t)qmax * k * 8),
                 sb = al((size_t)qmax * k * 4), cb = al((size_t)qmax * 4);
    const size_t need = qb + ib + sb + cb + 256 + pmax.total;
    for (auto& sl : pc.slot)
      if (sl.cap < need) {
        CUDA_TRY(cudaStreamSynchronize(pc.cs));
        if (sl.buf) cudaFree(sl.buf);
        sl.buf = nullptr;
        CUDA_TRY(cudaMalloc(&sl.buf, need));
        sl.cap = need;
      }
    for (int b = 0; b < nbatch; ++b) {
      PipeSlot& sl = pc.slot[b & 1];
      const int64_t n = nq[b];
      char* base = static_cast<char*>(sl.buf);
      float* dq = reinterpret_cast<float*>(base);
      int64_t* di = reinterpret_cast<int64_t*>(base + qb);
      float* dsc = reinterpret_cast<float*>(base + qb + ib);
      int32_t* dc = reinterpret_cast<int32_t*>(base + qb + ib + sb);
      int* dflag = reinterpret_cast<int*>(base + qb + ib + sb + cb);
      void* ws = base + qb + ib + sb + cb + 256;
      pc.hflags[b] = 0;
      if (n == 0) continue;
      // in: the slot's queries were last read by the search of batch b-2
      if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(pc.ci, sl.comp_done, 0));
      CUDA_TRY(cudaMemcpyAsync(dq, queries[b], (size_t)n * dim * 4, cudaMemcpyHostToDevice, pc.ci));
      CUDA_TRY(cudaEventRecord(sl.in_ready, pc.ci));
      // search: its outputs were last read by the D2H of batch b-2
      CUDA_TRY(cudaStreamWaitEvent(pc.cs, sl.in_ready, 0));
      if (b >= 2) CUDA_TRY(cudaStreamWaitEvent(pc.cs, sl.out_done, 0));
      CUDA_TRY(cudaMemsetAsync(dflag, 0, sizeof(int), pc.cs));
      search_impl(index, dq, n, k, w, t, rerank, di, dsc, dc, ws, pmax.total, pc.cs, nullptr, dflag);
      CUDA_TRY(cudaEventRecord(sl.comp_done, pc.cs));
      // out
      CUDA_TRY(cudaStreamWaitEvent(pc.co, sl.comp_done, 0));
      CUDA_TRY(cudaMemcpyAsync(ids[b], di, (size_t)n * k * 8, cudaMemcpyDeviceToHost, pc.co));
      CUDA_TRY(cudaMemcpyAsync(scores[b], dsc, (size_t)n * k * 4, cudaMemcpyDeviceToHost, pc.co));
      CUDA_TRY(cudaMemcpyAsync(count[b], dc, (size_t)n * 4, cudaMemcpyDeviceToHost, pc.co));
      CUDA_TRY(cudaMemcpyAsync(pc.hflags + b, dflag, sizeof(int), cudaMemcpyDeviceToHost, pc.co));
      CUDA_TRY(cudaEventRecord(sl.out_done, pc.co));
    }
    CUDA_TRY(cudaStreamSynchronize(pc.co));
    CUDA_TRY(cudaStreamSynchronize(pc.cs));
    for (int b = 0; b < nbatch; ++b)
      if (pc.hflags[b]) return fail(RRG_E_DATA, "DataError", "queries: contains non-finite values");
    return RRG_OK;
  });
}

int rrg_stage_project(RrgIndex* index, const float* queries, int64_t nq, float* xp,
                      int8_t* qcodes, float* qscale, float* qhead, void* stream) {
  return guarded([&] {
    const DevIndexView& v = index->view;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(index->device));
    double* pp = nullptr;
    float* xx = nullptr;
    CUDA_TRY(cudaMallocAsync(&pp, std::max<int64_t>(nq, 1) * 8, st));
    CUDA_TRY(cudaMallocAsync(&xx, std::max<int64_t>(nq, 1) * 4, st));
    int8_t* qpl = nullptr;
    int* qex = nullptr;
    if (v.opt.proj_sliced && nq > 0) {
      CUDA_TRY(cudaMallocAsync(&qpl, sliced_plane_bytes((int)nq, v.d, true), st));
      CUDA_TRY(cudaMallocAsync(&qex, (size_t)sliced_rows_pad((int)nq, true) * 4, st));
      launch_slice_rows(queries, (int)nq, v.d, v.d, true, qpl, qex, st);
      launch_gemm_sliced(qpl, qex, (int)nq, v.wt_planes, v.wt_exps, v.s, v.d, EPI_PROJ, xp, nullptr,
                         v.s, nullptr, nullptr, st);
      CUDA_TRY(cudaFreeAsync(qpl, st));
      CUDA_TRY(cudaFreeAsync(qex, st));
    } else {
      launch_project(queries, v.W, (int)nq, v.d, v.s, xp, v.opt.gemm_bk, st);
    }
    launch_prep(xp, queries, (int)nq, v.s, v.s_pad, v.d, qcodes, qscale, qhead, pp, xx, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaFreeAsync(pp, st));
    CUDA_TRY(cudaFreeAsync(xx, st));
    return RRG_OK;
  });
}

int rrg_stage_route(RrgIndex* index, const float* xp, int64_t nq, int32_t w, int32_t* selected,
                    void* workspace, size_t workspace_bytes, void* stream) {
  return guarded([&] {
    const DevIndexView& v = index->view;
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    size_t need = (size_t)nq * v.L * 8 + (size_t)nq * 8 + (size_t)nq * v.s_pad + 1024;
    if (workspace_bytes < need) raise_usage("ParameterError", "workspace too small");
    double* diss = static_cast<double*>(workspace);
    double* pp = diss + (size_t)nq * v.L;
    // recompute pp (f64 pairwise) via the prep kernel on xp; queries unused for xx
    int8_t* qc = reinterpret_cast<int8_t*>(pp + nq);
    float* dummy = nullptr;
    CUDA_TRY(cudaMallocAsync(&dummy, std::max<int64_t>(nq, 1) * 16, st));
    launch_prep(xp, xp, (int)nq, v.s, v.s_pad, v.s, qc, dummy, dummy + nq, pp, dummy + 2 * nq, st);
    int8_t* qpl = nullptr;
    int* qex = nullptr;
    if (v.opt.route_sliced) {
      CUDA_TRY(cudaMallocAsync(&qpl, sliced_plane_bytes((int)nq, v.s, true), st));
      CUDA_TRY(cudaMallocAsync(&qex, (size_t)sliced_rows_pad((int)nq, true) * 4, st));
    }
    route_dist(v, xp, (int)nq, pp, diss, qpl, qex, st);
    if (qpl) {
      CUDA_TRY(cudaFreeAsync(qpl, st));
      CUDA_TRY(cudaFreeAsync(qex, st));
    }
    launch_route_select(diss, (int)nq, v.L, w, selected, reinterpret_cast<int*>(dummy + 3 * nq), st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaFreeAsync(dummy, st));
    return RRG_OK;
  });
}

// Data-parallel front stages (SURVEY.md 8(e) "Queries"): the sharded search splits the
// batch's projection / quantization / routing over the ranks and all-gathers these rows.
size_t rrg_front_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t w) {
  if (!index || nq <= 0 || w < 1) return 0;
  return make_plan(index, nq, 1, w, 1, 0).total;
}

int rrg_search_front(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t w,
                     const RrgFront* out, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  return guarded([&] {
    if (!index || !out) return fail(RRG_E_USAGE, "ParameterError", "null argument");
    if (nq == 0) return RRG_OK;
    validate_search(index, dim, 1, w, 1, 0);
    CUDA_TRY(cudaSetDevice(index->device));
    search_impl(index, queries, nq, 1, w, 1, 0, nullptr, nullptr, nullptr, workspace, workspace_bytes,
                static_cast<cudaStream_t>(stream), nullptr, nullptr, nullptr, nullptr, out);
    return RRG_OK;
  });
}

int rrg_search_from_front(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                          int32_t w, int32_t t, int32_t rerank, const RrgFront* front, int64_t* ids,
                          float* scores, int32_t* count, void* workspace, size_t workspace_bytes,
                          void* stream) {
  g_launches = 0;
  return guarded([&] {
    if (!index || !front) return fail(RRG_E_USAGE, "ParameterError", "null argument");
    if (nq == 0) return RRG_OK;
    validate_search(index, dim, k, w, t, rerank);
    CUDA_TRY(cudaSetDevice(index->device));
    search_impl(index, queries, nq, k, w, t, rerank, ids, scores, count, workspace, workspace_bytes,
                static_cast<cudaStream_t>(stream), nullptr, nullptr, nullptr, front);
    return RRG_OK;
  });
}

// K4 stage outputs (score_cluster, rrr.py:181-203 / quantize.py:109-156) of the
// production cluster-major scoring kernel for caller-chosen probes: the projection
// and query quantization of the search path, then k_score_cluster with its stage
// outputs switched on.  Layout: raw1[q][c][j] (stage A, j < r, RRR clusters), and per
// candidate (query-major, probes in sel order: cand_off[q] + offset of probe c +
// point) raw2 = the last stage's int32 product (stage B, or stage A of an exact
// model) and the f32 score.
int rrg_stage_score(RrgIndex* index, const float* queries, int64_t nq, int32_t w,
                    const int32_t* sel, int32_t* raw1, int32_t* raw2, float* scores,
                    int32_t* cand_off, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  return guarded([&] {
    if (!index) return fail(RRG_E_USAGE, "ParameterError", "null index");
    if (nq == 0) return RRG_OK;
    const DevIndexView& v = index->view;
    if (!(1 <= w && w <= v.L)) raise_usage("ParameterError", "w=%d out of range [1, %d]", w, v.L);
    if (v.opt.score_query) raise_usage("ParameterError", "stage scoring runs the cluster-major kernel");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    CUDA_TRY(cudaSetDevice(index->device));
    Plan p = make_plan(index, nq, 1, w, 1, 0);
    if (p.qc < nq) raise_usage("ParameterError", "stage batch of %lld queries exceeds one chunk", (long long)nq);
    if (workspace_bytes < p.total)
      raise_usage("ParameterError", "workspace too small: %zu < %zu bytes", workspace_bytes, p.total);
    char* base = static_cast<char*>(workspace);
    float* xp = reinterpret_cast<float*>(base + p.off_xp);
    int8_t* qcodes = reinterpret_cast<int8_t*>(base + p.off_qc);
    float* qscale = reinterpret_cast<float*>(base + p.off_qs);
    float* qhead = reinterpret_cast<float*>(base + p.off_qh);
    float* xx = reinterpret_cast<float*>(base + p.off_xx);
    double* pp = reinterpret_cast<double*>(base + p.off_pp);
    const int n = (int)nq;
    if (n <= kSmallBatch) {
      launch_project_small(queries, v.Wt, n, v.d, v.s, xp, st);
    } else if (v.opt.proj_sliced) {
      int8_t* qpl = reinterpret_cast<int8_t*>(base + p.off_qpl);
      int* qex = reinterpret_cast<int*>(base + p.off_qex);
      launch_slice_rows(queries, n, v.d, v.d, true, qpl, qex, st);
      launch_gemm_sliced(qpl, qex, n, v.wt_planes, v.wt_exps, v.s, v.d, EPI_PROJ, xp, nullptr, v.s,
                         nullptr, nullptr, st);
    } else {
      launch_project(queries, v.W, n, v.d, v.s, xp, v.opt.gemm_bk, st);
    }
    launch_prep(xp, queries, n, v.s, v.s_pad, v.d, qcodes, qscale, qhead, pp, xx, st);
    ClusterScoringHost ch{};
    ch.ix = v; ch.xp = xp; ch.qcodes = qcodes; ch.qscale = qscale; ch.qhead = qhead; ch.sel = sel;
    ch.w = w;
    ch.qoff = reinterpret_cast<int*>(base + p.off_qoff);
    ch.ncand = reinterpret_cast<int*>(base + p.off_ncand);
    ch.pair_off = reinterpret_cast<int*>(base + p.off_pairoff);
    ch.item_off = reinterpret_cast<int*>(base + p.off_itemoff);
    ch.pairs = reinterpret_cast<int*>(base + p.off_pairs);
    ch.kbase = cand_off;
    ch.keys = reinterpret_cast<uint32_t*>(base + p.off_keys);
    ch.work_counter = reinterpret_cast<int*>(base + p.off_ctr);
    ch.dbg_raw1 = raw1; ch.dbg_raw2 = raw2; ch.dbg_score = scores;
    launch_cluster_scoring(ch, n, st);
    CUDA_TRY(cudaGetLastError());
    CUDA_TRY(cudaStreamSynchronize(st));
    return RRG_OK;
  });
}

size_t rrg_stage_score_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t w) {
  if (!index || nq <= 0 || w < 1) return 0;
  return make_plan(index, nq, 1, w, 1, 0).total;
}

// ---------------------------------------------------------- sharded search

size_t rrg_shard_workspace_bytes(const RrgIndex* index, int64_t nq, int32_t k, int32_t w,
                                 int32_t t) {
  if (!index || nq <= 0 || k < 1 || w < 1 || t < 1) return 0;
  size_t a = make_plan(index, nq, k, w, t, 1, true).total;
  size_t b = ((size_t)nq * t * 4 + 255) / 256 * 256 + ((size_t)nq * 4 + 255) / 256 * 256;
  return std::max(a, b);
}

int rrg_shard_phase1(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                     int32_t w, int32_t t, uint32_t* keys, uint32_t* ids, int32_t* count,
                     void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  return guarded([&] {
    if (!index) return fail(RRG_E_USAGE, "ParameterError", "null index");
    if (nq == 0) return RRG_OK;
    validate_search(index, dim, k, w, t, 1);
    CUDA_TRY(cudaSetDevice(index->device));
    Phase1Out o{keys, ids, count};
    search_impl(index, queries, nq, k, w, t, 1, nullptr, nullptr, nullptr, workspace,
                workspace_bytes, static_cast<cudaStream_t>(stream), &o);
    return RRG_OK;
  });
}

int rrg_shard_phase1_from_front(RrgIndex* index, const float* queries, int64_t nq, int32_t dim, int32_t k,
                                int32_t w, int32_t t, const RrgFront* front, uint32_t* keys, uint32_t* ids,
                                int32_t* count, void* workspace, size_t workspace_bytes, void* stream) {
  g_launches = 0;
  return guarded([&] {
    if (!index || !front) return fail(RRG_E_USAGE, "ParameterError", "null argument");
    if (nq == 0) return RRG_OK;
    validate_search(index, dim, k, w, t, 1);
    CUDA_TRY(cudaSetDevice(index->device));
    Phase1Out o{keys, ids, count};
    search_impl(index, queries, nq, k, w, t, 1, nullptr, nullptr, nullptr, workspace, workspace_bytes,
                static_cast<cudaStream_t>(stream), &o, nullptr, nullptr, front);
    return RRG_OK;
  });
}

int rrg_merge_candidates(int64_t nq, int32_t G, int32_t cap, const uint32_t* keys,
                         const uint32_t* ids, const int32_t* counts, int32_t take,
                         uint32_t* out_keys, uint32_t* out_ids, int32_t* out_count, void* stream) {
  return guarded([&] {
    if (G < 1 || G > 64) raise_usage("ParameterError", "G=%d out of range [1, 64]", G);
    if (nq == 0) return RRG_OK;
    staged(4, static_cast<cudaStream_t>(stream), [&] {
      launch_merge(0, 0, (int)nq, G, cap, keys, ids, counts, take, out_keys, out_ids, out_count,
                   static_cast<cudaStream_t>(stream));
    });
    CUDA_TRY(cudaGetLastError());
    return RRG_OK;
  });
}

int rrg_pack_candidates(int64_t nq, int32_t cap, const uint32_t* keys, const uint32_t* ids,
                        const int32_t* counts, uint32_t* packed_keys, uint32_t* packed_ids,
                        int32_t* offsets, void* stream) {
  return guarded([&] {
    if (nq < 0 || cap < 1) raise_usage("ParameterError", "bad list shape");
    // the packed offsets are int32: the exchange of one call holds < 2^31 entries
    if (nq * (int64_t)cap > (int64_t)INT32_MAX)
      raise_usage("ParameterError", "nq * cap = %lld exceeds the int32 offsets of the packed exchange; "
                  "split the batch", (long long)(nq * (int64_t)cap));
    if (nq == 0) return RRG_OK;
    staged(4, static_cast<cudaStream_t>(stream), [&] {
      launch_pack_candidates((int)nq, cap, keys, ids, counts, packed_keys, packed_ids, offsets,
                             static_cast<cudaStream_t>(stream));
    });
    return RRG_OK;
  });
}

int rrg_unpack_candidates(int64_t nq, int32_t G, int64_t stride, int32_t cap,
                          const uint32_t* packed_keys, const uint32_t* packed_ids,
                          const int32_t* offsets, uint32_t* keys, uint32_t* ids, int32_t* counts,
                          void* stream) {
  return guarded([&] {
    if (G < 1 || G > 64) raise_usage("ParameterError", "G=%d out of range [1, 64]", G);
    if (nq == 0) return RRG_OK;
    staged(4, static_cast<cudaStream_t>(stream), [&] {
      launch_unpack_candidates((int)nq, G, stride, cap, packed_keys, packed_ids, offsets, keys, ids,
                               counts, static_cast<cudaStream_t>(stream));
    });
    return RRG_OK;
  });
}

int rrg_shard_phase2(RrgIndex* index, const float* queries, int64_t nq, int32_t dim,
                     const uint32_t* cand_ids, const int32_t* cand_count, int32_t cap, int32_t k,
                     int64_t* ids, float* scores, int32_t* count, void* workspace,
                     size_t workspace_bytes, void* stream) {
  return guarded([&] {
    if (!index) return fail(RRG_E_USAGE, "ParameterError", "null index");
    if (nq == 0) return RRG_OK;
    validate_search(index, dim, k, 1, std::max(cap, k), 1);
    size_t need = ((size_t)nq * cap * 4 + 255) / 256 * 256 + ((size_t)nq * 4 + 255) / 256 * 256;
    if (workspace_bytes < need) raise_usage("ParameterError", "workspace too small");
    CUDA_TRY(cudaSetDevice(index->device));
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    int* cpos = static_cast<int*>(workspace);
    int* cn = reinterpret_cast<int*>(static_cast<char*>(workspace) +
                                     ((size_t)nq * cap * 4 + 255) / 256 * 256);
    staged(5, st, [&] { launch_ids_to_pos(index->view, (int)nq, cap, cand_ids, cand_count, cpos, cn, st); });
    RerankArgsHost ra{};
    ra.ix = index->view; ra.queries = queries; ra.cand_pos = cpos; ra.cand_n = cn;
    ra.take_cap = cap; ra.k = k; ra.out_ids = ids; ra.out_scores = scores; ra.out_count = count;
    ra.q0 = 0;
    staged(5, st, [&] { launch_rerank(ra, (int)nq, st); });
    CUDA_TRY(cudaGetLastError());
    return RRG_OK;
  });
}

int rrg_merge_results(int64_t nq, int32_t G, int32_t k, int32_t metric, const float* scores,
                      const int64_t* ids, const int32_t* counts, float* out_scores,
                      int64_t* out_ids, int32_t* out_count, void* stream) {
  return guarded([&] {
    if (G < 1 || G > 64) raise_usage("ParameterError", "G=%d out of range [1, 64]", G);
    if (nq == 0) return RRG_OK;
    staged(5, static_cast<cudaStream_t>(stream), [&] {
      launch_merge(1, metric, (int)nq, G, k, scores, ids, counts, k, out_scores, out_ids,
                   out_count, static_cast<cudaStream_t>(stream));
    });
    CUDA_TRY(cudaGetLastError());
    return RRG_OK;
  });
}

int64_t rrg_last_launch_count(void) { return g_launches; }

int rrg_search_counters(int64_t* out) {
  StageTimer& t = g_timer;
  for (int i = 0; i < RRG_N_COUNTERS; ++i) out[i] = 0;
  if (t.dcounters == nullptr) return RRG_OK;
  int prev = 0;
  cudaGetDevice(&prev);
  cudaSetDevice(t.cdev);
  cudaDeviceSynchronize();
  cudaMemcpy(out, t.dcounters, RRG_N_COUNTERS * 8, cudaMemcpyDeviceToHost);
  cudaMemset(t.dcounters, 0, RRG_N_COUNTERS * 8);
  cudaSetDevice(prev);
  return RRG_OK;
}

void rrg_set_stage_timing(int enabled) { g_timer.on = enabled != 0; }

int rrg_stage_times(double* ms, int64_t* launches) {
  StageTimer& t = g_timer;
  for (auto& r : t.pending) {
    cudaEventSynchronize(r.b);
    float el = 0.f;
    cudaEventElapsedTime(&el, r.a, r.b);
    t.ms[r.stage] += el;
    t.n[r.stage] += 1;
    t.pool.push_back(r.a);
    t.pool.push_back(r.b);
  }
  t.pending.clear();
  for (int i = 0; i < RRG_N_STAGES; ++i) {
    if (ms) ms[i] = t.ms[i];
    if (launches) launches[i] = t.n[i];
    t.ms[i] = 0;
    t.n[i] = 0;
  }
  return RRG_OK;
}
int rrg_path_times(double* ms, int64_t* count) {
  StageTimer& t = g_timer;
  for (auto& r : t.path_pending) {
    cudaEventSynchronize(r.b);
    float el = 0.f;
    cudaEventElapsedTime(&el, r.a, r.b);
    t.pms[r.stage] += el;
    t.pn[r.stage] += 1;
    t.pool.push_back(r.a);
    t.pool.push_back(r.b);
  }
  t.path_pending.clear();
  for (int i = 0; i < RRG_N_PATHS; ++i) {
    if (ms) ms[i] = t.pms[i];
    if (count) count[i] = t.pn[i];
    t.pms[i] = 0;
    t.pn[i] = 0;
  }
  return RRG_OK;
}
int rrg_ground_truth(const float* corpus, int64_t m, int32_t dim, const float* queries, int64_t nq,
                     int32_t k, int32_t metric, int64_t* ids, void* stream) {
  return guarded([&] {
    ground_truth_impl(corpus, m, dim, queries, nq, k, metric, ids, static_cast<cudaStream_t>(stream));
    return RRG_OK;
  });
}

const char* rrg_last_error(void) { return g_err.c_str(); }
const char* rrg_last_error_kind(void) { return g_kind.c_str(); }
const char* rrg_version(void) { return "rrg 0.1.0 (sm_100a)"; }

}  // extern "C"
