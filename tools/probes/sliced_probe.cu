// Probe: the sliced int8 tcgen05 GEMM vs a CPU f64 reference, and its speed.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -Iinclude tools/sliced_probe.cu -o /tmp/sp
#include "../paper_2410_18926_b200/csrc/rrg_sliced_gemm.cu"

#include <cmath>
#include <cstdio>
#include <random>
#include <vector>

using namespace rrg;
void rrg::note_launch() {}  // the library's launch counter (rrg_api.cu) is not linked here

static double run(int M, int N, int K, bool check, int reps) {
  std::mt19937 gen(M + N + K);
  std::normal_distribution<float> nd(0.f, 1.f);
  std::vector<float> a((size_t)M * K), b((size_t)N * K);
  for (auto& v : a) v = nd(gen) * 6.f;
  for (auto& v : b) v = nd(gen) * 0.05f;
  for (int i = 0; i < M; i += 7) a[(size_t)i * K + 3] = 0.f;         // zeros
  for (int i = 0; i < M; i += 11) a[(size_t)i * K + 5] *= 1e-6f;     // tiny entries
  if (M > 2) for (int k = 0; k < K; ++k) a[(size_t)2 * K + k] = 0.f;  // all-zero row
  float *da, *db;
  double* dout;
  int8_t *pa, *pb;
  int *ea, *eb;

  cudaMalloc(&da, a.size() * 4); cudaMalloc(&db, b.size() * 4);
  cudaMalloc(&pa, sliced_plane_bytes(M, K, true)); cudaMalloc(&pb, sliced_plane_bytes(N, K, false));
  cudaMalloc(&ea, sliced_rows_pad(M, true) * 4); cudaMalloc(&eb, sliced_rows_pad(N, false) * 4);
  cudaMalloc(&dout, (size_t)M * N * 8);
  cudaMemcpy(da, a.data(), a.size() * 4, cudaMemcpyHostToDevice);
  cudaMemcpy(db, b.data(), b.size() * 4, cudaMemcpyHostToDevice);
  launch_slice_rows(da, M, K, K, true, pa, ea, 0);
  launch_slice_rows(db, N, K, K, false, pb, eb, 0);
  launch_gemm_sliced(pa, ea, M, pb, eb, N, K, EPI_NEGIP, nullptr, dout, N, nullptr, nullptr, 0);
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) { printf("CUDA error %s\n", cudaGetErrorString(e)); exit(1); }
  if (check) {
    std::vector<double> out((size_t)M * N);
    cudaMemcpy(out.data(), dout, out.size() * 8, cudaMemcpyDeviceToHost);
    double maxrel = 0, maxabs = 0;
    long bad = 0;
    for (int i = 0; i < M; ++i)
      for (int j = 0; j < N; ++j) {
        double s = 0, sa = 0;
        for (int k = 0; k < K; ++k) {
          const double p = (double)a[(size_t)i * K + k] * (double)b[(size_t)j * K + k];
          s += p; sa += fabs(p);
        }
        const double g = -out[(size_t)i * N + j];
        const double err = fabs(g - s);
        maxabs = fmax(maxabs, err);
        if (sa > 0) maxrel = fmax(maxrel, err / sa);
        if ((float)g != (float)s) ++bad;
      }
    printf("M=%d N=%d K=%d  max |err|/sum|p| = %.3e  max abs %.3e  f32-rounding mismatches %ld/%ld\n",
           M, N, K, maxrel, maxabs, bad, (long)M * N);
  }
  cudaEvent_t t0, t1;
  cudaEventCreate(&t0); cudaEventCreate(&t1);
  cudaEventRecord(t0);
  for (int r = 0; r < reps; ++r) {
    launch_slice_rows(da, M, K, K, true, pa, ea, 0);
    launch_gemm_sliced(pa, ea, M, pb, eb, N, K, EPI_NEGIP, nullptr, dout, N, nullptr, nullptr, 0);
  }
  cudaEventRecord(t1); cudaEventSynchronize(t1);
  float ms; cudaEventElapsedTime(&ms, t0, t1);
  cudaFree(da); cudaFree(db); cudaFree(pa); cudaFree(pb); cudaFree(ea); cudaFree(eb); cudaFree(dout);
  return ms / reps;
}

static void time_parts(int M, int N, int K) {
  float *da, *db; double* dout; int8_t *pa, *pb; int *ea, *eb;
  cudaMalloc(&da, (size_t)M * K * 4); cudaMalloc(&db, (size_t)N * K * 4);
  cudaMemset(da, 0, (size_t)M * K * 4); cudaMemset(db, 0, (size_t)N * K * 4);
  cudaMalloc(&pa, sliced_plane_bytes(M, K, true)); cudaMalloc(&pb, sliced_plane_bytes(N, K, false));
  cudaMalloc(&ea, sliced_rows_pad(M, true) * 4); cudaMalloc(&eb, sliced_rows_pad(N, false) * 4);
  cudaMalloc(&dout, (size_t)M * N * 8);
  launch_slice_rows(db, N, K, K, false, pb, eb, 0);
  cudaEvent_t t0, t1, t2; cudaEventCreate(&t0); cudaEventCreate(&t1); cudaEventCreate(&t2);
  launch_slice_rows(da, M, K, K, true, pa, ea, 0);
  launch_gemm_sliced(pa, ea, M, pb, eb, N, K, EPI_NEGIP, nullptr, dout, N, nullptr, nullptr, 0);
  cudaEventRecord(t0);
  for (int r = 0; r < 10; ++r) launch_slice_rows(da, M, K, K, true, pa, ea, 0);
  cudaEventRecord(t1);
  for (int r = 0; r < 10; ++r)
    launch_gemm_sliced(pa, ea, M, pb, eb, N, K, EPI_NEGIP, nullptr, dout, N, nullptr, nullptr, 0);
  cudaEventRecord(t2); cudaEventSynchronize(t2);
  float a, b; cudaEventElapsedTime(&a, t0, t1); cudaEventElapsedTime(&b, t1, t2);
  const double mac = (double)M * N * K * 36;
  printf("M=%d N=%d K=%d: slice %.3f ms, gemm %.3f ms (%.2f P slice-MAC/s)\n", M, N, K, a / 10, b / 10,
         mac / (b / 10 * 1e-3) / 1e15);
  cudaFree(da); cudaFree(db); cudaFree(pa); cudaFree(pb); cudaFree(ea); cudaFree(eb); cudaFree(dout);
}

int main() {
  time_parts(10000, 256, 768);
  time_parts(10000, 1024, 256);
  time_parts(148 * 128, 64, 8192);
  time_parts(148 * 128, 64, 256);
  run(300, 64, 64, true, 1);
  run(517, 200, 768, true, 1);
  run(1000, 1024, 256, true, 1);
  printf("proj  10000x256x768: %.3f ms (slice + gemm)\n", run(10000, 256, 768, false, 20));
  printf("route 10000x1024x256: %.3f ms (slice + gemm)\n", run(10000, 1024, 256, false, 20));
  return 0;
}
