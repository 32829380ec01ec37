// Micro-probe: FP32 pipe throughput of scalar FADD vs packed FADD2/FFMA2 vs a mix
// (which SASS pipes the packed forms use on sm_100a).  nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>
constexpr int N = 4096;
__global__ void k_scalar(float* out, float a) {
  float r[16];
  for (int j = 0; j < 16; ++j) r[j] = threadIdx.x + j;
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < 16; ++j) r[j] = __fadd_rn(r[j], a);
  float s = 0; for (int j = 0; j < 16; ++j) s += r[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_packed(float* out, float a) {
  float2 r[8]; const float2 aa = make_float2(a, a);
  for (int j = 0; j < 8; ++j) r[j] = make_float2(threadIdx.x + j, j);
  for (int i = 0; i < N; ++i)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __fadd2_rn(r[j], aa);
  float s = 0; for (int j = 0; j < 8; ++j) s += r[j].x + r[j].y;
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_mix(float* out, float a) {  // 2/3 of lane-ops packed, 1/3 scalar
  float2 r[4]; float q[8]; const float2 aa = make_float2(a, a);
  for (int j = 0; j < 4; ++j) r[j] = make_float2(threadIdx.x + j, j);
  for (int j = 0; j < 8; ++j) q[j] = j;
  for (int i = 0; i < N; ++i) {
#pragma unroll
    for (int j = 0; j < 4; ++j) r[j] = __fadd2_rn(r[j], aa);
#pragma unroll
    for (int j = 0; j < 4; ++j) q[j] = __fadd_rn(q[j], a);
  }
  float s = 0; for (int j = 0; j < 4; ++j) s += r[j].x + r[j].y + q[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
template <typename K> void run(const char* name, K k, int lane_ops_per_iter) {
  float* out; cudaMalloc(&out, 148 * 8 * 1024 * 4);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  k<<<148 * 8, 256>>>(out, 1e-7f);
  cudaEventRecord(e0);
  for (int r = 0; r < 5; ++r) k<<<148 * 8, 256>>>(out, 1e-7f);
  cudaEventRecord(e1); cudaEventSynchronize(e1);
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  double ops = 5.0 * 148 * 8 * 256 * (double)N * lane_ops_per_iter;
  printf("%-8s %.3f ms  %.1f T lane-ops/s\n", name, ms, ops / ms / 1e9);
  cudaFree(out);
}
int main() {
  run("scalar", k_scalar, 16);
  run("packed", k_packed, 16);
  run("mix", k_mix, 12);
  return 0;
}
