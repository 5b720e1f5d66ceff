// FFMA operand-form throughput probe: shared-memory vs uniform (kernel-param) W.
#include <cstdio>
#include <cuda_runtime.h>
struct WP { float w[1024]; };
constexpr int NA = 16;
__global__ void k_smem(float *out, int iters, const float *wg) {
  __shared__ float ws[1024];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) ws[i] = wg[i];
  __syncthreads();
  float acc[NA], x[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) { acc[i] = 0.f; x[i] = threadIdx.x * 0.001f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int k = 0; k < 1024; ++k) {
      const float w = ws[k];
#pragma unroll
      for (int i = 0; i < NA; ++i) acc[i] = fmaf(x[i], w, acc[i]);
    }
  }
  float s = 0; for (int i = 0; i < NA; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
__global__ void k_param(float *out, int iters, const __grid_constant__ WP p) {
  float acc[NA], x[NA];
#pragma unroll
  for (int i = 0; i < NA; ++i) { acc[i] = 0.f; x[i] = threadIdx.x * 0.001f + i; }
  for (int it = 0; it < iters; ++it) {
#pragma unroll 8
    for (int k = 0; k < 1024; ++k) {
      const float w = p.w[k];
#pragma unroll
      for (int i = 0; i < NA; ++i) acc[i] = fmaf(x[i], w, acc[i]);
    }
  }
  float s = 0; for (int i = 0; i < NA; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
// register W: 8 distinct w in registers, reused
__global__ void k_reg(float *out, int iters, const float *wg) {
  float acc[NA], x[NA], w[8];
#pragma unroll
  for (int i = 0; i < NA; ++i) { acc[i] = 0.f; x[i] = threadIdx.x * 0.001f + i; }
#pragma unroll
  for (int j = 0; j < 8; ++j) w[j] = wg[j + (threadIdx.x & 1)];
  for (int it = 0; it < iters * 128; ++it) {
#pragma unroll
    for (int j = 0; j < 8; ++j)
#pragma unroll
      for (int i = 0; i < NA; ++i) acc[i] = fmaf(x[i], w[j], acc[i]);
  }
  float s = 0; for (int i = 0; i < NA; ++i) s += acc[i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float *out, *wg;
  const int blocks = 148 * 8, threads = 256, iters = 20;
  cudaMalloc(&out, blocks * threads * 4);
  cudaMalloc(&wg, 1024 * 4);
  cudaMemset(wg, 0, 4096);
  WP p{};
  for (int i = 0; i < 1024; ++i) p.w[i] = 1e-3f * i;
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  const double flops = 2.0 * blocks * threads * double(iters) * 1024 * NA;
  for (int kind = 0; kind < 3; ++kind) {
    for (int rep = 0; rep < 3; ++rep) {
      cudaEventRecord(a);
      if (kind == 0) k_smem<<<blocks, threads>>>(out, iters, wg);
      if (kind == 1) k_param<<<blocks, threads>>>(out, iters, p);
      if (kind == 2) k_reg<<<blocks, threads>>>(out, iters, wg);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms; cudaEventElapsedTime(&ms, a, b);
      if (rep == 2) printf("%s: %.3f ms  %.1f TFLOP/s\n", kind == 0 ? "smem-broadcast W" : kind == 1 ? "param (uniform) W" : "register W", ms, flops / ms / 1e9);
    }
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
