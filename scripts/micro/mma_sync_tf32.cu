// Throughput probe: legacy warp-level mma.sync tf32 (m16n8k8) on sm_100a.
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k_mma(float *out, int iters) {
  unsigned a[4], b[2];
  float c[8][4];
  for (int i = 0; i < 4; ++i) a[i] = __float_as_uint(1.0f + threadIdx.x * 1e-3f + i);
  for (int i = 0; i < 2; ++i) b[i] = __float_as_uint(0.5f + i);
  for (int t = 0; t < 8; ++t)
    for (int i = 0; i < 4; ++i) c[t][i] = 0.f;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int t = 0; t < 8; ++t)
      asm volatile(
          "mma.sync.aligned.m16n8k8.row.col.f32.tf32.tf32.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, "
          "{%8,%9}, {%0,%1,%2,%3};"
          : "+f"(c[t][0]), "+f"(c[t][1]), "+f"(c[t][2]), "+f"(c[t][3])
          : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b[0]), "r"(b[1]));
  }
  float s = 0;
  for (int t = 0; t < 8; ++t)
    for (int i = 0; i < 4; ++i) s += c[t][i];
  out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}
int main() {
  float *out;
  const int blocks = 148 * 4, threads = 256, iters = 4096;
  cudaMalloc(&out, blocks * threads * 4);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  for (int rep = 0; rep < 3; ++rep) {
    cudaEventRecord(a);
    k_mma<<<blocks, threads>>>(out, iters);
    cudaEventRecord(b);
    cudaEventSynchronize(b);
    float ms; cudaEventElapsedTime(&ms, a, b);
    const double flops = 2.0 * 16 * 8 * 8 * 8 * double(iters) * blocks * (threads / 32);
    if (rep == 2) printf("mma.sync tf32 m16n8k8: %.3f ms  %.1f TFLOP/s\n", ms, flops / ms / 1e9);
  }
  printf("err=%s\n", cudaGetErrorString(cudaGetLastError()));
}
