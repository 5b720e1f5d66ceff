// Bandwidth of persistent smem-ring copy kernels on B200 (1 CTA per SM, 148 CTAs):
//   mode 0: cp.async.bulk 1-D loads of CH bytes into an NS-stage ring, bulk stores out
//   mode 1: cp.async 16-byte gathers by 256 threads (LAG groups in flight), STG.128 out
//   mode 2: 2-D TMA boxes of 128 B x ROWS rows (rows 'stride' bytes apart), bulk stores
// Each mode copies N bytes X -> O. Prints GB/s (read + write).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t su32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void bar_init(uint64_t *b, int c) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(c));
}
__device__ __forceinline__ void bar_wait(uint64_t *b, uint32_t ph) {
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(su32(b)), "r"(ph)
        : "memory");
}

template <int NS, int CH>
__global__ void __launch_bounds__(128, 1) k_bulk(const char *X, char *O, int64_t nchunks) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t full[NS];
  if (threadIdx.x == 0) {
    for (int s = 0; s < NS; ++s) bar_init(&full[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x != 0) return;
  int64_t i0 = blockIdx.x;
  int issued = 0;
  // prologue
  for (int s = 0; s < NS && i0 + int64_t(s) * gridDim.x < nchunks; ++s, ++issued) {
    const int64_t c = i0 + int64_t(s) * gridDim.x;
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                 "r"(CH)
                 : "memory");
    asm volatile(
        "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
            su32(sm + s * CH)),
        "l"(X + c * CH), "r"(CH), "r"(su32(&full[s]))
        : "memory");
  }
  for (int g = 0;; ++g) {
    const int64_t c = i0 + int64_t(g) * gridDim.x;
    if (c >= nchunks) break;
    const int s = g % NS;
    bar_wait(&full[s], (g / NS) & 1);
    asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(O + c * CH),
                 "r"(su32(sm + s * CH)), "r"(CH)
                 : "memory");
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    // reuse slot s for chunk g + NS once its store has read smem
    const int64_t cn = i0 + int64_t(g + NS) * gridDim.x;
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
    if (cn < nchunks) {
      asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                   "r"(CH)
                   : "memory");
      asm volatile(
          "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
              su32(sm + s * CH)),
          "l"(X + cn * CH), "r"(CH), "r"(su32(&full[s]))
          : "memory");
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <int LAG>
__global__ void __launch_bounds__(256, 1) k_cpasync(const char *X, char *O, int64_t nchunks) {
  // chunk = 4 KiB per stage (256 threads x 16 B); ring of LAG+1 stages
  extern __shared__ __align__(1024) char sm[];
  const int t = threadIdx.x;
  int g = 0;
  for (int64_t c = blockIdx.x;; c += gridDim.x, ++g) {
    const bool valid = c < nchunks;
    const int s = g % (LAG + 1);
    if (valid)
      asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + s * 4096 + t * 16)),
                   "l"(X + c * 4096 + t * 16)
                   : "memory");
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
    const int64_t cp = c - int64_t(LAG) * gridDim.x;
    if (g >= LAG && cp < nchunks) {
      const int sp = (g - LAG) % (LAG + 1);
      const float4 v = *reinterpret_cast<const float4 *>(sm + sp * 4096 + t * 16);
      __stcs(reinterpret_cast<float4 *>(O + cp * 4096 + t * 16), v);
    }
    if (!valid && c - int64_t(LAG) * gridDim.x >= nchunks) break;
  }
}

__global__ void k_ldg(const float4 *X, float4 *O, int64_t n) {
  for (int64_t i = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x)
    __stcs(O + i, __ldcs(X + i));
}

int main() {
  const int64_t N = int64_t(1) << 30;
  char *X, *O;
  cudaMalloc(&X, N);
  cudaMalloc(&O, N);
  cudaMemset(X, 1, N);
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto timeit = [&](const char *name, auto launch) {
    launch();
    cudaDeviceSynchronize();
    cudaEventRecord(e0);
    for (int r = 0; r < 5; ++r) launch();
    cudaEventRecord(e1);
    cudaEventSynchronize(e1);
    float ms;
    cudaEventElapsedTime(&ms, e0, e1);
    cudaError_t err = cudaGetLastError();
    printf("%-40s %8.0f GB/s %s\n", name, 2.0 * N * 5 / (ms * 1e-3) / 1e9,
           err == cudaSuccess ? "" : cudaGetErrorString(err));
  };
  timeit("ldg/stg grid-stride (148x8 x 256)", [&] {
    k_ldg<<<148 * 8, 256>>>(reinterpret_cast<const float4 *>(X), reinterpret_cast<float4 *>(O),
                            N / 16);
  });
#define BULK(NSV, CHV)                                                                       \
  {                                                                                          \
    cudaFuncSetAttribute(k_bulk<NSV, CHV>, cudaFuncAttributeMaxDynamicSharedMemorySize,      \
                         NSV * CHV);                                                         \
    timeit("bulk NS=" #NSV " CH=" #CHV, [&] {                                                \
      k_bulk<NSV, CHV><<<148, 128, NSV * CHV>>>(X, O, N / CHV);                              \
    });                                                                                      \
  }
  BULK(4, 16384) BULK(8, 16384) BULK(12, 16384) BULK(6, 32768) BULK(16, 8192) BULK(32, 4096)
#define CPA(LAGV)                                                                            \
  {                                                                                          \
    cudaFuncSetAttribute(k_cpasync<LAGV>, cudaFuncAttributeMaxDynamicSharedMemorySize,       \
                         (LAGV + 1) * 4096);                                                 \
    timeit("cp.async LAG=" #LAGV, [&] {                                                      \
      k_cpasync<LAGV><<<148, 256, (LAGV + 1) * 4096>>>(X, O, N / 4096);                      \
    });                                                                                      \
  }
  CPA(4) CPA(8) CPA(16) CPA(32)
  return 0;
}
