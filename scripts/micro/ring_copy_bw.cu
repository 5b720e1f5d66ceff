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

// cp.async with a plane pattern: stage = 16 KiB = P planes x (16K / P) contiguous bytes;
// plane j of chunk c at c * (16K / P) + j * pstride (chunk index wraps within a plane).
template <int LAG>
__global__ void __launch_bounds__(256, 1) k_cpasync_planes(const char *X, char *O, int64_t nchunks,
                                                           int P, int64_t pstride) {
  extern __shared__ __align__(1024) char sm[];
  const int t = threadIdx.x;
  const int per = 16384 / P;
  int g = 0;
  for (int64_t c = blockIdx.x;; c += gridDim.x, ++g) {
    const bool valid = c < nchunks;
    const int s = g % (LAG + 1);
    if (valid) {
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int off = (t + 256 * u) * 16;  // byte in stage
        const int j = off / per, w = off % per;
        const int64_t src = (c * per) % pstride + int64_t(j) * pstride + w;
        asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(su32(sm + s * 16384 + off)),
                     "l"(X + src)
                     : "memory");
      }
    }
    asm volatile("cp.async.commit_group;" ::: "memory");
    asm volatile("cp.async.wait_group %0;" ::"n"(LAG) : "memory");
    const int64_t cp = c - int64_t(LAG) * gridDim.x;
    if (g >= LAG && cp < nchunks) {
      const int sp = (g - LAG) % (LAG + 1);
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const float4 v = *reinterpret_cast<const float4 *>(sm + sp * 16384 + (t + 256 * u) * 16);
        __stcs(reinterpret_cast<float4 *>(O + cp * 16384 + (t + 256 * u) * 16), v);
      }
    }
    if (!valid && c - int64_t(LAG) * gridDim.x >= nchunks) break;
  }
}

// Read-only TMA ring: 5-D boxes (dims/box/strides from the host), NS stages; one thread
// issues, waits, re-issues (the data is discarded).
__global__ void __launch_bounds__(32, 1) k_tma_read(const __grid_constant__ CUtensorMap map,
                                                   int64_t nbox, int bytes, int NS, int d1n,
                                                   int d2n, int d3n, int bx1, int bx2, int bx3) {
  extern __shared__ __align__(1024) char sm[];
  __shared__ uint64_t full[16];
  if (threadIdx.x != 0) return;
  for (int s = 0; s < NS; ++s) bar_init(&full[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  const int64_t b0 = nbox * blockIdx.x / gridDim.x, b1 = nbox * (blockIdx.x + 1) / gridDim.x;
  auto issue = [&](int64_t b, int s) {
    // box index -> coordinates of dims 1..3 (outer extents d1n, d2n, d3n boxes)
    // boxes iterate over dims 3 (fast) and 4; dims 1, 2 lie inside the box
    int c1 = 0, c2 = 0, c3 = int(b % d3n) * bx3, c4 = int(b / d3n);
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(&full[s])),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.5d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6, %7}], [%2];" ::"r"(su32(sm + s * bytes)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(su32(&full[s])), "r"(0), "r"(c1), "r"(c2),
        "r"(c3), "r"(c4)
        : "memory");
  };
  int g = 0;
  for (int64_t b = b0; b < b1 && g < NS; ++b, ++g) issue(b, g);
  for (int64_t b = b0, i = 0; b < b1; ++b, ++i) {
    const int s = int(i % NS);
    bar_wait(&full[s], (i / NS) & 1);
    if (b + NS < b1) issue(b + NS, s);
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
  cudaFuncSetAttribute(k_cpasync_planes<6>, cudaFuncAttributeMaxDynamicSharedMemorySize, 7 * 16384);
  const int64_t strides[] = {int64_t(1) << 19, int64_t(1) << 23, int64_t(1) << 27};
  for (int P : {1, 2, 8, 32})
    for (int64_t ps : strides) {
      char name[64];
      snprintf(name, sizeof name, "cp.async planes P=%d stride=2^%d", P, __builtin_ctzll(ps));
      // N bytes split over P planes of the region: chunk count so that P*per*n = N
      const int64_t nch = N / 16384;
      if (int64_t(P) * ps > N) continue;
      timeit(name, [&] { k_cpasync_planes<6><<<148, 256, 7 * 16384>>>(X, O, nch, P, ps); });
    }
  {
    // TMA read-only: X viewed as complex (8 B) array of 2^27; box = 128 B rows.
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
    using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                                  const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                                  const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                                  CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
    EncodeFn enc = reinterpret_cast<EncodeFn>(p);
    cudaFuncSetAttribute(k_tma_read, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024);
    struct Cfg {
      const char *name;
      int sw;  // 0 none, 1 128B_ATOM_32B
      cuuint64_t dims[5];
      cuuint64_t strides[4];  // bytes
      cuuint32_t box[5];
    };
    // 477-like: d0 = 32 floats (X bits 0..3), d1 = k bits 16,17 (4, stride 2^16 cx), d2 = k25
    // (2, stride 2^25 cx), d3 = m bits 4..15 (box 4 of 4096, stride 2^4 cx), d4 = m 18..24 etc.
    // all boxes 16 KiB (dims 0-2 in the box), iterated over dims 3 and 4; X = 1 GiB
    Cfg cfgs[] = {
        {"planes 2KiB x 8 @512K", 0, {32, 16, 8, 1u << 8, 1u << 8}, {128, 1u << 19, 2048, 1u << 22}, {32, 16, 8, 1, 1}},
        {"planes 2KiB x (4 @512K x 2 @256M)", 0, {32, 16, 4, 1u << 8, 1u << 7}, {128, 1u << 19, 2048, 1u << 21}, {32, 16, 4, 1, 1}},
        {"planes 4KiB x 2 @256M", 0, {32, 32, 2, 1u << 17, 2}, {128, 1u << 28, 4096, 1u << 29}, {32, 32, 2, 1, 1}},
        {"planes 4KiB x 2 @128M", 0, {32, 32, 2, 1u << 15, 4}, {128, 1u << 27, 4096, 1u << 28}, {32, 32, 2, 1, 1}},
        {"planes 4KiB x 2 @64M", 0, {32, 32, 2, 1u << 14, 8}, {128, 1u << 26, 4096, 1u << 27}, {32, 32, 2, 1, 1}},
        {"planes 8KiB x 2 @256M", 0, {32, 64, 2, 1u << 16, 2}, {128, 1u << 28, 8192, 1u << 29}, {32, 64, 2, 1, 1}},
    };
    for (auto &c : cfgs) {
      CUtensorMap map;
      cuuint32_t es[5] = {1, 1, 1, 1, 1};
      CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5, X, c.dims, c.strides, c.box, es,
                       CU_TENSOR_MAP_INTERLEAVE_NONE,
                       c.sw ? CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B : CU_TENSOR_MAP_SWIZZLE_NONE,
                       CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (r != CUDA_SUCCESS) {
        printf("%s: encode failed %d\n", c.name, int(r));
        continue;
      }
      const int bytes = int(c.box[0] * c.box[1] * c.box[2] * c.box[3] * c.box[4] * 4);
      // iterate over dims 3 (and 1, 2 beyond the box) with box-sized steps
      const int d1n = 1, d2n = 1, d3n = int(c.dims[3]);
      const int64_t nbox = int64_t(c.dims[3]) * c.dims[4];
      for (int ns : {4, 8, 12}) {
        if (ns * bytes > 200 * 1024) continue;
        cudaEventRecord(e0);
        for (int rr = 0; rr < 5; ++rr)
          k_tma_read<<<148, 32, ns * bytes>>>(map, nbox, bytes, ns, d1n, d2n, d3n, int(c.box[1]),
                                              int(c.box[2]), int(c.box[3]));
        cudaEventRecord(e1);
        cudaEventSynchronize(e1);
        float ms;
        cudaEventElapsedTime(&ms, e0, e1);
        cudaError_t err = cudaGetLastError();
        printf("%-36s NS=%2d box %6d B: read %6.0f GB/s %s\n", c.name, ns, bytes,
               double(nbox) * bytes * 5 / (ms * 1e-3) / 1e9, err == cudaSuccess ? "" : cudaGetErrorString(err));
      }
    }
  }
  return 0;
}
