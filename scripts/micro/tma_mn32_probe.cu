// Probe: does a multi-dimensional TMA box with CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B land
// in shared memory as the UMMA MN-major SWIZZLE_128B_BASE32B layout (dense box order,
// 32-byte chunk c of 128-byte row r stored at chunk c ^ (r & 3))? Tests a 128-byte inner
// box and a 32-byte inner box (MN row assembled from two dims).
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <vector>

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__global__ void k_load(const __grid_constant__ CUtensorMap map, int bytes, int c1, int c2,
                       float *out) {
  __shared__ __align__(1024) unsigned char buf[16384];
  __shared__ uint64_t bar;
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_u32(&bar)));
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(&bar)),
                 "r"(bytes)
                 : "memory");
    asm volatile(
        "cp.async.bulk.tensor.4d.shared::cluster.global.mbarrier::complete_tx::bytes"
        " [%0], [%1, {%3, %4, %5, %6}], [%2];" ::"r"(smem_u32(buf)),
        "l"(reinterpret_cast<uint64_t>(&map)), "r"(smem_u32(&bar)), "r"(0), "r"(c1), "r"(c2),
        "r"(0)
        : "memory");
  }
  uint32_t done = 0;
  while (!done)
    asm volatile(
        "{\n\t.reg .pred p;\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%1], 0;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_u32(&bar))
        : "memory");
  for (int i = threadIdx.x; i < bytes / 4; i += blockDim.x)
    out[i] = reinterpret_cast<const float *>(buf)[i];
}

using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main() {
  void *p = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q);
  EncodeFn enc = reinterpret_cast<EncodeFn>(p);
  const size_t n = size_t(1) << 22;  // floats
  std::vector<float> h(n);
  for (size_t i = 0; i < n; ++i) h[i] = float(i);
  float *dx, *dout;
  cudaMalloc(&dx, n * 4);
  cudaMalloc(&dout, 16384);
  cudaMemcpy(dx, h.data(), n * 4, cudaMemcpyHostToDevice);
  std::vector<float> got(4096);
  // Case A: inner 32 floats (stride 1), d1 = "k" 8 rows at stride 4096 floats,
  //         d2 = 4 "MN atoms" at stride 32 floats, d3 = 1.
  // Case B: inner 8 floats, d1 = 4 at stride 64 floats (MN row = 32 floats from 2 dims),
  //         d2 = 8 "k" rows at stride 4096 floats, d3 = 4 MN atoms at stride 512 floats.
  for (int cs = 0; cs < 2; ++cs) {
    CUtensorMap map;
    cuuint64_t dims[4], strides[3];
    cuuint32_t box[4], es[4] = {1, 1, 1, 1};
    if (cs == 0) {
      cuuint64_t d[4] = {32, 8, 4, 1}, s[3] = {4096 * 4, 32 * 4, 1 << 20};
      cuuint32_t b[4] = {32, 8, 4, 1};
      for (int i = 0; i < 4; ++i) dims[i] = d[i], box[i] = b[i];
      for (int i = 0; i < 3; ++i) strides[i] = s[i];
    } else {
      cuuint64_t d[4] = {8, 4, 8, 4}, s[3] = {64 * 4, 4096 * 4, 512 * 4};
      cuuint32_t b[4] = {8, 4, 8, 4};
      for (int i = 0; i < 4; ++i) dims[i] = d[i], box[i] = b[i];
      for (int i = 0; i < 3; ++i) strides[i] = s[i];
    }
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 4, dx, dims, strides, box, es,
                     CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B,
                     CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) {
      printf("case %d: encode failed %d\n", cs, int(r));
      continue;
    }
    const int bytes = 32 * 8 * 4 * 4;
    k_load<<<1, 128>>>(map, bytes, 0, 0, dout);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) {
      printf("case %d: %s\n", cs, cudaGetErrorString(e));
      return 1;
    }
    cudaMemcpy(got.data(), dout, bytes, cudaMemcpyDeviceToHost);
    // expected: MN index mn (0..127), k (0..7): source float index
    int bad = 0, bad_dense = 0;
    for (int mn = 0; mn < 128; ++mn)
      for (int k = 0; k < 8; ++k) {
        size_t src;
        if (cs == 0)
          src = size_t(mn & 31) + size_t(k) * 4096 + size_t(mn >> 5) * 32;
        else
          src = size_t(mn & 7) + size_t((mn >> 3) & 3) * 64 + size_t(k) * 4096 +
                size_t(mn >> 5) * 512;
        // dense box order: [mn atom][k][32 floats]; row = k + 8 * atom
        const int row = k + 8 * (mn >> 5);
        const int dense = row * 32 + (mn & 31);
        const int chunk = ((mn & 31) >> 3) ^ (row & 3);
        const int sw = row * 32 + chunk * 8 + (mn & 7);
        bad += got[sw] != float(src);
        bad_dense += got[dense] != float(src);
      }
    printf("case %d (%s inner): swizzled-32B mismatches %d/1024, dense mismatches %d/1024\n", cs,
           cs == 0 ? "128B" : "32B", bad, bad_dense);
  }
  return 0;
}
