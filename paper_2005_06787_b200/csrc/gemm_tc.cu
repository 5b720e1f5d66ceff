// tcgen05 split-TF32 ("3xTF32") complex GEMM for sm_100a.
//
//   C[z] (M x N complex) = A[z] (M x K complex, row-major) * B[z] (K x N complex, row-major)
//
// Complex -> real: with interleaved storage, A is an M x 2K real matrix that is
// already K-major. B becomes the 2N x 2K K-major real matrix
//   B''[2n+t][2k+s] = [[br, -bi], [bi, br]][t][s]
// so that C (M x 2N real, i.e. interleaved complex) = A . B''^T: 4 real MACs per
// complex MAC, like the 4M decomposition, in one real GEMM.
//
// Split-TF32: x = hi + lo with hi = tf32(x) (round to nearest) and lo = x - hi;
// C ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi, accumulated in fp32 in TMEM. The dropped
// Alo.Blo term is ~2^-22 relative, so results carry fp32-level accuracy.
//
// Kernel anatomy (one CTA per 128 x 128 real output tile):
//   warp 0      TMA producer: A hi/lo (128 x 32) and B'' hi/lo (128 x 32) tiles,
//               SWIZZLE_128B, three-stage mbarrier ring
//   warp 1      MMA issuer: 3 x 4 tcgen05.mma.kind::tf32 (128x128x8) per stage
//               into one of two TMEM buffers (hi*hi chain + correction chain);
//               tcgen05.commit frees the stage / hands a finished K chunk over
//   warps 2..5  epilogue: tcgen05.ld 32x32b.x32 of each K chunk, fp32 RN
//               accumulation in registers, then one row per thread to global
// The operand splits (A hi/lo, B'' hi/lo) are produced by two bandwidth-bound
// pre-pass kernels into a workspace.
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.h"

namespace stn {

namespace {

constexpr int BM = 128;        // rows of C per CTA (UMMA M)
constexpr int BN = 128;        // real columns of C per CTA (UMMA N)
constexpr int BK = 32;         // real K per stage (128 B rows -> SWIZZLE_128B)
constexpr int UK = 8;          // real K per tcgen05.mma (32 B of tf32)
constexpr int STAGES = 3;
constexpr int CHUNK = 8;       // k-blocks accumulated in TMEM before an fp32 RN flush
constexpr int A_TILE_BYTES = BM * BK * 4;  // 16 KiB
constexpr int B_TILE_BYTES = BN * BK * 4;  // 32 KiB
constexpr int STAGE_BYTES = 2 * A_TILE_BYTES + 2 * B_TILE_BYTES;
constexpr int THREADS = 192;
constexpr int TMEM_COLS = 512;  // 2 buffers x {hi*hi chain, hi*lo + lo*hi corrections} x BN
constexpr size_t SMEM_BYTES = size_t(STAGES) * STAGE_BYTES + 1024 /*align*/ + 256 /*barriers*/;

// ---- PTX wrappers -------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}

__device__ __forceinline__ void mbar_expect_tx(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)),
               "r"(bytes)
               : "memory");
}

// Bounded wait: a barrier that never completes traps (~60 s of clock: far beyond any
// legitimate wait, preemption included) instead of hanging the GPU.
__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t parity) {
  const uint32_t addr = smem_u32(bar);
  uint32_t done = 0;
  long long start = 0;
  for (int iter = 0;; ++iter) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(addr), "r"(parity)
        : "memory");
    if (done) return;
    if (iter == 0) start = clock64();
    if ((iter & 1023) == 1023 && clock64() - start > (120ll << 30)) __trap();
  }
}

__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}

__device__ __forceinline__ void tma_load_3d(void *dst, const CUtensorMap *map, uint64_t *bar,
                                            int x, int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}

__device__ __forceinline__ void umma_commit(uint64_t *bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
                   smem_u32(bar))
               : "memory");
}

__device__ __forceinline__ void umma_tf32(uint32_t tmem_d, uint64_t adesc, uint64_t bdesc,
                                          uint32_t idesc, uint32_t accumulate) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], %1, %2, %3, p;\n\t}" ::"r"(tmem_d),
      "l"(adesc), "l"(bdesc), "r"(idesc), "r"(accumulate));
}

__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}

// 32 lanes x 32 columns of fp32 from TMEM (one row per thread).
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32"
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15,"
      " %16, %17, %18, %19, %20, %21, %22, %23, %24, %25, %26, %27, %28, %29, %30, %31},"
      " [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15]), "=r"(v[16]), "=r"(v[17]), "=r"(v[18]), "=r"(v[19]),
        "=r"(v[20]), "=r"(v[21]), "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]),
        "=r"(v[26]), "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
}

// K-major SWIZZLE_128B shared-memory matrix descriptor (sm_100 "version 1").
// 8-row x 128 B swizzle atoms stacked every 1024 B (SBO); LBO unused.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;            // LBO (ignored for swizzled K-major)
  d |= uint64_t(1024 >> 4) << 32;    // SBO
  d |= uint64_t(1) << 46;            // descriptor version (Blackwell)
  d |= uint64_t(2) << 61;            // SWIZZLE_128B
  return d;
}

// kind::tf32 instruction descriptor: F32 accumulate, TF32 A/B, both K-major.
constexpr uint32_t kIdesc = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN >> 3) << 17) |
                            (uint32_t(BM >> 4) << 24);

__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// ---- the GEMM kernel ----------------------------------------------------------
struct TcArgs {
  float *c;          // C base (complex interleaved -> M x 2N floats per batch)
  int64_t c_bs;      // floats between slices
  int64_t c_ds;      // floats between D batches
  int D;
  int a_batched, b_batched;  // operand varies per slice
  int k_blocks;      // 2K / BK
  int two_n;         // 2N (row stride of C in floats)
  int n_tiles;       // 2N / BN
  int m_groups;      // M / BM / cluster size (k_gemm_tc256m)
  int gm;            // cluster m groups per raster band (k_gemm_tc256m)
};

__global__ void __launch_bounds__(THREADS, 1)
    k_gemm_tc(const __grid_constant__ CUtensorMap map_ahi, const __grid_constant__ CUtensorMap map_alo,
              const __grid_constant__ CUtensorMap map_bhi, const __grid_constant__ CUtensorMap map_blo,
              const TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES * STAGE_BYTES);
  uint64_t *empty = full + STAGES;
  uint64_t *tmem_full = empty + STAGES;   // [2]: chunk accumulated in TMEM buffer b
  uint64_t *tmem_empty = tmem_full + 2;   // [2]: epilogue drained TMEM buffer b
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x % args.n_tiles, m_tile = blockIdx.x / args.n_tiles;
  const int bz = blockIdx.z;
  const int slice = bz / args.D, d = bz % args.D;
  const int za = args.a_batched ? bz : d;
  const int zb = args.b_batched ? bz : d;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 4);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      // ---- TMA producer ----
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        mbar_wait(&empty[s], phase ^ 1);
        unsigned char *st = smem + s * STAGE_BYTES;
        mbar_expect_tx(&full[s], STAGE_BYTES);
        const int kx = kb * BK;
        tma_load_3d(st, &map_ahi, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + A_TILE_BYTES, &map_alo, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + 2 * A_TILE_BYTES, &map_bhi, &full[s], kx, n_tile * BN, zb);
        tma_load_3d(st + 2 * A_TILE_BYTES + B_TILE_BYTES, &map_blo, &full[s], kx, n_tile * BN, zb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      // ---- MMA issuer ----
      // K is accumulated in chunks of CHUNK k-blocks, alternating between two
      // TMEM buffers; the epilogue adds each finished chunk into fp32
      // registers with round-to-nearest, so long K chains do not accumulate the
      // tensor core's truncating adds.
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES;
        const uint32_t phase = (kb / STAGES) & 1;
        const int chunk = kb / CHUNK, buf = chunk & 1;
        const bool chunk_first = kb % CHUNK == 0;
        const bool chunk_last = kb % CHUNK == CHUNK - 1 || kb == args.k_blocks - 1;
        if (chunk_first) {
          mbar_wait(&tmem_empty[buf], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * STAGE_BYTES);
        const uint64_t ahi = smem_desc_sw128(st);
        const uint64_t alo = smem_desc_sw128(st + A_TILE_BYTES);
        const uint64_t bhi = smem_desc_sw128(st + 2 * A_TILE_BYTES);
        const uint64_t blo = smem_desc_sw128(st + 2 * A_TILE_BYTES + B_TILE_BYTES);
        const uint32_t tmain = tmem_base + uint32_t(buf * 2 * BN), tcorr = tmain + BN;
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          const uint64_t koff = uint64_t((k * UK * 4) >> 4);  // +32 B per K step
          const uint32_t acc0 = (!chunk_first || k > 0) ? 1u : 0u;
          // the small correction products get their own accumulator so their
          // additions do not round the large hi*hi partial sums
          umma_tf32(tmain, ahi + koff, bhi + koff, kIdesc, acc0);
          umma_tf32(tcorr, ahi + koff, blo + koff, kIdesc, acc0);
          umma_tf32(tcorr, alo + koff, bhi + koff, kIdesc, 1u);
        }
        umma_commit(&empty[s]);
        if (chunk_last) umma_commit(&tmem_full[buf]);
      }
    }
  } else {
    // ---- epilogue: drain TMEM chunks into fp32 registers, then global ----
    const int lane_base = 32 * (warp % 4);
    const int row = m_tile * BM + lane_base + lane;
    float acc[BN];
#pragma unroll
    for (int c = 0; c < BN; ++c) acc[c] = 0.f;
    const int n_chunks = (args.k_blocks + CHUNK - 1) / CHUNK;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(&tmem_full[buf], (chunk >> 1) & 1);
      tc_fence_after();
      const uint32_t tmain = tmem_base + (uint32_t(lane_base) << 16) + uint32_t(buf * 2 * BN);
#pragma unroll
      for (int cc = 0; cc < 2 * BN / 32; ++cc) {  // main columns, then corrections
        uint32_t v[32];
        tmem_ld32(tmain + uint32_t(cc * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        const int c0 = (cc * 32) % BN;
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[c0 + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
    }
    float *crow = args.c + int64_t(slice) * args.c_bs + int64_t(d) * args.c_ds +
                  int64_t(row) * args.two_n + int64_t(n_tile) * BN;
#pragma unroll
    for (int q = 0; q < BN / 4; ++q)
      reinterpret_cast<float4 *>(crow)[q] =
          make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(TMEM_COLS));
  }
}

// ---- 128 x 256 tiles -------------------------------------------------------------
// Same pipeline with UMMA N = 256: every A byte fetched from L2 now feeds twice the
// MMA work (the 128 x 128 kernel is bound by L2 -> SM operand traffic: 64 KiB per
// 810-cycle k-block). The three split-TF32 products go into ONE fp32 TMEM accumulator
// (256 columns; two buffers for the chunked round-to-nearest flush), two stages of
// 96 KiB, and 8 epilogue warps (two per TMEM lane quadrant, 128 columns each).
constexpr int BN2 = 256;
constexpr int STAGES2 = 2;
constexpr int B2_TILE_BYTES = BN2 * BK * 4;  // 32 KiB
constexpr int STAGE2_BYTES = 2 * A_TILE_BYTES + 2 * B2_TILE_BYTES;
constexpr int THREADS2 = 320;
constexpr size_t SMEM2_BYTES = size_t(STAGES2) * STAGE2_BYTES + 1024 + 256;
constexpr uint32_t kIdesc2 = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN2 >> 3) << 17) |
                             (uint32_t(BM >> 4) << 24);

__global__ void __launch_bounds__(THREADS2, 1)
    k_gemm_tc256(const __grid_constant__ CUtensorMap map_ahi,
                 const __grid_constant__ CUtensorMap map_alo,
                 const __grid_constant__ CUtensorMap map_bhi,
                 const __grid_constant__ CUtensorMap map_blo, const TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t *empty = full + STAGES2;
  uint64_t *tmem_full = empty + STAGES2;
  uint64_t *tmem_empty = tmem_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x % args.n_tiles, m_tile = blockIdx.x / args.n_tiles;
  const int bz = blockIdx.z;
  const int slice = bz / args.D, d = bz % args.D;
  const int za = args.a_batched ? bz : d;
  const int zb = args.b_batched ? bz : d;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 8);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES2;
        const uint32_t phase = (kb / STAGES2) & 1;
        mbar_wait(&empty[s], phase ^ 1);
        unsigned char *st = smem + s * STAGE2_BYTES;
        mbar_expect_tx(&full[s], STAGE2_BYTES);
        const int kx = kb * BK;
        tma_load_3d(st, &map_ahi, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + A_TILE_BYTES, &map_alo, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + 2 * A_TILE_BYTES, &map_bhi, &full[s], kx, n_tile * BN2, zb);
        tma_load_3d(st + 2 * A_TILE_BYTES + B2_TILE_BYTES, &map_blo, &full[s], kx, n_tile * BN2,
                    zb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES2;
        const uint32_t phase = (kb / STAGES2) & 1;
        const int chunk = kb / CHUNK, buf = chunk & 1;
        const bool chunk_first = kb % CHUNK == 0;
        const bool chunk_last = kb % CHUNK == CHUNK - 1 || kb == args.k_blocks - 1;
        if (chunk_first) {
          mbar_wait(&tmem_empty[buf], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * STAGE2_BYTES);
        const uint64_t ahi = smem_desc_sw128(st);
        const uint64_t alo = smem_desc_sw128(st + A_TILE_BYTES);
        const uint64_t bhi = smem_desc_sw128(st + 2 * A_TILE_BYTES);
        const uint64_t blo = smem_desc_sw128(st + 2 * A_TILE_BYTES + B2_TILE_BYTES);
        const uint32_t tacc = tmem_base + uint32_t(buf * BN2);
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          const uint64_t koff = uint64_t((k * UK * 4) >> 4);
          const uint32_t acc0 = (!chunk_first || k > 0) ? 1u : 0u;
          umma_tf32(tacc, ahi + koff, bhi + koff, kIdesc2, acc0);
          umma_tf32(tacc, ahi + koff, blo + koff, kIdesc2, 1u);
          umma_tf32(tacc, alo + koff, bhi + koff, kIdesc2, 1u);
        }
        umma_commit(&empty[s]);
        if (chunk_last) umma_commit(&tmem_full[buf]);
      }
    }
  } else {
    // ---- epilogue: warps 2..9; (warp % 4) = TMEM lane quadrant, half = 128-column half ----
    const int q4 = warp % 4, half = (warp - 2) / 4;
    const int lane_base = 32 * q4;
    const int row = m_tile * BM + lane_base + lane;
    float acc[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) acc[c] = 0.f;
    const int n_chunks = (args.k_blocks + CHUNK - 1) / CHUNK;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(&tmem_full[buf], (chunk >> 1) & 1);
      tc_fence_after();
      const uint32_t t0 =
          tmem_base + (uint32_t(lane_base) << 16) + uint32_t(buf * BN2 + 128 * half);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(t0 + uint32_t(cc * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[cc * 32 + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
    }
    float *crow = args.c + int64_t(slice) * args.c_bs + int64_t(d) * args.c_ds +
                  int64_t(row) * args.two_n + int64_t(n_tile) * BN2 + 128 * half;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      reinterpret_cast<float4 *>(crow)[q] =
          make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
  }
}

// ---- 128 x 256 tiles, BK = 16 (64-byte rows, SWIZZLE_64B), four stages ----------------
// The 128 x 256 kernel above holds two 96 KiB stages; a k-block's TMA latency is then
// barely covered by one stage of MMAs. Halving the stage (16 real K per stage, 64-byte
// rows) doubles the ring depth at the same shared memory; chunks stay 256 real K.
constexpr int BK3 = 16;
constexpr int STAGES3 = 4;
constexpr int CHUNK3 = 2 * CHUNK;
constexpr int A3_TILE_BYTES = BM * BK3 * 4;   // 8 KiB
constexpr int B3_TILE_BYTES = BN2 * BK3 * 4;  // 16 KiB
constexpr int STAGE3_BYTES = 2 * A3_TILE_BYTES + 2 * B3_TILE_BYTES;
constexpr size_t SMEM3_BYTES = size_t(STAGES3) * STAGE3_BYTES + 1024 + 256;

// K-major SWIZZLE_64B descriptor: 8-row x 64 B atoms every 512 B (SBO).
__device__ __forceinline__ uint64_t smem_desc_sw64(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;
  d |= uint64_t(512 >> 4) << 32;  // SBO
  d |= uint64_t(1) << 46;
  d |= uint64_t(4) << 61;         // SWIZZLE_64B
  return d;
}

__global__ void __launch_bounds__(THREADS2, 1)
    k_gemm_tc256s(const __grid_constant__ CUtensorMap map_ahi,
                 const __grid_constant__ CUtensorMap map_alo,
                 const __grid_constant__ CUtensorMap map_bhi,
                 const __grid_constant__ CUtensorMap map_blo, const TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES3 * STAGE3_BYTES);
  uint64_t *empty = full + STAGES3;
  uint64_t *tmem_full = empty + STAGES3;
  uint64_t *tmem_empty = tmem_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x % args.n_tiles, m_tile = blockIdx.x / args.n_tiles;
  const int bz = blockIdx.z;
  const int slice = bz / args.D, d = bz % args.D;
  const int za = args.a_batched ? bz : d;
  const int zb = args.b_batched ? bz : d;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES3; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 8);  // one arrive per epilogue warp
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES3;
        const uint32_t phase = (kb / STAGES3) & 1;
        mbar_wait(&empty[s], phase ^ 1);
        unsigned char *st = smem + s * STAGE3_BYTES;
        mbar_expect_tx(&full[s], STAGE3_BYTES);
        const int kx = kb * BK3;
        tma_load_3d(st, &map_ahi, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + A3_TILE_BYTES, &map_alo, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + 2 * A3_TILE_BYTES, &map_bhi, &full[s], kx, n_tile * BN2, zb);
        tma_load_3d(st + 2 * A3_TILE_BYTES + B3_TILE_BYTES, &map_blo, &full[s], kx, n_tile * BN2,
                    zb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES3;
        const uint32_t phase = (kb / STAGES3) & 1;
        const int chunk = kb / CHUNK3, buf = chunk & 1;
        const bool chunk_first = kb % CHUNK3 == 0;
        const bool chunk_last = kb % CHUNK3 == CHUNK3 - 1 || kb == args.k_blocks - 1;
        if (chunk_first) {
          mbar_wait(&tmem_empty[buf], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * STAGE3_BYTES);
        const uint64_t ahi = smem_desc_sw64(st);
        const uint64_t alo = smem_desc_sw64(st + A3_TILE_BYTES);
        const uint64_t bhi = smem_desc_sw64(st + 2 * A3_TILE_BYTES);
        const uint64_t blo = smem_desc_sw64(st + 2 * A3_TILE_BYTES + B3_TILE_BYTES);
        const uint32_t tacc = tmem_base + uint32_t(buf * BN2);
#pragma unroll
        for (int k = 0; k < BK3 / UK; ++k) {
          const uint64_t koff = uint64_t((k * UK * 4) >> 4);
          const uint32_t acc0 = (!chunk_first || k > 0) ? 1u : 0u;
          umma_tf32(tacc, ahi + koff, bhi + koff, kIdesc2, acc0);
          umma_tf32(tacc, ahi + koff, blo + koff, kIdesc2, 1u);
          umma_tf32(tacc, alo + koff, bhi + koff, kIdesc2, 1u);
        }
        umma_commit(&empty[s]);
        if (chunk_last) umma_commit(&tmem_full[buf]);
      }
    }
  } else {
    // ---- epilogue: warps 2..9; (warp % 4) = TMEM lane quadrant, half = 128-column half ----
    const int q4 = warp % 4, half = (warp - 2) / 4;
    const int lane_base = 32 * q4;
    const int row = m_tile * BM + lane_base + lane;
    float acc[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) acc[c] = 0.f;
    const int n_chunks = (args.k_blocks + CHUNK3 - 1) / CHUNK3;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(&tmem_full[buf], (chunk >> 1) & 1);
      tc_fence_after();
      const uint32_t t0 =
          tmem_base + (uint32_t(lane_base) << 16) + uint32_t(buf * BN2 + 128 * half);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(t0 + uint32_t(cc * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[cc * 32 + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
    }
    float *crow = args.c + int64_t(slice) * args.c_bs + int64_t(d) * args.c_ds +
                  int64_t(row) * args.two_n + int64_t(n_tile) * BN2 + 128 * half;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      reinterpret_cast<float4 *>(crow)[q] =
          make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
  }
}

// ---- 128 x 256 tiles, clusters of CL CTAs along M sharing the B tile ----------------
// The 128 x 256 kernel is bound by L2 -> SM operand traffic (96 KiB per k-block for
// ~1.5 M MACs). CL CTAs with consecutive m tiles and the same n tile form a cluster;
// each TMA-loads 1/CL of the B'' hi/lo tile and multicasts it into every CTA of the
// cluster, so a CTA pulls 32 KiB of A plus 64/CL KiB of B per k-block. A stage is
// written by every CTA of the cluster, so its "empty" barrier waits for the MMA
// commits of all CL CTAs (tcgen05.commit multicast).
__device__ __forceinline__ void tma_load_3d_mc(void *dst, const CUtensorMap *map, uint64_t *bar,
                                               int x, int y, int z, uint16_t mask) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      ".multicast::cluster [%0], [%1, {%3, %4, %5}], [%2], %6;" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<uint64_t>(map)), "r"(smem_u32(bar)), "r"(x), "r"(y), "r"(z),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void umma_commit_mc(uint64_t *bar, uint16_t mask) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(smem_u32(bar)),
      "h"(mask)
      : "memory");
}

__device__ __forceinline__ void cluster_sync() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}

__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}

template <int CL>
__global__ void __launch_bounds__(THREADS2, 1)
    k_gemm_tc256m(const __grid_constant__ CUtensorMap map_ahi,
                  const __grid_constant__ CUtensorMap map_alo,
                  const __grid_constant__ CUtensorMap map_bhi,
                  const __grid_constant__ CUtensorMap map_blo, const TcArgs args) {
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + STAGES2 * STAGE2_BYTES);
  uint64_t *empty = full + STAGES2;
  uint64_t *tmem_full = empty + STAGES2;
  uint64_t *tmem_empty = tmem_full + 2;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int rank = int(cluster_rank());
  // cluster index -> (m group, n tile), in bands of gm m groups: the CTAs resident at
  // one time cover ~gm x 148 / (gm CL) tiles, so a k-block of A and of B'' is fetched
  // from HBM once per band instead of once per m group
  const int group = blockIdx.x / CL;
  const int per_band = args.gm * args.n_tiles, band = group / per_band;
  const int first = band * args.gm, gs = min(args.m_groups - first, args.gm);
  const int r_in = group % per_band;
  const int n_tile = r_in / gs, m_tile = (first + r_in % gs) * CL + rank;
  const int bz = blockIdx.z;
  const int slice = bz / args.D, d = bz % args.D;
  const int za = args.a_batched ? bz : d;
  const int zb = args.b_batched ? bz : d;
  constexpr uint16_t kMask = uint16_t((1u << CL) - 1);
  constexpr int kBRows = BN2 / CL;                    // B'' rows this CTA loads
  constexpr int kBPart = B2_TILE_BYTES / CL;          // their bytes in the tile

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_ahi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_alo)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_bhi)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_blo)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < STAGES2; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], CL);  // the MMA commits of every CTA of the cluster
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], 8);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(512));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  cluster_sync();  // every CTA's barriers exist before any multicast lands
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES2;
        const uint32_t phase = (kb / STAGES2) & 1;
        mbar_wait(&empty[s], phase ^ 1);
        unsigned char *st = smem + s * STAGE2_BYTES;
        mbar_expect_tx(&full[s], STAGE2_BYTES);
        const int kx = kb * BK;
        tma_load_3d(st, &map_ahi, &full[s], kx, m_tile * BM, za);
        tma_load_3d(st + A_TILE_BYTES, &map_alo, &full[s], kx, m_tile * BM, za);
        const int brow = n_tile * BN2 + rank * kBRows;
        tma_load_3d_mc(st + 2 * A_TILE_BYTES + rank * kBPart, &map_bhi, &full[s], kx, brow, zb,
                       kMask);
        tma_load_3d_mc(st + 2 * A_TILE_BYTES + B2_TILE_BYTES + rank * kBPart, &map_blo, &full[s],
                       kx, brow, zb, kMask);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % STAGES2;
        const uint32_t phase = (kb / STAGES2) & 1;
        const int chunk = kb / CHUNK, buf = chunk & 1;
        const bool chunk_first = kb % CHUNK == 0;
        const bool chunk_last = kb % CHUNK == CHUNK - 1 || kb == args.k_blocks - 1;
        if (chunk_first) {
          mbar_wait(&tmem_empty[buf], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        mbar_wait(&full[s], phase);
        tc_fence_after();
        const uint32_t st = smem_u32(smem + s * STAGE2_BYTES);
        const uint64_t ahi = smem_desc_sw128(st);
        const uint64_t alo = smem_desc_sw128(st + A_TILE_BYTES);
        const uint64_t bhi = smem_desc_sw128(st + 2 * A_TILE_BYTES);
        const uint64_t blo = smem_desc_sw128(st + 2 * A_TILE_BYTES + B2_TILE_BYTES);
        const uint32_t tacc = tmem_base + uint32_t(buf * BN2);
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          const uint64_t koff = uint64_t((k * UK * 4) >> 4);
          const uint32_t acc0 = (!chunk_first || k > 0) ? 1u : 0u;
          umma_tf32(tacc, ahi + koff, bhi + koff, kIdesc2, acc0);
          umma_tf32(tacc, ahi + koff, blo + koff, kIdesc2, 1u);
          umma_tf32(tacc, alo + koff, bhi + koff, kIdesc2, 1u);
        }
        umma_commit_mc(&empty[s], kMask);  // frees stage s in every CTA of the cluster
        if (chunk_last) umma_commit(&tmem_full[buf]);
      }
    }
  } else {
    const int q4 = warp % 4, half = (warp - 2) / 4;
    const int lane_base = 32 * q4;
    const int row = m_tile * BM + lane_base + lane;
    float acc[128];
#pragma unroll
    for (int c = 0; c < 128; ++c) acc[c] = 0.f;
    const int n_chunks = (args.k_blocks + CHUNK - 1) / CHUNK;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(&tmem_full[buf], (chunk >> 1) & 1);
      tc_fence_after();
      const uint32_t t0 =
          tmem_base + (uint32_t(lane_base) << 16) + uint32_t(buf * BN2 + 128 * half);
#pragma unroll
      for (int cc = 0; cc < 4; ++cc) {
        uint32_t v[32];
        tmem_ld32(t0 + uint32_t(cc * 32), v);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 32; ++q) acc[cc * 32 + q] += __uint_as_float(v[q]);
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tmem_empty[buf]);
    }
    float *crow = args.c + int64_t(slice) * args.c_bs + int64_t(d) * args.c_ds +
                  int64_t(row) * args.two_n + int64_t(n_tile) * BN2 + 128 * half;
#pragma unroll
    for (int q = 0; q < 32; ++q)
      reinterpret_cast<float4 *>(crow)[q] =
          make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
  tc_fence_before();
  cluster_sync();  // no CTA leaves while a peer may still multicast into it
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(512));
  }
}

// ---- operand preparation --------------------------------------------------------
// A (complex M x K per batch) -> hi/lo planes, same M x 2K real layout.
__global__ void k_split_a(const float *__restrict__ a, int64_t a_bs, int64_t a_ds, int D,
                          int64_t per, int64_t nbatch, float *__restrict__ hi,
                          float *__restrict__ lo) {
  const int64_t total = per * nbatch;  // floats
  for (int64_t i = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 4; i < total;
       i += int64_t(gridDim.x) * blockDim.x * 4) {
    const int64_t z = i / per, r = i % per;
    const int64_t slice = z / D, d = z % D;
    const float4 x = *reinterpret_cast<const float4 *>(a + slice * a_bs + d * a_ds + r);
    float4 h, l;
    h.x = tf32_round(x.x), h.y = tf32_round(x.y), h.z = tf32_round(x.z), h.w = tf32_round(x.w);
    l.x = x.x - h.x, l.y = x.y - h.y, l.z = x.z - h.z, l.w = x.w - h.w;
    *reinterpret_cast<float4 *>(hi + i) = h;
    *reinterpret_cast<float4 *>(lo + i) = l;
  }
}

// B (complex K x N per batch) -> B'' (2N x 2K real, K-major) hi/lo planes.
// 32 x 32 complex tiles through shared memory: coalesced reads along n, writes along k.
__global__ void k_expand_b(const float2 *__restrict__ b, int64_t b_bs, int64_t b_ds, int D,
                           int K, int N, float *__restrict__ hi, float *__restrict__ lo) {
  __shared__ float2 tile[32][33];
  const int z = blockIdx.z;
  const int64_t slice = z / D, d = z % D;
  const float2 *src = b + slice * b_bs + d * b_ds;
  const int64_t plane = int64_t(4) * K * N;  // floats per batch in B''
  float *h = hi + z * plane, *l = lo + z * plane;
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y)
    tile[r][threadIdx.x] = src[int64_t(k0 + r) * N + n0 + threadIdx.x];
  __syncthreads();
  // thread (x, y): n = n0 + y, k = k0 + x
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const float2 v = tile[threadIdx.x][r];
    const int n = n0 + r, k = k0 + threadIdx.x;
    const float vals[4] = {v.x, -v.y, v.y, v.x};  // [t][s]: (0,0) br (0,1) -bi (1,0) bi (1,1) br
#pragma unroll
    for (int t = 0; t < 2; ++t) {
      const int64_t row = int64_t(2 * n + t) * (2 * K) + 2 * k;
#pragma unroll
      for (int s = 0; s < 2; ++s) {
        const float x = vals[2 * t + s];
        const float xh = tf32_round(x);
        h[row + s] = xh;
        l[row + s] = x - xh;
      }
    }
  }
}

// ---- host side --------------------------------------------------------------------
using EncodeFn = CUresult (*)(CUtensorMap *, CUtensorMapDataType, cuuint32_t, void *,
                              const cuuint64_t *, const cuuint64_t *, const cuuint32_t *,
                              const cuuint32_t *, CUtensorMapInterleave, CUtensorMapSwizzle,
                              CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

EncodeFn encode_fn() {
  static EncodeFn fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) ==
            cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<EncodeFn>(p);
  });
  return fn;
}

bool make_map(CUtensorMap *map, const float *base, int64_t inner, int64_t rows, int64_t batches,
              int box_rows, int box_k = BK) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(batches)};
  cuuint64_t strides[2] = {cuuint64_t(inner * 4), cuuint64_t(inner * rows * 4)};
  cuuint32_t box[3] = {cuuint32_t(box_k), cuuint32_t(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
             box_k == 16 ? CU_TENSOR_MAP_SWIZZLE_64B : CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

}  // namespace

bool gemm_tc_supported(const GemmShape &s) {
  return s.M % BM == 0 && (2 * s.N) % BN == 0 && s.K % 32 == 0 && s.M >= BM &&
         s.M <= (int64_t(1) << 31) && s.N <= (int64_t(1) << 30) && s.K <= (int64_t(1) << 30);
}

size_t gemm_tc_workspace_bytes(const GemmShape &s, const BatchPtrs &p) {
  const size_t nbA = size_t(p.a_bs ? p.nbatch : 1) * s.D;
  const size_t nbB = size_t(p.b_bs ? p.nbatch : 1) * s.D;
  return size_t(2) * 4 * (nbA * size_t(s.M) * 2 * s.K + nbB * size_t(4) * s.N * s.K);
}

void gemm_tc_a_planes(const GemmShape &s, const BatchPtrs &p, void *workspace, float **hi,
                      float **lo) {
  const int64_t nbA = (p.a_bs ? p.nbatch : 1) * s.D;
  *hi = static_cast<float *>(workspace);
  *lo = *hi + size_t(s.M) * 2 * s.K * nbA;
}

cudaError_t launch_gemm_tc(const GemmShape &s, const BatchPtrs &p, void *workspace,
                           size_t workspace_bytes, cudaStream_t stream, cudaEvent_t *gemm_events,
                           bool a_presplit) {
  if (!gemm_tc_supported(s)) return cudaErrorNotSupported;
  const int64_t nbA = (p.a_bs ? p.nbatch : 1) * s.D;
  const int64_t nbB = (p.b_bs ? p.nbatch : 1) * s.D;
  const size_t a_plane = size_t(s.M) * 2 * s.K;       // floats per batch
  const size_t b_plane = size_t(4) * s.N * s.K;
  const size_t need = 4 * 2 * (a_plane * nbA + b_plane * nbB);
  if (need > workspace_bytes) return cudaErrorNotSupported;
  float *ahi = static_cast<float *>(workspace);
  float *alo = ahi + a_plane * nbA;
  float *bhi = alo + a_plane * nbA;
  float *blo = bhi + b_plane * nbB;
  if (!a_presplit) {
    const int64_t total = int64_t(a_plane) * nbA;
    int64_t blocks = (total / 4 + 255) / 256;
    if (blocks > 148 * 32) blocks = 148 * 32;
    k_split_a<<<unsigned(blocks), 256, 0, stream>>>(
        static_cast<const float *>(p.a), 2 * p.a_bs, int64_t(2) * s.M * s.K, int(s.D),
        int64_t(a_plane), nbA, ahi, alo);
  }
  {
    dim3 grid(unsigned(s.N / 32), unsigned(s.K / 32), unsigned(nbB));
    if (s.N % 32 || s.K % 32) return cudaErrorNotSupported;
    k_expand_b<<<grid, dim3(32, 8), 0, stream>>>(static_cast<const float2 *>(p.b), p.b_bs,
                                                  s.K * s.N, int(s.D), int(s.K), int(s.N), bhi,
                                                  blo);
  }
  // 128 x 256 tiles where 2N allows (STN_GEMM_BN=128 forces the 128 x 128 kernel)
  const char *env_bn = stn::debug_opt("gemm_bn");
  const bool wide = (2 * s.N) % BN2 == 0 && !(env_bn && std::atoi(env_bn) == 128);
  const int bn = wide ? BN2 : BN;
  // 128 x 256 tiles with 16-K stages (four-deep ring): STN_DEBUG gemm_bk=16
  const char *env_bk = stn::debug_opt("gemm_bk");
  const bool deep = wide && env_bk && std::atoi(env_bk) == 16;
  const int bk = deep ? BK3 : BK;
  // clusters sharing the B tile (STN_DEBUG gemm_mc=1|2|4: cluster size, default 2)
  const char *env_mc = stn::debug_opt("gemm_mc");
  int cl = env_mc ? std::atoi(env_mc) : 2;
  if (!wide || deep || (cl != 2 && cl != 4) || (s.M / BM) % cl != 0) cl = 1;
  CUtensorMap mah, mal, mbh, mbl;
  if (!make_map(&mah, ahi, 2 * s.K, s.M, nbA, BM, bk) ||
      !make_map(&mal, alo, 2 * s.K, s.M, nbA, BM, bk) ||
      !make_map(&mbh, bhi, 2 * s.K, 2 * s.N, nbB, bn / cl, bk) ||
      !make_map(&mbl, blo, 2 * s.K, 2 * s.N, nbB, bn / cl, bk))
    return cudaErrorNotSupported;
  static bool attr_on[kMaxDevices] = {};
  bool &attr_set = attr_on[current_device()];
  if (!attr_set) {
    cudaError_t e =
        cudaFuncSetAttribute(k_gemm_tc, cudaFuncAttributeMaxDynamicSharedMemorySize, int(SMEM_BYTES));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gemm_tc256, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(SMEM2_BYTES));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gemm_tc256s, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(SMEM3_BYTES));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gemm_tc256m<2>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(SMEM2_BYTES));
    if (e != cudaSuccess) return e;
    e = cudaFuncSetAttribute(k_gemm_tc256m<4>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                             int(SMEM2_BYTES));
    if (e != cudaSuccess) return e;
    attr_set = true;
  }
  TcArgs args;
  args.c = static_cast<float *>(p.out);
  args.c_bs = 2 * p.out_bs;
  args.c_ds = int64_t(2) * s.M * s.N;
  args.D = int(s.D);
  args.a_batched = p.a_bs != 0;
  args.b_batched = p.b_bs != 0;
  args.k_blocks = int(2 * s.K / bk);
  args.two_n = int(2 * s.N);
  args.n_tiles = int(2 * s.N / bn);
  args.m_groups = int(s.M / BM / cl);
  {
    const char *env_gm = stn::debug_opt("gemm_gm");  // raster band height in m tiles
    const int gm_tiles = env_gm ? std::atoi(env_gm) : 16;
    args.gm = std::max(1, std::min(args.m_groups, gm_tiles / cl));
  }
  dim3 grid(unsigned((2 * s.N / bn) * (s.M / BM)), 1, unsigned(s.D * p.nbatch));
  if (gemm_events) cudaEventRecord(gemm_events[0], stream);
  if (cl > 1) {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = grid;
    cfg.blockDim = dim3(THREADS2);
    cfg.dynamicSmemBytes = SMEM2_BYTES;
    cfg.stream = stream;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = unsigned(cl);
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    const cudaError_t e = cl == 4 ? cudaLaunchKernelEx(&cfg, k_gemm_tc256m<4>, mah, mal, mbh, mbl, args)
                                  : cudaLaunchKernelEx(&cfg, k_gemm_tc256m<2>, mah, mal, mbh, mbl, args);
    if (e != cudaSuccess) return e;
  } else if (deep)
    k_gemm_tc256s<<<grid, THREADS2, SMEM3_BYTES, stream>>>(mah, mal, mbh, mbl, args);
  else if (wide)
    k_gemm_tc256<<<grid, THREADS2, SMEM2_BYTES, stream>>>(mah, mal, mbh, mbl, args);
  else
    k_gemm_tc<<<grid, THREADS, SMEM_BYTES, stream>>>(mah, mal, mbh, mbl, args);
  if (gemm_events) cudaEventRecord(gemm_events[1], stream);
  return cudaGetLastError();
}

}  // namespace stn
