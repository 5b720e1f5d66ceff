// tcgen05 split-TF32 complex GEMM with the operand split fused into shared memory.
//
//   C[z] (M x N complex) = A[z] (M x K complex, row-major) * B[z] (K x N complex)
//
// Same algebra as gemm_tc.cu (A is the M x 2K real K-major matrix of its own
// interleaved storage; B becomes the 2N x 2K real K-major B'' with
// B''[2n+t][2k+s] = [[br, -bi], [bi, br]][t][s]; C = A . B''^T), but no hi / lo
// planes exist in HBM:
//   * the TMA loads the RAW fp32 tiles of A (straight from the step operand when
//     its [D|M|K] order is the stored order, i.e. no transposed copy) and of B''
//     (one raw plane from the expansion pre-pass, B being the small operand);
//   * the tensor core truncates fp32 operands to TF32 (measured, round 1), so the
//     raw tile IS the "hi" operand; converter warps write lo = x - trunc(x) (exact
//     in fp32) at the same byte offsets -- the SWIZZLE_128B layout is a permutation
//     of 16-byte chunks, so an elementwise pass keeps it -- then release the stage;
//   * C ~= Ahi.Bhi + Ahi.Blo + Alo.Bhi into one fp32 TMEM accumulator, K in chunks
//     of CHUNK k-blocks alternating between two TMEM buffers and flushed into fp32
//     registers with round-to-nearest adds (long K chains do not accumulate the
//     tensor core's truncating adds).
// Per k-block the SM pulls 16 KiB of A and BN x 128 B of B'' from L2 instead of
// twice that (hi + lo planes), and HBM sees A once (4 bytes per real element)
// instead of split-pass read + 2 plane writes + 2 plane reads.
//
// Warp roles: 0 TMA producer, 1 MMA issuer (one elected thread), then the
// converters (4, or 2 at BN = 256), then the epilogue (BN / 128 warps per TMEM lane
// quadrant, at least one).
#include <cuda.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <mutex>

#include "kernels.h"

namespace stn {

namespace {

constexpr int BM = 128;  // rows of C per CTA (UMMA M)
constexpr int BK = 32;   // real K per stage (128-byte rows -> SWIZZLE_128B)
constexpr int UK = 8;    // real K per tcgen05.mma.kind::tf32
constexpr int CHUNK = 8; // k-blocks accumulated in TMEM before an fp32 RN flush
constexpr int A_BYTES = BM * BK * 4;  // 16 KiB
template <int BN>
struct Cfg {
  // converter warps (BN = 256: two, so the 8 epilogue warps keep 128 fp32 accumulators
  // each in registers at 384 threads)
  static constexpr int CONV_WARPS = BN >= 256 ? 2 : 4;
  static constexpr int B_BYTES = BN * BK * 4;
  // a ring of raw stages [A | B] (TMA / gather targets) and a shorter ring of lo buffers
  // [A lo | B lo] written by the converters: more raw bytes in flight per SM than
  // raw + lo stages side by side (6 / 4 / 2 raw stages at BN = 64 / 128 / 256)
  static constexpr int RAW_BYTES = A_BYTES + B_BYTES;
  static constexpr int NSL = 2;
  static constexpr int STAGES = (192 * 1024 - NSL * RAW_BYTES) / RAW_BYTES;
  static constexpr int EPI_WARPS = BN >= 256 ? 8 : 4;
  static constexpr int COLS_PER_EPI = BN >= 256 ? 128 : BN;
  static constexpr int THREADS = 32 * (2 + CONV_WARPS + EPI_WARPS);
  static constexpr int EPI_WARP0 = 2 + CONV_WARPS;
  static constexpr int GATHER_WARP0 = 2 + CONV_WARPS + EPI_WARPS;  // gather variant: 4 more
  static constexpr int GATHER_LAG = STAGES - 2;  // cp.async stages in flight per gatherer
  static constexpr int TMEM_COLS = 2 * BN;  // two accumulator buffers
  static constexpr size_t SMEM = size_t(STAGES + NSL) * RAW_BYTES + 1024 + 256;
  // kind::tf32: F32 accumulate (bit 4), A/B TF32 (bits 7, 10), both K-major, N >> 3, M >> 4
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (uint32_t(BN >> 3) << 17) | (uint32_t(BM >> 4) << 24);
};

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
__device__ __forceinline__ void mbar_arrive(uint64_t *bar) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(bar)) : "memory");
}
// Waits on an mbarrier phase; a wait that never completes (a pipeline bug) traps
// after ~60 s of clock instead of hanging the device.
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
    if ((iter & 4095) == 4095 && clock64() - start > (120ll << 30)) __trap();
  }
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
// K-major SWIZZLE_128B descriptor: 8-row x 128 B atoms every 1024 B (SBO).
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}

// lo = x - trunc_tf32(x), 4 floats (exact in fp32; the tensor core reads x itself as hi)
__device__ __forceinline__ float4 tf32_lo(const float4 x) {
  float4 r;
  r.x = x.x - __uint_as_float(__float_as_uint(x.x) & 0xFFFFE000u);
  r.y = x.y - __uint_as_float(__float_as_uint(x.y) & 0xFFFFE000u);
  r.z = x.z - __uint_as_float(__float_as_uint(x.z) & 0xFFFFE000u);
  r.w = x.w - __uint_as_float(__float_as_uint(x.w) & 0xFFFFE000u);
  return r;
}

struct TcfArgs {
  float *c;        // C (M x 2N floats per (slice, d))
  int64_t c_bs;    // floats between slices
  int64_t c_ds;    // floats between D batches
  int D;
  int a_batched, b_batched;
  int k_blocks;    // 2K / BK
  int two_n;
  int n_tiles;     // 2N / BN
  // gather variant: A[m][k] = X[moff_hi[m / 128] + moff_lo[m % 128] + koff[k]] (complex
  // elements; the operand permutation read straight from the stem layout)
  const float2 *x;
  int64_t x_bs;
  const int64_t *moff_lo, *moff_hi, *koff;
};

__device__ __forceinline__ void cp_async8(uint32_t dst, const void *src) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(dst), "l"(src) : "memory");
}

template <int BN, bool GATHER>
__global__ void __launch_bounds__(Cfg<BN>::THREADS + (GATHER ? 128 : 0), 1)
    k_gemm_tcf(const __grid_constant__ CUtensorMap map_a, const __grid_constant__ CUtensorMap map_b,
               const TcfArgs args) {
  using C = Cfg<BN>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = reinterpret_cast<unsigned char *>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint64_t *full = reinterpret_cast<uint64_t *>(smem + (C::STAGES + C::NSL) * C::RAW_BYTES);
  uint64_t *empty = full + C::STAGES;      // raw stage consumed by the MMAs
  uint64_t *conv = empty + C::STAGES;      // [NSL] lo buffer written
  uint64_t *lo_free = conv + C::NSL;       // [NSL] lo buffer consumed by the MMAs
  uint64_t *tmem_full = lo_free + C::NSL;  // [2]
  uint64_t *tmem_empty = tmem_full + 2;    // [2]
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(tmem_empty + 2);

  const int warp = threadIdx.x / 32, lane = threadIdx.x % 32;
  const int n_tile = blockIdx.x % args.n_tiles, m_tile = blockIdx.x / args.n_tiles;
  const int bz = blockIdx.z;
  const int slice = bz / args.D, d = bz % args.D;
  const int za = args.a_batched ? bz : d;
  const int zb = args.b_batched ? bz : d;

  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_a)) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(reinterpret_cast<uint64_t>(&map_b)) : "memory");
  }
  if (warp == 1 && lane == 0) {
    for (int s = 0; s < C::STAGES; ++s) {
      mbar_init(&full[s], GATHER ? 1 + 128 : 1);  // TMA (+ the 128 A gatherers)
      mbar_init(&empty[s], 1);
    }
    for (int l = 0; l < C::NSL; ++l) {
      mbar_init(&conv[l], C::CONV_WARPS);
      mbar_init(&lo_free[l], 1);
    }
    for (int b = 0; b < 2; ++b) {
      mbar_init(&tmem_full[b], 1);
      mbar_init(&tmem_empty[b], C::EPI_WARPS);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 2) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem_base = *tmem_slot;
  // raw stage s: [A raw | B raw]; lo buffer l: [A lo | B lo] (same offsets)
  auto stage = [&](int s) { return smem + s * C::RAW_BYTES; };
  auto lobuf = [&](int l) { return smem + (C::STAGES + l) * C::RAW_BYTES; };

  if (warp == 0) {
    if (lane == 0) {  // ---- TMA producer: raw tiles only ----
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % C::STAGES;
        mbar_wait(&empty[s], ((kb / C::STAGES) & 1) ^ 1);
        unsigned char *st = stage(s);
        mbar_expect_tx(&full[s], (GATHER ? 0 : A_BYTES) + C::B_BYTES);
        if (!GATHER) tma_load_3d(st, &map_a, &full[s], kb * BK, m_tile * BM, za);
        tma_load_3d(st + A_BYTES, &map_b, &full[s], kb * BK, n_tile * BN, zb);
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---- MMA issuer ----
      for (int kb = 0; kb < args.k_blocks; ++kb) {
        const int s = kb % C::STAGES;
        const int chunk = kb / CHUNK, buf = chunk & 1;
        const bool chunk_first = kb % CHUNK == 0;
        const bool chunk_last = kb % CHUNK == CHUNK - 1 || kb == args.k_blocks - 1;
        if (chunk_first) {
          mbar_wait(&tmem_empty[buf], ((chunk >> 1) & 1) ^ 1);
          tc_fence_after();
        }
        const int l = kb % C::NSL;
        mbar_wait(&conv[l], (kb / C::NSL) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(stage(s)), lt = smem_u32(lobuf(l));
        const uint64_t ahi = smem_desc_sw128(st), alo = smem_desc_sw128(lt);
        const uint64_t bhi = smem_desc_sw128(st + A_BYTES);
        const uint64_t blo = smem_desc_sw128(lt + A_BYTES);
        const uint32_t tacc = tmem_base + uint32_t(buf * BN);
#pragma unroll
        for (int k = 0; k < BK / UK; ++k) {
          const uint64_t koff = uint64_t((k * UK * 4) >> 4);  // +32 B per K step
          const uint32_t acc0 = (!chunk_first || k > 0) ? 1u : 0u;
          umma_tf32(tacc, ahi + koff, bhi + koff, C::IDESC, acc0);
          umma_tf32(tacc, ahi + koff, blo + koff, C::IDESC, 1u);
          umma_tf32(tacc, alo + koff, bhi + koff, C::IDESC, 1u);
        }
        umma_commit(&empty[s]);
        umma_commit(&lo_free[l]);
        if (chunk_last) umma_commit(&tmem_full[buf]);
      }
    }
  } else if (warp < C::EPI_WARP0) {
    // ---- converters: lo tiles next to the raw ones, same byte offsets ----
    const int ct = threadIdx.x - 64;  // 0 .. 32 * CONV_WARPS - 1
    constexpr int NV = (A_BYTES + C::B_BYTES) / 16;  // float4 per stage
    for (int kb = 0; kb < args.k_blocks; ++kb) {
      const int s = kb % C::STAGES, l = kb % C::NSL;
      mbar_wait(&full[s], (kb / C::STAGES) & 1);
      mbar_wait(&lo_free[l], ((kb / C::NSL) & 1) ^ 1);
      const unsigned char *st = stage(s);
      unsigned char *lt = lobuf(l);
#pragma unroll 4
      for (int i = ct; i < NV; i += 32 * C::CONV_WARPS) {
        const float4 x = *reinterpret_cast<const float4 *>(st + i * 16);
        *reinterpret_cast<float4 *>(lt + i * 16) = tf32_lo(x);
      }
      // generic-proxy smem writes -> visible to the tensor core (async proxy)
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&conv[l]);
    }
  } else if (GATHER && warp >= C::GATHER_WARP0) {
    // ---- A gatherers: row g of the tile, its 16 complex k of each stage, 8-byte
    // cp.async straight into the K-major SWIZZLE_128B layout TMA would have written
    // (16-byte chunk c of row r at chunk c ^ (r & 7)); lanes = consecutive rows ----
    const int g = threadIdx.x - 32 * C::GATHER_WARP0;  // 0 .. 127
    const float2 *xrow = args.x + int64_t(za) * args.x_bs + args.moff_hi[m_tile] + args.moff_lo[g];
    const uint32_t row_base = uint32_t(g) * 128u;
    const int sw = g & 7;
    // k offsets are linear in the bits of k: koff(16 kb + j) = koff(16 kb) + koff(j), so a
    // stage needs one table load (its base) and 16 register-held low offsets
    int64_t klo[BK / 2];
#pragma unroll
    for (int j = 0; j < BK / 2; ++j) klo[j] = __ldg(args.koff + j);
    int64_t khi = __ldg(args.koff);
    for (int kb = 0; kb < args.k_blocks + C::GATHER_LAG; ++kb) {
      if (kb < args.k_blocks) {
        const int s = kb % C::STAGES;
        const int64_t kbase = khi;
        if (kb + 1 < args.k_blocks) khi = __ldg(args.koff + int64_t(kb + 1) * (BK / 2));
        mbar_wait(&empty[s], ((kb / C::STAGES) & 1) ^ 1);
        const uint32_t dst = smem_u32(stage(s)) + row_base;
        const float2 *src = xrow + kbase;
#pragma unroll
        for (int j = 0; j < BK / 2; ++j)
          cp_async8(dst + uint32_t((((j >> 1) ^ sw) << 4) + ((j & 1) << 3)), src + klo[j]);
      }
      asm volatile("cp.async.commit_group;" ::: "memory");
      const int done = kb - C::GATHER_LAG;  // this thread's copies of stage `done` landed
      if (done >= 0) {
        asm volatile("cp.async.wait_group %0;" ::"n"(C::GATHER_LAG) : "memory");
        asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        mbar_arrive(&full[done % C::STAGES]);
      }
    }
  } else {
    // ---- epilogue: drain each K chunk into fp32 registers (RN adds), then store ----
    const int e = warp - C::EPI_WARP0;  // 0 .. EPI_WARPS-1
    const int quad = warp % 4;            // TMEM lane quadrant this warp may access
    const int half = e / 4;               // column half (BN = 256)
    const int row = m_tile * BM + 32 * quad + lane;
    float acc[C::COLS_PER_EPI];
#pragma unroll
    for (int c = 0; c < C::COLS_PER_EPI; ++c) acc[c] = 0.f;
    const int n_chunks = (args.k_blocks + CHUNK - 1) / CHUNK;
    for (int chunk = 0; chunk < n_chunks; ++chunk) {
      const int buf = chunk & 1;
      mbar_wait(&tmem_full[buf], (chunk >> 1) & 1);
      tc_fence_after();
      const uint32_t t0 = tmem_base + (uint32_t(32 * quad) << 16) +
                          uint32_t(buf * BN + C::COLS_PER_EPI * half);
#pragma unroll
      for (int cc = 0; cc < C::COLS_PER_EPI / 32; ++cc) {
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
                  int64_t(row) * args.two_n + int64_t(n_tile) * BN + C::COLS_PER_EPI * half;
    const int col0 = n_tile * BN + C::COLS_PER_EPI * half;  // 2N < 64: padded B'' columns
#pragma unroll
    for (int q = 0; q < C::COLS_PER_EPI / 4; ++q)
      if (col0 + 4 * q < args.two_n)
        reinterpret_cast<float4 *>(crow)[q] =
            make_float4(acc[4 * q], acc[4 * q + 1], acc[4 * q + 2], acc[4 * q + 3]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 2) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem_base),
                 "r"(C::TMEM_COLS));
  }
}

// Narrow B (N < 32): rows 2n, 2n+1 of a zeroed B'' with 2 * npad rows.
__global__ void k_expand_b_raw_small(const float2 *__restrict__ b, int64_t b_bs, int64_t b_ds,
                                     int D, int K, int N, int npad, float *__restrict__ out) {
  const int z = blockIdx.y;
  const int64_t slice = z / D, d = z % D;
  const float2 *src = b + slice * b_bs + d * b_ds;
  float *o = out + int64_t(z) * 4 * K * npad;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < int64_t(K) * N;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int k = int(i / N), n = int(i % N);
    const float2 v = src[i];
    const int64_t row0 = int64_t(2 * n) * (2 * K) + 2 * k, row1 = row0 + 2 * K;
    *reinterpret_cast<float2 *>(o + row0) = make_float2(v.x, -v.y);
    *reinterpret_cast<float2 *>(o + row1) = make_float2(v.y, v.x);
  }
}

// B (complex K x N per batch) -> raw B'' (2N x 2K real, K-major), one plane.
__global__ void k_expand_b_raw(const float2 *__restrict__ b, int64_t b_bs, int64_t b_ds, int D,
                               int K, int N, float *__restrict__ out) {
  __shared__ float2 tile[32][33];
  const int z = blockIdx.z;
  const int64_t slice = z / D, d = z % D;
  const float2 *src = b + slice * b_bs + d * b_ds;
  float *o = out + int64_t(z) * 4 * K * N;
  const int k0 = blockIdx.y * 32, n0 = blockIdx.x * 32;
  for (int r = threadIdx.y; r < 32; r += blockDim.y)
    tile[r][threadIdx.x] = src[int64_t(k0 + r) * N + n0 + threadIdx.x];
  __syncthreads();
  for (int r = threadIdx.y; r < 32; r += blockDim.y) {
    const float2 v = tile[threadIdx.x][r];
    const int n = n0 + r, k = k0 + threadIdx.x;
    const int64_t row0 = int64_t(2 * n) * (2 * K) + 2 * k, row1 = row0 + 2 * K;
    *reinterpret_cast<float2 *>(o + row0) = make_float2(v.x, -v.y);
    *reinterpret_cast<float2 *>(o + row1) = make_float2(v.y, v.x);
  }
}

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

// [batches][rows][inner] fp32, rows `row_stride` floats apart, batches `batch_stride`.
bool make_map(CUtensorMap *map, const float *base, int64_t inner, int64_t rows, int64_t batches,
              int64_t batch_stride, int box_rows) {
  EncodeFn enc = encode_fn();
  if (!enc) return false;
  cuuint64_t dims[3] = {cuuint64_t(inner), cuuint64_t(rows), cuuint64_t(batches)};
  cuuint64_t strides[2] = {cuuint64_t(inner * 4), cuuint64_t(batch_stride * 4)};
  cuuint32_t box[3] = {cuuint32_t(BK), cuuint32_t(box_rows), 1};
  cuuint32_t estr[3] = {1, 1, 1};
  return enc(map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 3, const_cast<float *>(base), dims, strides,
             box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
             CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) ==
         CUDA_SUCCESS;
}

template <int BN, bool GATHER>
cudaError_t launch_bn(const CUtensorMap &ma, const CUtensorMap &mb, const TcfArgs &args,
                      dim3 grid, cudaStream_t stream) {
  using C = Cfg<BN>;
  static bool set_on[kMaxDevices] = {};
  bool &set = set_on[current_device()];
  if (!set) {
    const cudaError_t attr = cudaFuncSetAttribute(
        k_gemm_tcf<BN, GATHER>, cudaFuncAttributeMaxDynamicSharedMemorySize, int(C::SMEM));
    if (attr != cudaSuccess) return attr;
    set = true;
  }
  k_gemm_tcf<BN, GATHER><<<grid, C::THREADS + (GATHER ? 128 : 0), C::SMEM, stream>>>(ma, mb, args);
  return cudaGetLastError();
}

int pick_bn(const GemmShape &s) {
  const char *o = debug_opt("tcf_bn");
  if (o) {
    const int bn = std::atoi(o);
    if ((bn == 64 || bn == 128 || bn == 256) && (2 * s.N) % bn == 0) return bn;
  }
  if ((2 * s.N) % 256 == 0) return 256;
  if ((2 * s.N) % 128 == 0) return 128;
  return 64;
}

}  // namespace

// padded B'' columns for a narrow N (8, 16: the tile's extra rows are zeros)
int64_t tcf_npad(const GemmShape &s) { return s.N < 32 ? 32 : s.N; }

bool gemm_tcf_supported(const GemmShape &s) {
  // narrow N (8, 16) only for tall A (>= 512 tiles): the skinny SIMT GEMM wins below
  return s.M % BM == 0 && (s.N % 32 == 0 || ((s.N == 8 || s.N == 16) && s.M >= (1 << 16))) &&
         s.K % 32 == 0 && s.M >= BM &&
         s.M <= (int64_t(1) << 31) && s.N <= (int64_t(1) << 30) && s.K <= (int64_t(1) << 30);
}

size_t gemm_tcf_workspace_bytes(const GemmShape &s, const BatchPtrs &p) {
  const size_t nbB = size_t(p.b_bs ? p.nbatch : 1) * size_t(s.D);
  return nbB * size_t(4) * size_t(tcf_npad(s)) * size_t(s.K) * 4;
}

cudaError_t launch_gemm_tcf(const GemmShape &s, const BatchPtrs &p, void *workspace,
                            size_t workspace_bytes, cudaStream_t stream, const TcfGather *ga) {
  if (!gemm_tcf_supported(s)) return cudaErrorNotSupported;
  if (gemm_tcf_workspace_bytes(s, p) > workspace_bytes) return cudaErrorNotSupported;
  // A is read in place: one [D|M|K] block per slice, or shared by every slice; or
  // gathered from the stem layout through offset tables (ga, D == 1)
  if (ga && s.D != 1) return cudaErrorNotSupported;
  if (!ga && p.a_bs != 0 && p.a_bs != s.D * s.M * s.K) return cudaErrorNotSupported;
  const int64_t nbA = (p.a_bs ? p.nbatch : 1) * s.D;
  const int64_t nbB = (p.b_bs ? p.nbatch : 1) * s.D;
  float *braw = static_cast<float *>(workspace);
  const int64_t npad = tcf_npad(s);
  if (npad != s.N) {
    const size_t bytes = size_t(nbB) * 4 * size_t(npad) * size_t(s.K) * 4;
    cudaError_t e = cudaMemsetAsync(braw, 0, bytes, stream);
    if (e != cudaSuccess) return e;
    k_expand_b_raw_small<<<dim3(unsigned(std::min<int64_t>((s.K * s.N + 255) / 256, 1024)),
                               unsigned(nbB)),
                           256, 0, stream>>>(static_cast<const float2 *>(p.b), p.b_bs, s.K * s.N,
                                             int(s.D), int(s.K), int(s.N), int(npad), braw);
  } else {
    if (s.N % 32 || s.K % 32) return cudaErrorNotSupported;
    dim3 grid(unsigned(s.N / 32), unsigned(s.K / 32), unsigned(nbB));
    k_expand_b_raw<<<grid, dim3(32, 8), 0, stream>>>(static_cast<const float2 *>(p.b), p.b_bs,
                                                      s.K * s.N, int(s.D), int(s.K), int(s.N),
                                                      braw);
  }
  // the gather variant runs 128 more threads: 64-column tiles keep its epilogue in registers
  const int bn = ga || npad != s.N ? 64 : pick_bn(s);
  CUtensorMap ma, mb;
  if ((!ga && !make_map(&ma, static_cast<const float *>(p.a), 2 * s.K, s.M, nbA, 2 * s.M * s.K,
                        BM)) ||
      !make_map(&mb, braw, 2 * s.K, 2 * npad, nbB, 4 * npad * s.K, bn))
    return cudaErrorNotSupported;
  if (ga) ma = mb;  // unused by the gather variant
  TcfArgs args;
  args.c = static_cast<float *>(p.out);
  args.c_bs = 2 * p.out_bs;
  args.c_ds = int64_t(2) * s.M * s.N;
  args.D = int(s.D);
  args.a_batched = p.a_bs != 0;
  args.b_batched = p.b_bs != 0;
  args.k_blocks = int(2 * s.K / BK);
  args.two_n = int(2 * s.N);
  args.n_tiles = int(2 * npad / bn);
  args.x = static_cast<const float2 *>(p.a);
  args.x_bs = p.a_bs;
  args.moff_lo = ga ? ga->moff_lo : nullptr;
  args.moff_hi = ga ? ga->moff_hi : nullptr;
  args.koff = ga ? ga->koff : nullptr;
  dim3 grid(unsigned((2 * npad / bn) * (s.M / BM)), 1, unsigned(s.D * p.nbatch));
  if (ga) return launch_bn<64, true>(ma, mb, args, grid, stream);  // bn = 64 (registers)
  switch (bn) {
    case 256:
      return launch_bn<256, false>(ma, mb, args, grid, stream);
    case 128:
      return launch_bn<128, false>(ma, mb, args, grid, stream);
    default:
      return launch_bn<64, false>(ma, mb, args, grid, stream);
  }
}

}  // namespace stn
