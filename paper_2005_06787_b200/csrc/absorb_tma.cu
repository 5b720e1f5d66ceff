// TMA-fed tensor-core absorb (FAST mode): the bond-2 stem step
//   O[m, n] = sum_k X[m, k] * W[k, n]        (complex64, 4 <= K <= 64, N <= 64)
// for stems whose four lowest X bits are M bits.
//
// The index permutation is fused into the tile loads: one multi-dimensional TMA
// box per stage gathers the X tile (64*MB complex m x KS k) straight from the
// canonical stem layout into shared memory, already in the UMMA MN-major
// SWIZZLE_128B_BASE32B operand layout (TMA swizzle 128B_ATOM_32B). The box
// dimensions are the runs of tile bits in the stem: dim 0 is X bits 0..3 with
// the (re, im) pair -- 32 floats, one MN row -- then the runs of K bits, then
// the runs of the remaining tile M bits; the bits above each run are its TMA
// coordinate. No thread touches the input on its way to the tensor core.
//
// De-interleaved real form (row 2m+s of A' is component s of X[m, :]):
//   A'[2m+s][k] = X_s[m, k]       B'[2n+t][k] = W_t[k, n]
//   D'[2m+s][2n+t] = sum_k A' B'
//   O[m, n] = (D'[2m][2n] - D'[2m+1][2n+1], D'[2m][2n+1] + D'[2m+1][2n])
// Split TF32: the tensor core truncates fp32 operands to TF32, so the raw TMA
// tile IS the "hi" operand; converter warps write lo = x - trunc(x) next to it.
// B'' = [B'hi ; B'lo] is one K-major operand of 2*NM rows, so
//   MMA 1: acc[0:2NM]  = A'raw . B''    (hi*hi and hi*lo in one instruction)
//   MMA 2: acc[NM:2NM] += A'lo . B'hi
// and the epilogue adds the two halves (runtime.hpp:386-418 is the reference
// step; the result is its GEMM within split-TF32 accuracy).
//
// Warp roles (persistent CTA, one per SM):
//   warp 0      TMA producer (one thread), ring of NS raw stages
//   warp 1      TMEM allocation + MMA issuer (one thread)
//   warps 2-5   converters: lo plane of each stage
//   warps 6-9   epilogue: TMEM -> registers, complex recombination, stores
#include <cuda.h>
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "kernels.h"
#include "tc_ptx.cuh"

namespace stn {

namespace {

using namespace ptx;

constexpr int kConvWarps = 4, kEpiWarps = 4;
constexpr int kMaxNSR = 10, kMaxNSL = 4;  // ring depths: raw X stages, lo planes
constexpr int kMaxLag = 6;  // cp.async groups in flight per loader thread (GATHER), <= nsr - 2

__device__ __forceinline__ void cp_async_wait(int n) {  // wait_group takes an immediate
  switch (n) {
    case 0: asm volatile("cp.async.wait_group 0;" ::: "memory"); break;
    case 1: asm volatile("cp.async.wait_group 1;" ::: "memory"); break;
    case 2: asm volatile("cp.async.wait_group 2;" ::: "memory"); break;
    case 3: asm volatile("cp.async.wait_group 3;" ::: "memory"); break;
    case 4: asm volatile("cp.async.wait_group 4;" ::: "memory"); break;
    case 5: asm volatile("cp.async.wait_group 5;" ::: "memory"); break;
    default: asm volatile("cp.async.wait_group 6;" ::: "memory"); break;
  }
}

template <int KSZ, int MB, int NM>
struct TmaLayout {
  static constexpr int STAGE = MB * KSZ * 512;       // bytes of one raw (or lo) stage
  static constexpr int LBO = KSZ * 128;              // MN-atom stride (32 m-floats x KSZ rows)
  static constexpr int BROWS = 2 * NM;               // B'' rows: hi then lo
  // DUAL (small N): MMA 1 = raw x [B'hi; B'lo] (N = 2NM) puts hi*hi and hi*lo in two column
  // halves, MMA 2 adds lo*hi to the second half -- 2 MMAs per k-step instead of 3 (the
  // single MMA thread is the limit there); the epilogue adds the halves.
  static constexpr bool DUAL = NM <= 32;
  static constexpr int BCOLS = DUAL ? 2 * NM : NM;    // TMEM columns of one M block
  static constexpr int ACC = MB * BCOLS;             // TMEM columns of one accumulator buffer
  static constexpr int NACC = 4 * ACC <= 512 ? 4 : 2;  // accumulator buffers
  static constexpr int TMEM_COLS = NACC * ACC <= 32 ? 32 : (NACC * ACC <= 64 ? 64 : (NACC * ACC <= 128 ? 128 : (NACC * ACC <= 256 ? 256 : 512)));
};

// Experiments (dbg & 32): cycles spent waiting on each barrier kind, CTA 0, printed at exit.
#define TW(slot, call)                                                 \
  do {                                                                 \
    const long long t0_ = (g.dbg & 32) ? clock64() : 0;                \
    call;                                                              \
    if (g.dbg & 32) wait_cyc[slot] += clock64() - t0_;                 \
  } while (0)

// Position in a ring of mbarrier-guarded slots: slot index and the parity of its phase.
struct RingPos {
  int idx = 0;
  uint32_t phase = 0;
  __device__ __forceinline__ void next(int n) {
    if (++idx == n) {
      idx = 0;
      phase ^= 1u;
    }
  }
};

__device__ __forceinline__ uint64_t pdep64(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t bit = 1; mask; bit <<= 1) {
    const uint64_t low = mask & (0 - mask);
    if (v & bit) r |= low;
    mask ^= low;
  }
  return r;
}

// Byte offset of real element (row, col) in a K-major SWIZZLE_128B plane of 32-column slabs.
__device__ __forceinline__ uint32_t kmajor_off(int row, int col, int rows) {
  const int slab = col >> 5, cc = col & 31;
  return uint32_t(slab * rows * 128 + row * 128 + (((cc >> 2) ^ (row & 7)) << 4) + (cc & 3) * 4);
}

template <bool GATHER>
struct Roles {
  // GATHER: warp 0 MMA, warps 1-8 loaders (cp.async gather + lo), warps 9-16 epilogue.
  // TMA:    warp 0 TMA, warp 1 MMA, warps 2-5 converters (lo), warps 6-13 epilogue.
  static constexpr int THREADS = GATHER ? 544 : 448;
  static constexpr int MMA_WARP = GATHER ? 0 : 1;
  static constexpr int LOAD_WARP0 = GATHER ? 1 : 2;
  static constexpr int LOAD_WARPS = GATHER ? 8 : 4;
  static constexpr int EPI_WARP0 = GATHER ? 9 : 6;  // 8 epilogue warps: 2 per TMEM quadrant
};

template <int KSZ, int MB, int NM, bool GATHER>
__global__ void __launch_bounds__(Roles<GATHER>::THREADS, 1)
    k_absorb_tma(const __grid_constant__ CUtensorMap map, const __grid_constant__ TmaAbsorbGeom g,
                 const float2 *__restrict__ X, const float2 *__restrict__ W,
                 float2 *__restrict__ O) {
  using Lay = TmaLayout<KSZ, MB, NM>;
  using R = Roles<GATHER>;
  constexpr int NT = R::THREADS;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  const int nsr = g.nsr, nsl = g.nsl;
  unsigned char *raw = smem;                          // nsr x STAGE
  unsigned char *lo = raw + nsr * Lay::STAGE;         // nsl x STAGE
  unsigned char *bmat = lo + nsl * Lay::STAGE;        // slabs x BROWS x 128 B
  const int nslabs = (g.K + 31) / 32;
  int64_t *o_m = reinterpret_cast<int64_t *>(bmat + nslabs * Lay::BROWS * 128);  // [64 MB]
  int64_t *o_n = o_m + 64 * MB;                                                   // [64]
  int64_t *x_m2 = o_n + 64;                                                       // [32 MB]
  int64_t *x_k = x_m2 + 32 * MB;                                                  // [KSZ]
  uint64_t *bars = reinterpret_cast<uint64_t *>(x_k + KSZ);
  uint64_t *full = bars, *empty = full + kMaxNSR;
  uint64_t *lofull = empty + kMaxNSR, *loempty = lofull + kMaxNSL;
  uint64_t *acc_full = loempty + kMaxNSL, *acc_empty = acc_full + 4;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + 4);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int spt = g.spt;  // stages per tile
  long long wait_cyc[7] = {0, 0, 0, 0, 0, 0, 0};
  const long long t_start = clock64();

  // ---- setup: B'' (K-major, rows 2n+t: hi rows then lo rows), offset tables ----
  for (int i = tid; i < nslabs * Lay::BROWS * 32; i += NT) reinterpret_cast<float *>(bmat)[i] = 0.f;
  __syncthreads();
  for (int i = tid; i < NM * g.K; i += NT) {
    const int row = i / g.K, k = i % g.K;  // row = 2n + t
    const int n = row >> 1, t = row & 1;
    float v = 0.f;
    if (n < g.N) {
      const float2 w = W[g.w_k_off[k] + g.w_n_off[n]];
      v = t ? w.y : w.x;
    }
    // round-to-nearest TF32 hi (exactly representable, so the truncating tensor core uses it as is)
    const float h = __uint_as_float((__float_as_uint(v) + 0x1000u) & 0xFFFFE000u);
    *reinterpret_cast<float *>(bmat + kmajor_off(row, k, Lay::BROWS)) = h;
    *reinterpret_cast<float *>(bmat + kmajor_off(NM + row, k, Lay::BROWS)) = v - h;
  }
  for (int i = tid; i < 64 * MB; i += NT) o_m[i] = g.o_m_off[i];
  for (int i = tid; i < g.N; i += NT) o_n[i] = g.w_n_off[64 + i];
  for (int i = tid; i < 32 * MB; i += NT) x_m2[i] = int64_t(pdep64(uint64_t(2 * i), g.tile_x_mask));
  for (int i = tid; i < KSZ; i += NT) x_k[i] = int64_t(pdep64(uint64_t(i), g.stagek_x_mask));
  if (tid == 0) {
    for (int s = 0; s < nsr; ++s) {
      mbar_init(&full[s], GATHER ? R::LOAD_WARPS : 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < nsl; ++s) {
      mbar_init(&lofull[s], R::LOAD_WARPS);
      mbar_init(&loempty[s], 1);
    }
    for (int a = 0; a < Lay::NACC; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], 2 * kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    if (!GATHER) prefetch_tensormap(&map);
  }
  if (warp == R::MMA_WARP) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(Lay::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B'' -> async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  // each CTA owns a contiguous range of tiles, so outer offsets advance by pdep increments
  const int64_t t_begin = g.n_tiles * blockIdx.x / gridDim.x;
  const int64_t t_end = g.n_tiles * (blockIdx.x + 1) / gridDim.x;

  if (!GATHER && warp == 0) {
    // ---------------- TMA producer ----------------
    if (lane == 0) {
      const uint64_t pol = policy_evict_first();
      RingPos rs;
      uint64_t xt = pdep64(uint64_t(t_begin), g.outer_x_mask);
      for (int64_t t = t_begin; t < t_end; ++t, xt = ((xt | ~g.outer_x_mask) + 1) & g.outer_x_mask) {
        for (int j = 0; j < spt; ++j, rs.next(nsr)) {
          const int s = rs.idx;
          TW(0, mbar_wait(&empty[s], rs.phase ^ 1));
          const uint64_t full_idx = xt | pdep64(uint64_t(j), g.loopk_x_mask);
          int c[5] = {0, 0, 0, 0, 0};
#pragma unroll
          for (int d = 0; d < 5; ++d)
            if (d < g.ndims)
              c[d] = int((full_idx >> g.dim_a[d]) & ((uint64_t(1) << (g.dim_c[d] - g.dim_a[d])) - 1)) *
                     (d == 0 ? 2 : 1);
          mbar_expect_tx(&full[s], Lay::STAGE);
          tma_load_5d(raw + s * Lay::STAGE, &map, &full[s], c, pol);
        }
      }
    }
  } else if (warp == R::MMA_WARP) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t b_base = smem_u32(bmat);
      const uint32_t raw_base = smem_u32(raw), lo_base = smem_u32(lo);
      constexpr uint32_t IDESC = idesc_tf32(NM, true);
      constexpr uint32_t IDESC2 = idesc_tf32(2 * NM, true);
      RingPos rs, rl;
      int i = 0;
      for (int64_t t = t_begin; t < t_end; ++t, ++i) {
        const int a = i % Lay::NACC;
        TW(1, mbar_wait(&acc_empty[a], ((i / Lay::NACC) & 1) ^ 1));
        tc_fence_after();
        const uint32_t acc_base = tmem + uint32_t(a * Lay::ACC);
        for (int j = 0; j < spt; ++j, rs.next(nsr), rl.next(nsl)) {
          const int s = rs.idx, l = rl.idx;
          TW(2, mbar_wait(&full[s], rs.phase));
          TW(3, mbar_wait(&lofull[l], rl.phase));
          tc_fence_after();
#pragma unroll
          for (int q = 0; q < (KSZ + 7) / 8; ++q) {
            const int kg = j * KSZ + q * 8;  // global k of this k-step
            const uint32_t boff = uint32_t((kg >> 5) * Lay::BROWS * 128 + (kg & 31) * 4);
            const uint64_t db = smem_desc(b_base + boff, 16, 1024, 2);
            const uint64_t dbl = smem_desc(b_base + boff + NM * 128, 16, 1024, 2);
            const uint32_t acc_flag = (j == 0 && q == 0) ? 0u : 1u;
#pragma unroll
            for (int b = 0; b < MB; ++b) {
              const uint32_t aoff = uint32_t(4 * b * Lay::LBO + q * 1024);
              // K = 4 stages hold one K atom: SBO = 0 makes the instruction's second atom
              // repeat the first, against B rows k = 4..7 that are zero
              constexpr uint32_t SBO = KSZ >= 8 ? 512 : 0;
              const uint64_t dr = smem_desc(raw_base + s * Lay::STAGE + aoff, Lay::LBO, SBO, 1);
              const uint64_t dl = smem_desc(lo_base + l * Lay::STAGE + aoff, Lay::LBO, SBO, 1);
              const uint32_t d = acc_base + uint32_t(b * Lay::BCOLS);
              if (g.dbg & 2) continue;
              if constexpr (Lay::DUAL) {
                umma_tf32(d, dr, db, IDESC2, acc_flag);
                umma_tf32(d + NM, dl, db, IDESC, 1u);
              } else {
                // one fp32 accumulator: hi*hi, then the hi*lo and lo*hi corrections
                umma_tf32(d, dr, db, IDESC, acc_flag);
                umma_tf32(d, dr, dbl, IDESC, 1u);
                umma_tf32(d, dl, db, IDESC, 1u);
              }
            }
          }
          umma_commit(&empty[s]);
          umma_commit(&loempty[l]);
        }
        umma_commit(&acc_full[a]);
      }
    }
  } else if (warp >= R::LOAD_WARP0 && warp < R::LOAD_WARP0 + R::LOAD_WARPS) {
    const int ct = tid - 32 * R::LOAD_WARP0;  // 0 .. 32 * LOAD_WARPS - 1
    constexpr int LT = 32 * R::LOAD_WARPS;
    constexpr int CPT = Lay::STAGE / 16 / LT;  // 16-byte chunks per thread and stage
    // lo = x - trunc_tf32(x) for this thread's chunks (GATHER) or a strided share (TMA)
    RingPos cs, cl;  // slot of the next stage to convert
    auto convert = [&]() {
      const int s = cs.idx, l = cl.idx;
      TW(4, mbar_wait(&loempty[l], cl.phase ^ 1));
      const float4 *src = reinterpret_cast<const float4 *>(raw + s * Lay::STAGE);
      float4 *dst = reinterpret_cast<float4 *>(lo + l * Lay::STAGE);
      if (!(g.dbg & 4)) {
#pragma unroll
        for (int u = 0; u < CPT; ++u) {
          const int c = ct + u * LT;
          const float4 v = src[c];
          dst[c] = make_float4(v.x - tf32_trunc(v.x), v.y - tf32_trunc(v.y),
                               v.z - tf32_trunc(v.z), v.w - tf32_trunc(v.w));
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) {
        if (GATHER) mbar_arrive(&full[s]);
        mbar_arrive(&lofull[l]);
      }
      cs.next(nsr);
      cl.next(nsl);
    };
    if constexpr (GATHER) {
      // ---------------- loaders: cp.async gather of the X tile, then lo ----------------
      // chunk c = 2 complex m (m pair p) at one k: row r = k + KSZ * (p >> 3) of the
      // MN-major BASE32B operand, 16-byte slot (p & 7) with the 32-byte pair swizzled by k.
      uint32_t dst_off[CPT];
      int64_t src_off[CPT];
#pragma unroll
      for (int u = 0; u < CPT; ++u) {
        const int c = ct + u * LT;
        const int plo = c & 7, r = c >> 3;
        const int k = r % KSZ, mm = r / KSZ;
        dst_off[u] = uint32_t(r * 128 + ((((plo >> 1) ^ (k & 3)) << 5) | ((plo & 1) << 4)));
        src_off[u] = x_m2[mm * 8 + plo] + x_k[k];
      }
      const uint32_t raw_base = smem_u32(raw);
      const int lag = g.lag;
      uint64_t pol;
      asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol));
      int gs = 0;
      RingPos rs;
      uint64_t xtu = pdep64(uint64_t(t_begin), g.outer_x_mask);
      for (int64_t t = t_begin; t < t_end;
           ++t, xtu = ((xtu | ~g.outer_x_mask) + 1) & g.outer_x_mask) {
        const int64_t xt = int64_t(xtu);
        for (int j = 0; j < spt; ++j, ++gs, rs.next(nsr)) {
          const int s = rs.idx;
          mbar_wait(&empty[s], rs.phase ^ 1);
          const float2 *base = X + xt + int64_t(pdep64(uint64_t(j), g.loopk_x_mask));
          const uint32_t sdst = raw_base + uint32_t(s * Lay::STAGE);
#pragma unroll
          for (int u = 0; u < CPT; ++u)
            asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2;" ::"r"(
                             sdst + dst_off[u]),
                         "l"(base + src_off[u]), "l"(pol)
                         : "memory");
          asm volatile("cp.async.commit_group;" ::: "memory");
          if (gs >= lag) {
            cp_async_wait(lag);
            convert();
          }
        }
      }
      asm volatile("cp.async.wait_group 0;" ::: "memory");
      for (int h = gs - lag < 0 ? 0 : gs - lag; h < gs; ++h) convert();
    } else {
      // ---------------- converters (TMA variant) ----------------
      for (int64_t t = t_begin; t < t_end; ++t)
        for (int j = 0; j < spt; ++j) {
          TW(5, mbar_wait(&full[cs.idx], cs.phase));
          convert();
        }
    }
  } else if (warp >= R::EPI_WARP0) {
    // ---------------- epilogue ----------------
    // Two warps per TMEM lane quadrant take alternate 16-column chunks of the tile's
    // accumulator (loaded in batches of up to 4, all in flight together); each warp hands
    // the buffer back as soon as its last batch is in registers, before shuffles and stores.
    constexpr int CH = MB * NM / 16;
    constexpr int MINE = (CH + 1) / 2, BATCH = MINE < 4 ? MINE : 4;
    const int q4 = warp & 3;                       // TMEM lane quadrant of this warp
    const int half = (warp - R::EPI_WARP0) >> 2;   // which alternate chunks
    const int row = 32 * q4 + lane;       // real row 2m + s within a 128-row block
    const int sc = row & 1;
    int i = 0;
    uint64_t oo = pdep64(uint64_t(t_begin), g.outer_o_mask);
    for (int64_t t = t_begin; t < t_end;
         ++t, ++i, oo = ((oo | ~g.outer_o_mask) + 1) & g.outer_o_mask) {
      const int a = i % Lay::NACC;
      TW(6, mbar_wait(&acc_full[a], (i / Lay::NACC) & 1));
      tc_fence_after();
      const int64_t o_outer = int64_t(oo);
      const uint32_t tq = tmem + (uint32_t(32 * q4) << 16) + uint32_t(a * Lay::ACC);
      if (half * 1 >= CH) {  // nothing for this warp (single-chunk tiles)
        tc_fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&acc_empty[a]);
        continue;
      }
#pragma unroll
      for (int j0 = 0; j0 < MINE; j0 += BATCH) {
        float vals[BATCH][16];
        {
          uint32_t vm[BATCH][16], vc[Lay::DUAL ? BATCH : 1][16];
#pragma unroll
          for (int u = 0; u < BATCH; ++u) {
            const int c = 2 * (j0 + u) + half;
            if (c < CH) {
              const int b = c / (NM / 16), cc = (c % (NM / 16)) * 16;
              tmem_ld16(tq + uint32_t(b * Lay::BCOLS + cc), vm[u]);
              if constexpr (Lay::DUAL) tmem_ld16(tq + uint32_t(b * Lay::BCOLS + NM + cc), vc[u]);
            }
          }
          tmem_wait_ld();
#pragma unroll
          for (int u = 0; u < BATCH; ++u)
#pragma unroll
            for (int q = 0; q < 16; ++q) {
              vals[u][q] = __uint_as_float(vm[u][q]);
              if constexpr (Lay::DUAL) vals[u][q] += __uint_as_float(vc[u][q]);
            }
        }
        if (j0 + BATCH >= MINE) {  // all of this warp's TMEM share is in registers
          tc_fence_before();
          __syncwarp();
          if (lane == 0) mbar_arrive(&acc_empty[a]);
        }
#pragma unroll
        for (int u = 0; u < BATCH; ++u) {
          const int c = 2 * (j0 + u) + half;
          if (c >= CH) break;
          const int b = c / (NM / 16), cc = (c % (NM / 16)) * 16;
          float2 *orow = O + o_outer + o_m[64 * b + (row >> 1)];
          float other[16];
#pragma unroll
          for (int q = 0; q < 16; ++q) other[q] = __shfl_xor_sync(0xffffffffu, vals[u][q], 1);
#pragma unroll
          for (int h = 0; h < 4; ++h) {
            const int nl = 4 * sc + h;  // this lane finishes n = cc/2 + nl
            const int n = (cc >> 1) + nl;
            const float xr_wr = sc ? other[2 * nl] : vals[u][2 * nl];
            const float xr_wi = sc ? other[2 * nl + 1] : vals[u][2 * nl + 1];
            const float xi_wr = sc ? vals[u][2 * nl] : other[2 * nl];
            const float xi_wi = sc ? vals[u][2 * nl + 1] : other[2 * nl + 1];
            if (n < g.N && !(g.dbg & 1))
              __stcs(orow + o_n[n], make_float2(xr_wr - xi_wi, xr_wi + xi_wr));
          }
        }
      }
    }
  }
  if ((g.dbg & 32) && blockIdx.x == 0 && lane == 0) {
    const long long tt = clock64() - t_start;
    printf("cta0 warp %2d: total %lld cyc, waits empty %lld acc_empty %lld full %lld lofull %lld "
           "loempty %lld conv_full %lld acc_full %lld\n",
           warp, tt, wait_cyc[0], wait_cyc[1], wait_cyc[2], wait_cyc[3], wait_cyc[4], wait_cyc[5],
           wait_cyc[6]);
  }
  tc_fence_before();
  __syncthreads();
  if (warp == R::MMA_WARP) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(Lay::TMEM_COLS));
  }
}

// Shared memory without the rings, and the ring depths that fit in 227 KiB.
template <int KSZ, int MB, int NM>
size_t tma_smem_bytes(TmaAbsorbGeom &g) {
  using Lay = TmaLayout<KSZ, MB, NM>;
  const int nslabs = (g.K + 31) / 32;
  const size_t fixed = 1024 + size_t(nslabs) * Lay::BROWS * 128 + 8 * (64 * MB + 64 + 32 * MB + KSZ) +
                       8 * (2 * kMaxNSR + 2 * kMaxNSL + 8) + 16;
  const size_t budget = size_t(227) * 1024;
  const int total = int((budget - fixed) / Lay::STAGE);
  g.nsl = total >= 11 ? 4 : 3;
  g.nsr = total - g.nsl;
  if (g.nsr > kMaxNSR) g.nsr = kMaxNSR;
  return fixed + size_t(g.nsr + g.nsl) * Lay::STAGE;
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

template <int KSZ, int MB, int NM, bool GATHER>
cudaError_t launch_tma_impl(const TmaAbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  auto kern = k_absorb_tma<KSZ, MB, NM, GATHER>;
  TmaAbsorbGeom gl = g;
  const size_t smem = tma_smem_bytes<KSZ, MB, NM>(gl);
  if (gl.nsr < (GATHER ? 4 : 2)) return cudaErrorNotSupported;
  gl.lag = gl.nsr - 3 < kMaxLag ? gl.nsr - 3 : kMaxLag;
  static const char *env_lag = stn::debug_opt("tma_lag");  // experiments
  if (env_lag && std::atoi(env_lag) >= 1 && std::atoi(env_lag) <= gl.nsr - 2 &&
      std::atoi(env_lag) <= kMaxLag)
    gl.lag = std::atoi(env_lag);
  static const int dbg = stn::debug_opt("tma_dbg") ? std::atoi(stn::debug_opt("tma_dbg")) : 0;
  gl.dbg = dbg;  // experiments: 1 no stores, 2 no MMAs, 4 no lo conversion
  if (dbg & 8) {  // experiments (wrong results): box order d0, M runs, K runs
    int order[5], n = 0;
    order[n++] = 0;
    for (int d = 1; d < gl.ndims; ++d)
      if (((gl.loopk_x_mask >> gl.dim_a[d]) & 1) == 0 && gl.dim_box[d] > 0 && d >= gl.ndims - 1) order[n++] = d;
    for (int d = 1; d < gl.ndims; ++d) {
      bool used = false;
      for (int i = 0; i < n; ++i) used |= order[i] == d;
      if (!used) order[n++] = d;
    }
    TmaAbsorbGeom t = gl;
    for (int i = 0; i < gl.ndims; ++i) {
      t.dim_a[i] = gl.dim_a[order[i]];
      t.dim_c[i] = gl.dim_c[order[i]];
      t.dim_box[i] = gl.dim_box[order[i]];
    }
    gl = t;
  }
  static bool set_on[kMaxDevices] = {};
  bool &set = set_on[current_device()];
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(227 * 1024));
    if (e != cudaSuccess) return e;
    set = true;
  }
  if (smem > size_t(227 * 1024)) return cudaErrorNotSupported;
  static const char *env_nsr = stn::debug_opt("tma_nsr");  // experiments: raw ring depth
  if (env_nsr && std::atoi(env_nsr) >= 2 && std::atoi(env_nsr) <= gl.nsr) gl.nsr = std::atoi(env_nsr);
  EncodeFn enc = encode_fn();
  if (!enc && !GATHER) return cudaErrorNotSupported;
  const int64_t ctas = g.n_tiles < 148 ? g.n_tiles : 148;
  for (int b = 0; b < p.nbatch; ++b) {
    const float *x = static_cast<const float *>(p.a) + 2 * p.a_bs * b;
    CUtensorMap map;
    std::memset(&map, 0, sizeof map);
    const float2 *w = static_cast<const float2 *>(p.b) + p.b_bs * b;
    float2 *o = static_cast<float2 *>(p.out) + p.out_bs * b;
    if (GATHER) {
      kern<<<unsigned(ctas), Roles<GATHER>::THREADS, smem, stream>>>(
          map, gl, reinterpret_cast<const float2 *>(x), w, o);
      cudaError_t e = cudaGetLastError();
      if (e != cudaSuccess) return e;
      continue;
    }
    cuuint64_t dims[5], strides[4];
    cuuint32_t box[5], es[5] = {1, 1, 1, 1, 1};
    // always rank 5 (the kernel issues 5-D loads): unused dims have extent 1
    int span = 0;
    for (int d = 0; d < g.ndims; ++d) span = g.dim_c[d] > span ? g.dim_c[d] : span;
    for (int d = 0; d < 5; ++d) {
      if (d < g.ndims) {
        const int w = g.dim_c[d] - g.dim_a[d];
        dims[d] = cuuint64_t(1) << (w + (d == 0 ? 1 : 0));
        box[d] = 1u << (g.dim_box[d] + (d == 0 ? 1 : 0));
        if (d > 0) strides[d - 1] = (cuuint64_t(8) << g.dim_a[d]);
      } else {
        dims[d] = 1;
        box[d] = 1;
        strides[d - 1] = cuuint64_t(8) << span;
      }
    }
    CUresult r = enc(&map, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 5,
                     const_cast<float *>(x), dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
                     CU_TENSOR_MAP_SWIZZLE_128B_ATOM_32B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                     CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaErrorNotSupported;
    kern<<<unsigned(ctas), Roles<GATHER>::THREADS, smem, stream>>>(
        map, gl, reinterpret_cast<const float2 *>(x), w, o);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

}  // namespace

bool build_tma_absorb(const std::vector<std::pair<int, int>> &kbits,
                      const std::vector<std::pair<int, int>> &mbits,
                      const std::vector<std::pair<int, int>> &nbits, int xr, TmaAbsorbGeom &g) {
  std::memset(&g, 0, sizeof g);
  const int kb = int(kbits.size()), nb = int(nbits.size());
  if (kb < 2 || kb > 6 || nb < 2 || nb > 6) return false;
  // classes of X positions: 0 = outer M, 1 = tile M, 2 = stage K, 3 = loop K
  std::vector<int> cls(xr, -1), opos(xr, -1);
  for (auto &[xp, op] : mbits) {
    cls[xp] = 0;
    opos[xp] = op;
  }
  for (auto &kw : kbits) cls[kw.first] = 3;
  if (xr < 8 || cls[0] != 0) return false;  // gather granule: 16 B = 2 complex m on X bit 0
  bool tma_ok = true;                        // TMA box rows: X bits 0..3 must be M bits
  for (int p = 0; p < 4; ++p) tma_ok &= cls[p] == 0;
  const int kstage = kb < 5 ? kb : 5;
  const int nm = (2 << nb) < 16 ? 16 : (2 << nb);
  int mbl = 5 - kstage;  // log2 MB: 32 k x 64 m per stage
  while (mbl > 0 && (1 << mbl) * 2 * nm > 256) --mbl;
  if (kstage + mbl < 3) return false;  // stages of >= 4 KiB (one 16-byte chunk per loader)
  const int tm = 6 + mbl;
  // tile M bits: the tm lowest M positions; stage K bits: the kstage lowest K positions
  int got = 0;
  for (int p = 0; p < xr && got < tm; ++p)
    if (cls[p] == 0) {
      cls[p] = 1;
      ++got;
    }
  if (got < tm) return false;
  int kgot = 0;
  for (int p = 0; p < xr && kgot < kstage; ++p)
    if (cls[p] == 3) {
      cls[p] = 2;
      ++kgot;
    }
  // dims: d0 = positions 0..3; then runs of stage-K bits, then runs of tile-M bits
  struct Run {
    int a, b, c, cl;
  };
  std::vector<Run> runs;
  for (int p = 4; p < xr;) {
    if (cls[p] != 1 && cls[p] != 2) {
      ++p;
      continue;
    }
    int q = p;
    while (q < xr && cls[q] == cls[p] && q - p < 8) ++q;
    runs.push_back({p, q, q, cls[p]});
    p = q;
  }
  // outer extent of each run (and of d0): up to the next in-box position
  auto next_inbox = [&](int from) {
    for (int p = from; p < xr; ++p)
      if (cls[p] == 1 || cls[p] == 2) return p;
    return xr;
  };
  std::vector<Run> dims;
  dims.push_back({0, 4, next_inbox(4), 1});
  for (auto &r : runs) r.c = next_inbox(r.b);
  for (auto &r : runs)
    if (r.cl == 2) dims.push_back(r);
  for (auto &r : runs)
    if (r.cl == 1) dims.push_back(r);
  if (dims.size() > 5) tma_ok = false;
  for (auto &d : dims)
    if (d.c - d.a > 31) tma_ok = false;
  g.tma_ok = tma_ok ? 1 : 0;
  g.ndims = tma_ok ? int(dims.size()) : 0;
  for (int d = 0; d < g.ndims; ++d) {
    g.dim_a[d] = dims[d].a;
    g.dim_c[d] = dims[d].c;
    g.dim_box[d] = dims[d].b - dims[d].a;
  }
  // outer masks: outer M bits in X / O (same relative order: canonical layouts), loop K bits
  int n_outer = 0;
  for (int p = 0; p < xr; ++p) {
    if (cls[p] == 0) {
      g.outer_x_mask |= uint64_t(1) << p;
      g.outer_o_mask |= uint64_t(1) << opos[p];
      ++n_outer;
    }
    if (cls[p] == 3) g.loopk_x_mask |= uint64_t(1) << p;
    if (cls[p] == 1) g.tile_x_mask |= uint64_t(1) << p;
    if (cls[p] == 2) g.stagek_x_mask |= uint64_t(1) << p;
  }
  if (n_outer > 40) return false;
  g.n_tiles = int64_t(1) << n_outer;
  g.K = 1 << kb;
  g.N = 1 << nb;
  g.kstage = kstage;
  g.mbl = mbl;
  g.nm = nm;
  g.spt = 1 << (kb - kstage);
  // tile-local m (ascending X position of the tile M bits) -> O offset
  std::vector<int> tile_o;
  for (int p = 0; p < xr; ++p)
    if (cls[p] == 1) tile_o.push_back(opos[p]);
  for (int ml = 0; ml < (64 << mbl); ++ml) {
    int64_t off = 0;
    for (int i = 0; i < tm; ++i)
      if ((ml >> i) & 1) off += int64_t(1) << tile_o[i];
    g.o_m_off[ml] = off;
  }
  // k (ascending X position == stage bits then loop bits) -> W offset; n -> W and O offsets
  for (int k = 0; k < g.K; ++k) {
    int64_t off = 0;
    for (int j = 0; j < kb; ++j)
      if ((k >> j) & 1) off += int64_t(1) << kbits[j].second;
    g.w_k_off[k] = off;
  }
  for (int n = 0; n < g.N; ++n) {
    int64_t woff = 0, ooff = 0;
    for (int j = 0; j < nb; ++j)
      if ((n >> j) & 1) {
        woff += int64_t(1) << nbits[j].second;
        ooff += int64_t(1) << nbits[j].first;
      }
    g.w_n_off[n] = woff;
    g.w_n_off[64 + n] = ooff;
  }
  return true;
}

cudaError_t launch_absorb_tma(const TmaAbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  const int ksz = 1 << g.kstage, mb = 1 << g.mbl;
  // loader: one TMA box per stage where the geometry allows it (measured faster), else the
  // cp.async gather; STN_ABSORB_LOADER=gather forces the gather (experiments)
  const char *ld = stn::debug_opt("absorb_loader");
  const bool use_tma = g.tma_ok && !(ld && std::strcmp(ld, "gather") == 0);
#define STN_TMA(KSZV, MBV, NMV)                                              \
  if (ksz == KSZV && mb == MBV && g.nm == NMV)                               \
    return use_tma ? launch_tma_impl<KSZV, MBV, NMV, false>(g, p, stream)    \
                   : launch_tma_impl<KSZV, MBV, NMV, true>(g, p, stream);
  STN_TMA(32, 1, 16) STN_TMA(32, 1, 32) STN_TMA(32, 1, 64) STN_TMA(32, 1, 128)
  STN_TMA(16, 2, 16) STN_TMA(16, 2, 32) STN_TMA(16, 2, 64) STN_TMA(16, 1, 128)
  STN_TMA(8, 4, 16) STN_TMA(8, 4, 32) STN_TMA(8, 2, 64) STN_TMA(8, 1, 128)
  STN_TMA(4, 8, 16) STN_TMA(4, 4, 32) STN_TMA(4, 2, 64)
#undef STN_TMA
  return cudaErrorNotSupported;
}

}  // namespace stn
