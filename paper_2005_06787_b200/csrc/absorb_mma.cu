// Tensor-core direct absorb (kernels.h DirectGeom, FAST mode):
//   O[m, n] = sum_k X[m, k] * W[k, n]      (complex64, K <= 64, N <= 64)
// on stems whose lowest L >= 2 bits are M bits at identical positions in X and
// O (the same geometry the SIMT direct kernel streams).
//
// The SIMT kernels spend 4*K FFMA per output element; from K*N >= 64 that, not
// HBM, bounds a stem pass (runtime.hpp:439-448 runs these steps as plain
// GEMMs). Here the contraction runs on tcgen05 in a de-interleaved real form
//   A'[2m+s][k]   = component s of X[m, k]        (M_mma = 128 = 64 complex m)
//   B'[2n+t][k]   = component t of W[k, n]        (N_mma = 2N, K-major)
//   D'[2m+s][2n+t] = sum_k A' B'
//   O[m, n] = (D'[2m][2n] - D'[2m+1][2n+1],  D'[2m][2n+1] + D'[2m+1][2n])
// with split-TF32 (hi*hi into one TMEM accumulator, hi*lo + lo*hi into a
// second), which keeps fp32-level accuracy.
//
// Warp roles of the persistent CTA (one per SM):
//   warps 0-3   epilogue: TMEM -> registers, pair rows 2m / 2m+1 with a lane
//               shuffle, stream the complex outputs to HBM;
//   warp  4     TMEM allocation + the single MMA-issuing thread;
//   warps 5-12  loaders: X tile (64 m x K) from HBM with 32-byte loads, split
//               into TF32 hi/lo, written into a ring of K-major SWIZZLE_128B
//               A' stages.
// mbarriers order the ring (full / empty) and the two TMEM accumulator
// buffers (acc_full / acc_empty), so loads of tile i+1.., the MMAs of tile i
// and the epilogue of tile i-1 overlap.
#include <cuda_runtime.h>

#include <cstdint>
#include <cstdlib>

#include "kernels.h"

namespace stn {

namespace {

constexpr int kMmaRowsC = 64;     // complex m per tile (M_mma = 128 real rows)
constexpr int kLoaderWarps = 8;
constexpr int kEpiWarps = 4;
constexpr int kThreads = 32 * (kEpiWarps + 1 + kLoaderWarps);
constexpr int kLoaderThreads = 32 * kLoaderWarps;

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
// TF32 "hi" part of x: round to nearest (ties away) on the 13 dropped bits,
// without the special-value branch of cvt.rna.tf32.f32; x - hi is exact.
__device__ __forceinline__ float tf32_hi(float x) {
  return __uint_as_float((__float_as_uint(x) + 0x1000u) & 0xFFFFE000u);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
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
// K-major SWIZZLE_128B descriptor: 8-row x 128 B atoms every 1024 B.
__device__ __forceinline__ uint64_t smem_desc_sw128(uint32_t saddr) {
  uint64_t d = 0;
  d |= uint64_t((saddr >> 4) & 0x3FFFu);
  d |= uint64_t(1) << 16;
  d |= uint64_t(1024 >> 4) << 32;
  d |= uint64_t(1) << 46;
  d |= uint64_t(2) << 61;
  return d;
}
__device__ __forceinline__ void tmem_ld16(uint32_t taddr, uint32_t (&v)[16]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x16.b32"
      "{%0, %1, %2, %3, %4, %5, %6, %7, %8, %9, %10, %11, %12, %13, %14, %15}, [%16];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]), "=r"(v[6]),
        "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]), "=r"(v[12]), "=r"(v[13]),
        "=r"(v[14]), "=r"(v[15])
      : "r"(taddr));
}
// Byte offset of real element (row, col) in a K-major SWIZZLE_128B plane made
// of 32-column slabs of `rows` x 128 B.
__device__ __forceinline__ uint32_t sw128_off(int row, int col, int rows) {
  const int slab = col >> 5, cc = col & 31;
  const int chunk = (cc >> 2) ^ (row & 7);
  return uint32_t(slab * rows * 128 + row * 128 + chunk * 16 + (cc & 3) * 4);
}

// KP: real K padded to the 32-column slab (32 or 64); NM: N_mma = 2N padded
// to >= 16; STAGES: A' ring depth.
template <int KP, int NM>
struct MmaLayout {
  static constexpr int STAGES = KP == 64 ? 2 : 4;
  static constexpr int ACC = NM == 128 ? 2 : 4;  // TMEM accumulator buffers (2 x NM columns each)
  static constexpr int GI = NM == 128 ? 1 : 2;   // tiles whose MMA chains are interleaved
  static constexpr int A_PLANE = 128 * KP * 4;
  static constexpr int B_PLANE = NM * KP * 4;
  static constexpr int STAGE_BYTES = 2 * A_PLANE;
  static constexpr int TMEM_COLS = (2 * ACC * NM) <= 32 ? 32 : ((2 * ACC * NM) <= 64 ? 64 : ((2 * ACC * NM) <= 128 ? 128 : ((2 * ACC * NM) <= 256 ? 256 : 512)));
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (uint32_t(NM >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  // pdep byte tables for the high M bits of X and O (5 bytes cover 40 bits)
  static constexpr int TABLE_BYTES = 2 * 5 * 256 * 8;
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * size_t(B_PLANE) +
                                 TABLE_BYTES + 8 * 64 /*xko*/ + 8 * 64 /*ono*/ + 256;
};

__device__ __forceinline__ int64_t pdep_tab(const int64_t *tab, uint64_t v) {
  return tab[v & 255] | tab[256 + ((v >> 8) & 255)] | tab[512 + ((v >> 16) & 255)] |
         tab[768 + ((v >> 24) & 255)] | tab[1024 + ((v >> 32) & 255)];
}

// KB = log2 K (4..6): K-padding KP, loader items per thread and tile
// (IPT = K / 16) and the register prefetch depth (D tiles, 8 items in flight).
template <int KB, int NM>
__global__ void __launch_bounds__(kThreads, 1)
    k_absorb_mma(const __grid_constant__ DirectGeom g, const BatchPtrs p, int64_t n_tiles, int dbg) {
  constexpr int KP = KB == 6 ? 64 : 32;
  constexpr int IPT = 1 << (KB - 4);
  constexpr int D = 8 / IPT;
  using Lay = MmaLayout<KP, NM>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align inside the shared window (keeps the pointer in the shared address
  // space, so the compiler emits STS/LDS rather than generic ST/LD)
  unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char *a_ring = smem;                                     // STAGES x {hi, lo}
  unsigned char *b_hi = a_ring + Lay::STAGES * Lay::STAGE_BYTES;
  unsigned char *b_lo = b_hi + Lay::B_PLANE;
  int64_t *tab_x = reinterpret_cast<int64_t *>(b_lo + Lay::B_PLANE);  // [5][256]
  int64_t *tab_o = tab_x + 5 * 256;
  int64_t *xko = tab_o + 5 * 256;  // [K] X offset of k
  int64_t *ono = xko + 64;         // [N] O offset of n
  uint64_t *bars = reinterpret_cast<uint64_t *>(ono + 64);
  uint64_t *full = bars, *empty = bars + Lay::STAGES;
  uint64_t *acc_full = empty + Lay::STAGES, *acc_empty = acc_full + Lay::ACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + Lay::ACC);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int K = 1 << g.kb, N = 1 << g.nb, L = g.L;
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  // ---- setup: pdep tables, k / n offsets, zeroed A' ring (K padding), B' ----
  for (int i = tid; i < 2 * 5 * 256; i += kThreads) {
    const bool ox = i < 5 * 256;
    const int j = ox ? i : i - 5 * 256;
    const uint64_t mask = ox ? g.hi_x_mask : g.hi_o_mask;
    const uint64_t v = uint64_t(j & 255) << (8 * (j >> 8));
    uint64_t r = 0, m = mask;
    for (uint64_t bit = 1; m; bit <<= 1) {
      const uint64_t low = m & (0 - m);
      if (v & bit) r |= low;
      m ^= low;
    }
    (ox ? tab_x : tab_o)[j] = int64_t(r);
  }
  for (int k = tid; k < K; k += kThreads) {
    int64_t off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off += int64_t(1) << g.k_xpos[j];
    xko[k] = off;
  }
  for (int n = tid; n < N; n += kThreads) {
    int64_t off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off += int64_t(1) << g.n_opos[j];
    ono[n] = off;
  }
  for (int i = tid; i < Lay::STAGES * Lay::STAGE_BYTES / 16; i += kThreads)
    reinterpret_cast<float4 *>(a_ring)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = tid; i < NM * KP; i += kThreads) {
    const int row = i / KP, k = i % KP;  // row = 2n + t
    const int n = row >> 1, t = row & 1;
    float v = 0.f;
    if (n < N && k < K) {
      int64_t off = 0;
      for (int j = 0; j < g.kb; ++j)
        if ((k >> j) & 1) off += g.w_k_stride[j];
      for (int j = 0; j < g.nb; ++j)
        if ((n >> j) & 1) off += g.w_n_stride[j];
      const float2 w = W[off];
      v = t ? w.y : w.x;
    }
    const float vh = tf32_round(v);
    const uint32_t o = sw128_off(row, k, NM);
    *reinterpret_cast<float *>(b_hi + o) = vh;
    *reinterpret_cast<float *>(b_lo + o) = v - vh;
  }
  if (tid == 0) {
    for (int s = 0; s < Lay::STAGES; ++s) {
      mbar_init(&full[s], kLoaderWarps);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < Lay::ACC; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kEpiWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(Lay::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");  // B' and zeroed A' -> async proxy
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int lmask = (1 << L) - 1;
  const int64_t G = gridDim.x;

  if (warp > kEpiWarps) {
    // ---------------- loaders ----------------
    // Item = (quad of 4 consecutive m, k): one 32-byte load (2 x float4), 8
    // TF32 values into each of the hi / lo planes. Consecutive lanes take
    // consecutive k, so the stores of a warp walk along a swizzled row.
    const int lt = tid - 32 * (kEpiWarps + 1);
    struct Regs {
      float4 v0[IPT], v1[IPT];
    };
    // loads of one tile into registers (issued, not waited on); item
    // e = lt + u * 256 -> (quad q = e / K, k = e % K)
    auto load = [&](int64_t tl, Regs &r) {
      if (tl >= n_tiles) return;
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int e = lt + u * kLoaderThreads;
        const int k = e & (K - 1), q = e >> KB;
        const int64_t m = tl * kMmaRowsC + 4 * q;
        const int64_t off = pdep_tab(tab_x, uint64_t(m >> L)) + (m & lmask) + xko[k];
        const float4 *src = reinterpret_cast<const float4 *>(X + off);
        if (dbg & 2) {
          r.v0[u] = make_float4(float(off & 7), 0.f, 0.f, 0.f);
          r.v1[u] = r.v0[u];
        } else {
          r.v0[u] = __ldcs(src);
          r.v1[u] = __ldcs(src + 1);
        }
      }
    };
    // split into the A' stage of tile number i and hand it to the MMA thread
    auto put = [&](int i, const Regs &r) {
      const int s = i % Lay::STAGES;
      mbar_wait(&empty[s], ((i / Lay::STAGES) & 1) ^ 1);
      unsigned char *ahi = a_ring + s * Lay::STAGE_BYTES;
      unsigned char *alo = ahi + Lay::A_PLANE;
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int e = lt + u * kLoaderThreads;
        const int k = e & (K - 1), q = e >> KB;
        const float vals[8] = {r.v0[u].x, r.v0[u].y, r.v0[u].z, r.v0[u].w,
                               r.v1[u].x, r.v1[u].y, r.v1[u].z, r.v1[u].w};
#pragma unroll
        for (int j = 0; j < 8; ++j) {  // real row 8q + j = 2m + s
          const uint32_t o = sw128_off(8 * q + j, k, 128);
          const float h = tf32_hi(vals[j]);
          *reinterpret_cast<float *>(ahi + o) = h;
          *reinterpret_cast<float *>(alo + o) = vals[j] - h;
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    };
    // D tiles of loads in flight per thread (a register ring, unrolled)
    Regs ring[D];
#pragma unroll
    for (int d = 0; d < D; ++d) load(blockIdx.x + d * G, ring[d]);
    for (int base = 0;; base += D) {
      bool done = false;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int i = base + d;
        const int64_t tl = blockIdx.x + int64_t(i) * G;
        if (tl >= n_tiles) {
          done = true;
          break;
        }
        put(i, ring[d]);
        load(tl + D * G, ring[d]);
      }
      if (done) break;
    }
  } else if (warp == kEpiWarps) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      // A dependent chain of small MMAs runs at its latency, not at the tensor
      // pipe's rate; the chains of GI consecutive tiles are issued interleaved.
      const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
      for (int i0 = 0;; i0 += Lay::GI) {
        int cnt = 0;
        uint32_t ah[Lay::GI], tmain[Lay::GI];
#pragma unroll
        for (int t = 0; t < Lay::GI; ++t) {
          const int i = i0 + t;
          if (blockIdx.x + int64_t(i) * G >= n_tiles) break;
          const int s = i % Lay::STAGES, a = i % Lay::ACC;
          mbar_wait(&acc_empty[a], ((i / Lay::ACC) & 1) ^ 1);
          mbar_wait(&full[s], (i / Lay::STAGES) & 1);
          ah[t] = smem_u32(a_ring + s * Lay::STAGE_BYTES);
          tmain[t] = tmem + uint32_t(a * 2 * NM);
          cnt = t + 1;
        }
        if (cnt == 0) break;
        tc_fence_after();
#pragma unroll
        for (int slab = 0; slab < KP / 32; ++slab) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t ao = slab * 128 * 128 + j * 32, bo = slab * NM * 128 + j * 32;
            const uint32_t acc = (slab == 0 && j == 0) ? 0u : 1u;
            const uint64_t dbh = smem_desc_sw128(bh + bo), dbl = smem_desc_sw128(bl + bo);
#pragma unroll
            for (int t = 0; t < Lay::GI; ++t) {
              if (t >= cnt) break;
              const uint64_t dah = smem_desc_sw128(ah[t] + ao);
              const uint64_t dal = smem_desc_sw128(ah[t] + Lay::A_PLANE + ao);
              if (dbg & 1) continue;
              umma_tf32(tmain[t], dah, dbh, Lay::IDESC, acc);
              umma_tf32(tmain[t] + NM, dah, dbl, Lay::IDESC, acc);
              umma_tf32(tmain[t] + NM, dal, dbh, Lay::IDESC, 1u);
            }
          }
        }
#pragma unroll
        for (int t = 0; t < Lay::GI; ++t) {
          if (t >= cnt) break;
          umma_commit(&empty[(i0 + t) % Lay::STAGES]);
          umma_commit(&acc_full[(i0 + t) % Lay::ACC]);
        }
        if (cnt < Lay::GI) break;
      }
    }
  } else {
    // ---------------- epilogue ----------------
    const int row = 32 * warp + lane;  // real row 2m + s of the tile
    const int r = row >> 1, sc = row & 1;
    int i = 0;
    for (int64_t tl = blockIdx.x; tl < n_tiles; tl += G, ++i) {
      const int a = i % Lay::ACC;
      mbar_wait(&acc_full[a], (i / Lay::ACC) & 1);
      tc_fence_after();
      const int64_t m = tl * kMmaRowsC + r;
      float2 *orow = O + pdep_tab(tab_o, uint64_t(m >> L)) + (m & lmask);
      const uint32_t tbase = tmem + (uint32_t(32 * warp) << 16) + uint32_t(a * 2 * NM);
      // rows 2m (Xr . W) and 2m+1 (Xi . W) sit in neighbouring lanes; each of
      // the two lanes finishes half of every 8-output group.
#pragma unroll
      for (int c0 = 0; c0 < NM; c0 += 16) {
        uint32_t vm[16], vc[16];
        tmem_ld16(tbase + uint32_t(c0), vm);
        tmem_ld16(tbase + uint32_t(NM + c0), vc);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
        float vals[16], other[16];
#pragma unroll
        for (int q = 0; q < 16; ++q) vals[q] = __uint_as_float(vm[q]) + __uint_as_float(vc[q]);
#pragma unroll
        for (int q = 0; q < 16; ++q) other[q] = __shfl_xor_sync(0xffffffffu, vals[q], 1);
#pragma unroll
        for (int h = 0; h < 4; ++h) {
          const int nl = 4 * sc + h;  // local n within the 8-group
          const int n = (c0 >> 1) + nl;
          const float er = sc ? other[2 * nl] : vals[2 * nl];           // Xr.Wr
          const float ei = sc ? other[2 * nl + 1] : vals[2 * nl + 1];   // Xr.Wi
          const float odr = sc ? vals[2 * nl] : other[2 * nl];          // Xi.Wr
          const float odi = sc ? vals[2 * nl + 1] : other[2 * nl + 1];  // Xi.Wi
          if (n < N && !(dbg & 4)) __stcs(orow + ono[n], make_float2(er - odi, ei + odr));
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kEpiWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(Lay::TMEM_COLS));
  }
}

template <int KB, int NM>
cudaError_t launch_mma_impl(const DirectGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  using Lay = MmaLayout<KB == 6 ? 64 : 32, NM>;
  auto kern = k_absorb_mma<KB, NM>;
  static bool set_on[kMaxDevices] = {};
  bool &set = set_on[current_device()];
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(Lay::SMEM));
    if (e != cudaSuccess) return e;
    set = true;
  }
  const int64_t n_tiles = int64_t(1) << (g.L + g.mh_bits - 6);
  int64_t ctas = 148 / (p.nbatch > 0 ? p.nbatch : 1);
  if (ctas < 1) ctas = 1;
  if (ctas > n_tiles) ctas = n_tiles;
  dim3 grid(unsigned(ctas), unsigned(p.nbatch));
  static const int dbg = stn::debug_opt("mma_dbg") ? std::atoi(stn::debug_opt("mma_dbg")) : 0;
  kern<<<grid, kThreads, Lay::SMEM, stream>>>(g, p, n_tiles, dbg);
  return cudaGetLastError();
}


// ---------------------------------------------------------------------------
// Interleaved variant for K in {16, 32}: complex rows stay whole,
//   A''[m][2k+s]   = component s of X[m, k]                (K-major, 2K real)
//   B''[2n+t][2k+s] = [[wr, -wi], [wi, wr]][t][s] of W[k, n]
//   D[m][2n+t]     = sum A'' B''  = (Re, Im) of O[m, n]
// so an M_mma = 128 block covers 128 complex m, the epilogue needs no lane
// exchange, and the loader writes (re, im) pairs with 8-byte stores. A tile is
// MB such blocks (MB = 2 for K = 16) to amortise the per-tile handshakes.
// Same warp roles and barriers as k_absorb_mma.
// ---------------------------------------------------------------------------
template <int KB, int NM>
struct Mma2Layout {
  static constexpr int K = 1 << KB;
  static constexpr int KP = 2 * K;                       // real K: 32 or 64
  static constexpr int MB = (K == 16 && NM <= 64) ? 2 : 1;  // 128-row blocks per tile
  static constexpr int STAGES = 2;
  static constexpr int ACC = 2;
  static constexpr int A_BLOCK = 128 * KP * 4;           // one plane of one block
  static constexpr int STAGE_BYTES = 2 * MB * A_BLOCK;   // {hi, lo} x MB blocks
  static constexpr int B_PLANE = NM * KP * 4;
  static constexpr int COLS = ACC * MB * 2 * NM;
  static constexpr int TMEM_COLS = COLS <= 32 ? 32 : (COLS <= 64 ? 64 : (COLS <= 128 ? 128 : (COLS <= 256 ? 256 : 512)));
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) |
                                    (uint32_t(NM >> 3) << 17) | (uint32_t(128 >> 4) << 24);
  static constexpr int TABLE_BYTES = 2 * 5 * 256 * 8;
  static constexpr size_t SMEM = 1024 + size_t(STAGES) * STAGE_BYTES + 2 * size_t(B_PLANE) +
                                 TABLE_BYTES + 8 * 64 + 8 * 64 + 256;
  static constexpr int ROWS = 128 * MB;                  // complex m per tile
};

template <int KB, int NM>
__global__ void __launch_bounds__(kThreads, 1)
    k_absorb_mma2(const __grid_constant__ DirectGeom g, const BatchPtrs p, int64_t n_tiles) {
  using Lay = Mma2Layout<KB, NM>;
  constexpr int K = Lay::K, KP = Lay::KP, MB = Lay::MB;
  constexpr int IPT = 32 * MB * K / kLoaderThreads;  // quads x K items per loader thread
  constexpr int D = IPT >= 4 ? 2 : 8 / IPT;           // tiles of loads in flight
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char *a_ring = smem;
  unsigned char *b_hi = a_ring + Lay::STAGES * Lay::STAGE_BYTES;
  unsigned char *b_lo = b_hi + Lay::B_PLANE;
  int64_t *tab_x = reinterpret_cast<int64_t *>(b_lo + Lay::B_PLANE);
  int64_t *tab_o = tab_x + 5 * 256;
  int64_t *xko = tab_o + 5 * 256;
  int64_t *ono = xko + 64;
  uint64_t *bars = reinterpret_cast<uint64_t *>(ono + 64);
  uint64_t *full = bars, *empty = bars + Lay::STAGES;
  uint64_t *acc_full = empty + Lay::STAGES, *acc_empty = acc_full + Lay::ACC;
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(acc_empty + Lay::ACC);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int N = 1 << g.nb, L = g.L;
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  for (int i = tid; i < 2 * 5 * 256; i += kThreads) {
    const bool ox = i < 5 * 256;
    const int j = ox ? i : i - 5 * 256;
    const uint64_t mask = ox ? g.hi_x_mask : g.hi_o_mask;
    const uint64_t v = uint64_t(j & 255) << (8 * (j >> 8));
    uint64_t r = 0, m = mask;
    for (uint64_t bit = 1; m; bit <<= 1) {
      const uint64_t low = m & (0 - m);
      if (v & bit) r |= low;
      m ^= low;
    }
    (ox ? tab_x : tab_o)[j] = int64_t(r);
  }
  for (int k = tid; k < K; k += kThreads) {
    int64_t off = 0;
    for (int j = 0; j < KB; ++j)
      if ((k >> j) & 1) off += int64_t(1) << g.k_xpos[j];
    xko[k] = off;
  }
  for (int n = tid; n < N; n += kThreads) {
    int64_t off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off += int64_t(1) << g.n_opos[j];
    ono[n] = off;
  }
  for (int i = tid; i < NM * KP; i += kThreads) {
    const int row = i / KP, c = i % KP;  // row = 2n + t, c = 2k + s
    const int n = row >> 1, t = row & 1, k = c >> 1, sc = c & 1;
    float v = 0.f;
    if (n < N) {
      int64_t off = 0;
      for (int j = 0; j < KB; ++j)
        if ((k >> j) & 1) off += g.w_k_stride[j];
      for (int j = 0; j < g.nb; ++j)
        if ((n >> j) & 1) off += g.w_n_stride[j];
      const float2 w = W[off];
      v = t == 0 ? (sc == 0 ? w.x : -w.y) : (sc == 0 ? w.y : w.x);
    }
    const float vh = tf32_hi(v);
    const uint32_t o = sw128_off(row, c, NM);
    *reinterpret_cast<float *>(b_hi + o) = vh;
    *reinterpret_cast<float *>(b_lo + o) = v - vh;
  }
  if (tid == 0) {
    for (int s = 0; s < Lay::STAGES; ++s) {
      mbar_init(&full[s], kLoaderWarps);
      mbar_init(&empty[s], 1);
    }
    for (int a = 0; a < Lay::ACC; ++a) {
      mbar_init(&acc_full[a], 1);
      mbar_init(&acc_empty[a], kEpiWarps);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == kEpiWarps) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(Lay::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  const int lmask = (1 << L) - 1;
  const int64_t G = gridDim.x;

  if (warp > kEpiWarps) {
    // ---------------- loaders: item = (quad of 4 m, k) ----------------
    const int lt = tid - 32 * (kEpiWarps + 1);
    struct Regs {
      float4 v0[IPT], v1[IPT];
    };
    auto load = [&](int64_t tl, Regs &r) {
      if (tl >= n_tiles) return;
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int e = lt + u * kLoaderThreads;
        const int k = e & (K - 1), q = e >> KB;
        const int64_t m = tl * Lay::ROWS + 4 * q;
        const int64_t off = pdep_tab(tab_x, uint64_t(m >> L)) + (m & lmask) + xko[k];
        const float4 *src = reinterpret_cast<const float4 *>(X + off);
        r.v0[u] = __ldcs(src);
        r.v1[u] = __ldcs(src + 1);
      }
    };
    auto put = [&](int i, const Regs &r) {
      const int s = i % Lay::STAGES;
      mbar_wait(&empty[s], ((i / Lay::STAGES) & 1) ^ 1);
      unsigned char *st = a_ring + s * Lay::STAGE_BYTES;
#pragma unroll
      for (int u = 0; u < IPT; ++u) {
        const int e = lt + u * kLoaderThreads;
        const int k = e & (K - 1), q = e >> KB;
        const int blk = (4 * q) >> 7, row0 = (4 * q) & 127;
        unsigned char *hi = st + blk * 2 * Lay::A_BLOCK, *lo = hi + Lay::A_BLOCK;
        const float4 v[2] = {r.v0[u], r.v1[u]};
#pragma unroll
        for (int j = 0; j < 4; ++j) {  // m = 4q + j: (re, im) at (row, 2k)
          const float re = (j & 1) ? v[j >> 1].z : v[j >> 1].x;
          const float im = (j & 1) ? v[j >> 1].w : v[j >> 1].y;
          const uint32_t o = sw128_off(row0 + j, 2 * k, 128);
          const float rh = tf32_hi(re), ih = tf32_hi(im);
          *reinterpret_cast<float2 *>(hi + o) = make_float2(rh, ih);
          *reinterpret_cast<float2 *>(lo + o) = make_float2(re - rh, im - ih);
        }
      }
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      __syncwarp();
      if (lane == 0) mbar_arrive(&full[s]);
    };
    Regs ring[D];
#pragma unroll
    for (int d = 0; d < D; ++d) load(blockIdx.x + d * G, ring[d]);
    for (int base = 0;; base += D) {
      bool done = false;
#pragma unroll
      for (int d = 0; d < D; ++d) {
        const int i = base + d;
        const int64_t tl = blockIdx.x + int64_t(i) * G;
        if (tl >= n_tiles) {
          done = true;
          break;
        }
        put(i, ring[d]);
        load(tl + D * G, ring[d]);
      }
      if (done) break;
    }
  } else if (warp == kEpiWarps) {
    // ---------------- MMA issuer ----------------
    if (lane == 0) {
      const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
      int i = 0;
      for (int64_t tl = blockIdx.x; tl < n_tiles; tl += G, ++i) {
        const int s = i % Lay::STAGES, a = i % Lay::ACC;
        mbar_wait(&acc_empty[a], ((i / Lay::ACC) & 1) ^ 1);
        mbar_wait(&full[s], (i / Lay::STAGES) & 1);
        tc_fence_after();
        const uint32_t st = smem_u32(a_ring + s * Lay::STAGE_BYTES);
#pragma unroll
        for (int slab = 0; slab < KP / 32; ++slab) {
#pragma unroll
          for (int j = 0; j < 4; ++j) {
            const uint32_t ao = slab * 128 * 128 + j * 32, bo = slab * NM * 128 + j * 32;
            const uint32_t acc = (slab == 0 && j == 0) ? 0u : 1u;
            const uint64_t dbh = smem_desc_sw128(bh + bo), dbl = smem_desc_sw128(bl + bo);
#pragma unroll
            for (int blk = 0; blk < MB; ++blk) {  // independent chains, interleaved
              const uint32_t ah = st + blk * 2 * Lay::A_BLOCK, al = ah + Lay::A_BLOCK;
              const uint32_t tm = tmem + uint32_t((a * MB + blk) * 2 * NM);
              const uint64_t dah = smem_desc_sw128(ah + ao), dal = smem_desc_sw128(al + ao);
              umma_tf32(tm, dah, dbh, Lay::IDESC, acc);
              umma_tf32(tm + NM, dah, dbl, Lay::IDESC, acc);
              umma_tf32(tm + NM, dal, dbh, Lay::IDESC, 1u);
            }
          }
        }
        umma_commit(&empty[s]);
        umma_commit(&acc_full[a]);
      }
    }
  } else {
    // ---------------- epilogue: lane = complex row ----------------
    int i = 0;
    for (int64_t tl = blockIdx.x; tl < n_tiles; tl += G, ++i) {
      const int a = i % Lay::ACC;
      mbar_wait(&acc_full[a], (i / Lay::ACC) & 1);
      tc_fence_after();
#pragma unroll
      for (int blk = 0; blk < MB; ++blk) {
        const int64_t m = tl * Lay::ROWS + blk * 128 + 32 * warp + lane;
        float2 *orow = O + pdep_tab(tab_o, uint64_t(m >> L)) + (m & lmask);
        const uint32_t tb = tmem + (uint32_t(32 * warp) << 16) + uint32_t((a * MB + blk) * 2 * NM);
#pragma unroll
        for (int c0 = 0; c0 < NM; c0 += 16) {
          uint32_t vm[16], vc[16];
          tmem_ld16(tb + uint32_t(c0), vm);
          tmem_ld16(tb + uint32_t(NM + c0), vc);
          asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
          for (int q = 0; q < 8; ++q) {
            const int n = (c0 >> 1) + q;
            if (n < N)
              __stcs(orow + ono[n],
                     make_float2(__uint_as_float(vm[2 * q]) + __uint_as_float(vc[2 * q]),
                                 __uint_as_float(vm[2 * q + 1]) + __uint_as_float(vc[2 * q + 1])));
          }
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&acc_empty[a]);
    }
  }
  tc_fence_before();
  __syncthreads();
  if (warp == kEpiWarps) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(Lay::TMEM_COLS));
  }
}

template <int KB, int NM>
cudaError_t launch_mma2_impl(const DirectGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  using Lay = Mma2Layout<KB, NM>;
  auto kern = k_absorb_mma2<KB, NM>;
  static bool set_on[kMaxDevices] = {};
  bool &set = set_on[current_device()];
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(Lay::SMEM));
    if (e != cudaSuccess) return e;
    set = true;
  }
  const int64_t n_tiles = (int64_t(1) << (g.L + g.mh_bits)) / Lay::ROWS;
  int64_t ctas = 148 / (p.nbatch > 0 ? p.nbatch : 1);
  if (ctas < 1) ctas = 1;
  if (ctas > n_tiles) ctas = n_tiles;
  dim3 grid(unsigned(ctas), unsigned(p.nbatch));
  kern<<<grid, kThreads, Lay::SMEM, stream>>>(g, p, n_tiles);
  return cudaGetLastError();
}

}  // namespace

bool mma_absorb_supported(const DirectGeom &g) {
  return g.L >= 2 && g.kb >= 4 && g.kb <= 6 && g.nb <= 6 && g.L + g.mh_bits >= 8 &&
         g.mh_bits <= 40;
}

cudaError_t launch_absorb_mma(const DirectGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  if (!mma_absorb_supported(g)) return cudaErrorNotSupported;
  const int nm = (2 << g.nb) < 16 ? 16 : (2 << g.nb);
  static const char *force1 = stn::debug_opt("mma_v1");  // experiments: de-interleaved kernel only
  if (!force1 && g.kb <= 5) {  // interleaved kernel: whole complex rows, larger tiles
#define STN_MMA2(KBV, NMV) \
  if (g.kb == KBV && nm == NMV) return launch_mma2_impl<KBV, NMV>(g, p, stream);
    STN_MMA2(4, 16) STN_MMA2(4, 32) STN_MMA2(4, 64) STN_MMA2(4, 128)
    STN_MMA2(5, 16) STN_MMA2(5, 32) STN_MMA2(5, 64) STN_MMA2(5, 128)
#undef STN_MMA2
  }
#define STN_MMA(KBV, NMV) \
  if (g.kb == KBV && nm == NMV) return launch_mma_impl<KBV, NMV>(g, p, stream);
#define STN_MMA_ROW(KBV) STN_MMA(KBV, 16) STN_MMA(KBV, 32) STN_MMA(KBV, 64) STN_MMA(KBV, 128)
  STN_MMA_ROW(4) STN_MMA_ROW(5) STN_MMA_ROW(6)
#undef STN_MMA_ROW
#undef STN_MMA
  return cudaErrorNotSupported;
}

}  // namespace stn
