// tcgen05 "absorb": bond-2 stem step O[t, n] = sum_k X[t, k] * W[k, n] with a
// small branch W (K <= 32, N <= 64 complex) on the 5th-generation tensor cores.
//
// Same tiling as the SIMT absorb (kernels.h AbsorbGeom, T = 7 bits = 128 rows):
// each CTA streams X tiles (128 rows x K) from HBM with 16 B loads, splits
// them on the fly into TF32 hi/lo planes laid out as the UMMA K-major
// SWIZZLE_128B canonical layout, and one thread issues the split-TF32 MMAs
//   acc_main  = Xhi . W''hi            (128 x 2N x 2K real)
//   acc_corr  = Xhi . W''lo + Xlo . W''hi
// into TMEM (W'' = the 2N x 2K real expansion of W, built once per CTA).
// The epilogue reads TMEM (tcgen05.ld), adds the two accumulators and scatters
// the 128 x N complex outputs into the O tile in shared memory, which is then
// written with coalesced 16 B stores. Tensor work per tile is a few hundred
// cycles; the kernel is bound by the HBM stream like the SIMT absorb, but its
// instruction count no longer grows with K * N.
#include <cuda_runtime.h>

#include <cstdint>

#include "kernels.h"

namespace stn {

namespace {

constexpr int kThreads = 128;
constexpr int kRows = 128;  // UMMA M = tile rows (T = 7 bits)

__device__ __forceinline__ uint32_t smem_u32(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ float tf32_round(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}
__device__ __forceinline__ void mbar_init(uint64_t *bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
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

template <int KP, int NP>
struct TcAbsorbLayout {
  static constexpr int AK = 2 * KP;  // real K (multiple of 32)
  static constexpr int BN = 2 * NP;  // real N (multiple of 16)
  static constexpr int A_PLANE = kRows * AK * 4;
  static constexpr int B_PLANE = BN * AK * 4;
  static constexpr int TMEM_COLS = (2 * BN) <= 32 ? 32 : ((2 * BN) <= 64 ? 64 : ((2 * BN) <= 128 ? 128 : 256));
  static constexpr uint32_t IDESC = (1u << 4) | (2u << 7) | (2u << 10) | (uint32_t(BN >> 3) << 17) |
                                    (uint32_t(kRows >> 4) << 24);
};

template <int KP, int NP>
__global__ void __launch_bounds__(kThreads, 1)
    k_absorb_tc(const __grid_constant__ AbsorbGeom g, const BatchPtrs p, int64_t n_tiles) {
  using L = TcAbsorbLayout<KP, NP>;
  extern __shared__ __align__(1024) unsigned char smem_raw[];
  // align inside the shared window (keeps the pointer in the shared address
  // space, so the compiler emits STS/LDS rather than generic ST/LD)
  unsigned char *smem = smem_raw + ((1024 - (smem_u32(smem_raw) & 1023)) & 1023);
  unsigned char *a_hi = smem;
  unsigned char *a_lo = a_hi + L::A_PLANE;
  unsigned char *b_hi = a_lo + L::A_PLANE;
  unsigned char *b_lo = b_hi + L::B_PLANE;
  const int K = 1 << g.kb, N = 1 << g.nb;
  const int xt = g.xt_bits, ot = g.ot_bits;
  float2 *os = reinterpret_cast<float2 *>(b_lo + L::B_PLANE);
  const int x_hi_n = 1 << (xt - g.x_run), o_hi_n = 1 << (ot - g.o_run);
  int64_t *xhi = reinterpret_cast<int64_t *>(os + (1 << ot));
  int64_t *ohi = xhi + x_hi_n;
  uint32_t *tk_hi = reinterpret_cast<uint32_t *>(ohi + o_hi_n);  // (t | k << 16) of high tile bits
  uint32_t *tk_lo = tk_hi + x_hi_n;                              // ... of the low run bits
  int *on = reinterpret_cast<int *>(tk_lo + (1 << g.x_run));
  int *oo_t = on + N;                                            // O-tile offset of row t
  uint64_t *mbar = reinterpret_cast<uint64_t *>(
      (reinterpret_cast<uintptr_t>(oo_t + kRows) + 7) & ~uintptr_t(7));
  uint32_t *tmem_slot = reinterpret_cast<uint32_t *>(mbar + 1);

  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  // ---- one-time setup: tables, zeroed A planes (K padding), W'' hi/lo ----
  for (int i = tid; i < x_hi_n; i += kThreads) {
    int64_t off = 0;
    for (int l = g.x_run; l < xt; ++l)
      if ((i >> (l - g.x_run)) & 1) off += int64_t(1) << g.x_tile_pos[l];
    xhi[i] = off;
  }
  for (int i = tid; i < o_hi_n; i += kThreads) {
    int64_t off = 0;
    for (int l = g.o_run; l < ot; ++l)
      if ((i >> (l - g.o_run)) & 1) off += int64_t(1) << g.o_tile_pos[l];
    ohi[i] = off;
  }
  // tile-local X bit -> (t bit | k bit) contribution
  {
    // inverse maps of t_xl / k_xl
    for (int i = tid; i < x_hi_n + (1 << g.x_run); i += kThreads) {
      const bool hi = i < x_hi_n;
      const int v = hi ? i : i - x_hi_n;
      const int lo_bit = hi ? g.x_run : 0;
      const int nbits = hi ? xt - g.x_run : g.x_run;
      uint32_t t = 0, k = 0;
      for (int l = 0; l < nbits; ++l) {
        if (!((v >> l) & 1)) continue;
        const int tl = lo_bit + l;  // tile-local X bit
        for (int j = 0; j < g.tb; ++j)
          if (g.t_xl[j] == tl) t |= 1u << j;
        for (int j = 0; j < g.kb; ++j)
          if (g.k_xl[j] == tl) k |= 1u << j;
      }
      if (hi)
        tk_hi[v] = t | (k << 16);
      else
        tk_lo[v] = t | (k << 16);
    }
  }
  for (int n = tid; n < N; n += kThreads) {
    int off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off |= 1 << g.n_ol[j];
    on[n] = off;
  }
  for (int t = tid; t < kRows; t += kThreads) {
    int off = 0;
    for (int j = 0; j < g.tb; ++j)
      if ((t >> j) & 1) off |= 1 << g.t_ol[j];
    oo_t[t] = off;
  }
  for (int i = tid; i < 2 * L::A_PLANE / 16; i += kThreads)
    reinterpret_cast<float4 *>(a_hi)[i] = make_float4(0.f, 0.f, 0.f, 0.f);
  for (int i = tid; i < L::BN * L::AK; i += kThreads) {
    const int nr = i / L::AK, c = i % L::AK;
    const int n = nr >> 1, tt = nr & 1, k = c >> 1, s = c & 1;
    float v = 0.f;
    if (n < N && k < K) {
      int64_t off = 0;
      for (int j = 0; j < g.kb; ++j)
        if ((k >> j) & 1) off += g.w_k_stride[j];
      for (int j = 0; j < g.nb; ++j)
        if ((n >> j) & 1) off += g.w_n_stride[j];
      const float2 w = W[off];
      // B''[2n+t][2k+s] = [[wr, -wi], [wi, wr]][t][s]
      v = tt == 0 ? (s == 0 ? w.x : -w.y) : (s == 0 ? w.y : w.x);
    }
    const float vh = tf32_round(v);
    const uint32_t o = sw128_off(nr, c, L::BN);
    *reinterpret_cast<float *>(b_hi + o) = vh;
    *reinterpret_cast<float *>(b_lo + o) = v - vh;
  }
  if (warp == 0) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     smem_u32(tmem_slot)),
                 "r"(L::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (tid == 0) {
    mbar_init(mbar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
  __syncthreads();
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
  const uint32_t tmem = *tmem_slot;

  const int x_run_mask = (1 << g.x_run) - 1, o_run_mask = (1 << g.o_run) - 1;
  const int x_pairs = 1 << (xt - 1), o_pairs = 1 << (ot - 1);
  uint32_t phase = 0;
  // X pairs are prefetched into registers one tile ahead, so the HBM latency
  // of tile i+1 overlaps the MMA, epilogue and store of tile i.
  constexpr int LD = KP == 16 ? 8 : 16;  // max float4 per thread (x_pairs / 128)
  float4 pre[LD];
  auto tile_base = [&](int64_t tile, int64_t &bx, int64_t &bo) {
    bx = 0;
    bo = 0;
    for (int j = 0; j < g.ob; ++j)
      if ((tile >> j) & 1) {
        bx += int64_t(1) << g.outer_x[j];
        bo += int64_t(1) << g.outer_o[j];
      }
  };
  auto prefetch = [&](int64_t tile) {
    if (tile >= n_tiles) return;
    int64_t bx, bo;
    tile_base(tile, bx, bo);
#pragma unroll
    for (int u = 0; u < LD; ++u) {
      const int q = tid + u * kThreads;
      if (q < x_pairs) {
        const int i = q << 1;
        pre[u] = __ldcs(reinterpret_cast<const float4 *>(X + bx + xhi[i >> g.x_run] +
                                                         (i & x_run_mask)));
      }
    }
  };
  prefetch(blockIdx.x);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    int64_t bx, bo;
    tile_base(tile, bx, bo);
    // ---- prefetched X pairs -> TF32 hi/lo planes ----
#pragma unroll
    for (int u = 0; u < LD; ++u) {
      const int q = tid + u * kThreads;
      if (q >= x_pairs) break;
      const int i = q << 1;
      const float4 v = pre[u];
      const uint32_t base_tk = tk_hi[i >> g.x_run];
#pragma unroll
      for (int e = 0; e < 2; ++e) {
        const uint32_t tk = base_tk | tk_lo[(i + e) & x_run_mask];
        const int t = int(tk & 0xFFFFu), k = int(tk >> 16);
        const float re = e ? v.z : v.x, im = e ? v.w : v.y;
        const float rh = tf32_round(re), ih = tf32_round(im);
        const uint32_t o = sw128_off(t, 2 * k, kRows);
        *reinterpret_cast<float2 *>(a_hi + o) = make_float2(rh, ih);
        *reinterpret_cast<float2 *>(a_lo + o) = make_float2(re - rh, im - ih);
      }
    }
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    // ---- MMA ----
    if (tid == 0) {
      asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
      const uint32_t ah = smem_u32(a_hi), al = smem_u32(a_lo);
      const uint32_t bh = smem_u32(b_hi), bl = smem_u32(b_lo);
#pragma unroll
      for (int slab = 0; slab < L::AK / 32; ++slab) {
#pragma unroll
        for (int j = 0; j < 4; ++j) {
          const uint32_t ao = slab * kRows * 128 + j * 32, bo2 = slab * L::BN * 128 + j * 32;
          const uint32_t first = (slab == 0 && j == 0) ? 0u : 1u;
          umma_tf32(tmem, smem_desc_sw128(ah + ao), smem_desc_sw128(bh + bo2), L::IDESC, first);
          umma_tf32(tmem + L::BN, smem_desc_sw128(ah + ao), smem_desc_sw128(bl + bo2), L::IDESC,
                    first);
          umma_tf32(tmem + L::BN, smem_desc_sw128(al + ao), smem_desc_sw128(bh + bo2), L::IDESC,
                    1u);
        }
      }
      umma_commit(mbar);
    }
    prefetch(tile + gridDim.x);
    mbar_wait(mbar, phase);
    phase ^= 1;
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    // ---- epilogue: TMEM -> O tile (smem) ----
    {
      const int t = warp * 32 + lane;
      const int oo = oo_t[t];
#pragma unroll
      for (int c0 = 0; c0 < L::BN; c0 += 16) {
        uint32_t v[16], w[16];
        const uint32_t ta = tmem + (uint32_t(warp * 32) << 16) + uint32_t(c0);
        tmem_ld16(ta, v);
        tmem_ld16(ta + L::BN, w);
        asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
#pragma unroll
        for (int q = 0; q < 8; ++q) {
          const int n = (c0 >> 1) + q;
          if (n < N)
            os[oo | on[n]] = make_float2(__uint_as_float(v[2 * q]) + __uint_as_float(w[2 * q]),
                                         __uint_as_float(v[2 * q + 1]) +
                                             __uint_as_float(w[2 * q + 1]));
        }
      }
    }
    asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
    __syncthreads();
    // ---- store O tile ----
    for (int q = tid; q < o_pairs; q += kThreads) {
      const int i = q << 1;
      const float4 v = reinterpret_cast<const float4 *>(os)[q];
      __stcs(reinterpret_cast<float4 *>(O + bo + ohi[i >> g.o_run] + (i & o_run_mask)), v);
    }
    __syncthreads();
  }
  if (warp == 0) {
    asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(L::TMEM_COLS));
  }
}

template <int KP, int NP>
size_t tc_absorb_smem(const AbsorbGeom &g) {
  using L = TcAbsorbLayout<KP, NP>;
  const size_t x_hi_n = size_t(1) << (g.xt_bits - g.x_run);
  const size_t o_hi_n = size_t(1) << (g.ot_bits - g.o_run);
  return 1024 + 2 * size_t(L::A_PLANE) + 2 * size_t(L::B_PLANE) + 8 * (size_t(1) << g.ot_bits) +
         8 * (x_hi_n + o_hi_n) + 4 * (x_hi_n + (size_t(1) << g.x_run)) +
         4 * ((size_t(1) << g.nb) + kRows) + 64 + 8;
}

template <int KP, int NP>
cudaError_t launch_tc_absorb_impl(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  const size_t smem = tc_absorb_smem<KP, NP>(g);
  if (smem > 220 * 1024) return cudaErrorNotSupported;
  auto kern = k_absorb_tc<KP, NP>;
  static bool set_on[kMaxDevices] = {};
  bool &set = set_on[current_device()];
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    set = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  if (per_sm > 512 / TcAbsorbLayout<KP, NP>::TMEM_COLS)  // TMEM: 512 columns per SM
    per_sm = 512 / TcAbsorbLayout<KP, NP>::TMEM_COLS;
  const int64_t n_tiles = int64_t(1) << g.ob;
  int64_t ctas = int64_t(148) * per_sm / (p.nbatch > 0 ? p.nbatch : 1);
  if (ctas < 1) ctas = 1;
  if (ctas > n_tiles) ctas = n_tiles;
  dim3 grid(unsigned(ctas), unsigned(p.nbatch));
  kern<<<grid, kThreads, smem, stream>>>(g, p, n_tiles);
  return cudaGetLastError();
}

}  // namespace

bool tc_absorb_supported(const AbsorbGeom &g) {
  return g.tb == 7 && g.kb <= 5 && g.nb <= 6 && g.x_run >= 1 && g.o_run >= 1;
}

cudaError_t launch_absorb_tc(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  if (!tc_absorb_supported(g)) return cudaErrorNotSupported;
  const int kp = g.kb <= 4 ? 16 : 32;
  const int np = g.nb <= 3 ? 8 : (1 << g.nb);
#define STN_TCA(KPV, NPV) \
  if (kp == KPV && np == NPV) return launch_tc_absorb_impl<KPV, NPV>(g, p, stream);
  STN_TCA(16, 8) STN_TCA(16, 16) STN_TCA(16, 32) STN_TCA(16, 64)
  STN_TCA(32, 8) STN_TCA(32, 16) STN_TCA(32, 32) STN_TCA(32, 64)
#undef STN_TCA
  return cudaErrorNotSupported;
}

}  // namespace stn
