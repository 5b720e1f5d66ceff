// Tile-free bond-2 absorb (kernels.h DirectGeom): 16-byte streaming of
// consecutive m pairs, pdep-increment addressing, W in shared memory.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace stn {

namespace {
using namespace dev;

// ---------------------------------------------------------------------------
// Direct absorb (kernels.h DirectGeom): every thread owns a pair of consecutive
// m (one 16-byte vector per k and per n) and walks R consecutive m_hi values
// with pdep increments; W lives in shared memory. Loads and stores of a warp
// cover 512 contiguous bytes per k / per n; no tiles, no barriers in the loop.
// ---------------------------------------------------------------------------
constexpr int kDirThreads = 256;
constexpr int kDirR = 8;   // m_hi values per thread
constexpr int kDirPf = 2;  // L2 prefetch distance (m_hi values) in FAST mode

__device__ __forceinline__ uint64_t pdep_mask(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t bit = 1; mask; bit <<= 1) {
    const uint64_t low = mask & (0 - mask);
    if (v & bit) r |= low;
    mask ^= low;
  }
  return r;
}

// Blackwell packed FP32 FMA (FFMA2) on 64-bit register pairs: acc += x * w, lane-wise.
__device__ __forceinline__ void ffma2(unsigned long long &acc, const unsigned long long x,
                                      const unsigned long long w) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(acc) : "l"(x), "l"(w));
}
__device__ __forceinline__ float2 unpack2(const unsigned long long v) {
  float2 r;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(r.x), "=f"(r.y) : "l"(v));
  return r;
}

// KC / NC: K and N chunks held in registers (compile time, <= 16). FULLK:
// K == KC, so the K inputs of an m pair are loaded once and reused for every
// N chunk; otherwise every (N chunk, K chunk) reloads (an L1/L2 hit).
template <bool EXACT, int KC, int NC, bool FULLK>
__global__ void __launch_bounds__(kDirThreads)
    k_absorb_direct(const __grid_constant__ DirectGeom g, const BatchPtrs p) {
  extern __shared__ __align__(16) unsigned char dsm[];
  const int K = FULLK ? KC : (1 << g.kb), N = 1 << g.nb;
  // EXACT: W as [N][K] float2. FAST (FFMA2 form): [N][K] float4 (wr, wr, wi, -wi), so
  // that with x = (xr, xi) as loaded, U += x * (wr, wr) and V += x * (wi, -wi) give
  // re = U.x + V.y and im = U.y + V.x without repacking any operand.
  float2 *wsm = reinterpret_cast<float2 *>(dsm);
  float4 *wq = reinterpret_cast<float4 *>(dsm);
  int64_t *xko = reinterpret_cast<int64_t *>(EXACT ? (void *)(wsm + K * N) : (void *)(wq + K * N));
  int64_t *ono = xko + K;                                         // [N] O offset of n
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  const float2 *Wg = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;
  for (int i = threadIdx.x; i < K * N; i += kDirThreads) {
    const int n = i / K, k = i % K;
    int64_t off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off += g.w_k_stride[j];
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off += g.w_n_stride[j];
    const float2 w = Wg[off];
    if constexpr (EXACT) {
      wsm[i] = w;
    } else {
      wq[i] = make_float4(w.x, w.x, w.y, -w.y);
    }
  }
  for (int k = threadIdx.x; k < K; k += kDirThreads) {
    int64_t off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off += int64_t(1) << g.k_xpos[j];
    xko[k] = off / 2;
  }
  for (int n = threadIdx.x; n < N; n += kDirThreads) {
    int64_t off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off += int64_t(1) << g.n_opos[j];
    ono[n] = off;
  }
  __syncthreads();
  const int pairs_lo = 1 << (g.L - 1);  // m pairs per m_hi
  const int64_t t = int64_t(blockIdx.x) * kDirThreads + threadIdx.x;
  const int lo = int(t % pairs_lo) * 2;
  const int64_t hi0 = (t / pairs_lo) * kDirR;
  const int64_t n_hi = int64_t(1) << g.mh_bits;
  if (hi0 >= n_hi) return;
  uint64_t px = pdep_mask(uint64_t(hi0), g.hi_x_mask);
  uint64_t po = pdep_mask(uint64_t(hi0), g.hi_o_mask);
  for (int r = 0; r < kDirR && hi0 + r < n_hi; ++r) {
    const float4 *xs = reinterpret_cast<const float4 *>(X + px + lo);
    float2 *os = O + po + lo;
    float4 xv[KC];
    if constexpr (FULLK && EXACT) {
#pragma unroll
      for (int k = 0; k < KC; ++k) xv[k] = __ldcs(xs + xko[k]);
    }
    if constexpr (!EXACT) {
      const ulonglong2 *xq = reinterpret_cast<const ulonglong2 *>(xs);
      const ulonglong2 *wq2 = reinterpret_cast<const ulonglong2 *>(wq);
      ulonglong2 xp[KC];  // (x m0, x m1) as 64-bit (re, im) pairs
      if constexpr (FULLK) {
#pragma unroll
        for (int k = 0; k < KC; ++k) xp[k] = __ldcs(xq + xko[k]);
        // pull the X inputs kDirPf m_hi ahead into L2 while this one computes
        uint64_t pxn = px;
        for (int d = 1; d <= kDirPf; ++d) {
          pxn = ((pxn | ~g.hi_x_mask) + 1) & g.hi_x_mask;
          if ((r == 0 || d == kDirPf) && r + d < kDirR && hi0 + r + d < n_hi) {
            const float2 *xn = X + pxn + lo;
#pragma unroll
            for (int k = 0; k < KC; ++k)
              asm volatile("prefetch.global.L2 [%0];" ::"l"(xn + 2 * xko[k]));
          }
        }
      }
      for (int n0 = 0; n0 < N; n0 += NC) {
        unsigned long long u0[NC], v0[NC], u1[NC], v1[NC];
#pragma unroll
        for (int c = 0; c < NC; ++c) u0[c] = v0[c] = u1[c] = v1[c] = 0ull;
        for (int k0 = 0; k0 < K; k0 += KC) {
          if constexpr (!FULLK) {
#pragma unroll
            for (int k = 0; k < KC; ++k) xp[k] = xq[xko[k0 + k]];
          }
#pragma unroll
          for (int c = 0; c < NC; ++c) {
            const ulonglong2 *qr = wq2 + (n0 + c) * K + k0;
#pragma unroll
            for (int k = 0; k < KC; ++k) {
              const ulonglong2 q = qr[k];  // ((wr, wr), (wi, -wi))
              ffma2(u0[c], xp[k].x, q.x);
              ffma2(v0[c], xp[k].x, q.y);
              ffma2(u1[c], xp[k].y, q.x);
              ffma2(v1[c], xp[k].y, q.y);
            }
          }
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const float2 U0 = unpack2(u0[c]), V0 = unpack2(v0[c]);
          const float2 U1 = unpack2(u1[c]), V1 = unpack2(v1[c]);
          __stcs(reinterpret_cast<float4 *>(os + ono[n0 + c]),
                 make_float4(U0.x + V0.y, U0.y + V0.x, U1.x + V1.y, U1.y + V1.x));
        }
      }
    } else
    for (int n0 = 0; n0 < N; n0 += NC) {
      float2 a0[NC], a1[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) a0[c] = a1[c] = make_float2(0.f, 0.f);
      for (int k0 = 0; k0 < K; k0 += KC) {
        if constexpr (!FULLK) {
#pragma unroll
          for (int k = 0; k < KC; ++k) xv[k] = xs[xko[k0 + k]];
        }
#pragma unroll
        for (int c = 0; c < NC; ++c) {
          const float2 *wr = wsm + (n0 + c) * K + k0;
#pragma unroll
          for (int k = 0; k < KC; ++k) {
            const float2 wk = wr[k];
            cmac<EXACT>(a0[c], make_float2(xv[k].x, xv[k].y), wk);
            cmac<EXACT>(a1[c], make_float2(xv[k].z, xv[k].w), wk);
          }
        }
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
        __stcs(reinterpret_cast<float4 *>(os + ono[n0 + c]),
               make_float4(a0[c].x, a0[c].y, a1[c].x, a1[c].y));
    }
    // next subset of the high-bit masks (pdep(v + 1) from pdep(v))
    px = ((px | ~g.hi_x_mask) + 1) & g.hi_x_mask;
    po = ((po | ~g.hi_o_mask) + 1) & g.hi_o_mask;
  }
}

bool direct_ok_impl(const DirectGeom &g) {
  return g.L >= 2 && g.kb <= 6 && g.nb <= 12 && g.kb + g.nb <= 12;
}

template <bool EXACT>
cudaError_t launch_direct_exact(const DirectGeom &g, const BatchPtrs &p, cudaStream_t st) {
  const int64_t threads = (int64_t(1) << (g.L - 1)) *
                          (((int64_t(1) << g.mh_bits) + kDirR - 1) / kDirR);
  dim3 grid(unsigned((threads + kDirThreads - 1) / kDirThreads), unsigned(p.nbatch));
  const size_t smem = (size_t(EXACT ? 8 : 24) << (g.kb + g.nb)) +
                      8 * ((size_t(1) << g.kb) + (size_t(1) << g.nb));
  // FAST keeps two accumulator pairs per (m, n): at most 8 n per register tile
  const int kc = g.kb >= 4 ? 16 : (1 << g.kb), nc = g.nb >= (EXACT ? 4 : 3) ? (EXACT ? 16 : 8) : (1 << g.nb);
  const bool full = g.kb <= 4;
#define STN_DIR(KV, NV, FULL)                                                          \
  if (kc == KV && nc == NV && full == FULL) {                                          \
    if (smem > 48 * 1024)                                                              \
      cudaFuncSetAttribute(k_absorb_direct<EXACT, KV, NV, FULL>,                      \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem));   \
    k_absorb_direct<EXACT, KV, NV, FULL><<<grid, kDirThreads, smem, st>>>(g, p);      \
    return cudaGetLastError();                                                         \
  }
#define STN_DIR_ROW(KV, FULL) \
  STN_DIR(KV, 1, FULL) STN_DIR(KV, 2, FULL) STN_DIR(KV, 4, FULL) STN_DIR(KV, 8, FULL) STN_DIR(KV, 16, FULL)
  STN_DIR_ROW(1, true) STN_DIR_ROW(2, true) STN_DIR_ROW(4, true) STN_DIR_ROW(8, true)
  STN_DIR_ROW(16, true) STN_DIR_ROW(16, false)
#undef STN_DIR_ROW
#undef STN_DIR
  return cudaErrorNotSupported;
}

cudaError_t launch_direct_impl(const DirectGeom &g, const BatchPtrs &p, bool exact,
                               cudaStream_t stream) {
  if (!direct_ok_impl(g)) return cudaErrorNotSupported;
  return exact ? launch_direct_exact<true>(g, p, stream) : launch_direct_exact<false>(g, p, stream);
}

}  // namespace

bool direct_absorb_launchable(const DirectGeom &g) { return direct_ok_impl(g); }

cudaError_t launch_absorb_direct(const DirectGeom &g, const BatchPtrs &p, bool exact,
                                 cudaStream_t stream) {
  return launch_direct_impl(g, p, exact, stream);
}


}  // namespace stn
