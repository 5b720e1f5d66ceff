// Tiled bond-2 absorb kernels (shared-memory tiles): v2 (cp.async ring) and v3
// (bulk async copies + mbarrier ring + bulk stores), plus the tiled bit
// permutation. See kernels.h AbsorbGeom for the tile geometry.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace stn {

namespace {
using namespace dev;

// ---------------------------------------------------------------------------
// Absorb v2: persistent CTAs, cp.async double-buffered X tiles, one tile row
// per thread with its K inputs in registers and W^T broadcast from smem
// (8 FMA per shared load), O tile staged in smem for coalesced 16 B stores.
// Per output the K terms are summed in ascending k (exact mode = reference).
// ---------------------------------------------------------------------------
constexpr int kAb2Threads = 256;
constexpr int kAb2Stages = 3;  // X tiles in flight per CTA (cp.async ring)

__device__ __forceinline__ void cp_async16(void *smem, const void *gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// KC / NC: K and N chunk sizes held in registers (compile-time, <= 16).
// Tile math shared by the absorb kernels: O tile (os) from X tile (xs).
template <bool EXACT, bool PERMUTE, int KC, int NC, bool BLOCKED>
__device__ __forceinline__ void absorb_tile_math(const AbsorbGeom &g, const float2 *xs,
                                                 float2 *os, const float2 *wt, const int *xk,
                                                 const int *on, int tid, int nthreads) {
  const int K = 1 << g.kb, N = 1 << g.nb;
  const int T = 1 << g.tb;
  const int tpr = T >= nthreads ? 1 : nthreads / T;  // threads per tile row
    // ---- math ----
    if constexpr (BLOCKED) {
      constexpr int RB = KC, CB = NC;
      const int row_groups = T / RB, items = row_groups * (N / CB);
      for (int item = tid; item < items; item += nthreads) {
        const int r0 = (item % row_groups) * RB, c0 = (item / row_groups) * CB;
        int xo[RB], oo[RB];
#pragma unroll
        for (int i = 0; i < RB; ++i) {
          xo[i] = 0;
          oo[i] = 0;
          for (int j = 0; j < g.tb; ++j)
            if (((r0 + i) >> j) & 1) {
              xo[i] |= 1 << g.t_xl[j];
              oo[i] |= 1 << g.t_ol[j];
            }
        }
        float2 acc[RB][CB];
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < CB; ++j) acc[i][j] = make_float2(0.f, 0.f);
        for (int k = 0; k < K; ++k) {
          const int xkk = xk[k];
          float2 xv[RB], wv[CB];
#pragma unroll
          for (int i = 0; i < RB; ++i) xv[i] = xs[xo[i] | xkk];
#pragma unroll
          for (int j = 0; j < CB; ++j) wv[j] = wt[(c0 + j) * K + k];
#pragma unroll
          for (int i = 0; i < RB; ++i)
#pragma unroll
            for (int j = 0; j < CB; ++j) cmac<EXACT>(acc[i][j], xv[i], wv[j]);
        }
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < CB; ++j) os[oo[i] | on[c0 + j]] = acc[i][j];
      }
    } else
    for (int r = tid / tpr; r < T; r += nthreads / tpr) {
      const int sub = tid % tpr;
      int xo = 0, oo = 0;
      for (int j = 0; j < g.tb; ++j)
        if ((r >> j) & 1) {
          xo |= 1 << g.t_xl[j];
          oo |= 1 << g.t_ol[j];
        }
      if constexpr (PERMUTE) {
        if (sub == 0) os[oo] = xs[xo];
      } else {
        for (int n0 = sub * NC; n0 < N; n0 += tpr * NC) {
          float2 acc[NC];
#pragma unroll
          for (int c = 0; c < NC; ++c) acc[c] = make_float2(0.f, 0.f);
          for (int k0 = 0; k0 < K; k0 += KC) {
            float2 x[KC];
#pragma unroll
            for (int kk = 0; kk < KC; ++kk)
              if (KC <= 1 || k0 + kk < K) x[kk] = xs[xo | xk[k0 + kk]];
#pragma unroll
            for (int c = 0; c < NC; ++c) {
              const float2 *w = wt + (n0 + c) * K + k0;
#pragma unroll
              for (int kk = 0; kk < KC; ++kk)
                if (k0 + kk < K) cmac<EXACT>(acc[c], x[kk], w[kk]);
            }
          }
#pragma unroll
          for (int c = 0; c < NC; ++c) os[oo | on[n0 + c]] = acc[c];
        }
      }
    }
}

// BLOCKED (large K x N): each thread owns a KC x NC = RB x CB block of (rows,
// columns) and runs the k loop as an outer product (8 FMA per shared load).
template <bool EXACT, bool PERMUTE, int KC, int NC, bool BLOCKED = false>
__global__ void __launch_bounds__(kAb2Threads, 2)
    k_absorb2(const __grid_constant__ AbsorbGeom g, const BatchPtrs p, int64_t n_tiles) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int xt = g.xt_bits, ot = g.ot_bits;
  const int K = 1 << g.kb, N = 1 << g.nb;
  const int x_hi_n = 1 << (xt - g.x_run), o_hi_n = 1 << (ot - g.o_run);
  float2 *xs_ring = reinterpret_cast<float2 *>(smem_raw);
  float2 *os = xs_ring + kAb2Stages * (1 << xt);
  float2 *wt = os + (1 << ot);  // W^T: [n][k]
  int64_t *xhi = reinterpret_cast<int64_t *>(wt + (PERMUTE ? 0 : K * N));
  int64_t *ohi = xhi + x_hi_n;
  int *xk = reinterpret_cast<int *>(ohi + o_hi_n);
  int *on = xk + K;
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  for (int i = tid; i < x_hi_n; i += kAb2Threads) {
    int64_t off = 0;
    for (int l = g.x_run; l < xt; ++l)
      if ((i >> (l - g.x_run)) & 1) off += int64_t(1) << g.x_tile_pos[l];
    xhi[i] = off;
  }
  for (int i = tid; i < o_hi_n; i += kAb2Threads) {
    int64_t off = 0;
    for (int l = g.o_run; l < ot; ++l)
      if ((i >> (l - g.o_run)) & 1) off += int64_t(1) << g.o_tile_pos[l];
    ohi[i] = off;
  }
  for (int k = tid; k < K; k += kAb2Threads) {
    int off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off |= 1 << g.k_xl[j];
    xk[k] = off;
  }
  for (int n = tid; n < N; n += kAb2Threads) {
    int off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off |= 1 << g.n_ol[j];
    on[n] = off;
  }
  if constexpr (!PERMUTE) {
    const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
    for (int i = tid; i < K * N; i += kAb2Threads) {
      const int n = i / K, k = i % K;
      int64_t off = 0;
      for (int j = 0; j < g.kb; ++j)
        if ((k >> j) & 1) off += g.w_k_stride[j];
      for (int j = 0; j < g.nb; ++j)
        if ((n >> j) & 1) off += g.w_n_stride[j];
      wt[i] = W[off];
    }
  }
  __syncthreads();

  auto tile_bases = [&](int64_t tile, int64_t &bx, int64_t &bo) {
    bx = 0;
    bo = 0;
    for (int j = 0; j < g.ob; ++j)
      if ((tile >> j) & 1) {
        bx += int64_t(1) << g.outer_x[j];
        bo += int64_t(1) << g.outer_o[j];
      }
  };
  const int x_run_mask = (1 << g.x_run) - 1, o_run_mask = (1 << g.o_run) - 1;
  const int x_pairs = 1 << (xt - 1), o_pairs = 1 << (ot - 1);
  auto issue_load = [&](int64_t tile, float2 *dst) {
    if (tile < n_tiles) {
      int64_t bx, bo;
      tile_bases(tile, bx, bo);
      for (int q = tid; q < x_pairs; q += kAb2Threads) {
        const int i = q << 1;
        cp_async16(dst + i, X + bx + xhi[i >> g.x_run] + (i & x_run_mask));
      }
    }
    cp_async_commit();  // (possibly empty) group keeps the ring arithmetic uniform
  };

  const int64_t first = blockIdx.x, stride = gridDim.x;
#pragma unroll 1
  for (int s = 0; s < kAb2Stages - 1; ++s)
    issue_load(first + s * stride, xs_ring + s * (1 << xt));
  int it = 0;
  for (int64_t tile = first; tile < n_tiles; tile += stride, ++it) {
    issue_load(tile + (kAb2Stages - 1) * stride,
               xs_ring + ((it + kAb2Stages - 1) % kAb2Stages) * (1 << xt));
    cp_async_wait<kAb2Stages - 1>();
    __syncthreads();
    const float2 *xs = xs_ring + (it % kAb2Stages) * (1 << xt);
    absorb_tile_math<EXACT, PERMUTE, KC, NC, BLOCKED>(g, xs, os, wt, xk, on, tid, kAb2Threads);
    __syncthreads();
    // ---- store ----
    {
      int64_t bx, bo;
      tile_bases(tile, bx, bo);
      for (int q = tid; q < o_pairs; q += kAb2Threads) {
        const int i = q << 1;
        const float4 v = reinterpret_cast<const float4 *>(os)[q];
        float4 *dst = reinterpret_cast<float4 *>(O + bo + ohi[i >> g.o_run] + (i & o_run_mask));
        __stcs(dst, v);
      }
    }
    // os is rewritten only after the next iteration's __syncthreads
  }
  cp_async_wait<0>();
}

// ---------------------------------------------------------------------------
// Absorb v3: the X and O tiles move as bulk async copies (cp.async.bulk, the
// TMA engine's 1-D path): one copy per contiguous run of 2^x_run elements,
// completion on an mbarrier (4-stage ring) and bulk stores from a double-
// buffered O tile. The SMs only do the tile math.
// ---------------------------------------------------------------------------
constexpr int kAb3Threads = 256;
constexpr int kAb3Stages = 4;

__device__ __forceinline__ uint32_t smem_addr(const void *p) {
  return static_cast<uint32_t>(__cvta_generic_to_shared(p));
}
__device__ __forceinline__ void ab3_mbar_init(uint64_t *bar) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(smem_addr(bar)));
}
__device__ __forceinline__ void ab3_expect(uint64_t *bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_addr(bar)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void ab3_wait(uint64_t *bar, uint32_t parity) {
  uint32_t done = 0;
  long long start = 0;
  for (int iter = 0;; ++iter) {
    asm volatile(
        "{\n\t.reg .pred p;\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t}"
        : "=r"(done)
        : "r"(smem_addr(bar)), "r"(parity)
        : "memory");
    if (done) return;
    if (iter == 0) start = clock64();
    if ((iter & 1023) == 1023 && clock64() - start > (120ll << 30)) __trap();
  }
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, uint32_t bytes, uint64_t *bar) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
          smem_addr(dst)),
      "l"(src), "r"(bytes), "r"(smem_addr(bar))
      : "memory");
}
__device__ __forceinline__ void bulk_s2g(void *dst, const void *src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst),
               "r"(smem_addr(src)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void bulk_commit() { asm volatile("cp.async.bulk.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void bulk_wait_read() {
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait() {
  asm volatile("cp.async.bulk.wait_group %0;" ::"n"(N) : "memory");
}

template <bool EXACT, bool PERMUTE, int KC, int NC, bool BLOCKED>
__global__ void __launch_bounds__(kAb3Threads, 1)
    k_absorb3(const __grid_constant__ AbsorbGeom g, const BatchPtrs p, int64_t n_tiles) {
  extern __shared__ __align__(128) unsigned char smem_raw[];
  const int xt = g.xt_bits, ot = g.ot_bits;
  const int K = 1 << g.kb, N = 1 << g.nb;
  const int x_hi_n = 1 << (xt - g.x_run), o_hi_n = 1 << (ot - g.o_run);
  float2 *xs_ring = reinterpret_cast<float2 *>(smem_raw);
  float2 *os_buf = xs_ring + kAb3Stages * (1 << xt);
  float2 *wt = os_buf + 2 * (1 << ot);
  int64_t *xhi = reinterpret_cast<int64_t *>(wt + (PERMUTE ? 0 : K * N));
  int64_t *ohi = xhi + x_hi_n;
  uint64_t *full = reinterpret_cast<uint64_t *>(ohi + o_hi_n);
  int *xk = reinterpret_cast<int *>(full + kAb3Stages);
  int *on = xk + K;
  const int tid = threadIdx.x, warp = tid / 32, lane = tid % 32;
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  for (int i = tid; i < x_hi_n; i += kAb3Threads) {
    int64_t off = 0;
    for (int l = g.x_run; l < xt; ++l)
      if ((i >> (l - g.x_run)) & 1) off += int64_t(1) << g.x_tile_pos[l];
    xhi[i] = off;
  }
  for (int i = tid; i < o_hi_n; i += kAb3Threads) {
    int64_t off = 0;
    for (int l = g.o_run; l < ot; ++l)
      if ((i >> (l - g.o_run)) & 1) off += int64_t(1) << g.o_tile_pos[l];
    ohi[i] = off;
  }
  for (int k = tid; k < K; k += kAb3Threads) {
    int off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off |= 1 << g.k_xl[j];
    xk[k] = off;
  }
  for (int n = tid; n < N; n += kAb3Threads) {
    int off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off |= 1 << g.n_ol[j];
    on[n] = off;
  }
  if constexpr (!PERMUTE) {
    const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
    for (int i = tid; i < K * N; i += kAb3Threads) {
      const int n = i / K, k = i % K;
      int64_t off = 0;
      for (int j = 0; j < g.kb; ++j)
        if ((k >> j) & 1) off += g.w_k_stride[j];
      for (int j = 0; j < g.nb; ++j)
        if ((n >> j) & 1) off += g.w_n_stride[j];
      wt[i] = W[off];
    }
  }
  if (tid == 0) {
    for (int s = 0; s < kAb3Stages; ++s) ab3_mbar_init(&full[s]);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  __syncthreads();

  auto tile_bases = [&](int64_t tile, int64_t &bx, int64_t &bo) {
    bx = 0;
    bo = 0;
    for (int j = 0; j < g.ob; ++j)
      if ((tile >> j) & 1) {
        bx += int64_t(1) << g.outer_x[j];
        bo += int64_t(1) << g.outer_o[j];
      }
  };
  const uint32_t x_run_bytes = 8u << g.x_run, o_run_bytes = 8u << g.o_run;
  // warp 0 issues the bulk loads of one tile into ring stage s
  auto issue_load = [&](int64_t tile, int s) {
    if (tile >= n_tiles) return;
    if (lane == 0) ab3_expect(&full[s], 8u << xt);
    __syncwarp();
    int64_t bx, bo;
    tile_bases(tile, bx, bo);
    float2 *dst = xs_ring + s * (1 << xt);
    for (int r = lane; r < x_hi_n; r += 32)
      bulk_g2s(dst + (r << g.x_run), X + bx + xhi[r], x_run_bytes, &full[s]);
  };
  const int64_t first = blockIdx.x, stride = gridDim.x;
  if (warp == 0)
    for (int s = 0; s < kAb3Stages - 1; ++s) issue_load(first + s * stride, s);
  int it = 0;
  for (int64_t tile = first; tile < n_tiles; tile += stride, ++it) {
    if (warp == 0) bulk_wait_read<1>();  // O buffer it&1 was read out two tiles ago
    __syncthreads();                      // ... and stage (it-1)%S is consumed
    if (warp == 0) issue_load(tile + (kAb3Stages - 1) * stride, (it + kAb3Stages - 1) % kAb3Stages);
    ab3_wait(&full[it % kAb3Stages], (it / kAb3Stages) & 1);
    const float2 *xs = xs_ring + (it % kAb3Stages) * (1 << xt);
    float2 *os = os_buf + (it & 1) * (1 << ot);
    absorb_tile_math<EXACT, PERMUTE, KC, NC, BLOCKED>(g, xs, os, wt, xk, on, tid, kAb3Threads);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    __syncthreads();
    if (warp == 0) {
      int64_t bx, bo;
      tile_bases(tile, bx, bo);
      for (int r = lane; r < o_hi_n; r += 32)
        bulk_s2g(O + bo + ohi[r], os + (r << g.o_run), o_run_bytes);
      bulk_commit();
    }
  }
  if (warp == 0) bulk_wait<0>();
}

size_t absorb3_smem_bytes(const AbsorbGeom &g, bool permute) {
  const size_t K = size_t(1) << g.kb, N = size_t(1) << g.nb;
  return 8 * (kAb3Stages * (size_t(1) << g.xt_bits) + 2 * (size_t(1) << g.ot_bits) +
              (permute ? 0 : K * N)) +
         8 * ((size_t(1) << (g.xt_bits - g.x_run)) + (size_t(1) << (g.ot_bits - g.o_run))) +
         8 * kAb3Stages + 4 * (K + N);
}

template <bool EXACT, bool PERMUTE, int KC, int NC, bool BLOCKED>
cudaError_t launch_absorb3_impl(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  const size_t smem = absorb3_smem_bytes(g, PERMUTE);
  if (smem > 220 * 1024) return cudaErrorNotSupported;
  auto kern = k_absorb3<EXACT, PERMUTE, KC, NC, BLOCKED>;
  static bool set_on[kMaxDevices] = {};
  bool &set = set_on[current_device()];
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         220 * 1024);
    if (e != cudaSuccess) return e;
    set = true;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kAb3Threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t n_tiles = int64_t(1) << g.ob;
  int64_t ctas = int64_t(148) * per_sm / (p.nbatch > 0 ? p.nbatch : 1);
  if (ctas < 1) ctas = 1;
  if (ctas > n_tiles) ctas = n_tiles;
  dim3 grid(unsigned(ctas), unsigned(p.nbatch));
  kern<<<grid, kAb3Threads, smem, stream>>>(g, p, n_tiles);
  return cudaGetLastError();
}

bool absorb3_ok(const AbsorbGeom &g) {
  return g.x_run >= 3 && g.o_run >= 3 && (g.xt_bits - g.x_run) <= 8 &&
         (g.ot_bits - g.o_run) <= 8;
}

size_t absorb2_smem_bytes(const AbsorbGeom &g, bool permute) {
  const size_t K = size_t(1) << g.kb, N = size_t(1) << g.nb;
  return 8 * (kAb2Stages * (size_t(1) << g.xt_bits) + (size_t(1) << g.ot_bits) +
              (permute ? 0 : K * N)) +
         8 * ((size_t(1) << (g.xt_bits - g.x_run)) + (size_t(1) << (g.ot_bits - g.o_run))) +
         4 * (K + N);
}

template <bool EXACT, bool PERMUTE, int KC, int NC, bool BLOCKED = false>
cudaError_t launch_absorb2_impl(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream) {
  const size_t smem = absorb2_smem_bytes(g, PERMUTE);
  auto kern = k_absorb2<EXACT, PERMUTE, KC, NC, BLOCKED>;
  static int set_bytes_on[kMaxDevices] = {};
  int &set_bytes = set_bytes_on[current_device()];
  if (int(smem) > set_bytes) {
    const int want = smem > 48 * 1024 ? 200 * 1024 : 48 * 1024;
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, want);
    if (e != cudaSuccess) return e;
    set_bytes = want;
  }
  int per_sm = 0;
  cudaError_t e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kAb2Threads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t n_tiles = int64_t(1) << g.ob;
  int64_t ctas = int64_t(148) * per_sm / (p.nbatch > 0 ? p.nbatch : 1);
  if (ctas < 1) ctas = 1;
  if (ctas > n_tiles) ctas = n_tiles;
  dim3 grid(unsigned(ctas), unsigned(p.nbatch));
  kern<<<grid, kAb2Threads, smem, stream>>>(g, p, n_tiles);
  return cudaGetLastError();
}

template <bool EXACT, int KC, int NC, bool BLOCKED>
cudaError_t launch_absorb_best(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t st) {
  static const bool no_bulk = stn::debug_opt("no_bulk") != nullptr;  // experiments only
  if (!no_bulk && absorb3_ok(g)) {
    cudaError_t e = launch_absorb3_impl<EXACT, false, KC, NC, BLOCKED>(g, p, st);
    if (e != cudaErrorNotSupported) return e;
  }
  return launch_absorb2_impl<EXACT, false, KC, NC, BLOCKED>(g, p, st);
}

template <bool EXACT>
cudaError_t launch_absorb2_dispatch(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t st) {
  // large K x N: register-blocked outer products (4 rows x CB columns)
  if (g.kb + g.nb >= 8 && g.tb >= 2) {
    if (g.nb >= 2) return launch_absorb_best<EXACT, 4, 4, true>(g, p, st);
    if (g.nb == 1) return launch_absorb_best<EXACT, 4, 2, true>(g, p, st);
    return launch_absorb_best<EXACT, 4, 1, true>(g, p, st);
  }
  const int kc = g.kb >= 4 ? 16 : (1 << g.kb), nc = g.nb >= 4 ? 16 : (1 << g.nb);
#define STN_AB2(KCV, NCV) \
  if (kc == KCV && nc == NCV) return launch_absorb_best<EXACT, KCV, NCV, false>(g, p, st);
#define STN_AB2_ROW(KCV) \
  STN_AB2(KCV, 1) STN_AB2(KCV, 2) STN_AB2(KCV, 4) STN_AB2(KCV, 8) STN_AB2(KCV, 16)
  STN_AB2_ROW(1) STN_AB2_ROW(2) STN_AB2_ROW(4) STN_AB2_ROW(8) STN_AB2_ROW(16)
#undef STN_AB2_ROW
#undef STN_AB2
  return cudaErrorNotSupported;
}

}  // namespace

cudaError_t launch_absorb(const AbsorbGeom &g, const BatchPtrs &p, bool exact,
                          cudaStream_t stream) {
  return exact ? launch_absorb2_dispatch<true>(g, p, stream)
               : launch_absorb2_dispatch<false>(g, p, stream);
}

cudaError_t launch_bitperm(const AbsorbGeom &g, const void *in, void *out, int64_t in_bs,
                           int64_t out_bs, int nbatch, cudaStream_t stream) {
  BatchPtrs p{in, nullptr, out, in_bs, 0, out_bs, nbatch};
  if (absorb3_ok(g)) {
    cudaError_t e = launch_absorb3_impl<false, true, 1, 1, false>(g, p, stream);
    if (e != cudaErrorNotSupported) return e;
  }
  return launch_absorb2_impl<false, true, 1, 1>(g, p, stream);
}


}  // namespace stn
