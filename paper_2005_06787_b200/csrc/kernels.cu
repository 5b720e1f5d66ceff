// SIMT kernels of the B200 stem executor (sm_100a).
//
// Arithmetic modes:
//   exact  - every complex product is (ar*br - ai*bi, ar*bi + ai*br) with
//            separately rounded IEEE operations (__fmul_rn/__fadd_rn never
//            contract into FMA) and every output sums its K terms in ascending
//            k order starting from zero. That is the reference loop
//            (runtime.hpp:396-407) operation for operation, so results are
//            bitwise identical to the reference CPU executor.
//   fast   - the same order with fused multiply-adds.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "kernels.h"

namespace stn {

namespace {

template <class R>
struct Cx;
template <>
struct Cx<float> {
  using T = float2;
};
template <>
struct Cx<double> {
  using T = double2;
};
template <class R>
using cx_t = typename Cx<R>::T;

__device__ __forceinline__ float mul_rn(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ double mul_rn(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ float add_rn(float a, float b) { return __fadd_rn(a, b); }
__device__ __forceinline__ double add_rn(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float sub_rn(float a, float b) { return __fsub_rn(a, b); }
__device__ __forceinline__ double sub_rn(double a, double b) { return __dsub_rn(a, b); }

// acc += a * b
template <bool EXACT, class T>
__device__ __forceinline__ void cmac(T &acc, const T a, const T b) {
  if constexpr (EXACT) {
    auto re = sub_rn(mul_rn(a.x, b.x), mul_rn(a.y, b.y));
    auto im = add_rn(mul_rn(a.x, b.y), mul_rn(a.y, b.x));
    acc.x = add_rn(acc.x, re);
    acc.y = add_rn(acc.y, im);
  } else {
    acc.x = fma(a.x, b.x, acc.x);
    acc.x = fma(-a.y, b.y, acc.x);
    acc.y = fma(a.x, b.y, acc.y);
    acc.y = fma(a.y, b.x, acc.y);
  }
}

inline int grid_for(int64_t n, int threads, int max_blocks = 148 * 16) {
  int64_t b = (n + threads - 1) / threads;
  if (b > max_blocks) b = max_blocks;
  if (b < 1) b = 1;
  return int(b);
}

// ---------------------------------------------------------------------------
// Generic strided contraction. One thread per output element (grid-stride);
// the K sum runs over an odometer in ascending k. POW2: every (merged) dim is a
// power of two and indices decompose with shifts (all circuit networks).
// ---------------------------------------------------------------------------
template <class R, bool EXACT, bool POW2>
__global__ void __launch_bounds__(256)
    k_generic(const __grid_constant__ StridedGeom g, const BatchPtrs p) {
  using T = cx_t<R>;
  const int b = blockIdx.y;
  const T *A = static_cast<const T *>(p.a) + int64_t(b) * p.a_bs;
  const T *B = static_cast<const T *>(p.b) + int64_t(b) * p.b_bs;
  T *O = static_cast<T *>(p.out) + int64_t(b) * p.out_bs;
  const int last = g.n_k - 1;
  const int64_t kd_last = last >= 0 ? g.k_dim[last] : 1;
  const int64_t ka_last = last >= 0 ? g.k_sa[last] : 0;
  const int64_t kb_last = last >= 0 ? g.k_sb[last] : 0;
  const int64_t k_outer = g.k_size / kd_last;
  for (int64_t o = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < g.out_size;
       o += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = o, ao = 0, bo = 0;
    for (int i = g.n_out - 1; i >= 0; --i) {
      int64_t idx;
      if constexpr (POW2) {
        const int sh = __ffsll(g.out_dim[i]) - 1;
        idx = rem & (g.out_dim[i] - 1);
        rem >>= sh;
      } else {
        idx = rem % g.out_dim[i];
        rem /= g.out_dim[i];
      }
      ao += idx * g.out_sa[i];
      bo += idx * g.out_sb[i];
    }
    T acc;
    acc.x = 0;
    acc.y = 0;
    for (int64_t ko = 0; ko < k_outer; ++ko) {
      int64_t r2 = ko, ka = ao, kb = bo;
      for (int i = last - 1; i >= 0; --i) {
        int64_t idx;
        if constexpr (POW2) {
          const int sh = __ffsll(g.k_dim[i]) - 1;
          idx = r2 & (g.k_dim[i] - 1);
          r2 >>= sh;
        } else {
          idx = r2 % g.k_dim[i];
          r2 /= g.k_dim[i];
        }
        ka += idx * g.k_sa[i];
        kb += idx * g.k_sb[i];
      }
      for (int64_t kk = 0; kk < kd_last; ++kk) {
        cmac<EXACT>(acc, A[ka], B[kb]);
        ka += ka_last;
        kb += kb_last;
      }
    }
    O[o] = acc;
  }
}

// out[o] = in[a_off(o)] : axis permutation (the reference's permute,
// runtime.hpp:113-140, as a gather over the output index).
template <class R, bool POW2>
__global__ void __launch_bounds__(256)
    k_permute(const __grid_constant__ StridedGeom g, const void *in_, void *out_, int64_t in_bs,
              int64_t out_bs) {
  using T = cx_t<R>;
  const int b = blockIdx.y;
  const T *in = static_cast<const T *>(in_) + int64_t(b) * in_bs;
  T *out = static_cast<T *>(out_) + int64_t(b) * out_bs;
  for (int64_t o = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; o < g.out_size;
       o += int64_t(gridDim.x) * blockDim.x) {
    int64_t rem = o, ao = 0;
    for (int i = g.n_out - 1; i >= 0; --i) {
      int64_t idx;
      if constexpr (POW2) {
        const int sh = __ffsll(g.out_dim[i]) - 1;
        idx = rem & (g.out_dim[i] - 1);
        rem >>= sh;
      } else {
        idx = rem % g.out_dim[i];
        rem /= g.out_dim[i];
      }
      ao += idx * g.out_sa[i];
    }
    out[o] = in[ao];
  }
}

// ---------------------------------------------------------------------------
// Bond-2 absorb: stream the big operand X once through shared memory.
//   load : X tile (tile M bits x all K bits) -> xs, 16-byte coalesced runs
//   math : O[t, n] = sum_k xs[t, k] * W[k, n], k ascending, W from smem
//   store: O tile (tile M bits x all N bits) -> global, 16-byte coalesced runs
// One CTA per assignment of the outer M bits (and per slice in the batch).
// ---------------------------------------------------------------------------
constexpr int kAbsorbThreads = 256;

template <bool EXACT, int NC, bool PERMUTE>
__global__ void __launch_bounds__(kAbsorbThreads)
    k_absorb(const __grid_constant__ AbsorbGeom g, const BatchPtrs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  const int xt = g.xt_bits, ot = g.ot_bits;
  const int K = 1 << g.kb, N = 1 << g.nb;
  const int x_hi_n = 1 << (xt - g.x_run), o_hi_n = 1 << (ot - g.o_run);
  float2 *xs = reinterpret_cast<float2 *>(smem_raw);
  float2 *os = xs + (1 << xt);
  float2 *ws = os + (1 << ot);                              // [k][n]
  int64_t *xhi = reinterpret_cast<int64_t *>(ws + K * N);   // X offset of high tile bits
  int64_t *ohi = xhi + x_hi_n;                              // O offset of high tile bits
  int *xk = reinterpret_cast<int *>(ohi + o_hi_n);          // tile-local X offset of k
  int *on = xk + K;                                         // tile-local O offset of n

  // base offsets of this CTA's outer M bits
  const uint64_t outer = blockIdx.x;
  int64_t base_x = 0, base_o = 0;
  for (int j = 0; j < g.ob; ++j)
    if ((outer >> j) & 1) {
      base_x += int64_t(1) << g.outer_x[j];
      base_o += int64_t(1) << g.outer_o[j];
    }

  const int tid = threadIdx.x;
  for (int i = tid; i < x_hi_n; i += kAbsorbThreads) {
    int64_t off = 0;
    for (int l = g.x_run; l < xt; ++l)
      if ((i >> (l - g.x_run)) & 1) off += int64_t(1) << g.x_tile_pos[l];
    xhi[i] = off;
  }
  for (int i = tid; i < o_hi_n; i += kAbsorbThreads) {
    int64_t off = 0;
    for (int l = g.o_run; l < ot; ++l)
      if ((i >> (l - g.o_run)) & 1) off += int64_t(1) << g.o_tile_pos[l];
    ohi[i] = off;
  }
  for (int k = tid; k < K; k += kAbsorbThreads) {
    int off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off |= 1 << g.k_xl[j];
    xk[k] = off;
  }
  for (int n = tid; n < N; n += kAbsorbThreads) {
    int off = 0;
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off |= 1 << g.n_ol[j];
    on[n] = off;
  }
  for (int i = tid; i < (PERMUTE ? 0 : K * N); i += kAbsorbThreads) {
    const int k = i / N, n = i % N;
    int64_t off = 0;
    for (int j = 0; j < g.kb; ++j)
      if ((k >> j) & 1) off += g.w_k_stride[j];
    for (int j = 0; j < g.nb; ++j)
      if ((n >> j) & 1) off += g.w_n_stride[j];
    ws[i] = W[off];
  }
  __syncthreads();

  // load the X tile: pairs of consecutive elements (x_run >= 1)
  {
    const int run_mask = (1 << g.x_run) - 1;
    const int pairs = 1 << (xt - 1);
    for (int q = tid; q < pairs; q += kAbsorbThreads) {
      const int i = q << 1;
      const int64_t src = base_x + xhi[i >> g.x_run] + (i & run_mask);
      const float4 v = __ldg(reinterpret_cast<const float4 *>(X + src));
      reinterpret_cast<float4 *>(xs)[q] = v;
    }
  }
  __syncthreads();

  // math: each thread owns tile rows t; NC outputs per pass over K
  const int T = 1 << g.tb;
  for (int t = tid; t < T; t += kAbsorbThreads) {
    int xo = 0, oo = 0;
    for (int j = 0; j < g.tb; ++j)
      if ((t >> j) & 1) {
        xo |= 1 << g.t_xl[j];
        oo |= 1 << g.t_ol[j];
      }
    if constexpr (PERMUTE) {
      os[oo] = xs[xo];
      continue;
    }
    for (int n0 = 0; n0 < N; n0 += NC) {
      float2 acc[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[c] = make_float2(0.f, 0.f);
      for (int k = 0; k < K; ++k) {
        const float2 x = xs[xo | xk[k]];
        const float2 *wr = ws + k * N + n0;
#pragma unroll
        for (int c = 0; c < NC; ++c)
          if (n0 + c < N) cmac<EXACT>(acc[c], x, wr[c]);
      }
#pragma unroll
      for (int c = 0; c < NC; ++c)
        if (n0 + c < N) os[oo | on[n0 + c]] = acc[c];
    }
  }
  __syncthreads();

  // store the O tile
  {
    const int run_mask = (1 << g.o_run) - 1;
    const int pairs = 1 << (ot - 1);
    for (int q = tid; q < pairs; q += kAbsorbThreads) {
      const int i = q << 1;
      const int64_t dst = base_o + ohi[i >> g.o_run] + (i & run_mask);
      reinterpret_cast<float4 *>(O + dst)[0] = reinterpret_cast<const float4 *>(os)[q];
    }
  }
}

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
    if ((iter & 1023) == 1023 && clock64() - start > (4ll << 30)) __trap();
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
  static bool set = false;
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
  static int set_bytes = 0;
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
  static const bool no_bulk = std::getenv("STN_NO_BULK") != nullptr;  // experiments only
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

// ---------------------------------------------------------------------------
// Direct absorb (kernels.h DirectGeom): every thread owns a pair of consecutive
// m (one 16-byte vector per k and per n) and walks R consecutive m_hi values
// with pdep increments; W lives in shared memory. Loads and stores of a warp
// cover 512 contiguous bytes per k / per n; no tiles, no barriers in the loop.
// ---------------------------------------------------------------------------
constexpr int kDirThreads = 256;
constexpr int kDirR = 8;  // m_hi values per thread

__device__ __forceinline__ uint64_t pdep_mask(uint64_t v, uint64_t mask) {
  uint64_t r = 0;
  for (uint64_t bit = 1; mask; bit <<= 1) {
    const uint64_t low = mask & (0 - mask);
    if (v & bit) r |= low;
    mask ^= low;
  }
  return r;
}

// KC / NC: K and N chunks held in registers; K and N are runtime multiples.
template <bool EXACT, int KC, int NC>
__global__ void __launch_bounds__(kDirThreads)
    k_absorb_direct(const __grid_constant__ DirectGeom g, const BatchPtrs p) {
  extern __shared__ __align__(16) float2 wsm[];  // [N][K]
  const int K = 1 << g.kb, N = 1 << g.nb;
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
    wsm[i] = Wg[off];
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
    for (int n0 = 0; n0 < N; n0 += NC) {
      float2 a0[NC], a1[NC];
#pragma unroll
      for (int c = 0; c < NC; ++c) a0[c] = a1[c] = make_float2(0.f, 0.f);
      for (int k0 = 0; k0 < K; k0 += KC) {
        float4 xv[KC];
#pragma unroll
        for (int k = 0; k < KC; ++k) xv[k] = __ldcs(xs + g.x_koff[k0 + k] / 2);
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
        __stcs(reinterpret_cast<float4 *>(O + po + lo + g.o_noff[n0 + c]),
               make_float4(a0[c].x, a0[c].y, a1[c].x, a1[c].y));
    }
    // next subset of the high-bit masks (pdep(v + 1) from pdep(v))
    px = ((px | ~g.hi_x_mask) + 1) & g.hi_x_mask;
    po = ((po | ~g.hi_o_mask) + 1) & g.hi_o_mask;
  }
}

bool direct_ok_impl(const DirectGeom &g) { return g.L >= 2 && g.kb <= 6 && g.nb <= 6; }

template <bool EXACT>
cudaError_t launch_direct_exact(const DirectGeom &g, const BatchPtrs &p, cudaStream_t st) {
  const int64_t threads = (int64_t(1) << (g.L - 1)) *
                          (((int64_t(1) << g.mh_bits) + kDirR - 1) / kDirR);
  dim3 grid(unsigned((threads + kDirThreads - 1) / kDirThreads), unsigned(p.nbatch));
  const size_t smem = size_t(8) << (g.kb + g.nb);
  const int kc = g.kb >= 4 ? 16 : (1 << g.kb), nc = g.nb >= 4 ? 16 : (1 << g.nb);
#define STN_DIR(KV, NV)                                                          \
  if (kc == KV && nc == NV) {                                                    \
    if (smem > 48 * 1024)                                                        \
      cudaFuncSetAttribute(k_absorb_direct<EXACT, KV, NV>,                      \
                           cudaFuncAttributeMaxDynamicSharedMemorySize, int(smem)); \
    k_absorb_direct<EXACT, KV, NV><<<grid, kDirThreads, smem, st>>>(g, p);      \
    return cudaGetLastError();                                                   \
  }
#define STN_DIR_ROW(KV) STN_DIR(KV, 1) STN_DIR(KV, 2) STN_DIR(KV, 4) STN_DIR(KV, 8) STN_DIR(KV, 16)
  STN_DIR_ROW(1) STN_DIR_ROW(2) STN_DIR_ROW(4) STN_DIR_ROW(8) STN_DIR_ROW(16)
#undef STN_DIR_ROW
#undef STN_DIR
  return cudaErrorNotSupported;
}

cudaError_t launch_direct_impl(const DirectGeom &g, const BatchPtrs &p, bool exact,
                               cudaStream_t stream) {
  if (!direct_ok_impl(g)) return cudaErrorNotSupported;
  return exact ? launch_direct_exact<true>(g, p, stream) : launch_direct_exact<false>(g, p, stream);
}

// ---------------------------------------------------------------------------
// Tiled SIMT complex GEMM, C[d] = A[d] (MxK, row-major) * B[d] (KxN, row-major).
// 64x64 output tile per CTA, 16-wide K steps, 4x4 outputs per thread; every
// output accumulates k in ascending order.
// ---------------------------------------------------------------------------
template <class R, bool EXACT>
__global__ void __launch_bounds__(256)
    k_gemm_simt(const GemmShape s, const BatchPtrs p) {
  using T = cx_t<R>;
  constexpr int BM = 64, BN = 64, BK = 16;
  __shared__ T As[BK][BM + 1];
  __shared__ T Bs[BK][BN + 1];
  const int64_t batch = blockIdx.z;  // = slice * D + d
  const int64_t slice = batch / s.D, d = batch % s.D;
  const T *A = static_cast<const T *>(p.a) + slice * p.a_bs + d * s.M * s.K;
  const T *B = static_cast<const T *>(p.b) + slice * p.b_bs + d * s.K * s.N;
  T *C = static_cast<T *>(p.out) + slice * p.out_bs + d * s.M * s.N;
  const int64_t m_tiles = (s.M + BM - 1) / BM;
  const int64_t m0 = (int64_t(blockIdx.x) % m_tiles) * BM, n0 = (int64_t(blockIdx.x) / m_tiles) * BN;
  const int tx = threadIdx.x % 16, ty = threadIdx.x / 16;
  T acc[4][4];
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[i][j].x = acc[i][j].y = 0;
  for (int64_t k0 = 0; k0 < s.K; k0 += BK) {
    for (int e = threadIdx.x; e < BM * BK; e += 256) {
      const int mm = e / BK, kk = e % BK;
      const int64_t gm = m0 + mm, gk = k0 + kk;
      T v;
      v.x = v.y = 0;
      if (gm < s.M && gk < s.K) v = A[gm * s.K + gk];
      As[kk][mm] = v;
    }
    for (int e = threadIdx.x; e < BK * BN; e += 256) {
      const int kk = e / BN, nn = e % BN;
      const int64_t gk = k0 + kk, gn = n0 + nn;
      T v;
      v.x = v.y = 0;
      if (gk < s.K && gn < s.N) v = B[gk * s.N + gn];
      Bs[kk][nn] = v;
    }
    __syncthreads();
    const int kmax = int(s.K - k0 < BK ? s.K - k0 : BK);
    for (int kk = 0; kk < kmax; ++kk) {
      T a[4], bb[4];
#pragma unroll
      for (int i = 0; i < 4; ++i) a[i] = As[kk][ty * 4 + i];
#pragma unroll
      for (int j = 0; j < 4; ++j) bb[j] = Bs[kk][tx + 16 * j];
#pragma unroll
      for (int i = 0; i < 4; ++i)
#pragma unroll
        for (int j = 0; j < 4; ++j) cmac<EXACT>(acc[i][j], a[i], bb[j]);
    }
    __syncthreads();
  }
#pragma unroll
  for (int i = 0; i < 4; ++i)
#pragma unroll
    for (int j = 0; j < 4; ++j) {
      const int64_t gm = m0 + ty * 4 + i, gn = n0 + tx + 16 * j;
      if (gm < s.M && gn < s.N) C[gm * s.N + gn] = acc[i][j];
    }
}

// ---------------------------------------------------------------------------
// Per-slice leaf preparation (runtime.hpp:367-384): digit restriction, cast,
// canonical layout, for every sliced leaf and every slice of the batch.
// ---------------------------------------------------------------------------
template <class R>
__global__ void k_leaf_gather(const LeafGatherTable t, void *arena_, const int32_t *digits,
                              int nbatch) {
  using T = cx_t<R>;
  T *arena = static_cast<T *>(arena_);
  const int64_t total = t.total_out * nbatch;
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < total;
       i += int64_t(gridDim.x) * blockDim.x) {
    const int b = int(i / t.total_out);
    const int64_t e = i % t.total_out;
    const int leaf = t.elem_leaf[e];
    int64_t src = t.src_base[e];
    for (int a = t.ax_begin[leaf]; a < t.ax_begin[leaf + 1]; ++a)
      src += t.ax_stride[a] * digits[int64_t(b) * t.n_sliced + t.ax_slice[a]];
    T v;
    v.x = R(t.values[2 * src]);
    v.y = R(t.values[2 * src + 1]);
    arena[t.dst_off[leaf] * nbatch + int64_t(b) * t.dst_bs[leaf] + t.elem_local[e]] = v;
  }
}

// Root of each slice -> double; optional per-slice copy; ascending-order
// accumulation over the batch (runtime.hpp:601-605).
template <class R>
__global__ void k_root_accumulate(const void *root_, int64_t root_bs, int64_t n, int nbatch,
                                  double *acc, double *per_slice) {
  using T = cx_t<R>;
  const T *root = static_cast<const T *>(root_);
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double sr = acc ? acc[2 * i] : 0.0, si = acc ? acc[2 * i + 1] : 0.0;
    for (int b = 0; b < nbatch; ++b) {
      const T v = root[int64_t(b) * root_bs + i];
      const double vr = double(v.x), vi = double(v.y);
      if (per_slice) {
        per_slice[2 * (int64_t(b) * n + i)] = vr;
        per_slice[2 * (int64_t(b) * n + i) + 1] = vi;
      }
      sr = __dadd_rn(sr, vr);
      si = __dadd_rn(si, vi);
    }
    if (acc) {
      acc[2 * i] = sr;
      acc[2 * i + 1] = si;
    }
  }
}

__global__ void k_sum_ordered(const double *per_slice, uint64_t n_slices, int64_t n, double *out) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < 2 * n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double s = 0.0;
    for (uint64_t a = 0; a < n_slices; ++a) s = __dadd_rn(s, per_slice[a * 2 * n + i]);
    out[i] = s;
  }
}

bool all_pow2(const StridedGeom &g) {
  for (int i = 0; i < g.n_out; ++i)
    if (g.out_dim[i] & (g.out_dim[i] - 1)) return false;
  for (int i = 0; i < g.n_k; ++i)
    if (g.k_dim[i] & (g.k_dim[i] - 1)) return false;
  return true;
}

}  // namespace

bool direct_absorb_launchable(const DirectGeom &g) { return direct_ok_impl(g); }

cudaError_t launch_absorb_direct(const DirectGeom &g, const BatchPtrs &p, bool exact,
                                 cudaStream_t stream) {
  return launch_direct_impl(g, p, exact, stream);
}

template <class R>
cudaError_t launch_generic(const StridedGeom &g, const BatchPtrs &p, bool exact,
                           cudaStream_t stream) {
  if (g.out_size == 0 || p.nbatch == 0) return cudaSuccess;
  dim3 grid(grid_for(g.out_size, 256), p.nbatch);
  const bool pow2 = all_pow2(g);
  if (exact) {
    if (pow2)
      k_generic<R, true, true><<<grid, 256, 0, stream>>>(g, p);
    else
      k_generic<R, true, false><<<grid, 256, 0, stream>>>(g, p);
  } else {
    if (pow2)
      k_generic<R, false, true><<<grid, 256, 0, stream>>>(g, p);
    else
      k_generic<R, false, false><<<grid, 256, 0, stream>>>(g, p);
  }
  return cudaGetLastError();
}

template <class R>
cudaError_t launch_permute(const StridedGeom &g, const void *in, void *out, int64_t in_bs,
                           int64_t out_bs, int nbatch, cudaStream_t stream) {
  if (g.out_size == 0 || nbatch == 0) return cudaSuccess;
  dim3 grid(grid_for(g.out_size, 256), nbatch);
  if (all_pow2(g))
    k_permute<R, true><<<grid, 256, 0, stream>>>(g, in, out, in_bs, out_bs);
  else
    k_permute<R, false><<<grid, 256, 0, stream>>>(g, in, out, in_bs, out_bs);
  return cudaGetLastError();
}

size_t absorb_smem_bytes(const AbsorbGeom &g) {
  const size_t K = size_t(1) << g.kb, N = size_t(1) << g.nb;
  return 8 * ((size_t(1) << g.xt_bits) + (size_t(1) << g.ot_bits) + K * N) +
         8 * ((size_t(1) << (g.xt_bits - g.x_run)) + (size_t(1) << (g.ot_bits - g.o_run))) +
         4 * (K + N);
}

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

// ---------------------------------------------------------------------------
// Split-K reduction for steps with a small output and a long K (e.g. the
// 16 x 16 x 2^20 inner products of two big stem tensors). FAST mode only: the
// K range is cut into fixed chunks (deterministic order, not the reference's
// single running sum). Pass 1: per (chunk, batch) partial outputs; pass 2:
// ascending-chunk sum.
// ---------------------------------------------------------------------------
template <class R>
__global__ void __launch_bounds__(256)
    k_splitk_partial(const __grid_constant__ StridedGeom g, const BatchPtrs p, DotTables t,
                     int kc, int nchunks, void *partial_) {
  using T = cx_t<R>;
  extern __shared__ __align__(16) unsigned char smem_raw[];
  T *sA = reinterpret_cast<T *>(smem_raw);  // [M][kc + 1]
  T *sB = sA + t.M * (kc + 1);              // [N][kc + 1]
  const int b = blockIdx.y, chunk = blockIdx.x;
  const T *A = static_cast<const T *>(p.a) + int64_t(b) * p.a_bs;
  const T *B = static_cast<const T *>(p.b) + int64_t(b) * p.b_bs;
  T *partial = static_cast<T *>(partial_) + (int64_t(b) * nchunks + chunk) * g.out_size;
  const int64_t k0 = int64_t(chunk) * kc;
  const int len = int(min(int64_t(kc), g.k_size - k0));
  // pow2 axes: operand offsets are linear in the bits of k, so
  // off(k0 + kk) = off(k0) + off(kk) for kk < kc (kc a power of two, k0 aligned)
  int64_t *ka_tab = reinterpret_cast<int64_t *>(sB + t.N * (kc + 1));
  int64_t *kb_tab = ka_tab + kc;
  auto koff = [&](int64_t k, int64_t &ka, int64_t &kb) {
    ka = 0;
    kb = 0;
    for (int i = g.n_k - 1; i >= 0; --i) {
      const int sh = __ffsll(g.k_dim[i]) - 1;
      const int64_t idx = k & (g.k_dim[i] - 1);
      k >>= sh;
      ka += idx * g.k_sa[i];
      kb += idx * g.k_sb[i];
    }
  };
  for (int kk = threadIdx.x; kk < kc; kk += blockDim.x) koff(kk, ka_tab[kk], kb_tab[kk]);
  int64_t ka0, kb0;
  koff(k0, ka0, kb0);
  __syncthreads();
  // stage A[:, chunk] and B[:, chunk]: consecutive threads take consecutive k
  for (int idx = threadIdx.x; idx < (t.M + t.N) * kc; idx += blockDim.x) {
    const int row = idx / kc, kk = idx % kc;
    T v;
    v.x = v.y = 0;
    if (kk < len)
      v = row < t.M ? A[t.a_row[row] + ka0 + ka_tab[kk]] : B[t.b_col[row - t.M] + kb0 + kb_tab[kk]];
    sA[row * (kc + 1) + kk] = v;  // sB follows sA contiguously
  }
  __syncthreads();
  for (int o = threadIdx.x; o < g.out_size; o += blockDim.x) {
    const int mn = t.o_mn[o];
    const T *ra = sA + (mn & 0xFFFF) * (kc + 1);
    const T *rb = sB + (mn >> 16) * (kc + 1);
    T acc;
    acc.x = acc.y = 0;
    for (int kk = 0; kk < len; ++kk) cmac<false>(acc, ra[kk], rb[kk]);
    partial[o] = acc;
  }
}

// One CTA per (batch, output): 256 threads sum strided chunk subsets, then a
// fixed-shape tree in shared memory -- deterministic for a given chunk count.
template <class R>
__global__ void __launch_bounds__(256)
    k_splitk_sum(const void *partial_, int nchunks, int64_t out_size, int nbatch, void *out_,
                 int64_t out_bs) {
  using T = cx_t<R>;
  __shared__ T red[256];
  const T *partial = static_cast<const T *>(partial_);
  T *out = static_cast<T *>(out_);
  const int64_t b = blockIdx.x / out_size, o = blockIdx.x % out_size;
  T s;
  s.x = s.y = 0;
  for (int c = threadIdx.x; c < nchunks; c += 256) {
    const T v = partial[(b * nchunks + c) * out_size + o];
    s.x += v.x;
    s.y += v.y;
  }
  red[threadIdx.x] = s;
  __syncthreads();
  for (int w = 128; w > 0; w >>= 1) {
    if (threadIdx.x < w) {
      red[threadIdx.x].x += red[threadIdx.x + w].x;
      red[threadIdx.x].y += red[threadIdx.x + w].y;
    }
    __syncthreads();
  }
  if (threadIdx.x == 0) out[b * out_bs + o] = red[0];
}

// k per chunk: A and B rows of the chunk fit in 48 KiB of shared memory
int splitk_kc(const DotTables &t, size_t esize) {
  int kc = 256;
  while (kc > 8 && size_t(t.M + t.N) * (kc + 1) * esize > 48 * 1024) kc /= 2;
  return kc;
}

int splitk_chunks(const StridedGeom &g, const DotTables &t, size_t esize) {
  const int64_t kc = splitk_kc(t, esize);
  return int((g.k_size + kc - 1) / kc);
}

template <class R>
cudaError_t launch_splitk(const StridedGeom &g, const BatchPtrs &p, const DotTables &t,
                          void *workspace, cudaStream_t stream) {
  const int kc = splitk_kc(t, sizeof(cx_t<R>));
  const int nchunks = splitk_chunks(g, t, sizeof(cx_t<R>));
  const size_t smem = size_t(t.M + t.N) * (kc + 1) * sizeof(cx_t<R>) + 16 * size_t(kc);
  k_splitk_partial<R><<<dim3(nchunks, p.nbatch), 256, smem, stream>>>(g, p, t, kc, nchunks,
                                                                      workspace);
  k_splitk_sum<R><<<unsigned(g.out_size * p.nbatch), 256, 0, stream>>>(
      workspace, nchunks, g.out_size, p.nbatch, p.out, p.out_bs);
  return cudaGetLastError();
}

size_t splitk_workspace_bytes(const StridedGeom &g, const DotTables &t, int nbatch,
                              size_t esize) {
  return size_t(splitk_chunks(g, t, esize)) * g.out_size * nbatch * esize;
}

template <class R>
cudaError_t launch_gemm_simt(const GemmShape &s, const BatchPtrs &p, bool exact,
                             cudaStream_t stream) {
  if (s.M == 0 || s.N == 0 || p.nbatch == 0) return cudaSuccess;
  const int64_t tiles = ((s.M + 63) / 64) * ((s.N + 63) / 64);
  dim3 grid(unsigned(tiles), 1, unsigned(s.D * p.nbatch));
  if (exact)
    k_gemm_simt<R, true><<<grid, 256, 0, stream>>>(s, p);
  else
    k_gemm_simt<R, false><<<grid, 256, 0, stream>>>(s, p);
  return cudaGetLastError();
}

template <class R>
cudaError_t launch_leaf_gather(const LeafGatherTable &t, void *arena, const int32_t *digits,
                               int nbatch, cudaStream_t stream) {
  if (t.total_out == 0 || nbatch == 0) return cudaSuccess;
  k_leaf_gather<R><<<grid_for(t.total_out * nbatch, 256), 256, 0, stream>>>(t, arena, digits,
                                                                            nbatch);
  return cudaGetLastError();
}

template <class R>
cudaError_t launch_root_accumulate(const void *root, int64_t root_bs, int64_t n, int nbatch,
                                   double *acc, double *per_slice, cudaStream_t stream) {
  k_root_accumulate<R><<<grid_for(n, 256), 256, 0, stream>>>(root, root_bs, n, nbatch, acc,
                                                            per_slice);
  return cudaGetLastError();
}

cudaError_t launch_sum_ordered(const double *per_slice, uint64_t n_slices, int64_t n, double *out,
                               cudaStream_t stream) {
  k_sum_ordered<<<grid_for(2 * n, 256), 256, 0, stream>>>(per_slice, n_slices, n, out);
  return cudaGetLastError();
}

template cudaError_t launch_generic<float>(const StridedGeom &, const BatchPtrs &, bool,
                                           cudaStream_t);
template cudaError_t launch_generic<double>(const StridedGeom &, const BatchPtrs &, bool,
                                            cudaStream_t);
template cudaError_t launch_permute<float>(const StridedGeom &, const void *, void *, int64_t,
                                           int64_t, int, cudaStream_t);
template cudaError_t launch_permute<double>(const StridedGeom &, const void *, void *, int64_t,
                                            int64_t, int, cudaStream_t);
template cudaError_t launch_gemm_simt<float>(const GemmShape &, const BatchPtrs &, bool,
                                             cudaStream_t);
template cudaError_t launch_gemm_simt<double>(const GemmShape &, const BatchPtrs &, bool,
                                              cudaStream_t);
template cudaError_t launch_splitk<float>(const StridedGeom &, const BatchPtrs &,
                                          const DotTables &, void *, cudaStream_t);
template cudaError_t launch_splitk<double>(const StridedGeom &, const BatchPtrs &,
                                           const DotTables &, void *, cudaStream_t);
template cudaError_t launch_leaf_gather<float>(const LeafGatherTable &, void *, const int32_t *,
                                               int, cudaStream_t);
template cudaError_t launch_leaf_gather<double>(const LeafGatherTable &, void *, const int32_t *,
                                                int, cudaStream_t);
template cudaError_t launch_root_accumulate<float>(const void *, int64_t, int64_t, int, double *,
                                                   double *, cudaStream_t);
template cudaError_t launch_root_accumulate<double>(const void *, int64_t, int64_t, int,
                                                    double *, double *, cudaStream_t);

}  // namespace stn
