// Lane-mapped bond-2 absorb (kernels.h LaneGeom): the reference's
// transpose -> GEMM -> transpose of a stem step (runtime.hpp:386-418) computed
// straight from the stem's own layout, for any interleaving of the low output
// bits (M bits from the stem X, N bits from the small operand W).
//
// A warp owns one "row" of the output: 32 lanes x 1 or 2 consecutive complex
// outputs, i.e. the lowest 5 (+1) output bits, so every store of the warp is one
// contiguous 256/512-byte run. Each lane gathers its X inputs through per-lane
// and per-k offset tables (the permutation of the step lives only in these
// tables), W sits in shared memory, and the higher output bits ("row bits")
// map to X / W offsets through per-byte tables. The k terms are summed in
// ascending k with separately rounded products and sums in EXACT mode (bitwise
// the reference's crow[n] += amk * brow[n] order) and with FMAs in FAST mode.
// Persistent grid: CTAs stride over rows, so the 12 KiB of tables are staged
// once per CTA.
#include <algorithm>
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace stn {

namespace {
using namespace dev;

constexpr int kLaneThreads = 256;

__device__ __forceinline__ int64_t row_x(const int64_t (*xr)[256], uint32_t r) {
  return xr[0][r & 255] + xr[1][(r >> 8) & 255] + xr[2][(r >> 16) & 255] + xr[3][r >> 24];
}
__device__ __forceinline__ int32_t row_w(const int32_t (*wr)[256], uint32_t r) {
  return wr[0][r & 255] + wr[1][(r >> 8) & 255] + wr[2][(r >> 16) & 255] + wr[3][r >> 24];
}

// MODE 0: one output per lane; 1: an m pair (O bit 0 = X bit 0, 16-byte X loads);
// 2: an n pair (O bit 0 = an N bit: one X load feeds two outputs).
// RB rows per warp iteration (rows r, r + W, ... for W warps in the grid, so all
// warps together still sweep a contiguous range): RB x KC loads are in flight per
// lane before any math, KC = 8 / RB k terms per chunk. PF: prefetch the next row
// group's X inputs into L2 while this one computes.
template <int MODE, bool EXACT, int RB, bool PF>
__global__ void __launch_bounds__(kLaneThreads, RB == 1 ? 4 : 3)
    k_absorb_lanes(const LaneTables *__restrict__ T, const LaneGeom g, const BatchPtrs p) {
  constexpr int KC = 8 / RB;
  __shared__ int64_t sxr[4][256];
  __shared__ int32_t swr[4][256];
  __shared__ int64_t sxk[kLaneMaxK];
  __shared__ int32_t swk[kLaneMaxK];
  extern __shared__ float2 sw[];  // W of this batch: g.w_elems complex
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  const float2 *W = static_cast<const float2 *>(p.b) + int64_t(b) * p.b_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;
  for (int i = threadIdx.x; i < 1024; i += kLaneThreads) {
    sxr[i >> 8][i & 255] = T->xr[i >> 8][i & 255];
    swr[i >> 8][i & 255] = T->wr[i >> 8][i & 255];
  }
  for (int i = threadIdx.x; i < g.K; i += kLaneThreads) {
    sxk[i] = T->xk[i];
    swk[i] = T->wk[i];
  }
  for (int i = threadIdx.x; i < g.w_elems; i += kLaneThreads) sw[i] = W[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const int64_t xl = T->xl[lane];
  const int32_t wl = T->wl[lane];
  const int64_t warps = int64_t(gridDim.x) * (kLaneThreads / 32);
  const int K = g.K;
  constexpr int U = MODE == 0 ? 1 : 2;  // outputs per lane
  for (int64_t row0 = int64_t(blockIdx.x) * (kLaneThreads / 32) + (threadIdx.x >> 5);
       row0 < g.rows; row0 += warps * RB) {
    int64_t xb[RB];
    int32_t wb[RB];
    bool live[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int64_t row = row0 + i * warps;
      live[i] = row < g.rows;
      const uint32_t r = uint32_t(live[i] ? row : row0);
      xb[i] = row_x(sxr, r) + xl;
      wb[i] = row_w(swr, r) + wl;
    }
    if constexpr (PF) {
#pragma unroll
      for (int i = 0; i < RB; ++i) {
        const int64_t nrow = row0 + (RB + i) * warps;
        if (nrow < g.rows) {
          const int64_t nx = row_x(sxr, uint32_t(nrow)) + xl;
          for (int k = 0; k < K; ++k)
            asm volatile("prefetch.global.L2 [%0];" ::"l"(X + nx + sxk[k]));
        }
      }
    }
    float2 a0[RB], a1[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) a0[i] = a1[i] = make_float2(0.f, 0.f);
    for (int k0 = 0; k0 < K; k0 += KC) {
      if constexpr (MODE == 1) {
        float4 xv[RB][KC];
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < KC; ++j)
            if (k0 + j < K && live[i])
              xv[i][j] = __ldcs(reinterpret_cast<const float4 *>(X + xb[i] + sxk[k0 + j]));
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < KC; ++j)
            if (k0 + j < K && live[i]) {
              const float2 w = sw[wb[i] + swk[k0 + j]];
              cmac<EXACT>(a0[i], make_float2(xv[i][j].x, xv[i][j].y), w);
              cmac<EXACT>(a1[i], make_float2(xv[i][j].z, xv[i][j].w), w);
            }
      } else {
        float2 xv[RB][KC];
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < KC; ++j)
            if (k0 + j < K && live[i]) xv[i][j] = __ldcs(X + xb[i] + sxk[k0 + j]);
#pragma unroll
        for (int i = 0; i < RB; ++i)
#pragma unroll
          for (int j = 0; j < KC; ++j)
            if (k0 + j < K && live[i]) {
              const int32_t wi = wb[i] + swk[k0 + j];
              cmac<EXACT>(a0[i], xv[i][j], sw[wi]);
              if constexpr (MODE == 2) cmac<EXACT>(a1[i], xv[i][j], sw[wi + g.w_pair]);
            }
      }
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      if (!live[i]) continue;
      float2 *o = O + ((row0 + i * warps) * 32 + lane) * U;
      if constexpr (MODE == 0) {
        __stcs(o, a0[i]);
      } else {
        __stcs(reinterpret_cast<float4 *>(o), make_float4(a0[i].x, a0[i].y, a1[i].x, a1[i].y));
      }
    }
  }
}

template <int MODE, int RB, bool PF>
cudaError_t launch_rb(const LaneTables *T, const LaneGeom &g, const BatchPtrs &p, bool exact,
                      cudaStream_t st) {
  const size_t smem = size_t(g.w_elems) * sizeof(float2);
  auto kern = exact ? k_absorb_lanes<MODE, true, RB, PF> : k_absorb_lanes<MODE, false, RB, PF>;
  if (smem > 48 * 1024) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         int(smem));
    if (e != cudaSuccess) return e;
  }
  // persistent over rows: 4 CTAs of 256 threads per SM, shared by the batch
  const int64_t per_cta = (kLaneThreads / 32) * RB * 4;
  const int64_t want = (g.rows + per_cta - 1) / per_cta;
  const int64_t cap = std::max<int64_t>(1, 148 * (RB == 1 ? 4 : 3) / std::max(1, p.nbatch));
  const int64_t gx = std::max<int64_t>(1, std::min(want, cap));
  dim3 grid(unsigned(gx), unsigned(p.nbatch));
  kern<<<grid, kLaneThreads, smem, st>>>(T, g, p);
  return cudaGetLastError();
}

template <int MODE>
cudaError_t launch_mode(const LaneTables *T, const LaneGeom &g, const BatchPtrs &p, bool exact,
                        cudaStream_t st) {
  // rows per warp iteration: >= 8 loads in flight per lane; L2 prefetch of the next
  // row group for short K (STN_DEBUG lanes_pf=0|1 overrides)
  const char *pf_opt = debug_opt("lanes_pf");
  const bool pf = pf_opt ? std::atoi(pf_opt) != 0 : g.K <= 4;
  // (16-byte m-pair loads: at most 2 rows, so the loads fit in registers)
  constexpr int RBMAX = MODE == 1 ? 2 : 4;
  if (g.K >= 8) return pf ? launch_rb<MODE, 1, true>(T, g, p, exact, st)
                          : launch_rb<MODE, 1, false>(T, g, p, exact, st);
  if (g.K >= 4 || RBMAX == 2) return pf ? launch_rb<MODE, 2, true>(T, g, p, exact, st)
                                        : launch_rb<MODE, 2, false>(T, g, p, exact, st);
  return pf ? launch_rb<MODE, RBMAX, true>(T, g, p, exact, st)
            : launch_rb<MODE, RBMAX, false>(T, g, p, exact, st);
}

}  // namespace

cudaError_t launch_absorb_lanes(const LaneTables *T, const LaneGeom &g, const BatchPtrs &p,
                                bool exact, cudaStream_t stream) {
  if (g.rows == 0 || p.nbatch == 0) return cudaSuccess;
  switch (g.mode) {
    case 0:
      return launch_mode<0>(T, g, p, exact, stream);
    case 1:
      return launch_mode<1>(T, g, p, exact, stream);
    case 2:
      return launch_mode<2>(T, g, p, exact, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace stn
