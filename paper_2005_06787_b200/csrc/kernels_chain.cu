// Fused stem chain (kernels.h ChainGeom): a run of consecutive bond-2 absorbs
//   S_1 = S_0 x W_0,  S_2 = S_1 x W_1,  ...,  S_r = S_{r-1} x W_{r-1}
// in ONE pass over HBM: S_0 is read once, S_r written once, the intermediate stems
// (each as large as the stem itself -- 64 GiB at cfg5) never exist in memory.
//
// The reference materialises every stem of the chain (runtime.hpp:439-448, one
// Engine::gemm per step). Here the bits of the stem are split into
//   * passive lines: stem bits no stage of the chain contracts; they only move
//     (the operand / output permutations of runtime.hpp:387-388 and 417 reduce to
//     a relabelling of positions), and
//   * active lines: stem bits some stage contracts (K bits) and W bits a stage
//     creates (N bits).
// A warp owns 32 values of the passive index (the "lane" bits: the lowest
// passive bits, so every load and store of the warp is a contiguous run) and a
// thread keeps the whole active tile of its column -- at most 16 complex values --
// in a per-warp shared-memory buffer laid out [slot][lane] (every access of the
// warp hits 32 consecutive 8-byte words). Each stage reads its R x K inputs in the
// reference's [r][k] order through a slot table, forms the R x N outputs with the
// K terms in ascending k (EXACT: separately rounded products and sums, so the
// intermediate tiles are bitwise the reference's stems; FAST: FMAs), and writes
// them back through a slot table. Higher passive bits ("rows") map to X / O
// offsets through per-byte tables; the grid is persistent over rows.
#include <algorithm>
#include <cstdint>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace stn {

namespace {
using namespace dev;

constexpr int kChThreads = 256;
constexpr int kChWarps = kChThreads / 32;
constexpr int kChTile = 1 << kChainMaxLog;  // slots per column

__device__ __forceinline__ int64_t row_off(const int64_t (*t)[256], uint32_t r) {
  return t[0][r & 255] + t[1][(r >> 8) & 255] + t[2][(r >> 16) & 255] + t[3][r >> 24];
}

// One stage on one column: y[r][n] = sum_k x[r][k] w[k][n], r processed in chunks of
// RC rows so the live registers stay at RC x (K + N) <= 16 complex values (a separate
// function per shape: its registers do not add up with the other shapes').
template <bool EXACT, int LR, int LK, int LN>
__device__ __noinline__ void chain_stage(float2 *__restrict__ tile, int lane,
                                            const uint8_t *__restrict__ rd,
                                            const uint8_t *__restrict__ wr,
                                            const float2 *__restrict__ w) {
  constexpr int R = 1 << LR, K = 1 << LK, N = 1 << LN;
  // rows per chunk: RC (K + N) <= 16 complex values live
  constexpr int RCMAX = 16 / (K + N) > 0 ? 16 / (K + N) : 1;
  constexpr int RC = RCMAX >= R ? R : (RCMAX >= 8 ? 8 : (RCMAX >= 4 ? 4 : (RCMAX >= 2 ? 2 : 1)));
  float2 x[RC * K], y[RC * N];
#pragma unroll 1
  for (int r0 = 0; r0 < R; r0 += RC) {
#pragma unroll
    for (int i = 0; i < RC * K; ++i) x[i] = tile[rd[r0 * K + i] * 32 + lane];
#pragma unroll
    for (int i = 0; i < RC * N; ++i) y[i] = make_float2(0.f, 0.f);
#pragma unroll
    for (int n = 0; n < N; ++n)
#pragma unroll
      for (int k = 0; k < K; ++k) {
        const float2 wv = w[k * N + n];
#pragma unroll
        for (int r = 0; r < RC; ++r) cmac<EXACT>(y[r * N + n], x[r * K + k], wv);
      }
#pragma unroll
    for (int i = 0; i < RC * N; ++i) tile[wr[r0 * N + i] * 32 + lane] = y[i];
  }
}

template <bool EXACT>
__device__ __forceinline__ void run_stage(const ChainStage &st, float2 *tile, int lane,
                                          const uint8_t *rd, const uint8_t *wr, const float2 *w) {
  // every (log R, log K, log N) with R K <= 16 and R N <= 16 (kChainMaxLog = 4)
#define STN_CH(a, b, c)                                                          \
  if (st.lr == a && st.lk == b && st.ln == c) {                                  \
    chain_stage<EXACT, a, b, c>(tile, lane, rd, wr, w);                          \
    return;                                                                      \
  }
  STN_CH(0, 0, 0) STN_CH(0, 0, 1) STN_CH(0, 0, 2) STN_CH(0, 0, 3) STN_CH(0, 0, 4)
  STN_CH(0, 1, 0) STN_CH(0, 1, 1) STN_CH(0, 1, 2) STN_CH(0, 1, 3) STN_CH(0, 1, 4)
  STN_CH(0, 2, 0) STN_CH(0, 2, 1) STN_CH(0, 2, 2) STN_CH(0, 2, 3) STN_CH(0, 2, 4)
  STN_CH(0, 3, 0) STN_CH(0, 3, 1) STN_CH(0, 3, 2) STN_CH(0, 3, 3) STN_CH(0, 3, 4)
  STN_CH(0, 4, 0) STN_CH(0, 4, 1) STN_CH(0, 4, 2) STN_CH(0, 4, 3) STN_CH(0, 4, 4)
  STN_CH(1, 0, 0) STN_CH(1, 0, 1) STN_CH(1, 0, 2) STN_CH(1, 0, 3) STN_CH(1, 1, 0)
  STN_CH(1, 1, 1) STN_CH(1, 1, 2) STN_CH(1, 1, 3) STN_CH(1, 2, 0) STN_CH(1, 2, 1)
  STN_CH(1, 2, 2) STN_CH(1, 2, 3) STN_CH(1, 3, 0) STN_CH(1, 3, 1) STN_CH(1, 3, 2)
  STN_CH(1, 3, 3) STN_CH(2, 0, 0) STN_CH(2, 0, 1) STN_CH(2, 0, 2) STN_CH(2, 1, 0)
  STN_CH(2, 1, 1) STN_CH(2, 1, 2) STN_CH(2, 2, 0) STN_CH(2, 2, 1) STN_CH(2, 2, 2)
  STN_CH(3, 0, 0) STN_CH(3, 0, 1) STN_CH(3, 1, 0) STN_CH(3, 1, 1) STN_CH(4, 0, 0)
#undef STN_CH
}

template <bool EXACT>
__global__ void __launch_bounds__(kChThreads, 3)
    k_chain(const ChainTables *__restrict__ T, const __grid_constant__ ChainGeom g,
            const BatchPtrs p) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  int64_t(*sxr)[256] = reinterpret_cast<int64_t(*)[256]>(smem_raw);
  int64_t(*sor)[256] = sxr + 4;
  int64_t *sxin = reinterpret_cast<int64_t *>(sor + 4);  // [kChTile]
  int64_t *sout = sxin + kChTile;                        // [kChTile]
  uint8_t *stab = reinterpret_cast<uint8_t *>(sout + kChTile);  // rd / wr tables
  float2 *sw = reinterpret_cast<float2 *>(stab + kChainMaxTab);  // W of all stages
  float2 *tiles = sw + g.w_total;                                 // [warp][slot][lane]
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;
  for (int i = threadIdx.x; i < 1024; i += kChThreads) {
    sxr[i >> 8][i & 255] = T->xr[i >> 8][i & 255];
    sor[i >> 8][i & 255] = T->orow[i >> 8][i & 255];
  }
  for (int i = threadIdx.x; i < kChTile; i += kChThreads) {
    sxin[i] = T->xin[i];
    sout[i] = T->oout[i];
  }
  for (int i = threadIdx.x; i < kChainMaxTab; i += kChThreads) stab[i] = T->tab[i];
  for (int s = 0; s < g.n_stages; ++s) {
    const ChainStage &st = g.st[s];
    const float2 *W = static_cast<const float2 *>(g.w[s]) + int64_t(b) * g.w_bs[s];
    const int kn = 1 << (st.lk + st.ln);
    for (int i = threadIdx.x; i < kn; i += kChThreads) sw[st.w_smem + i] = W[T->widx[st.w_off + i]];
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t xl = T->xl[lane], ol = T->ol[lane];
  float2 *tile = tiles + warp * kChTile * 32;
  const int ni = 1 << g.li, no = 1 << g.lo;
  const int64_t warps = int64_t(gridDim.x) * kChWarps;
  for (int64_t row = int64_t(blockIdx.x) * kChWarps + warp; row < g.rows; row += warps) {
    const int64_t bx = row_off(sxr, uint32_t(row)) + xl;
    const int64_t bo = row_off(sor, uint32_t(row)) + ol;
    {  // every input of the column in flight before any is stored
      float2 v[kChTile];
#pragma unroll
      for (int i = 0; i < kChTile; ++i)
        if (i < ni) v[i] = __ldcs(X + bx + sxin[i]);
#pragma unroll
      for (int i = 0; i < kChTile; ++i)
        if (i < ni) tile[i * 32 + lane] = v[i];
    }
    for (int s = 0; s < g.n_stages; ++s) {
      const ChainStage &st = g.st[s];
      run_stage<EXACT>(st, tile, lane, stab + st.rd_off, stab + st.wr_off, sw + st.w_smem);
    }
    {
      float2 v[kChTile];
#pragma unroll
      for (int i = 0; i < kChTile; ++i)
        if (i < no) v[i] = tile[i * 32 + lane];
#pragma unroll
      for (int i = 0; i < kChTile; ++i)
        if (i < no) __stcs(O + bo + sout[i], v[i]);
    }
  }
}

}  // namespace

size_t chain_smem_bytes(const ChainGeom &g) {
  return 8 * 2 * 1024 + 8 * 2 * kChTile + kChainMaxTab + 8 * size_t(g.w_total) +
         size_t(kChWarps) * kChTile * 32 * 8;
}

cudaError_t launch_chain(const ChainTables *T, const ChainGeom &g, const BatchPtrs &p, bool exact,
                         cudaStream_t stream) {
  if (g.rows == 0 || p.nbatch == 0) return cudaSuccess;
  const size_t smem = chain_smem_bytes(g);
  auto kern = exact ? k_chain<true> : k_chain<false>;
  static bool set_on[kMaxDevices][2] = {};
  bool &set = set_on[current_device()][exact ? 1 : 0];
  if (!set) {
    cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         110 * 1024);
    if (e != cudaSuccess) return e;
    set = true;
  }
  if (smem > 110 * 1024) return cudaErrorNotSupported;
  const int64_t want = (g.rows + kChWarps * 4 - 1) / (kChWarps * 4);
  const int64_t cap = std::max<int64_t>(1, 148 * 3 / std::max(1, p.nbatch));
  dim3 grid(unsigned(std::max<int64_t>(1, std::min(want, cap))), unsigned(p.nbatch));
  kern<<<grid, kChThreads, smem, stream>>>(T, g, p);
  return cudaGetLastError();
}

}  // namespace stn
