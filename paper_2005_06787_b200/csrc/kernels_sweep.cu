// Fused stem sweep (kernels.h SweepGeom): a chain of consecutive skinny absorbs
// on the stem, executed tile by tile in shared memory.
//
// The reference materialises every stem tensor of the chain
// (runtime.hpp:439-448: each Engine::gemm writes its full output); on cfg2 the
// stem chains move ~26 GB per slice through HBM just to write and re-read
// intermediate stems. Here a persistent CTA loads a tile of S_0 (the tile holds
// every bit the chain touches plus the low bits for coalescing), applies all
// stages in shared memory, and writes the tile of S_r.
//
// Stage math is register tiled like a GEMM micro-kernel: a thread owns RB M
// indices x NC outputs along N and per k loads RB inputs and NC weights
// (warp-uniform broadcast loads), so the FMA pipe rather than the
// shared-memory pipe bounds the stage. Per output element the K terms
// are accumulated in ascending k with the same complex multiply-add as the
// single-step kernels, so a sweep is bitwise identical to its steps run one by
// one in EXACT mode.
//
// Three tile buffers of 2^max_bits elements rotate: the stages of tile t
// ping-pong between two of them while tile t+1 streams into the third
// (cp.async), so HBM traffic overlaps the stage math within every CTA.
//
// Tile buffers are XOR-swizzled, phys(l) = l ^ ((l>>4 ^ l>>8) & 15), so a label
// at tile position p selects bank pair bit p mod 4 wherever it sits. The swizzle
// is linear over GF(2), so the host bakes it into the index tables
// (phys(base | koff) = phys(base) ^ phys(koff)) and the stage loop pays nothing
// for it; the host also picks the lane bits of r so that a warp's 16-lane
// wavefronts hit 16 distinct bank pairs on both the loads and the stores.
#include <cstdint>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace stn {

namespace {
using namespace dev;

constexpr int kSwThreads = 128;

__device__ __forceinline__ int sw_phys(int l) { return l ^ (((l >> 4) ^ (l >> 8)) & 15); }
__device__ __forceinline__ void sw_cp_async8(void *smem, const void *gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 8;" ::"r"(
                   static_cast<uint32_t>(__cvta_generic_to_shared(smem))),
               "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void sw_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void sw_wait_prev() {  // all but the most recent group
  asm volatile("cp.async.wait_group 1;" ::: "memory");
}
__device__ __forceinline__ void sw_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

// One stage, GEMM-style register tiling: a thread owns RB M indices x NC
// outputs along N; per k it loads RB inputs (distinct per lane) and NC weights
// (warp-uniform broadcast, [k][n] layout so NC consecutive n are one vector
// load) and issues RB*NC complex multiply-adds. Each output still sums its K
// terms in ascending k.
template <bool EXACT, int RB, int NC>
__device__ __forceinline__ void sweep_stage(const SweepStage &st, const float2 *__restrict__ cur,
                                            float2 *__restrict__ out,
                                            const float2 *__restrict__ ws,
                                            const uint16_t *__restrict__ koff,
                                            const uint16_t *__restrict__ nofs) {
  const int rbits = st.out_bits - st.nb;
  const int R = 1 << rbits, N = 1 << st.nb, K = 1 << st.kb;
  const int rl_bits = rbits - st.rb_log;  // lanes vary the low r bits
  const int RL = 1 << rl_bits;
  const int items = RL << (st.nb - st.nc_log);
  for (int item = threadIdx.x; item < items; item += kSwThreads) {
    const int rlo = item & (RL - 1);
    const int n0 = (item >> rl_bits) * NC;
    int base[RB];
#pragma unroll
    for (int i = 0; i < RB; ++i) base[i] = __ldg(st.rb + rlo + i * RL);
    float2 acc[RB][NC];
#pragma unroll
    for (int i = 0; i < RB; ++i)
#pragma unroll
      for (int c = 0; c < NC; ++c) acc[i][c] = make_float2(0.f, 0.f);
    const float2 *wk = ws + n0;
#pragma unroll 2
    for (int k = 0; k < K; ++k, wk += N) {
      const int ko = koff[k];
      float2 x[RB], w[NC];
#pragma unroll
      for (int i = 0; i < RB; ++i) x[i] = cur[base[i] ^ ko];
      if constexpr (NC >= 2) {
#pragma unroll
        for (int c = 0; c < NC; c += 2) {
          const float4 w2 = *reinterpret_cast<const float4 *>(wk + c);
          w[c] = make_float2(w2.x, w2.y);
          w[c + 1] = make_float2(w2.z, w2.w);
        }
      } else {
        w[0] = wk[0];
      }
#pragma unroll
      for (int i = 0; i < RB; ++i)
#pragma unroll
        for (int c = 0; c < NC; ++c) cmac<EXACT>(acc[i][c], x[i], w[c]);
    }
#pragma unroll
    for (int i = 0; i < RB; ++i) {
      const int ob = __ldg(st.ro + rlo + i * RL);
#pragma unroll
      for (int c = 0; c < NC; ++c) out[ob ^ nofs[n0 + c]] = acc[i][c];
    }
  }
  (void)R;
}

#define STN_SWEEP_ARGS st, cur, out, ws, koff, nofs
template <bool EXACT, int RB>
__device__ __forceinline__ void sweep_stage_nc(const SweepStage &st, const float2 *cur,
                                               float2 *out, const float2 *ws,
                                               const uint16_t *koff, const uint16_t *nofs) {
  switch (st.nc_log) {
    case 0: sweep_stage<EXACT, RB, 1>(STN_SWEEP_ARGS); break;
    case 1: sweep_stage<EXACT, RB, 2>(STN_SWEEP_ARGS); break;
    case 2: sweep_stage<EXACT, RB, 4>(STN_SWEEP_ARGS); break;
    default: if constexpr (RB <= 4) sweep_stage<EXACT, RB, 8>(STN_SWEEP_ARGS); break;
  }
}

template <bool EXACT>
__device__ __forceinline__ void sweep_stage_any(const SweepStage &st, const float2 *cur,
                                                float2 *out, const float2 *ws,
                                                const uint16_t *koff, const uint16_t *nofs) {
  switch (st.rb_log) {
    case 0: sweep_stage_nc<EXACT, 1>(STN_SWEEP_ARGS); break;
    case 1: sweep_stage_nc<EXACT, 2>(STN_SWEEP_ARGS); break;
    case 2: sweep_stage_nc<EXACT, 4>(STN_SWEEP_ARGS); break;
    default: sweep_stage_nc<EXACT, 8>(STN_SWEEP_ARGS); break;
  }
}
#undef STN_SWEEP_ARGS

template <bool EXACT>
__global__ void __launch_bounds__(kSwThreads, 2)
    k_sweep(const __grid_constant__ SweepGeom g, const BatchPtrs p, int64_t n_tiles, int dbg) {
  extern __shared__ __align__(16) unsigned char smem_raw[];
  const AbsorbGeom &io = g.io;
  const int xt = io.xt_bits, ot = io.ot_bits;
  const int x_hi_n = 1 << (xt - io.x_run), o_hi_n = 1 << (ot - io.o_run);
  float2 *bufs = reinterpret_cast<float2 *>(smem_raw);  // 3 x [2^max_bits]
  float2 *wsm = bufs + 3 * (1 << g.max_bits);            // all stages' W^T
  int64_t *xhi = reinterpret_cast<int64_t *>(wsm + g.w_total);
  int64_t *ohi = xhi + x_hi_n;
  uint16_t *tabs = reinterpret_cast<uint16_t *>(ohi + o_hi_n);  // koff / nofs of all stages
  const int tid = threadIdx.x;
  const int b = blockIdx.y;
  const float2 *X = static_cast<const float2 *>(p.a) + int64_t(b) * p.a_bs;
  float2 *O = static_cast<float2 *>(p.out) + int64_t(b) * p.out_bs;

  for (int i = tid; i < x_hi_n; i += kSwThreads) {
    int64_t off = 0;
    for (int l = io.x_run; l < xt; ++l)
      if ((i >> (l - io.x_run)) & 1) off += int64_t(1) << io.x_tile_pos[l];
    xhi[i] = off;
  }
  for (int i = tid; i < o_hi_n; i += kSwThreads) {
    int64_t off = 0;
    for (int l = io.o_run; l < ot; ++l)
      if ((i >> (l - io.o_run)) & 1) off += int64_t(1) << io.o_tile_pos[l];
    ohi[i] = off;
  }
  for (int s = 0; s < g.n_stages; ++s) {
    const SweepStage &st = g.st[s];
    const int KN = 1 << (st.kb + st.nb);
    const float2 *W = static_cast<const float2 *>(g.w[s]) + int64_t(b) * g.w_bs[s];
    for (int i = tid; i < KN; i += kSwThreads) wsm[st.w_smem + i] = W[st.w_idx[i]];
    for (int i = tid; i < (1 << st.kb); i += kSwThreads) tabs[st.t_smem + i] = st.koff[i];
    for (int i = tid; i < (1 << st.nb); i += kSwThreads)
      tabs[st.t_smem + (1 << st.kb) + i] = st.nofs[i];
  }
  __syncthreads();

  auto tile_bases = [&](int64_t tile, int64_t &bx, int64_t &bo) {
    bx = 0;
    bo = 0;
    for (int j = 0; j < io.ob; ++j)
      if ((tile >> j) & 1) {
        bx += int64_t(1) << io.outer_x[j];
        bo += int64_t(1) << io.outer_o[j];
      }
  };
  const int x_run_mask = (1 << io.x_run) - 1, o_run_mask = (1 << io.o_run) - 1;
  // Three tile buffers rotate: the next tile's input streams into the third
  // while the stages of the current tile ping-pong between the other two.
  auto issue_load = [&](int64_t tile, float2 *dst) {
    if (tile < n_tiles && !(dbg & 2)) {
      int64_t bx, bo;
      tile_bases(tile, bx, bo);
      for (int i = tid; i < (1 << xt); i += kSwThreads)
        sw_cp_async8(dst + sw_phys(i), X + bx + xhi[i >> io.x_run] + (i & x_run_mask));
    }
    sw_commit();
  };
  const int bsz = 1 << g.max_bits;
  int pin = 0, pw = 1, pf = 2;  // input, work, prefetch buffer
  issue_load(blockIdx.x, bufs);
  for (int64_t tile = blockIdx.x; tile < n_tiles; tile += gridDim.x) {
    issue_load(tile + gridDim.x, bufs + pf * bsz);
    sw_wait_prev();
    __syncthreads();
    float2 *cur = bufs + pin * bsz;
    float2 *out = bufs + pw * bsz;
    for (int s = 0; s < ((dbg & 1) ? 0 : g.n_stages); ++s) {
      const SweepStage &st = g.st[s];
      sweep_stage_any<EXACT>(st, cur, out, wsm + st.w_smem, tabs + st.t_smem,
                             tabs + st.t_smem + (1 << st.kb));
      __syncthreads();
      float2 *t = out;
      out = cur;
      cur = t;
    }
    int64_t bx, bo;
    tile_bases(tile, bx, bo);
    if (!(dbg & 2))
      for (int q = tid; q < (1 << (ot - 1)); q += kSwThreads) {
        const int i = q << 1, ph = sw_phys(i);
        float4 v = reinterpret_cast<const float4 *>(cur)[ph >> 1];
        if (ph & 1) v = make_float4(v.z, v.w, v.x, v.y);  // the pair sits swapped
        __stcs(reinterpret_cast<float4 *>(O + bo + ohi[i >> io.o_run] + (i & o_run_mask)), v);
      }
    __syncthreads();  // the buffers of this tile are reused as prefetch target
    const int npin = pf;
    pf = pw;
    pw = pin;
    pin = npin;
  }
  sw_wait_all();
}

}  // namespace

size_t sweep_smem_bytes(const SweepGeom &g) {
  const AbsorbGeom &io = g.io;
  return 8 * (3 * (size_t(1) << g.max_bits) + size_t(g.w_total)) +
         8 * ((size_t(1) << (io.xt_bits - io.x_run)) + (size_t(1) << (io.ot_bits - io.o_run))) +
         2 * size_t(g.t_total);
}

cudaError_t launch_sweep(const SweepGeom &g, const BatchPtrs &p, bool exact,
                         cudaStream_t stream) {
  const size_t smem = sweep_smem_bytes(g);
  if (smem > 220 * 1024) return cudaErrorNotSupported;
  auto kern = exact ? k_sweep<true> : k_sweep<false>;
  cudaError_t e = cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                       220 * 1024);
  if (e != cudaSuccess) return e;
  int per_sm = 0;
  e = cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kern, kSwThreads, smem);
  if (e != cudaSuccess) return e;
  if (per_sm < 1) per_sm = 1;
  const int64_t n_tiles = int64_t(1) << g.io.ob;
  int64_t ctas = int64_t(148) * per_sm / (p.nbatch > 0 ? p.nbatch : 1);
  if (ctas < 1) ctas = 1;
  if (ctas > n_tiles) ctas = n_tiles;
  dim3 grid(unsigned(ctas), unsigned(p.nbatch));
  static const int dbg = stn::debug_opt("sweep_dbg") ? std::atoi(stn::debug_opt("sweep_dbg")) : 0;
  kern<<<grid, kSwThreads, smem, stream>>>(g, p, n_tiles, dbg);
  return cudaGetLastError();
}

}  // namespace stn
