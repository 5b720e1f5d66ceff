// Tiled bond-2 bit permutation (kernels.h PermTileGeom): out[perm(i)] = in[i] for the
// operand / result transposes of the GEMM-shaped steps (runtime.hpp:113-140 is the
// reference's permute). One CTA moves one tile of 2^TB complex elements: the tile bits
// hold the lowest input bits and the positions of the lowest output bits, so both the
// 16-byte loads (input order) and the 16-byte stores (output order) run along
// contiguous memory; the transpose happens in shared memory. Non-persistent, many
// CTAs per SM: the memory-level parallelism comes from occupancy.
#include <cstdint>
#include <cstdlib>
#include <cstring>
#include <cuda_runtime.h>

#include "kernels.h"

namespace stn {

namespace {

constexpr int kPermThreads = 256;

__device__ __forceinline__ float tf32_rna(float x) {
  uint32_t r;
  asm("cvt.rna.tf32.f32 %0, %1;" : "=r"(r) : "f"(x));
  return __uint_as_float(r);
}

// SPLIT: instead of the permuted tensor, write its TF32 hi / lo planes (out, out_lo),
// the operand preparation of the tcgen05 GEMM (gemm_tc.cu k_split_a) fused in.
template <int TB, bool SPLIT>
__global__ void __launch_bounds__(kPermThreads)
    k_perm_tiles(const __grid_constant__ PermTileGeom g, const int64_t *__restrict__ bases,
                 const float2 *__restrict__ in, float2 *__restrict__ out,
                 float2 *__restrict__ out_lo, int64_t in_bs, int64_t out_bs) {
  constexpr int E = 1 << TB;
  __shared__ __align__(16) float2 tile[E];
  __shared__ int64_t io[2][64], oo[2][64];
  __shared__ uint16_t lt[2][64];
  const int tid = threadIdx.x;
  if (tid < 128) {
    const int h = tid >> 6, i = tid & 63;
    io[h][i] = g.in_off[h][i];
    oo[h][i] = g.out_off[h][i];
    lt[h][i] = g.li_of_lo[h][i];
  }
  const int64_t t = blockIdx.x;
  const float2 *src = in + int64_t(blockIdx.y) * in_bs + bases[2 * t];
  const int64_t dst_off = int64_t(blockIdx.y) * out_bs + bases[2 * t + 1];
  float2 *dst = out + dst_off;
  __syncthreads();
  // input order: pairs of consecutive elements (input bit 0 is tile bit 0)
#pragma unroll
  for (int p = tid; p < E / 2; p += kPermThreads) {
    const int li = 2 * p;
    const float4 v = __ldcs(reinterpret_cast<const float4 *>(src + io[0][li & 63] + io[1][li >> 6]));
    reinterpret_cast<float4 *>(tile)[p] = v;
  }
  __syncthreads();
  // output order: pairs of consecutive output elements (output bit 0 is tile bit 0 of lo)
#pragma unroll
  for (int p = tid; p < E / 2; p += kPermThreads) {
    const int lo = 2 * p;
    const int a = lt[0][lo & 63] | lt[1][lo >> 6];
    const int b = lt[0][(lo + 1) & 63] | lt[1][(lo + 1) >> 6];
    const float2 x = tile[a], y = tile[b];
    const int64_t o = oo[0][lo & 63] + oo[1][lo >> 6];
    if constexpr (SPLIT) {
      const float4 h = make_float4(tf32_rna(x.x), tf32_rna(x.y), tf32_rna(y.x), tf32_rna(y.y));
      __stcs(reinterpret_cast<float4 *>(dst + o), h);
      __stcs(reinterpret_cast<float4 *>(out_lo + dst_off + o),
             make_float4(x.x - h.x, x.y - h.y, y.x - h.z, y.y - h.w));
    } else {
      __stcs(reinterpret_cast<float4 *>(dst + o), make_float4(x.x, x.y, y.x, y.y));
    }
  }
}

}  // namespace

// perm: output axis i = input axis perm[i] (all dims 2, axis 0 most significant).
bool build_perm_tiles(const std::vector<int> &perm, PermTileGeom &g, std::vector<int64_t> &bases) {
  const int r = int(perm.size());
  if (r < 10 || r > 40) return false;
  std::vector<int> outpos(r), inpos_of_out(r);
  for (int i = 0; i < r; ++i) {
    const int p = r - 1 - perm[i], q = r - 1 - i;
    outpos[p] = q;
    inpos_of_out[q] = p;
  }
  std::vector<char> in_s(r, 0);
  int n = 0;
  auto add = [&](int p) {
    if (!in_s[p]) {
      in_s[p] = 1;
      ++n;
    }
  };
  static const char *env_tb = stn::debug_opt("perm_tb");  // experiments: tile bits
  const int target = env_tb ? std::atoi(env_tb) : 11;  // 16 KiB tiles: measured best on B200
  for (int p = 0; p < 5; ++p) add(p);
  for (int q = 0; q < 5 && n < target; ++q) add(inpos_of_out[q]);
  for (int k = 5; n < target && k < r; ++k) {
    add(k);
    if (n < target) add(inpos_of_out[k]);
  }
  if (n < 8 || n > 12) return false;
  std::vector<int> sin, sout, outer;
  for (int p = 0; p < r; ++p) (in_s[p] ? sin : outer).push_back(p);
  for (int q = 0; q < r; ++q)
    if (in_s[inpos_of_out[q]]) sout.push_back(inpos_of_out[q]);
  std::vector<int> idx_in(r, -1);
  for (int j = 0; j < n; ++j) idx_in[sin[j]] = j;
  std::memset(&g, 0, sizeof g);
  g.tb = n;
  for (int h = 0; h < 2; ++h)
    for (int v = 0; v < 64; ++v) {
      int64_t io = 0, oo = 0;
      int li = 0;
      for (int j = 0; j < 6; ++j) {
        const int bit = 6 * h + j;
        if (!((v >> j) & 1) || bit >= n) continue;
        io += int64_t(1) << sin[bit];
        oo += int64_t(1) << outpos[sout[bit]];
        li |= 1 << idx_in[sout[bit]];
      }
      g.in_off[h][v] = io;
      g.out_off[h][v] = oo;
      g.li_of_lo[h][v] = uint16_t(li);
    }
  const int nout = int(outer.size());
  g.n_tiles = int64_t(1) << nout;
  if (g.n_tiles > (int64_t(1) << 24)) return false;
  bases.assign(size_t(2 * g.n_tiles), 0);
  // tile t's bits enumerate the outer input positions in ascending order
  for (int64_t t = 0; t < g.n_tiles; ++t) {
    int64_t ib = 0, ob = 0;
    for (int j = 0; j < nout; ++j)
      if ((t >> j) & 1) {
        ib += int64_t(1) << outer[j];
        ob += int64_t(1) << outpos[outer[j]];
      }
    bases[2 * t] = ib;
    bases[2 * t + 1] = ob;
  }
  return true;
}

cudaError_t launch_perm_tiles(const PermTileGeom &g, const int64_t *bases, const void *in,
                              void *out, int64_t in_bs, int64_t out_bs, int nbatch,
                              cudaStream_t stream, void *out_lo) {
  dim3 grid(unsigned(g.n_tiles), unsigned(nbatch));
  const float2 *x = static_cast<const float2 *>(in);
  float2 *y = static_cast<float2 *>(out), *ylo = static_cast<float2 *>(out_lo);
#define STN_PERM(TBV)                                                                    \
  case TBV:                                                                              \
    if (ylo)                                                                             \
      k_perm_tiles<TBV, true><<<grid, kPermThreads, 0, stream>>>(g, bases, x, y, ylo, in_bs, \
                                                                 out_bs);                \
    else                                                                                 \
      k_perm_tiles<TBV, false><<<grid, kPermThreads, 0, stream>>>(g, bases, x, y, nullptr,   \
                                                                  in_bs, out_bs);        \
    break;
  switch (g.tb) {
    STN_PERM(8) STN_PERM(9) STN_PERM(10) STN_PERM(11) STN_PERM(12)
    default: return cudaErrorNotSupported;
  }
#undef STN_PERM
  return cudaGetLastError();
}

}  // namespace stn
