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
#include <type_traits>
#include <cstdlib>
#include <cuda_runtime.h>

#include "device_common.cuh"
#include "kernels.h"

namespace stn {


namespace {
using namespace dev;

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
// Tiled SIMT complex GEMM, C[d] = A[d] (MxK, row-major) * B[d] (KxN, row-major).
// 64x64 output tile per CTA, 16-wide K steps, 4x4 outputs per thread; every
// output accumulates k in ascending order.
// ---------------------------------------------------------------------------
// ---------------------------------------------------------------------------
// "Outer" steps (kernels.h OuterGeom): both operands small, the output large
// (e.g. the first stem step, a 2^11 x 2^14 -> 2^23 expansion with K = 2). The
// operand offsets of an output index come from per-byte tables in shared memory
// instead of a per-axis div/mod walk; the K sum runs in k_generic's order with
// the same complex MAC, so results are bitwise those of k_generic.
// ---------------------------------------------------------------------------
template <class R, bool EXACT>
__global__ void __launch_bounds__(256)
    k_outer(const __grid_constant__ OuterGeom g, const BatchPtrs p) {
  using T = cx_t<R>;
  __shared__ int32_t ta[4][256], tb[4][256], ka[64], kb[64];
  for (int i = threadIdx.x; i < 1024; i += blockDim.x) {
    ta[i >> 8][i & 255] = g.ta[i >> 8][i & 255];
    tb[i >> 8][i & 255] = g.tb[i >> 8][i & 255];
  }
  for (int i = threadIdx.x; i < g.nk; i += blockDim.x) {
    ka[i] = g.ka[i];
    kb[i] = g.kb[i];
  }
  __syncthreads();
  const int b = blockIdx.y;
  const T *A = static_cast<const T *>(p.a) + int64_t(b) * p.a_bs;
  const T *B = static_cast<const T *>(p.b) + int64_t(b) * p.b_bs;
  T *O = static_cast<T *>(p.out) + int64_t(b) * p.out_bs;
  const int64_t n = int64_t(1) << g.obits;
  // 8 consecutive outputs per thread: base offsets from the tables once, the three low
  // output bits from register copies of the first table entries
  int32_t la[8], lb[8];
#pragma unroll
  for (int v = 0; v < 8; ++v) {
    la[v] = ta[0][v];
    lb[v] = tb[0][v];
  }
  for (int64_t o = (int64_t(blockIdx.x) * blockDim.x + threadIdx.x) * 8; o < n;
       o += int64_t(gridDim.x) * blockDim.x * 8) {
    const uint32_t ou = uint32_t(o);
    const int32_t ao = ta[0][ou & 255] + ta[1][(ou >> 8) & 255] + ta[2][(ou >> 16) & 255] +
                       ta[3][ou >> 24];
    const int32_t bo = tb[0][ou & 255] + tb[1][(ou >> 8) & 255] + tb[2][(ou >> 16) & 255] +
                       tb[3][ou >> 24];
    T acc[8];
#pragma unroll
    for (int e = 0; e < 8; ++e) {
      acc[e].x = 0;
      acc[e].y = 0;
    }
    for (int k = 0; k < g.nk; ++k) {
      const T *ak = A + ao + ka[k];
      const T *bk = B + bo + kb[k];
#pragma unroll
      for (int e = 0; e < 8; ++e) cmac<EXACT>(acc[e], __ldg(ak + la[e]), __ldg(bk + lb[e]));
    }
#pragma unroll
    for (int e = 0; e < 8; ++e) O[o + e] = acc[e];
  }
}

}  // namespace

template <class R>
cudaError_t launch_outer(const OuterGeom &g, const BatchPtrs &p, bool exact, cudaStream_t stream) {
  const int64_t groups = (int64_t(1) << g.obits) / 8;
  dim3 grid(unsigned(grid_for(groups, 256, 148 * 16)), unsigned(p.nbatch));
  if (exact)
    k_outer<R, true><<<grid, 256, 0, stream>>>(g, p);
  else
    k_outer<R, false><<<grid, 256, 0, stream>>>(g, p);
  return cudaGetLastError();
}
template cudaError_t launch_outer<float>(const OuterGeom &, const BatchPtrs &, bool, cudaStream_t);
template cudaError_t launch_outer<double>(const OuterGeom &, const BatchPtrs &, bool, cudaStream_t);

namespace {

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

// out[i] = (((init + r_0[i]) + r_1[i]) + ...) in ascending slice order, init = 0 or out[i]
// (continuing a fold another device started: the chained cross-GPU reduction)
__global__ void k_sum_ordered(const double *per_slice, uint64_t n_slices, int64_t n, double *out,
                              bool accumulate) {
  for (int64_t i = int64_t(blockIdx.x) * blockDim.x + threadIdx.x; i < 2 * n;
       i += int64_t(gridDim.x) * blockDim.x) {
    double s = accumulate ? out[i] : 0.0;
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
  int64_t *rows = kb_tab + kc;  // [M] A row offsets + ka0, then [N] B column offsets + kb0
  for (int kk = threadIdx.x; kk < kc; kk += blockDim.x) koff(kk, ka_tab[kk], kb_tab[kk]);
  {
    int64_t ka0, kb0;
    koff(k0, ka0, kb0);
    for (int r = threadIdx.x; r < t.M + t.N; r += blockDim.x)
      rows[r] = r < t.M ? t.a_row[r] + ka0 : t.b_col[r - t.M] + kb0;
  }
  __syncthreads();
  // stage A[:, chunk] and B[:, chunk]: consecutive threads take consecutive k;
  // kBatch independent loads in flight per thread before any shared store
  constexpr int kBatch = 8;
  const int kc_log = __ffs(kc) - 1;
  const int total = (t.M + t.N) << kc_log;
  for (int base = 0; base < total; base += kBatch * 256) {
    T v[kBatch];
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int idx = base + j * 256 + int(threadIdx.x);
      const int row = idx >> kc_log, kk = idx & (kc - 1);
      v[j].x = v[j].y = 0;
      if (idx < total && kk < len) {
        const T *src = row < t.M ? A : B;
        v[j] = src[rows[row] + (row < t.M ? ka_tab[kk] : kb_tab[kk])];
      }
    }
#pragma unroll
    for (int j = 0; j < kBatch; ++j) {
      const int idx = base + j * 256 + int(threadIdx.x);
      if (idx < total) sA[(idx >> kc_log) * (kc + 1) + (idx & (kc - 1))] = v[j];  // sB follows sA
    }
  }
  __syncthreads();
  for (int o = threadIdx.x; o < g.out_size; o += blockDim.x) {
    const int mn = t.o_mn[o];
    const T *ra = sA + (mn & 0xFFFF) * (kc + 1);
    const T *rb = sB + (mn >> 16) * (kc + 1);
    // four independent accumulators (k mod 4), summed in a fixed order
    T acc[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) acc[j].x = acc[j].y = 0;
    int kk = 0;
    for (; kk + 4 <= len; kk += 4) {
#pragma unroll
      for (int j = 0; j < 4; ++j) cmac<false>(acc[j], ra[kk + j], rb[kk + j]);
    }
    for (; kk < len; ++kk) cmac<false>(acc[0], ra[kk], rb[kk]);
    T r;
    r.x = (acc[0].x + acc[1].x) + (acc[2].x + acc[3].x);
    r.y = (acc[0].y + acc[1].y) + (acc[2].y + acc[3].y);
    partial[o] = r;
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
  while (kc > 8 && size_t(t.M + t.N) * (kc + 1) * esize + 8 * size_t(t.M + t.N) > 44 * 1024)
    kc /= 2;
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
  const size_t smem = size_t(t.M + t.N) * (kc + 1) * sizeof(cx_t<R>) + 16 * size_t(kc) +
                      8 * size_t(t.M + t.N);
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

// Skinny GEMM (FAST, N <= 8, K * N <= 4096): C[m][:] = A[m][:] . B for very tall A
// (e.g. 2^20 x 512 x 8). The 64 x 64 tile kernel wastes 7/8 of its math on N = 8; here
// B^T sits in shared memory ([n][k]: lanes read consecutive k, no bank conflicts) and
// each warp streams kSkRows rows of A with 16-byte loads along k, every B load serving
// all its rows; the 32 lane partials of each output are summed with xor shuffles.
constexpr int kSkRows = 4, kSkN = 8;
__global__ void __launch_bounds__(256)
    k_gemm_skinny(const GemmShape s, const BatchPtrs p, const int64_t *gtab, int mbits) {
  extern __shared__ __align__(16) float2 bt[];  // [kSkN][K], then (gather) [K] k offsets
  const int64_t batch = blockIdx.z;  // = slice * D + d
  const int64_t slice = batch / s.D, d = batch % s.D;
  const float2 *A = static_cast<const float2 *>(p.a) + slice * p.a_bs + d * s.M * s.K;
  const float2 *B = static_cast<const float2 *>(p.b) + slice * p.b_bs + d * s.K * s.N;
  float2 *C = static_cast<float2 *>(p.out) + slice * p.out_bs + d * s.M * s.N;
  const int K = int(s.K), N = int(s.N);
  // gather form (gtab): A is the step's operand in its own layout; element (m, k) sits
  // at mo(m) + ko(k), ko = gtab[0..K), mo = sum of the bit strides gtab[K + j]
  int64_t *ko = reinterpret_cast<int64_t *>(bt + kSkN * K);
  if (gtab) {
    A = static_cast<const float2 *>(p.a) + slice * p.a_bs;
    for (int k = threadIdx.x; k < K; k += 256) ko[k] = gtab[k];
  }
  for (int e = threadIdx.x; e < kSkN * K; e += 256) {
    const int n = e / K, k = e % K;
    bt[e] = n < N ? B[int64_t(k) * N + n] : make_float2(0.f, 0.f);
  }
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const int64_t m0 = (int64_t(blockIdx.x) * 8 + warp) * kSkRows;
  if (m0 >= s.M) return;
  float2 acc[kSkRows][kSkN];
#pragma unroll
  for (int r = 0; r < kSkRows; ++r)
#pragma unroll
    for (int n = 0; n < kSkN; ++n) acc[r][n] = make_float2(0.f, 0.f);
  int64_t row[kSkRows];
#pragma unroll
  for (int r = 0; r < kSkRows; ++r) {
    row[r] = (m0 + r) * K;
    if (gtab) {
      int64_t o = 0;
      for (int j = 0; j < mbits; ++j)
        if (((m0 + r) >> j) & 1) o += gtab[K + j];
      row[r] = o;
    }
  }
  for (int k = 2 * lane; k < K; k += 64) {
    const int64_t kof = gtab ? ko[k] : k;
    float4 x[kSkRows];
#pragma unroll
    for (int r = 0; r < kSkRows; ++r)
      x[r] = m0 + r < s.M ? __ldcs(reinterpret_cast<const float4 *>(A + row[r] + kof))
                          : make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int n = 0; n < kSkN; ++n) {
      const float4 w = *reinterpret_cast<const float4 *>(bt + n * K + k);
#pragma unroll
      for (int r = 0; r < kSkRows; ++r) {
        cmac<false>(acc[r][n], make_float2(x[r].x, x[r].y), make_float2(w.x, w.y));
        cmac<false>(acc[r][n], make_float2(x[r].z, x[r].w), make_float2(w.z, w.w));
      }
    }
  }
#pragma unroll
  for (int r = 0; r < kSkRows; ++r)
#pragma unroll
    for (int n = 0; n < kSkN; ++n)
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) {
        acc[r][n].x += __shfl_xor_sync(0xffffffffu, acc[r][n].x, o);
        acc[r][n].y += __shfl_xor_sync(0xffffffffu, acc[r][n].y, o);
      }
#pragma unroll
  for (int r = 0; r < kSkRows; ++r) {
    float2 v = acc[r][0];
#pragma unroll
    for (int n = 1; n < kSkN; ++n)
      if (lane == n) v = acc[r][n];
    if (lane < N && m0 + r < s.M) C[(m0 + r) * N + lane] = v;
  }
}

bool gemm_skinny_supported(const GemmShape &s) {
  return s.D == 1 && s.N <= kSkN && s.K % 2 == 0 && s.K >= 64 && s.K * kSkN <= 4096 &&
         s.M >= 4096;
}

cudaError_t launch_gemm_skinny_gather(const GemmShape &s, const BatchPtrs &p, const int64_t *gtab,
                                      int mbits, cudaStream_t stream) {
  if (!gemm_skinny_supported(s)) return cudaErrorNotSupported;
  const int64_t rows_per_cta = 8 * kSkRows;
  dim3 grid(unsigned((s.M + rows_per_cta - 1) / rows_per_cta), 1, unsigned(p.nbatch));
  k_gemm_skinny<<<grid, 256, size_t(kSkN) * s.K * sizeof(float2) + 8 * size_t(s.K), stream>>>(
      s, p, gtab, mbits);
  return cudaGetLastError();
}

template <class R>
cudaError_t launch_gemm_simt(const GemmShape &s, const BatchPtrs &p, bool exact,
                             cudaStream_t stream) {
  if (s.M == 0 || s.N == 0 || p.nbatch == 0) return cudaSuccess;
  if constexpr (std::is_same<R, float>::value) {
    if (!exact && s.N <= kSkN && s.K % 2 == 0 && s.K >= 64 && s.K * kSkN <= 4096 &&
        s.M >= 4096) {
      const int64_t rows_per_cta = 8 * kSkRows;
      dim3 grid(unsigned((s.M + rows_per_cta - 1) / rows_per_cta), 1, unsigned(s.D * p.nbatch));
      k_gemm_skinny<<<grid, 256, size_t(kSkN) * s.K * sizeof(float2), stream>>>(s, p, nullptr, 0);
      return cudaGetLastError();
    }
  }
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
                               cudaStream_t stream, bool accumulate) {
  k_sum_ordered<<<grid_for(2 * n, 256), 256, 0, stream>>>(per_slice, n_slices, n, out, accumulate);
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
