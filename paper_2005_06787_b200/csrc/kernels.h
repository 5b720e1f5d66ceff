// Internal interface between the host executor (stn_exec.cpp) and the sm_100a
// kernels (kernels.cu, gemm_tc.cu). Not part of the C ABI.
//
// Every tensor is complex, interleaved (re, im), in the reference's canonical
// layout: axes sorted by ascending edge id, row-major (runtime.hpp:341-346).
// A "batch" is a set of slices executed together; operand batch strides are in
// complex elements and are 0 for slice-invariant operands.
#pragma once

#include <cstdint>
#include <cuda_runtime.h>

#include <cstdlib>
#include <mutex>
#include <set>
#include <string>
#include <utility>
#include <vector>

namespace stn {

// Experiment and diagnostic switches of the executor, all behind ONE environment
// variable (unset in production): STN_DEBUG="key=value,key,...". Keys:
//   lanes=0|1|all          lane-mapped absorb off / default policy / every eligible step
//   lanes_pf=0|1           lane absorb: L2 prefetch of the next row group (default K <= 4)
//   direct_max_bits=B      direct absorb only for K x N <= 2^B (default 12)
//   direct_min_l=L         direct absorb needs >= L identity low bits (default 2)
//   mma_min_bits=B         tensor-core direct absorb from K x N >= 2^B (default 10)
//   tma_min_bits=B         TMA absorb for every K x N >= 2^B
//   absorb_policy=simt|tc  tiled absorb: never / from K x N >= 64 on tensor cores
//   sweep_bits=B, sweep_debug, sweep_dbg=N   stem-sweep fusion tile size / traces
//   plan_dump, plan_timing                 per-step kernel choice / plan-build timing
//   graphs=0               no CUDA graphs: every batch launched kernel by kernel
//   chain=0, chain_min_bits=B, chain_jit=0   fused stem chains off / only with
//                          intermediates >= 2^B elements (default 24) / table kernel only
//   chain_single=0|2       one-stage chains off / for every step that fits (measurements)
//   chain_multi_log=L      tile limit of multi-stage chains (default 6 = 64 values)
//   chain_exp=0, chain_exp_pen=0   no expansion rows / no penalty for large expanded operands
//   chain_vec=0|1|2        widest tile access (1, 2, 4 complex); chain_swap=0: no exchanges
//   chain_pf_log=L         software-pipeline rows of tiles up to 2^L values
//   chain_ffma2=1, chain_wreg=V, chain_wreg_exp=V, chain_alt=1   stage-math experiments
//   chain_why=S, chain_src  why segments from step S do not fit / NVRTC source in the log
//   side=1                 small steps on a second stream of the lane
//   gemm_mc=1|2|4, gemm_gm=G   wide GEMM cluster size / raster band height in m tiles
//   tcf_gather=0           fused-split GEMM reads a permuted A from a permuted copy
//   bitperm_legacy         legacy bit-permute kernel for the selftest
//   sweep_only=..., no_bulk, tma_lag=N, tma_nsr=N, perm_tb=N   pipeline experiments
//   tcf=0|1|2              fused-split GEMM never / for 2N <= 128 (default) / always
//   tcf_bn=64|128|256      fused-split GEMM tile width
//   mma_v1, mma_dbg=N, tma_dbg=N, absorb_loader=tma|gather, gemm_bn=N   kernel experiments
// Returns the value ("" for a bare key) or nullptr when the key is absent. Read at
// every call (tests change it at run time); returned strings stay valid.
inline const char *debug_opt(const char *key) {
  static std::mutex mu;
  static std::set<std::string> interned;
  const char *e = std::getenv("STN_DEBUG");
  if (!e) return nullptr;
  std::string s = e, item;
  for (size_t i = 0; i <= s.size(); ++i) {
    if (i == s.size() || s[i] == ',') {
      const size_t eq = item.find('=');
      if (item.substr(0, eq) == key) {
        std::lock_guard<std::mutex> lk(mu);
        return interned.insert(eq == std::string::npos ? std::string() : item.substr(eq + 1))
            .first->c_str();
      }
      item.clear();
    } else {
      item += s[i];
    }
  }
  return nullptr;
}

// Index of the current CUDA device: function attributes (dynamic shared-memory
// opt-in) are per device context, so "set once" flags are kept per device.
constexpr int kMaxDevices = 64;
inline int current_device() {
  int d = 0;
  if (cudaGetDevice(&d) != cudaSuccess || d < 0 || d >= kMaxDevices) d = 0;
  return d;
}

constexpr int kMaxAxes = 40;

// Generic strided contraction (any bond dimensions, D batches included):
//   out[o] = sum_k A[a_off(o) + ka_off(k)] * B[b_off(o) + kb_off(k)]
// with o running over the canonical output index and k over the K axes in the
// reference's [D|M|K] order (ascending edge id, first axis most significant).
// Axes are listed outermost first; adjacent axes are pre-merged where both
// operand strides allow it.
struct StridedGeom {
  int n_out;
  int n_k;
  int64_t out_size;
  int64_t k_size;
  int64_t out_dim[kMaxAxes];
  int64_t out_sa[kMaxAxes];
  int64_t out_sb[kMaxAxes];
  int64_t k_dim[kMaxAxes];
  int64_t k_sa[kMaxAxes];
  int64_t k_sb[kMaxAxes];
};

// Batched operand pointers.
struct BatchPtrs {
  const void *a;
  const void *b;
  void *out;
  int64_t a_bs, b_bs, out_bs;  // complex-element batch strides
  int nbatch;
};

// Small operands, large output (kernels.cu k_outer): output index bits -> operand
// offsets through per-byte tables (4 bytes cover <= 32 output bits), K terms in the
// reference order (bitwise equal to k_generic in both modes).
struct OuterGeom {
  int obits;                 // log2 output size (pow2 dims)
  int nk;                    // K terms (<= 64)
  int32_t ta[4][256], tb[4][256];
  int32_t ka[64], kb[64];    // operand offsets of k, row-major over the K axes
};
template <class R>
cudaError_t launch_outer(const OuterGeom &g, const BatchPtrs &p, bool exact, cudaStream_t stream);

// Bond-2 "absorb": one big operand X (the stem side) contracted with a small
// operand W over K bits, producing N new bits:
//   O[m, n] = sum_k X[m, k] * W[k, n]
// X/O/W bits are positions in the flat canonical index (bit 0 = fastest axis).
// A CTA owns one assignment of the "outer" M bits and the full tile over the
// "tile" M bits T, all K bits and all N bits. Tile-local indices list the tile
// bits in ascending position of the respective tensor, so the lowest bits of X
// and O (always inside the tile) give coalesced runs.
constexpr int kAbsorbMaxTileBits = 14;  // X/O tile <= 2^14 complex (128 KiB)
constexpr int kAbsorbMaxKN = 6;         // K, N <= 64
struct AbsorbGeom {
  int x_bits, o_bits;       // log2 |X|, log2 |O|
  int kb, nb, tb, ob;       // #K, #N, #tile M, #outer M bits
  int xt_bits, ot_bits;     // tile bits in X (kb+tb) and in O (nb+tb)
  int x_run, o_run;         // lowest X / O bits that are contiguous inside the tile
  int w_is_lhs;             // 1: W is the lhs operand (product order w*x)
  int64_t w_k_stride[kAbsorbMaxKN];  // W element stride of each K bit (k bit j, LSB first)
  int64_t w_n_stride[kAbsorbMaxKN];  // W element stride of each N bit (n bit j, LSB first)
  uint8_t x_tile_pos[kAbsorbMaxTileBits + kAbsorbMaxKN];  // X position of tile-local X bit i
  uint8_t o_tile_pos[kAbsorbMaxTileBits + kAbsorbMaxKN];  // O position of tile-local O bit i
  uint8_t t_xl[kAbsorbMaxTileBits];  // tile-local X bit of T bit j (T bits in ascending X pos)
  uint8_t t_ol[kAbsorbMaxTileBits];  // tile-local O bit of T bit j
  uint8_t k_xl[kAbsorbMaxKN];        // tile-local X bit of K bit j (ascending X pos)
  uint8_t n_ol[kAbsorbMaxKN];        // tile-local O bit of N bit j (ascending O pos)
  uint8_t outer_x[34];               // X position of outer M bit j
  uint8_t outer_o[34];               // O position of outer M bit j
};

// "Direct" bond-2 absorb: no shared-memory tile. Valid when the lowest L bits
// of X are M bits that are also the lowest L bits of O (same order), so a warp
// streams 16-byte pairs of consecutive m straight from X to O for every k / n.
// M index m = m_hi << L | m_lo; the high M bits scatter to positions given by
// the bit masks hi_x (in X) and hi_o (in O), enumerated with pdep increments.
struct DirectGeom {
  int L;                     // identity low bits (>= 2)
  int kb, nb;                // K bits (<= 6), N bits (<= 12), K*N <= 4096
  int mh_bits;               // high M bits
  uint64_t hi_x_mask, hi_o_mask;
  uint8_t k_xpos[6];         // X position of K bit j (ascending)
  uint8_t n_opos[12];        // O position of N bit j (ascending)
  int64_t w_k_stride[6];     // W stride of K bit j
  int64_t w_n_stride[12];    // W stride of N bit j
};
bool direct_absorb_launchable(const DirectGeom &g);

// Lane-mapped bond-2 absorb (kernels_lanes.cu), single precision: any
// interleaving of M bits (from the stem X) and N bits (from W) in the output.
// Output index o = ((row << 5) | lane) << U | pair, U = 0 (mode 0) or 1 (mode 1:
// the pair bit is X bit 0, so X is read as 16-byte m pairs; mode 2: the pair bit
// is an N bit whose W offset is w_pair). Every output bit maps to an X offset or
// a W offset: lane bits through xl / wl, row bits through per-byte tables.
constexpr int kLaneMaxK = 64;
struct LaneTables {        // device memory, one per step
  int64_t xr[4][256];      // X offset of row byte c with value v
  int32_t wr[4][256];      // W offset of row byte c with value v
  int64_t xl[32];          // X offset of lane bits
  int32_t wl[32];          // W offset of lane bits
  int64_t xk[kLaneMaxK];   // X offset of k (bit j of k = K bit j, ascending X position)
  int32_t wk[kLaneMaxK];   // W offset of k
};
struct LaneGeom {
  int mode;                // 0, 1, 2 (above)
  int K;                   // k terms (<= 64)
  int64_t rows;            // output rows of 32 lanes per batch
  int32_t w_pair;          // mode 2: W offset of the pair bit
  int32_t w_elems;         // W elements staged in shared memory (<= 8192)
};
cudaError_t launch_absorb_lanes(const LaneTables *T, const LaneGeom &g, const BatchPtrs &p,
                                bool exact, cudaStream_t stream);
cudaError_t launch_absorb_direct(const DirectGeom &g, const BatchPtrs &p, bool exact,
                                 cudaStream_t stream);

// Fused stem chain (kernels_chain.cu): consecutive bond-2 absorbs in one HBM pass,
// a warp = 32 columns of the passive (never contracted) stem bits, a thread = the
// active tile of its column (<= 2^kChainMaxLog complex values).
constexpr int kChainMaxStages = 8;
constexpr int kChainMaxLog = 6;      // tile limit of the NVRTC-specialised kernels (chain_jit.cpp)
constexpr int kChainMultiLog = 6;    // ... for chains of more than one stage (spilling
                                     // kernels are re-planned: stn_exec.cpp plan_chains)
constexpr int kChainTableLog = 4;    // tile limit of the table-driven kernel (kernels_chain.cu)
constexpr int kChainMaxTab = 2 * kChainMaxStages * (1 << kChainMaxLog);  // rd + wr slots
constexpr int kChainMaxW = 5120;  // W elements of a chain (shared memory, 40 KiB)
struct ChainStage {
  int lr, lk, ln;   // log2 of the stage's R (other active lines), K and N
  int rd_off;       // tab offset: slot of input (r, k), [R][K]
  int wr_off;       // tab offset: slot of output (r, n), [R][N]
  int w_off;        // widx offset: W element of (k, n), [K][N]
  int w_smem;       // offset of the stage's W in shared memory
};
struct ChainGeom {
  int n_stages;
  int li, lo;                       // log2 input / output elements per column
  int ma;                           // log2 of the largest tile (slots per column)
  int64_t rows;                     // rows of 32 columns (per batch)
  int w_total;                      // W elements of all stages
  int n_exp;                        // expansion row bits of stage 0 (specialised kernel)
  ChainStage st[kChainMaxStages];
  const void *w[kChainMaxStages];   // filled at launch
  int64_t w_bs[kChainMaxStages];
};
struct ChainTables {                // device memory, one per chain
  int64_t xr[4][256], orow[4][256]; // X / O offsets of the row bytes
  int64_t xl[32], ol[32];           // X / O offsets of the lane bits
  int64_t xin[1 << kChainMaxLog];   // X offset of input element i (first stage's layout)
  int64_t oout[1 << kChainMaxLog];  // O offset of output element j (last stage's layout)
  uint8_t tab[kChainMaxTab];        // rd / wr slot tables of all stages
  int32_t widx[kChainMaxW];         // W element offsets, [K][N] per stage
};
size_t chain_smem_bytes(const ChainGeom &g);
cudaError_t launch_chain(const ChainTables *T, const ChainGeom &g, const BatchPtrs &p, bool exact,
                         cudaStream_t stream);

// Fused stem sweep: a chain of consecutive bond-2 absorbs S_{j+1} = S_j x W_j
// executed tile by tile in shared memory. Only S_0 is read from and S_r written
// to HBM; the intermediate stems never exist in memory. Every stage sums its K
// terms in ascending k exactly like the single-step kernels, so a sweep is
// bitwise identical to running its steps one by one.
constexpr int kSweepMaxStages = 24;
constexpr int kSweepMaxTileBits = 12;
struct SweepStage {
  int in_bits, out_bits;  // tile bits before / after the stage
  int kb, nb;             // K and N bits of the stage
  int nc_log;             // outputs per thread along N (register tile), log2
  int rb_log;             // M indices per thread (register tile), log2; rb+nc <= 5
  const uint16_t *rb;     // [2^(out_bits-nb)] input tile offset of M index r
  const uint16_t *ro;     // [2^(out_bits-nb)] output tile offset of M index r
  const uint16_t *koff;   // [2^kb] input tile offset of k
  const uint16_t *nofs;   // [2^nb] output tile offset of n
  const int64_t *w_idx;   // [K*N] W element offset of (k, n), k-major
  int w_smem;             // offset of this stage's W^T in the smem W area (elements)
  int t_smem;             // offset of this stage's koff/nofs in the smem table area
};
struct SweepGeom {
  AbsorbGeom io;            // input tile (x_*) / output tile (o_*) / outer bits; kb = nb = 0
  int n_stages;
  int max_bits;             // largest tile over all stages
  int w_total;              // W elements of all stages
  int t_total;              // koff + nofs entries of all stages
  SweepStage st[kSweepMaxStages];
  const void *w[kSweepMaxStages];  // per-launch W pointers
  int64_t w_bs[kSweepMaxStages];   // and batch strides
};
cudaError_t launch_sweep(const SweepGeom &g, const BatchPtrs &p, bool exact, cudaStream_t stream);
size_t sweep_smem_bytes(const SweepGeom &g);  // dynamic shared memory of one CTA

// Dense batched complex GEMM on materialised operands:
//   C[d] (M x N) = A[d] (M x K, row-major) * B[d] (K x N, row-major)
struct GemmShape {
  int64_t D, M, N, K;
};

// Slice-dependent leaf gather: for every sliced leaf and every slice in the
// batch, restrict the double-precision vertex tensor on its sliced axes
// (digits), convert to the executor's real type and lay it out canonically.
struct LeafGatherTable {
  const double *values;        // device: all sliced leaves' values, concatenated
  const int64_t *src_base;     // [total_out] source complex index with sliced axes at 0
  const int32_t *elem_leaf;    // [total_out] leaf id of output element
  const int64_t *dst_off;      // [n_leaves] per-slice arena offset (scaled by the batch size)
  const int64_t *dst_bs;       // [n_leaves] batch stride of the leaf's output
  const int32_t *elem_local;   // [total_out] element index inside its leaf
  const int32_t *ax_begin;     // [n_leaves + 1] range into ax_stride/ax_slice
  const int64_t *ax_stride;    // source stride of each sliced axis
  const int32_t *ax_slice;     // sliced-edge index of each sliced axis
  int64_t total_out;
  int n_sliced;
};

// ---- launchers (kernels.cu); all asynchronous on `stream` ----
template <class R>
cudaError_t launch_generic(const StridedGeom &g, const BatchPtrs &p, bool exact,
                           cudaStream_t stream);
cudaError_t launch_absorb(const AbsorbGeom &g, const BatchPtrs &p, bool exact, cudaStream_t stream);
template <class R>
cudaError_t launch_permute(const StridedGeom &g, const void *in, void *out, int64_t in_bs,
                           int64_t out_bs, int nbatch, cudaStream_t stream);
// tcgen05 split-TF32 absorb (absorb_tc.cu): AbsorbGeom with exactly 7 tile
// bits (128 rows), K <= 32, N <= 64. FAST mode only.
bool tc_absorb_supported(const AbsorbGeom &g);
// tcgen05 direct absorb (absorb_mma.cu, FAST mode): DirectGeom with 4 <= K <= 64, N <= 64
bool mma_absorb_supported(const DirectGeom &g);
cudaError_t launch_absorb_mma(const DirectGeom &g, const BatchPtrs &p, cudaStream_t stream);
cudaError_t launch_absorb_tc(const AbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream);
// Gather-fed tcgen05 absorb (absorb_tma.cu, FAST mode): 4 <= K <= 64, 4 <= N <= 64, X bit
// 0 an M bit. The X tile of every stage is gathered straight into the UMMA MN-major
// operand layout (the step's permutation fused into the load): by cp.async 16-byte
// chunks (default), or -- when X bits 0..3 are M bits and the tile bits form <= 5 runs --
// by one TMA box whose dims are [0] X bits 0..3 (+ re/im), the runs of K bits, the runs
// of tile M bits, each extended over the outer bits above it (its TMA coordinate).
struct TmaAbsorbGeom {
  int ndims;
  int dim_a[5], dim_c[5], dim_box[5];  // X positions [a, c) of dim d; the box covers [a, a+box)
  uint64_t outer_x_mask, outer_o_mask;  // outer M bits (tile index) in X and in O
  uint64_t loopk_x_mask;                // K bits iterated by the stages of a tile
  uint64_t tile_x_mask, stagek_x_mask;  // tile M bits, stage K bits (gather loader)
  int tma_ok;                           // the box loader applies (X bits 0..3 in M, <= 5 dims)
  int64_t n_tiles;
  int K, N, kstage, mbl, nm, spt;       // stage K bits, log2 M blocks, N_mma, stages/tile
  int nsr, nsl, lag;                    // ring depths, loads in flight (set at launch)
  int dbg;
  int64_t o_m_off[512];                 // O offset of tile-local m
  int64_t w_k_off[64];                  // W offset of k (k bits in ascending X position)
  int64_t w_n_off[128];                 // [0, 64): W offset of n; [64, 128): O offset of n
};
bool build_tma_absorb(const std::vector<std::pair<int, int>> &kbits,
                      const std::vector<std::pair<int, int>> &mbits,
                      const std::vector<std::pair<int, int>> &nbits, int xr, TmaAbsorbGeom &g);
cudaError_t launch_absorb_tma(const TmaAbsorbGeom &g, const BatchPtrs &p, cudaStream_t stream);
// Tiled bond-2 bit permutation (the absorb tile machinery with K = N = 0).
cudaError_t launch_bitperm(const AbsorbGeom &g, const void *in, void *out, int64_t in_bs,
                           int64_t out_bs, int nbatch, cudaStream_t stream);
// Tiled bond-2 bit permutation (kernels_perm.cu): one CTA per tile of 2^tb complex
// elements whose bits hold the lowest input and the lowest output bits. Tile-local input
// index li (tile bits in ascending input position) and output index lo (ascending output
// position) map to offsets through two 64-entry halves; bases[2t], bases[2t+1] are the
// input / output offsets of tile t (device table, built at plan creation).
struct PermTileGeom {
  int tb;
  int64_t n_tiles;
  int64_t in_off[2][64];     // input offset of li bits [0,6) / [6,12)
  int64_t out_off[2][64];    // output offset of lo bits [0,6) / [6,12)
  uint16_t li_of_lo[2][64];  // li of lo bits [0,6) / [6,12)
};
bool build_perm_tiles(const std::vector<int> &perm, PermTileGeom &g, std::vector<int64_t> &bases);
// out_lo != nullptr: write the TF32 hi (out) / lo (out_lo) planes of the permuted tensor.
cudaError_t launch_perm_tiles(const PermTileGeom &g, const int64_t *bases, const void *in,
                              void *out, int64_t in_bs, int64_t out_bs, int nbatch,
                              cudaStream_t stream, void *out_lo = nullptr);
// Split-K reduction (small output, long K; FAST mode). Pow2 geometries, out_size <= 256.
// The output factorises into A rows (M) x B columns (N); o_mn[o] = m | n << 16.
struct DotTables {
  int M, N;
  const int64_t *a_row;  // [M] A offset of row m
  const int64_t *b_col;  // [N] B offset of column n
  const int32_t *o_mn;   // [out_size]
};
template <class R>
cudaError_t launch_splitk(const StridedGeom &g, const BatchPtrs &p, const DotTables &t,
                          void *workspace, cudaStream_t stream);
size_t splitk_workspace_bytes(const StridedGeom &g, const DotTables &t, int nbatch,
                              size_t esize);
// Skinny GEMM reading A straight from the step operand's own layout (FAST, float):
// gtab = [K] offsets of k, then [mbits] offsets of the M index bits.
bool gemm_skinny_supported(const GemmShape &s);
cudaError_t launch_gemm_skinny_gather(const GemmShape &s, const BatchPtrs &p, const int64_t *gtab,
                                      int mbits, cudaStream_t stream);
template <class R>
cudaError_t launch_gemm_simt(const GemmShape &s, const BatchPtrs &p, bool exact,
                             cudaStream_t stream);
template <class R>
cudaError_t launch_leaf_gather(const LeafGatherTable &t, void *arena, const int32_t *digits,
                               int nbatch, cudaStream_t stream);
template <class R>
cudaError_t launch_root_accumulate(const void *root, int64_t root_bs, int64_t n, int nbatch,
                                   double *acc, double *per_slice, cudaStream_t stream);
cudaError_t launch_sum_ordered(const double *per_slice, uint64_t n_slices, int64_t n,
                               double *out, cudaStream_t stream, bool accumulate = false);

// tcgen05 split-TF32 complex GEMM (gemm_tc.cu). Requires M % 128 == 0,
// N % 128 == 0, K % 32 == 0 (complex elements); returns cudaErrorNotSupported
// otherwise so the caller can pick another kernel.
// gemm_events (optional, 2 events) bracket the GEMM kernel alone (no pre-pass).
// a_presplit: the workspace already holds A's hi / lo planes (a fused permute-split wrote
// them; see gemm_tc_a_planes), so the A pre-pass is skipped.
cudaError_t launch_gemm_tc(const GemmShape &s, const BatchPtrs &p, void *workspace,
                           size_t workspace_bytes, cudaStream_t stream,
                           cudaEvent_t *gemm_events = nullptr, bool a_presplit = false);
// A hi / lo plane pointers inside the workspace (float offsets of the planes).
void gemm_tc_a_planes(const GemmShape &s, const BatchPtrs &p, void *workspace, float **hi,
                      float **lo);
size_t gemm_tc_workspace_bytes(const GemmShape &s, const BatchPtrs &p);
bool gemm_tc_supported(const GemmShape &s);

// tcgen05 split-TF32 complex GEMM with the split fused into shared memory
// (gemm_tcf.cu): A (the [D|M|K] operand, read in place) and the raw B'' plane are
// TMA-loaded as fp32 tiles, lo = x - trunc_tf32(x) is formed in shared memory.
// Requires M % 128 == 0, N % 32 == 0, K % 32 == 0; A batch stride 0 or D*M*K.
// Workspace: the raw B'' plane(s).
bool gemm_tcf_supported(const GemmShape &s);
size_t gemm_tcf_workspace_bytes(const GemmShape &s, const BatchPtrs &p);
// Operand A gathered from the stem layout (no permuted copy): A[m][k] = X[moff_hi[m/128] +
// moff_lo[m%128] + koff[k]] in complex elements, device tables.
struct TcfGather {
  const int64_t *moff_lo, *moff_hi, *koff;
};
cudaError_t launch_gemm_tcf(const GemmShape &s, const BatchPtrs &p, void *workspace,
                            size_t workspace_bytes, cudaStream_t stream,
                            const TcfGather *gather = nullptr);

}  // namespace stn
