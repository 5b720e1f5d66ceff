// Host side of the B200 stem executor: the C ABI of include/stn_exec.h.
//
// What happens where:
//   stn_plan_create   validates the flattened ExecutablePlan, derives the
//                     contraction geometry of every step (the reference's
//                     transpose-GEMM-transpose of runtime.hpp:386-418 becomes a
//                     stride/bit description), picks a kernel per step, builds
//                     three programs (branch-cache build, per-slice with cache,
//                     per-slice without cache) with liveness-planned arenas, and
//                     uploads the leaf tensors.
//   stn_cache_build   runs the branch program once; consumed outputs stay in HBM
//                     (runtime.hpp:456-500).
//   stn_run_*         run the per-slice program for batches of slices: one
//                     leaf-gather launch, one launch per step, one ordered
//                     fp64 accumulation (runtime.hpp:420-453, 601-605).
#include <algorithm>
#include <array>
#include <chrono>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <functional>
#include <map>
#include <mutex>
#include <memory>
#include <numeric>
#include <set>
#include <string>
#include <vector>

#include <cuda_runtime.h>

#include "chain_jit.h"
#include "kernels.h"
#include "stn_exec.h"

namespace {

thread_local std::string g_last_error;

int set_error(int status, const std::string &msg) {
  g_last_error = msg;
  return status;
}

struct Failure {
  int status;
  std::string msg;
};

[[noreturn]] void fail(int status, const std::string &msg) { throw Failure{status, msg}; }
void require(bool cond, int status, const std::string &msg) {
  if (!cond) fail(status, msg);
}
void cuda_check(cudaError_t e, const char *what) {
  if (e != cudaSuccess)
    fail(e == cudaErrorMemoryAllocation ? STN_ERR_OUT_OF_MEMORY : STN_ERR_CUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
}

template <class F>
int guarded(F &&f) {
  try {
    f();
    return STN_OK;
  } catch (const Failure &e) {
    return set_error(e.status, e.msg);
  } catch (const std::bad_alloc &) {
    return set_error(STN_ERR_OUT_OF_MEMORY, "host allocation failed");
  } catch (const std::exception &e) {
    return set_error(STN_ERR_INVALID_ARGUMENT, e.what());
  }
}

// ---------------------------------------------------------------------------
// device buffers
// ---------------------------------------------------------------------------
// Process-wide cache of large device blocks (arenas, workspaces): plans created and
// destroyed back to back (a sampler loop, the bench's end-to-end path) reuse their
// multi-GiB arenas instead of paying cudaMalloc / cudaFree each time. A block goes
// back to the cache only after a device synchronisation (cudaFree's own guarantee).
struct BlockCache {
  struct Block {
    int device;
    size_t bytes;
    void *ptr;
  };
  std::mutex mu;
  std::vector<Block> blocks;
  size_t total = 0;
  // only arena-sized blocks are worth keeping: small tables go straight to cudaFree
  static constexpr size_t kMinBytes = size_t(64) << 20;
  static constexpr size_t kMaxTotal = size_t(48) << 30;
  static BlockCache &get() {
    static BlockCache *c = new BlockCache;  // never destroyed: no cudaFree at exit
    return *c;
  }
  static bool disabled() {
    static const bool off = std::getenv("STN_BLOCK_CACHE") &&
                            std::string(std::getenv("STN_BLOCK_CACHE")) == "0";
    return off;
  }
  void *take(int dev, size_t n) {
    if (disabled() || n < kMinBytes) return nullptr;
    std::lock_guard<std::mutex> lk(mu);
    for (size_t i = 0; i < blocks.size(); ++i)
      if (blocks[i].device == dev && blocks[i].bytes >= n && blocks[i].bytes <= 2 * n) {
        void *p = blocks[i].ptr;
        total -= blocks[i].bytes;
        blocks.erase(blocks.begin() + long(i));
        return p;
      }
    return nullptr;
  }
  // Frees every cached block of `dev` (all devices when dev < 0).
  void flush(int dev = -1) {
    std::lock_guard<std::mutex> lk(mu);
    int cur = 0;
    cudaGetDevice(&cur);
    std::vector<Block> keep;
    for (auto &bl : blocks) {
      if (dev >= 0 && bl.device != dev) {
        keep.push_back(bl);
        continue;
      }
      cudaSetDevice(bl.device);
      cudaFree(bl.ptr);
      total -= bl.bytes;
    }
    blocks.swap(keep);
    cudaSetDevice(cur);
  }
  // The caller has made `dev` current and synchronised it.
  bool give(int dev, void *p, size_t n) {
    if (disabled() || n < kMinBytes) return false;
    std::lock_guard<std::mutex> lk(mu);
    if (total + n > kMaxTotal) return false;
    blocks.push_back({dev, n, p});
    total += n;
    return true;
  }
};

// Makes `dev` current for a scope and restores the previous device.
struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    if (cudaGetDevice(&prev) != cudaSuccess) prev = -1;
    if (prev != dev) cudaSetDevice(dev);
  }
  ~DeviceGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
};

struct DevBuf {
  void *ptr = nullptr;
  size_t bytes = 0;
  int device = 0;  // device the block was allocated on
  DevBuf() = default;
  DevBuf(const DevBuf &) = delete;
  DevBuf &operator=(const DevBuf &) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (ptr) {
      DeviceGuard g(device);
      // cudaFree's own guarantee: no kernel of this device still uses the block
      cudaDeviceSynchronize();
      if (!BlockCache::get().give(device, ptr, bytes)) cudaFree(ptr);
    }
    ptr = nullptr;
    bytes = 0;
  }
  void reserve(size_t n) {
    if (n <= bytes) return;
    release();
    cuda_check(cudaGetDevice(&device), "cudaGetDevice");
    if (void *p = BlockCache::get().take(device, n)) {
      ptr = p;
      bytes = n;  // usable size; the block may be larger (returned with this size)
      return;
    }
    if (cudaMalloc(&ptr, n) != cudaSuccess) {  // out of memory: drop the cached blocks, retry
      cudaGetLastError();
      BlockCache::get().flush(device);
      cuda_check(cudaMalloc(&ptr, n), "cudaMalloc");
    }
    bytes = n;
  }
  template <class T>
  void upload(const std::vector<T> &v) {
    reserve(std::max<size_t>(v.size() * sizeof(T), 16));
    if (!v.empty())
      cuda_check(cudaMemcpy(ptr, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice),
                 "upload");
  }
  template <class T>
  T *as() const {
    return static_cast<T *>(ptr);
  }
};

// ---------------------------------------------------------------------------
// plan model
// ---------------------------------------------------------------------------
enum class Kern { Generic, Absorb, AbsorbTc, AbsorbDirect, AbsorbMma, SplitK, GemmSimt, GemmTc, AbsorbTma, Outer, Lanes };

struct Node {
  bool is_leaf = false;
  int step = -1;  // producing step index
  int leaf = -1;  // leaf index
  std::vector<int> dims;  // canonical dims
  int64_t size = 1;
  bool sliced_leaf = false;
  int consumer = -1;  // step index consuming this node (-1: root or unused)
};

struct StepPlan {
  stn_step_desc d{};
  std::vector<int> lperm, rperm, operm, out_dims;
  Kern kern = Kern::Generic;
  stn::StridedGeom geo{};  // generic
  std::shared_ptr<stn::OuterGeom> og;  // small operands, large output
  // absorb
  stn::AbsorbGeom ag{};
  stn::AbsorbGeom agtc{};  // 128-row tiles for the tensor-core absorb
  bool tc_ok = false;
  stn::DirectGeom dg{};     // tile-free variant (identity low bits)
  bool direct_ok = false;
  std::shared_ptr<stn::TmaAbsorbGeom> tg;  // TMA-fed tensor-core variant (X bits 0..3 in M)
  stn::LaneGeom lg{};                      // lane-mapped SIMT variant (any low-bit interleave)
  std::shared_ptr<DevBuf> lane_tab;        // its stn::LaneTables
  double lane_eff = 0;                     // X sector efficiency of one warp row (all k)
  // absorb bit geometry (positions in X / W / O), kept for stem-sweep fusion
  bool has_bits = false;
  int xr = 0, wr = 0, orank_ = 0;
  std::vector<std::pair<int, int>> kbits, mbits, nbits;  // (x,w), (x,o), (o,w)
  bool x_is_lhs = true;
  // gemm path
  bool a_id = true, b_id = true, c_id = true;
  stn::StridedGeom pa{}, pb{}, pc{};
  bool pa_tiled = false, pb_tiled = false, pc_tiled = false;  // bond-2 tiled permutes
  stn::PermTileGeom pat{}, pbt{}, pct{};                         // high-occupancy tile permutes
  std::shared_ptr<DevBuf> pa_bases, pb_bases, pc_bases;
  std::shared_ptr<DevBuf> skinny_tab;  // gathered skinny GEMM: k offsets, M bit strides
  std::shared_ptr<DevBuf> tcf_gather;  // fused-split GEMM gathering A: m / k offset tables
  int skinny_mbits = 0;
  stn::AbsorbGeom pag{}, pbg{}, pcg{};
  stn::GemmShape gs{};
  bool gemm_swap = false;            // operands exchanged: C^T = B^T A^T
  bool tcf = false;                  // fused-split tcgen05 GEMM (gemm_tcf.cu)
  std::vector<int> gl, gr, go;       // GEMM operand A / B permutations, product -> output
  int64_t lsize = 0, rsize = 0, osize = 0;
  // split-K dot tables (device)
  std::shared_ptr<DevBuf> dot_buf, dot_mn;
  stn::DotTables dot{};
};

enum class Src { ConstLeaf, SliceLeaf, Cache, Arena, Persist };

struct Ref {
  Src kind = Src::Arena;
  int node = -1;
  int64_t off = 0;  // per-slice arena offset (elements) / cache or constant offset
  int64_t size = 0;
};

struct Op {
  int step = -1;
  int sweep = -1;          // >= 0: fused stem sweep over several steps
  std::vector<Ref> wrefs;  // sweep: W operand of every stage
  Ref a, b, out;
  int64_t scr_a = -1, scr_b = -1, scr_c = -1;  // arena scratch offsets (gemm path)
};

struct Program {
  std::vector<Op> ops;
  // intra-slice concurrency: small independent steps (branch-side work that feeds a
  // later stem absorb) run on a second stream of the lane; wait_other[k] = the latest
  // op of the other stream op k must follow (RAW / WAR / WAW on arena regions), -1 none
  std::vector<char> side, need_event;
  std::vector<int> wait_other;
  bool has_side = false;
  int n_steps = 0;  // plan steps covered (a sweep op covers several)
  int64_t arena_elems = 0;  // per slice
  std::vector<int> slice_leaves;           // leaf node ids gathered per slice
  std::map<int, int64_t> slice_leaf_off;   // node -> arena offset
  Ref root;
  bool has_root = false;
  uint64_t mults = 0;
  uint64_t peak = 0;
  // device leaf-gather table
  DevBuf t_src_base, t_elem_leaf, t_dst_off, t_dst_bs, t_elem_local, t_ax_begin, t_ax_stride,
      t_ax_slice;
  stn::LeafGatherTable table{};
};

// One execution lane of a plan: a stream with its own arena, digit buffer,
// workspaces and root staging rows, plus the CUDA graph of a full batch of the
// per-slice program captured on it. Several lanes run batches of slices
// concurrently (run_scheme's `parallelism`, runtime.hpp:564-598); lane 0 runs on
// the caller's stream.
struct ExecCtx {
  cudaStream_t st = nullptr;
  bool own_stream = false;
  DevBuf arena, digits, tc_workspace, splitk_ws, rows;
  cudaEvent_t done = nullptr;  // recorded after this lane's last fold
  // captured graph and what it was captured for
  cudaGraphExec_t graph = nullptr;
  const void *g_prog = nullptr, *g_cache = nullptr, *g_arena = nullptr, *g_rows = nullptr;
  int g_nb = 0;
  uint64_t g_epoch = 0;
  const void *w_prog = nullptr;  // last program run eagerly at full batch (pre-capture warm-up)
  int w_nb = 0;
  uint64_t w_epoch = 0;
  // the side stream of the intra-slice schedule (Program::side) and its events
  cudaStream_t side = nullptr;
  cudaEvent_t fork = nullptr, join = nullptr;
  std::vector<cudaEvent_t> op_ev;
  ~ExecCtx() {
    if (graph) cudaGraphExecDestroy(graph);
    if (done) cudaEventDestroy(done);
    if (fork) cudaEventDestroy(fork);
    if (join) cudaEventDestroy(join);
    for (cudaEvent_t e : op_ev)
      if (e) cudaEventDestroy(e);
    if (side) cudaStreamDestroy(side);
    if (own_stream && st) cudaStreamDestroy(st);
  }
};

}  // namespace

struct stn_cache {
  int device = 0;
  uint64_t identity = 0;
  uint64_t leaf_epoch = 0;
  uint64_t mults = 0;
  uint64_t elements = 0;
  const stn_plan *plan = nullptr;
  DevBuf storage;
};

struct stn_plan {
  int device = 0;
  int mode = STN_MODE_FAST;
  int precision = STN_SINGLE;
  size_t esize = 8;  // bytes per complex element
  uint64_t identity = 0, subtasks = 0;
  int merged_groups = 0, exec_cw = 0;
  int root = -1;
  std::vector<int32_t> sliced_dims;
  std::vector<Node> nodes;
  std::vector<StepPlan> steps;
  std::vector<stn_leaf_desc> leaf_desc;  // arrays below own the data
  std::vector<std::vector<int32_t>> leaf_dims, leaf_sax, leaf_sidx, leaf_perm;
  std::vector<std::vector<double>> leaf_values;
  std::map<int, int> leaf_of_vertex;
  // leaves feeding branch steps (cache staleness tracking)
  std::vector<char> leaf_feeds_branch;
  uint64_t leaf_epoch = 0;
  // constants: canonical unsliced leaves (executor precision)
  std::map<int, int64_t> const_off;  // node -> element offset
  DevBuf consts;
  int64_t consts_elems = 0;
  // sliced leaves: double values, concatenated
  std::map<int, int64_t> sliced_val_off;  // leaf node -> complex offset into sliced_vals
  DevBuf sliced_vals;
  // fused stem sweeps (chains of skinny absorbs)
  struct Sweep {
    std::vector<int> steps;
    stn::SweepGeom geom{};
    std::shared_ptr<DevBuf> tables;
    double io_bytes = 0;  // S_0 + S_r + W's per slice, in elements
    bool chain = false;   // lane-column fused chain (kernels_chain.cu) instead of a tile sweep
    stn::ChainGeom cgeom{};
    std::shared_ptr<stn::ChainTables> host_tables;  // for the NVRTC-specialised kernel
    void *jit_fn = nullptr;                          // its CUfunction (chain_jit.cpp)
    void *jit_alt = nullptr;   // the same kernel capped at 128 registers (two CTAs per SM)
    mutable int jit_pick = 0;  // 0: not yet timed, 1: jit_fn, 2: jit_alt (first-run choice)
  };
  std::vector<Sweep> sweeps;
  std::map<int, int> sweep_of_step;
  std::set<std::vector<int>> chain_banned;  // segments whose specialised kernel spilled
  // programs
  Program build, with_cache, no_cache;
  std::map<int, int64_t> cache_off;  // node -> element offset in cache storage
  int64_t cache_elems = 0;
  // runtime state
  DevBuf scratch_out;
  std::vector<std::unique_ptr<ExecCtx>> lanes;  // lane 0 always exists
  ExecCtx *cur = nullptr;                        // lane the launches go to
  int streams = 1;                               // lanes used by run_slices (stn_plan_set_streams)
  bool graphs = true;                            // capture full batches as CUDA graphs
  uint64_t graph_epoch = 0;                      // bumped when captured graphs become invalid
  int64_t out_elements = 1;
  std::vector<int> out_dims;
  int max_batch = 0;
  int kernel_launches = 0;
  // per-launch profiling (CUDA events on the launch stream)
  bool profiling = false;
  struct Pending {
    int kind;
    int step;
    double bytes, flops;
    cudaEvent_t e0, e1;
  };
  std::map<int, stn_step_profile> step_totals;
  std::vector<Pending> pending;
  std::vector<cudaEvent_t> event_pool;
  stn_kernel_profile totals[STN_KERNEL_KINDS] = {};
  ~stn_plan() {
    for (auto &p : pending) {
      cudaEventDestroy(p.e0);
      cudaEventDestroy(p.e1);
    }
    for (auto e : event_pool) cudaEventDestroy(e);
  }
};

namespace {

// ---------------------------------------------------------------------------
// geometry helpers
// ---------------------------------------------------------------------------
std::vector<int64_t> row_major_strides(const std::vector<int> &dims) {
  std::vector<int64_t> s(dims.size(), 1);
  for (int i = int(dims.size()) - 2; i >= 0; --i) s[i] = s[i + 1] * dims[i + 1];
  return s;
}

struct Axis {
  int64_t dim, sa, sb;
};

// merges adjacent axes whose strides are contiguous in both operands
std::vector<Axis> merge_axes(const std::vector<Axis> &in) {
  std::vector<Axis> out;
  for (const Axis &a : in) {
    if (a.dim == 1) continue;
    if (!out.empty()) {
      Axis &p = out.back();
      if (p.sa == a.sa * a.dim && p.sb == a.sb * a.dim) {
        p.dim *= a.dim;
        p.sa = a.sa;
        p.sb = a.sb;
        continue;
      }
    }
    out.push_back(a);
  }
  return out;
}

void fill_geom(stn::StridedGeom &g, const std::vector<Axis> &out_axes,
               const std::vector<Axis> &k_axes) {
  std::vector<Axis> o = merge_axes(out_axes), k = merge_axes(k_axes);
  require(int(o.size()) <= stn::kMaxAxes && int(k.size()) <= stn::kMaxAxes,
          STN_ERR_INVALID_ARGUMENT, "contraction rank exceeds executor limit");
  memset(&g, 0, sizeof g);
  g.n_out = int(o.size());
  g.n_k = int(k.size());
  g.out_size = 1;
  g.k_size = 1;
  for (int i = 0; i < g.n_out; ++i) {
    g.out_dim[i] = o[i].dim;
    g.out_sa[i] = o[i].sa;
    g.out_sb[i] = o[i].sb;
    g.out_size *= o[i].dim;
  }
  for (int i = 0; i < g.n_k; ++i) {
    g.k_dim[i] = k[i].dim;
    g.k_sa[i] = k[i].sa;
    g.k_sb[i] = k[i].sb;
    g.k_size *= k[i].dim;
  }
}

// permutation as a gather: out axis i = in axis perm[i]
void fill_permute(stn::StridedGeom &g, const std::vector<int> &in_dims,
                  const std::vector<int> &perm) {
  std::vector<int64_t> s = row_major_strides(in_dims);
  std::vector<Axis> ax;
  for (size_t i = 0; i < perm.size(); ++i) ax.push_back({in_dims[perm[i]], s[perm[i]], 0});
  fill_geom(g, ax, {});
}

bool is_identity(const std::vector<int> &p) {
  for (size_t i = 0; i < p.size(); ++i)
    if (p[i] != int(i)) return false;
  return true;
}

// ---------------------------------------------------------------------------
// absorb geometry (bond-2, D == 1): see kernels.h AbsorbGeom
// ---------------------------------------------------------------------------
// Tile geometry shared by the absorb and bit-permute kernels (kernels.h AbsorbGeom).
// kbits: (x pos, w pos) ascending; mbits: (x pos, o pos); nbits: (o pos, w pos) ascending.
bool make_tile_geom(const std::vector<std::pair<int, int>> &kbits,
                    const std::vector<std::pair<int, int>> &mbits,
                    const std::vector<std::pair<int, int>> &nbits, int x_bits, int o_bits,
                    stn::AbsorbGeom &g, int force_tb = 0) {
  const int kb = int(kbits.size()), nb = int(nbits.size()), mb = int(mbits.size());
  // choose tile M bits T: low X bits, low O bits, then ascending X position
  const int Lx = std::min(5, x_bits), Lo = std::min(5, o_bits);
  std::vector<char> in_t(mbits.size(), 0);
  int tb = 0;
  for (size_t j = 0; j < mbits.size(); ++j)
    if (mbits[j].first < Lx || mbits[j].second < Lo) {
      in_t[j] = 1;
      tb++;
    }
  const int target = 11;
  if (force_tb > 0 && tb > force_tb) return false;
  {
    std::vector<size_t> order(mbits.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(),
              [&](size_t a, size_t b) { return mbits[a].first < mbits[b].first; });
    for (size_t j : order) {
      if (in_t[j]) continue;
      if (force_tb > 0 ? tb >= force_tb : (kb + tb >= target || nb + tb >= target)) break;
      in_t[j] = 1;
      tb++;
    }
  }
  if (force_tb > 0 && tb != force_tb) return false;
  if (kb + tb > 13 || nb + tb > 13) return false;  // <= 64 KiB per tile
  if (kb + tb < 2 || nb + tb < 2) return false;
  const int ob = mb - tb;
  if (ob > 31) return false;

  memset(&g, 0, sizeof g);
  g.x_bits = x_bits;
  g.o_bits = o_bits;
  g.kb = kb;
  g.nb = nb;
  g.tb = tb;
  g.ob = ob;
  g.xt_bits = kb + tb;
  g.ot_bits = nb + tb;
  for (int j = 0; j < kb; ++j) g.w_k_stride[j] = int64_t(1) << kbits[j].second;
  for (int j = 0; j < nb; ++j) g.w_n_stride[j] = int64_t(1) << nbits[j].second;
  // tile-local X bits: K bits and T bits by ascending X position
  std::vector<std::pair<int, int>> xt;  // (xpos, tag) tag: -1-k for K bit k, j for M bit j
  for (int j = 0; j < kb; ++j) xt.push_back({kbits[j].first, -1 - j});
  for (size_t j = 0; j < mbits.size(); ++j)
    if (in_t[j]) xt.push_back({mbits[j].first, int(j)});
  std::sort(xt.begin(), xt.end());
  std::vector<std::pair<int, int>> otl;  // (opos, tag) tag: -1-n for N bit n, j for M bit j
  for (int j = 0; j < nb; ++j) otl.push_back({nbits[j].first, -1 - j});
  for (size_t j = 0; j < mbits.size(); ++j)
    if (in_t[j]) otl.push_back({mbits[j].second, int(j)});
  std::sort(otl.begin(), otl.end());
  std::map<int, int> xl_of_m, ol_of_m;
  for (int i = 0; i < int(xt.size()); ++i) {
    g.x_tile_pos[i] = uint8_t(xt[i].first);
    if (xt[i].second < 0)
      g.k_xl[-1 - xt[i].second] = uint8_t(i);
    else
      xl_of_m[xt[i].second] = i;
  }
  for (int i = 0; i < int(otl.size()); ++i) {
    g.o_tile_pos[i] = uint8_t(otl[i].first);
    if (otl[i].second < 0)
      g.n_ol[-1 - otl[i].second] = uint8_t(i);
    else
      ol_of_m[otl[i].second] = i;
  }
  // T bits in ascending X position
  int tj = 0, oj = 0;
  {
    std::vector<size_t> order(mbits.size());
    std::iota(order.begin(), order.end(), 0);
    std::sort(order.begin(), order.end(),
              [&](size_t a, size_t b) { return mbits[a].first < mbits[b].first; });
    for (size_t j : order) {
      if (in_t[j]) {
        g.t_xl[tj] = uint8_t(xl_of_m[int(j)]);
        g.t_ol[tj] = uint8_t(ol_of_m[int(j)]);
        tj++;
      } else {
        g.outer_x[oj] = uint8_t(mbits[j].first);
        g.outer_o[oj] = uint8_t(mbits[j].second);
        oj++;
      }
    }
  }
  g.x_run = 0;
  while (g.x_run < g.xt_bits && g.x_tile_pos[g.x_run] == g.x_run) g.x_run++;
  g.o_run = 0;
  while (g.o_run < g.ot_bits && g.o_tile_pos[g.o_run] == g.o_run) g.o_run++;
  if (g.x_run < 1 || g.o_run < 1) return false;
  return true;
}

// Lane-mapped absorb tables (kernels.h LaneGeom / LaneTables). kbits: (x, w) by
// ascending X position (k bit j = kbits[j], the reference's k order);
// mbits: (x, o); nbits: (o, w).
void build_lanes(StepPlan &sp, const std::vector<std::pair<int, int>> &kbits,
                 const std::vector<std::pair<int, int>> &mbits,
                 const std::vector<std::pair<int, int>> &nbits, int xr, int wr, int orank) {
  const int kb = int(kbits.size());
  if (kb > 6 || wr > 13) return;  // K <= 64, W <= 8192 complex in shared memory
  std::vector<int64_t> xs(size_t(orank), 0);
  std::vector<int32_t> ws(size_t(orank), 0);
  for (auto &[xp, op] : mbits) xs[size_t(op)] = int64_t(1) << xp;
  for (auto &[op, wp] : nbits) ws[size_t(op)] = int32_t(1) << wp;
  int mode = 0;
  if (xs[0] == 1) mode = 1;       // O bit 0 = X bit 0: m pairs
  else if (ws[0] != 0) mode = 2;  // O bit 0 = an N bit: n pairs
  const int U = mode ? 1 : 0;
  const int row_bits = orank - U - 5;
  if (row_bits < 0 || row_bits > 32) return;
  auto T = std::make_unique<stn::LaneTables>();
  memset(T.get(), 0, sizeof(stn::LaneTables));
  for (int l = 0; l < 32; ++l)
    for (int j = 0; j < 5; ++j)
      if ((l >> j) & 1) {
        T->xl[l] += xs[size_t(U + j)];
        T->wl[l] += ws[size_t(U + j)];
      }
  for (int c = 0; c < 4; ++c)
    for (int v = 0; v < 256; ++v)
      for (int j = 0; j < 8; ++j)
        if (((v >> j) & 1) && 8 * c + j < row_bits) {
          T->xr[c][v] += xs[size_t(U + 5 + 8 * c + j)];
          T->wr[c][v] += ws[size_t(U + 5 + 8 * c + j)];
        }
  const int K = 1 << kb;
  for (int k = 0; k < K; ++k)
    for (int j = 0; j < kb; ++j)
      if ((k >> j) & 1) {
        T->xk[k] += int64_t(1) << kbits[size_t(j)].first;
        T->wk[k] += int32_t(1) << kbits[size_t(j)].second;
      }
  // X sector efficiency of one warp row over all k (L1 / L2 serve the re-reads)
  std::set<int64_t> elems, sectors;
  for (int l = 0; l < 32; ++l)
    for (int k = 0; k < K; ++k)
      for (int u = 0; u < (mode == 1 ? 2 : 1); ++u) {
        const int64_t e = T->xl[l] + T->xk[k] + u;
        elems.insert(e);
        sectors.insert(e / 4);
      }
  sp.lane_eff = double(elems.size()) / (4.0 * double(sectors.size()));
  sp.lg.mode = mode;
  sp.lg.K = K;
  sp.lg.rows = int64_t(1) << row_bits;
  sp.lg.w_pair = mode == 2 ? ws[0] : 0;
  sp.lg.w_elems = int32_t(1) << wr;
  sp.lane_tab = std::make_shared<DevBuf>();
  sp.lane_tab->reserve(sizeof(stn::LaneTables));
  cuda_check(cudaMemcpy(sp.lane_tab->ptr, T.get(), sizeof(stn::LaneTables), cudaMemcpyHostToDevice),
             "lane tables");
}

bool build_absorb(StepPlan &sp, const std::vector<int> &ldims, const std::vector<int> &rdims) {
  const stn_step_desc &d = sp.d;
  if (d.nd != 0) return false;
  for (int x : ldims)
    if (x != 2) return false;
  for (int x : rdims)
    if (x != 2) return false;
  const int lr = int(ldims.size()), rr = int(rdims.size()), orank = int(sp.out_dims.size());
  const bool x_lhs = sp.lsize >= sp.rsize;
  const int xr = x_lhs ? lr : rr, wr = x_lhs ? rr : lr;
  const int kb = d.nk;
  const int nb = wr - kb;  // W-side free bits
  const int mb = xr - kb;
  if (kb > stn::kAbsorbMaxKN || nb > 12 || xr < 12) return false;
  // K bits: (x position, w position)
  std::vector<std::pair<int, int>> kbits;
  for (int q = 0; q < d.nk; ++q) {
    int la = sp.lperm[d.nd + d.nm + q], rb = sp.rperm[d.nd + q];
    int xa = x_lhs ? la : rb, wa = x_lhs ? rb : la;
    kbits.push_back({xr - 1 - xa, wr - 1 - wa});
  }
  std::sort(kbits.begin(), kbits.end());
  // output bits: M pairs (x pos, o pos) from X, N pairs (w pos, o pos) from W
  std::vector<std::pair<int, int>> mbits, nbits;  // (xpos, opos), (opos, wpos)
  for (int i = 0; i < orank; ++i) {
    int p = sp.operm[i];
    int opos = orank - 1 - i;
    bool from_lhs = p < d.nd + d.nm;
    if (from_lhs) {
      int la = sp.lperm[p];
      if (x_lhs)
        mbits.push_back({lr - 1 - la, opos});
      else
        nbits.push_back({opos, lr - 1 - la});
    } else {
      int q = p - d.nd - d.nm;
      int rb = sp.rperm[d.nd + d.nk + q];
      if (x_lhs)
        nbits.push_back({opos, rr - 1 - rb});
      else
        mbits.push_back({rr - 1 - rb, opos});
    }
  }
  std::sort(nbits.begin(), nbits.end());
  if (int(mbits.size()) != mb || int(nbits.size()) != nb) return false;
  // W positions of K and N bits must be ascending with their X/O order
  for (size_t j = 1; j < kbits.size(); ++j)
    if (kbits[j].second < kbits[j - 1].second) return false;
  for (size_t j = 1; j < nbits.size(); ++j)
    if (nbits[j].second < nbits[j - 1].second) return false;

  sp.x_is_lhs = x_lhs;
  sp.has_bits = true;
  {
    auto tg = std::make_shared<stn::TmaAbsorbGeom>();
    if (stn::build_tma_absorb(kbits, mbits, nbits, xr, *tg)) sp.tg = tg;
  }
  sp.xr = xr;
  sp.wr = wr;
  sp.orank_ = orank;
  sp.kbits = kbits;
  sp.mbits = mbits;
  sp.nbits = nbits;
  build_lanes(sp, kbits, mbits, nbits, xr, wr, orank);
  // tile-free geometry: the lowest L bits of X are M bits at the same O positions
  {
    std::map<int, int> o_of_x;
    for (auto &[xp, op] : mbits) o_of_x[xp] = op;
    int L = 0;
    while (o_of_x.count(L) && o_of_x[L] == L) ++L;
    stn::DirectGeom &dg = sp.dg;
    memset(&dg, 0, sizeof dg);
    dg.L = L;
    dg.kb = kb;
    dg.nb = nb;
    dg.mh_bits = mb - L;
    for (auto &[xp, op] : mbits)
      if (xp >= L) {
        dg.hi_x_mask |= uint64_t(1) << xp;
        dg.hi_o_mask |= uint64_t(1) << op;
      }
    if (kb <= 6 && nb <= 12) {
      for (int j = 0; j < kb; ++j) {
        dg.k_xpos[j] = uint8_t(kbits[j].first);
        dg.w_k_stride[j] = int64_t(1) << kbits[j].second;
      }
      for (int j = 0; j < nb; ++j) {
        dg.n_opos[j] = uint8_t(nbits[j].first);
        dg.w_n_stride[j] = int64_t(1) << nbits[j].second;
      }
    }
    sp.direct_ok = L >= 2 && stn::direct_absorb_launchable(dg) && dg.mh_bits <= 40;
  }
  if (nb > stn::kAbsorbMaxKN) return sp.direct_ok;  // tiled kernels: N <= 64
  stn::AbsorbGeom g;
  if (!make_tile_geom(kbits, mbits, nbits, xr, orank, g)) return sp.direct_ok;
  g.w_is_lhs = x_lhs ? 0 : 1;
  sp.ag = g;
  sp.x_is_lhs = x_lhs;
  // tensor-core variant: exactly 128 tile rows
  sp.tc_ok = make_tile_geom(kbits, mbits, nbits, xr, orank, sp.agtc, 7) &&
             stn::tc_absorb_supported(sp.agtc);
  return true;
}

// Bond-2 permutation (out axis i = in axis perm[i]) as a tiled bit permutation.
bool build_bitperm(const std::vector<int> &in_dims, const std::vector<int> &perm,
                   stn::AbsorbGeom &g) {
  const int r = int(in_dims.size());
  if (r < 12) return false;
  for (int x : in_dims)
    if (x != 2) return false;
  std::vector<std::pair<int, int>> mbits;
  for (int i = 0; i < r; ++i) mbits.push_back({r - 1 - perm[i], r - 1 - i});
  return make_tile_geom({}, mbits, {}, r, r, g);
}


// ---------------------------------------------------------------------------
// plan construction
// ---------------------------------------------------------------------------
void choose_kernel(stn_plan &P, StepPlan &sp, const std::vector<int> &ldims,
                   const std::vector<int> &rdims) {
  const stn_step_desc &d = sp.d;
  const bool single = P.precision == STN_SINGLE;
  const bool exact = P.mode == STN_MODE_EXACT;
  // generic geometry (always built: also the fallback)
  {
    std::vector<int64_t> ls = row_major_strides(ldims), rs = row_major_strides(rdims);
    std::vector<Axis> out_axes, k_axes;
    for (int i = 0; i < d.orank; ++i) {
      int p = sp.operm[i];
      if (p < d.nd) {
        out_axes.push_back({sp.out_dims[i], ls[sp.lperm[p]], rs[sp.rperm[p]]});
      } else if (p < d.nd + d.nm) {
        out_axes.push_back({sp.out_dims[i], ls[sp.lperm[p]], 0});
      } else {
        int q = p - d.nd - d.nm;
        out_axes.push_back({sp.out_dims[i], 0, rs[sp.rperm[d.nd + d.nk + q]]});
      }
    }
    for (int q = 0; q < d.nk; ++q) {
      int la = sp.lperm[d.nd + d.nm + q], rb = sp.rperm[d.nd + q];
      k_axes.push_back({ldims[la], ls[la], rs[rb]});
    }
    fill_geom(sp.geo, out_axes, k_axes);
  }
  sp.kern = Kern::Generic;
  // small operands, large output: table-driven outer kernel (bitwise k_generic)
  if (sp.lsize <= (int64_t(1) << 16) && sp.rsize <= (int64_t(1) << 16) &&
      sp.osize >= (int64_t(1) << 20) && sp.osize <= (int64_t(1) << 31) &&
      sp.geo.k_size <= 64) {
    bool pow2 = true;
    for (int i = 0; i < sp.geo.n_out; ++i) pow2 &= (sp.geo.out_dim[i] & (sp.geo.out_dim[i] - 1)) == 0;
    for (int i = 0; i < sp.geo.n_k; ++i) pow2 &= (sp.geo.k_dim[i] & (sp.geo.k_dim[i] - 1)) == 0;
    if (pow2) {
      auto og = std::make_shared<stn::OuterGeom>();
      memset(og.get(), 0, sizeof(stn::OuterGeom));
      std::vector<int64_t> abit, bbit;  // per output bit (LSB first)
      for (int i = sp.geo.n_out - 1; i >= 0; --i)
        for (int64_t v = 1; v < sp.geo.out_dim[i]; v <<= 1) {
          abit.push_back(v * sp.geo.out_sa[i]);
          bbit.push_back(v * sp.geo.out_sb[i]);
        }
      og->obits = int(abit.size());
      for (int c = 0; c < 4; ++c)
        for (int v = 0; v < 256; ++v) {
          int64_t a = 0, b = 0;
          for (int j = 0; j < 8; ++j)
            if (((v >> j) & 1) && 8 * c + j < og->obits) {
              a += abit[8 * c + j];
              b += bbit[8 * c + j];
            }
          og->ta[c][v] = int32_t(a);
          og->tb[c][v] = int32_t(b);
        }
      og->nk = int(sp.geo.k_size);
      for (int64_t k = 0; k < sp.geo.k_size; ++k) {  // row-major over the K axes
        int64_t rem = k, a = 0, b = 0;
        for (int i = sp.geo.n_k - 1; i >= 0; --i) {
          const int64_t idx = rem % sp.geo.k_dim[i];
          rem /= sp.geo.k_dim[i];
          a += idx * sp.geo.k_sa[i];
          b += idx * sp.geo.k_sb[i];
        }
        og->ka[k] = int32_t(a);
        og->kb[k] = int32_t(b);
      }
      if (og->obits >= 3) {
        sp.og = og;
        sp.kern = Kern::Outer;
        return;
      }
    }
  }
  const int64_t small = std::min(sp.lsize, sp.rsize);
  const int64_t big = std::max(sp.lsize, sp.rsize);
  // bandwidth-bound absorb: one big operand, a small K x N side
  if (single && big >= (int64_t(1) << 12) && small <= 4096 && build_absorb(sp, ldims, rdims)) {
    sp.kern = Kern::Absorb;
    // tile-free streaming when the low bits line up (K x N <= 2^STN_DIRECT_MAX_BITS)
    static const char *dmax = stn::debug_opt("direct_max_bits");
    const int direct_max = dmax ? std::atoi(dmax) : 12;
    static const char *dminl = stn::debug_opt("direct_min_l");
    const int direct_min_L = dminl ? std::atoi(dminl) : 2;
    // FAST mode, K x N >= 2^STN_MMA_MIN_BITS: tensor-core direct absorb
    const char *mmin = stn::debug_opt("mma_min_bits");
    const int mma_min = mmin ? std::atoi(mmin) : 10;
    // FAST mode: the gather/TMA-fed tensor-core absorb where the SIMT streams are weak --
    // no or short identity run of low bits (L <= 2, measured on B200: the tensor-core
    // kernel streams at 3-4 TB/s, the SIMT kernels at 1.3-3 TB/s there) and 64 x 64
    // W's -- while long identity runs stay on the SIMT direct kernel (6+ TB/s).
    // STN_TMA_MIN_BITS=<bits> (experiments) forces it for every K x N >= 2^bits.
    const char *tmin = stn::debug_opt("tma_min_bits");
    // lane-mapped SIMT absorb (any interleave of the low output bits): where neither
    // the direct stream (identity run of >= 3 low bits) nor the TMA-fed tensor-core
    // absorb takes the step, it replaces the tiled SIMT absorb (measured on B200:
    // cfg5 step 1606, 2^32 x 2 x 2: 28.6 -> 12.4 ms; step 693: 9.1 -> 1.9 ms), and it
    // also takes the TMA steps with K x N <= 16 (cfg5 steps 1624 / 1628: 3.6 -> 2.7 ms;
    // larger K x N stay on the tensor cores, e.g. cfg4 step 1040: 2.4 vs 4.9 ms).
    // STN_DEBUG lanes=0 disables it, lanes=all takes every eligible step.
    const char *lp = stn::debug_opt("lanes");
    const int lanes_policy = lp ? (std::string(lp) == "all" ? 2 : std::atoi(lp) != 0) : 1;
    const bool lanes_ok = sp.lane_tab && sp.lane_eff >= 0.5 && big >= (int64_t(1) << 16) &&
                          lanes_policy > 0;
    const int kn_bits = int(sp.kbits.size() + sp.nbits.size());
    if (lanes_ok && (lanes_policy == 2 || (kn_bits <= 4 && !(sp.direct_ok && sp.dg.L >= 3)))) {
      sp.kern = Kern::Lanes;
      return;
    }
    if (!exact && sp.tg) {
      const int kn = int(sp.kbits.size() + sp.nbits.size());
      const bool pick = tmin ? kn >= std::atoi(tmin)
                             : (big >= (int64_t(1) << 22) &&
                                (!sp.direct_ok || sp.dg.L <= 2 || kn >= 12));
      if (pick) {
        sp.kern = Kern::AbsorbTma;
        return;
      }
    }
    if (!exact && sp.direct_ok && stn::mma_absorb_supported(sp.dg) &&
        sp.dg.kb + sp.dg.nb >= mma_min) {
      sp.kern = Kern::AbsorbMma;
      return;
    }
    if (sp.direct_ok && sp.dg.L >= direct_min_L && sp.dg.kb + sp.dg.nb <= direct_max) {
      sp.kern = Kern::AbsorbDirect;
      return;
    }
    if (lanes_ok && !(sp.direct_ok && sp.dg.L >= 3)) {  // instead of the tiled SIMT absorb
      sp.kern = Kern::Lanes;
      return;
    }
    if (!sp.tc_ok && sp.ag.xt_bits == 0) {  // no tile geometry: direct or generic
      sp.kern = sp.direct_ok ? Kern::AbsorbDirect : Kern::Generic;
      return;
    }
    // large K x N: SIMT math would bound the stream; use the tensor cores.
    // STN_ABSORB_POLICY (experiments only): "simt" never, "tc" from K*N >= 64.
    static const char *policy = stn::debug_opt("absorb_policy");
    int tc_min_bits = 10;
    if (policy && std::string(policy) == "simt") tc_min_bits = 99;
    if (policy && std::string(policy) == "tc") tc_min_bits = 6;
    if (!exact && sp.tc_ok && sp.ag.kb + sp.ag.nb >= tc_min_bits) sp.kern = Kern::AbsorbTc;
    return;
  }
  // long-K reduction to a small output (FAST mode: chunked K order)
  if (!exact && sp.geo.out_size <= 256 && sp.geo.k_size >= (int64_t(1) << 14)) {
    bool pow2 = true;
    for (int i = 0; i < sp.geo.n_out; ++i) pow2 &= (sp.geo.out_dim[i] & (sp.geo.out_dim[i] - 1)) == 0;
    for (int i = 0; i < sp.geo.n_k; ++i) pow2 &= (sp.geo.k_dim[i] & (sp.geo.k_dim[i] - 1)) == 0;
    // factorise the output into A rows x B columns (no D axes)
    bool factor = pow2;
    std::vector<int> m_ax, n_ax;
    for (int i = 0; i < sp.geo.n_out && factor; ++i) {
      if (sp.geo.out_sa[i] != 0 && sp.geo.out_sb[i] != 0) factor = false;
      else if (sp.geo.out_sb[i] == 0) m_ax.push_back(i);
      else n_ax.push_back(i);
    }
    if (factor) {
      auto enumerate = [&](const std::vector<int> &ax, bool use_a) {
        std::vector<int64_t> offs{0};
        for (int i : ax) {  // outermost first -> row-major enumeration
          std::vector<int64_t> nx;
          for (int64_t base : offs)
            for (int64_t v = 0; v < sp.geo.out_dim[i]; ++v)
              nx.push_back(base + v * (use_a ? sp.geo.out_sa[i] : sp.geo.out_sb[i]));
          offs.swap(nx);
        }
        return offs;
      };
      std::vector<int64_t> a_row = enumerate(m_ax, true), b_col = enumerate(n_ax, false);
      // output o -> (m, n): decompose o over the out axes
      std::vector<int32_t> o_mn(size_t(sp.geo.out_size));
      for (int64_t o = 0; o < sp.geo.out_size; ++o) {
        int64_t rem = o, m = 0, n = 0, mstride = 1, nstride = 1;
        for (int i = sp.geo.n_out - 1; i >= 0; --i) {
          const int64_t idx = rem % sp.geo.out_dim[i];
          rem /= sp.geo.out_dim[i];
          if (sp.geo.out_sb[i] == 0) {
            m += idx * mstride;
            mstride *= sp.geo.out_dim[i];
          } else {
            n += idx * nstride;
            nstride *= sp.geo.out_dim[i];
          }
        }
        o_mn[size_t(o)] = int32_t(m | (n << 16));
      }
      std::vector<int64_t> packed(a_row);
      packed.insert(packed.end(), b_col.begin(), b_col.end());
      sp.dot_buf = std::make_shared<DevBuf>();
      sp.dot_buf->upload(packed);
      auto mn_buf = std::make_shared<DevBuf>();
      mn_buf->upload(o_mn);
      sp.dot.M = int(a_row.size());
      sp.dot.N = int(b_col.size());
      sp.dot.a_row = sp.dot_buf->as<int64_t>();
      sp.dot.b_col = sp.dot_buf->as<int64_t>() + a_row.size();
      sp.dot.o_mn = mn_buf->as<int32_t>();
      sp.dot_mn = mn_buf;
      sp.kern = Kern::SplitK;
      return;
    }
  }
  // dense GEMM path: materialise [D|M|K], [D|K|N], run GEMM, permute [D|M|N]
  if (d.M >= 8 && d.N >= 8 && d.K >= 8 && d.mults >= (uint64_t(1) << 18)) {
    sp.gs = {d.D, d.M, d.N, d.K};
    // fused-split kernel (gemm_tcf.cu) unless STN_DEBUG tcf=0; else the pre-split one
    // Measured on B200 (profiles/r02_gemm_tcf.txt): the fused-split kernel wins where
    // the GEMM is operand-bandwidth bound (2N <= 128: cfg5's 32 x 32768 x 8192 step
    // 7.6 -> 2.6 ms on tensor cores at all), the pre-split 128 x 256 kernel on the
    // compute-bound wide GEMMs (212 vs 95 TFLOP/s at 4096 x 1024 x 1024).
    const char *tcf_opt = stn::debug_opt("tcf");
    const int tcf_mode = tcf_opt ? std::atoi(tcf_opt) : 1;  // 0 never, 1 narrow, 2 always
    auto use_tcf = [&](const stn::GemmShape &g) {
      if (tcf_mode == 0 || !stn::gemm_tcf_supported(g)) return false;
      return tcf_mode == 2 || 2 * g.N <= 128 || !stn::gemm_tc_supported(g);
    };
    auto tc_ok = [&](const stn::GemmShape &g) {
      return stn::gemm_tc_supported(g) || use_tcf(g);
    };
    const bool tc_fwd = single && !exact && tc_ok(sp.gs);
    // tcgen05 GEMM: the operand it expands (B -> 2N x 2K real) should be the small one;
    // with a larger rhs compute C^T = B^T A^T ([D|N|K] x [D|K|M] -> [D|N|M])
    sp.gemm_swap = false;
    const stn::GemmShape t{d.D, d.N, d.M, d.K};
    const bool tc_swp = single && !exact && tc_ok(t);
    if (tc_swp && (sp.rsize > sp.lsize || !tc_fwd)) {
      sp.gemm_swap = true;
      sp.gs = t;
    }
    const bool tc = sp.gemm_swap || tc_fwd;
    sp.kern = tc ? Kern::GemmTc : Kern::GemmSimt;
    sp.tcf = tc && use_tcf(sp.gs);
    const int nd = d.nd, nm = d.nm, nk = d.nk, nn = d.nn;
    if (!sp.gemm_swap) {
      sp.gl = sp.lperm;
      sp.gr = sp.rperm;
      sp.go = sp.operm;
    } else {
      sp.gl.assign(sp.rperm.begin(), sp.rperm.begin() + nd);  // A' = rhs as [D|N|K]
      sp.gl.insert(sp.gl.end(), sp.rperm.begin() + nd + nk, sp.rperm.end());
      sp.gl.insert(sp.gl.end(), sp.rperm.begin() + nd, sp.rperm.begin() + nd + nk);
      sp.gr.assign(sp.lperm.begin(), sp.lperm.begin() + nd);  // B' = lhs as [D|K|M]
      sp.gr.insert(sp.gr.end(), sp.lperm.begin() + nd + nm, sp.lperm.end());
      sp.gr.insert(sp.gr.end(), sp.lperm.begin() + nd, sp.lperm.begin() + nd + nm);
      sp.go.resize(sp.operm.size());  // product axes [D|M|N] -> [D|N|M]
      for (size_t i = 0; i < sp.operm.size(); ++i) {
        const int p = sp.operm[i];
        sp.go[i] = p < nd ? p : (p < nd + nm ? p + nn : p - nm);
      }
    }
    const std::vector<int> &adims = sp.gemm_swap ? rdims : ldims;
    const std::vector<int> &bdims = sp.gemm_swap ? ldims : rdims;
    std::vector<int> prod_dims(d.orank);
    for (int i = 0; i < d.orank; ++i) prod_dims[sp.go[i]] = sp.out_dims[i];
    sp.a_id = is_identity(sp.gl);
    sp.b_id = is_identity(sp.gr);
    sp.c_id = is_identity(sp.go);
    fill_permute(sp.pa, adims, sp.gl);
    fill_permute(sp.pb, bdims, sp.gr);
    fill_permute(sp.pc, prod_dims, sp.go);
    if (single) {
      sp.pa_tiled = !sp.a_id && build_bitperm(adims, sp.gl, sp.pag);
      sp.pb_tiled = !sp.b_id && build_bitperm(bdims, sp.gr, sp.pbg);
      sp.pc_tiled = !sp.c_id && build_bitperm(prod_dims, sp.go, sp.pcg);
      auto tiles = [&](bool id, const std::vector<int> &dims, const std::vector<int> &perm,
                       stn::PermTileGeom &g, std::shared_ptr<DevBuf> &buf) {
        if (id) return;
        for (int x : dims)
          if (x != 2) return;
        std::vector<int64_t> bases;
        if (!stn::build_perm_tiles(perm, g, bases)) return;
        buf = std::make_shared<DevBuf>();
        buf->upload(bases);
      };
      tiles(sp.a_id, adims, sp.gl, sp.pat, sp.pa_bases);
      tiles(sp.b_id, bdims, sp.gr, sp.pbt, sp.pb_bases);
      tiles(sp.c_id, prod_dims, sp.go, sp.pct, sp.pc_bases);
      // FAST skinny GEMM (N <= 8): read A through offset tables instead of permuting it
      bool all2 = true;
      for (int x : adims) all2 &= x == 2;
      const int nmb = __builtin_ctzll(uint64_t(sp.gs.M)), nkb = __builtin_ctzll(uint64_t(sp.gs.K));
      if (!exact && sp.kern == Kern::GemmSimt && !sp.gemm_swap && !sp.a_id && all2 &&
          stn::gemm_skinny_supported(sp.gs) && int(adims.size()) == nmb + nkb &&
          (int64_t(1) << nmb) == sp.gs.M && (int64_t(1) << nkb) == sp.gs.K) {
        const int r = int(adims.size());
        std::vector<int64_t> tab(size_t(sp.gs.K + nmb));
        for (int64_t k = 0; k < sp.gs.K; ++k) {
          int64_t off = 0;
          for (int j = 0; j < nkb; ++j)
            if ((k >> j) & 1) off += int64_t(1) << (r - 1 - sp.gl[r - 1 - j]);
          tab[size_t(k)] = off;
        }
        for (int j = 0; j < nmb; ++j)
          tab[size_t(sp.gs.K + j)] = int64_t(1) << (r - 1 - sp.gl[r - 1 - nkb - j]);
        if (tab[1] == 1) {  // k pairs contiguous: 16-byte loads
          sp.skinny_tab = std::make_shared<DevBuf>();
          sp.skinny_tab->upload(tab);
          sp.skinny_mbits = nmb;
        }
      }
      // fused-split tcgen05 GEMM with a permuted A: gather A from the stem layout inside
      // the GEMM (offset tables) instead of materialising the permuted operand
      const char *tg = stn::debug_opt("tcf_gather");  // STN_DEBUG tcf_gather=0: permute
      if (sp.kern == Kern::GemmTc && sp.tcf && !sp.a_id && all2 && sp.gs.D == 1 &&
          !(tg && std::atoi(tg) == 0) && int(adims.size()) == nmb + nkb &&
          (int64_t(1) << nmb) == sp.gs.M && (int64_t(1) << nkb) == sp.gs.K && sp.gs.M >= 128) {
        const int r = int(adims.size());
        auto mbit = [&](int j) { return int64_t(1) << (r - 1 - sp.gl[size_t(r - 1 - nkb - j)]); };
        auto moff = [&](int64_t m) {
          int64_t off = 0;
          for (int j = 0; j < nmb; ++j)
            if ((m >> j) & 1) off += mbit(j);
          return off;
        };
        std::vector<int64_t> tab;  // [128 moff_lo | M/128 moff_hi | K koff]
        for (int64_t m = 0; m < 128; ++m) tab.push_back(moff(m));
        for (int64_t t = 0; t < sp.gs.M / 128; ++t) tab.push_back(moff(t * 128));
        for (int64_t k = 0; k < sp.gs.K; ++k) {
          int64_t off = 0;
          for (int j = 0; j < nkb; ++j)
            if ((k >> j) & 1) off += int64_t(1) << (r - 1 - sp.gl[size_t(r - 1 - j)]);
          tab.push_back(off);
        }
        sp.tcf_gather = std::make_shared<DevBuf>();
        sp.tcf_gather->upload(tab);
      }
    }
  }
}

// Diagnostics (STN_PLAN_DUMP): one line per large step with its kernel and bit geometry.
void dump_step(const StepPlan &sp, int i) {
  static const char *names[] = {"generic", "absorb", "absorb_tc", "direct", "mma", "splitk",
                                "gemm_simt", "gemm_tc", "tma", "outer", "lanes"};
  auto lg = [](int64_t v) { int b = 0; while ((int64_t(1) << b) < v) ++b; return b; };
  std::string s = "step " + std::to_string(i) + " " + names[int(sp.kern)] + " l2^" +
                  std::to_string(lg(sp.lsize)) + " r2^" + std::to_string(lg(sp.rsize)) + " o2^" +
                  std::to_string(lg(sp.osize)) + " D" + std::to_string(sp.d.D) + " M" +
                  std::to_string(sp.d.M) + " N" + std::to_string(sp.d.N) + " K" +
                  std::to_string(sp.d.K);
  if (sp.has_bits) {
    s += " x_lhs=" + std::to_string(sp.x_is_lhs) + " L=" + std::to_string(sp.dg.L) + " k(x,w):";
    for (auto &p : sp.kbits) s += " " + std::to_string(p.first) + "," + std::to_string(p.second);
    s += " n(o,w):";
    for (auto &p : sp.nbits) s += " " + std::to_string(p.first) + "," + std::to_string(p.second);
    s += " m(x,o)<16:";
    for (auto &p : sp.mbits)
      if (p.first < 16 || p.second < 16)
        s += " " + std::to_string(p.first) + "," + std::to_string(p.second);
  }
  if (sp.kern == Kern::GemmTc || sp.kern == Kern::GemmSimt) {
    s += " a_id=" + std::to_string(sp.a_id) + " b_id=" + std::to_string(sp.b_id) +
         " c_id=" + std::to_string(sp.c_id);
    auto perm = [&](const char *n, const std::vector<int> &p) {
      s += std::string(" ") + n + "=[";
      for (int v : p) s += std::to_string(v) + " ";
      s += "]";
    };
    perm("lperm", sp.lperm);
    perm("rperm", sp.rperm);
    perm("operm", sp.operm);
  }
  fprintf(stderr, "%s\n", s.c_str());
}

// ---------------------------------------------------------------------------
// Stem sweeps: fuse chains of consecutive skinny absorbs (kernels.h SweepGeom)
// ---------------------------------------------------------------------------
bool sweep_candidate(const stn_plan &P, const StepPlan &sp) {
  return P.precision == STN_SINGLE && !sp.d.is_branch && sp.has_bits &&
         (sp.kern == Kern::Absorb || sp.kern == Kern::AbsorbDirect || sp.kern == Kern::AbsorbTc) &&
         sp.kbits.size() <= 6 && sp.nbits.size() <= 6;
}

bool chain_candidate(const stn_plan &P, const StepPlan &sp) {
  return P.precision == STN_SINGLE && !sp.d.is_branch && sp.has_bits &&
         (sp.kern == Kern::Absorb || sp.kern == Kern::AbsorbDirect || sp.kern == Kern::AbsorbTc ||
          sp.kern == Kern::AbsorbTma || sp.kern == Kern::AbsorbMma || sp.kern == Kern::Lanes) &&
         int(sp.kbits.size()) <= stn::kChainMaxLog &&
         int(sp.nbits.size()) <= stn::kChainMaxLog + 10;  // growth steps: expansion rows
}

// Fused stem chain over steps [steps] (kernels.h ChainGeom). Follows every bit
// ("line") of the stem through the chain: X bits no stage contracts are passive
// (they only move; the lowest five are the warp's lanes, the rest rows), the
// others are active and live in a thread's tile (<= 2^kChainMaxLog values). Slot
// layout at a stage boundary: element index over the alive active lines in list
// order. Stage s reads [r][k] (k bit j = the step's K bit j, ascending X position:
// the reference's k order) and writes [r][n] (n bit j = N bit j, ascending O
// position). False when the chain does not fit or would not coalesce.
// Sector efficiency of ONE warp access of a tile (what the L1/L2 see per instruction,
// not what eventually reaches DRAM): the lanes' offsets plus the vector group the
// specialised kernel moves per access (tile elements at offsets 1, 2: chain_jit.cpp
// vec_bits), against the 32-byte sectors they touch.
double access_efficiency(const int64_t *lane_off_in, const int64_t *elem_off_in, int n_log,
                         bool jit, bool swaps) {
  const int vmax = jit ? stn::chain_vec_max() : 0;
  int64_t lane_sw[32], elem_sw[1 << stn::kChainMaxLog];
  const int64_t *lane_off = lane_off_in, *elem_off = elem_off_in;
  int j, sb;
  if (vmax >= 2 && swaps && stn::chain_lane_swap(lane_off_in, elem_off_in, n_log, &j, &sb)) {
    stn::chain_apply_swap(lane_off_in, elem_off_in, n_log, j, sb, lane_sw, elem_sw);
    lane_off = lane_sw;
    elem_off = elem_sw;
  }
  int v = 0;
  if (jit) {
    bool b0 = false, b1 = false;
    for (int j = 0; j < n_log; ++j) {
      b0 = b0 || elem_off[1 << j] == 1;
      b1 = b1 || elem_off[1 << j] == 2;
    }
    v = std::min(vmax, b0 ? (b1 ? 2 : 1) : 0);
  }
  std::set<int64_t> sectors;
  for (int l = 0; l < 32; ++l)
    for (int e = 0; e < (1 << v); ++e) sectors.insert((lane_off[l] + e) >> 2);
  return double(32 << v) / (4.0 * double(sectors.size()));
}

bool build_chain(const stn_plan &P, const std::vector<int> &steps, stn_plan::Sweep *out,
                 bool jit, double *eff_in, double *eff_out) {
  // STN_DEBUG chain_why=<step>: why segments starting at that step do not fit
  const char *why = stn::debug_opt("chain_why");
  const bool trace = why && !steps.empty() && std::atoi(why) == steps.front();
#define CHAIN_FAIL(at)                                                                  \
  do {                                                                                  \
    if (trace) fprintf(stderr, "chain from %d (%zu steps): no fit at stn_exec.cpp:%d\n", \
                       steps.front(), steps.size(), at);                                \
    return false;                                                                       \
  } while (0)
  // the NVRTC-specialised kernel holds up to 32 values per column in registers (64 in a
  // one-stage chain); the table-driven one 16 in shared memory, K, N <= 8 and K x N <= 16
  // per stage
  const int ns = int(steps.size());
  const char *ml = stn::debug_opt("chain_multi_log");  // tile limit of multi-stage chains (6)
  const int multi_log = ml ? std::max(2, std::min(stn::kChainMaxLog, std::atoi(ml)))
                           : stn::kChainMultiLog;
  const int max_log = !jit ? stn::kChainTableLog : ns == 1 ? stn::kChainMaxLog : multi_log;
  if (ns < 1 || ns > stn::kChainMaxStages || (ns == 1 && !jit)) CHAIN_FAIL(1180);
  const StepPlan &s0 = P.steps[steps[0]];
  const int xr0 = s0.xr;
  // line bookkeeping
  std::vector<int> pos2line(static_cast<size_t>(xr0));
  std::iota(pos2line.begin(), pos2line.end(), 0);
  int n_lines = xr0;
  std::vector<int> consumed_by(64, -1);  // line -> stage
  struct StageLines {
    std::vector<int> k, n;  // K lines (k bit order), N lines (n bit order)
    std::vector<int> nw;    // W bit position of each N line
  };
  std::vector<StageLines> sl(static_cast<size_t>(ns));
  for (int si = 0; si < ns; ++si) {
    const StepPlan &sp = P.steps[steps[si]];
    if (int(pos2line.size()) != sp.xr) CHAIN_FAIL(1195);
    for (auto &[xp, wp] : sp.kbits) {
      const int ln = pos2line[size_t(xp)];
      sl[size_t(si)].k.push_back(ln);
      consumed_by[size_t(ln)] = si;
    }
    std::vector<int> nxt(static_cast<size_t>(sp.orank_), -1);
    for (auto &[xp, op] : sp.mbits) nxt[size_t(op)] = pos2line[size_t(xp)];
    for (auto &[op, wp] : sp.nbits) {
      if (n_lines >= 64) CHAIN_FAIL(1204);
      nxt[size_t(op)] = n_lines;
      sl[size_t(si)].n.push_back(n_lines++);
      sl[size_t(si)].nw.push_back(wp);
    }
    for (int v : nxt)
      if (v < 0) CHAIN_FAIL(1210);
    pos2line.swap(nxt);
  }
  // Expansion rows: a first stage that grows the stem (many N lines from W, e.g. cfg5
  // 1605: 2^24 -> 2^32 elements) keeps the N lines no later stage consumes out of the
  // tile; they become the lowest row bits (each row reads the same X tile, from L1 /
  // L2, and a W column selected by its row). Specialised kernel only.
  std::vector<int> exp_lines, exp_w;
  const char *eo = stn::debug_opt("chain_exp");  // STN_DEBUG chain_exp=0: no expansion rows
  const char *es1 = stn::debug_opt("chain_exp_single");  // experiments: one-stage expansion
  const bool exp_single = es1 && std::atoi(es1) != 0;
  if (jit && (ns >= 2 || exp_single) && !(eo && std::atoi(eo) == 0)) {
    StageLines &z = sl[0];
    std::vector<int> keep, keep_w;
    for (size_t j = 0; j < z.n.size(); ++j)
      if (consumed_by[size_t(z.n[j])] < 0) {
        exp_lines.push_back(z.n[j]);
        exp_w.push_back(z.nw[j]);
      } else {
        keep.push_back(z.n[j]);
        keep_w.push_back(z.nw[j]);
      }
    if (exp_lines.size() >= 3 && int(z.n.size()) > 2) {
      z.n = keep;
      z.nw = keep_w;
    } else {
      exp_lines.clear();
      exp_w.clear();
    }
  }
  const int n_exp = int(exp_lines.size());
  if (n_exp > 10) CHAIN_FAIL(1239);  // W column block in shared memory
  const std::vector<int> &final_pos2line = pos2line;
  std::vector<int> opos_of(static_cast<size_t>(n_lines), -1);
  for (int op = 0; op < int(final_pos2line.size()); ++op) opos_of[size_t(final_pos2line[size_t(op)])] = op;
  // input-active: X lines consumed in the chain (ascending X position)
  std::vector<int> L;
  std::vector<int> passive;  // X lines never consumed
  for (int xp = 0; xp < xr0; ++xp) (consumed_by[size_t(xp)] >= 0 ? L : passive).push_back(xp);
  if (int(L.size()) > max_log || passive.size() < 5) CHAIN_FAIL(1247);
  // largest tile along the chain (alive active lines at a stage's input or output)
  int ma = int(L.size());
  {
    int alive = int(L.size());
    for (int si = 0; si < ns; ++si) {
      const int a_out = alive - int(sl[size_t(si)].k.size()) + int(sl[size_t(si)].n.size());
      ma = std::max(ma, std::max(alive, a_out));
      alive = a_out;
    }
  }
  // small tiles carry a fixed per-row cost (table lookups, the stage dispatch): the
  // passive lines right above the lanes ride along in the tile as lines no stage
  // touches, so a column holds 2^kChainMaxLog values and there are fewer rows
  const int extra = std::max(0, std::min(stn::kChainTableLog - ma, int(passive.size()) - 5));
  for (int q = 0; q < extra; ++q) L.push_back(passive[size_t(5 + q)]);
  passive.erase(passive.begin() + 5, passive.begin() + 5 + extra);
  const int li = int(L.size());
  for (int ln : passive)
    if (opos_of[size_t(ln)] < 0) CHAIN_FAIL(1266);
  auto T = std::make_unique<stn::ChainTables>();
  memset(T.get(), 0, sizeof(stn::ChainTables));
  stn::ChainGeom g{};
  g.n_stages = ns;
  g.li = li;
  for (int e = 0; e < (1 << li); ++e)
    for (int i = 0; i < li; ++i)
      if ((e >> i) & 1) T->xin[e] += int64_t(1) << L[size_t(i)];
  int tab = 0, widx = 0, wsm = 0;
  for (int si = 0; si < ns; ++si) {
    const StepPlan &sp = P.steps[steps[si]];
    const StageLines &st = sl[size_t(si)];
    std::vector<int> R;
    for (int ln : L)
      if (std::find(st.k.begin(), st.k.end(), ln) == st.k.end()) R.push_back(ln);
    const int lr = int(R.size()), lk = int(st.k.size()), ln_ = int(st.n.size());
    if (lr + lk > max_log || lr + ln_ > max_log) CHAIN_FAIL(1283);
    // table kernel: the stage shapes it instantiates (K, N <= 8), and K x N <= 16 (with
    // larger ones its per-column math is slower than the separate HBM-rate steps: cfg5
    // chain 1613-1614, K x N = 32, 41 ms fused vs 37 ms unfused, measured on B200)
    if (!jit && (lk > 3 || ln_ > 3 || lk + ln_ > 4)) CHAIN_FAIL(1287);
    g.ma = std::max(g.ma, std::max(lr + lk, lr + ln_));
    if (int(R.size()) + lk != int(L.size())) CHAIN_FAIL(1289);  // a K line not in the tile
    auto slot_in = [&](int ln) {
      return int(std::find(L.begin(), L.end(), ln) - L.begin());
    };
    stn::ChainStage &cs = g.st[si];
    cs.lr = lr;
    cs.lk = lk;
    cs.ln = ln_;
    const int le = si == 0 ? n_exp : 0;  // expansion bits of this stage's W block
    if (tab + (1 << lr) * ((1 << lk) + (1 << ln_)) > stn::kChainMaxTab ||
        widx + (1 << (lk + ln_ + le)) > stn::kChainMaxW)
      CHAIN_FAIL(1300);
    cs.rd_off = tab;
    for (int r = 0; r < (1 << lr); ++r)
      for (int k = 0; k < (1 << lk); ++k) {
        int e = 0;
        for (int i = 0; i < lr; ++i)
          if ((r >> i) & 1) e |= 1 << slot_in(R[size_t(i)]);
        for (int j = 0; j < lk; ++j)
          if ((k >> j) & 1) e |= 1 << slot_in(st.k[size_t(j)]);
        T->tab[tab++] = uint8_t(e);
      }
    cs.wr_off = tab;
    for (int r = 0; r < (1 << lr); ++r)
      for (int n = 0; n < (1 << ln_); ++n) T->tab[tab++] = uint8_t(r | (n << lr));
    cs.w_off = widx;
    cs.w_smem = wsm;
    // W block [k][e][n]: e = expansion column (row bits), n = tile N index
    for (int k = 0; k < (1 << lk); ++k)
      for (int e = 0; e < (1 << le); ++e)
        for (int n = 0; n < (1 << ln_); ++n) {
          int32_t off = 0;
          for (int j = 0; j < lk; ++j)
            if ((k >> j) & 1) off += int32_t(1) << sp.kbits[size_t(j)].second;
          for (int j = 0; j < ln_; ++j)
            if ((n >> j) & 1) off += int32_t(1) << st.nw[size_t(j)];
          for (int j = 0; j < le; ++j)
            if ((e >> j) & 1) off += int32_t(1) << exp_w[size_t(j)];
          T->widx[widx++] = off;
        }
    wsm += 1 << (lk + ln_ + le);
    // next layout: R lines, then the stage's N lines
    L = R;
    L.insert(L.end(), st.n.begin(), st.n.end());
  }
  g.lo = int(L.size());
  for (int ln : L)
    if (opos_of[size_t(ln)] < 0) CHAIN_FAIL(1336);
  for (int e = 0; e < (1 << g.lo); ++e)
    for (int i = 0; i < g.lo; ++i)
      if ((e >> i) & 1) T->oout[e] += int64_t(1) << opos_of[size_t(L[size_t(i)])];
  g.w_total = wsm;
  // passive lines: the 5 lowest X positions are the lanes, the rest the rows (after
  // the expansion lines, which are the lowest row bits and have no X offset)
  for (int ln : exp_lines)
    if (opos_of[size_t(ln)] < 0) CHAIN_FAIL(1344);
  std::vector<int> row_lines = exp_lines;
  row_lines.insert(row_lines.end(), passive.begin() + 5, passive.end());
  const int rb = int(row_lines.size());
  if (rb > 32) CHAIN_FAIL(1348);
  g.n_exp = n_exp;
  for (int l = 0; l < 32; ++l)
    for (int j = 0; j < 5; ++j)
      if ((l >> j) & 1) {
        T->xl[l] += int64_t(1) << passive[size_t(j)];
        T->ol[l] += int64_t(1) << opos_of[size_t(passive[size_t(j)])];
      }
  for (int c = 0; c < 4; ++c)
    for (int v = 0; v < 256; ++v)
      for (int j = 0; j < 8; ++j)
        if (((v >> j) & 1) && 8 * c + j < rb) {
          const int ln = row_lines[size_t(8 * c + j)];
          if (ln < xr0) T->xr[c][v] += int64_t(1) << ln;  // expansion lines: not in X
          T->orow[c][v] += int64_t(1) << opos_of[size_t(ln)];
        }
  g.rows = int64_t(1) << rb;
  // coalescing: 32-byte sectors one warp row touches, against the bytes it moves
  auto efficiency = [&](const int64_t *lane_off, const int64_t *elem_off, int ne) {
    std::set<int64_t> sectors;
    for (int e = 0; e < ne; ++e)
      for (int l = 0; l < 32; ++l) sectors.insert((lane_off[l] + elem_off[e]) >> 2);
    return double(32 * ne) / (4.0 * double(sectors.size()));
  };
  if (efficiency(T->xl, T->xin, 1 << li) < 0.5 || efficiency(T->ol, T->oout, 1 << g.lo) < 0.5)
    CHAIN_FAIL(1373);
  const bool swaps = jit && stn::chain_swaps_allowed(g);
  if (eff_in) *eff_in = access_efficiency(T->xl, T->xin, li, jit, swaps);
  if (eff_out) *eff_out = access_efficiency(T->ol, T->oout, g.lo, jit, swaps);
  if (!jit && stn::chain_smem_bytes(g) > 110 * 1024) CHAIN_FAIL(1377);  // table kernel's tiles
  if (out) {
    out->steps = steps;
    out->chain = true;
    out->cgeom = g;
    out->tables = std::make_shared<DevBuf>();
    out->tables->reserve(sizeof(stn::ChainTables));
    cuda_check(cudaMemcpy(out->tables->ptr, T.get(), sizeof(stn::ChainTables),
                          cudaMemcpyHostToDevice),
               "chain tables");
    out->host_tables = std::shared_ptr<stn::ChainTables>(T.release());
  }
  return true;
#undef CHAIN_FAIL
}

bool build_chain(const stn_plan &P, const std::vector<int> &steps, stn_plan::Sweep *out,
                 bool jit) {
  return build_chain(P, steps, out, jit, nullptr, nullptr);
}

// Tile-buffer swizzle of kernels_sweep.cu (linear over GF(2)).
int sweep_phys(int l) { return l ^ (((l >> 4) ^ (l >> 8)) & 15); }

// Builds the sweep geometry of chain steps [steps]; false if a tile does not fit.
bool build_sweep(const stn_plan &P, const std::vector<int> &steps, int max_bits,
                 stn_plan::Sweep *out) {
  if (steps.size() < 2 || int(steps.size()) > stn::kSweepMaxStages) return false;
  // labels by position, stage by stage
  std::vector<std::vector<int>> lab;  // lab[j][pos] for S_j
  const StepPlan &s0 = P.steps[steps[0]];
  std::vector<int> cur(s0.xr);
  for (int i = 0; i < s0.xr; ++i) cur[i] = i;
  int next_label = s0.xr;
  lab.push_back(cur);
  std::vector<std::vector<int>> klab(steps.size()), nlab(steps.size());
  std::set<int> touched;
  for (size_t j = 0; j < steps.size(); ++j) {
    const StepPlan &sp = P.steps[steps[j]];
    if (int(cur.size()) != sp.xr) return false;
    std::vector<int> nx(sp.orank_, -1);
    for (auto &[xp, wp] : sp.kbits) {
      klab[j].push_back(cur[xp]);
      touched.insert(cur[xp]);
    }
    for (auto &[xp, op] : sp.mbits) nx[op] = cur[xp];
    for (auto &[op, wp] : sp.nbits) {
      nx[op] = next_label;
      nlab[j].push_back(next_label);
      touched.insert(next_label++);
    }
    for (int x : nx)
      if (x < 0) return false;
    cur = nx;
    lab.push_back(cur);
  }
  std::set<int> keep = touched;  // + the lowest positions of S_0 and S_r (coalescing)
  for (int pos = 0; pos < 5; ++pos) {
    if (pos < int(lab.front().size())) keep.insert(lab.front()[pos]);
    if (pos < int(lab.back().size())) keep.insert(lab.back()[pos]);
  }
  // tile label lists per stage, in ascending position of that stage's tensor
  std::vector<std::vector<int>> tile(lab.size());
  int maxb = 0;
  for (size_t j = 0; j < lab.size(); ++j) {
    for (int pos = 0; pos < int(lab[j].size()); ++pos)
      if (keep.count(lab[j][pos])) tile[j].push_back(lab[j][pos]);
    maxb = std::max(maxb, int(tile[j].size()));
  }
  if (maxb > max_bits || maxb > stn::kSweepMaxTileBits) return false;
  // outer (pass-through) labels: in S_0 and S_r at their positions
  std::map<int, int> pos_first, pos_last;
  for (int pos = 0; pos < int(lab.front().size()); ++pos) pos_first[lab.front()[pos]] = pos;
  for (int pos = 0; pos < int(lab.back().size()); ++pos) pos_last[lab.back()[pos]] = pos;
  stn::SweepGeom g;
  memset(&g, 0, sizeof g);
  stn::AbsorbGeom &io = g.io;
  io.x_bits = int(lab.front().size());
  io.o_bits = int(lab.back().size());
  io.xt_bits = int(tile.front().size());
  io.ot_bits = int(tile.back().size());
  for (int i = 0; i < io.xt_bits; ++i) io.x_tile_pos[i] = uint8_t(pos_first.at(tile.front()[i]));
  for (int i = 0; i < io.ot_bits; ++i) io.o_tile_pos[i] = uint8_t(pos_last.at(tile.back()[i]));
  int ob = 0;
  for (int pos = 0; pos < int(lab.front().size()); ++pos) {
    const int l = lab.front()[pos];
    if (keep.count(l)) continue;
    if (!pos_last.count(l) || ob >= 34) return false;
    io.outer_x[ob] = uint8_t(pos);
    io.outer_o[ob] = uint8_t(pos_last.at(l));
    ob++;
  }
  io.ob = ob;
  if (ob > 31) return false;
  while (io.x_run < io.xt_bits && io.x_tile_pos[io.x_run] == io.x_run) io.x_run++;
  while (io.o_run < io.ot_bits && io.o_tile_pos[io.o_run] == io.o_run) io.o_run++;
  if (io.x_run < 1 || io.o_run < 1) return false;
  // per-stage tables
  std::vector<uint16_t> u16;
  std::vector<int64_t> i64;
  struct Off {
    size_t rb, ro, koff, nofs, w_idx;
  };
  std::vector<Off> offs;
  int w_total = 0, t_total = 0;
  g.n_stages = int(steps.size());
  g.max_bits = maxb;
  for (size_t j = 0; j < steps.size(); ++j) {
    const StepPlan &sp = P.steps[steps[j]];
    std::map<int, int> local_in, local_out;
    for (int i = 0; i < int(tile[j].size()); ++i) local_in[tile[j][i]] = i;
    for (int i = 0; i < int(tile[j + 1].size()); ++i) local_out[tile[j + 1][i]] = i;
    std::set<int> nset(nlab[j].begin(), nlab[j].end());
    std::vector<int> mlab;  // M labels of the stage tile, ascending output position
    for (int l : tile[j + 1])
      if (!nset.count(l)) mlab.push_back(l);
    {  // lane bits r0..r3: labels whose positions cover distinct swizzled bank bits
      const int m = int(mlab.size());
      int best_score = -1;
      std::vector<int> best;
      std::vector<int> pick;
      std::function<void(int)> rec = [&](int from) {
        if (int(pick.size()) == std::min(4, m)) {
          int in_mask = 0, out_mask = 0;
          for (int q : pick) {
            in_mask |= 1 << (local_in.at(mlab[q]) & 3);
            out_mask |= 1 << (local_out.at(mlab[q]) & 3);
          }
          const int score = __builtin_popcount(in_mask) + __builtin_popcount(out_mask);
          if (score > best_score) best_score = score, best = pick;
          return;
        }
        for (int q = from; q < m; ++q) {
          pick.push_back(q);
          rec(q + 1);
          pick.pop_back();
        }
      };
      rec(0);
      std::vector<int> order;
      for (int q : best) order.push_back(mlab[q]);
      for (int q = 0; q < m; ++q)
        if (std::find(best.begin(), best.end(), q) == best.end()) order.push_back(mlab[q]);
      mlab = order;
    }
    stn::SweepStage &st = g.st[j];
    st.in_bits = int(tile[j].size());
    st.out_bits = int(tile[j + 1].size());
    st.kb = int(klab[j].size());
    st.nb = int(nlab[j].size());
    const int R = 1 << int(mlab.size());
    // register tile RB x NC: up to 32 outputs per thread while all 128 threads have work
    {
      const int mbits_n = int(mlab.size());
      const int tile_log = std::max(0, std::min(5, st.out_bits - 7));
      st.nc_log = std::min({st.nb, 3, tile_log});
      st.rb_log = std::max(0, std::min({mbits_n - 4, 3, tile_log - st.nc_log}));
      st.nc_log = std::min({st.nb, 3, tile_log - st.rb_log});
      if (st.rb_log == 3) st.nc_log = std::min(st.nc_log, 2);
    }
    Off o;
    o.rb = u16.size();
    for (int r = 0; r < R; ++r) {
      int v = 0;
      for (int i = 0; i < int(mlab.size()); ++i)
        if ((r >> i) & 1) v |= 1 << local_in.at(mlab[i]);
      u16.push_back(uint16_t(sweep_phys(v)));
    }
    o.ro = u16.size();
    for (int r = 0; r < R; ++r) {
      int v = 0;
      for (int i = 0; i < int(mlab.size()); ++i)
        if ((r >> i) & 1) v |= 1 << local_out.at(mlab[i]);
      u16.push_back(uint16_t(sweep_phys(v)));
    }
    o.koff = u16.size();
    for (int k = 0; k < (1 << st.kb); ++k) {
      int v = 0;
      for (int i = 0; i < st.kb; ++i)
        if ((k >> i) & 1) v |= 1 << local_in.at(klab[j][i]);
      u16.push_back(uint16_t(sweep_phys(v)));
    }
    o.nofs = u16.size();
    for (int n = 0; n < (1 << st.nb); ++n) {
      int v = 0;
      for (int i = 0; i < st.nb; ++i)
        if ((n >> i) & 1) v |= 1 << local_out.at(nlab[j][i]);
      u16.push_back(uint16_t(sweep_phys(v)));
    }
    while (u16.size() % 4) u16.push_back(0);
    o.w_idx = i64.size();
    const int K = 1 << st.kb, N = 1 << st.nb;
    for (int k = 0; k < K; ++k)
      for (int n = 0; n < N; ++n) {
        int64_t off = 0;
        for (int i = 0; i < st.kb; ++i)
          if ((k >> i) & 1) off += int64_t(1) << sp.kbits[i].second;
        for (int i = 0; i < st.nb; ++i)
          if ((n >> i) & 1) off += int64_t(1) << sp.nbits[i].second;
        i64.push_back(off);
      }
    st.w_smem = w_total;
    w_total += (K * N + 1) & ~1;  // 16-byte aligned rows for the float4 W loads
    st.t_smem = t_total;
    t_total += K + N;
    offs.push_back(o);
  }
  g.w_total = w_total;
  g.t_total = t_total;
  if (stn::sweep_smem_bytes(g) > 110 * 1024) return false;  // >= 2 CTAs per SM
  if (!out) return true;
  // one device buffer: int64 w_idx first, then the uint16 tables
  std::vector<unsigned char> blob(i64.size() * 8 + u16.size() * 2);
  memcpy(blob.data(), i64.data(), i64.size() * 8);
  memcpy(blob.data() + i64.size() * 8, u16.data(), u16.size() * 2);
  out->tables = std::make_shared<DevBuf>();
  out->tables->upload(blob);
  const int64_t *d64 = out->tables->as<int64_t>();
  const uint16_t *d16 = reinterpret_cast<const uint16_t *>(d64 + i64.size());
  for (size_t j = 0; j < steps.size(); ++j) {
    g.st[j].rb = d16 + offs[j].rb;
    g.st[j].ro = d16 + offs[j].ro;
    g.st[j].koff = d16 + offs[j].koff;
    g.st[j].nofs = d16 + offs[j].nofs;
    g.st[j].w_idx = d64 + offs[j].w_idx;
  }
  out->steps = steps;
  out->geom = g;
  return true;
}

// Fused stem chains (default): maximal runs of consecutive stem absorbs (a step's
// output is the next step's stem operand) cut greedily into the longest segments
// build_chain accepts; only segments whose intermediate stems are large enough to
// matter are fused. STN_DEBUG chain=0 disables it; chain_min_bits=B (default 24):
// fuse only when an intermediate stem has >= 2^B elements.
void plan_chains(stn_plan &P, bool jit);

void plan_chains(stn_plan &P) {
  const char *opt = stn::debug_opt("chain");
  if (opt && std::atoi(opt) == 0) return;
  const char *jo = stn::debug_opt("chain_jit");
  const bool jit = stn::chain_jit_available() && !(jo && std::atoi(jo) == 0);
  P.chain_banned.clear();
  std::string log;
  for (int round = 0; round < 4; ++round) {
    plan_chains(P, jit);
    if (!jit || P.sweeps.empty()) return;
    // specialise every chain of the plan with NVRTC; a kernel that spills (its tiles
    // exceed the registers: > 64 B of local memory) bans its segment and the runs are
    // segmented again; if NVRTC fails, plan again for the table-driven kernel
    std::vector<stn::ChainJitSpec> specs;
    for (auto &sw : P.sweeps) specs.push_back({&sw.cgeom, sw.host_tables.get()});
    std::vector<void *> fns, alt;
    std::vector<int> local;
    // STN_DEBUG chain_alt=1: also compile every chain capped at 128 registers and keep the
    // faster variant on its first run (cfg5: 249 3.09 -> 2.77, 1185 3.09 -> 2.68 ms, the
    // big chains spill when capped; no measurable change per slice, twice the NVRTC work)
    const char *ao = stn::debug_opt("chain_alt");
    const bool want_alt = ao && std::atoi(ao) != 0;
    if (!stn::chain_jit_compile(specs, P.mode == STN_MODE_EXACT, P.device, &fns, &log, &local,
                                want_alt ? &alt : nullptr))
      break;
    bool banned = false;
    for (size_t i = 0; i < fns.size(); ++i) {
      P.sweeps[i].jit_fn = fns[i];
      P.sweeps[i].jit_alt = want_alt ? alt[i] : nullptr;
      P.sweeps[i].jit_pick = 0;
      if (local[i] > 64 && round < 3) {
        P.chain_banned.insert(P.sweeps[i].steps);
        banned = true;
      }
    }
    if (!banned) return;
    P.sweeps.clear();
    P.sweep_of_step.clear();
  }
  if (!P.sweeps.empty() && P.sweeps.front().jit_fn) return;
  if (stn::debug_opt("sweep_debug"))
    fprintf(stderr, "chain jit failed, table kernel instead: %s\n", log.substr(0, 2000).c_str());
  P.sweeps.clear();
  P.sweep_of_step.clear();
  plan_chains(P, false);
}

void plan_chains(stn_plan &P, bool jit) {
  const char *mb = stn::debug_opt("chain_min_bits");
  const int min_bits = mb ? std::atoi(mb) : 24;
  // one-stage chains (the specialised kernel) for slow single absorbs; STN_DEBUG
  // chain_single=0 disables them, =2 takes every step that fits (measurements)
  const char *so = stn::debug_opt("chain_single");
  const bool single = jit && !(so && std::atoi(so) == 0);
  const bool single_all = single && so && std::atoi(so) == 2;
  const char *ep = stn::debug_opt("chain_exp_pen");
  const bool exp_pen = !(ep && std::atoi(ep) == 0);
  const int n = int(P.steps.size());
  std::vector<int> next(n, -1), has_prev(n, 0);
  for (int i = 0; i < n; ++i) {
    const StepPlan &sp = P.steps[i];
    if (!chain_candidate(P, sp)) continue;
    const int c = P.nodes[sp.d.node].consumer;
    if (c < 0 || !chain_candidate(P, P.steps[c])) continue;
    const StepPlan &cp = P.steps[c];
    if ((cp.x_is_lhs ? cp.d.lhs : cp.d.rhs) != sp.d.node) continue;
    next[i] = c;
    has_prev[c] = 1;
  }
  for (int i = 0; i < n; ++i) {
    if (has_prev[i] || (next[i] < 0 && !(single && chain_candidate(P, P.steps[i])))) continue;
    std::vector<int> chain{i};
    while (next[chain.back()] >= 0) chain.push_back(next[chain.back()]);
    // Segmentation by dynamic programming over the run: a fused segment [a, b] gains
    // the HBM bytes of its intermediate stems (written and read back when unfused),
    // plus half the bytes of the steps it takes off the slower tile / tensor-core
    // absorbs (~3.3 TB/s measured, against ~6 TB/s for the fused pass). Only segments
    // whose largest intermediate has >= 2^min_bits elements are fused.
    const int m = int(chain.size());
    std::vector<std::vector<char>> fits(size_t(m), std::vector<char>(size_t(m), 0));
    std::vector<std::vector<char>> buildable = fits;  // fits, or built but banned
    // warp-access sector efficiency of each segment's stem input and output
    std::vector<std::vector<double>> e_in(size_t(m), std::vector<double>(size_t(m), 0.0));
    std::vector<std::vector<double>> e_out = e_in;
    for (int a = 0; a < m; ++a)
      for (int b = single ? a : a + 1; b < m; ++b) {
        std::vector<int> seg(chain.begin() + a, chain.begin() + b + 1);
        if (!build_chain(P, seg, nullptr, jit, &e_in[size_t(a)][size_t(b)],
                         &e_out[size_t(a)][size_t(b)])) {
          if (b == a) continue;
          break;  // longer ones from a fail too
        }
        buildable[size_t(a)][size_t(b)] = 1;
        if (P.chain_banned.count(seg)) continue;
        fits[size_t(a)][size_t(b)] = 1;
      }
    auto gain = [&](int a, int b) -> double {
      double g = 0;
      int64_t largest_mid = 0;
      for (int q = a; q <= b; ++q) {
        const StepPlan &sp = P.steps[chain[size_t(q)]];
        if (q < b) {
          g += 2.0 * double(sp.osize);
          largest_mid = std::max<int64_t>(largest_mid, sp.osize);
        }
        if (sp.kern == Kern::AbsorbTma || sp.kern == Kern::AbsorbTc || sp.kern == Kern::Absorb)
          g += 0.5 * double(sp.lsize + sp.rsize + sp.osize);
      }
      if (a == b) {
        // a one-stage chain (the specialised kernel as a single absorb) replaces the
        // slower absorb kernels when every warp access of its stem operand moves whole
        // 32-byte sectors and so do its stores, unless the output is small; measured on
        // B200 (cfg5 1185: tma 3.2 -> 5.9 TB/s; 1155, stores half-sector: 3.5 -> 3.3)
        const StepPlan &sp = P.steps[chain[size_t(a)]];
        const int64_t xsize = sp.x_is_lhs ? sp.lsize : sp.rsize;
        const bool slow = sp.kern == Kern::AbsorbTma || sp.kern == Kern::AbsorbTc ||
                          sp.kern == Kern::Absorb || sp.kern == Kern::Lanes ||
                          sp.kern == Kern::AbsorbMma;
        // ... and while its math stays under the HBM stream: K x N <= 12 (K + N) complex
        // multiply-adds per column element moved (cfg2 494 / 536, K x N = 1024 against
        // 80 / 64 elements: 3.6 -> 2.7 TB/s; cfg5 1365, 512 against 48, is kept)
        const int64_t K = int64_t(1) << sp.kbits.size(), N = int64_t(1) << sp.nbits.size();
        const char *es1 = stn::debug_opt("chain_exp_single");
        const bool exp_single = es1 && std::atoi(es1) != 0 && sp.nbits.size() >= 3;
        const bool coalesced = e_in[size_t(a)][size_t(a)] > 0.99 &&
                               (e_out[size_t(a)][size_t(a)] > 0.99 || 4 * sp.osize <= xsize ||
                                exp_single) &&
                               (K * N <= 12 * (K + N) || exp_single);
        g = (single_all || (slow && coalesced)) ? 0.5 * double(sp.lsize + sp.rsize + sp.osize)
                                                : 0.0;
        return sp.osize >= (int64_t(1) << min_bits) ? g - 1.0 : -1.0;
      }
      // half-sector warp accesses on the chain's stem input / output cost about a second
      // pass over those bytes (cfg5 1155-1161, output at 0.5: 13.1 ms unfused, 18.8 fused)
      const StepPlan &s0 = P.steps[chain[size_t(a)]], &s1 = P.steps[chain[size_t(b)]];
      const double xin = double(s0.x_is_lhs ? s0.lsize : s0.rsize);
      g -= (1.0 / std::max(e_in[size_t(a)][size_t(b)], 0.25) - 1.0) * xin;
      g -= (1.0 / std::max(e_out[size_t(a)][size_t(b)], 0.25) - 1.0) * double(s1.osize);
      // a growth step fused as expansion rows re-reads its stem operand once per row
      // group (8 warps of a CTA share it in L1): costly once that operand outgrows L2
      if (exp_pen && b > a && double(s0.osize) > 4.0 * xin && xin > double(int64_t(1) << 24))
        g -= 8.0 * xin;
      return largest_mid >= (int64_t(1) << min_bits) ? g : -1.0;
    };
    std::vector<double> best(size_t(m) + 1, 0.0);  // best[i]: steps [i, m)
    std::vector<int> cut(size_t(m) + 1, -1);
    for (int a = m - 1; a >= 0; --a) {
      best[size_t(a)] = best[size_t(a) + 1];  // step a alone
      cut[size_t(a)] = a;
      for (int b = single ? a : a + 1; b < m && (b == a || buildable[size_t(a)][size_t(b)]); ++b) {
        if (!fits[size_t(a)][size_t(b)]) continue;
        const double g = gain(a, b);
        if (g > 0 && g + best[size_t(b) + 1] > best[size_t(a)]) {
          best[size_t(a)] = g + best[size_t(b) + 1];
          cut[size_t(a)] = b;
        }
      }
    }
    for (int a = 0; a < m;) {
      const int b = cut[size_t(a)];
      if (b > a || (single && b == a && best[size_t(a)] > best[size_t(a) + 1])) {
        std::vector<int> seg(chain.begin() + a, chain.begin() + b + 1);
        stn_plan::Sweep sw;
        double ei = 0, eo = 0;
        if (build_chain(P, seg, &sw, jit, &ei, &eo)) {
          const int id = int(P.sweeps.size());
          if (stn::debug_opt("sweep_debug")) {
            fprintf(stderr, "chain %d: steps", id);
            for (int q : seg) fprintf(stderr, " %d", q);
            fprintf(stderr, " | li %d lo %d rows 2^%d | access efficiency in %.2f out %.2f\n",
                    sw.cgeom.li, sw.cgeom.lo, __builtin_ctzll(uint64_t(sw.cgeom.rows)), ei, eo);
          }
          for (int st : seg) P.sweep_of_step[st] = id;
          P.sweeps.push_back(std::move(sw));
        }
      }
      a = b + 1;
    }
  }
}

void plan_sweeps(stn_plan &P) {
  P.sweeps.clear();
  P.sweep_of_step.clear();
  // Off by default: measured on B200 (profiles/r01_sweep_vs_unfused.txt) the
  // per-tile stage math of a sweep is FFMA-issue bound and loses to the
  // unfused HBM-rate direct / tensor-core absorbs. STN_SWEEP_BITS=<tile bits>
  // (e.g. 12) enables it; read per plan so tests can toggle it.
  const char *env_bits = stn::debug_opt("sweep_bits");
  const int max_bits = env_bits ? std::atoi(env_bits) : 0;
  if (max_bits <= 0) return plan_chains(P);
  const int n = int(P.steps.size());
  std::vector<int> next(n, -1), has_prev(n, 0);
  for (int i = 0; i < n; ++i) {
    const StepPlan &sp = P.steps[i];
    if (!sweep_candidate(P, sp)) continue;
    const int c = P.nodes[sp.d.node].consumer;
    if (c < 0 || !sweep_candidate(P, P.steps[c])) continue;
    const StepPlan &cp = P.steps[c];
    if ((cp.x_is_lhs ? cp.d.lhs : cp.d.rhs) != sp.d.node) continue;
    next[i] = c;
    has_prev[c] = 1;
  }
  for (int i = 0; i < n; ++i) {
    if (has_prev[i] || next[i] < 0) continue;
    std::vector<int> chain{i};
    while (next[chain.back()] >= 0) chain.push_back(next[chain.back()]);
    size_t a = 0;
    while (a < chain.size()) {
      size_t best = a;
      for (size_t b = a + 1; b < chain.size(); ++b) {
        std::vector<int> seg(chain.begin() + a, chain.begin() + b + 1);
        if (build_sweep(P, seg, max_bits, nullptr))
          best = b;
        else
          break;
      }
      if (best > a) {
        stn_plan::Sweep sw;
        std::vector<int> seg(chain.begin() + a, chain.begin() + best + 1);
        static const char *env_only = stn::debug_opt("sweep_only");  // profiling aid
        static int seen = 0;
        const bool take = !env_only || std::atoi(env_only) == seen;
        ++seen;
        if (take && build_sweep(P, seg, max_bits, &sw)) {
          const int id = int(P.sweeps.size());
          if (stn::debug_opt("sweep_debug")) {
            const stn::SweepGeom &g = sw.geom;
            fprintf(stderr, "sweep %d: steps", id);
            for (int q : seg) fprintf(stderr, " %d", q);
            fprintf(stderr, " | xt %d ot %d max %d ob %d xrun %d orun %d smem %zu\n",
                    g.io.xt_bits, g.io.ot_bits, g.max_bits, g.io.ob, g.io.x_run, g.io.o_run,
                    stn::sweep_smem_bytes(g));
            for (int q = 0; q < g.n_stages; ++q)
              fprintf(stderr, "   stage %d: in %d out %d kb %d nb %d nc_log %d rb_log %d\n", q,
                      g.st[q].in_bits, g.st[q].out_bits, g.st[q].kb, g.st[q].nb, g.st[q].nc_log,
                      g.st[q].rb_log);
          }
          for (int st : seg) P.sweep_of_step[st] = id;
          P.sweeps.push_back(std::move(sw));
        }
      }
      a = best + 1;
    }
  }
}

void build_program(stn_plan &P, Program &prog, int which /*0 build, 1 cache, 2 no cache*/) {
  prog.ops.clear();
  prog.slice_leaves.clear();
  prog.slice_leaf_off.clear();
  prog.mults = 0;
  prog.peak = 0;
  struct Item {
    int64_t size, start, end;
    int64_t *off;
  };
  std::vector<Item> items;
  std::vector<std::unique_ptr<int64_t>> offs;
  auto new_item = [&](int64_t size, int64_t start, int64_t end) {
    offs.emplace_back(new int64_t(0));
    items.push_back({size, start, end, offs.back().get()});
    return offs.back().get();
  };
  // which steps run
  std::vector<int> run;
  for (int i = 0; i < int(P.steps.size()); ++i) {
    bool br = P.steps[i].d.is_branch != 0;
    if (which == 0 && br) run.push_back(i);
    if (which == 1 && !br) run.push_back(i);
    if (which == 2) run.push_back(i);
  }
  // units: single steps, or a fused sweep emitted at the position of its last step
  std::vector<std::vector<int>> units;
  std::vector<int> unit_sweep;
  for (int k = 0; k < int(run.size()); ++k) {
    const int st = run[k];
    auto sw = which == 0 ? P.sweep_of_step.end() : P.sweep_of_step.find(st);
    if (sw == P.sweep_of_step.end()) {
      units.push_back({st});
      unit_sweep.push_back(-1);
    } else if (P.sweeps[sw->second].steps.back() == st) {
      units.push_back(P.sweeps[sw->second].steps);
      unit_sweep.push_back(sw->second);
    }
  }
  std::map<int, int> op_of_step;
  for (int u = 0; u < int(units.size()); ++u)
    for (int st : units[u]) op_of_step[st] = u;
  const int64_t n_ops = int64_t(units.size());
  // consumer op of each node within this program (chain-internal stems excluded)
  std::map<int, int64_t> consumer_op;
  for (int u = 0; u < int(units.size()); ++u) {
    std::set<int> internal;
    for (int st : units[u]) internal.insert(P.steps[st].d.node);
    for (int st : units[u]) {
      const StepPlan &sp = P.steps[st];
      for (int in : {sp.d.lhs, sp.d.rhs})
        if (!internal.count(in)) consumer_op[in] = u;
    }
  }
  auto end_of = [&](int node) -> int64_t {
    auto it = consumer_op.find(node);
    return it == consumer_op.end() ? n_ops : it->second;  // root lives to the end
  };
  // where a program input comes from
  std::map<int, int64_t *> out_off_ptr;   // node produced in this program -> arena offset
  std::map<int, int64_t *> leaf_off_ptr;  // sliced leaf -> arena offset
  auto make_input = [&](int node) -> Ref {
    Ref r;
    r.node = node;
    r.size = P.nodes[node].size;
    const Node &nd = P.nodes[node];
    if (!nd.is_leaf) {
      int st = nd.step;
      if (op_of_step.count(st)) {
        if (which == 0 && P.cache_off.count(node)) {
          r.kind = Src::Persist;
          r.off = P.cache_off.at(node);
        } else {
          r.kind = Src::Arena;  // offset resolved after allocation
        }
      } else {
        require(which == 1 && P.cache_off.count(node), STN_ERR_SUBTASK_FAILURE,
                "operand for node " + std::to_string(node) + " unavailable");
        r.kind = Src::Cache;
        r.off = P.cache_off.at(node);
      }
    } else if (nd.sliced_leaf) {
      require(which != 0, STN_ERR_SUBTASK_FAILURE, "sliced leaf feeds a branch step");
      r.kind = Src::SliceLeaf;
      if (!leaf_off_ptr.count(node)) {
        leaf_off_ptr[node] = new_item(nd.size, -1, end_of(node));
        prog.slice_leaves.push_back(node);
      }
    } else {
      r.kind = Src::ConstLeaf;
      r.off = P.const_off.at(node);
    }
    return r;
  };
  // side-stream candidates (per-slice programs): small steps on kernels that use no
  // lane workspace; their outputs live from the start of the program so that no stem
  // step's buffer shares their memory (no write-after-read waits between the streams).
  // Off unless STN_DEBUG side=1: measured on B200 it neither helps nor hurts (cfg5
  // 122.1 / 122.3, cfg4 51.1 / 51.4, cfg2 7.52 / 7.48 ms per slice without / with)
  const char *side_opt = stn::debug_opt("side");
  const bool side_on = which != 0 && side_opt && std::atoi(side_opt) != 0;
  auto side_ok = [&](int u) {
    if (!side_on || unit_sweep[u] >= 0) return false;
    const StepPlan &sp = P.steps[units[u].back()];
    const bool kern_ok = sp.kern == Kern::Generic || sp.kern == Kern::Outer ||
                         sp.kern == Kern::AbsorbDirect || sp.kern == Kern::Lanes ||
                         sp.kern == Kern::Absorb;
    return kern_ok && sp.osize <= (int64_t(1) << 22);
  };
  prog.side.assign(units.size(), 0);
  for (int u = 0; u < int(units.size()); ++u) {
    const StepPlan &last = P.steps[units[u].back()];
    Op op;
    op.step = units[u].back();
    op.sweep = unit_sweep[u];
    prog.side[size_t(u)] = side_ok(u) ? 1 : 0;
    if (op.sweep >= 0) {
      const StepPlan &first = P.steps[units[u].front()];
      op.a = make_input(first.x_is_lhs ? first.d.lhs : first.d.rhs);
      for (int st : units[u]) {
        const StepPlan &sp = P.steps[st];
        op.wrefs.push_back(make_input(sp.x_is_lhs ? sp.d.rhs : sp.d.lhs));
      }
    } else {
      op.a = make_input(last.d.lhs);
      op.b = make_input(last.d.rhs);
    }
    op.out.node = last.d.node;
    op.out.size = last.osize;
    if (which == 0 && P.cache_off.count(last.d.node)) {
      op.out.kind = Src::Persist;
      op.out.off = P.cache_off.at(last.d.node);
    } else {
      op.out.kind = Src::Arena;
      out_off_ptr[last.d.node] =
          new_item(last.osize, prog.side[size_t(u)] ? -1 : u, end_of(last.d.node));
    }
    prog.ops.push_back(op);
    for (int st : units[u]) {  // SubtaskResult bookkeeping counts every step
      prog.mults += P.steps[st].d.mults;
      prog.peak = std::max<uint64_t>(prog.peak, uint64_t(P.steps[st].osize));
    }
  }
  prog.n_steps = int(run.size());
  // gemm-path scratch (lifetime: the op itself)
  std::vector<std::array<int64_t *, 3>> scr(prog.ops.size(), {nullptr, nullptr, nullptr});
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    const StepPlan &sp = P.steps[prog.ops[k].step];
    if (prog.ops[k].sweep >= 0) continue;
    if (sp.kern != Kern::GemmSimt && sp.kern != Kern::GemmTc) continue;
    // A needs no scratch when the skinny GEMM gathers it through its offset table or the
    // tile permute writes it straight into the tcgen05 workspace (a_fused in launch_op)
    const bool a_in_place = sp.skinny_tab || sp.tcf_gather ||
                            (sp.kern == Kern::GemmTc && !sp.tcf && sp.pa_bases &&
                                              stn::gemm_tc_supported(sp.gs));
    if (!sp.a_id && !a_in_place)
      scr[k][0] = new_item(sp.gemm_swap ? sp.rsize : sp.lsize, int64_t(k), int64_t(k));
    if (!sp.b_id) scr[k][1] = new_item(sp.gemm_swap ? sp.lsize : sp.rsize, int64_t(k), int64_t(k));
    if (!sp.c_id) scr[k][2] = new_item(sp.osize, int64_t(k), int64_t(k));
  }
  // liveness allocation: biggest first, lowest non-conflicting offset
  std::vector<size_t> order(items.size());
  std::iota(order.begin(), order.end(), 0);
  std::stable_sort(order.begin(), order.end(),
                   [&](size_t a, size_t b) { return items[a].size > items[b].size; });
  const int64_t align = 64;  // elements (512 B in single precision)
  auto aligned = [&](int64_t x) { return (x + align - 1) / align * align; };
  std::vector<size_t> placed;
  int64_t arena = 0;
  for (size_t i : order) {
    Item &it = items[i];
    std::vector<std::pair<int64_t, int64_t>> busy;
    for (size_t j : placed) {
      const Item &o = items[j];
      if (o.start <= it.end && it.start <= o.end) busy.push_back({*o.off, *o.off + aligned(o.size)});
    }
    std::sort(busy.begin(), busy.end());
    int64_t cand = 0;
    for (auto &[lo, hi] : busy) {
      if (cand + aligned(it.size) <= lo) break;
      cand = std::max(cand, hi);
    }
    *it.off = cand;
    arena = std::max(arena, cand + aligned(it.size));
    placed.push_back(i);
  }
  prog.arena_elems = arena;
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    Op &op = prog.ops[k];
    std::vector<Ref *> refs{&op.a};
    if (op.sweep < 0) refs.push_back(&op.b);
    for (Ref &w : op.wrefs) refs.push_back(&w);
    for (Ref *r : refs)
      if (r->kind == Src::Arena)
        r->off = *out_off_ptr.at(r->node);
      else if (r->kind == Src::SliceLeaf)
        r->off = *leaf_off_ptr.at(r->node);
    if (op.out.kind == Src::Arena) op.out.off = *out_off_ptr.at(op.out.node);
    op.scr_a = scr[k][0] ? *scr[k][0] : -1;
    op.scr_b = scr[k][1] ? *scr[k][1] : -1;
    op.scr_c = scr[k][2] ? *scr[k][2] : -1;
  }
  for (int node : prog.slice_leaves) prog.slice_leaf_off[node] = *leaf_off_ptr.at(node);
  // cross-stream ordering of the side-stream schedule
  {
    const size_t n_ops = prog.ops.size();
    prog.wait_other.assign(n_ops, -1);
    prog.need_event.assign(n_ops, 0);
    for (size_t k = 0; k < n_ops; ++k) prog.has_side = prog.has_side || prog.side[k];
    if (prog.has_side) {
      using Reg = std::pair<int64_t, int64_t>;
      std::vector<std::vector<Reg>> rd(n_ops), wr(n_ops);
      auto region = [&](const Ref &r, std::vector<Reg> &v) {
        if (r.kind == Src::Arena || r.kind == Src::SliceLeaf)
          v.push_back({r.off, r.off + aligned(r.size)});
      };
      for (size_t k = 0; k < n_ops; ++k) {
        const Op &op = prog.ops[k];
        region(op.a, rd[k]);
        if (op.sweep < 0) region(op.b, rd[k]);
        for (const Ref &w : op.wrefs) region(w, rd[k]);
        region(op.out, wr[k]);
        const StepPlan &sp = P.steps[op.step];
        if (op.scr_a >= 0) wr[k].push_back({op.scr_a, op.scr_a + aligned(sp.gemm_swap ? sp.rsize : sp.lsize)});
        if (op.scr_b >= 0) wr[k].push_back({op.scr_b, op.scr_b + aligned(sp.gemm_swap ? sp.lsize : sp.rsize)});
        if (op.scr_c >= 0) wr[k].push_back({op.scr_c, op.scr_c + aligned(sp.osize)});
      }
      auto meet = [](const std::vector<Reg> &x, const std::vector<Reg> &y) {
        for (const Reg &a : x)
          for (const Reg &b : y)
            if (a.first < b.second && b.first < a.second) return true;
        return false;
      };
      for (size_t k = 0; k < n_ops; ++k)
        for (size_t j = k; j-- > 0;) {
          if (prog.side[j] == prog.side[k]) continue;
          if (meet(wr[j], rd[k]) || meet(rd[j], wr[k]) || meet(wr[j], wr[k])) {
            prog.wait_other[k] = int(j);
            prog.need_event[j] = 1;
            break;
          }
        }
    }
  }
  // root
  prog.has_root = which != 0;
  if (prog.has_root) {
    int root = P.root;
    if (out_off_ptr.count(root)) {
      prog.root = Ref{Src::Arena, root, *out_off_ptr.at(root), P.nodes[root].size};
    } else if (P.nodes[root].is_leaf) {
      prog.root = Ref{};
      prog.root.node = root;
      prog.root.size = P.nodes[root].size;
      if (P.nodes[root].sliced_leaf) {
        prog.root.kind = Src::SliceLeaf;
        if (!leaf_off_ptr.count(root)) {
          // a lone sliced leaf: give it its own arena slot at the end
          prog.slice_leaves.push_back(root);
          prog.slice_leaf_off[root] = prog.arena_elems;
          prog.arena_elems += aligned(P.nodes[root].size);
        }
        prog.root.off = prog.slice_leaf_off.at(root);
      } else {
        prog.root.kind = Src::ConstLeaf;
        prog.root.off = P.const_off.at(root);
      }
    } else {
      require(which == 1 && P.cache_off.count(root), STN_ERR_SUBTASK_FAILURE,
              "root unavailable");
      prog.root = Ref{Src::Cache, root, P.cache_off.at(root), P.nodes[root].size};
    }
  }
  // leaf-gather table
  std::vector<int64_t> src_base, dst_off, dst_bs, ax_stride;
  std::vector<int32_t> elem_leaf, elem_local, ax_begin, ax_slice;
  ax_begin.push_back(0);
  for (size_t li = 0; li < prog.slice_leaves.size(); ++li) {
    int node = prog.slice_leaves[li];
    const stn_leaf_desc &L = P.leaf_desc[P.nodes[node].leaf];
    std::vector<int> dims(L.dims, L.dims + L.rank);
    std::vector<int64_t> st = row_major_strides(dims);
    std::vector<char> sliced(L.rank, 0);
    for (int s = 0; s < L.n_sliced; ++s) {
      sliced[L.sliced_axis[s]] = 1;
      ax_stride.push_back(st[L.sliced_axis[s]]);
      ax_slice.push_back(L.sliced_index[s]);
    }
    ax_begin.push_back(int32_t(ax_stride.size()));
    std::vector<int> kept_axes;
    for (int a = 0; a < L.rank; ++a)
      if (!sliced[a]) kept_axes.push_back(a);
    // canonical axis i = kept axis perm[i]
    std::vector<int> cdims(L.perm_rank);
    std::vector<int64_t> cstr(L.perm_rank);
    for (int i = 0; i < L.perm_rank; ++i) {
      cdims[i] = dims[kept_axes[L.perm[i]]];
      cstr[i] = st[kept_axes[L.perm[i]]];
    }
    int64_t n = 1;
    for (int x : cdims) n *= x;
    const int64_t voff = P.sliced_val_off.at(node);
    for (int64_t e = 0; e < n; ++e) {
      int64_t rem = e, src = 0;
      for (int i = L.perm_rank - 1; i >= 0; --i) {
        src += (rem % cdims[i]) * cstr[i];
        rem /= cdims[i];
      }
      src_base.push_back(voff + src);
      elem_leaf.push_back(int32_t(li));
      elem_local.push_back(int32_t(e));
    }
    dst_off.push_back(prog.slice_leaf_off.at(node));
    dst_bs.push_back(P.nodes[node].size);
  }
  prog.t_src_base.upload(src_base);
  prog.t_elem_leaf.upload(elem_leaf);
  prog.t_elem_local.upload(elem_local);
  prog.t_dst_off.upload(dst_off);
  prog.t_dst_bs.upload(dst_bs);
  prog.t_ax_begin.upload(ax_begin);
  prog.t_ax_stride.upload(ax_stride);
  prog.t_ax_slice.upload(ax_slice);
  stn::LeafGatherTable &t = prog.table;
  t.values = P.sliced_vals.as<double>();
  t.src_base = prog.t_src_base.as<int64_t>();
  t.elem_leaf = prog.t_elem_leaf.as<int32_t>();
  t.dst_off = prog.t_dst_off.as<int64_t>();
  t.dst_bs = prog.t_dst_bs.as<int64_t>();
  t.elem_local = prog.t_elem_local.as<int32_t>();
  t.ax_begin = prog.t_ax_begin.as<int32_t>();
  t.ax_stride = prog.t_ax_stride.as<int64_t>();
  t.ax_slice = prog.t_ax_slice.as<int32_t>();
  t.total_out = int64_t(src_base.size());
  t.n_sliced = int(P.sliced_dims.size());
}

// canonical, executor-precision copy of an unsliced leaf (load_leaf without
// restriction: from_tensor + permute, runtime.hpp:382-383)
void canonical_leaf(const stn_plan &P, int leaf, std::vector<double> &out) {
  const stn_leaf_desc &L = P.leaf_desc[leaf];
  std::vector<int> dims(L.dims, L.dims + L.rank);
  std::vector<int64_t> st = row_major_strides(dims);
  std::vector<int> cdims(L.perm_rank);
  std::vector<int64_t> cstr(L.perm_rank);
  for (int i = 0; i < L.perm_rank; ++i) {
    cdims[i] = dims[L.perm[i]];
    cstr[i] = st[L.perm[i]];
  }
  int64_t n = 1;
  for (int x : cdims) n *= x;
  out.resize(2 * n);
  for (int64_t e = 0; e < n; ++e) {
    int64_t rem = e, src = 0;
    for (int i = L.perm_rank - 1; i >= 0; --i) {
      src += (rem % cdims[i]) * cstr[i];
      rem /= cdims[i];
    }
    out[2 * e] = L.values[2 * src];
    out[2 * e + 1] = L.values[2 * src + 1];
  }
}

void upload_consts(stn_plan &P) {
  std::vector<unsigned char> host(size_t(P.consts_elems) * P.esize);
  for (auto &[node, off] : P.const_off) {
    std::vector<double> v;
    canonical_leaf(P, P.nodes[node].leaf, v);
    for (size_t i = 0; i < v.size(); ++i) {
      if (P.precision == STN_SINGLE) {
        float f = float(v[i]);
        memcpy(host.data() + (size_t(off) * 2 + i) * 4, &f, 4);
      } else {
        memcpy(host.data() + (size_t(off) * 2 + i) * 8, &v[i], 8);
      }
    }
  }
  P.consts.upload(host);
}

void upload_sliced_values(stn_plan &P) {
  std::vector<double> vals;
  for (auto &[node, off] : P.sliced_val_off) {
    const stn_leaf_desc &L = P.leaf_desc[P.nodes[node].leaf];
    int64_t n = 1;
    for (int a = 0; a < L.rank; ++a) n *= L.dims[a];
    vals.resize(std::max<size_t>(vals.size(), size_t(2 * (off + n))));
    memcpy(vals.data() + 2 * off, L.values, size_t(16 * n));
  }
  P.sliced_vals.upload(vals);
}

void create_plan(const stn_plan_desc *desc, int device, int mode, stn_plan *P) {
  const auto t_begin = std::chrono::steady_clock::now();
  double choose_ms[16] = {0};  // per kernel kind (STN_PLAN_TIMING)
  require(desc != nullptr, STN_ERR_INVALID_ARGUMENT, "NULL plan descriptor");
  require(desc->precision == STN_SINGLE || desc->precision == STN_DOUBLE,
          STN_ERR_INVALID_ARGUMENT, "bad precision");
  require(mode == STN_MODE_FAST || mode == STN_MODE_EXACT, STN_ERR_INVALID_ARGUMENT, "bad mode");
  int ndev = 0;
  cudaError_t e = cudaGetDeviceCount(&ndev);
  require(e == cudaSuccess && ndev > 0, STN_ERR_NO_DEVICE, "no CUDA device available");
  require(device >= 0 && device < ndev, STN_ERR_NO_DEVICE, "device index out of range");
  cuda_check(cudaSetDevice(device), "cudaSetDevice");
  {  // STN_DEBUG graphs=0: every batch launched eagerly (no CUDA graphs)
    const char *g = stn::debug_opt("graphs");
    P->graphs = !(g && std::atoi(g) == 0);
  }
  // (attribute queries: cudaGetDeviceProperties costs milliseconds per call)
  int cc_major = 0, cc_minor = 0;
  cuda_check(cudaDeviceGetAttribute(&cc_major, cudaDevAttrComputeCapabilityMajor, device),
             "cudaDeviceGetAttribute");
  cuda_check(cudaDeviceGetAttribute(&cc_minor, cudaDevAttrComputeCapabilityMinor, device),
             "cudaDeviceGetAttribute");
  require(cc_major == 10, STN_ERR_NO_DEVICE,
          "executor is built for sm_100a; device is sm_" + std::to_string(cc_major) +
              std::to_string(cc_minor));
  const auto t_dev = std::chrono::steady_clock::now();
  P->device = device;
  P->mode = mode;
  P->precision = desc->precision;
  P->esize = desc->precision == STN_SINGLE ? 8 : 16;
  P->identity = desc->identity;
  P->subtasks = desc->subtasks;
  P->merged_groups = desc->merged_groups;
  P->exec_cw = desc->exec_cw;
  P->root = desc->root;
  require(desc->n_nodes > 0 && desc->root >= 0 && desc->root < desc->n_nodes,
          STN_ERR_MALFORMED_NETWORK, "bad node count / root");
  P->sliced_dims.assign(desc->sliced_dims, desc->sliced_dims + desc->n_sliced);
  for (int32_t d : P->sliced_dims) require(d > 0, STN_ERR_MALFORMED_NETWORK, "bad sliced dim");
  P->nodes.assign(desc->n_nodes, Node{});
  // leaves (copied: the descriptor may be freed after create)
  const int nl = desc->n_leaves;
  P->leaf_desc.resize(nl);
  P->leaf_dims.resize(nl);
  P->leaf_sax.resize(nl);
  P->leaf_sidx.resize(nl);
  P->leaf_perm.resize(nl);
  P->leaf_values.resize(nl);
  for (int i = 0; i < nl; ++i) {
    const stn_leaf_desc &L = desc->leaves[i];
    require(L.node >= 0 && L.node < desc->n_nodes && L.rank >= 0 && L.rank <= 64 &&
                L.n_sliced >= 0 && L.n_sliced <= L.rank && L.perm_rank == L.rank - L.n_sliced,
            STN_ERR_MALFORMED_NETWORK, "malformed leaf " + std::to_string(i));
    P->leaf_dims[i].assign(L.dims, L.dims + L.rank);
    P->leaf_sax[i].assign(L.sliced_axis, L.sliced_axis + L.n_sliced);
    P->leaf_sidx[i].assign(L.sliced_index, L.sliced_index + L.n_sliced);
    P->leaf_perm[i].assign(L.perm, L.perm + L.perm_rank);
    int64_t n = 1;
    for (int a = 0; a < L.rank; ++a) {
      require(L.dims[a] > 0, STN_ERR_MALFORMED_NETWORK, "bond dimension must be positive");
      n *= L.dims[a];
    }
    P->leaf_values[i].assign(L.values, L.values + 2 * n);
    for (int s = 0; s < L.n_sliced; ++s)
      require(L.sliced_axis[s] >= 0 && L.sliced_axis[s] < L.rank && L.sliced_index[s] >= 0 &&
                  L.sliced_index[s] < desc->n_sliced &&
                  L.dims[L.sliced_axis[s]] == desc->sliced_dims[L.sliced_index[s]],
              STN_ERR_MALFORMED_NETWORK, "malformed sliced axis");
    for (int s = 1; s < L.n_sliced; ++s)
      require(L.sliced_axis[s] < L.sliced_axis[s - 1], STN_ERR_MALFORMED_NETWORK,
              "sliced axes must be in descending order");
    stn_leaf_desc c = L;
    c.dims = P->leaf_dims[i].data();
    c.sliced_axis = P->leaf_sax[i].data();
    c.sliced_index = P->leaf_sidx[i].data();
    c.perm = P->leaf_perm[i].data();
    c.values = P->leaf_values[i].data();
    P->leaf_desc[i] = c;
    Node &nd = P->nodes[L.node];
    require(!nd.is_leaf, STN_ERR_MALFORMED_NETWORK, "duplicate leaf node");
    nd.is_leaf = true;
    nd.leaf = i;
    nd.sliced_leaf = L.n_sliced > 0;
    std::vector<int> kept;
    std::vector<char> sl(L.rank, 0);
    for (int s = 0; s < L.n_sliced; ++s) sl[L.sliced_axis[s]] = 1;
    for (int a = 0; a < L.rank; ++a)
      if (!sl[a]) kept.push_back(L.dims[a]);
    std::vector<char> seen(L.perm_rank, 0);
    for (int a = 0; a < L.perm_rank; ++a) {
      require(L.perm[a] >= 0 && L.perm[a] < L.perm_rank && !seen[L.perm[a]],
              STN_ERR_MALFORMED_NETWORK, "leaf perm is not a permutation");
      seen[L.perm[a]] = 1;
      nd.dims.push_back(kept[L.perm[a]]);
    }
    nd.size = 1;
    for (int x : nd.dims) nd.size *= x;
    P->leaf_of_vertex[L.vertex] = i;
  }
  // steps
  P->steps.resize(desc->n_steps);
  for (int i = 0; i < desc->n_steps; ++i) {
    const stn_step_desc &d = desc->steps[i];
    StepPlan &sp = P->steps[i];
    sp.d = d;
    require(d.node >= 0 && d.node < desc->n_nodes && d.lhs >= 0 && d.lhs < desc->n_nodes &&
                d.rhs >= 0 && d.rhs < desc->n_nodes,
            STN_ERR_MALFORMED_NETWORK, "step node id out of range");
    require(d.lrank == d.nd + d.nm + d.nk && d.rrank == d.nd + d.nk + d.nn &&
                d.orank == d.nd + d.nm + d.nn && d.orank <= 64,
            STN_ERR_MALFORMED_NETWORK, "step axis groups inconsistent");
    sp.lperm.assign(d.lperm, d.lperm + d.lrank);
    sp.rperm.assign(d.rperm, d.rperm + d.rrank);
    sp.operm.assign(d.operm, d.operm + d.orank);
    sp.out_dims.assign(d.out_dims, d.out_dims + d.orank);
    sp.d.lperm = sp.d.rperm = sp.d.operm = sp.d.out_dims = nullptr;
    Node &nd = P->nodes[d.node];
    require(!nd.is_leaf && nd.step < 0, STN_ERR_MALFORMED_NETWORK, "node produced twice");
    nd.step = i;
    nd.dims = sp.out_dims;
    nd.size = 1;
    for (int x : nd.dims) nd.size *= x;
  }
  // consumers, operand shapes and per-step geometry (post-order: children first)
  P->leaf_feeds_branch.assign(nl, 0);
  for (int i = 0; i < desc->n_steps; ++i) {
    StepPlan &sp = P->steps[i];
    const stn_step_desc &d = sp.d;
    for (int c : {d.lhs, d.rhs}) {
      Node &cn = P->nodes[c];
      require(cn.is_leaf || (cn.step >= 0 && cn.step < i), STN_ERR_MALFORMED_NETWORK,
              "steps are not in post-order");
      require(cn.consumer < 0, STN_ERR_MALFORMED_NETWORK, "node consumed twice");
      cn.consumer = i;
      if (cn.is_leaf && d.is_branch) P->leaf_feeds_branch[cn.leaf] = 1;
    }
    const std::vector<int> &ld = P->nodes[d.lhs].dims, &rd = P->nodes[d.rhs].dims;
    require(int(ld.size()) == d.lrank && int(rd.size()) == d.rrank, STN_ERR_MALFORMED_NETWORK,
            "operand rank mismatch at node " + std::to_string(d.node));
    sp.lsize = P->nodes[d.lhs].size;
    sp.rsize = P->nodes[d.rhs].size;
    sp.osize = P->nodes[d.node].size;
    // group dims must agree with the recorded D, M, N, K
    int64_t D = 1, M = 1, N = 1, K = 1;
    for (int q = 0; q < d.nd; ++q) D *= ld[sp.lperm[q]];
    for (int q = 0; q < d.nm; ++q) M *= ld[sp.lperm[d.nd + q]];
    for (int q = 0; q < d.nk; ++q) K *= ld[sp.lperm[d.nd + d.nm + q]];
    for (int q = 0; q < d.nn; ++q) N *= rd[sp.rperm[d.nd + d.nk + q]];
    require(D == d.D && M == d.M && N == d.N && K == d.K && sp.osize == D * M * N,
            STN_ERR_MALFORMED_NETWORK, "step shape inconsistent at node " + std::to_string(d.node));
    const auto t_ck = std::chrono::steady_clock::now();
    choose_kernel(*P, sp, ld, rd);
    choose_ms[int(sp.kern)] +=
        std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - t_ck).count();
    if (stn::debug_opt("plan_dump") && !d.is_branch && sp.osize + sp.lsize + sp.rsize >= (1 << 20))
      dump_step(sp, i);
  }
  // root
  {
    const Node &r = P->nodes[P->root];
    require(r.is_leaf || r.step >= 0, STN_ERR_MALFORMED_NETWORK, "root is neither leaf nor step");
    P->out_dims = r.dims;
    P->out_elements = r.size;
  }
  // constant (unsliced) leaves and sliced-leaf values
  int64_t coff = 0, soff = 0;
  for (int i = 0; i < nl; ++i) {
    int node = desc->leaves[i].node;
    const Node &nd = P->nodes[node];
    if (nd.sliced_leaf) {
      P->sliced_val_off[node] = soff;
      int64_t n = 1;
      for (int a = 0; a < desc->leaves[i].rank; ++a) n *= desc->leaves[i].dims[a];
      soff += n;
    } else {
      P->const_off[node] = coff;
      coff += (nd.size + 7) / 8 * 8;
    }
  }
  P->consts_elems = std::max<int64_t>(coff, 1);
  const auto t_up0 = std::chrono::steady_clock::now();
  upload_consts(*P);
  upload_sliced_values(*P);
  const auto t_up1 = std::chrono::steady_clock::now();
  // branch outputs that survive the cache build (runtime.hpp:473-487)
  {
    std::vector<char> needed(desc->n_nodes, 0);
    for (auto &sp : P->steps)
      if (!sp.d.is_branch) needed[sp.d.lhs] = needed[sp.d.rhs] = 1;
    needed[P->root] = 1;
    int64_t off = 0;
    for (auto &sp : P->steps)
      if (sp.d.is_branch && needed[sp.d.node]) {
        P->cache_off[sp.d.node] = off;
        off += (sp.osize + 63) / 64 * 64;
      }
    P->cache_elems = off;
  }
  const auto t_steps = std::chrono::steady_clock::now();
  plan_sweeps(*P);
  build_program(*P, P->build, 0);
  build_program(*P, P->with_cache, 1);
  build_program(*P, P->no_cache, 2);
  if (stn::debug_opt("plan_timing")) {
    const auto t_end = std::chrono::steady_clock::now();
    auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
    fprintf(stderr, "plan create: steps+leaves %.2f ms, programs %.2f ms\n", ms(t_begin, t_steps),
            ms(t_steps, t_end));
    fprintf(stderr, "  device query %.2f ms, leaf/const uploads %.2f ms\n", ms(t_begin, t_dev),
            ms(t_up0, t_up1));
    fprintf(stderr, "  choose_kernel ms by kind:");
    for (int k = 0; k < 16; ++k)
      if (choose_ms[k] > 0.05) fprintf(stderr, " %d:%.2f", k, choose_ms[k]);
    fprintf(stderr, "\n");
  }
}

// ---------------------------------------------------------------------------
// execution
// ---------------------------------------------------------------------------
// ---- per-launch profiling ----
cudaEvent_t take_event(stn_plan &P) {
  if (!P.event_pool.empty()) {
    cudaEvent_t e = P.event_pool.back();
    P.event_pool.pop_back();
    return e;
  }
  cudaEvent_t e;
  cuda_check(cudaEventCreate(&e), "cudaEventCreate");
  return e;
}

struct ProfScope {
  stn_plan &P;
  cudaStream_t st;
  int step;
  cudaEvent_t e0 = nullptr;
  ProfScope(stn_plan &p, cudaStream_t s, int step_index = -1) : P(p), st(s), step(step_index) {
    if (P.profiling) {
      e0 = take_event(P);
      cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
    }
  }
  void done(int kind, double bytes, double flops) {
    P.kernel_launches++;
    if (!P.profiling) return;
    cudaEvent_t e1 = take_event(P);
    cuda_check(cudaEventRecord(e1, st), "cudaEventRecord");
    P.pending.push_back({kind, step, bytes, flops, e0, e1});
    e0 = take_event(P);
    cuda_check(cudaEventRecord(e0, st), "cudaEventRecord");
  }
  ~ProfScope() {
    if (e0) P.event_pool.push_back(e0);
  }
};

void collect_profile(stn_plan &P) {
  for (auto &p : P.pending) {
    cuda_check(cudaEventSynchronize(p.e1), "cudaEventSynchronize");
    float ms = 0;
    cuda_check(cudaEventElapsedTime(&ms, p.e0, p.e1), "cudaEventElapsedTime");
    stn_kernel_profile &t = P.totals[p.kind];
    t.kind = p.kind;
    t.launches++;
    t.ms += ms;
    t.bytes += p.bytes;
    t.flops += p.flops;
    if (p.step >= 0) {
      stn_step_profile &sp = P.step_totals[p.step];
      const StepPlan &stp = P.steps[p.step];
      sp.step = p.step;
      if (p.kind != STN_KERNEL_PERMUTE || sp.launches == 0) sp.kind = p.kind;
      sp.M = stp.d.M;
      sp.N = stp.d.N;
      sp.K = stp.d.K;
      sp.launches++;
      sp.ms += ms;
      sp.bytes += p.bytes;
      sp.flops += p.flops;
    }
    P.event_pool.push_back(p.e0);
    P.event_pool.push_back(p.e1);
  }
  P.pending.clear();
}

void *elem_ptr(const stn_plan &P, void *base, int64_t elems) {
  return static_cast<unsigned char *>(base) + size_t(elems) * P.esize;
}

struct Resolved {
  const void *ptr;
  int64_t bs;
};

Resolved resolve(stn_plan &P, const Ref &r, const stn_cache *cache, int nb) {
  switch (r.kind) {
    case Src::ConstLeaf:
      return {elem_ptr(P, P.consts.ptr, r.off), 0};
    case Src::Cache:
    case Src::Persist:
      return {elem_ptr(P, cache->storage.ptr, r.off), 0};
    case Src::Arena:
    case Src::SliceLeaf:
      return {elem_ptr(P, P.cur->arena.ptr, r.off * nb), r.size};
  }
  return {nullptr, 0};
}

void launch_chain_op(stn_plan &P, const Op &op, const stn_cache *cache, int nb, cudaStream_t st) {
  const stn_plan::Sweep &sw = P.sweeps[op.sweep];
  stn::ChainGeom g = sw.cgeom;
  Resolved x = resolve(P, op.a, cache, nb), o = resolve(P, op.out, cache, nb);
  double bytes = 8.0 * (x.bs ? nb : 1) * op.a.size + 8.0 * nb * op.out.size, flops = 0;
  for (size_t j = 0; j < op.wrefs.size(); ++j) {
    Resolved w = resolve(P, op.wrefs[j], cache, nb);
    g.w[j] = w.ptr;
    g.w_bs[j] = w.bs;
    bytes += 8.0 * (w.bs ? nb : 1) * op.wrefs[j].size;
  }
  for (int stp : sw.steps) flops += 8.0 * double(P.steps[stp].d.mults) * nb;
  stn::BatchPtrs p{x.ptr, nullptr, const_cast<void *>(o.ptr), x.bs, 0, o.bs, nb};
  if (sw.jit_fn && sw.jit_alt && sw.jit_pick == 0) {
    // first run outside a capture: time both variants (they write the same output, bit for
    // bit) and keep the faster one for every later launch and graph capture
    cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
    cuda_check(cudaStreamIsCapturing(st, &cs), "capture status");
    if (cs == cudaStreamCaptureStatusNone) {
      cudaEvent_t ev[3];
      for (auto &e : ev) cuda_check(cudaEventCreate(&e), "event");
      float ms[2] = {0, 0};
      cuda_check(cudaEventRecord(ev[0], st), "event");
      cuda_check(stn::chain_jit_launch(sw.jit_fn, g, sw.tables->as<stn::ChainTables>(), p, st),
                 "fused stem chain kernel (specialised)");
      cuda_check(cudaEventRecord(ev[1], st), "event");
      cuda_check(stn::chain_jit_launch(sw.jit_alt, g, sw.tables->as<stn::ChainTables>(), p, st),
                 "fused stem chain kernel (specialised, 128 registers)");
      cuda_check(cudaEventRecord(ev[2], st), "event");
      cuda_check(cudaEventSynchronize(ev[2]), "event sync");
      cudaEventElapsedTime(&ms[0], ev[0], ev[1]);
      cudaEventElapsedTime(&ms[1], ev[1], ev[2]);
      for (auto &e : ev) cudaEventDestroy(e);
      sw.jit_pick = ms[1] < 0.97f * ms[0] ? 2 : 1;
      if (stn::debug_opt("sweep_debug"))
        fprintf(stderr, "chain from step %d: %.3f ms, 128-register variant %.3f ms -> %s\n",
                sw.steps.front(), ms[0], ms[1], sw.jit_pick == 2 ? "variant" : "primary");
      P.kernel_launches++;
      return;
    }
  }
  ProfScope prof(P, st, sw.steps.front());
  if (sw.jit_fn)
    cuda_check(stn::chain_jit_launch(sw.jit_pick == 2 ? sw.jit_alt : sw.jit_fn, g,
                                     sw.tables->as<stn::ChainTables>(), p, st),
               "fused stem chain kernel (specialised)");
  else if (g.ma > stn::kChainTableLog)
    fail(STN_ERR_CUDA, "fused stem chain planned for the specialised kernel has none");
  else
    cuda_check(stn::launch_chain(sw.tables->as<stn::ChainTables>(), g, p,
                                 P.mode == STN_MODE_EXACT, st),
               "fused stem chain kernel");
  prof.done(STN_KERNEL_SWEEP, bytes, flops);
}

void launch_sweep_op(stn_plan &P, const Op &op, const stn_cache *cache, int nb, cudaStream_t st) {
  if (P.sweeps[op.sweep].chain) return launch_chain_op(P, op, cache, nb, st);
  const stn_plan::Sweep &sw = P.sweeps[op.sweep];
  stn::SweepGeom g = sw.geom;
  Resolved x = resolve(P, op.a, cache, nb), o = resolve(P, op.out, cache, nb);
  double bytes = 8.0 * (x.bs ? nb : 1) * op.a.size + 8.0 * nb * op.out.size, flops = 0;
  for (size_t j = 0; j < op.wrefs.size(); ++j) {
    Resolved w = resolve(P, op.wrefs[j], cache, nb);
    g.w[j] = w.ptr;
    g.w_bs[j] = w.bs;
    bytes += 8.0 * (w.bs ? nb : 1) * op.wrefs[j].size;
  }
  for (int stp : sw.steps) flops += 8.0 * double(P.steps[stp].d.mults) * nb;
  ProfScope prof(P, st, sw.steps.front());
  stn::BatchPtrs p{x.ptr, nullptr, const_cast<void *>(o.ptr), x.bs, 0, o.bs, nb};
  cuda_check(stn::launch_sweep(g, p, P.mode == STN_MODE_EXACT, st), "stem sweep kernel");
  prof.done(STN_KERNEL_SWEEP, bytes, flops);
}

template <class R>
void launch_op(stn_plan &P, const Op &op, const stn_cache *cache, int nb, cudaStream_t st) {
  if (op.sweep >= 0) return launch_sweep_op(P, op, cache, nb, st);
  const StepPlan &sp = P.steps[op.step];
  Resolved a = resolve(P, op.a, cache, nb), b = resolve(P, op.b, cache, nb);
  Resolved o = resolve(P, op.out, cache, nb);
  void *out = const_cast<void *>(o.ptr);
  const bool exact = P.mode == STN_MODE_EXACT;
  const double es = double(P.esize);
  // algorithmic traffic: slice-invariant operands once per batch
  auto reads = [&](const Resolved &r, int64_t size) { return es * size * (r.bs ? nb : 1); };
  const double io_bytes = reads(a, sp.lsize) + reads(b, sp.rsize) + es * sp.osize * nb;
  const double flops = 8.0 * double(sp.d.mults) * nb;
  ProfScope prof(P, st, op.step);
  switch (sp.kern) {
    case Kern::Generic: {
      stn::BatchPtrs p{a.ptr, b.ptr, out, a.bs, b.bs, o.bs, nb};
      cuda_check(stn::launch_generic<R>(sp.geo, p, exact, st), "generic kernel");
      prof.done(STN_KERNEL_GENERIC, io_bytes, flops);
      break;
    }
    case Kern::Outer: {
      stn::BatchPtrs p{a.ptr, b.ptr, out, a.bs, b.bs, o.bs, nb};
      cuda_check(stn::launch_outer<R>(*sp.og, p, exact, st), "outer kernel");
      prof.done(STN_KERNEL_GENERIC, io_bytes, flops);
      break;
    }
    case Kern::SplitK: {
      stn::BatchPtrs p{a.ptr, b.ptr, out, a.bs, b.bs, o.bs, nb};
      P.cur->splitk_ws.reserve(
          std::max<size_t>(stn::splitk_workspace_bytes(sp.geo, sp.dot, nb, P.esize), 16));
      cuda_check(stn::launch_splitk<R>(sp.geo, p, sp.dot, P.cur->splitk_ws.ptr, st),
                 "split-K kernel");
      prof.done(STN_KERNEL_GENERIC, io_bytes, flops);
      P.kernel_launches++;  // second (ordered-sum) launch
      break;
    }
    case Kern::AbsorbTc: {
      const Resolved &x = sp.x_is_lhs ? a : b;
      const Resolved &w = sp.x_is_lhs ? b : a;
      stn::BatchPtrs p{x.ptr, w.ptr, out, x.bs, w.bs, o.bs, nb};
      cuda_check(stn::launch_absorb_tc(sp.agtc, p, st), "tensor-core absorb kernel");
      prof.done(STN_KERNEL_ABSORB_TC, io_bytes, flops);
      break;
    }
    case Kern::AbsorbTma: {
      const Resolved &x = sp.x_is_lhs ? a : b;
      const Resolved &w = sp.x_is_lhs ? b : a;
      stn::BatchPtrs p{x.ptr, w.ptr, out, x.bs, w.bs, o.bs, nb};
      cuda_check(stn::launch_absorb_tma(*sp.tg, p, st), "TMA tensor-core absorb kernel");
      prof.done(STN_KERNEL_ABSORB_TC, io_bytes, flops);
      break;
    }
    case Kern::AbsorbMma: {
      const Resolved &x = sp.x_is_lhs ? a : b;
      const Resolved &w = sp.x_is_lhs ? b : a;
      stn::BatchPtrs p{x.ptr, w.ptr, out, x.bs, w.bs, o.bs, nb};
      cuda_check(stn::launch_absorb_mma(sp.dg, p, st), "tensor-core direct absorb kernel");
      prof.done(STN_KERNEL_ABSORB_TC, io_bytes, flops);
      break;
    }
    case Kern::AbsorbDirect: {
      const Resolved &x = sp.x_is_lhs ? a : b;
      const Resolved &w = sp.x_is_lhs ? b : a;
      stn::BatchPtrs p{x.ptr, w.ptr, out, x.bs, w.bs, o.bs, nb};
      cuda_check(stn::launch_absorb_direct(sp.dg, p, exact, st), "direct absorb kernel");
      prof.done(STN_KERNEL_ABSORB, io_bytes, flops);
      break;
    }
    case Kern::Lanes: {
      const Resolved &x = sp.x_is_lhs ? a : b;
      const Resolved &w = sp.x_is_lhs ? b : a;
      stn::BatchPtrs p{x.ptr, w.ptr, out, x.bs, w.bs, o.bs, nb};
      cuda_check(stn::launch_absorb_lanes(sp.lane_tab->as<stn::LaneTables>(), sp.lg, p, exact, st),
                 "lane absorb kernel");
      prof.done(STN_KERNEL_ABSORB, io_bytes, flops);
      break;
    }
    case Kern::Absorb: {
      const Resolved &x = sp.x_is_lhs ? a : b;
      const Resolved &w = sp.x_is_lhs ? b : a;
      stn::BatchPtrs p{x.ptr, w.ptr, out, x.bs, w.bs, o.bs, nb};
      cuda_check(stn::launch_absorb(sp.ag, p, exact, st), "absorb kernel");
      prof.done(STN_KERNEL_ABSORB, io_bytes, flops);
      break;
    }
    case Kern::GemmSimt:
    case Kern::GemmTc: {
      const Resolved &ra = sp.gemm_swap ? b : a, &rb = sp.gemm_swap ? a : b;
      const int64_t asize = sp.gemm_swap ? sp.rsize : sp.lsize;
      const int64_t bsize = sp.gemm_swap ? sp.lsize : sp.rsize;
      const void *ga = ra.ptr, *gb = rb.ptr;
      int64_t ga_bs = ra.bs, gb_bs = rb.bs;
      // tcgen05 GEMM with a permuted A: the tile permute writes A's TF32 hi / lo planes
      // straight into the GEMM workspace (one pass instead of permute + split)
      const bool a_fused = sp.kern == Kern::GemmTc && !sp.tcf && !sp.a_id && sp.pa_bases &&
                           stn::gemm_tc_supported(sp.gs);
      if (a_fused) {
        stn::BatchPtrs pp{nullptr, rb.ptr, nullptr, asize, rb.bs, 0, nb};
        size_t ws = stn::gemm_tc_workspace_bytes(sp.gs, pp);
        P.cur->tc_workspace.reserve(std::max<size_t>(ws, 16));
        float *hi, *lo;
        stn::gemm_tc_a_planes(sp.gs, pp, P.cur->tc_workspace.ptr, &hi, &lo);
        cuda_check(stn::launch_perm_tiles(sp.pat, sp.pa_bases->as<int64_t>(), ra.ptr, hi, ra.bs,
                                          asize, nb, st, lo),
                   "tile permute + split");
        prof.done(STN_KERNEL_PERMUTE, (es + 2 * es) * asize * nb, 0);
        ga = nullptr;
        ga_bs = asize;
      } else if (sp.skinny_tab || sp.tcf_gather) {
        // gathered by the GEMM itself (skinny SIMT / fused-split tcgen05)
      } else if (!sp.a_id) {
        void *dst = elem_ptr(P, P.cur->arena.ptr, op.scr_a * nb);
        if (sp.pa_bases)
          cuda_check(stn::launch_perm_tiles(sp.pat, sp.pa_bases->as<int64_t>(), ra.ptr, dst,
                                            ra.bs, asize, nb, st),
                     "tile permute");
        else if (sp.pa_tiled)
          cuda_check(stn::launch_bitperm(sp.pag, ra.ptr, dst, ra.bs, asize, nb, st), "bitperm");
        else
          cuda_check(stn::launch_permute<R>(sp.pa, ra.ptr, dst, ra.bs, asize, nb, st), "permute");
        prof.done(STN_KERNEL_PERMUTE, 2 * es * asize * nb, 0);
        ga = dst;
        ga_bs = asize;
      }
      if (!sp.b_id) {
        void *dst = elem_ptr(P, P.cur->arena.ptr, op.scr_b * nb);
        if (sp.pb_bases)
          cuda_check(stn::launch_perm_tiles(sp.pbt, sp.pb_bases->as<int64_t>(), rb.ptr, dst,
                                            rb.bs, bsize, nb, st),
                     "tile permute");
        else if (sp.pb_tiled)
          cuda_check(stn::launch_bitperm(sp.pbg, rb.ptr, dst, rb.bs, bsize, nb, st), "bitperm");
        else
          cuda_check(stn::launch_permute<R>(sp.pb, rb.ptr, dst, rb.bs, bsize, nb, st), "permute");
        prof.done(STN_KERNEL_PERMUTE, 2 * es * bsize * nb, 0);
        gb = dst;
        gb_bs = bsize;
      }
      void *gc = sp.c_id ? out : elem_ptr(P, P.cur->arena.ptr, op.scr_c * nb);
      int64_t gc_bs = sp.c_id ? o.bs : sp.osize;
      stn::BatchPtrs p{ga, gb, gc, ga_bs, gb_bs, gc_bs, nb};
      const double gbytes = es * (asize * (ga_bs ? nb : 1) + bsize * (gb_bs ? nb : 1) +
                                  double(sp.osize) * nb);
      bool done = false;
      if (sp.kern == Kern::GemmTc && sp.tcf) {
        const size_t ws = stn::gemm_tcf_workspace_bytes(sp.gs, p);
        P.cur->tc_workspace.reserve(std::max<size_t>(ws, 16));
        stn::TcfGather tg{};
        if (sp.tcf_gather) {
          const int64_t *t = sp.tcf_gather->as<int64_t>();
          tg = {t, t + 128, t + 128 + sp.gs.M / 128};
          p.a = ra.ptr;  // the stem itself
          p.a_bs = ra.bs;
        }
        cuda_check(stn::launch_gemm_tcf(sp.gs, p, P.cur->tc_workspace.ptr, ws, st,
                                        sp.tcf_gather ? &tg : nullptr),
                   "tcgen05 fused-split gemm");
        prof.done(STN_KERNEL_GEMM_TC, gbytes, flops);
        done = true;
      }
      if (sp.kern == Kern::GemmTc && !done) {
        size_t ws = stn::gemm_tc_workspace_bytes(sp.gs, p);
        P.cur->tc_workspace.reserve(std::max<size_t>(ws, 16));
        cudaError_t e =
            stn::launch_gemm_tc(sp.gs, p, P.cur->tc_workspace.ptr, ws, st, nullptr, a_fused);
        require(!a_fused || e == cudaSuccess, STN_ERR_CUDA,
                std::string("tcgen05 gemm (pre-split A): ") + cudaGetErrorString(e));
        if (e == cudaSuccess) {
          done = true;
          prof.done(STN_KERNEL_GEMM_TC, gbytes, flops);
        } else {
          require(e == cudaErrorNotSupported, STN_ERR_CUDA,
                  std::string("tcgen05 gemm: ") + cudaGetErrorString(e));
          cudaGetLastError();
        }
      }
      if (!done && sp.skinny_tab) {
        cuda_check(stn::launch_gemm_skinny_gather(sp.gs, p, sp.skinny_tab->as<int64_t>(),
                                                  sp.skinny_mbits, st),
                   "skinny gemm");
        prof.done(STN_KERNEL_GEMM_SIMT, gbytes, flops);
        done = true;
      }
      if (!done) {
        cuda_check(stn::launch_gemm_simt<R>(sp.gs, p, exact, st), "gemm kernel");
        prof.done(STN_KERNEL_GEMM_SIMT, gbytes, flops);
      }
      if (!sp.c_id) {
        if (sp.pc_bases)
          cuda_check(stn::launch_perm_tiles(sp.pct, sp.pc_bases->as<int64_t>(), gc, out, sp.osize,
                                            o.bs, nb, st),
                     "tile permute");
        else if (sp.pc_tiled)
          cuda_check(stn::launch_bitperm(sp.pcg, gc, out, sp.osize, o.bs, nb, st), "bitperm");
        else
          cuda_check(stn::launch_permute<R>(sp.pc, gc, out, sp.osize, o.bs, nb, st), "permute");
        prof.done(STN_KERNEL_PERMUTE, 2 * es * sp.osize * nb, 0);
      }
      break;
    }
  }
}

int auto_batch(const stn_plan &P, const Program &prog) {
  const int64_t per = std::max<int64_t>(prog.arena_elems, 1) * int64_t(P.esize);
  int64_t nb = P.max_batch > 0 ? int64_t(P.max_batch)
                               : (int64_t(256) << 20) / per;  // aim for >= 256 MiB per pass
  // batched launches put D x nbatch in gridDim.z (<= 65535)
  int64_t max_d = 1;
  for (const StepPlan &sp : P.steps) max_d = std::max<int64_t>(max_d, sp.gs.D);
  return int(std::max<int64_t>(1, std::min<int64_t>({nb, 256, 65535 / max_d})));
}

// Lane `i` of the plan (created on first use; lane 0 runs on the caller's stream).
ExecCtx *get_lane(stn_plan &P, int i, cudaStream_t caller) {
  while (int(P.lanes.size()) <= i) P.lanes.push_back(std::make_unique<ExecCtx>());
  ExecCtx &c = *P.lanes[size_t(i)];
  if (i == 0) {
    c.st = caller;
  } else if (!c.st) {
    cuda_check(cudaStreamCreateWithFlags(&c.st, cudaStreamNonBlocking), "lane stream");
    c.own_stream = true;
  }
  if (!c.done) cuda_check(cudaEventCreateWithFlags(&c.done, cudaEventDisableTiming), "lane event");
  return &c;
}

// The device work of one batch of `n` slices on lane P.cur (digits already on the
// device): leaf gather, every step, root accumulation. Captured as-is into graphs.
void batch_kernels(stn_plan &P, Program &prog, const stn_cache *cache, int n, cudaStream_t st,
                   double *acc, double *per_slice) {
  ExecCtx &L = *P.cur;
  if (!prog.slice_leaves.empty()) {
    ProfScope prof(P, st);
    if (P.precision == STN_SINGLE)
      cuda_check(stn::launch_leaf_gather<float>(prog.table, L.arena.ptr, L.digits.as<int32_t>(),
                                                n, st),
                 "leaf gather");
    else
      cuda_check(stn::launch_leaf_gather<double>(prog.table, L.arena.ptr, L.digits.as<int32_t>(),
                                                 n, st),
                 "leaf gather");
    prof.done(STN_KERNEL_LEAF, double(prog.table.total_out) * n * (16 + P.esize), 0);
  }
  // side stream: small independent steps overlap the stem steps (not while profiling,
  // which times every step on one stream)
  const bool two = prog.has_side && !P.profiling;
  if (two) {
    if (!L.side) cuda_check(cudaStreamCreateWithFlags(&L.side, cudaStreamNonBlocking), "side stream");
    for (cudaEvent_t *e : {&L.fork, &L.join})
      if (!*e) cuda_check(cudaEventCreateWithFlags(e, cudaEventDisableTiming), "side event");
    if (L.op_ev.size() < prog.ops.size()) L.op_ev.resize(prog.ops.size(), nullptr);
    for (size_t k = 0; k < prog.ops.size(); ++k)
      if (prog.need_event[k] && !L.op_ev[k])
        cuda_check(cudaEventCreateWithFlags(&L.op_ev[k], cudaEventDisableTiming), "op event");
    cuda_check(cudaEventRecord(L.fork, st), "fork");
    cuda_check(cudaStreamWaitEvent(L.side, L.fork, 0), "fork wait");
  }
  for (size_t k = 0; k < prog.ops.size(); ++k) {
    const Op &op = prog.ops[k];
    cudaStream_t s = two && prog.side[k] ? L.side : st;
    if (two && prog.wait_other[k] >= 0)
      cuda_check(cudaStreamWaitEvent(s, L.op_ev[size_t(prog.wait_other[k])], 0), "op wait");
    if (P.precision == STN_SINGLE)
      launch_op<float>(P, op, cache, n, s);
    else
      launch_op<double>(P, op, cache, n, s);
    if (two && prog.need_event[k]) cuda_check(cudaEventRecord(L.op_ev[k], s), "op event");
  }
  if (two) {
    cuda_check(cudaEventRecord(L.join, L.side), "join");
    cuda_check(cudaStreamWaitEvent(st, L.join, 0), "join wait");
  }
  if (prog.has_root && (acc || per_slice)) {
    ProfScope prof(P, st);
    Resolved r = resolve(P, prog.root, cache, n);
    if (P.precision == STN_SINGLE)
      cuda_check(stn::launch_root_accumulate<float>(r.ptr, r.bs, P.out_elements, n, acc,
                                                    per_slice, st),
                 "root accumulate");
    else
      cuda_check(stn::launch_root_accumulate<double>(r.ptr, r.bs, P.out_elements, n, acc,
                                                     per_slice, st),
                 "root accumulate");
    prof.done(STN_KERNEL_ROOT, double(P.out_elements) * n * (P.esize + 16), 0);
  }
}

// Runs `n` slices (digits row-major n x n_sliced on the host) of `prog` on lane
// P.cur's buffers, on stream `st`.
void run_batch(stn_plan &P, Program &prog, const stn_cache *cache, const int32_t *digits_host,
               int n, cudaStream_t st, double *acc, double *per_slice) {
  ExecCtx &L = *P.cur;
  const size_t arena_bytes = size_t(std::max<int64_t>(prog.arena_elems, 1)) * n * P.esize;
  L.arena.reserve(arena_bytes);
  const int ns = int(P.sliced_dims.size());
  if (ns > 0 && !prog.slice_leaves.empty()) {
    L.digits.reserve(size_t(n) * ns * 4);
    cuda_check(cudaMemcpyAsync(L.digits.ptr, digits_host, size_t(n) * ns * 4,
                               cudaMemcpyHostToDevice, st),
               "digits upload");
  }
  batch_kernels(P, prog, cache, n, st, acc, per_slice);
}

// Same batch through the lane's CUDA graph (one launch for the whole per-slice program
// of a full batch; the roots go to the lane's staging rows). Captured on first use and
// whenever what it was captured for changed; any capture problem turns graphs off for
// the plan and the batch runs eagerly.
void run_batch_graph(stn_plan &P, Program &prog, const stn_cache *cache,
                     const int32_t *digits_host, int n, cudaStream_t st) {
  ExecCtx &L = *P.cur;
  const size_t arena_bytes = size_t(std::max<int64_t>(prog.arena_elems, 1)) * n * P.esize;
  L.arena.reserve(arena_bytes);
  L.rows.reserve(16 * size_t(P.out_elements) * size_t(n));
  const int ns = int(P.sliced_dims.size());
  if (ns > 0 && !prog.slice_leaves.empty()) {
    L.digits.reserve(size_t(n) * ns * 4);
    cuda_check(cudaMemcpyAsync(L.digits.ptr, digits_host, size_t(n) * ns * 4,
                               cudaMemcpyHostToDevice, st),
               "digits upload");
  }
  const void *cstore = cache ? cache->storage.ptr : nullptr;
  const bool fresh = L.graph && L.g_prog == &prog && L.g_cache == cstore &&
                     L.g_arena == L.arena.ptr && L.g_rows == L.rows.ptr && L.g_nb == n &&
                     L.g_epoch == P.graph_epoch;
  if (!fresh && !(L.w_prog == &prog && L.w_nb == n && L.w_epoch == P.graph_epoch)) {
    // first full batch of this program on this lane: eager, so every workspace the
    // launches reserve exists before a capture (no allocation inside a graph)
    batch_kernels(P, prog, cache, n, st, nullptr, L.rows.as<double>());
    L.w_prog = &prog;
    L.w_nb = n;
    L.w_epoch = P.graph_epoch;
    return;
  }
  if (!fresh && P.graphs) {
    if (L.graph) {
      cudaGraphExecDestroy(L.graph);
      L.graph = nullptr;
    }
    cudaGraph_t g = nullptr;
    bool ok = cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal) == cudaSuccess;
    if (ok) {
      const int launches = P.kernel_launches;
      try {
        batch_kernels(P, prog, cache, n, st, nullptr, L.rows.as<double>());
      } catch (const Failure &) {
        ok = false;
      }
      P.kernel_launches = launches;
      ok = cudaStreamEndCapture(st, &g) == cudaSuccess && ok;
    }
    if (ok) ok = cudaGraphInstantiate(&L.graph, g, 0) == cudaSuccess;
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    if (!ok) {
      L.graph = nullptr;
      P.graphs = false;  // eager from now on
    } else {
      L.g_prog = &prog;
      L.g_cache = cstore;
      L.g_arena = L.arena.ptr;
      L.g_rows = L.rows.ptr;
      L.g_nb = n;
      L.g_epoch = P.graph_epoch;
    }
  }
  if (L.graph) {
    cuda_check(cudaGraphLaunch(L.graph, st), "graph launch");
    P.kernel_launches += int(prog.ops.size()) + 2;
  } else {
    batch_kernels(P, prog, cache, n, st, nullptr, L.rows.as<double>());
  }
}

void decode(const stn_plan &P, uint64_t a, int32_t *digits) {
  uint64_t rest = a;
  for (size_t i = P.sliced_dims.size(); i-- > 0;) {
    uint64_t d = uint64_t(P.sliced_dims[i]);
    digits[i] = int32_t(rest % d);
    rest /= d;
  }
}

void check_cache(const stn_plan &P, const stn_cache *cache) {
  if (!cache) return;
  require(cache->identity == P.identity && cache->plan == &P, STN_ERR_SUBTASK_FAILURE,
          "branch cache belongs to a different plan");
  require(cache->leaf_epoch == P.leaf_epoch, STN_ERR_SUBTASK_FAILURE,
          "branch cache is stale: leaf values feeding branch steps changed");
}

// Runs slices given by a digit generator over [0, n) in batches. With one lane and
// no graph this is the plain sequence: per batch, digits upload + kernels, roots
// accumulated into `acc` in ascending slice order. With `lanes` > 1 (and/or graphs)
// batches rotate over lanes, each on its own stream and arena, so the small
// launch-bound steps of one batch overlap the HBM-bound stem steps of another; a
// batch's roots land in its lane's staging rows, are copied to `per_slice`, and are
// folded into `acc` after the previous batch's fold (an event chain), so the sum
// keeps the reference's ascending order bit for bit (runtime.hpp:601-605).
template <class DigitsOf>
void run_slices_impl(stn_plan &P, const stn_cache *cache, uint64_t n, DigitsOf &&digits_of,
                     cudaStream_t st, double *acc, double *per_slice,
                     std::vector<double> *batch_ms = nullptr, int lanes = 1) {
  Program &prog = cache ? P.with_cache : P.no_cache;
  const int ns = int(P.sliced_dims.size());
  const int nb = auto_batch(P, prog);
  const uint64_t n_batches = (n + uint64_t(nb) - 1) / uint64_t(nb);
  // lanes: bounded by the batches and by free device memory for their arenas
  int par = int(std::max<uint64_t>(1, std::min<uint64_t>(uint64_t(std::max(lanes, 1)), n_batches)));
  if (par > 1) {
    size_t free_b = 0, total_b = 0;
    cudaMemGetInfo(&free_b, &total_b);
    const size_t per = size_t(std::max<int64_t>(prog.arena_elems, 1)) * nb * P.esize;
    int have = 0;
    for (auto &l : P.lanes) have += l->arena.bytes >= per ? 1 : 0;
    const size_t room = free_b > (size_t(2) << 30) ? free_b - (size_t(2) << 30) : 0;
    par = std::max(1, std::min(par, have + int(room / std::max<size_t>(per, 1))));
  }
  const bool staged = par > 1 || (P.graphs && !P.profiling && !batch_ms);
  std::vector<int32_t> dig;
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  if (batch_ms) {
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
  }
  ExecCtx *lv[64];
  par = std::min(par, 64);
  for (int i = 0; i < par; ++i) lv[i] = get_lane(P, i, st);
  cudaEvent_t start = nullptr, fold_done = nullptr;
  if (par > 1) {  // the lanes start after the work already queued on the caller's stream
    start = lv[0]->done;
    cuda_check(cudaEventRecord(start, st), "event");
    for (int i = 1; i < par; ++i) cuda_check(cudaStreamWaitEvent(lv[i]->st, start), "wait");
  }
  const size_t row = 2 * size_t(P.out_elements);
  for (uint64_t b = 0; b < n_batches; ++b) {
    const uint64_t a0 = b * uint64_t(nb);
    const int cnt = int(std::min<uint64_t>(uint64_t(nb), n - a0));
    ExecCtx &C = *lv[b % uint64_t(par)];
    P.cur = &C;
    dig.assign(size_t(cnt) * std::max(ns, 1), 0);
    for (int i = 0; i < cnt; ++i) digits_of(a0 + i, dig.data() + size_t(i) * ns);
    if (batch_ms) cuda_check(cudaEventRecord(e0, C.st), "event");
    double *ps = per_slice ? per_slice + row * a0 : nullptr;
    if (!staged) {
      run_batch(P, prog, cache, dig.data(), cnt, C.st, acc, ps);
    } else {
      if (cnt == nb && P.graphs && !P.profiling)
        run_batch_graph(P, prog, cache, dig.data(), cnt, C.st);
      else {
        C.rows.reserve(8 * row * size_t(nb));
        run_batch(P, prog, cache, dig.data(), cnt, C.st, nullptr, C.rows.as<double>());
      }
      if (ps)
        cuda_check(cudaMemcpyAsync(ps, C.rows.ptr, 8 * row * size_t(cnt),
                                   cudaMemcpyDeviceToDevice, C.st),
                   "per-slice copy");
      if (acc) {
        if (fold_done) cuda_check(cudaStreamWaitEvent(C.st, fold_done), "wait");
        cuda_check(stn::launch_sum_ordered(C.rows.as<double>(), uint64_t(cnt), P.out_elements,
                                           acc, C.st, true),
                   "ordered fold");
        P.kernel_launches++;
      }
      cuda_check(cudaEventRecord(C.done, C.st), "event");
      fold_done = C.done;
    }
    if (batch_ms) {
      cuda_check(cudaEventRecord(e1, C.st), "event");
      cuda_check(cudaEventSynchronize(e1), "event sync");
      float ms = 0;
      cuda_check(cudaEventElapsedTime(&ms, e0, e1), "event time");
      for (int i = 0; i < cnt; ++i) batch_ms->push_back(double(ms) / cnt);
    }
  }
  if (par > 1)  // join: the caller's stream waits for every lane
    for (int i = 1; i < par; ++i) {
      cuda_check(cudaEventRecord(lv[i]->done, lv[i]->st), "event");
      cuda_check(cudaStreamWaitEvent(st, lv[i]->done), "wait");
    }
  P.cur = P.lanes[0].get();
  if (e0) cudaEventDestroy(e0);
  if (e1) cudaEventDestroy(e1);
}

void build_cache(stn_plan &P, cudaStream_t st, stn_cache *c) {
  c->device = P.device;
  c->identity = P.identity;
  c->leaf_epoch = P.leaf_epoch;
  c->plan = &P;
  c->storage.reserve(size_t(std::max<int64_t>(P.cache_elems, 1)) * P.esize);
  P.cur = get_lane(P, 0, st);
  for (auto &sp : P.steps)
    if (sp.d.is_branch) c->mults += sp.d.mults;
  for (auto &[node, off] : P.cache_off) c->elements += uint64_t(P.nodes[node].size);
  run_batch(P, P.build, c, nullptr, 1, st, nullptr, nullptr);
}

void run_one(stn_plan &P, const int32_t *digits, const stn_cache *cache, cudaStream_t st,
             double *out_host, stn_subtask_info *info) {
  check_cache(P, cache);
  Program &prog = cache ? P.with_cache : P.no_cache;
  P.cur = get_lane(P, 0, st);
  P.scratch_out.reserve(16 * size_t(P.out_elements));
  std::vector<int32_t> dig(digits, digits + P.sliced_dims.size());
  if (dig.empty()) dig.push_back(0);
  run_batch(P, prog, cache, dig.data(), 1, st, nullptr, P.scratch_out.as<double>());
  cuda_check(cudaMemcpyAsync(out_host, P.scratch_out.ptr, 16 * size_t(P.out_elements),
                             cudaMemcpyDeviceToHost, st),
             "result download");
  cuda_check(cudaStreamSynchronize(st), "stream sync");
  if (info) {
    info->step_count = int32_t(prog.n_steps);
    info->mults = prog.mults;
    info->peak_elements = prog.peak;
  }
}

}  // namespace

// ---------------------------------------------------------------------------
// C ABI
// ---------------------------------------------------------------------------
extern "C" {

void stn_set_error_c(const char *msg) { g_last_error = msg ? msg : ""; }

const char *stn_version(void) { return "stn_exec 0.1 (sm_100a)"; }
int stn_abi_version(void) { return STN_ABI_VERSION; }
const char *stn_last_error(void) { return g_last_error.c_str(); }

const char *stn_status_name(int status) {
  static const char *kinds[] = {"MalformedNetwork", "CapExceeded",       "OpenEdgeSliced",
                                "IndexOutOfRange",  "MissingParams",     "SyntaxError",
                                "InvariantViolation", "QubitCoverage",   "LayoutTooSmall",
                                "Infeasible",       "EdgeNotFound",      "SchemaError",
                                "Stuck",            "HashMismatch",      "WidthExceedsBudget",
                                "SubtaskFailure",   "MissingResult",     "ChecksumMismatch",
                                "EmptySamples"};
  if (status == 0) return "Ok";
  if (status >= 1 && status <= 19) return kinds[status - 1];
  switch (status) {
    case STN_ERR_CUDA: return "CudaError";
    case STN_ERR_INVALID_ARGUMENT: return "InvalidArgument";
    case STN_ERR_OUT_OF_MEMORY: return "OutOfMemory";
    case STN_ERR_NO_DEVICE: return "NoDevice";
    case STN_ERR_IO: return "IOError";
  }
  return "Unknown";
}

int stn_plan_create(const stn_plan_desc *desc, int device, int mode, stn_plan **out) {
  if (!out) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL output pointer");
  *out = nullptr;
  auto P = std::make_unique<stn_plan>();
  int st = guarded([&] { create_plan(desc, device, mode, P.get()); });
  if (st == STN_OK) *out = P.release();
  return st;
}

int stn_plan_destroy(stn_plan *plan) {
  if (plan) {
    cudaSetDevice(plan->device);
    delete plan;
  }
  return STN_OK;
}

int stn_plan_get_info(const stn_plan *P, stn_plan_info *info) {
  if (!P || !info) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  memset(info, 0, sizeof *info);
  info->identity = P->identity;
  info->subtasks = P->subtasks;
  info->n_sliced = int32_t(P->sliced_dims.size());
  info->out_rank = int32_t(P->out_dims.size());
  info->out_elements = P->out_elements;
  for (size_t i = 0; i < P->out_dims.size() && i < 64; ++i) info->out_dims[i] = P->out_dims[i];
  info->per_slice_steps = int32_t(P->with_cache.n_steps);
  info->per_slice_mults = P->with_cache.mults;
  for (auto &sp : P->steps)
    if (sp.d.is_branch) info->branch_mults += sp.d.mults;
  info->peak_elements = P->with_cache.peak;
  info->arena_bytes_per_slice = uint64_t(P->with_cache.arena_elems) * P->esize;
  info->cache_bytes = uint64_t(P->cache_elems) * P->esize;
  for (auto &op : P->with_cache.ops) {
    if (op.sweep >= 0) {
      info->sweeps++;
      info->steps_in_sweeps += int32_t(P->sweeps[op.sweep].steps.size());
      continue;
    }
    Kern k = P->steps[op.step].kern;
    if (k == Kern::GemmTc) info->steps_tensor_core++;
    else if (k == Kern::GemmSimt) info->steps_generic++;
    else if (k == Kern::Absorb || k == Kern::AbsorbTc || k == Kern::AbsorbDirect ||
             k == Kern::AbsorbMma || k == Kern::AbsorbTma || k == Kern::Lanes)
      info->steps_absorb++;
    else info->steps_generic++;
  }
  return STN_OK;
}

int stn_plan_set_leaf_values(stn_plan *P, int32_t vertex, const double *values, int64_t n) {
  if (!P || !values) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    auto it = P->leaf_of_vertex.find(vertex);
    require(it != P->leaf_of_vertex.end(), STN_ERR_INDEX_OUT_OF_RANGE,
            "vertex " + std::to_string(vertex) + " is not a leaf of this plan");
    const int li = it->second;
    require(int64_t(P->leaf_values[li].size()) == 2 * n, STN_ERR_MALFORMED_NETWORK,
            "tensor data length does not match the vertex tensor");
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    std::copy(values, values + 2 * n, P->leaf_values[li].begin());
    const int node = P->leaf_desc[li].node;
    if (P->nodes[node].sliced_leaf)
      upload_sliced_values(*P);
    else
      upload_consts(*P);
    if (P->leaf_feeds_branch[li]) P->leaf_epoch++;
    P->graph_epoch++;  // buffers may have moved: recapture
  });
}

int stn_plan_set_max_batch(stn_plan *P, int32_t max_batch) {
  if (!P || max_batch < 0) return set_error(STN_ERR_INVALID_ARGUMENT, "bad argument");
  P->max_batch = max_batch;
  P->graph_epoch++;
  return STN_OK;
}

int stn_plan_set_streams(stn_plan *P, int32_t streams) {
  if (!P || streams < 1) return set_error(STN_ERR_INVALID_ARGUMENT, "bad argument");
  P->streams = streams;
  return STN_OK;
}

int stn_plan_set_profiling(stn_plan *P, int enable) {
  if (!P) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL plan");
  P->profiling = enable != 0;
  return STN_OK;
}

int stn_plan_get_profile(stn_plan *P, stn_kernel_profile *out) {
  if (!P || !out) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    collect_profile(*P);
    for (int k = 0; k < STN_KERNEL_KINDS; ++k) {
      out[k] = P->totals[k];
      out[k].kind = k;
    }
  });
}

int stn_plan_reset_profile(stn_plan *P) {
  if (!P) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL plan");
  return guarded([&] {
    collect_profile(*P);
    for (auto &t : P->totals) t = stn_kernel_profile{};
    P->step_totals.clear();
  });
}

int stn_plan_get_step_profile(stn_plan *P, stn_step_profile *out, int32_t cap, int32_t *n) {
  if (!P || !n) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    collect_profile(*P);
    *n = int32_t(P->step_totals.size());
    int32_t i = 0;
    for (auto &[step, e] : P->step_totals) {
      if (i >= cap || !out) break;
      out[i++] = e;
    }
  });
}

int stn_cache_build(stn_plan *P, void *stream, stn_cache **out) {
  if (!P || !out) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  *out = nullptr;
  auto c = std::make_unique<stn_cache>();
  int st = guarded([&] {
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    build_cache(*P, static_cast<cudaStream_t>(stream), c.get());
    cuda_check(cudaStreamSynchronize(static_cast<cudaStream_t>(stream)), "cache build");
  });
  if (st == STN_OK) *out = c.release();
  return st;
}

int stn_cache_destroy(stn_cache *c) {
  if (c) {
    DeviceGuard g(c->device);
    delete c;
  }
  return STN_OK;
}

int stn_flush_block_cache(void) {
  BlockCache::get().flush();
  return STN_OK;
}

int stn_cache_info(const stn_cache *c, uint64_t *identity, uint64_t *mults, uint64_t *elements) {
  if (!c) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL cache");
  if (identity) *identity = c->identity;
  if (mults) *mults = c->mults;
  if (elements) *elements = c->elements;
  return STN_OK;
}

int stn_run_subtask(stn_plan *P, uint64_t assignment, const stn_cache *cache, void *stream,
                    double *out_host, stn_subtask_info *info) {
  if (!P || !out_host) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    require(assignment < P->subtasks, STN_ERR_SUBTASK_FAILURE, "assignment out of range");
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    std::vector<int32_t> dig(std::max<size_t>(P->sliced_dims.size(), 1), 0);
    decode(*P, assignment, dig.data());
    run_one(*P, dig.data(), cache, static_cast<cudaStream_t>(stream), out_host, info);
    if (info) info->assignment = assignment;
  });
}

int stn_run_subtask_digits(stn_plan *P, const int32_t *digits, const stn_cache *cache,
                           void *stream, double *out_host, stn_subtask_info *info) {
  if (!P || !out_host || (!digits && !P->sliced_dims.empty()))
    return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    for (size_t i = 0; i < P->sliced_dims.size(); ++i)
      require(digits[i] >= 0 && digits[i] < P->sliced_dims[i], STN_ERR_INDEX_OUT_OF_RANGE,
              "slice digit out of range");
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    int32_t zero = 0;
    run_one(*P, digits ? digits : &zero, cache, static_cast<cudaStream_t>(stream), out_host, info);
    if (info) info->assignment = 0;
  });
}

int stn_run_slices(stn_plan *P, const stn_cache *cache, uint64_t lo, uint64_t hi, void *stream,
                   double *acc_dev, double *per_slice_dev) {
  if (!P) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL plan");
  return guarded([&] {
    require(lo <= hi && hi <= P->subtasks, STN_ERR_SUBTASK_FAILURE, "assignment out of range");
    require(cache != nullptr, STN_ERR_INVALID_ARGUMENT, "stn_run_slices needs a branch cache");
    check_cache(*P, cache);
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    run_slices_impl(
        *P, cache, hi - lo, [&](uint64_t i, int32_t *d) { decode(*P, lo + i, d); },
        static_cast<cudaStream_t>(stream), acc_dev, per_slice_dev, nullptr, P->streams);
  });
}

int stn_run_slices_digits(stn_plan *P, const stn_cache *cache, const int32_t *digits,
                          uint64_t n_slices, void *stream, double *acc_dev,
                          double *per_slice_dev) {
  if (!P || (!digits && n_slices && !P->sliced_dims.empty()))
    return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    require(cache != nullptr, STN_ERR_INVALID_ARGUMENT, "stn_run_slices needs a branch cache");
    check_cache(*P, cache);
    const size_t ns = P->sliced_dims.size();
    for (uint64_t i = 0; i < n_slices * ns; ++i)
      require(digits[i] >= 0 && digits[i] < P->sliced_dims[i % ns], STN_ERR_INDEX_OUT_OF_RANGE,
              "slice digit out of range");
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    run_slices_impl(
        *P, cache, n_slices,
        [&](uint64_t i, int32_t *d) { std::copy(digits + i * ns, digits + (i + 1) * ns, d); },
        static_cast<cudaStream_t>(stream), acc_dev, per_slice_dev, nullptr, P->streams);
  });
}

int stn_run_scheme(stn_plan *P, int parallelism, double *out_host, stn_run_report *rep) {
  if (!P || !out_host) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    require(parallelism >= 1, STN_ERR_SUBTASK_FAILURE, "parallelism must be positive");
    require(P->subtasks >= 1, STN_ERR_SUBTASK_FAILURE,
            "plan has no enumerable subtasks (uint64 subtask count overflowed)");
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    auto t0 = std::chrono::steady_clock::now();
    P->kernel_launches = 0;
    cudaStream_t st = nullptr;
    stn_cache cache;
    build_cache(*P, st, &cache);
    DevBuf acc;
    acc.reserve(16 * size_t(P->out_elements));
    cuda_check(cudaMemsetAsync(acc.ptr, 0, 16 * size_t(P->out_elements), st), "memset");
    std::vector<double> ms;
    // per-slice times need one batch at a time; with parallelism > 1 the batches
    // rotate over `parallelism` streams and the reported times are per-batch wall
    // shares of the whole run
    if (parallelism > 1) {
      auto t_a = std::chrono::steady_clock::now();
      run_slices_impl(
          *P, &cache, P->subtasks, [&](uint64_t i, int32_t *d) { decode(*P, i, d); }, st,
          acc.as<double>(), nullptr, nullptr, parallelism);
      cuda_check(cudaStreamSynchronize(st), "stream sync");
      const double per = std::chrono::duration<double, std::milli>(
                             std::chrono::steady_clock::now() - t_a).count() /
                         double(std::max<uint64_t>(P->subtasks, 1));
      ms.assign(size_t(P->subtasks), per);
    } else {
      run_slices_impl(
          *P, &cache, P->subtasks, [&](uint64_t i, int32_t *d) { decode(*P, i, d); }, st,
          acc.as<double>(), nullptr, &ms);
    }
    cuda_check(cudaMemcpyAsync(out_host, acc.ptr, 16 * size_t(P->out_elements),
                               cudaMemcpyDeviceToHost, st),
               "result download");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
    auto t1 = std::chrono::steady_clock::now();
    if (rep) {
      memset(rep, 0, sizeof *rep);
      rep->subtasks = P->subtasks;
      rep->branch_mults = cache.mults;
      rep->mult_count = cache.mults + P->with_cache.mults * P->subtasks;
      rep->wall_seconds = std::chrono::duration<double>(t1 - t0).count();
      std::sort(ms.begin(), ms.end());
      auto q = [&](double f) {
        if (ms.empty()) return 0.0;
        size_t i = size_t(f * double(ms.size() - 1) + 0.5);
        return ms[std::min(i, ms.size() - 1)];
      };
      rep->p50_ms = q(0.5);
      rep->p90_ms = q(0.9);
      rep->p99_ms = q(0.99);
      rep->parallelism = parallelism;
      rep->precision = P->precision;
      rep->peak_elements = P->with_cache.peak;
      rep->merged_groups = P->merged_groups;
      rep->slices_per_batch = auto_batch(*P, P->with_cache);
      rep->kernel_launches = P->kernel_launches;
    }
  });
}

int stn_sum_slices_ordered(const double *per_slice_dev, uint64_t n_slices, int64_t out_elements,
                           double *out_dev, void *stream) {
  if (!per_slice_dev || !out_dev) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    cuda_check(stn::launch_sum_ordered(per_slice_dev, n_slices, out_elements, out_dev,
                                       static_cast<cudaStream_t>(stream)),
               "ordered sum");
  });
}

int stn_run_slices_host(stn_plan *P, const stn_cache *cache, const int32_t *digits, uint64_t lo,
                        uint64_t n_slices, void *stream, double *per_slice_host,
                        double *sum_host) {
  if (!P) return set_error(STN_ERR_INVALID_ARGUMENT, "NULL plan");
  return guarded([&] {
    require(cache != nullptr, STN_ERR_INVALID_ARGUMENT, "stn_run_slices_host needs a branch cache");
    check_cache(*P, cache);
    const size_t ns = P->sliced_dims.size();
    if (digits) {
      for (uint64_t i = 0; i < n_slices * ns; ++i)
        require(digits[i] >= 0 && digits[i] < P->sliced_dims[i % ns], STN_ERR_INDEX_OUT_OF_RANGE,
                "slice digit out of range");
    } else {
      require(lo <= P->subtasks && n_slices <= P->subtasks - lo, STN_ERR_SUBTASK_FAILURE,
              "assignment out of range");
    }
    cuda_check(cudaSetDevice(P->device), "cudaSetDevice");
    cudaStream_t st = static_cast<cudaStream_t>(stream);
    const size_t row = 2 * size_t(P->out_elements);
    DevBuf rows, acc;
    if (per_slice_host) rows.reserve(8 * row * std::max<uint64_t>(n_slices, 1));
    if (sum_host) {
      acc.reserve(8 * row);
      cuda_check(cudaMemsetAsync(acc.ptr, 0, 8 * row, st), "memset");
    }
    auto gen = [&](uint64_t i, int32_t *d) {
      if (digits)
        std::copy(digits + i * ns, digits + (i + 1) * ns, d);
      else
        decode(*P, lo + i, d);
    };
    run_slices_impl(*P, cache, n_slices, gen, st, sum_host ? acc.as<double>() : nullptr,
                    per_slice_host ? rows.as<double>() : nullptr, nullptr, P->streams);
    if (per_slice_host && n_slices)
      cuda_check(cudaMemcpyAsync(per_slice_host, rows.ptr, 8 * row * n_slices,
                                 cudaMemcpyDeviceToHost, st),
                 "per-slice download");
    if (sum_host)
      cuda_check(cudaMemcpyAsync(sum_host, acc.ptr, 8 * row, cudaMemcpyDeviceToHost, st),
                 "sum download");
    cuda_check(cudaStreamSynchronize(st), "stream sync");
  });
}

int stn_fold_slices_ordered(const double *per_slice_dev, uint64_t n_slices, int64_t out_elements,
                            double *acc_dev, void *stream) {
  if ((!per_slice_dev && n_slices) || !acc_dev)
    return set_error(STN_ERR_INVALID_ARGUMENT, "NULL argument");
  return guarded([&] {
    if (n_slices == 0) return;
    cuda_check(stn::launch_sum_ordered(per_slice_dev, n_slices, out_elements, acc_dev,
                                       static_cast<cudaStream_t>(stream), true),
               "ordered fold");
  });
}

int stn_selftest_gemm_tc(int64_t M, int64_t N, int64_t K, int32_t batches, int32_t a_batched,
                         int32_t b_batched, int32_t reps, double *max_rel_err, double *ms_total,
                         double *ms_gemm, double *ms_simt, double *simt_rel_err) {
  return guarded([&] {
    stn::GemmShape s{1, M, N, K};
    // the fused-split kernel (gemm_tcf.cu) unless STN_DEBUG tcf=0 selects the pre-split one
    const char *tcf_opt = stn::debug_opt("tcf");
    const bool tcf = !(tcf_opt && std::atoi(tcf_opt) == 0);  // selftest: 0 pre-split, else fused
    require((tcf ? stn::gemm_tcf_supported(s) : stn::gemm_tc_supported(s)) && batches >= 1 &&
                reps >= 1,
            STN_ERR_INVALID_ARGUMENT, "shape not supported by the tensor-core GEMM");
    auto run_tc = [&](const stn::BatchPtrs &pp, void *w, size_t wb, cudaStream_t ss,
                      cudaEvent_t *gev) {
      if (!tcf) return stn::launch_gemm_tc(s, pp, w, wb, ss, gev);
      if (gev) cudaEventRecord(gev[0], ss);
      cudaError_t e = stn::launch_gemm_tcf(s, pp, w, wb, ss);
      if (gev) cudaEventRecord(gev[1], ss);
      return e;
    };
    const int64_t na = a_batched ? batches : 1, nbb = b_batched ? batches : 1;
    std::vector<float> ha(size_t(2 * M * K * na)), hb(size_t(2 * K * N * nbb));
    uint64_t x = 0x9E3779B97F4A7C15ull;
    auto rnd = [&] {
      x ^= x << 13;
      x ^= x >> 7;
      x ^= x << 17;
      return float(double(x >> 11) * 0x1.0p-53 * 2.0 - 1.0);
    };
    for (auto &v : ha) v = rnd();
    for (auto &v : hb) v = rnd();
    std::vector<double> da(ha.begin(), ha.end()), db(hb.begin(), hb.end());
    DevBuf A, B, Cf, Ad, Bd, Cd, ws;
    A.upload(ha);
    B.upload(hb);
    Ad.upload(da);
    Bd.upload(db);
    Cf.reserve(size_t(8 * M * N * batches));
    Cd.reserve(size_t(16 * M * N * batches));
    stn::BatchPtrs p{A.ptr, B.ptr, Cf.ptr, a_batched ? M * K : 0, b_batched ? K * N : 0, M * N,
                     batches};
    stn::BatchPtrs pd{Ad.ptr, Bd.ptr, Cd.ptr, a_batched ? M * K : 0, b_batched ? K * N : 0,
                      M * N, batches};
    size_t wsb = tcf ? stn::gemm_tcf_workspace_bytes(s, p) : stn::gemm_tc_workspace_bytes(s, p);
    ws.reserve(std::max<size_t>(wsb, 16));
    cudaStream_t st = nullptr;
    cudaEvent_t ev[4];
    for (auto &e : ev) cuda_check(cudaEventCreate(&e), "event");
    cuda_check(run_tc(p, ws.ptr, wsb, st, nullptr), "tc gemm");
    cuda_check(stn::launch_gemm_simt<double>(s, pd, false, st), "simt gemm");
    cuda_check(cudaStreamSynchronize(st), "sync");
    std::vector<float> cf(size_t(2 * M * N * batches));
    std::vector<double> cd(size_t(2 * M * N * batches));
    cuda_check(cudaMemcpy(cf.data(), Cf.ptr, cf.size() * 4, cudaMemcpyDeviceToHost), "dl");
    cuda_check(cudaMemcpy(cd.data(), Cd.ptr, cd.size() * 8, cudaMemcpyDeviceToHost), "dl");
    double scale = 0, err = 0;
    for (size_t i = 0; i < cd.size(); i += 2) scale = std::max(scale, std::hypot(cd[i], cd[i + 1]));
    for (size_t i = 0; i < cd.size(); i += 2)
      err = std::max(err, std::hypot(double(cf[i]) - cd[i], double(cf[i + 1]) - cd[i + 1]));
    *max_rel_err = err / std::max(scale, 1e-300);
    double tot = 0, gm = 0;
    for (int r = 0; r < reps; ++r) {
      cuda_check(cudaEventRecord(ev[0], st), "event");
      cuda_check(run_tc(p, ws.ptr, wsb, st, &ev[2]), "tc gemm");
      cuda_check(cudaEventRecord(ev[1], st), "event");
      cuda_check(cudaEventSynchronize(ev[1]), "sync");
      float a = 0, b = 0;
      cudaEventElapsedTime(&a, ev[0], ev[1]);
      cudaEventElapsedTime(&b, ev[2], ev[3]);
      tot += a;
      gm += b;
    }
    *ms_total = tot / reps;
    *ms_gemm = gm / reps;
    double sm = 0;
    for (int r = 0; r < reps; ++r) {
      cuda_check(cudaEventRecord(ev[0], st), "event");
      cuda_check(stn::launch_gemm_simt<float>(s, p, false, st), "simt gemm");
      cuda_check(cudaEventRecord(ev[1], st), "event");
      cuda_check(cudaEventSynchronize(ev[1]), "sync");
      float a = 0;
      cudaEventElapsedTime(&a, ev[0], ev[1]);
      sm += a;
    }
    if (ms_simt) *ms_simt = sm / reps;
    if (simt_rel_err) {
      cuda_check(cudaMemcpy(cf.data(), Cf.ptr, cf.size() * 4, cudaMemcpyDeviceToHost), "dl");
      double e2 = 0;
      for (size_t i = 0; i < cd.size(); i += 2)
        e2 = std::max(e2, std::hypot(double(cf[i]) - cd[i], double(cf[i + 1]) - cd[i + 1]));
      *simt_rel_err = e2 / std::max(scale, 1e-300);
    }
    for (auto &e : ev) cudaEventDestroy(e);
  });
}

int stn_selftest_chain_jit(int exact, char *log, int32_t log_cap) {
  return guarded([&] {
    // a synthetic two-stage chain (K = N = 2 each) through the NVRTC code generator
    stn::ChainGeom g{};
    auto t = std::make_unique<stn::ChainTables>();
    memset(t.get(), 0, sizeof(stn::ChainTables));
    g.n_stages = 2;
    g.li = 2;
    g.lo = 2;
    g.ma = 2;
    g.rows = 1 << 10;
    g.w_total = 8;
    g.st[0] = {1, 1, 1, 0, 4, 0, 0};
    g.st[1] = {1, 1, 1, 8, 12, 4, 4};
    const uint8_t tab[16] = {0, 1, 2, 3, 0, 1, 2, 3, 0, 2, 1, 3, 0, 1, 2, 3};
    memcpy(t->tab, tab, sizeof tab);
    for (int i = 0; i < 4; ++i) {
      t->xin[i] = i * 64;
      t->oout[i] = i * 128;
      t->widx[i] = t->widx[4 + i] = i;
    }
    // the same chain with 32-byte loads and 16-byte stores (tile lines at the lowest
    // positions of X and O)
    stn::ChainGeom gv = g;
    auto tv = std::make_unique<stn::ChainTables>(*t);
    for (int i = 0; i < 4; ++i) {
      tv->xin[i] = i;
      tv->oout[i] = (i & 1) + (i >> 1) * 128;
    }
    // the same chain with lane / tile exchanges: position 0 is a lane bit, position 1 a
    // tile line, on both sides
    auto tx = std::make_unique<stn::ChainTables>(*t);
    const int64_t lane_bits[5] = {1, 4, 8, 16, 32};
    for (int l = 0; l < 32; ++l) {
      tx->xl[l] = tx->ol[l] = 0;
      for (int q = 0; q < 5; ++q)
        if ((l >> q) & 1) tx->xl[l] = tx->ol[l] += lane_bits[q];
    }
    for (int i = 0; i < 4; ++i) tx->xin[i] = tx->oout[i] = (i & 1) * 2 + (i >> 1) * 64;
    // a one-stage chain with a 64-value input tile (no software pipelining), K = 64, N = 2
    stn::ChainGeom g1{};
    auto t1 = std::make_unique<stn::ChainTables>();
    memset(t1.get(), 0, sizeof(stn::ChainTables));
    g1.n_stages = 1;
    g1.li = 6;
    g1.lo = 1;
    g1.ma = 6;
    g1.rows = 1 << 10;
    g1.w_total = 128;
    g1.st[0] = {0, 6, 1, 0, 64, 0, 0};
    for (int k = 0; k < 64; ++k) t1->tab[k] = uint8_t(k);
    t1->tab[64] = 0;
    t1->tab[65] = 1;
    for (int i = 0; i < 64; ++i) t1->xin[i] = i;
    t1->oout[1] = 1;
    for (int i = 0; i < 128; ++i) t1->widx[i] = i;
    // the two-stage chain with 3 expansion row bits on its first stage (W block [k][e][n])
    stn::ChainGeom ge = g;
    ge.n_exp = 3;
    ge.st[1].w_smem = 32;
    ge.st[1].w_off = 32;
    ge.w_total = 36;
    std::string l;
    const bool ok = stn::chain_jit_compile_only(
        {{&g, t.get()}, {&gv, tv.get()}, {&g, tx.get()}, {&g1, t1.get()}, {&ge, t.get()}},
        exact != 0, &l);
    if (log && log_cap > 0) {
      strncpy(log, l.c_str(), size_t(log_cap) - 1);
      log[log_cap - 1] = 0;
    }
    require(ok, STN_ERR_CUDA, "NVRTC compilation of a chain kernel failed: " + l.substr(0, 400));
  });
}

int stn_selftest_bitperm(int32_t log2_elems, const int32_t *perm, int32_t reps, double *gbs_kernel,
                         double *gbs_memcpy, int32_t *correct) {
  return guarded([&] {
    require(log2_elems >= 12 && log2_elems <= 31 && reps >= 1, STN_ERR_INVALID_ARGUMENT,
            "bad size");
    const int r = log2_elems;
    // out bit i (position) <- in bit perm[i]; as axes: out axis a = in axis p
    std::vector<int> dims(r, 2), axis_perm(r);
    for (int i = 0; i < r; ++i) {
      const int src_bit = perm ? perm[i] : i;
      axis_perm[r - 1 - i] = r - 1 - src_bit;
    }
    stn::AbsorbGeom g;
    require(build_bitperm(dims, axis_perm, g), STN_ERR_INVALID_ARGUMENT, "no tile geometry");
    // the executor's permute: the high-occupancy tile permute where it applies
    stn::PermTileGeom tg;
    std::vector<int64_t> tbases;
    DevBuf tb_dev;
    const bool tiles = stn::debug_opt("bitperm_legacy") == nullptr &&
                       stn::build_perm_tiles(axis_perm, tg, tbases);
    if (tiles) tb_dev.upload(tbases);
    auto launch = [&](const void *src, void *dst, cudaStream_t s) {
      return tiles ? stn::launch_perm_tiles(tg, tb_dev.as<int64_t>(), src, dst, 0, 0, 1, s)
                   : stn::launch_bitperm(g, src, dst, 0, 0, 1, s);
    };
    const size_t n = size_t(1) << r, bytes = n * 8;
    DevBuf in, out, ref;
    in.reserve(bytes);
    out.reserve(bytes);
    ref.reserve(bytes);
    std::vector<uint32_t> host(2 * n);
    for (size_t i = 0; i < n; ++i) host[2 * i] = uint32_t(i), host[2 * i + 1] = uint32_t(~i);
    cuda_check(cudaMemcpy(in.ptr, host.data(), bytes, cudaMemcpyHostToDevice), "upload");
    cudaStream_t st = nullptr;
    cudaEvent_t e0, e1;
    cuda_check(cudaEventCreate(&e0), "event");
    cuda_check(cudaEventCreate(&e1), "event");
    cuda_check(launch(in.ptr, out.ptr, st), "bitperm");
    cuda_check(cudaStreamSynchronize(st), "sync");
    std::vector<uint32_t> got(2 * n);
    cuda_check(cudaMemcpy(got.data(), out.ptr, bytes, cudaMemcpyDeviceToHost), "download");
    bool ok = true;
    for (size_t o = 0; o < n && ok; ++o) {
      size_t src = 0;
      for (int i = 0; i < r; ++i)
        if ((o >> i) & 1) src |= size_t(1) << (perm ? perm[i] : i);
      ok = got[2 * o] == uint32_t(src) && got[2 * o + 1] == uint32_t(~src);
    }
    *correct = ok ? 1 : 0;
    cuda_check(cudaEventRecord(e0, st), "event");
    for (int i = 0; i < reps; ++i) cuda_check(launch(in.ptr, out.ptr, st), "bitperm");
    cuda_check(cudaEventRecord(e1, st), "event");
    cuda_check(cudaEventSynchronize(e1), "sync");
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    *gbs_kernel = 2.0 * bytes * reps / (ms / 1e3) / 1e9;
    cuda_check(cudaEventRecord(e0, st), "event");
    for (int i = 0; i < reps; ++i)
      cuda_check(cudaMemcpyAsync(ref.ptr, in.ptr, bytes, cudaMemcpyDeviceToDevice, st), "memcpy");
    cuda_check(cudaEventRecord(e1, st), "event");
    cuda_check(cudaEventSynchronize(e1), "sync");
    cudaEventElapsedTime(&ms, e0, e1);
    *gbs_memcpy = 2.0 * bytes * reps / (ms / 1e3) / 1e9;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
  });
}

}  // extern "C"
