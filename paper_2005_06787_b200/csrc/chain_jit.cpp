// Plan-specialised fused stem chains, compiled at plan creation with NVRTC.
//
// kernels_chain.cu runs any chain through slot tables and a shared-memory tile;
// its per-element table lookups and shared-memory round trips cost more issue
// slots than the HBM stream leaves (measured on B200: ~3 TB/s). Here the plan's
// chains are known, so each one is emitted as straight-line CUDA: the column's
// inputs are registers loaded from constant offsets, every stage is a fixed
// sequence of complex multiply-adds between named registers (k ascending; EXACT:
// separately rounded products and sums, bitwise the reference's order), and the
// next row's inputs are loaded before the current row's stages run (software
// pipelining instead of a shared-memory ring). All chains of a plan go into one
// NVRTC program; the cubin is loaded per device and cached per process.
// NVRTC and the driver's module API are resolved at run time (dlopen /
// cudaGetDriverEntryPoint): without NVRTC the chains run on kernels_chain.cu.
#include "chain_jit.h"

#include <dlfcn.h>
#include <sys/stat.h>
#include <unistd.h>

#include <algorithm>
#include <atomic>
#include <cstddef>
#include <cstdlib>
#include <thread>

#include <cstdio>
#include <cstring>
#include <map>
#include <mutex>
#include <sstream>
#include <string>
#include <vector>

#include <cuda.h>
#include <cuda_runtime.h>

namespace stn {

namespace {

// ---- NVRTC (dlopen) -----------------------------------------------------------------
struct Nvrtc {
  void *h = nullptr;
  int (*Create)(void **, const char *, const char *, int, const char *const *,
                const char *const *) = nullptr;
  int (*Compile)(void *, int, const char *const *) = nullptr;
  int (*GetCubinSize)(void *, size_t *) = nullptr;
  int (*GetCubin)(void *, char *) = nullptr;
  int (*GetLogSize)(void *, size_t *) = nullptr;
  int (*GetLog)(void *, char *) = nullptr;
  int (*Destroy)(void **) = nullptr;
  int major = 0, minor = 0;
  bool ok = false;
  static Nvrtc &get() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] { n.load(); });
    return n;
  }
  void load() {
    // the toolkit's NVRTC first: a process that imported torch already has torch's
    // bundled (older) libnvrtc.so.12 loaded, which the bare soname would return
    for (const char *name : {"/usr/local/cuda/lib64/libnvrtc.so.12", "/usr/local/cuda/lib64/libnvrtc.so",
                             "libnvrtc.so.12", "libnvrtc.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) return;
    auto version = reinterpret_cast<int (*)(int *, int *)>(dlsym(h, "nvrtcVersion"));
    if (version) version(&major, &minor);
    Create = reinterpret_cast<decltype(Create)>(dlsym(h, "nvrtcCreateProgram"));
    Compile = reinterpret_cast<decltype(Compile)>(dlsym(h, "nvrtcCompileProgram"));
    GetCubinSize = reinterpret_cast<decltype(GetCubinSize)>(dlsym(h, "nvrtcGetCUBINSize"));
    GetCubin = reinterpret_cast<decltype(GetCubin)>(dlsym(h, "nvrtcGetCUBIN"));
    GetLogSize = reinterpret_cast<decltype(GetLogSize)>(dlsym(h, "nvrtcGetProgramLogSize"));
    GetLog = reinterpret_cast<decltype(GetLog)>(dlsym(h, "nvrtcGetProgramLog"));
    Destroy = reinterpret_cast<decltype(Destroy)>(dlsym(h, "nvrtcDestroyProgram"));
    ok = Create && Compile && GetCubinSize && GetCubin && GetLogSize && GetLog && Destroy;
  }
};

// ---- driver module API (entry points through the runtime) -----------------------------
struct Driver {
  CUresult (*ModuleLoadData)(CUmodule *, const void *) = nullptr;
  CUresult (*ModuleGetFunction)(CUfunction *, CUmodule, const char *) = nullptr;
  CUresult (*LaunchKernel)(CUfunction, unsigned, unsigned, unsigned, unsigned, unsigned, unsigned,
                           unsigned, CUstream, void **, void **) = nullptr;
  CUresult (*FuncGetAttribute)(int *, CUfunction_attribute, CUfunction) = nullptr;
  CUresult (*FuncSetAttribute)(CUfunction, CUfunction_attribute, int) = nullptr;
  bool ok = false;
  static Driver &get() {
    static Driver d;
    static std::once_flag once;
    std::call_once(once, [] { d.load(); });
    return d;
  }
  template <class F>
  void sym(F &f, const char *name) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint(name, &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      f = reinterpret_cast<F>(p);
  }
  void load() {
    sym(ModuleLoadData, "cuModuleLoadData");
    sym(ModuleGetFunction, "cuModuleGetFunction");
    sym(LaunchKernel, "cuLaunchKernel");
    sym(FuncGetAttribute, "cuFuncGetAttribute");
    sym(FuncSetAttribute, "cuFuncSetAttribute");
    ok = ModuleLoadData && ModuleGetFunction && LaunchKernel;
  }
};

// Same layout on both sides (generated source declares it identically).
struct JitArgs {
  const void *x;
  void *o;
  long long x_bs, o_bs;
  const void *w[kChainMaxStages];
  long long w_bs[kChainMaxStages];
  const void *tabs;  // ChainTables
  long long rows;
};

const char *kPrelude = R"(
struct JitArgs {
  const float2 *x; float2 *o; long long x_bs, o_bs;
  const float2 *w[8]; long long w_bs[8]; const long long *tabs; long long rows;
};
__device__ __forceinline__ float2 ldcs2(const float2 *p) {
  float2 v; asm volatile("ld.global.cs.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void stcs2(float2 *p, float2 v) {
  asm volatile("st.global.cs.v2.f32 [%0], {%1, %2};" :: "l"(p), "f"(v.x), "f"(v.y) : "memory");
}
__device__ __forceinline__ void ldcs4(const float2 *p, float2 &a, float2 &b) {
  asm volatile("ld.global.cs.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y) : "l"(p));
}
__device__ __forceinline__ void ldcs8(const float2 *p, float2 &a, float2 &b, float2 &c, float2 &d) {
  asm volatile("ld.global.cs.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y), "=f"(c.x), "=f"(c.y), "=f"(d.x),
                 "=f"(d.y) : "l"(p));
}
// plain (L1-allocating) loads for X tiles that several rows re-read (expansion rows)
__device__ __forceinline__ float2 ldg2(const float2 *p) {
  float2 v; asm volatile("ld.global.v2.f32 {%0, %1}, [%2];" : "=f"(v.x), "=f"(v.y) : "l"(p));
  return v;
}
__device__ __forceinline__ void ldg4(const float2 *p, float2 &a, float2 &b) {
  asm volatile("ld.global.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y) : "l"(p));
}
__device__ __forceinline__ void ldg8(const float2 *p, float2 &a, float2 &b, float2 &c, float2 &d) {
  asm volatile("ld.global.v8.f32 {%0, %1, %2, %3, %4, %5, %6, %7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(b.x), "=f"(b.y), "=f"(c.x), "=f"(c.y), "=f"(d.x),
                 "=f"(d.y) : "l"(p));
}
__device__ __forceinline__ void stcs4(float2 *p, float2 a, float2 b) {
  asm volatile("st.global.cs.v4.f32 [%0], {%1, %2, %3, %4};"
               :: "l"(p), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y) : "memory");
}
__device__ __forceinline__ void stcs8(float2 *p, float2 a, float2 b, float2 c, float2 d) {
  asm volatile("st.global.cs.v8.f32 [%0], {%1, %2, %3, %4, %5, %6, %7, %8};"
               :: "l"(p), "f"(a.x), "f"(a.y), "f"(b.x), "f"(b.y), "f"(c.x), "f"(c.y),
                  "f"(d.x), "f"(d.y) : "memory");
}
// acc + x * w
__device__ __forceinline__ float2 cmx(float2 acc, float2 x, float2 w) {  // EXACT
  float re = __fsub_rn(__fmul_rn(x.x, w.x), __fmul_rn(x.y, w.y));
  float im = __fadd_rn(__fmul_rn(x.x, w.y), __fmul_rn(x.y, w.x));
  return make_float2(__fadd_rn(acc.x, re), __fadd_rn(acc.y, im));
}
// FAST with packed FP32 FMAs (FFMA2): W staged as (wr, wr, wi, -wi); U += x (wr, wr),
// V += x (wi, -wi) with x = (xr, xi) as held; re = U.x + V.y, im = U.y + V.x
__device__ __forceinline__ unsigned long long pk(float2 v) {
  unsigned long long r; asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(v.x), "f"(v.y)); return r;
}
__device__ __forceinline__ void f2(unsigned long long &a, unsigned long long x, unsigned long long w) {
  asm("fma.rn.f32x2 %0, %1, %2, %0;" : "+l"(a) : "l"(x), "l"(w));
}
__device__ __forceinline__ float2 fin(unsigned long long u, unsigned long long v) {
  float2 a, c;
  asm("mov.b64 {%0, %1}, %2;" : "=f"(a.x), "=f"(a.y) : "l"(u));
  asm("mov.b64 {%0, %1}, %2;" : "=f"(c.x), "=f"(c.y) : "l"(v));
  return make_float2(a.x + c.y, a.y + c.x);
}
__device__ __forceinline__ float2 cmf(float2 acc, float2 x, float2 w) {  // FAST
  acc.x = fmaf(x.x, w.x, acc.x); acc.x = fmaf(-x.y, w.y, acc.x);
  acc.y = fmaf(x.x, w.y, acc.y); acc.y = fmaf(x.y, w.x, acc.y);
  return acc;
}
)";

}  // namespace

// 16 / 32-byte accesses for tiles holding the tensors' lowest positions: log2 of the
// widest group (STN_DEBUG chain_vec=0|1|2 caps it); 32-byte (v8) accesses need PTX
// ISA 8.8 (NVRTC >= 12.9)
int chain_vec_max() {
  const char *cv = debug_opt("chain_vec");
  const Nvrtc &nv = Nvrtc::get();
  return std::min(cv ? std::atoi(cv) : 2, nv.major > 12 || (nv.major == 12 && nv.minor >= 9) ? 2 : 1);
}

namespace {

// Vector width of a tile's HBM accesses: the tile lines at positions 0 and 1 of the
// tensor (offsets 1 and 2) make groups of 2 or 4 adjacent complex values that one
// 16- or 32-byte access moves (a whole 32-byte sector per thread instead of one
// element of it per lane). Returns log2 of the group size and the slot bits.
int vec_bits(const int64_t *off, int n_log, int *s0, int *s1) {
  *s0 = *s1 = -1;
  for (int j = 0; j < n_log; ++j) {
    if (off[1 << j] == 1) *s0 = j;
    if (off[1 << j] == 2) *s1 = j;
  }
  if (*s0 < 0) return 0;
  return *s1 < 0 ? 1 : 2;
}

// "dst = ld(p + off)" for every element of a tile, grouped into vector accesses.
// `name(i)` is the register of element i; `v` the vector log (<= vmax).
template <class Name>
void emit_tile_io(std::ostringstream &s, bool load, const char *ptr, const int64_t *off,
                  int n_log, int vmax, Name name, const char *indent, bool declare = true,
                  const std::string &ld = "ldcs") {
  int s0, s1;
  int v = std::min(vec_bits(off, n_log, &s0, &s1), vmax);
  const int m0 = s0 >= 0 ? 1 << s0 : 0, m1 = s1 >= 0 ? 1 << s1 : 0;
  for (int i = 0; i < (1 << n_log); ++i) {
    if (v >= 1 && (i & m0)) continue;
    if (v >= 2 && (i & m1)) continue;
    s << indent;
    if (v == 0) {
      if (load)
        s << (declare ? "float2 " : "") << name(i) << " = " << ld << "2(" << ptr << " + " << off[i]
          << "LL);\n";
      else s << "stcs2(" << ptr << " + " << off[i] << "LL, " << name(i) << ");\n";
    } else if (v == 1) {
      if (load && !declare)
        s << ld << "4(" << ptr << " + " << off[i] << "LL, " << name(i) << ", " << name(i | m0)
          << ");\n";
      else if (load)
        s << "float2 " << name(i) << ", " << name(i | m0) << "; " << ld << "4(" << ptr << " + " << off[i]
          << "LL, " << name(i) << ", " << name(i | m0) << ");\n";
      else
        s << "stcs4(" << ptr << " + " << off[i] << "LL, " << name(i) << ", " << name(i | m0)
          << ");\n";
    } else {
      if (load && !declare)
        s << ld << "8(" << ptr << " + " << off[i] << "LL, " << name(i) << ", " << name(i | m0)
          << ", " << name(i | m1) << ", " << name(i | m0 | m1) << ");\n";
      else if (load)
        s << "float2 " << name(i) << ", " << name(i | m0) << ", " << name(i | m1) << ", "
          << name(i | m0 | m1) << "; " << ld << "8(" << ptr << " + " << off[i] << "LL, " << name(i)
          << ", " << name(i | m0) << ", " << name(i | m1) << ", " << name(i | m0 | m1) << ");\n";
      else
        s << "stcs8(" << ptr << " + " << off[i] << "LL, " << name(i) << ", " << name(i | m0)
          << ", " << name(i | m1) << ", " << name(i | m0 | m1) << ");\n";
    }
  }
}

// Warp exchange of tile slot bit s with lane bit j (an involution): afterwards slot
// bit s indexes what lane bit j did and vice versa.
void emit_exchange(std::ostringstream &s, const std::string &prefix, int n_log, int j, int sb) {
  s << "    { const bool lam = (lane >> " << j << ") & 1;\n";
  for (int i = 0; i < (1 << n_log); ++i) {
    if ((i >> sb) & 1) continue;
    const std::string a = prefix + std::to_string(i), b = prefix + std::to_string(i | (1 << sb));
    s << "      { float2 v = lam ? " << a << " : " << b << "; v.x = __shfl_xor_sync(0xffffffffu, v.x, "
      << (1 << j) << "); v.y = __shfl_xor_sync(0xffffffffu, v.y, " << (1 << j) << "); if (lam) "
      << a << " = v; else " << b << " = v; }\n";
  }
  s << "    }\n";
}

// Emits the kernel of one chain. `kt` is the host copy of its tables.
std::string emit(const ChainGeom &g, const ChainTables &kt, int id, bool exact, int minb = 1) {
  std::ostringstream s;
  const int ni = 1 << g.li;
  const char *cm = exact ? "cmx" : "cmf";
  // FAST with packed FP32 FMAs only on request (STN_DEBUG chain_ffma2=1): the U / V
  // accumulator pairs raise register pressure, more chains spill and are re-planned;
  // measured on B200 cfg5 88.1 -> 94.5, cfg2 6.78 -> 7.03 ms per slice with them
  const char *fo = debug_opt("chain_ffma2");
  const bool ff2 = !exact && fo && std::atoi(fo) != 0;
  // software pipelining holds two input tiles in registers: only for tiles of up to
  // 2^chain_pf_log values (STN_DEBUG chain_pf_log, default 5)
  const bool prefetch = chain_prefetch(g);
  const int vmax = chain_vec_max();
  // lane / tile exchanges that make the HBM accesses whole sectors (chain_lane_swap)
  int xj = -1, xs = -1, oj = -1, os_ = -1;
  int64_t xl_p[32], xin_p[1 << kChainMaxLog], ol_p[32], oout_p[1 << kChainMaxLog];
  const int64_t *xin = kt.xin, *oout = kt.oout;
  const bool swaps = vmax >= 2 && chain_swaps_allowed(g);
  const bool xswap = swaps && chain_lane_swap(kt.xl, kt.xin, g.li, &xj, &xs);
  const bool oswap = swaps && chain_lane_swap(kt.ol, kt.oout, g.lo, &oj, &os_);
  if (xswap) {
    chain_apply_swap(kt.xl, kt.xin, g.li, xj, xs, xl_p, xin_p);
    xin = xin_p;
  }
  if (oswap) {
    chain_apply_swap(kt.ol, kt.oout, g.lo, oj, os_, ol_p, oout_p);
    oout = oout_p;
  }
  s << "extern \"C\" __global__ void __launch_bounds__(256"
    << (minb > 1 ? ", " + std::to_string(minb) : std::string()) << ") stn_chain_" << id
    << "(const JitArgs a) {\n"
    << "  __shared__ long long sxr[1024], sor[1024];\n"
    << (ff2 ? "  extern __shared__ ulonglong2 sw[];  // W of every stage as (wr, wr, wi, -wi)\n"
            : "  extern __shared__ float2 sw[];  // W of every stage (dynamic)\n")
    << "  for (int i = threadIdx.x; i < 1024; i += 256) { sxr[i] = a.tabs[i]; sor[i] = a.tabs[1024 + i]; }\n"
    << "  const long long b = blockIdx.y;\n";
  // W: staged through the element offsets of the chain's tables (ChainTables::widx)
  s << "  const int *widx = (const int *)((const char *)a.tabs + "
    << offsetof(ChainTables, widx) << ");\n";
  const std::string ld = "ldcs";
  for (int st = 0; st < g.n_stages; ++st) {
    const ChainStage &cs = g.st[st];
    const int kn = 1 << (cs.lk + cs.ln + (st == 0 ? g.n_exp : 0));
    if (ff2)
      s << "  for (int i = threadIdx.x; i < " << kn << "; i += 256) { const float2 w = a.w[" << st
        << "][b * a.w_bs[" << st << "] + widx[" << cs.w_off << " + i]]; sw[" << cs.w_smem
        << " + i] = make_ulonglong2(pk(make_float2(w.x, w.x)), pk(make_float2(w.y, -w.y))); }\n";
    else
      s << "  for (int i = threadIdx.x; i < " << kn << "; i += 256) sw[" << cs.w_smem
        << " + i] = a.w[" << st << "][b * a.w_bs[" << st << "] + widx[" << cs.w_off << " + i]];\n";
  }
  // W operands of small stages (K x N <= 16, not an expansion stage) held in registers for
  // the whole kernel instead of one shared-memory load per multiply-add: only on request
  // (STN_DEBUG chain_wreg=V, at most V values) -- the registers they take cost more than
  // the loads they save (measured on B200: cfg5 86.9 -> 106.3 ms per slice with 16)
  const char *wo = debug_opt("chain_wreg");
  const char *we = debug_opt("chain_wreg_exp");  // experiments: expansion kernels only
  const int wreg_max = wo ? std::atoi(wo) : (we && g.n_exp > 0) ? std::atoi(we) : 0;
  std::vector<char> hoist(size_t(g.n_stages), 0);
  {
    int used = 0;
    for (int st = 0; st < g.n_stages; ++st) {
      const ChainStage &cs = g.st[st];
      const int kn = 1 << (cs.lk + cs.ln);
      if (ff2 || (st == 0 && g.n_exp > 0) || kn > 16 || used + kn > wreg_max) continue;
      hoist[size_t(st)] = 1;
      used += kn;
    }
  }
  s << "  __syncthreads();\n";
  for (int st = 0; st < g.n_stages; ++st) {
    if (!hoist[size_t(st)]) continue;
    const ChainStage &cs = g.st[st];
    for (int i = 0; i < (1 << (cs.lk + cs.ln)); ++i)
      s << "  const float2 w" << st << "_" << i << " = sw[" << cs.w_smem + i << "];\n";
  }
  s << "  const int lane = threadIdx.x & 31;\n"
    << "  const long long xl = a.tabs[2048 + lane]"
    << (xswap ? " + (((lane >> " + std::to_string(xj) + ") & 1) ? " +
                    std::to_string(xl_p[1 << xj] - kt.xl[1 << xj]) + "LL : 0LL)"
              : std::string())
    << ", ol = a.tabs[2080 + lane]"
    << (oswap ? " + (((lane >> " + std::to_string(oj) + ") & 1) ? " +
                    std::to_string(ol_p[1 << oj] - kt.ol[1 << oj]) + "LL : 0LL)"
              : std::string())
    << ";\n"
    << "  const float2 *X = a.x + b * a.x_bs;\n  float2 *O = a.o + b * a.o_bs;\n"
    << "  const long long step = (long long)gridDim.x * 8;\n"
    << "  long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);\n"
    << "#define RX(r) (sxr[(r) & 255] + sxr[256 + (((r) >> 8) & 255)] + sxr[512 + (((r) >> 16) & 255)] + sxr[768 + (((r) >> 24) & 255)])\n"
    << "#define RO(r) (sor[(r) & 255] + sor[256 + (((r) >> 8) & 255)] + sor[512 + (((r) >> 16) & 255)] + sor[768 + (((r) >> 24) & 255)])\n";
  if (g.n_exp > 0) {
    // expansion rows: a warp loads its X tile once per group of 2^n_exp rows (they share
    // it) and runs the chain for every expansion column of the group in an inner loop
    s << "  const long long groups = a.rows >> " << g.n_exp << ";\n"
      << "  for (long long grp = row; grp < groups; grp += step) {\n"
      << "    const float2 *p = X + RX((unsigned)(grp << " << g.n_exp << ")) + xl;\n";
    emit_tile_io(s, true, "p", xin, g.li, vmax, [](int i) { return "t0_" + std::to_string(i); },
                 "    ", true);
    if (xswap) emit_exchange(s, "t0_", g.li, xj, xs);
    s << "  for (int e = 0; e < " << (1 << g.n_exp) << "; ++e) {\n"
      << "    const long long row = (grp << " << g.n_exp << ") | e;\n"
      << "    const int wr = e * " << (1 << g.st[0].ln) << ";  // W column block of stage 0\n";
  } else if (prefetch) {
    for (int i = 0; i < ni; ++i) s << "  float2 n" << i << " = make_float2(0.f, 0.f);\n";
    auto nn = [](int i) { return "n" + std::to_string(i); };
    s << "  if (row < a.rows) {\n    const float2 *p = X + RX((unsigned)row) + xl;\n";
    emit_tile_io(s, true, "p", xin, g.li, vmax, nn, "    ", false, ld);
    s << "  }\n  for (; row < a.rows; row += step) {\n";
    for (int i = 0; i < ni; ++i) s << "    float2 t0_" << i << " = n" << i << ";\n";
    if (xswap) emit_exchange(s, "t0_", g.li, xj, xs);
    s << "    { const long long nr = row + step;\n      if (nr < a.rows) {\n"
      << "        const float2 *p = X + RX((unsigned)nr) + xl;\n";
    emit_tile_io(s, true, "p", xin, g.li, vmax, nn, "        ", false, ld);
    s << "      }\n    }\n";
  } else {  // large tiles: the other warps of the SM hide the load latency
    s << "  for (; row < a.rows; row += step) {\n"
      << "    const float2 *p = X + RX((unsigned)row) + xl;\n";
    emit_tile_io(s, true, "p", xin, g.li, vmax, [](int i) { return "t0_" + std::to_string(i); },
                 "    ", true, ld);
    if (xswap) emit_exchange(s, "t0_", g.li, xj, xs);
  }

  for (int st = 0; st < g.n_stages; ++st) {
    const ChainStage &cs = g.st[st];
    const int R = 1 << cs.lr, K = 1 << cs.lk, N = 1 << cs.ln;
    for (int r = 0; r < R; ++r)
      for (int n = 0; n < N; ++n) {
        const int out_slot = kt.tab[cs.wr_off + r * N + n];
        if (ff2) {
          s << "    float2 t" << st + 1 << "_" << out_slot << ";\n    { unsigned long long u = 0ull, v = 0ull;\n";
          for (int k = 0; k < K; ++k) {
            const int in_slot = kt.tab[cs.rd_off + r * K + k];
            const bool ex = st == 0 && g.n_exp > 0;
            s << "      { const ulonglong2 w = sw[" << (ex ? "wr + " : "")
              << cs.w_smem + k * (N << (ex ? g.n_exp : 0)) + n << "]; const unsigned long long x = pk(t"
              << st << "_" << in_slot << "); f2(u, x, w.x); f2(v, x, w.y); }\n";
          }
          s << "      t" << st + 1 << "_" << out_slot << " = fin(u, v); }\n";
          continue;
        }
        s << "    float2 t" << st + 1 << "_" << out_slot << " = make_float2(0.f, 0.f);\n";
        for (int k = 0; k < K; ++k) {
          const int in_slot = kt.tab[cs.rd_off + r * K + k];
          const bool ex = st == 0 && g.n_exp > 0;  // W block [k][e][n]
          s << "    t" << st + 1 << "_" << out_slot << " = " << cm << "(t" << st + 1 << "_"
            << out_slot << ", t" << st << "_" << in_slot << ", ";
          if (hoist[size_t(st)])
            s << "w" << st << "_" << k * N + n << ");\n";
          else
            s << "sw[" << (ex ? "wr + " : "") << cs.w_smem + k * (N << (ex ? g.n_exp : 0)) + n
              << "]);\n";
        }
      }
  }
  s << "    float2 *q = O + RO((unsigned)row) + ol;\n";
  const int last = g.n_stages;
  if (oswap) emit_exchange(s, "t" + std::to_string(last) + "_", g.lo, oj, os_);
  emit_tile_io(s, false, "q", oout, g.lo, vmax,
               [last](int j) { return "t" + std::to_string(last) + "_" + std::to_string(j); },
               "    ");
  s << (g.n_exp > 0 ? "  }\n  }\n" : "  }\n") << "#undef RX\n#undef RO\n}\n";
  return s.str();
}

// One compiled chain kernel per (source, device).
std::mutex g_mu;
std::map<std::pair<std::string, int>, CUfunction> g_fns;
std::map<std::string, std::vector<char>> g_cubins;  // source -> cubin (any device)

const char *const kOpts[] = {"--gpu-architecture=sm_100a", "-std=c++17", "--fmad=false"};
constexpr int kNOpts = 3;

uint64_t fnv1a(const std::string &s) {
  uint64_t h = 1469598103934665603ull;
  for (unsigned char c : s) h = (h ^ c) * 1099511628211ull;
  return h;
}

// On-disk cubin cache shared by the processes of one host (tests, smoke, bench each
// create plans): $STN_JIT_CACHE, else jit_cache/ next to this library. Best effort:
// any I/O problem just means a recompile.
std::string cache_dir() {
  const char *e = std::getenv("STN_JIT_CACHE");
  if (e && *e) return e;
  Dl_info info;
  if (dladdr(reinterpret_cast<void *>(&cache_dir), &info) && info.dli_fname) {
    std::string so = info.dli_fname;
    const size_t slash = so.rfind('/');
    if (slash != std::string::npos) return so.substr(0, slash) + "/jit_cache";
  }
  return "/tmp/stn_exec_jit";
}

std::string cache_path(const std::string &src) {
  char name[64];
  snprintf(name, sizeof name, "/chain_%016llx_%zu.cubin", (unsigned long long)fnv1a(src),
           src.size());
  return cache_dir() + name;
}

bool read_file(const std::string &path, std::vector<char> *out) {
  FILE *f = fopen(path.c_str(), "rb");
  if (!f) return false;
  fseek(f, 0, SEEK_END);
  const long n = ftell(f);
  fseek(f, 0, SEEK_SET);
  out->resize(size_t(n > 0 ? n : 0));
  const bool ok = n > 0 && fread(out->data(), 1, size_t(n), f) == size_t(n);
  fclose(f);
  return ok;
}

void write_file(const std::string &path, const std::vector<char> &data) {
  std::string dir = cache_dir(), cur;
  for (size_t i = 0; i <= dir.size(); ++i)  // mkdir -p
    if (i == dir.size() || dir[i] == '/') {
      if (!cur.empty()) mkdir(cur.c_str(), 0755);
      if (i < dir.size()) cur += '/';
    } else {
      cur += dir[i];
    }
  const std::string tmp = path + ".tmp" + std::to_string(getpid());
  FILE *f = fopen(tmp.c_str(), "wb");
  if (!f) return;
  const bool ok = fwrite(data.data(), 1, data.size(), f) == data.size();
  fclose(f);
  if (ok) rename(tmp.c_str(), path.c_str());
  else unlink(tmp.c_str());
}

bool nvrtc_compile(const std::string &src, std::vector<char> *cubin, std::string *log) {
  Nvrtc &nv = Nvrtc::get();
  void *prog = nullptr;
  if (nv.Create(&prog, src.c_str(), "stn_chain.cu", 0, nullptr, nullptr) != 0) return false;
  const int rc = nv.Compile(prog, kNOpts, kOpts);
  if (rc != 0) {
    size_t n = 0;
    nv.GetLogSize(prog, &n);
    std::string l(n, '\0');
    nv.GetLog(prog, &l[0]);
    if (log) *log = l;
    nv.Destroy(&prog);
    return false;
  }
  size_t n = 0;
  nv.GetCubinSize(prog, &n);
  cubin->resize(n);
  nv.GetCubin(prog, cubin->data());
  nv.Destroy(&prog);
  return true;
}

}  // namespace

bool chain_jit_available() { return Nvrtc::get().ok && Driver::get().ok; }

bool chain_jit_compile_only(const std::vector<ChainJitSpec> &chains, bool exact,
                            std::string *log) {
  Nvrtc &nv = Nvrtc::get();
  if (!nv.ok) {
    if (log) *log = "NVRTC not available";
    return false;
  }
  std::string src = kPrelude;
  for (size_t i = 0; i < chains.size(); ++i)
    src += emit(*chains[i].geom, *chains[i].tables, int(i), exact);
  void *prog = nullptr;
  if (nv.Create(&prog, src.c_str(), "stn_chains.cu", 0, nullptr, nullptr) != 0) return false;
  const int rc = nv.Compile(prog, kNOpts, kOpts);
  size_t n = 0;
  nv.GetLogSize(prog, &n);
  std::string l(n, '\0');
  nv.GetLog(prog, &l[0]);
  l.resize(strlen(l.c_str()));  // the log's terminating NUL
  if (log)
    *log = l + (rc == 0 && !debug_opt("chain_src") ? "" : "\n--- source ---\n" + src);
  nv.Destroy(&prog);
  return rc == 0;
}

bool chain_jit_compile(const std::vector<ChainJitSpec> &chains, bool exact, int device,
                       std::vector<void *> *fns_out, std::string *log,
                       std::vector<int> *local_out, std::vector<void *> *alt_out) {
  const size_t nc = chains.size();
  fns_out->assign(nc, nullptr);
  if (local_out) local_out->assign(nc, 0);
  if (alt_out) alt_out->assign(nc, nullptr);
  if (chains.empty()) return true;
  if (!chain_jit_available()) {
    if (log) *log = "NVRTC or the driver module API is not available";
    return false;
  }
  // one program per chain: independent, so they compile on parallel host threads. With
  // alt_out, a second variant of every chain capped at 128 registers (two CTAs per SM);
  // launch_chain_op times both on their first run and keeps the faster
  const size_t nv = alt_out ? 2 * nc : nc;
  std::vector<std::string> srcs(nv);
  for (size_t i = 0; i < nv; ++i)
    srcs[i] = std::string(kPrelude) +
              emit(*chains[i % nc].geom, *chains[i % nc].tables, 0, exact, i < nc ? 1 : 2);
  std::vector<void *> fnv(nv, nullptr);
  std::vector<int> localv(nv, 0);
  std::vector<void *> *fns = &fnv;
  std::vector<int> *local_bytes = &localv;
  std::vector<std::vector<char>> cubins(nv);
  std::vector<char> have(nv, 0);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < nv; ++i) {
      auto it = g_fns.find({srcs[i], device});
      if (it != g_fns.end()) {
        (*fns)[i] = it->second;
        have[i] = 2;
        continue;
      }
      auto c = g_cubins.find(srcs[i]);
      if (c != g_cubins.end()) {
        cubins[i] = c->second;
        have[i] = 1;
      }
    }
  }
  for (size_t i = 0; i < nv; ++i)
    if (!have[i] && read_file(cache_path(srcs[i]), &cubins[i])) have[i] = 1;
  std::vector<size_t> todo;
  for (size_t i = 0; i < nv; ++i)
    if (!have[i]) todo.push_back(i);
  std::vector<std::string> logs(nv);
  std::vector<char> ok(nv, 1);
  if (!todo.empty()) {
    const unsigned hw = std::max(1u, std::thread::hardware_concurrency());
    const size_t nt = std::min<size_t>(todo.size(), hw);
    std::atomic<size_t> next{0};
    std::vector<std::thread> pool;
    for (size_t t = 0; t < nt; ++t)
      pool.emplace_back([&] {
        for (;;) {
          const size_t q = next.fetch_add(1);
          if (q >= todo.size()) return;
          const size_t i = todo[q];
          ok[i] = nvrtc_compile(srcs[i], &cubins[i], &logs[i]) ? 1 : 0;
          if (ok[i]) write_file(cache_path(srcs[i]), cubins[i]);
        }
      });
    for (auto &t : pool) t.join();
  }
  std::lock_guard<std::mutex> lk(g_mu);
  for (size_t i = 0; i < nv; ++i) {
    if (have[i] == 2) {
      if (local_bytes && Driver::get().FuncGetAttribute)
        Driver::get().FuncGetAttribute(&(*local_bytes)[i], CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES,
                                       static_cast<CUfunction>((*fns)[i]));
      continue;
    }
    if (!ok[i]) {
      if (log) *log = logs[i];
      return false;
    }
    g_cubins[srcs[i]] = cubins[i];
    CUmodule mod = nullptr;
    CUfunction f = nullptr;
    if (Driver::get().ModuleLoadData(&mod, cubins[i].data()) != CUDA_SUCCESS ||
        Driver::get().ModuleGetFunction(&f, mod, "stn_chain_0") != CUDA_SUCCESS) {
      if (log) *log = "cuModuleLoadData / cuModuleGetFunction failed";
      return false;
    }
    // W lives in dynamic shared memory next to 16 KiB of row tables: opt in to 80 KiB
    if (Driver::get().FuncSetAttribute)
      Driver::get().FuncSetAttribute(f, CU_FUNC_ATTRIBUTE_MAX_DYNAMIC_SHARED_SIZE_BYTES,
                                     16 * kChainMaxW);
    g_fns[{srcs[i], device}] = f;
    (*fns)[i] = f;
    if (local_bytes && Driver::get().FuncGetAttribute)
      Driver::get().FuncGetAttribute(&(*local_bytes)[i], CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
    if (debug_opt("sweep_debug") && Driver::get().FuncGetAttribute) {
      int regs = 0, local = 0;
      Driver::get().FuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
      Driver::get().FuncGetAttribute(&local, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
      fprintf(stderr, "chain kernel %zu%s: li %d lo %d stages %d, %d registers, %d B local\n",
              i % nc, i < nc ? "" : " (128-register variant)", chains[i % nc].geom->li,
              chains[i % nc].geom->lo, chains[i % nc].geom->n_stages, regs, local);
    }
  }
  for (size_t i = 0; i < nc; ++i) {
    (*fns_out)[i] = fnv[i];
    if (local_out) (*local_out)[i] = localv[i];
    // the capped variant only where it does not spill
    if (alt_out && localv[nc + i] == 0) (*alt_out)[i] = fnv[nc + i];
  }
  return true;
}

bool chain_prefetch(const ChainGeom &g) {
  // the next row's input tile costs 2 registers per complex value: pipelined while
  // both input tiles and the largest stage tile stay within ~200 registers (a 64-value
  // output tile with an 8-value input, cfg5 1155, keeps it; 64-value inputs do not)
  const char *pf = debug_opt("chain_pf_log");
  const int pf_log = pf ? std::atoi(pf) : 5;
  return g.li <= pf_log && 4 * (1 << g.li) + 2 * (1 << g.ma) <= 200;
}

bool chain_swaps_allowed(const ChainGeom &g) {
  // the exchange keeps both halves of every pair live: only for kernels whose tiles
  // leave registers to spare (~2 per float of the input tile(s) and the largest tile)
  // -- cfg5 chain 1162-1170 (li 5, prefetched, ma 5) spilled with it: 10.3 -> 13.4 ms
  const int est = 2 * (1 << g.li) * (chain_prefetch(g) ? 2 : 1) + 2 * (1 << g.ma);
  return est <= 160;
}

bool chain_lane_swap(const int64_t *lane_off, const int64_t *elem_off, int n_log, int *j, int *s) {
  const char *sw = debug_opt("chain_swap");  // STN_DEBUG chain_swap=0: no exchanges
  if (sw && std::atoi(sw) == 0) return false;
  int l0 = -1, s1 = -1, s0 = -1;
  for (int b = 0; b < 5; ++b)
    if (lane_off[1 << b] == 1) l0 = b;
  for (int b = 0; b < n_log; ++b) {
    if (elem_off[1 << b] == 1) s0 = b;
    if (elem_off[1 << b] == 2) s1 = b;
  }
  if (l0 < 0 || s1 < 0 || s0 >= 0) return false;
  int best = -1;  // the tile line at the highest position moves to the lanes
  for (int b = 0; b < n_log; ++b)
    if (b != s1 && (best < 0 || elem_off[1 << b] > elem_off[1 << best])) best = b;
  if (best < 0) return false;
  *j = l0;
  *s = best;
  return true;
}

void chain_apply_swap(const int64_t *lane_off, const int64_t *elem_off, int n_log, int j, int s,
                      int64_t *lane_out, int64_t *elem_out) {
  const int64_t dl = lane_off[1 << j], ds = elem_off[1 << s];
  for (int l = 0; l < 32; ++l) lane_out[l] = lane_off[l] + (((l >> j) & 1) ? ds - dl : 0);
  for (int i = 0; i < (1 << n_log); ++i) elem_out[i] = elem_off[i] + (((i >> s) & 1) ? dl - ds : 0);
}

cudaError_t chain_jit_launch(void *fn, const ChainGeom &g, const ChainTables *T,
                             const BatchPtrs &p, cudaStream_t stream) {
  // the 32-byte tile accesses need 32-byte aligned tensors (arena blocks are)
  if ((reinterpret_cast<uintptr_t>(p.a) | reinterpret_cast<uintptr_t>(p.out)) % 32 != 0 ||
      (p.nbatch > 1 && (p.a_bs % 4 != 0 || p.out_bs % 4 != 0)))
    return cudaErrorMisalignedAddress;
  JitArgs a{};
  a.x = p.a;
  a.o = p.out;
  a.x_bs = p.a_bs;
  a.o_bs = p.out_bs;
  for (int s = 0; s < g.n_stages; ++s) {
    a.w[s] = g.w[s];
    a.w_bs[s] = g.w_bs[s];
  }
  a.tabs = T;
  a.rows = g.rows;
  void *params[] = {&a};
  // persistent over rows: up to 8 CTAs of 256 threads per SM
  const long long want = (g.rows + 8 * 4 - 1) / (8 * 4);
  long long gx = 148LL * 8 / (p.nbatch > 0 ? p.nbatch : 1);
  if (gx > want) gx = want;
  if (gx < 1) gx = 1;
  // W bytes: 8 per element, 16 in the (opt-in) FFMA2 form
  const unsigned smem = unsigned((debug_opt("chain_ffma2") ? 16 : 8) * std::max(g.w_total, 1));
  const CUresult r = Driver::get().LaunchKernel(static_cast<CUfunction>(fn), unsigned(gx),
                                                unsigned(p.nbatch), 1, 256, 1, 1, smem,
                                                reinterpret_cast<CUstream>(stream), params,
                                                nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

}  // namespace stn
