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
  bool ok = false;
  static Nvrtc &get() {
    static Nvrtc n;
    static std::once_flag once;
    std::call_once(once, [] { n.load(); });
    return n;
  }
  void load() {
    for (const char *name : {"libnvrtc.so.12", "libnvrtc.so", "/usr/local/cuda/lib64/libnvrtc.so.12",
                             "/usr/local/cuda/lib64/libnvrtc.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_LOCAL);
      if (h) break;
    }
    if (!h) return;
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
// acc + x * w
__device__ __forceinline__ float2 cmx(float2 acc, float2 x, float2 w) {  // EXACT
  float re = __fsub_rn(__fmul_rn(x.x, w.x), __fmul_rn(x.y, w.y));
  float im = __fadd_rn(__fmul_rn(x.x, w.y), __fmul_rn(x.y, w.x));
  return make_float2(__fadd_rn(acc.x, re), __fadd_rn(acc.y, im));
}
__device__ __forceinline__ float2 cmf(float2 acc, float2 x, float2 w) {  // FAST
  acc.x = fmaf(x.x, w.x, acc.x); acc.x = fmaf(-x.y, w.y, acc.x);
  acc.y = fmaf(x.x, w.y, acc.y); acc.y = fmaf(x.y, w.x, acc.y);
  return acc;
}
)";

// Emits the kernel of one chain. `kt` is the host copy of its tables.
std::string emit(const ChainGeom &g, const ChainTables &kt, int id, bool exact) {
  std::ostringstream s;
  const int ni = 1 << g.li, no = 1 << g.lo;
  const char *cm = exact ? "cmx" : "cmf";
  s << "extern \"C\" __global__ void __launch_bounds__(256) stn_chain_" << id
    << "(const JitArgs a) {\n"
    << "  __shared__ long long sxr[1024], sor[1024];\n"
    << "  __shared__ float2 sw[" << (g.w_total > 0 ? g.w_total : 1) << "];\n"
    << "  for (int i = threadIdx.x; i < 1024; i += 256) { sxr[i] = a.tabs[i]; sor[i] = a.tabs[1024 + i]; }\n"
    << "  const long long b = blockIdx.y;\n";
  // W: one staging statement per element (constant offsets)
  int wi = 0;
  for (int st = 0; st < g.n_stages; ++st) {
    const ChainStage &cs = g.st[st];
    const int kn = 1 << (cs.lk + cs.ln);
    s << "  if (threadIdx.x < " << kn << ") {\n    const int i = threadIdx.x;\n"
      << "    const int widx[" << kn << "] = {";
    for (int i = 0; i < kn; ++i) s << (i ? "," : "") << kt.widx[cs.w_off + i];
    s << "};\n    sw[" << cs.w_smem << " + i] = a.w[" << st << "][b * a.w_bs[" << st
      << "] + widx[i]];\n  }\n";
    wi += kn;
  }
  (void)wi;
  s << "  __syncthreads();\n"
    << "  const int lane = threadIdx.x & 31;\n"
    << "  const long long xl = a.tabs[2048 + lane], ol = a.tabs[2080 + lane];\n"
    << "  const float2 *X = a.x + b * a.x_bs;\n  float2 *O = a.o + b * a.o_bs;\n"
    << "  const long long step = (long long)gridDim.x * 8;\n"
    << "  long long row = (long long)blockIdx.x * 8 + (threadIdx.x >> 5);\n"
    << "#define RX(r) (sxr[(r) & 255] + sxr[256 + (((r) >> 8) & 255)] + sxr[512 + (((r) >> 16) & 255)] + sxr[768 + (((r) >> 24) & 255)])\n"
    << "#define RO(r) (sor[(r) & 255] + sor[256 + (((r) >> 8) & 255)] + sor[512 + (((r) >> 16) & 255)] + sor[768 + (((r) >> 24) & 255)])\n";
  for (int i = 0; i < ni; ++i) s << "  float2 n" << i << " = make_float2(0.f, 0.f);\n";
  s << "  if (row < a.rows) {\n    const float2 *p = X + RX((unsigned)row) + xl;\n";
  for (int i = 0; i < ni; ++i) s << "    n" << i << " = ldcs2(p + " << kt.xin[i] << "LL);\n";
  s << "  }\n  for (; row < a.rows; row += step) {\n";
  for (int i = 0; i < ni; ++i) s << "    const float2 t0_" << i << " = n" << i << ";\n";
  s << "    { const long long nr = row + step;\n      if (nr < a.rows) {\n"
    << "        const float2 *p = X + RX((unsigned)nr) + xl;\n";
  for (int i = 0; i < ni; ++i) s << "        n" << i << " = ldcs2(p + " << kt.xin[i] << "LL);\n";
  s << "      }\n    }\n";
  for (int st = 0; st < g.n_stages; ++st) {
    const ChainStage &cs = g.st[st];
    const int R = 1 << cs.lr, K = 1 << cs.lk, N = 1 << cs.ln;
    for (int r = 0; r < R; ++r)
      for (int n = 0; n < N; ++n) {
        const int out_slot = kt.tab[cs.wr_off + r * N + n];
        s << "    float2 t" << st + 1 << "_" << out_slot << " = make_float2(0.f, 0.f);\n";
        for (int k = 0; k < K; ++k) {
          const int in_slot = kt.tab[cs.rd_off + r * K + k];
          s << "    t" << st + 1 << "_" << out_slot << " = " << cm << "(t" << st + 1 << "_"
            << out_slot << ", t" << st << "_" << in_slot << ", sw[" << cs.w_smem + k * N + n
            << "]);\n";
        }
      }
  }
  s << "    float2 *q = O + RO((unsigned)row) + ol;\n";
  for (int j = 0; j < no; ++j)
    s << "    stcs2(q + " << kt.oout[j] << "LL, t" << g.n_stages << "_" << j << ");\n";
  s << "  }\n#undef RX\n#undef RO\n}\n";
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
  if (log) *log = l + (rc == 0 ? "" : "\n--- source ---\n" + src);
  nv.Destroy(&prog);
  return rc == 0;
}

bool chain_jit_compile(const std::vector<ChainJitSpec> &chains, bool exact, int device,
                       std::vector<void *> *fns, std::string *log) {
  fns->assign(chains.size(), nullptr);
  if (chains.empty()) return true;
  if (!chain_jit_available()) {
    if (log) *log = "NVRTC or the driver module API is not available";
    return false;
  }
  // one program per chain: independent, so they compile on parallel host threads
  std::vector<std::string> srcs(chains.size());
  for (size_t i = 0; i < chains.size(); ++i)
    srcs[i] = std::string(kPrelude) + emit(*chains[i].geom, *chains[i].tables, 0, exact);
  std::vector<std::vector<char>> cubins(chains.size());
  std::vector<char> have(chains.size(), 0);
  {
    std::lock_guard<std::mutex> lk(g_mu);
    for (size_t i = 0; i < chains.size(); ++i) {
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
  for (size_t i = 0; i < chains.size(); ++i)
    if (!have[i] && read_file(cache_path(srcs[i]), &cubins[i])) have[i] = 1;
  std::vector<size_t> todo;
  for (size_t i = 0; i < chains.size(); ++i)
    if (!have[i]) todo.push_back(i);
  std::vector<std::string> logs(chains.size());
  std::vector<char> ok(chains.size(), 1);
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
  for (size_t i = 0; i < chains.size(); ++i) {
    if (have[i] == 2) continue;
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
    g_fns[{srcs[i], device}] = f;
    (*fns)[i] = f;
    if (debug_opt("sweep_debug") && Driver::get().FuncGetAttribute) {
      int regs = 0, local = 0;
      Driver::get().FuncGetAttribute(&regs, CU_FUNC_ATTRIBUTE_NUM_REGS, f);
      Driver::get().FuncGetAttribute(&local, CU_FUNC_ATTRIBUTE_LOCAL_SIZE_BYTES, f);
      fprintf(stderr, "chain kernel %zu: li %d lo %d stages %d, %d registers, %d B local\n", i,
              chains[i].geom->li, chains[i].geom->lo, chains[i].geom->n_stages, regs, local);
    }
  }
  return true;
}

cudaError_t chain_jit_launch(void *fn, const ChainGeom &g, const ChainTables *T,
                             const BatchPtrs &p, cudaStream_t stream) {
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
  const CUresult r = Driver::get().LaunchKernel(static_cast<CUfunction>(fn), unsigned(gx),
                                                unsigned(p.nbatch), 1, 256, 1, 1, 0,
                                                reinterpret_cast<CUstream>(stream), params,
                                                nullptr);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorLaunchFailure;
}

}  // namespace stn
