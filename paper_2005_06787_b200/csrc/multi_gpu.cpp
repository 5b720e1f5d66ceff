// Several GPUs of one box behind the C ABI (include/stn_exec.h, "several GPUs").
//
// Replaces the reference's multi-worker layer -- envelopes of slices claimed by
// worker processes through a shared directory and summed by agent_collect in
// ascending envelope order (queue.hpp:197-336) -- and the worker threads of
// run_scheme (runtime.hpp:564-598): one device plan with its HBM-resident branch
// cache per GPU, one host thread per GPU, each GPU a contiguous balanced shard of
// the slices (ascending devices own ascending slices). The only cross-GPU data
// is the 2*out_elements fp64 accumulator (1 KiB for 64 amplitudes):
//   deterministic: the ascending fold (runtime.hpp:601-605) starts on the first
//                  GPU and continues on the next with the handed-over accumulator
//                  (one peer copy over NVLink per hop), so the result is bitwise
//                  run_scheme's for any device count;
//   otherwise:     every GPU folds its own shard and one ncclAllReduce (sum) over
//                  NVLink combines them. NCCL is loaded with dlopen on first use,
//                  so the library itself has no link-time NCCL dependency.
// Built only on the public ABI of stn_exec.cpp plus the CUDA runtime.
#include <dlfcn.h>

#include <algorithm>
#include <chrono>
#include <cstring>
#include <exception>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

#include "stn_exec.h"

extern "C" void stn_set_error_c(const char *msg);

namespace {

// ---- NCCL, resolved at run time ------------------------------------------------
// The handful of nccl.h (2.x) declarations this file needs; the ABI of these has
// been stable since NCCL 2.0.
typedef struct ncclComm *ncclComm_t;
enum { kNcclSuccess = 0, kNcclFloat64 = 8, kNcclSum = 0 };

struct Nccl {
  void *h = nullptr;
  int (*CommInitAll)(ncclComm_t *, int, const int *) = nullptr;
  int (*CommDestroy)(ncclComm_t) = nullptr;
  int (*AllReduce)(const void *, void *, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
  int (*GroupStart)() = nullptr;
  int (*GroupEnd)() = nullptr;
  const char *(*GetErrorString)(int) = nullptr;
  std::string error;

  static Nccl &get() {
    static Nccl n;
    static std::once_flag once;
    std::call_once(once, [] { n.load(); });
    return n;
  }
  void load() {
    for (const char *name : {"libnccl.so.2", "libnccl.so"}) {
      h = dlopen(name, RTLD_NOW | RTLD_GLOBAL);
      if (h) break;
    }
    if (!h) {
      error = std::string("cannot load NCCL (libnccl.so.2): ") + dlerror();
      return;
    }
    auto sym = [&](const char *n) {
      void *p = dlsym(h, n);
      if (!p) error = std::string("NCCL symbol missing: ") + n;
      return p;
    };
    CommInitAll = reinterpret_cast<decltype(CommInitAll)>(sym("ncclCommInitAll"));
    CommDestroy = reinterpret_cast<decltype(CommDestroy)>(sym("ncclCommDestroy"));
    AllReduce = reinterpret_cast<decltype(AllReduce)>(sym("ncclAllReduce"));
    GroupStart = reinterpret_cast<decltype(GroupStart)>(sym("ncclGroupStart"));
    GroupEnd = reinterpret_cast<decltype(GroupEnd)>(sym("ncclGroupEnd"));
    GetErrorString = reinterpret_cast<decltype(GetErrorString)>(sym("ncclGetErrorString"));
  }
  bool ok() const { return h && error.empty(); }
};

struct Failure {
  int status;
  std::string msg;
};

void check(int st, const char *what) {
  if (st != STN_OK) throw Failure{st, std::string(what) + ": " + stn_last_error()};
}
void cuda(cudaError_t e, const char *what) {
  if (e != cudaSuccess)
    throw Failure{e == cudaErrorMemoryAllocation ? STN_ERR_OUT_OF_MEMORY : STN_ERR_CUDA,
                  std::string(what) + ": " + cudaGetErrorString(e)};
}

template <class F>
int guarded(F &&f) {
  try {
    f();
    return STN_OK;
  } catch (const Failure &e) {
    stn_set_error_c(e.msg.c_str());
    return e.status;
  } catch (const std::bad_alloc &) {
    stn_set_error_c("host allocation failed");
    return STN_ERR_OUT_OF_MEMORY;
  } catch (const std::exception &e) {
    stn_set_error_c(e.what());
    return STN_ERR_INVALID_ARGUMENT;
  }
}

// Contiguous balanced shard of [0, n) owned by rank r of w (distributed.py's shard_range).
void shard(uint64_t n, int r, int w, uint64_t *lo, uint64_t *hi) {
  const uint64_t base = n / uint64_t(w), extra = n % uint64_t(w);
  *lo = uint64_t(r) * base + std::min<uint64_t>(uint64_t(r), extra);
  *hi = *lo + base + (uint64_t(r) < extra ? 1 : 0);
}

struct DeviceMem {
  int dev = 0;
  void *p = nullptr;
  size_t bytes = 0;
  void reserve(int d, size_t n) {
    if (n <= bytes && d == dev) return;
    release();
    dev = d;
    cuda(cudaSetDevice(d), "cudaSetDevice");
    cuda(cudaMalloc(&p, std::max<size_t>(n, 16)), "cudaMalloc");
    bytes = n;
  }
  void release() {
    if (p) {
      cudaSetDevice(dev);
      cudaFree(p);
    }
    p = nullptr;
    bytes = 0;
  }
  ~DeviceMem() { release(); }
  double *d() const { return static_cast<double *>(p); }
};

}  // namespace

struct stn_multi {
  std::vector<int> devices;
  std::vector<stn_plan *> plans;
  std::vector<stn_cache *> caches;
  std::vector<cudaStream_t> streams;
  std::vector<DeviceMem> rows, acc;
  std::vector<ncclComm_t> comms;
  stn_plan_info info{};
  int n_sliced = 0;
  int precision = STN_SINGLE;
  ~stn_multi() {
    if (!comms.empty() && Nccl::get().ok())
      for (auto c : comms) Nccl::get().CommDestroy(c);
    for (size_t i = 0; i < plans.size(); ++i) {
      cudaSetDevice(devices[i]);
      if (i < caches.size() && caches[i]) stn_cache_destroy(caches[i]);
      if (i < streams.size() && streams[i]) cudaStreamDestroy(streams[i]);
      rows[i].release();
      acc[i].release();
      stn_plan_destroy(plans[i]);
    }
  }
  int n() const { return int(devices.size()); }

  // Runs f(i) on one host thread per GPU; the first failure is rethrown.
  template <class F>
  void on_all(F &&f) {
    std::vector<Failure> errs(devices.size(), Failure{STN_OK, ""});
    std::vector<std::thread> th;
    for (int i = 0; i < n(); ++i)
      th.emplace_back([&, i] {
        int st = guarded([&] {
          cuda(cudaSetDevice(devices[i]), "cudaSetDevice");
          f(i);
        });
        if (st != STN_OK) errs[i] = Failure{st, stn_last_error()};
      });
    for (auto &t : th) t.join();
    for (auto &e : errs)
      if (e.status != STN_OK) throw e;
  }

  void build_caches() {
    on_all([&](int i) {
      if (caches[i]) stn_cache_destroy(caches[i]);
      caches[i] = nullptr;
      check(stn_cache_build(plans[i], streams[i], &caches[i]), "branch cache");
    });
  }

  // Runs every GPU's shard of the n slices; per-slice roots stay in rows[i]
  // (deterministic) or are folded into acc[i] (not).
  void run_shards(const int32_t *digits, uint64_t lo, uint64_t n_slices, bool keep_rows,
                  std::vector<double> *ms) {
    const size_t row = 2 * size_t(info.out_elements);
    std::vector<double> dev_ms(devices.size(), 0.0);
    on_all([&](int i) {
      uint64_t a, b;
      shard(n_slices, i, n(), &a, &b);
      acc[i].reserve(devices[i], 8 * row);
      cuda(cudaMemsetAsync(acc[i].p, 0, 8 * row, streams[i]), "memset");
      if (keep_rows) rows[i].reserve(devices[i], 8 * row * std::max<uint64_t>(b - a, 1));
      cudaEvent_t e0, e1;
      cuda(cudaEventCreate(&e0), "event");
      cuda(cudaEventCreate(&e1), "event");
      cuda(cudaEventRecord(e0, streams[i]), "event");
      if (b > a) {
        if (digits)
          check(stn_run_slices_digits(plans[i], caches[i], digits + a * size_t(n_sliced), b - a,
                                      streams[i], keep_rows ? nullptr : acc[i].d(),
                                      keep_rows ? rows[i].d() : nullptr),
                "run slices");
        else
          check(stn_run_slices(plans[i], caches[i], lo + a, lo + b, streams[i],
                               keep_rows ? nullptr : acc[i].d(),
                               keep_rows ? rows[i].d() : nullptr),
                "run slices");
      }
      cuda(cudaEventRecord(e1, streams[i]), "event");
      cuda(cudaEventSynchronize(e1), "event sync");
      float t = 0;
      cuda(cudaEventElapsedTime(&t, e0, e1), "event time");
      dev_ms[i] = double(t);
      cudaEventDestroy(e0);
      cudaEventDestroy(e1);
    });
    if (ms) *ms = dev_ms;
  }

  // Ascending fold chained across the GPUs; the result ends on the last GPU's acc.
  void chained_fold(uint64_t n_slices, double *sum_host) {
    const size_t row = 2 * size_t(info.out_elements);
    for (int i = 0; i < n(); ++i) {
      uint64_t a, b;
      shard(n_slices, i, n(), &a, &b);
      cuda(cudaSetDevice(devices[i]), "cudaSetDevice");
      if (i > 0) {  // hand the accumulator over (NVLink peer copy), then continue the fold
        cuda(cudaStreamSynchronize(streams[i - 1]), "stream sync");
        cuda(cudaMemcpyPeerAsync(acc[i].p, devices[i], acc[i - 1].p, devices[i - 1], 8 * row,
                                 streams[i]),
             "accumulator hand-over");
      }
      check(stn_fold_slices_ordered(rows[i].d(), b - a, info.out_elements, acc[i].d(),
                                    streams[i]),
            "ordered fold");
    }
    const int last = n() - 1;
    cuda(cudaSetDevice(devices[last]), "cudaSetDevice");
    cuda(cudaMemcpyAsync(sum_host, acc[last].p, 8 * row, cudaMemcpyDeviceToHost, streams[last]),
         "sum download");
    cuda(cudaStreamSynchronize(streams[last]), "stream sync");
  }

  bool distinct() const {
    std::vector<int> d(devices);
    std::sort(d.begin(), d.end());
    return std::adjacent_find(d.begin(), d.end()) == d.end();
  }

  // One NCCL all-reduce of the per-GPU partial folds. Several device plans on one
  // GPU (tests on a 1-GPU box) cannot form an NCCL communicator; their partials
  // are added on the first plan's device instead.
  void allreduce(double *sum_host) {
    const size_t row = 2 * size_t(info.out_elements);
    if (n() > 1 && !distinct()) {
      DeviceMem tmp;
      tmp.reserve(devices[0], 8 * row);
      for (int i = 1; i < n(); ++i) {
        cuda(cudaSetDevice(devices[i]), "cudaSetDevice");
        cuda(cudaStreamSynchronize(streams[i]), "stream sync");
        cuda(cudaSetDevice(devices[0]), "cudaSetDevice");
        cuda(cudaMemcpyPeerAsync(tmp.p, devices[0], acc[i].p, devices[i], 8 * row, streams[0]),
             "partial copy");
        check(stn_fold_slices_ordered(tmp.d(), 1, info.out_elements, acc[0].d(), streams[0]),
              "partial add");
      }
      cuda(cudaMemcpyAsync(sum_host, acc[0].p, 8 * row, cudaMemcpyDeviceToHost, streams[0]),
           "sum download");
      cuda(cudaStreamSynchronize(streams[0]), "stream sync");
      return;
    }
    if (n() > 1) {
      Nccl &nc = Nccl::get();
      if (!nc.ok()) throw Failure{STN_ERR_CUDA, nc.error};
      if (comms.empty()) {
        comms.resize(devices.size());
        int st = nc.CommInitAll(comms.data(), n(), devices.data());
        if (st != kNcclSuccess) {
          comms.clear();
          throw Failure{STN_ERR_CUDA, std::string("ncclCommInitAll: ") + nc.GetErrorString(st)};
        }
      }
      nc.GroupStart();
      for (int i = 0; i < n(); ++i) {
        cuda(cudaSetDevice(devices[i]), "cudaSetDevice");
        int st = nc.AllReduce(acc[i].p, acc[i].p, row, kNcclFloat64, kNcclSum, comms[i],
                              streams[i]);
        if (st != kNcclSuccess)
          throw Failure{STN_ERR_CUDA, std::string("ncclAllReduce: ") + nc.GetErrorString(st)};
      }
      int st = nc.GroupEnd();
      if (st != kNcclSuccess)
        throw Failure{STN_ERR_CUDA, std::string("ncclGroupEnd: ") + nc.GetErrorString(st)};
    }
    cuda(cudaSetDevice(devices[0]), "cudaSetDevice");
    cuda(cudaMemcpyAsync(sum_host, acc[0].p, 8 * row, cudaMemcpyDeviceToHost, streams[0]),
         "sum download");
    for (int i = 0; i < n(); ++i) {
      cuda(cudaSetDevice(devices[i]), "cudaSetDevice");
      cuda(cudaStreamSynchronize(streams[i]), "stream sync");
    }
  }

  void download_rows(uint64_t n_slices, double *per_slice_host) {
    const size_t row = 2 * size_t(info.out_elements);
    on_all([&](int i) {
      uint64_t a, b;
      shard(n_slices, i, n(), &a, &b);
      if (b > a)
        cuda(cudaMemcpyAsync(per_slice_host + a * row, rows[i].p, 8 * row * (b - a),
                             cudaMemcpyDeviceToHost, streams[i]),
             "per-slice download");
      cuda(cudaStreamSynchronize(streams[i]), "stream sync");
    });
  }
};

extern "C" {

int stn_device_count(void) {
  int n = 0;
  if (cudaGetDeviceCount(&n) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return n;
}

int stn_multi_create(const stn_plan_desc *desc, int n_devices, const int32_t *devices, int mode,
                     stn_multi **out) {
  if (!desc || !out || n_devices < 1) {
    stn_set_error_c("bad argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  *out = nullptr;
  auto m = new stn_multi;
  int st = guarded([&] {
    int count = 0;
    cuda(cudaGetDeviceCount(&count), "cudaGetDeviceCount");
    for (int i = 0; i < n_devices; ++i) {
      const int d = devices ? devices[i] : i;
      if (d < 0 || d >= count)
        throw Failure{STN_ERR_NO_DEVICE, "device " + std::to_string(d) + " not present"};
      m->devices.push_back(d);
    }
    const size_t k = m->devices.size();
    m->plans.assign(k, nullptr);
    m->caches.assign(k, nullptr);
    m->streams.assign(k, nullptr);
    m->rows.resize(k);
    m->acc.resize(k);
    m->on_all([&](int i) {
      check(stn_plan_create(desc, m->devices[i], mode, &m->plans[i]), "plan");
      cuda(cudaStreamCreateWithFlags(&m->streams[i], cudaStreamNonBlocking), "stream");
    });
    check(stn_plan_get_info(m->plans[0], &m->info), "plan info");
    m->n_sliced = m->info.n_sliced;
    m->precision = desc->precision;
    // peer access for the accumulator hand-over (a staged copy works without it)
    for (size_t i = 1; i < k; ++i) {
      int can = 0;
      cudaDeviceCanAccessPeer(&can, m->devices[i], m->devices[i - 1]);
      if (can) {
        cudaSetDevice(m->devices[i]);
        if (cudaDeviceEnablePeerAccess(m->devices[i - 1], 0) != cudaSuccess) cudaGetLastError();
      }
    }
    m->build_caches();
  });
  if (st != STN_OK) {
    delete m;
    return st;
  }
  *out = m;
  return STN_OK;
}

int stn_multi_destroy(stn_multi *m) {
  delete m;
  return STN_OK;
}

int stn_multi_device_count(const stn_multi *m) { return m ? m->n() : 0; }

stn_plan *stn_multi_plan(stn_multi *m, int i) {
  return m && i >= 0 && i < m->n() ? m->plans[size_t(i)] : nullptr;
}

int stn_multi_build_caches(stn_multi *m) {
  if (!m) {
    stn_set_error_c("NULL argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] { m->build_caches(); });
}

int stn_multi_set_leaf_values(stn_multi *m, int32_t vertex, const double *values,
                              int64_t n_complex) {
  if (!m || !values) {
    stn_set_error_c("NULL argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    for (int i = 0; i < m->n(); ++i)
      check(stn_plan_set_leaf_values(m->plans[size_t(i)], vertex, values, n_complex),
            "leaf values");
  });
}

int stn_multi_run_scheme(stn_multi *m, int deterministic, double *out_host,
                         stn_run_report *rep) {
  if (!m || !out_host) {
    stn_set_error_c("NULL argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    const uint64_t n = m->info.subtasks;
    if (n < 1)
      throw Failure{STN_ERR_SUBTASK_FAILURE,
                    "plan has no enumerable subtasks (uint64 subtask count overflowed)"};
    auto t0 = std::chrono::steady_clock::now();
    std::vector<double> ms;
    m->run_shards(nullptr, 0, n, deterministic != 0, &ms);
    if (deterministic)
      m->chained_fold(n, out_host);
    else
      m->allreduce(out_host);
    auto t1 = std::chrono::steady_clock::now();
    if (rep) {
      memset(rep, 0, sizeof *rep);
      uint64_t cm = 0, ce = 0, id = 0;
      check(stn_cache_info(m->caches[0], &id, &cm, &ce), "cache info");
      rep->subtasks = n;
      rep->branch_mults = cm;
      rep->mult_count = cm + m->info.per_slice_mults * n;
      rep->wall_seconds = std::chrono::duration<double>(t1 - t0).count();
      // per-slice device time: each GPU's shard time / its slice count
      std::vector<double> per;
      for (int i = 0; i < m->n(); ++i) {
        uint64_t a, b;
        shard(n, i, m->n(), &a, &b);
        for (uint64_t s = a; s < b; ++s) per.push_back(ms[size_t(i)] / double(b - a));
      }
      std::sort(per.begin(), per.end());
      auto q = [&](double f) {
        return per.empty() ? 0.0
                           : per[std::min(per.size() - 1, size_t(f * double(per.size() - 1) + 0.5))];
      };
      rep->p50_ms = q(0.5);
      rep->p90_ms = q(0.9);
      rep->p99_ms = q(0.99);
      rep->parallelism = m->n();
      rep->precision = m->precision;
      rep->peak_elements = m->info.peak_elements;
    }
  });
}

int stn_multi_run_slices(stn_multi *m, const int32_t *digits, uint64_t lo, uint64_t n_slices,
                         int deterministic, double *per_slice_host, double *sum_host) {
  if (!m) {
    stn_set_error_c("NULL argument");
    return STN_ERR_INVALID_ARGUMENT;
  }
  return guarded([&] {
    if (!digits && (lo > m->info.subtasks || n_slices > m->info.subtasks - lo))
      throw Failure{STN_ERR_SUBTASK_FAILURE, "assignment out of range"};
    const bool rows = per_slice_host || deterministic;
    m->run_shards(digits, lo, n_slices, rows, nullptr);
    if (per_slice_host) m->download_rows(n_slices, per_slice_host);
    if (sum_host) {
      if (deterministic) {
        m->chained_fold(n_slices, sum_host);
      } else {
        if (rows) {  // fold each GPU's rows first (the per-slice rows were kept)
          for (int i = 0; i < m->n(); ++i) {
            uint64_t a, b;
            shard(n_slices, i, m->n(), &a, &b);
            cuda(cudaSetDevice(m->devices[size_t(i)]), "cudaSetDevice");
            check(stn_fold_slices_ordered(m->rows[size_t(i)].d(), b - a, m->info.out_elements,
                                          m->acc[size_t(i)].d(), m->streams[size_t(i)]),
                  "ordered fold");
          }
        }
        m->allreduce(sum_host);
      }
    }
  });
}

int stn_run_scheme_multi(const stn_plan_desc *desc, int n_devices, const int32_t *devices,
                         int mode, int deterministic, double *out_host, stn_run_report *rep) {
  stn_multi *m = nullptr;
  int st = stn_multi_create(desc, n_devices, devices, mode, &m);
  if (st != STN_OK) return st;
  st = stn_multi_run_scheme(m, deterministic, out_host, rep);
  std::string err = st == STN_OK ? "" : stn_last_error();
  stn_multi_destroy(m);
  if (st != STN_OK) stn_set_error_c(err.c_str());
  return st;
}

}  // extern "C"
