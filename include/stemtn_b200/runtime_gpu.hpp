// Drop-in GPU executor for the reference `stemtn` runtime.
//
// A reference caller switches by replacing
//     BranchCache cache = build_branch_cache(plan);            // runtime.hpp:492
//     SubtaskResult r   = run_subtask(plan, a, &cache);         // runtime.hpp:502
//     auto [sum, rep]   = run_scheme(plan, parallelism);        // runtime.hpp:555
// with
//     stemtn::b200::GpuPlan gp(plan);                           // upload once
//     stemtn::b200::GpuBranchCache cache = stemtn::b200::build_branch_cache(gp);
//     SubtaskResult r = stemtn::b200::run_subtask(gp, a, &cache);
//     auto [sum, rep] = stemtn::b200::run_scheme(gp, parallelism);
// Results come back in the reference's own types (Tensor, SubtaskResult,
// RunReport); failures throw stemtn::Error with the reference ErrorKind.
// Header-only; link with libstn_exec.so.
#pragma once

#include <algorithm>
#include <cmath>
#include <memory>
#include <string>
#include <utility>
#include <vector>

#include "stemtn/runtime.hpp"
#include "stemtn_b200/flatten.hpp"
#include "stn_exec.h"

namespace stemtn::b200 {

inline void check(int status) {
  if (status == STN_OK) return;
  std::string msg = stn_last_error();
  if (status >= 1 && status <= 19) throw Error(ErrorKind(status - 1), msg);
  // executor-side conditions (CUDA, memory, device) surface as SubtaskFailure,
  // the reference's kind for "a subtask could not be executed"
  throw Error(ErrorKind::SubtaskFailure, std::string(stn_status_name(status)) + ": " + msg);
}

// Device-resident copy of an ExecutablePlan. `mode` is STN_MODE_FAST (default)
// or STN_MODE_EXACT (bitwise identical to the reference CPU path).
class GpuPlan {
 public:
  explicit GpuPlan(const ExecutablePlan &plan, int device = 0, int mode = STN_MODE_FAST)
      : plan_(&plan), flat_(flatten(plan)) {
    stn_plan *p = nullptr;
    check(stn_plan_create(flat_.view(), device, mode, &p));
    handle_.reset(p);
    check(stn_plan_get_info(p, &info_));
  }
  stn_plan *handle() const { return handle_.get(); }
  const ExecutablePlan &plan() const { return *plan_; }
  const stn_plan_info &info() const { return info_; }
  // Re-uploads a vertex tensor the caller changed in plan.net (what
  // frugal_sample does to the output projectors, sampler.hpp:206-213).
  void refresh_vertex(int vertex) {
    const Tensor &t = plan_->net.vertices.at(vertex).tensor;
    std::vector<double> v(2 * t.data.size());
    for (size_t i = 0; i < t.data.size(); ++i) {
      v[2 * i] = t.data[i].real();
      v[2 * i + 1] = t.data[i].imag();
    }
    check(stn_plan_set_leaf_values(handle(), vertex, v.data(), int64_t(t.data.size())));
  }

 private:
  struct Deleter {
    void operator()(stn_plan *p) const { stn_plan_destroy(p); }
  };
  const ExecutablePlan *plan_;
  FlatPlan flat_;
  std::unique_ptr<stn_plan, Deleter> handle_;
  stn_plan_info info_{};
};

class GpuBranchCache {
 public:
  GpuBranchCache() = default;
  explicit GpuBranchCache(stn_cache *c) : handle_(c) {
    check(stn_cache_info(c, &plan_identity, &mults, &elements));
  }
  stn_cache *handle() const { return handle_.get(); }
  std::uint64_t plan_identity = 0, mults = 0, elements = 0;

 private:
  struct Deleter {
    void operator()(stn_cache *c) const { stn_cache_destroy(c); }
  };
  std::unique_ptr<stn_cache, Deleter> handle_;
};

inline GpuBranchCache build_branch_cache(GpuPlan &gp) {
  stn_cache *c = nullptr;
  check(stn_cache_build(gp.handle(), nullptr, &c));
  return GpuBranchCache(c);
}

inline Tensor to_tensor(const GpuPlan &gp, const std::vector<double> &v) {
  std::vector<int> dims(gp.info().out_dims, gp.info().out_dims + gp.info().out_rank);
  Tensor t(dims);
  for (size_t i = 0; i < t.data.size(); ++i) t.data[i] = cx(v[2 * i], v[2 * i + 1]);
  return t;
}

inline SubtaskResult run_subtask(GpuPlan &gp, std::uint64_t assignment,
                                 const GpuBranchCache *cache = nullptr) {
  std::vector<double> out(2 * size_t(gp.info().out_elements));
  stn_subtask_info info{};
  check(stn_run_subtask(gp.handle(), assignment, cache ? cache->handle() : nullptr, nullptr,
                        out.data(), &info));
  SubtaskResult r;
  r.assignment = assignment;
  r.value = to_tensor(gp, out);
  r.step_count = info.step_count;
  r.mults = info.mults;
  r.peak_elements = info.peak_elements;
  return r;
}

inline std::pair<Tensor, RunReport> run_scheme(GpuPlan &gp, int parallelism = 1) {
  std::vector<double> out(2 * size_t(gp.info().out_elements));
  stn_run_report rep{};
  check(stn_run_scheme(gp.handle(), parallelism, out.data(), &rep));
  RunReport r;
  auto costs = gp.plan().scheme.costs();
  r.log2_tc = costs.log2_tc;
  r.cw = costs.cw;
  r.subtasks = rep.subtasks;
  r.mult_count = rep.mult_count;
  r.branch_mults = rep.branch_mults;
  r.wall_seconds = rep.wall_seconds;
  r.p50_ms = rep.p50_ms;
  r.p90_ms = rep.p90_ms;
  r.p99_ms = rep.p99_ms;
  r.parallelism = rep.parallelism;
  r.precision = precision_name(gp.plan().options.precision);
  r.peak_elements = rep.peak_elements;
  r.merged_groups = rep.merged_groups;
  return {to_tensor(gp, out), r};
}

// The GPUs of one box as one executor: what the reference's C++ consumers
// (frugal_sample's run_scheme, sampler.hpp:214; the worker/agent pair,
// queue.hpp:197-336) switch to for 8 GPUs. One device plan + branch cache per
// GPU, contiguous slice shards, and either the chained ascending fold (bitwise
// run_scheme for any device count) or one NCCL all-reduce.
class GpuMultiPlan {
 public:
  GpuMultiPlan(const ExecutablePlan &plan, const std::vector<int> &devices,
               int mode = STN_MODE_FAST)
      : plan_(&plan), flat_(flatten(plan)) {
    std::vector<int32_t> d(devices.begin(), devices.end());
    stn_multi *m = nullptr;
    check(stn_multi_create(flat_.view(), int(d.size()), d.data(), mode, &m));
    handle_.reset(m);
    check(stn_plan_get_info(stn_multi_plan(m, 0), &info_));
  }
  // All visible GPUs (or `n` of them).
  static std::vector<int> all_devices(int n = -1) {
    int c = stn_device_count();
    if (n > 0 && n < c) c = n;
    std::vector<int> d(size_t(std::max(c, 0)));
    for (int i = 0; i < c; ++i) d[size_t(i)] = i;
    return d;
  }
  stn_multi *handle() const { return handle_.get(); }
  const stn_plan_info &info() const { return info_; }
  // Re-uploads a poked vertex tensor on every GPU and rebuilds the branch caches
  // (frugal_sample's per-batch projector update, sampler.hpp:206-213).
  void refresh_vertex(int vertex) {
    const Tensor &t = plan_->net.vertices.at(vertex).tensor;
    std::vector<double> v(2 * t.data.size());
    for (size_t i = 0; i < t.data.size(); ++i) {
      v[2 * i] = t.data[i].real();
      v[2 * i + 1] = t.data[i].imag();
    }
    check(stn_multi_set_leaf_values(handle(), vertex, v.data(), int64_t(t.data.size())));
    stale_ = true;
  }
  std::pair<Tensor, RunReport> run_scheme(bool deterministic = true) {
    if (stale_) {
      check(stn_multi_build_caches(handle()));
      stale_ = false;
    }
    std::vector<double> out(2 * size_t(info_.out_elements));
    stn_run_report rep{};
    check(stn_multi_run_scheme(handle(), deterministic ? 1 : 0, out.data(), &rep));
    RunReport r;
    auto costs = plan_->scheme.costs();
    r.log2_tc = costs.log2_tc;
    r.cw = costs.cw;
    r.subtasks = rep.subtasks;
    r.mult_count = rep.mult_count;
    r.branch_mults = rep.branch_mults;
    r.wall_seconds = rep.wall_seconds;
    r.p50_ms = rep.p50_ms;
    r.p90_ms = rep.p90_ms;
    r.p99_ms = rep.p99_ms;
    r.parallelism = rep.parallelism;
    r.precision = precision_name(plan_->options.precision);
    r.peak_elements = rep.peak_elements;
    r.merged_groups = plan_->merged_groups;
    std::vector<int> dims(info_.out_dims, info_.out_dims + info_.out_rank);
    Tensor t(dims);
    for (size_t i = 0; i < t.data.size(); ++i) t.data[i] = cx(out[2 * i], out[2 * i + 1]);
    return {t, r};
  }

 private:
  struct Deleter {
    void operator()(stn_multi *m) const { stn_multi_destroy(m); }
  };
  const ExecutablePlan *plan_;
  FlatPlan flat_;
  std::unique_ptr<stn_multi, Deleter> handle_;
  stn_plan_info info_{};
  bool stale_ = false;
};

}  // namespace stemtn::b200
