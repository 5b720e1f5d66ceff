// Flattens a reference `stemtn::ExecutablePlan` (runtime.hpp:60-73) into the
// plain-old-data `stn_plan_desc` of the C ABI (include/stn_exec.h).
//
// Header-only; include it after the reference headers are on the include path
// (`-I <reference>/proj/include`). It reads only public fields of the plan:
//   - steps:        Step (runtime.hpp:41-49), group sizes recomputed from the
//                   exec tree exactly as compile() does (runtime.hpp:303-319)
//   - leaf_prep:    LeafPrep (runtime.hpp:51-58) + the vertex tensor
//                   (plan.net.vertices, network.hpp Vertex)
//   - sliced dims:  scheme.sliced_edges / sliced_dims (scheme.hpp:26-31)
#pragma once

#include <algorithm>
#include <cstdint>
#include <iterator>
#include <vector>

#include "stemtn/runtime.hpp"
#include "stn_exec.h"

namespace stemtn::b200 {

// Owns every array the descriptor points to. Moving it keeps the pointers valid
// (vectors move their buffers); copying is disabled.
struct FlatPlan {
  struct StepArrays {
    std::vector<int32_t> lperm, rperm, operm, out_dims;
  };
  struct LeafArrays {
    std::vector<int32_t> dims, sliced_axis, sliced_index, perm;
    std::vector<double> values;
  };
  std::vector<int32_t> sliced_dims;
  std::vector<StepArrays> step_arrays;
  std::vector<LeafArrays> leaf_arrays;
  std::vector<stn_step_desc> steps;
  std::vector<stn_leaf_desc> leaves;
  stn_plan_desc desc{};

  FlatPlan() = default;
  FlatPlan(const FlatPlan &) = delete;
  FlatPlan &operator=(const FlatPlan &) = delete;
  FlatPlan(FlatPlan &&) = default;
  FlatPlan &operator=(FlatPlan &&) = default;

  // Re-points the descriptor at the owned arrays (call after any mutation).
  const stn_plan_desc *view() {
    for (std::size_t i = 0; i < steps.size(); ++i) {
      steps[i].lperm = step_arrays[i].lperm.data();
      steps[i].rperm = step_arrays[i].rperm.data();
      steps[i].operm = step_arrays[i].operm.data();
      steps[i].out_dims = step_arrays[i].out_dims.data();
    }
    for (std::size_t i = 0; i < leaves.size(); ++i) {
      leaves[i].dims = leaf_arrays[i].dims.data();
      leaves[i].values = leaf_arrays[i].values.data();
      leaves[i].sliced_axis = leaf_arrays[i].sliced_axis.data();
      leaves[i].sliced_index = leaf_arrays[i].sliced_index.data();
      leaves[i].perm = leaf_arrays[i].perm.data();
    }
    desc.sliced_dims = sliced_dims.data();
    desc.n_sliced = int32_t(sliced_dims.size());
    desc.steps = steps.data();
    desc.n_steps = int32_t(steps.size());
    desc.leaves = leaves.data();
    desc.n_leaves = int32_t(leaves.size());
    return &desc;
  }
};

// Copies the current vertex tensor of `vertex` into the flat leaf (used after
// callers poke plan.net, e.g. the sampler's projector update).
inline void refresh_leaf_values(FlatPlan &fp, const ExecutablePlan &plan, int vertex) {
  for (std::size_t i = 0; i < fp.leaves.size(); ++i) {
    if (fp.leaves[i].vertex != vertex) continue;
    const Tensor &t = plan.net.vertices.at(vertex).tensor;
    auto &vals = fp.leaf_arrays[i].values;
    vals.resize(2 * t.data.size());
    for (std::size_t j = 0; j < t.data.size(); ++j) {
      vals[2 * j] = t.data[j].real();
      vals[2 * j + 1] = t.data[j].imag();
    }
  }
  fp.view();
}

inline FlatPlan flatten(const ExecutablePlan &plan) {
  FlatPlan fp;
  const ContractionTree &t = plan.exec_tree;
  fp.desc.precision = plan.options.precision == Precision::Single ? STN_SINGLE : STN_DOUBLE;
  fp.desc.merge_min_dim = plan.options.merge_min_dim;
  fp.desc.n_nodes = int32_t(t.nodes.size());
  fp.desc.root = t.root;
  fp.desc.identity = plan.identity;
  fp.desc.subtasks = plan.subtasks;
  fp.desc.merged_groups = plan.merged_groups;
  fp.desc.exec_cw = plan.exec_cw;
  fp.desc.n_open = int32_t(plan.open_edges.size());
  for (int e : plan.scheme.sliced_edges) fp.sliced_dims.push_back(plan.scheme.sliced_dims.at(e));

  for (const Step &s : plan.steps) {
    // axis-group sizes, as compile() partitions the edge sets (runtime.hpp:303-319)
    std::vector<int> la = t.nodes[s.lhs].alive_ids();
    std::vector<int> lb = t.nodes[s.rhs].alive_ids();
    std::vector<int> lu = t.nodes[s.node].alive_ids();
    std::vector<int> shared;
    std::set_intersection(la.begin(), la.end(), lb.begin(), lb.end(), std::back_inserter(shared));
    int nd = 0, nk = 0;
    for (int e : shared) (std::binary_search(lu.begin(), lu.end(), e) ? nd : nk)++;
    stn_step_desc d{};
    d.node = s.node;
    d.lhs = s.lhs;
    d.rhs = s.rhs;
    d.is_branch = s.is_branch ? 1 : 0;
    d.nd = nd;
    d.nk = nk;
    d.nm = int32_t(la.size()) - int32_t(shared.size());
    d.nn = int32_t(lb.size()) - int32_t(shared.size());
    d.D = s.D;
    d.M = s.M;
    d.N = s.N;
    d.K = s.K;
    d.mults = s.mults;
    d.lrank = int32_t(s.lperm.size());
    d.rrank = int32_t(s.rperm.size());
    d.orank = int32_t(s.operm.size());
    FlatPlan::StepArrays arr;
    arr.lperm.assign(s.lperm.begin(), s.lperm.end());
    arr.rperm.assign(s.rperm.begin(), s.rperm.end());
    arr.operm.assign(s.operm.begin(), s.operm.end());
    arr.out_dims.assign(s.out_dims.begin(), s.out_dims.end());
    fp.steps.push_back(d);
    fp.step_arrays.push_back(std::move(arr));
  }

  for (const auto &[node, prep] : plan.leaf_prep) {
    const Tensor &tensor = plan.net.vertices.at(prep.vertex).tensor;
    stn_leaf_desc d{};
    d.node = node;
    d.vertex = prep.vertex;
    d.rank = int32_t(tensor.dims.size());
    d.n_sliced = int32_t(prep.sliced_axes.size());
    d.perm_rank = int32_t(prep.perm.size());
    FlatPlan::LeafArrays arr;
    arr.dims.assign(tensor.dims.begin(), tensor.dims.end());
    arr.values.resize(2 * tensor.data.size());
    for (std::size_t j = 0; j < tensor.data.size(); ++j) {
      arr.values[2 * j] = tensor.data[j].real();
      arr.values[2 * j + 1] = tensor.data[j].imag();
    }
    for (const auto &[axis, slice_idx] : prep.sliced_axes) {
      arr.sliced_axis.push_back(axis);
      arr.sliced_index.push_back(slice_idx);
    }
    arr.perm.assign(prep.perm.begin(), prep.perm.end());
    fp.leaves.push_back(d);
    fp.leaf_arrays.push_back(std::move(arr));
  }
  fp.view();
  return fp;
}

}  // namespace stemtn::b200
