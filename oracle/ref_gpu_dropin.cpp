// TEST INFRASTRUCTURE -- the reference's own runtime tests, re-run with the B200
// executor swapped in through include/stemtn_b200/runtime_gpu.hpp.
//
// Built against the reference headers (so it can only be compiled where
// /root/reference exists) into oracle/_ref/ref_gpu_dropin and run on the GPU
// box by tests/test_gpu_dropin.py. Each case restates a TEST_CASE of
// /root/reference/proj/tests/test_runtime.cpp with `stemtn::b200::` calls in
// place of the CPU executor; the expected values come from the reference
// itself (statevector, feynman_value, the CPU run_scheme) in the same process.
#include <cstdio>
#include <cstring>
#include <functional>
#include <set>

#include "stemtn/circuit.hpp"
#include "stemtn/planner.hpp"
#include "stemtn/runtime.hpp"
#include "stemtn/statevector.hpp"
#include "test_support.hpp"

#include "stemtn_b200/runtime_gpu.hpp"

using namespace stemtn;
using stemtn::testing::random_network;
using stemtn::testing::tensor_close;

namespace {

int failures = 0;

void check(bool ok, const char *name, const std::string &detail = "") {
  std::printf("[%s] %s %s\n", ok ? "PASS" : "FAIL", name, detail.c_str());
  if (!ok) failures++;
}

ContractionScheme plan_light(const TensorNetwork &net, int target_cw, std::uint64_t seed) {
  PlannerParams p;  // test_runtime.cpp:17-24
  p.iterations = {6, 4, 2, 4};
  p.restarts = 2;
  p.seed = seed;
  p.target_cw = target_cw;
  return plan(net, p).scheme;
}

bool bits_equal(const Tensor &a, const Tensor &b) {
  return a.dims == b.dims &&
         std::memcmp(a.data.data(), b.data.data(), a.data.size() * sizeof(cx)) == 0;
}

double rel(const Tensor &a, const Tensor &b) {
  double scale = std::max(max_abs(b), 1e-300), w = 0;
  for (size_t i = 0; i < a.data.size(); ++i) w = std::max(w, std::abs(a.data[i] - b.data[i]));
  return w / scale;
}

}  // namespace

int main() {
  // test_runtime.cpp:54-72 -- unmerged plans replay the tree exactly (hyperedges -> D > 1)
  {
    double worst = 0;
    for (std::uint64_t seed = 0; seed < 8; ++seed) {
      Rng rng(stream_seed(1400, seed));
      stemtn::testing::RandomNetOptions opt;
      opt.vertices = 9;
      opt.extra_edges = 6;
      opt.open_edges = 2;
      opt.hyper_prob = 0.3;
      TensorNetwork net = random_network(rng, opt);
      ContractionScheme s = plan_light(net, 29, seed);
      CompileOptions co;
      co.merge_min_dim = 1;
      co.precision = Precision::Double;
      ExecutablePlan p = compile(net, s, co);
      b200::GpuPlan gp(p);
      auto [value, rep] = b200::run_scheme(gp, 1);
      worst = std::max(worst, rel(value, net.feynman_value()));
    }
    check(worst <= 1e-9, "unmerged plans replay the tree exactly", std::to_string(worst));
  }
  // test_runtime.cpp:176-200 -- branch cache is bitwise sound, both precisions
  {
    Rng rng(77);
    stemtn::testing::RandomNetOptions opt;
    opt.vertices = 10;
    opt.extra_edges = 8;
    opt.open_edges = 1;
    TensorNetwork net = random_network(rng, opt);
    ContractionScheme s = plan_light(net, 3, 3);
    bool ok = !s.sliced_edges.empty();
    for (Precision prec : {Precision::Single, Precision::Double}) {
      CompileOptions co;
      co.precision = prec;
      ExecutablePlan p = compile(net, s, co);
      b200::GpuPlan gp(p);
      b200::GpuBranchCache cache = b200::build_branch_cache(gp);
      ok &= cache.plan_identity == p.identity;
      for (std::uint64_t a = 0; a < std::min<std::uint64_t>(p.subtasks, 4); ++a) {
        SubtaskResult with = b200::run_subtask(gp, a, &cache);
        SubtaskResult without = b200::run_subtask(gp, a, nullptr);
        ok &= bits_equal(with.value, without.value) && with.mults < without.mults;
      }
    }
    check(ok, "branch cache is bitwise sound");
  }
  // test_runtime.cpp:202-213 -- stale branch caches are rejected
  {
    Rng rng(15);
    TensorNetwork net = random_network(rng);
    ContractionScheme s = plan_light(net, 29, 1);
    ExecutablePlan p = compile(net, s, CompileOptions{32, Precision::Double, 30});
    ExecutablePlan p2 = compile(net, s, CompileOptions{1, Precision::Double, 30});
    b200::GpuPlan g1(p), g2(p2);
    b200::GpuBranchCache cache = b200::build_branch_cache(g2);
    bool threw = false;
    try {
      b200::run_subtask(g1, 0, &cache);
    } catch (const Error &e) {
      threw = e.kind() == ErrorKind::SubtaskFailure;
    }
    check(threw, "stale branch caches are rejected");
  }
  // test_runtime.cpp:244-256 -- slicing-sum identity on the runtime path
  {
    Rng rng(99);
    stemtn::testing::RandomNetOptions opt;
    opt.vertices = 9;
    opt.extra_edges = 7;
    opt.open_edges = 2;
    TensorNetwork net = random_network(rng, opt);
    ContractionScheme s = plan_light(net, 3, 4);
    ExecutablePlan p = compile(net, s, CompileOptions{32, Precision::Double, 30});
    b200::GpuPlan gp(p);
    auto [sum, rep] = b200::run_scheme(gp, 1);
    check(!s.sliced_edges.empty() && tensor_close(sum, net.feynman_value(), 1e-10),
          "slicing-sum identity holds on the GPU runtime path");
  }
  // test_runtime.cpp:258-277 -- output bits identical across parallelism levels,
  // and (exact mode) identical to the reference CPU executor
  {
    Circuit c = generate_random_circuit(2, 5, 4, 77);
    std::set<int> open = {0, 1, 2};
    std::map<int, int> fixed;
    for (int q = 0; q < 10; ++q)
      if (!open.count(q)) fixed[q] = 0;
    TensorNetwork net = circuit_to_network(c, open, fixed).net;
    ContractionScheme s = plan_light(net, 10, 6);
    bool ok = true;
    for (Precision prec : {Precision::Single, Precision::Double}) {
      CompileOptions co;
      co.precision = prec;
      ExecutablePlan p = compile(net, s, co);
      b200::GpuPlan gp(p, 0, STN_MODE_EXACT);
      auto [v1, r1] = b200::run_scheme(gp, 1);
      auto [v8, r8] = b200::run_scheme(gp, 8);
      auto [vc, rc] = run_scheme(p, 2);  // the reference CPU executor
      ok &= bits_equal(v1, v8) && bits_equal(v1, vc) &&
            r1.deterministic_json() == rc.deterministic_json();
    }
    check(ok, "output bits identical across parallelism and equal to the CPU reference");
  }
  // test_runtime.cpp:279-306 -- batch amplitudes for a 12-qubit circuit match the oracle
  {
    Circuit c = generate_random_circuit(3, 4, 4, 900);
    std::set<int> open = {0, 1, 2, 3, 4, 5};
    std::map<int, int> fixed;
    Rng rng(31);
    for (int q = 0; q < 12; ++q)
      if (!open.count(q)) fixed[q] = int(rng.next_below(2));
    CircuitNetwork cn = circuit_to_network(c, open, fixed);
    ContractionScheme s = plan_light(cn.net, 16, 11);
    ExecutablePlan p = compile(cn.net, s, CompileOptions{32, Precision::Single, 30});
    b200::GpuPlan gp(p);  // FAST mode
    auto [amps, rep] = b200::run_scheme(gp, 2);
    std::vector<cx> psi = statevector(c);
    double scale = 0;
    for (const cx &v : psi) scale = std::max(scale, std::abs(v));
    double worst = 0;
    for (std::uint64_t x = 0; x < 64; ++x) {
      std::vector<int> bits(12, 0);
      for (auto &[q, b] : fixed) bits[q] = b;
      std::vector<int> tidx(6);
      for (int i = 0; i < 6; ++i) {
        int bit = int((x >> (5 - i)) & 1);
        bits[i] = bit;
        tidx[i] = bit;
      }
      worst = std::max(worst, std::abs(amps.at(tidx) - psi[bits_to_index(bits)]) / scale);
    }
    check(amps.data.size() == 64 && worst <= 1e-6, "batch amplitudes match the state vector",
          std::to_string(worst));
  }
  // test_runtime.cpp:308-322 -- empty circuit with one open qubit yields [1, 0]
  {
    Circuit c;
    c.layout = Layout::grid(1, 1);
    c.cycles = 0;
    Layer final_layer;
    final_layer.gates.push_back(make_custom({0}, {cx(1, 0), cx(0, 0), cx(0, 0), cx(1, 0)}));
    c.layers.push_back(std::move(final_layer));
    TensorNetwork net = circuit_to_network(c, {0}, {}).net;
    ContractionScheme s = plan_light(net, 29, 1);
    ExecutablePlan p = compile(net, s, CompileOptions{32, Precision::Double, 30});
    b200::GpuPlan gp(p);
    auto [v, rep] = b200::run_scheme(gp, 1);
    check(v.dims == std::vector<int>{2} && std::abs(v.data[0] - cx(1, 0)) < 1e-12 &&
              std::abs(v.data[1]) < 1e-12,
          "empty circuit with one open qubit yields [1, 0]");
  }
  // sampler.hpp:206-214 -- projector pokes between batches, cache rebuilt per batch
  {
    Circuit c = generate_random_circuit(3, 4, 6, 5);
    std::set<int> open = {0, 1, 2, 3, 4, 5};
    std::map<int, int> fixed;
    for (int q = 0; q < 12; ++q)
      if (!open.count(q)) fixed[q] = 0;
    CircuitNetwork cn = circuit_to_network(c, open, fixed);
    ContractionScheme s = plan_light(cn.net, 8, 2);
    ExecutablePlan p = compile(cn.net, s, CompileOptions{32, Precision::Single, 30});
    b200::GpuPlan gp(p, 0, STN_MODE_EXACT);
    bool ok = true;
    for (int batch = 0; batch < 3; ++batch) {
      for (const auto &[q, vid] : cn.out_vertex_of_qubit) {
        int bit = int(stream_seed(7, batch + 1, q) & 1);
        Tensor &t = p.net.vertices.at(vid).tensor;
        t.data[0] = cx(bit == 0 ? 1 : 0, 0);
        t.data[1] = cx(bit == 1 ? 1 : 0, 0);
        gp.refresh_vertex(vid);
      }
      auto [vg, rg] = b200::run_scheme(gp, 1);
      auto [vc, rc] = run_scheme(p, 1);
      ok &= bits_equal(vg, vc);
    }
    check(ok, "sampler-style projector updates stay bitwise equal to the CPU reference");
  }
  // runtime.hpp:555-605 across GPUs -- the multi-device executor (one plan + cache per
  // GPU, contiguous shards, chained ascending fold) gives the reference's run_scheme bits;
  // with one GPU present, three device plans share it
  {
    Circuit c = generate_random_circuit(3, 4, 8, 12);
    std::set<int> open = {0, 1, 2, 3, 4, 5};
    std::map<int, int> fixed;
    for (int q = 0; q < 12; ++q)
      if (!open.count(q)) fixed[q] = 0;
    CircuitNetwork cn = circuit_to_network(c, open, fixed);
    ContractionScheme s = plan_light(cn.net, 6, 3);
    ExecutablePlan p = compile(cn.net, s, CompileOptions{32, Precision::Single, 30});
    std::vector<int> devs = b200::GpuMultiPlan::all_devices(8);
    if (devs.size() < 2) devs = {0, 0, 0};
    b200::GpuMultiPlan mp(p, devs, STN_MODE_EXACT);
    auto [vm, rm] = mp.run_scheme(true);
    auto [vc, rc] = run_scheme(p, 4);
    check(p.subtasks > 1 && bits_equal(vm, vc) &&
              rm.deterministic_json() == rc.deterministic_json(),
          "multi-GPU run_scheme equals the CPU reference bitwise",
          std::to_string(devs.size()) + " device plan(s), " + std::to_string(p.subtasks) +
              " slices");
    auto [vf, rf] = mp.run_scheme(false);  // one NCCL all-reduce (no NCCL call on a single GPU)
    check(rel(vf, vc) <= 1e-12, "multi-GPU all-reduce sum within 1e-12",
          std::to_string(rel(vf, vc)));
  }
  std::printf("%d failure(s)\n", failures);
  return failures ? 1 : 0;
}
