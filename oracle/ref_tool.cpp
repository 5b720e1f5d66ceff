// TEST INFRASTRUCTURE ONLY -- the reference oracle driver (`oracle/_ref/ref_tool`).
//
// Compiled from the reference's own headers where they lie
// (`/root/reference/proj/include`, read-only, never copied) with the two build
// shims in oracle/shim (Boost cpp_int, nlohmann json). It is used to
//   (1) produce workloads through the reference pipeline: circuit generation
//       (circuit.hpp:307), circuit_to_network (circuit.hpp:570), the planner
//       (planner.hpp:605) and compile (runtime.hpp:243), writing the reference
//       file formats (network.json: network.hpp:361; order.json: scheme.hpp:52)
//       plus the flattened plan for the B200 executor (include/stemtn_b200/flatten.hpp);
//   (2) record golden outputs of the reference CPU executor: run_subtask
//       (runtime.hpp:502) per slice and run_scheme (runtime.hpp:555) sums;
//   (3) time the reference CPU executor on this host (bench.py --impl reference).
// Nothing in the product links or executes this tool.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <fstream>
#include <iostream>
#include <sstream>
#include <string>
#include <thread>

#include "stemtn/circuit.hpp"
#include "stemtn/planner.hpp"
#include "stemtn/runtime.hpp"
#include "stemtn/sampler.hpp"
#include "stemtn/statevector.hpp"
#include "test_support.hpp"  // reference test fixtures (random_network), proj/tests

#include "stemtn_b200/flatten.hpp"

extern "C" void stn_set_error_c(const char *msg) { std::fprintf(stderr, "plan_io: %s\n", msg); }

using namespace stemtn;
using clk = std::chrono::steady_clock;

namespace {

struct Args {
  std::map<std::string, std::string> kv;
  std::vector<std::string> pos;
  Args(int argc, char **argv, int from) {
    for (int i = from; i < argc; ++i) {
      std::string a = argv[i];
      if (a.rfind("--", 0) == 0 && i + 1 < argc) {
        kv[a.substr(2)] = argv[++i];
      } else {
        pos.push_back(a);
      }
    }
  }
  std::string get(const std::string &k, const std::string &def) const {
    auto it = kv.find(k);
    return it == kv.end() ? def : it->second;
  }
  long long geti(const std::string &k, long long def) const {
    auto it = kv.find(k);
    return it == kv.end() ? def : std::atoll(it->second.c_str());
  }
  double getd(const std::string &k, double def) const {
    auto it = kv.find(k);
    return it == kv.end() ? def : std::atof(it->second.c_str());
  }
};

nlohmann::json read_json(const std::string &path) {
  std::ifstream in(path);
  require(bool(in), ErrorKind::MissingResult, "cannot read " + path);
  nlohmann::json j;
  in >> j;
  return j;
}

void write_text(const std::string &path, const std::string &s) {
  std::ofstream out(path);
  out << s;
  require(bool(out), ErrorKind::MissingResult, "cannot write " + path);
}

void write_plans(const std::string &dir, const TensorNetwork &net, const ContractionScheme &s,
                 int merge_min_dim, int width_budget) {
  for (Precision p : {Precision::Single, Precision::Double}) {
    CompileOptions co{merge_min_dim, p, width_budget};
    ExecutablePlan ep = compile(net, s, co);
    b200::FlatPlan fp = b200::flatten(ep);
    std::string path = dir + "/plan_" + precision_name(p) + ".stnplan";
    require(stn_plan_save(fp.view(), path.c_str()) == STN_OK, ErrorKind::MissingResult,
            "cannot write " + path);
  }
}

nlohmann::json plan_summary(const ExecutablePlan &ep) {
  std::uint64_t bm = 0, sm = 0;
  int nb = 0, ns = 0;
  for (const Step &s : ep.steps) {
    if (s.is_branch) {
      nb++;
      bm += s.mults;
    } else {
      ns++;
      sm += s.mults;
    }
  }
  auto c = ep.scheme.costs();
  double log2_slices = 0;
  for (int e : ep.scheme.sliced_edges) log2_slices += std::log2(double(ep.scheme.sliced_dims.at(e)));
  return {{"vertices", ep.net.vertex_count()},
          {"edges", ep.net.edge_count()},
          {"open_edges", ep.open_edges.size()},
          {"sliced_edges", ep.scheme.sliced_edges.size()},
          {"log2_slices", log2_slices},
          {"subtasks_u64", ep.subtasks},
          {"scheme_cw", c.cw},
          {"scheme_log2_tc", c.log2_tc},
          {"exec_cw", ep.exec_cw},
          {"log2_exec_tc", log2_big(ep.exec_tc)},
          {"merged_groups", ep.merged_groups},
          {"steps", ep.steps.size()},
          {"branch_steps", nb},
          {"per_slice_steps", ns},
          {"branch_mults", bm},
          {"per_slice_mults", sm},
          {"identity", ep.identity}};
}

ContractionScheme plan_with(const TensorNetwork &net, const Args &a) {
  PlannerParams p;
  p.seed = std::uint64_t(a.geti("plan-seed", 1));
  p.target_cw = int(a.geti("target-cw", 29));
  if (a.kv.count("restarts")) p.restarts = int(a.geti("restarts", 5));
  if (a.get("light", "0") == "1") {  // plan_light of test_runtime.cpp:17-24
    p.iterations = {6, 4, 2, 4};
    p.restarts = 2;
  }
  return plan(net, p).scheme;
}

// gen-circuit <outdir> --layout L --cycles m --open k --target-cw c [--circuit-seed s]
int cmd_gen_circuit(const Args &a) {
  std::string dir = a.pos.at(0);
  Layout L = Layout::named(a.get("layout", "grid4x5"));
  int m = int(a.geti("cycles", 14));
  int nopen = int(a.geti("open", 0));
  Circuit c = generate_random_circuit(L, m, std::uint64_t(a.geti("circuit-seed", 1)));
  std::set<int> open;
  if (nopen == 6) {
    for (int q : batch_qubit_selector(L, m)) open.insert(q);
  } else {
    for (int q = 0; q < nopen; ++q) open.insert(q);
  }
  std::map<int, int> fixed;
  for (int q = 0; q < L.qubit_count(); ++q)
    if (!open.count(q)) fixed[q] = 0;
  CircuitNetwork cn = circuit_to_network(c, open, fixed);
  auto t0 = clk::now();
  ContractionScheme s = plan_with(cn.net, a);
  double plan_s = std::chrono::duration<double>(clk::now() - t0).count();
  int merge = int(a.geti("merge-min-dim", 32)), width = int(a.geti("width-budget", 40));
  write_text(dir + "/network.json", cn.net.to_json().dump());
  write_text(dir + "/order.json", serialize_scheme(s).dump());
  write_plans(dir, cn.net, s, merge, width);
  ExecutablePlan ep = compile(cn.net, s, CompileOptions{merge, Precision::Single, width});
  nlohmann::json meta = {{"kind", "circuit"},
                         {"layout", L.name},
                         {"qubits", L.qubit_count()},
                         {"cycles", m},
                         {"open_qubits", std::vector<int>(open.begin(), open.end())},
                         {"circuit_seed", a.geti("circuit-seed", 1)},
                         {"plan_seed", a.geti("plan-seed", 1)},
                         {"target_cw", a.geti("target-cw", 29)},
                         {"merge_min_dim", merge},
                         {"width_budget", width},
                         {"plan_seconds", plan_s},
                         {"plan", plan_summary(ep)}};
  write_text(dir + "/meta.json", meta.dump(1));
  std::cout << meta.dump() << "\n";
  return 0;
}

// gen-random <outdir> --seed s [--vertices v --extra e --open o --hyper p --mixed 0/1]
//            --target-cw c [--light 1] [--merge-min-dim d]
int cmd_gen_random(const Args &a) {
  std::string dir = a.pos.at(0);
  Rng rng(std::uint64_t(a.geti("seed", 1)));
  stemtn::testing::RandomNetOptions opt;
  opt.vertices = int(a.geti("vertices", 6));
  opt.extra_edges = int(a.geti("extra", 3));
  opt.open_edges = int(a.geti("open", 1));
  opt.hyper_prob = a.getd("hyper", 0.2);
  opt.mixed_dims = a.get("mixed", "0") == "1";
  TensorNetwork net = stemtn::testing::random_network(rng, opt);
  ContractionScheme s = plan_with(net, a);
  int merge = int(a.geti("merge-min-dim", 32)), width = int(a.geti("width-budget", 30));
  write_text(dir + "/network.json", net.to_json().dump());
  write_text(dir + "/order.json", serialize_scheme(s).dump());
  write_plans(dir, net, s, merge, width);
  ExecutablePlan ep = compile(net, s, CompileOptions{merge, Precision::Double, width});
  Tensor fv = net.feynman_value();
  std::vector<double> fvals;
  for (const cx &v : fv.data) {
    fvals.push_back(v.real());
    fvals.push_back(v.imag());
  }
  nlohmann::json meta = {{"kind", "random"},
                         {"seed", a.geti("seed", 1)},
                         {"options",
                          {{"vertices", opt.vertices},
                           {"extra_edges", opt.extra_edges},
                           {"open_edges", opt.open_edges},
                           {"hyper_prob", opt.hyper_prob},
                           {"mixed_dims", opt.mixed_dims}}},
                         {"merge_min_dim", merge},
                         {"width_budget", width},
                         {"feynman_dims", fv.dims},
                         {"feynman_value", fvals},
                         {"plan", plan_summary(ep)}};
  write_text(dir + "/meta.json", meta.dump(1));
  std::cout << meta.dump() << "\n";
  return 0;
}

ExecutablePlan load_plan(const std::string &dir, Precision p, int merge, int width) {
  TensorNetwork net = TensorNetwork::from_json(read_json(dir + "/network.json"));
  ContractionScheme s = parse_scheme(read_json(dir + "/order.json"), net);
  return compile(net, s, CompileOptions{merge, p, width});
}

std::vector<std::uint64_t> parse_slices(const std::string &spec, std::uint64_t n) {
  std::vector<std::uint64_t> out;
  if (spec == "all") {
    for (std::uint64_t a = 0; a < n; ++a) out.push_back(a);
  } else if (spec.rfind("sample:", 0) == 0) {
    // first, last and K-2 seeded picks, ascending and de-duplicated
    std::uint64_t k = std::strtoull(spec.c_str() + 7, nullptr, 10);
    std::set<std::uint64_t> s{0, n - 1};
    Rng rng(0x5A17CE5ull);
    while (s.size() < std::min<std::uint64_t>(k, n)) s.insert(rng.next_below(n));
    out.assign(s.begin(), s.end());
  } else {
    std::stringstream ss(spec);
    std::string tok;
    while (std::getline(ss, tok, ',')) out.push_back(std::strtoull(tok.c_str(), nullptr, 10));
  }
  return out;
}

// golden <dir> --precision single|double --slices all|sample:K|a,b,c [--scheme 1] [--threads t]
// Writes ref_<precision>.bin:
//   u64 n_slices, u64 out_elems, u64 assignments[n], f64 values[n][2*out_elems],
//   u64 has_sum, f64 sum[2*out_elems], u64 step_count, u64 mults, u64 peak_elements
int cmd_golden(const Args &a) {
  std::string dir = a.pos.at(0);
  std::string prec = a.get("precision", "single");
  Precision p = prec == "double" ? Precision::Double : Precision::Single;
  int merge = int(a.geti("merge-min-dim", 32)), width = int(a.geti("width-budget", 40));
  auto tstart = clk::now();
  ExecutablePlan ep = load_plan(dir, p, merge, width);
  std::vector<std::uint64_t> slices = parse_slices(a.get("slices", "all"), ep.subtasks);
  BranchCache cache = build_branch_cache(ep);
  int threads = int(a.geti("threads", 1));
  std::vector<SubtaskResult> res(slices.size());
  std::atomic<std::size_t> next{0};
  auto worker = [&] {
    for (;;) {
      std::size_t i = next.fetch_add(1);
      if (i >= slices.size()) return;
      if (ep.subtasks == 0) {
        // subtasks() overflowed (>= 64 sliced bond-2 edges, scheme.hpp:33-37), so
        // run_subtask refuses every assignment (runtime.hpp:504). Engine::run itself
        // decodes a uint64 assignment as the mixed-radix digit vector whose leading
        // (most significant) digits are 0 (runtime.hpp:371-378): drive it directly.
        if (p == Precision::Single)
          res[i] = detail_rt::Engine<float>{ep, &cache.single}.run(slices[i]);
        else
          res[i] = detail_rt::Engine<double>{ep, &cache.dbl}.run(slices[i]);
      } else {
        res[i] = run_subtask(ep, slices[i], &cache);
      }
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
  for (auto &th : pool) th.join();
  std::uint64_t out_elems = res.empty() ? 0 : res[0].value.data.size();
  std::string path = dir + "/ref_" + prec + ".bin";
  // written to a temporary name and renamed at the end: a long run never leaves a
  // truncated fixture where the tests read it
  std::string tmp = path + ".partial";
  FILE *f = std::fopen(tmp.c_str(), "wb");
  require(f != nullptr, ErrorKind::MissingResult, "cannot write " + path);
  std::uint64_t n = slices.size();
  std::fwrite(&n, 8, 1, f);
  std::fwrite(&out_elems, 8, 1, f);
  std::fwrite(slices.data(), 8, n, f);
  for (const auto &r : res) std::fwrite(r.value.data.data(), 16, out_elems, f);
  std::uint64_t has_sum = a.get("scheme", "0") == "1" ? 1 : 0;
  std::fwrite(&has_sum, 8, 1, f);
  if (has_sum) {
    auto [sum, rep] = run_scheme(ep, threads);
    require(sum.data.size() == out_elems, ErrorKind::SubtaskFailure, "sum shape");
    std::fwrite(sum.data.data(), 16, out_elems, f);
  }
  std::uint64_t sc = res.empty() ? 0 : std::uint64_t(res[0].step_count);
  std::uint64_t mu = res.empty() ? 0 : res[0].mults;
  std::uint64_t pk = res.empty() ? 0 : res[0].peak_elements;
  std::fwrite(&sc, 8, 1, f);
  std::fwrite(&mu, 8, 1, f);
  std::fwrite(&pk, 8, 1, f);
  std::fclose(f);
  require(std::rename(tmp.c_str(), path.c_str()) == 0, ErrorKind::MissingResult,
          "cannot rename " + tmp);
  nlohmann::json j = {{"slices", n},
                      {"out_elems", out_elems},
                      {"precision", prec},
                      {"has_sum", has_sum},
                      {"cached", {{"step_count", sc}, {"mults", mu}, {"peak_elements", pk}}},
                      {"cache", {{"mults", cache.mults}, {"elements", cache.elements}}}};
  // no-cache run of slice 0 for the bookkeeping of SubtaskResult without a cache
  // (--uncached 0 skips it: it doubles the CPU time of the 53-qubit goldens)
  if (a.get("uncached", "1") == "1" && ep.subtasks != 0) {
    SubtaskResult nc = run_subtask(ep, slices.empty() ? 0 : slices[0], nullptr);
    j["uncached"] = {{"step_count", nc.step_count},
                     {"mults", nc.mults},
                     {"peak_elements", nc.peak_elements}};
  }
  j["cpu_seconds_wall"] = std::chrono::duration<double>(clk::now() - tstart).count();
  write_text(dir + "/ref_" + prec + ".json", j.dump(1));
  std::cout << j.dump() << "\n";
  return 0;
}

// bench <dir> --threads t --slices n [--first a]: reference CPU executor timing.
int cmd_bench(const Args &a) {
  std::string dir = a.pos.at(0);
  int threads = int(a.geti("threads", int(std::thread::hardware_concurrency())));
  int merge = int(a.geti("merge-min-dim", 32)), width = int(a.geti("width-budget", 40));
  auto t0 = clk::now();
  ExecutablePlan ep = load_plan(dir, Precision::Single, merge, width);
  auto t1 = clk::now();
  BranchCache cache = build_branch_cache(ep);
  auto t2 = clk::now();
  std::uint64_t n = std::uint64_t(a.geti("slices", 1));
  std::uint64_t first = std::uint64_t(a.geti("first", 0));
  std::atomic<std::uint64_t> next{0};
  std::vector<double> ms(n, 0.0);
  auto worker = [&] {
    for (;;) {
      std::uint64_t i = next.fetch_add(1);
      if (i >= n) return;
      auto s0 = clk::now();
      run_subtask(ep, (first + i) % std::max<std::uint64_t>(ep.subtasks, 1), &cache);
      ms[i] = std::chrono::duration<double, std::milli>(clk::now() - s0).count();
    }
  };
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t) pool.emplace_back(worker);
  for (auto &th : pool) th.join();
  auto t3 = clk::now();
  double run_s = std::chrono::duration<double>(t3 - t2).count();
  std::uint64_t per_slice = 0;
  for (const Step &s : ep.steps)
    if (!s.is_branch) per_slice += s.mults;
  nlohmann::json j = {{"slices", n},
                      {"threads", threads},
                      {"compile_seconds", std::chrono::duration<double>(t1 - t0).count()},
                      {"cache_seconds", std::chrono::duration<double>(t2 - t1).count()},
                      {"run_seconds", run_s},
                      {"slices_per_sec", double(n) / run_s},
                      {"flops_per_slice", 8.0 * double(per_slice)},
                      {"gflops", 8.0 * double(per_slice) * double(n) / run_s / 1e9},
                      {"slice_ms", ms}};
  std::cout << j.dump() << "\n";
  return 0;
}

// Mirror of Engine<float>::run (runtime.hpp:420-453) built from the reference's
// own Engine members (load_leaf, gemm) with a timer around every per-slice step.
// Stops after the step during which `budget_s` elapsed (budget_s <= 0: run all).
struct StepTimes {
  std::vector<double> ms;        // per executed per-slice step
  std::vector<std::uint64_t> mults;
  bool complete = false;
};

StepTimes time_slice_steps(const ExecutablePlan &ep, const BranchCache &cache,
                           std::uint64_t assignment, double budget_s) {
  detail_rt::Engine<float> eng{ep, &cache.single};
  std::map<int, detail_rt::TypedTensor<float>> live;
  StepTimes out;
  auto fetch = [&](int node) {
    auto it = live.find(node);
    if (it != live.end()) {
      auto v = std::move(it->second);
      live.erase(it);
      return v;
    }
    auto c = cache.single.find(node);
    if (c != cache.single.end()) return c->second;
    return eng.load_leaf(node, assignment);
  };
  auto t0 = clk::now();
  for (const Step &s : ep.steps) {
    if (s.is_branch) continue;
    auto s0 = clk::now();
    auto a = fetch(s.lhs);
    auto b = fetch(s.rhs);
    live.emplace(s.node, eng.gemm(s, a, b));
    out.ms.push_back(std::chrono::duration<double, std::milli>(clk::now() - s0).count());
    out.mults.push_back(s.mults);
    if (budget_s > 0 && std::chrono::duration<double>(clk::now() - t0).count() > budget_s)
      return out;
  }
  out.complete = true;
  return out;
}

// step-times <dir> [--slice a]: one full slice, single thread, per-step ms
int cmd_step_times(const Args &a) {
  std::string dir = a.pos.at(0);
  ExecutablePlan ep = load_plan(dir, Precision::Single, int(a.geti("merge-min-dim", 32)),
                                int(a.geti("width-budget", 40)));
  BranchCache cache = build_branch_cache(ep);
  StepTimes st = time_slice_steps(ep, cache, std::uint64_t(a.geti("slice", 0)), 0);
  double total = 0;
  for (double x : st.ms) total += x;
  nlohmann::json j = {{"slice", a.geti("slice", 0)}, {"total_ms", total}, {"step_ms", st.ms},
                      {"step_mults", st.mults}, {"threads", 1},
                      {"host_threads", std::thread::hardware_concurrency()}};
  std::cout << j.dump() << "\n";
  return 0;
}

// bench-prefix <dir> --threads T --budget S: every thread runs the per-slice
// steps of its own slice (the reference executor's own code) until S seconds
// have passed; reports per-thread per-step ms of the executed prefix.
int cmd_bench_prefix(const Args &a) {
  std::string dir = a.pos.at(0);
  int threads = int(a.geti("threads", int(std::thread::hardware_concurrency())));
  double budget = a.getd("budget", 20.0);
  ExecutablePlan ep = load_plan(dir, Precision::Single, int(a.geti("merge-min-dim", 32)),
                                int(a.geti("width-budget", 40)));
  BranchCache cache = build_branch_cache(ep);
  std::vector<StepTimes> res(threads);
  auto w0 = clk::now();
  std::vector<std::thread> pool;
  for (int t = 0; t < threads; ++t)
    pool.emplace_back([&, t] {
      res[t] = time_slice_steps(ep, cache, std::uint64_t(t) % std::max<std::uint64_t>(ep.subtasks, 1),
                                budget);
    });
  for (auto &th : pool) th.join();
  double wall = std::chrono::duration<double>(clk::now() - w0).count();
  nlohmann::json per = nlohmann::json::array();
  for (auto &r : res) per.push_back({{"step_ms", r.ms}, {"complete", r.complete}});
  nlohmann::json j = {{"threads", threads}, {"budget_s", budget}, {"wall_s", wall},
                      {"per_thread", per}};
  std::cout << j.dump() << "\n";
  return 0;
}

}  // namespace

int main(int argc, char **argv) {
  if (argc < 2) {
    std::fprintf(stderr, "usage: ref_tool gen-circuit|gen-random|golden|bench ...\n");
    return 2;
  }
  std::string cmd = argv[1];
  Args a(argc, argv, 2);
  try {
    if (cmd == "gen-circuit") return cmd_gen_circuit(a);
    if (cmd == "gen-random") return cmd_gen_random(a);
    if (cmd == "golden") return cmd_golden(a);
    if (cmd == "bench") return cmd_bench(a);
    if (cmd == "step-times") return cmd_step_times(a);
    if (cmd == "bench-prefix") return cmd_bench_prefix(a);
  } catch (const std::exception &e) {
    std::fprintf(stderr, "ref_tool: %s\n", e.what());
    return 3;
  }
  std::fprintf(stderr, "ref_tool: unknown command %s\n", cmd.c_str());
  return 2;
}
