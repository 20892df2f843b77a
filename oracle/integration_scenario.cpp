// TEST INFRASTRUCTURE — the reference's own simulated cluster (run_scenario,
// proj/src/harness.cpp) with the GPU executor wired where the harness builds
// each node's executor (harness.cpp:255: std::make_unique<ToyExecutor>(),
// then PerturbingExecutor and, for corrupt_result, OffsetExecutor around it).
//
// The maintainer's one-line change there (ToyExecutor -> CudaExecutor) is made
// at link time, without touching a reference source: oracle/Makefile links
// the reference's compiled objects with ToyExecutor::run weakened in a copy of
// model.o, and this file supplies the strong definition, which runs the
// LinearToyModel batch on the GPU through credo::gpu::CudaExecutor (the
// reference's body, model.cpp:67-73, when g_gpu is off).
//
// For each scenario of the reference's own harness tests
// (tests/test_harness.cpp:233-296) it runs the cluster twice -- stock CPU
// executor, then GPU executor -- and checks: no deadlock, every request
// certified, check_invariants() empty, and the two rendered traces
// byte-identical (the fp64 GPU path is bit-exact, so every digest, vote and
// certificate in the run is the same).
//
// Then the reference's own strategy benchmark (bench_strategies,
// src/experiments.cpp:60-80: execute-then-agree vs agree-then-execute over
// the same workload) with the GPU executor, under three device-time models
// for a batch (ExecCost, include/credo/engine.hpp:38-45): the reference's
// default, the measured wall time of CudaExecutor::run on the harness's
// LinearToyModel, and (argv[1], argv[2] = fixed_us, per_item_us) the
// measured device time of one ResNet-50 replica's forward on the B200.
#include <chrono>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <optional>
#include <random>
#include <string>

#include "credo/harness.hpp"
#include "credo/model.hpp"
#include "credo_gpu_adapters.hpp"

namespace {
bool g_gpu = false;
uint64_t g_gpu_runs = 0, g_gpu_inputs = 0;
std::unique_ptr<credo::gpu::Context> g_ctx;
std::unique_ptr<credo::gpu::CudaExecutor> g_exec;
}  // namespace

namespace credo {
std::vector<std::vector<double>> ToyExecutor::run(const LinearToyModel& model,
                                                  const std::vector<std::vector<double>>& inputs) {
  if (g_gpu) {
    g_gpu_runs++;
    g_gpu_inputs += inputs.size();
    return g_exec->run(model, inputs);
  }
  std::vector<std::vector<double>> out;  // model.cpp:67-73
  out.reserve(inputs.size());
  for (const auto& x : inputs) out.push_back(model.run(x));
  return out;
}
}  // namespace credo

using namespace credo;
using namespace credo::harness;

// ExecCost of CudaExecutor::run on the harness's default model shape
// (WorkloadSpec defaults): wall time per call, H2D + kernel + D2H + sync,
// fitted as fixed + per_item * n over batches of 1 and 4 requests.
static ExecCost measure_linear_cost() {
  WorkloadSpec w;
  auto gen = generate_group("bench", w, 0);
  const LinearToyModel model = LinearToyModel::from_file_bytes(
      ByteView(gen.model_files.begin()->second.data(), gen.model_files.begin()->second.size()));
  std::mt19937_64 rng(3);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  auto batch = [&](size_t n) {
    std::vector<std::vector<double>> xs(n, std::vector<double>(model.input_dim));
    for (auto& x : xs)
      for (double& v : x) v = uni(rng);
    return xs;
  };
  auto time_us = [&](size_t n) {
    auto xs = batch(n);
    for (int i = 0; i < 20; i++) g_exec->run(model, xs);  // warm: residency, plans
    const int reps = 200;
    auto t0 = std::chrono::steady_clock::now();
    for (int i = 0; i < reps; i++) g_exec->run(model, xs);
    return std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0)
               .count() / reps;
  };
  const double t1 = time_us(1), t4 = time_us(4);
  ExecCost c;
  c.per_item_us = (uint64_t)std::llround(std::max(0.0, (t4 - t1) / 3.0));
  c.fixed_us = (uint64_t)std::llround(std::max(1.0, t1 - (double)c.per_item_us));
  return c;
}

int main(int argc, char** argv) {
  g_ctx = std::make_unique<gpu::Context>(0);
  g_exec = std::make_unique<gpu::CudaExecutor>(*g_ctx);
  auto small_spec = [] {  // tests/test_harness.cpp:19-28
    ScenarioSpec spec;
    spec.workload.n_requests = 8;
    spec.workload.input_dim = 4;
    spec.workload.output_dim = 3;
    spec.workload.models_per_group = 4;
    spec.workload.arrival_gap_us = 3'000;
    spec.duration_us = 120'000'000;
    return spec;
  };
  struct Case {
    const char* name;
    ScenarioSpec spec;
  };
  std::vector<Case> cases;
  cases.push_back({"honest", small_spec()});
  {
    ScenarioSpec s = small_spec();
    s.strategy = Coordinator::Strategy::agree_then_execute;
    cases.push_back({"agree_then_execute", s});
  }
  {
    ScenarioSpec s = small_spec();
    s.faults[2].behavior = FaultSpec::Behavior::corrupt_result;
    s.faults[2].magnitude = 1.0;  // beyond epsilon 0.05
    cases.push_back({"corrupt_beyond_eps", s});
  }
  {
    ScenarioSpec s = small_spec();
    s.faults[2].behavior = FaultSpec::Behavior::corrupt_result;
    s.faults[2].magnitude = 1e-4;  // within epsilon
    cases.push_back({"corrupt_within_eps", s});
  }
  {
    ScenarioSpec s = small_spec();  // C1-sized models: 3072 -> 10
    s.workload.input_dim = 3072;
    s.workload.output_dim = 10;
    s.workload.n_requests = 12;
    cases.push_back({"c1_shape", s});
  }
  int failures = 0;
  for (auto& c : cases) {
    g_gpu = false;
    ScenarioResult cpu = run_scenario(c.spec);
    g_gpu = true;
    const uint64_t runs0 = g_gpu_runs;
    ScenarioResult gpu = run_scenario(c.spec);
    g_gpu = false;
    auto violations = check_invariants(gpu);
    const bool ok = !gpu.deadlocked && gpu.certified() == c.spec.workload.n_requests &&
                    violations.empty() && gpu.trace == cpu.trace && g_gpu_runs > runs0;
    std::printf("%-20s gpu executor runs %4lu  certified %lu/%lu  violations %zu  "
                "trace %s (%zu bytes)  %s\n",
                c.name, (unsigned long)(g_gpu_runs - runs0), (unsigned long)gpu.certified(),
                (unsigned long)c.spec.workload.n_requests, violations.size(),
                gpu.trace == cpu.trace ? "identical" : "DIFFERS", gpu.trace.size(),
                ok ? "ok" : "FAIL");
    for (auto& v : violations) std::printf("  violation: %s\n", v.c_str());
    if (!ok) failures++;
  }
  // the reference's strategy benchmark with real device-time models
  {
    struct Model {
      const char* name;
      std::optional<ExecCost> cost;
    };
    std::vector<Model> models{{"reference default ExecCost", std::nullopt},
                              {"B200 LinearToyModel (measured)", measure_linear_cost()}};
    if (argc > 2) {
      ExecCost rn;
      rn.fixed_us = std::strtoull(argv[1], nullptr, 10);
      rn.per_item_us = std::strtoull(argv[2], nullptr, 10);
      models.push_back({"B200 ResNet-50 replica (measured)", rn});
    }
    g_gpu = true;
    for (uint64_t gap : {1000ull, 100ull})  // BenchSpec default arrival gap, and 10x the rate
      for (const auto& m : models) {
        BenchSpec bs;
        bs.exec_cost = m.cost;
        bs.arrival_gap_us = gap;
        const ExecCost c = m.cost.value_or(ExecCost{});
        BenchReport rep = bench_strategies(bs);
        std::printf("strategies [%s: %lu + %lu*n us, arrival gap %lu us]: execute-agree-attest "
                    "%.1f req/s, agree-execute %.1f req/s (%lu requests, all certified %d)\n",
                    m.name, (unsigned long)c.fixed_us, (unsigned long)c.per_item_us,
                    (unsigned long)gap, rep.execute_agree_attest_tps, rep.agree_execute_tps,
                    (unsigned long)rep.n_requests, (int)rep.all_certified);
        if (!rep.all_certified) failures++;
      }
    g_gpu = false;
  }
  std::printf("integration_scenario: %zu scenarios, %lu GPU executor calls (%lu inputs), "
              "%d failures\n",
              cases.size(), (unsigned long)g_gpu_runs, (unsigned long)g_gpu_inputs, failures);
  g_exec.reset();
  g_ctx.reset();
  return failures == 0 ? 0 : 1;
}
