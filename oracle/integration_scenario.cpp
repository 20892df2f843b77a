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
#include <cstdio>
#include <memory>
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

int main() {
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
  std::printf("integration_scenario: %zu scenarios, %lu GPU executor calls (%lu inputs), "
              "%d failures\n",
              cases.size(), (unsigned long)g_gpu_runs, (unsigned long)g_gpu_inputs, failures);
  g_exec.reset();
  g_ctx.reset();
  return failures == 0 ? 0 : 1;
}
