// TEST INFRASTRUCTURE — drop-in demonstration. Runs the reference's own
// InferenceEngine (src/engine.cpp, unmodified, linked from oracle/_ref) with
// the GPU executor from include/credo_gpu_adapters.hpp next to the stock
// ToyExecutor on the same generated group and signed requests, and checks:
//   * execute_batch results bit-identical (LinearToyModel fp64 path),
//   * distance::select_quorum == gpu_select_quorum on every request,
//   * crypto::hash == gpu_hash_many on the result leaves.
// Built by `make -C oracle integration`; run by tests/test_gpu_integration.py.
#include <cstdio>
#include <map>
#include <memory>
#include <random>

#include "credo/domain.hpp"
#include "credo/engine.hpp"
#include "credo/harness.hpp"
#include "credo/merkle.hpp"
#include "credo/messages.hpp"
#include "credo_gpu_adapters.hpp"

using namespace credo;

int main() {
  harness::WorkloadSpec w;
  w.input_dim = 3072;
  w.output_dim = 10;
  w.models_per_group = 4;
  w.epsilon = 0.05;
  auto gen = harness::generate_group("group-0", w, 0);
  std::map<std::string, Bytes> files(gen.model_files.begin(), gen.model_files.end());
  ModelFetcher fetch = [&](const std::string& url) -> std::optional<Bytes> {
    auto it = files.find(url);
    if (it == files.end()) return std::nullopt;
    return it->second;
  };
  ModelGroup group;
  group.group_id = "group-0";
  group.version = 1;
  group.models = gen.definition.models;
  group.distance = gen.definition.distance;
  group.status = GroupStatus::active;

  gpu::Context ctx(0);
  const uint64_t N = 4, B = 16;
  KeyPair client = KeyPair::from_seed(std::array<uint8_t, 32>{7});
  std::mt19937_64 rng(11);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::vector<InferenceRequest> reqs;
  for (uint64_t i = 0; i < B; i++) {
    std::vector<double> x(w.input_dim);
    for (double& v : x) v = uni(rng);
    Encoder ne;
    ne.u64(i);
    reqs.push_back(make_signed_request(client, ne.take(), "group-0", x, std::nullopt));
  }
  int mismatches = 0, checked = 0;
  std::map<uint64_t, std::map<uint64_t, std::vector<double>>> outs;  // req -> node -> out
  for (uint64_t node = 0; node < N; node++) {
    NodeIdentity self;
    self.index = node;
    InferenceEngine gpu_engine(self, N, B, 2000, std::make_unique<gpu::CudaExecutor>(ctx), fetch);
    InferenceEngine cpu_engine(self, N, B, 2000, std::make_unique<ToyExecutor>(), fetch);
    if (gpu_engine.load_group(group) || cpu_engine.load_group(group)) {
      std::fprintf(stderr, "load_group failed\n");
      return 2;
    }
    std::vector<ExecutionBatch> gb, cb;
    for (auto& r : reqs) {
      auto a = gpu_engine.submit(r, 0);
      auto b = cpu_engine.submit(r, 0);
      gb.insert(gb.end(), a.ready.begin(), a.ready.end());
      cb.insert(cb.end(), b.ready.begin(), b.ready.end());
    }
    if (gb.size() != 1 || cb.size() != 1) {
      std::fprintf(stderr, "expected one full batch\n");
      return 2;
    }
    auto g = gpu_engine.execute_batch(gb[0]);
    auto c = cpu_engine.execute_batch(cb[0]);
    for (size_t k = 0; k < g.size(); k++) {
      checked++;
      if (!(g[k] == c[k])) mismatches++;
      outs[k][node] = g[k].output;
    }
    // result leaves hashed on the GPU == crypto::hash on the CPU
    std::vector<Bytes> leaves;
    for (size_t k = 0; k < g.size(); k++) {
      Bytes leaf = result_leaf(reqs[k], g[k]);
      leaf.insert(leaf.begin(), 0x00);  // merkle leaf domain
      leaves.push_back(leaf);
    }
    auto hs = gpu::gpu_hash_many(ctx, leaves);
    for (size_t k = 0; k < g.size(); k++) {
      checked++;
      if (!(hs[k] == merkle::leaf_hash(result_leaf(reqs[k], g[k])))) mismatches++;
    }
  }
  // PerturbingExecutor(ToyExecutor, node, magnitude) (the harness wiring,
  // harness.cpp:255-258) == CudaExecutor(ctx, node, magnitude), and a model
  // is serialised + hashed once, not on every run
  {
    std::vector<std::vector<double>> xs;
    for (auto& r : reqs) xs.push_back(r.input);
    for (const auto& [url, bytes] : files) {
      LinearToyModel model = LinearToyModel::from_file_bytes(ByteView(bytes.data(), bytes.size()));
      for (uint64_t node : {0ull, 3ull}) {
        PerturbingExecutor cpu(std::make_unique<ToyExecutor>(), node, 1e-9);
        gpu::CudaExecutor g(ctx, node, 1e-9);
        auto want = cpu.run(model, xs);
        for (int rep = 0; rep < 3; rep++) {
          checked++;
          if (g.run(model, xs) != want) mismatches++;
        }
        checked++;
        if (g.files_hashed() != 1) mismatches++;
      }
    }
  }
  for (auto& [k, m] : outs) {
    auto want = distance::select_quorum(m, N, 1, distance::Metric::euclidean, 0.05);
    auto got = gpu::gpu_select_quorum(ctx, m, N, 1, distance::Metric::euclidean, 0.05);
    checked++;
    if (want.selected != got.selected || want.diameter != got.diameter ||
        want.satisfied != got.satisfied)
      mismatches++;
  }
  std::printf("integration: %d checks, %d mismatches\n", checked, mismatches);
  return mismatches == 0 ? 0 : 1;
}
