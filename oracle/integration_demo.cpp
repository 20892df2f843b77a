// TEST INFRASTRUCTURE — drop-in demonstration. Runs the reference's own
// InferenceEngine (src/engine.cpp, unmodified, linked from oracle/_ref) with
// the GPU executor from include/credo_gpu_adapters.hpp next to the stock
// ToyExecutor on the same generated group and signed requests, and checks:
//   * execute_batch results bit-identical (LinearToyModel fp64 path),
//   * distance::select_quorum == gpu_select_quorum on every request,
//   * crypto::hash == gpu_hash_many on the result leaves,
//   * adjacency_batches + GroupServer::execute_batches filling per-node
//     PendingResultStores == the reference engines' execute_batch results.
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
  // agree_then_execute's execution path: an ordered slot's ok request ops
  // (two live versions interleaved, one misfit input) chunked by
  // adjacency_batches (coordinator.cpp:26-43), dispatched through
  // GroupServer::execute_batches, every provider's results in its own
  // PendingResultStore == each node's InferenceEngine::execute_batch results
  // (engine.cpp:269-306, stored in results()), bit for bit
  {
    ModelGroup g2 = group;
    g2.version = 2;
    gpu::GroupServer srv(ctx, B, 2000);
    if (srv.load_group(group, fetch, 1) || srv.load_group(g2, fetch, 1)) {
      std::fprintf(stderr, "GroupServer load_group failed\n");
      return 2;
    }
    std::vector<InferenceRequest> slot_reqs(reqs.begin(), reqs.begin() + 11);
    slot_reqs[6].input.resize(5);  // does not fit: skipped by execute_batch
    std::vector<const InferenceRequest*> ptrs;
    std::vector<uint64_t> versions;
    const uint64_t pattern[11] = {1, 1, 1, 1, 1, 2, 2, 1, 2, 2, 2};
    for (size_t i = 0; i < slot_reqs.size(); i++) {
      ptrs.push_back(&slot_reqs[i]);
      versions.push_back(pattern[i]);
    }
    auto batches = gpu::adjacency_batches(ptrs, versions, 4);
    checked++;
    if (batches.size() != 5) mismatches++;  // [1x4] [1] [2x2] [1] [2x3]
    std::vector<PendingResultStore> stores(N);
    std::map<uint64_t, PendingResultStore*> sp;
    for (uint64_t p = 0; p < N; p++) sp[p] = &stores[p];
    srv.execute_batches(batches, sp);
    for (uint64_t node = 0; node < N; node++) {
      NodeIdentity self;
      self.index = node;
      InferenceEngine cpu_engine(self, N, B, 2000, std::make_unique<ToyExecutor>(), fetch);
      if (cpu_engine.load_group(group) || cpu_engine.load_group(g2)) return 2;
      for (const auto& b : batches) cpu_engine.execute_batch(b);
      for (size_t i = 0; i < slot_reqs.size(); i++)
        for (uint64_t ver : {1ull, 2ull}) {
          checked++;
          auto want = cpu_engine.results().get(slot_reqs[i].request_id, ver);
          auto got = stores[node].get(slot_reqs[i].request_id, ver);
          if (want != got) mismatches++;
        }
      checked++;
      if (stores[node].request_count() != cpu_engine.results().request_count()) mismatches++;
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
