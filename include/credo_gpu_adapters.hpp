// Reference-side bindings a credo maintainer adds to use the B200 path as a
// drop-in (header-only; compiles against the reference's own headers,
// proj/include/credo/*.hpp, and links libcredo_gpu.so). See INTEGRATION.md.
//
//   CudaExecutor      : credo::ModelExecutor   (include/credo/model.hpp:41-51)
//   gpu_select_quorum : distance::select_quorum (include/credo/distance.hpp:65-67)
//   gpu_hash_many     : crypto::hash, batched   (include/credo/crypto.hpp:26-30)
#pragma once

#include <map>
#include <stdexcept>
#include <string>
#include <vector>

#include "credo/distance.hpp"
#include "credo/model.hpp"
#include "credo_gpu.h"

namespace credo::gpu {

inline void check(cg_ctx* ctx, int rc) {
  if (rc == CG_OK) return;
  std::string msg = cg_last_error(ctx);
  if (rc == CG_EINVAL) throw std::invalid_argument(msg);  // same class as the reference
  throw std::runtime_error(msg);
}

class Context {
 public:
  explicit Context(int device = 0) {
    if (cg_ctx_create(device, &ctx_) != CG_OK)
      throw std::runtime_error("credo_gpu: no sm_100a device");
  }
  ~Context() { cg_ctx_destroy(ctx_); }
  Context(const Context&) = delete;
  Context& operator=(const Context&) = delete;
  cg_ctx* get() const { return ctx_; }

 private:
  cg_ctx* ctx_ = nullptr;
};

// ModelExecutor::run on the GPU. Models become resident on first use, keyed
// by their weights digest (the same key load_group checks, engine.cpp:79).
class CudaExecutor final : public ModelExecutor {
 public:
  explicit CudaExecutor(Context& ctx) : ctx_(ctx) {}
  ~CudaExecutor() override {
    for (auto& kv : resident_) cg_model_free(kv.second);
  }

  std::vector<std::vector<double>> run(
      const LinearToyModel& model,
      const std::vector<std::vector<double>>& inputs) override {
    if (inputs.empty()) return {};
    for (const auto& x : inputs)
      if (x.size() != model.input_dim)
        throw std::invalid_argument("model input dimension mismatch");
    cg_model* m = resident(model);
    const uint64_t u = model.input_dim, v = model.output_dim, B = inputs.size();
    std::vector<double> in(B * u), out(B * v);
    for (uint64_t i = 0; i < B; i++) std::copy(inputs[i].begin(), inputs[i].end(), in.begin() + i * u);
    check(ctx_.get(), cg_exec_run(ctx_.get(), m, in.data(), B, u, out.data(), v));
    std::vector<std::vector<double>> y(B);
    for (uint64_t i = 0; i < B; i++) y[i].assign(out.begin() + i * v, out.begin() + (i + 1) * v);
    return y;
  }

 private:
  cg_model* resident(const LinearToyModel& model) {
    Bytes file = model.to_file_bytes();
    Hash32 d = hash(file);
    auto it = resident_.find(d);
    if (it != resident_.end()) return it->second;
    cg_model* m = nullptr;
    check(ctx_.get(), cg_model_load_linear(ctx_.get(), file.data(), file.size(), d.data.data(), &m));
    resident_[d] = m;
    return m;
  }

  Context& ctx_;
  std::map<Hash32, cg_model*> resident_;
};

// distance::select_quorum with the reference's signature and exceptions.
inline distance::AgreementOutcome gpu_select_quorum(
    Context& ctx, const std::map<uint64_t, std::vector<double>>& results,
    uint64_t n_nodes, uint64_t f, distance::Metric metric, double epsilon) {
  if (n_nodes == 0 || n_nodes > 20 || f >= n_nodes)
    throw std::invalid_argument("select_quorum: bad n/f");
  if (results.empty()) throw std::invalid_argument("select_quorum: fewer than N-f results present");
  const size_t v = results.begin()->second.size();
  std::vector<double> outs(n_nodes * std::max<size_t>(v, 1), 0.0);
  uint32_t present = 0;
  for (const auto& [node, vec] : results) {
    if (node >= n_nodes) throw std::invalid_argument("select_quorum: node index out of range");
    if (vec.size() != v) throw std::invalid_argument("delta: result dimensionality mismatch");
    std::copy(vec.begin(), vec.end(), outs.begin() + node * v);
    present |= 1u << node;
  }
  uint32_t sel = 0;
  double diam = 0;
  uint8_t sat = 0;
  int8_t status = 0;
  check(ctx.get(), cg_select_quorum_batch(ctx.get(), outs.data(), &present, &epsilon, 1,
                                          (uint32_t)n_nodes, (uint32_t)f, (uint32_t)v,
                                          (uint32_t)metric, &sel, &diam, &sat, &status,
                                          nullptr));
  distance::AgreementOutcome o;
  o.satisfied = sat != 0;
  o.diameter = diam;
  for (uint64_t i = 0; i < n_nodes; i++)
    if (sel >> i & 1) o.selected.insert(i);
  return o;
}

// crypto::hash over many messages in one launch.
inline std::vector<Hash32> gpu_hash_many(Context& ctx, const std::vector<Bytes>& msgs) {
  std::vector<uint8_t> buf;
  std::vector<uint64_t> off, len;
  for (const auto& m : msgs) {
    off.push_back(buf.size());
    len.push_back(m.size());
    buf.insert(buf.end(), m.begin(), m.end());
  }
  std::vector<Hash32> out(msgs.size());
  std::vector<uint8_t> raw(32 * msgs.size());
  check(ctx.get(), cg_sha256_batch(ctx.get(), buf.data(), off.data(), len.data(), msgs.size(),
                                   raw.data()));
  for (size_t i = 0; i < msgs.size(); i++)
    std::copy(raw.begin() + 32 * i, raw.begin() + 32 * i + 32, out[i].data.begin());
  return out;
}

}  // namespace credo::gpu
