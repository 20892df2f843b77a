// Reference-side bindings a credo maintainer adds to use the B200 path as a
// drop-in (header-only; compiles against the reference's own headers,
// proj/include/credo/*.hpp, and links libcredo_gpu.so). See INTEGRATION.md.
//
//   CudaExecutor      : credo::ModelExecutor   (include/credo/model.hpp:41-51),
//                       optionally PerturbingExecutor-wrapped (model.hpp:60-79)
//   GroupServer       : InferenceEngine::load_group / submit / flush_* /
//                       execute_batch + try_attest's digests for any model
//                       family (src/engine.cpp:67-306, coordinator.cpp:727-865)
//                       execute_batches: dispatch_batches for adjacency_batches
//                       of an ordered slot, results into PendingResultStore
//                       (coordinator.cpp:26-43,1030-1048; engine.cpp:11-34)
//   gpu_select_quorum : distance::select_quorum (include/credo/distance.hpp:65-67)
//   gpu_hash_many     : crypto::hash, batched   (include/credo/crypto.hpp:26-30)
#pragma once

#include <cstring>
#include <map>
#include <optional>
#include <stdexcept>
#include <string>
#include <tuple>
#include <vector>

#include "credo/distance.hpp"
#include "credo/domain.hpp"
#include "credo/engine.hpp"
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

inline Hash32 host_hash(const Bytes& b) {
  Hash32 h;
  if (cg_host_sha256(b.data(), b.size(), h.data.data()) != CG_OK)
    throw std::runtime_error("cg_host_sha256 failed");
  return h;
}

// ModelExecutor::run on the GPU; with (node_index, magnitude) it is
// PerturbingExecutor(inner, node_index, magnitude) with the SHA-256 lane
// offsets computed on the device (model.cpp:75-105). A model becomes
// resident on first use: its canonical file is serialised and hashed once
// (the weights digest, the key load_group checks, engine.cpp:79); later runs
// find it by identity (address, buffers, shape, a strided content
// fingerprint) without re-serialising or re-hashing the file.
class CudaExecutor final : public ModelExecutor {
 public:
  explicit CudaExecutor(Context& ctx) : ctx_(ctx) {}
  CudaExecutor(Context& ctx, uint64_t node_index, double magnitude)
      : ctx_(ctx), node_index_(node_index), magnitude_(magnitude) {
    if (!(magnitude >= 0.0)) throw std::invalid_argument("negative magnitude");
  }
  ~CudaExecutor() override {
    for (auto& kv : by_digest_) cg_model_free(kv.second);
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
    check(ctx_.get(), magnitude_ == 0.0
                          ? cg_exec_run(ctx_.get(), m, in.data(), B, u, out.data(), v)
                          : cg_exec_run_perturbed(ctx_.get(), m, in.data(), B, u, out.data(), v,
                                                  node_index_, magnitude_));
    std::vector<std::vector<double>> y(B);
    for (uint64_t i = 0; i < B; i++) y[i].assign(out.begin() + i * v, out.begin() + (i + 1) * v);
    return y;
  }

  uint64_t files_hashed() const { return files_hashed_; }

 private:
  using Key = std::tuple<const void*, const double*, const double*, uint64_t, uint64_t, bool,
                         uint64_t>;
  static uint64_t fingerprint(const LinearToyModel& m) {
    uint64_t h = 1469598103934665603ull;  // FNV-1a over <= 64 strided weights + bias
    auto mix = [&](double d) {
      uint64_t b;
      std::memcpy(&b, &d, 8);
      for (int i = 0; i < 8; i++) h = (h ^ ((b >> (8 * i)) & 0xff)) * 1099511628211ull;
    };
    const size_t n = m.weights.size(), step = n > 64 ? n / 64 : 1;
    for (size_t i = 0; i < n; i += step) mix(m.weights[i]);
    for (double d : m.bias) mix(d);
    return h;
  }
  cg_model* resident(const LinearToyModel& model) {
    const Key key{&model, model.weights.data(), model.bias.data(), model.input_dim,
                  model.output_dim, model.softmax, fingerprint(model)};
    auto it = by_key_.find(key);
    if (it != by_key_.end()) return it->second;
    Bytes file = model.to_file_bytes();
    const Hash32 d = host_hash(file);
    files_hashed_++;
    auto dit = by_digest_.find(d);
    cg_model* m = nullptr;
    if (dit != by_digest_.end()) {
      m = dit->second;
    } else {
      check(ctx_.get(), cg_model_load_linear(ctx_.get(), file.data(), file.size(), d.data.data(), &m));
      by_digest_[d] = m;
    }
    by_key_[key] = m;
    return m;
  }

  Context& ctx_;
  uint64_t node_index_ = 0;
  double magnitude_ = 0.0;
  uint64_t files_hashed_ = 0;
  std::map<Key, cg_model*> by_key_;
  std::map<Hash32, cg_model*> by_digest_;
};

// InferenceEngine's batch path for model groups of any family on one GPU:
// load_group fetches every descriptor's file through the reference's
// ModelFetcher and makes it resident as an opaque cg_model keyed by its
// weights_digest (params["arch"] names a CNN -- cg_model_load_cnn -- else the
// file is a LinearToyModel), with the digest checked as engine.cpp:79 does.
// submit/flush_* are the reference's batch-former semantics (cg_engine:
// seen-dedup, per-version FIFO, exec_batch_max, flush deadline, one batch per
// live version); dispatch certifies every released batch: the replica
// forwards, select_quorum + label vote, result leaves and R roots, the
// attestation manifest and A root (try_prepare / try_attest's digests).
class GroupServer {
 public:
  struct Certified {
    std::string group_id;
    uint64_t version = 0;
    std::vector<uint32_t> selected;  // B requests, in submission (FIFO) order
    std::vector<double> diameter;
    std::vector<uint8_t> satisfied;
    std::vector<int64_t> label;
    std::vector<Hash32> r_roots;  // per provider
    Hash32 a_root{};
    uint64_t manifest_len = 0;
    std::vector<double> outputs;  // N x B x v (provider-major), when keep_outputs
  };

  GroupServer(Context& ctx, uint64_t exec_batch_max, uint64_t flush_interval_us,
              int pack_threads = 4)
      : ctx_(ctx), max_(exec_batch_max) {
    check(ctx_.get(), cg_engine_create(ctx_.get(), exec_batch_max, flush_interval_us, pack_threads,
                                       &eng_));
  }
  ~GroupServer() {
    cg_engine_free(eng_);
    for (auto& [key, g] : groups_) cg_group_free(g.h);
    for (auto& kv : models_) cg_model_free(kv.second);
  }
  GroupServer(const GroupServer&) = delete;
  GroupServer& operator=(const GroupServer&) = delete;

  // load_group (engine.cpp:67-97): every model of the group is served on
  // this GPU (replicas time-sliced; node p answers as provider p).
  std::optional<std::string> load_group(const ModelGroup& group, const ModelFetcher& fetch,
                                        uint64_t f, uint32_t topk = 5) {
    if (auto err = group.validate()) return err;
    if (groups_.count({group.group_id, group.version})) return "version already loaded";
    std::vector<cg_model*> ms;
    for (const auto& desc : group.models) {
      auto it = models_.find(desc.weights_digest);
      if (it == models_.end()) {
        auto file = fetch(desc.model_url);
        if (!file) return "model file unavailable: " + desc.model_url;
        cg_model* m = nullptr;
        const bool cnn = desc.params.count("arch") > 0;
        int rc = cnn ? cg_model_load_cnn(ctx_.get(), file->data(), file->size(),
                                         desc.weights_digest.data.data(), &m)
                     : cg_model_load_linear(ctx_.get(), file->data(), file->size(),
                                            desc.weights_digest.data.data(), &m);
        if (rc == CG_EDIGEST) return "weights digest mismatch: " + desc.model_url;
        if (rc != CG_OK) return std::string("bad model file: ") + cg_last_error(ctx_.get());
        uint64_t u = 0, v = 0;
        cg_model_dims(m, &u, &v);
        if (u != desc.input_dim || v != desc.output_dim) {
          cg_model_free(m);
          return "model file dimensions disagree with descriptor";
        }
        it = models_.emplace(desc.weights_digest, m).first;
      }
      ms.push_back(it->second);
    }
    cg_group* g = nullptr;
    check(ctx_.get(), cg_group_create(ctx_.get(), ms.data(), (uint32_t)ms.size(), (uint32_t)f,
                                      (uint32_t)group.distance.metric,
                                      group.distance.default_epsilon, group.group_id.data(),
                                      group.group_id.size(), group.version, (uint32_t)max_, topk,
                                      &g));
    const int st = group.status == GroupStatus::retired  ? CG_GROUP_RETIRED
                   : group.status == GroupStatus::active ? CG_GROUP_ACTIVE
                                                         : CG_GROUP_DEFINED;
    check(ctx_.get(), cg_engine_load_group(eng_, g, st));
    Group G{g, (uint32_t)ms.size(), group.models.front().output_dim,
            group.models.front().input_dim, {}};
    for (const auto& desc : group.models) G.digests.push_back(desc.weights_digest);
    groups_[{group.group_id, group.version}] = std::move(G);
    return std::nullopt;
  }

  void set_status(const std::string& gid, uint64_t version, GroupStatus s) {
    check(ctx_.get(), cg_engine_set_status(eng_, gid.data(), gid.size(), version,
                                           s == GroupStatus::retired  ? CG_GROUP_RETIRED
                                           : s == GroupStatus::active ? CG_GROUP_ACTIVE
                                                                      : CG_GROUP_DEFINED));
  }

  // submit (engine.cpp:182-209): nullopt or the SubmitOutcome error string.
  // Run verify_request's Ed25519 check first (or set a verifier on the
  // engine); the structural checks run here.
  std::optional<std::string> submit(const InferenceRequest& r, uint64_t now_us) {
    return submit_many(&r, 1, now_us)[0];
  }
  std::vector<std::optional<std::string>> submit_many(const InferenceRequest* rs, size_t n,
                                                      uint64_t now_us) {
    std::vector<cg_request> cr(n);
    for (size_t i = 0; i < n; i++) {
      const InferenceRequest& r = rs[i];
      cr[i] = cg_request{r.request_id.data.data(), r.group_id.data(), r.group_id.size(),
                         r.input.data(), r.input.size(), r.epsilon_override.has_value() ? 1 : 0,
                         r.epsilon_override.value_or(0.0), r.client_pub.data(),
                         r.client_nonce.data(), r.client_nonce.size(), r.client_sig.data()};
    }
    std::vector<int> err(n);
    check(ctx_.get(), cg_engine_submit(eng_, cr.data(), (uint32_t)n, now_us, err.data()));
    std::vector<std::optional<std::string>> out(n);
    for (size_t i = 0; i < n; i++) {
      if (err[i] == CG_SUBMIT_INVALID) out[i] = "invalid request signature";
      else if (err[i] == CG_SUBMIT_UNKNOWN_GROUP) out[i] = "unknown group";
      else if (err[i] == CG_SUBMIT_RETIRED) out[i] = "group retired";
    }
    return out;
  }

  void flush_due(uint64_t now_us) { check(ctx_.get(), cg_engine_flush_due(eng_, now_us)); }
  void flush_version(const std::string& gid, uint64_t version) {
    check(ctx_.get(), cg_engine_flush_version(eng_, gid.data(), gid.size(), version));
  }
  void flush_all() { check(ctx_.get(), cg_engine_flush_all(eng_)); }
  std::optional<uint64_t> next_flush_deadline() {
    uint64_t d = 0;
    int has = 0;
    check(ctx_.get(), cg_engine_next_flush_deadline(eng_, &d, &has));
    return has ? std::optional<uint64_t>(d) : std::nullopt;
  }

  // Coordinator::dispatch_batches (coordinator.cpp:1030-1048) for batches
  // formed outside the batch former -- adjacency_batches of an ordered slot
  // under agree_then_execute (coordinator.cpp:26-43, :588-624): each batch is
  // ingested and certified as it is (a request whose input does not fit the
  // group is skipped by execute_batch, engine.cpp:286-291: missing results).
  // With stores[p], provider p's results go into that PendingResultStore as
  // InferenceEngine::execute_batch puts them (engine.cpp:293-303): node p,
  // the batch's version, the output, p's weights_digest.
  std::vector<Certified> execute_batches(const std::vector<ExecutionBatch>& batches,
                                         const std::map<uint64_t, PendingResultStore*>& stores = {},
                                         bool keep_outputs = false) {
    std::vector<Certified> out;
    for (const ExecutionBatch& b : batches) {
      if (b.requests.empty()) continue;
      auto git = groups_.find({b.group_id, b.group_version});
      if (git == groups_.end()) throw std::invalid_argument("execute_batches: version not loaded");
      const Group& G = git->second;
      const uint32_t B = (uint32_t)b.requests.size();
      const uint64_t u = G.u;
      std::vector<uint8_t> ids(32 * (size_t)B), has_eps(B), pubs(32 * (size_t)B),
          sigs(64 * (size_t)B), nonces;
      std::vector<double> eps(B), in((size_t)B * u, 0.0);
      std::vector<uint64_t> nonce_lens(B), dims(B);
      std::vector<const double*> mis(B, nullptr);
      bool any_mis = false;
      for (uint32_t k = 0; k < B; k++) {
        const InferenceRequest& r = b.requests[k];
        std::memcpy(&ids[32 * (size_t)k], r.request_id.data.data(), 32);
        dims[k] = r.input.size();
        if (dims[k] == u) std::copy(r.input.begin(), r.input.end(), in.begin() + (size_t)k * u);
        else mis[k] = r.input.data(), any_mis = true;
        has_eps[k] = r.epsilon_override.has_value();
        eps[k] = r.epsilon_override.value_or(0.0);
        std::memcpy(&pubs[32 * (size_t)k], r.client_pub.data(), 32);
        nonces.insert(nonces.end(), r.client_nonce.begin(), r.client_nonce.end());
        nonce_lens[k] = r.client_nonce.size();
        std::memcpy(&sigs[64 * (size_t)k], r.client_sig.data(), 64);
      }
      cg_request_batch bt{};
      bt.B = B;
      bt.u = u;
      bt.request_ids = ids.data();
      bt.inputs = in.data();
      bt.has_eps = has_eps.data();
      bt.eps = eps.data();
      bt.client_pubs = pubs.data();
      bt.nonces = nonces.data();
      bt.nonce_lens = nonce_lens.data();
      bt.client_sigs = sigs.data();
      if (any_mis) {
        bt.input_dims = dims.data();
        bt.misfit_inputs = mis.data();
      }
      uint64_t ticket = 0;
      check(ctx_.get(), cg_ingest_batch(G.h, &bt, &ticket));
      auto [c, Gp] = certify_group(cg_ready_batch{G.h, b.group_version, ticket, B},
                                   keep_outputs || !stores.empty());
      for (const auto& [p, store] : stores) {
        if (p >= G.N || !store) continue;
        for (uint32_t k = 0; k < B; k++) {
          if (dims[k] != u) continue;
          InferenceResult r;
          r.request_id = b.requests[k].request_id;
          r.node_index = p;
          r.group_id = b.group_id;
          r.group_version = b.group_version;
          const double* o = c.outputs.data() + ((size_t)p * B + k) * G.v;
          r.output.assign(o, o + G.v);
          r.model_digest = G.digests[p];
          store->put(r);
        }
      }
      if (!keep_outputs) c.outputs.clear();
      out.push_back(std::move(c));
    }
    return out;
  }

  // dispatch_batches + execute_batch + try_prepare/try_attest digests for
  // every released batch, in release order.
  std::vector<Certified> dispatch(bool keep_outputs = false) {
    std::vector<Certified> out;
    cg_ready_batch rb[64];
    for (;;) {
      uint32_t n = 0;
      check(ctx_.get(), cg_engine_ready(eng_, rb, 64, &n));
      for (uint32_t i = 0; i < n; i++) out.push_back(certify(rb[i], keep_outputs));
      if (n < 64) break;
    }
    return out;
  }

 private:
  struct Group {
    cg_group* h;
    uint32_t N;
    uint64_t v, u;
    std::vector<Hash32> digests;  // provider p's weights_digest
  };
  Certified certify(const cg_ready_batch& rb, bool keep_outputs) {
    return certify_group(rb, keep_outputs).first;
  }
  std::pair<Certified, const Group*> certify_group(const cg_ready_batch& rb, bool keep_outputs) {
    const Group* G = nullptr;
    Certified c;
    for (auto& [key, g] : groups_)
      if (g.h == rb.group) {
        G = &g;
        c.group_id = key.first;
      }
    if (!G) throw std::runtime_error("ready batch of an unknown group");
    c.version = rb.version;
    const uint32_t B = rb.B, N = G->N;
    c.selected.resize(B);
    c.diameter.resize(B);
    c.satisfied.resize(B);
    c.label.resize(B);
    c.r_roots.resize(N);
    std::vector<uint8_t> rr(32 * N);
    if (keep_outputs) c.outputs.resize((size_t)N * B * G->v);
    cg_certify_out o{};
    o.selected = c.selected.data();
    o.diameter = c.diameter.data();
    o.satisfied = c.satisfied.data();
    o.label = c.label.data();
    o.r_roots = rr.data();
    o.a_root = c.a_root.data.data();
    o.manifest_len = &c.manifest_len;
    if (keep_outputs) o.outputs = c.outputs.data();
    check(ctx_.get(), cg_certify_ticket(rb.group, rb.ticket, &o));
    for (uint32_t p = 0; p < N; p++) std::memcpy(c.r_roots[p].data.data(), &rr[32 * p], 32);
    return {std::move(c), G};
  }

  Context& ctx_;
  uint64_t max_;
  cg_engine* eng_ = nullptr;
  std::map<Hash32, cg_model*> models_;
  std::map<std::pair<std::string, uint64_t>, Group> groups_;
};

// adjacency_batches (coordinator.cpp:24-43, file-local there): consecutive
// ok request ops sharing a (group, version), chunked to batch_max, batch
// order kept -- how an ordered slot becomes execution batches under
// agree_then_execute.
inline std::vector<ExecutionBatch> adjacency_batches(
    const std::vector<const InferenceRequest*>& reqs, const std::vector<uint64_t>& versions,
    uint64_t batch_max) {
  std::vector<ExecutionBatch> out;
  for (size_t i = 0; i < reqs.size(); i++) {
    if (out.empty() || out.back().group_id != reqs[i]->group_id ||
        out.back().group_version != versions[i] || out.back().requests.size() >= batch_max) {
      out.emplace_back();
      out.back().group_id = reqs[i]->group_id;
      out.back().group_version = versions[i];
    }
    out.back().requests.push_back(*reqs[i]);
  }
  return out;
}

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
