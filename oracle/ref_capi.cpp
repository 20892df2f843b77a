// TEST INFRASTRUCTURE — oracle only. Never linked into the product.
//
// extern "C" shims over the UNMODIFIED reference library (compiled in place
// from /root/reference/proj/src by oracle/Makefile into oracle/_ref/). Used by
//   * tests/golden/make_golden.py to generate the committed golden fixtures,
//   * tests/ (CPU, when oracle/_ref exists) to pin the C restatement,
//   * bench.py --impl reference / cpu_baseline to time the reference's own
//     CPU path on the box's host cores.
// Every function calls reference symbols; the few the reference keeps in
// anonymous namespaces are restated here with a file:line citation.

#include <algorithm>
#include <atomic>
#include <cstring>
#include <map>
#include <memory>
#include <random>
#include <set>
#include <stdexcept>
#include <thread>
#include <vector>

#include "credo/crypto.hpp"
#include "credo/distance.hpp"
#include "credo/domain.hpp"
#include "credo/harness.hpp"
#include "credo/merkle.hpp"
#include "credo/messages.hpp"
#include "credo/model.hpp"

using namespace credo;

namespace {

// Restated: src/harness.cpp:188-196 (anonymous namespace there).
std::array<uint8_t, 32> derive_seed(uint64_t master, const char* role,
                                    uint64_t index) {
  Encoder e;
  e.u64(master);
  e.str(role);
  e.u64(index);
  Bytes b = e.take();
  return hash(ByteView(b.data(), b.size())).data;
}

// Restated: src/harness.cpp:428-431.
std::mt19937_64 seeded_rng(uint64_t a, uint64_t b, uint64_t c) {
  std::seed_seq q{a, b, c};
  return std::mt19937_64(q);
}

// Restated: src/experiments.cpp:99-101 (anonymous namespace there).
size_t argmax(const std::vector<double>& v) {
  return static_cast<size_t>(std::max_element(v.begin(), v.end()) - v.begin());
}

// Restated: src/experiments.cpp:106-125 (anonymous namespace there).
std::optional<size_t> ensemble_label(
    const std::map<uint64_t, std::vector<double>>& quorum_outputs, uint64_t f) {
  std::map<size_t, std::pair<uint64_t, double>> votes;
  for (const auto& [node, v] : quorum_outputs) {
    size_t label = argmax(v);
    auto& entry = votes[label];
    entry.first++;
    entry.second = std::max(entry.second, v[label]);
  }
  std::optional<size_t> best;
  double best_conf = -1.0;
  for (const auto& [label, entry] : votes) {
    if (entry.first <= f) continue;
    if (entry.second > best_conf) {
      best = label;
      best_conf = entry.second;
    }
  }
  return best;
}

Hash32 to_h32(const uint8_t* p) {
  Hash32 h;
  std::memcpy(h.data.data(), p, 32);
  return h;
}

}  // namespace

extern "C" {

int ref_sha256(const uint8_t* buf, uint64_t len, uint8_t* out) {
  Hash32 h = hash(ByteView(buf, len));
  std::memcpy(out, h.data.data(), 32);
  return 0;
}

// merkle::leaf_hash (src/merkle.cpp:22-25).
int ref_leaf_hash(const uint8_t* leaf, uint64_t len, uint8_t* out) {
  Hash32 h = merkle::leaf_hash(ByteView(leaf, len));
  std::memcpy(out, h.data.data(), 32);
  return 0;
}

// merkle::Tree::build (src/merkle.cpp:47-67) over n leaves given back to back.
int ref_merkle_root(const uint8_t* leaves, const uint64_t* lens, uint64_t n,
                    uint8_t* root_out) {
  try {
    std::vector<Bytes> ls;
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; i++) {
      ls.emplace_back(leaves + off, leaves + off + lens[i]);
      off += lens[i];
    }
    Hash32 r = merkle::Tree::build(ls).root();
    std::memcpy(root_out, r.data.data(), 32);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// merkle::Tree::build(leaves).auth_path(index) (merkle.cpp:69-84): writes
// up to 64 steps (sibling 32 B, side 0 left / 1 right); returns the step
// count or -1.
int ref_auth_path(const uint8_t* leaves, const uint64_t* lens, uint64_t n, uint64_t index,
                  uint8_t* siblings, uint8_t* sides) {
  try {
    std::vector<Bytes> ls;
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; i++) {
      ls.emplace_back(leaves + off, leaves + off + lens[i]);
      off += lens[i];
    }
    merkle::AuthPath p = merkle::Tree::build(ls).auth_path(index);
    if (p.siblings.size() > 64) return -1;
    for (size_t i = 0; i < p.siblings.size(); i++) {
      std::memcpy(siblings + 32 * i, p.siblings[i].sibling.data.data(), 32);
      sides[i] = p.siblings[i].side == merkle::Side::left ? 0 : 1;
    }
    return (int)p.siblings.size();
  } catch (const std::exception&) {
    return -1;
  }
}

// merkle::get_merkle_root(path, leaf) (merkle.cpp:86-93).
int ref_path_root(const uint8_t* leaf, uint64_t leaf_len, const uint8_t* siblings,
                  const uint8_t* sides, uint32_t steps, uint8_t* root_out) {
  try {
    merkle::AuthPath p;
    for (uint32_t i = 0; i < steps; i++) {
      merkle::PathStep st;
      std::memcpy(st.sibling.data.data(), siblings + 32 * i, 32);
      st.side = sides[i] ? merkle::Side::right : merkle::Side::left;
      p.siblings.push_back(st);
    }
    Hash32 r = merkle::get_merkle_root(p, ByteView(leaf, leaf_len));
    std::memcpy(root_out, r.data.data(), 32);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

uint64_t ref_model_file_len(uint64_t in, uint64_t out) {
  return 8 + 8 + 1 + 4 + 8 * in * out + 4 + 8 * out;
}

// harness::generate_group (src/harness.cpp:346-395). softmax=1 re-encodes
// each model file with softmax=true and recomputes the
// digest. files_out: models × ref_model_file_len bytes; digests_out: models×32.
int ref_generate_group(const char* gid, uint64_t in, uint64_t out,
                       uint64_t models, uint32_t metric, double eps,
                       uint64_t seed, uint64_t salt, int softmax,
                       uint8_t* files_out, uint8_t* digests_out) {
  try {
    harness::WorkloadSpec w;
    w.input_dim = in;
    w.output_dim = out;
    w.models_per_group = models;
    w.metric = static_cast<distance::Metric>(metric);
    w.epsilon = eps;
    w.seed = seed;
    auto g = harness::generate_group(gid, w, salt);
    const uint64_t flen = ref_model_file_len(in, out);
    for (uint64_t m = 0; m < models; m++) {
      Bytes file = g.model_files[m].second;
      Hash32 d = g.definition.models[m].weights_digest;
      if (softmax) {
        auto mdl = LinearToyModel::from_file_bytes(file);
        mdl.softmax = true;
        file = mdl.to_file_bytes();
        d = mdl.digest();
      }
      if (file.size() != flen) return -2;
      std::memcpy(files_out + m * flen, file.data(), flen);
      std::memcpy(digests_out + 32 * m, d.data.data(), 32);
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

uint64_t ref_request_len(uint64_t gid_len, uint64_t in, uint64_t nonce_len,
                         int has_eps) {
  return 32 + 4 + gid_len + 4 + 8 * in + 1 + (has_eps ? 8 : 0) + 32 + 4 +
         nonce_len + 64;
}

// The run_scenario driver's request stream (src/harness.cpp:449-458,
// 564-575): client key derive_seed(seed,"client-key",0), rng seeded
// (seed, workload_seed, 0x647276), input U(-1,1), nonce u64 ctr || u64 rng.
// inputs_out: n×in doubles; enc_out: n × ref_request_len(...) bytes.
int ref_make_requests(uint64_t scenario_seed, uint64_t workload_seed,
                      uint64_t n, uint64_t in, const char* gid,
                      double* inputs_out, uint8_t* enc_out) {
  try {
    KeyPair client =
        KeyPair::from_seed(derive_seed(scenario_seed, "client-key", 0));
    auto rng = seeded_rng(scenario_seed, workload_seed, 0x647276);
    std::uniform_real_distribution<double> uni(-1.0, 1.0);
    const uint64_t rlen = ref_request_len(std::strlen(gid), in, 16, 0);
    for (uint64_t i = 0; i < n; i++) {
      std::vector<double> input(in);
      for (double& v : input) v = uni(rng);
      Encoder ne;
      ne.u64(i);
      ne.u64(rng());
      auto req = make_signed_request(client, ne.take(), gid, input,
                                     std::nullopt);
      Encoder e;
      req.encode(e);
      if (e.data().size() != rlen) return -2;
      std::memcpy(enc_out + i * rlen, e.data().data(), rlen);
      std::memcpy(inputs_out + i * in, input.data(), 8 * in);
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// make_signed_request (src/domain.cpp:184-202) for a caller-supplied input,
// seeded client key and nonce; with an optional epsilon override.
int ref_make_request(uint64_t key_seed, const uint8_t* nonce,
                     uint64_t nonce_len, const char* gid, const double* input,
                     uint64_t in, int has_eps, double eps, uint8_t* enc_out,
                     uint64_t cap, uint64_t* len_out) {
  try {
    KeyPair client = KeyPair::from_seed(derive_seed(key_seed, "client-key", 0));
    std::optional<double> e_o;
    if (has_eps) e_o = eps;
    auto req = make_signed_request(client, Bytes(nonce, nonce + nonce_len),
                                   gid, std::vector<double>(input, input + in),
                                   e_o);
    Encoder e;
    req.encode(e);
    *len_out = e.data().size();
    if (e.data().size() > cap) return -2;
    std::memcpy(enc_out, e.data().data(), e.data().size());
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_verify_request(const uint8_t* enc, uint64_t len) {
  try {
    Decoder d(ByteView(enc, len));
    auto req = InferenceRequest::decode(d);
    return verify_request(req) ? 1 : 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_signing_digest(const uint8_t* enc, uint64_t len, uint8_t* out) {
  try {
    Decoder d(ByteView(enc, len));
    auto req = InferenceRequest::decode(d);
    Hash32 h = req.signing_digest();
    std::memcpy(out, h.data.data(), 32);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// LinearToyModel::from_file_bytes + run (src/model.cpp:12-36, 46-60).
int ref_linear_run(const uint8_t* file, uint64_t len, const double* in,
                   uint64_t n, double* out) {
  try {
    auto m = LinearToyModel::from_file_bytes(ByteView(file, len));
    for (uint64_t i = 0; i < n; i++) {
      std::vector<double> x(in + i * m.input_dim, in + (i + 1) * m.input_dim);
      auto y = m.run(x);
      std::memcpy(out + i * m.output_dim, y.data(), 8 * m.output_dim);
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// PerturbingExecutor(ToyExecutor) over n inputs (src/model.cpp:75-105).
int ref_perturbing_run(const uint8_t* file, uint64_t len, const double* in,
                       uint64_t n, uint64_t node, double magnitude, double* out) {
  try {
    auto m = LinearToyModel::from_file_bytes(ByteView(file, len));
    PerturbingExecutor ex(std::make_unique<ToyExecutor>(), node, magnitude);
    std::vector<std::vector<double>> xs;
    for (uint64_t i = 0; i < n; i++)
      xs.emplace_back(in + i * m.input_dim, in + (i + 1) * m.input_dim);
    auto ys = ex.run(m, xs);
    for (uint64_t i = 0; i < n; i++)
      std::memcpy(out + i * m.output_dim, ys[i].data(), 8 * m.output_dim);
    return 0;
  } catch (const std::invalid_argument&) {
    return -2;
  } catch (const std::exception&) {
    return -1;
  }
}

// distance::select_quorum (src/distance.cpp:138-216). outs: m×v, node ids in
// node_idx. selected_mask: bit k set when node k is selected.
int ref_select_quorum(const double* outs, const uint64_t* node_idx, uint64_t m,
                      uint64_t v, uint64_t n, uint64_t f, uint32_t metric,
                      double eps, uint64_t* selected_mask, double* diam,
                      int* satisfied) {
  try {
    std::map<uint64_t, std::vector<double>> r;
    for (uint64_t i = 0; i < m; i++)
      r[node_idx[i]] = std::vector<double>(outs + i * v, outs + (i + 1) * v);
    auto o = distance::select_quorum(r, n, f,
                                     static_cast<distance::Metric>(metric), eps);
    uint64_t mask = 0;
    for (auto k : o.selected) mask |= uint64_t{1} << k;
    *selected_mask = mask;
    *diam = o.diameter;
    *satisfied = o.satisfied ? 1 : 0;
    return 0;
  } catch (const std::invalid_argument&) {
    return -1;
  }
}

// Restated ensemble_label over the members in `mask`; -1 when no label.
int64_t ref_ensemble_label(const double* outs, uint64_t m, uint64_t v,
                           uint64_t mask, uint64_t f) {
  std::map<uint64_t, std::vector<double>> q;
  for (uint64_t i = 0; i < m; i++)
    if (mask >> i & 1) q[i] = std::vector<double>(outs + i * v, outs + (i + 1) * v);
  auto l = ensemble_label(q, f);
  return l ? static_cast<int64_t>(*l) : -1;
}

// leaf_hash(result_leaf(req, res)) (src/messages.cpp:204-211,
// src/merkle.cpp:22-25) for one (request, provider).
int ref_result_leaf_hash(const uint8_t* req_enc, uint64_t req_len,
                         uint64_t node, const char* gid, uint64_t version,
                         const double* output, uint64_t v,
                         const uint8_t* model_digest, uint8_t* out) {
  try {
    Decoder d(ByteView(req_enc, req_len));
    auto req = InferenceRequest::decode(d);
    InferenceResult res;
    res.request_id = req.request_id;
    res.node_index = node;
    res.group_id = gid;
    res.group_version = version;
    res.output.assign(output, output + v);
    res.model_digest = to_h32(model_digest);
    Hash32 h = merkle::leaf_hash(result_leaf(req, res));
    std::memcpy(out, h.data.data(), 32);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// ---------------------------------------------------------------------------
// Batch certification on the CPU: the reference's functions in hot-path order
// (SURVEY.md §8(d) CPU baseline). A handle holds the decoded requests so the
// timed call does only the per-batch work.

struct RefBatch {
  std::vector<InferenceRequest> reqs;
  std::vector<OpEntry> ops;
  std::string gid;
};

void* ref_batch_new(const uint8_t* enc, const uint64_t* lens, uint64_t B,
                    uint64_t version) {
  try {
    auto* b = new RefBatch();
    uint64_t off = 0;
    for (uint64_t i = 0; i < B; i++) {
      Decoder d(ByteView(enc + off, lens[i]));
      b->reqs.push_back(InferenceRequest::decode(d));
      off += lens[i];
      OpEntry op;
      op.kind = OpKind::request_inf;
      op.request = b->reqs.back();
      op.version = version;
      op.status = OpStatus::ok;
      b->ops.push_back(std::move(op));
    }
    if (B) b->gid = b->reqs[0].group_id;
    return b;
  } catch (const std::exception&) {
    return nullptr;
  }
}

void ref_batch_free(void* h) { delete static_cast<RefBatch*>(h); }

// outputs: N × B × v (provider-major). Writes per request: selected mask,
// diameter, satisfied, label (-1 none); per provider the R root; the A root
// and manifest length. threads<=1 runs the reference's Tree::build verbatim;
// threads>1 shards leaf hashing across std::threads and folds with the same
// H(0x01||L||R) rule (src/merkle.cpp:14-19), giving identical roots.
// missing (optional, B flags): request k has no result from any provider
// (execute_batch skipped it as a misfit, engine.cpp:286-291): its R leaves are
// missing_result_leaf and try_attest leaves it unsatisfied without running
// select_quorum (coordinator.cpp:748-771).
int ref_certify_batch_ex(void* h, uint64_t N, uint64_t f, uint32_t metric,
                         double eps_default, const double* outputs, uint64_t v,
                         uint64_t version, const uint8_t* model_digests,
                         uint64_t view, uint64_t seq, int threads,
                         uint64_t* sel_mask, double* diam, uint8_t* satisfied,
                         int64_t* label, uint8_t* r_roots, uint8_t* a_root,
                         uint64_t* manifest_len, const uint8_t* missing) {
  try {
    auto* b = static_cast<RefBatch*>(h);
    const uint64_t B = b->reqs.size();
    auto miss = [&](uint64_t k) { return missing && missing[k]; };
    // results[p][k]
    std::vector<std::map<uint64_t, InferenceResult>> results(N);
    for (uint64_t p = 0; p < N; p++) {
      for (uint64_t k = 0; k < B; k++) {
        if (miss(k)) continue;
        InferenceResult r;
        r.request_id = b->reqs[k].request_id;
        r.node_index = p;
        r.group_id = b->gid;
        r.group_version = version;
        const double* o = outputs + (p * B + k) * v;
        r.output.assign(o, o + v);
        r.model_digest = to_h32(model_digests + 32 * p);
        results[p][k] = std::move(r);
      }
    }
    const int T = std::max(1, threads);
    auto parallel_for = [&](uint64_t n, auto&& fn) {
      if (T <= 1 || n < 2) {
        for (uint64_t i = 0; i < n; i++) fn(i);
        return;
      }
      std::atomic<uint64_t> next{0};
      std::vector<std::thread> ws;
      for (int t = 0; t < T; t++)
        ws.emplace_back([&] {
          for (uint64_t i; (i = next++) < n;) fn(i);
        });
      for (auto& w : ws) w.join();
    };

    // Agreement: select_quorum over all N outputs + label vote.
    std::vector<distance::AgreementOutcome> outc(B);
    parallel_for(B, [&](uint64_t k) {
      if (miss(k)) {  // fewer than N-f outputs: unsatisfied, select_quorum not run
        sel_mask[k] = 0;
        diam[k] = 0;
        satisfied[k] = 0;
        label[k] = -1;
        return;
      }
      std::map<uint64_t, std::vector<double>> outs;
      for (uint64_t p = 0; p < N; p++) outs[p] = results[p][k].output;
      double eps = b->reqs[k].epsilon_override ? *b->reqs[k].epsilon_override
                                               : eps_default;
      outc[k] = distance::select_quorum(
          outs, N, f, static_cast<distance::Metric>(metric), eps);
      uint64_t mask = 0;
      for (auto i : outc[k].selected) mask |= uint64_t{1} << i;
      sel_mask[k] = mask;
      diam[k] = outc[k].diameter;
      satisfied[k] = outc[k].satisfied ? 1 : 0;
      std::map<uint64_t, std::vector<double>> q;
      for (auto i : outc[k].selected) q[i] = outs[i];
      auto l = outc[k].satisfied ? ensemble_label(q, f) : std::nullopt;
      label[k] = l ? static_cast<int64_t>(*l) : -1;
    });

    // R trees (build_result_tree, src/messages.cpp:235-258).
    std::map<uint64_t, Hash32> r_root_map;
    if (T <= 1) {
      for (uint64_t p = 0; p < N; p++)
        r_root_map[p] = build_result_tree(view, seq, b->ops, results[p]).root();
    } else {
      std::vector<Hash32> leaves(N * B);
      parallel_for(N * B, [&](uint64_t i) {
        uint64_t p = i / B, k = i % B;
        leaves[i] = miss(k) ? merkle::leaf_hash(missing_result_leaf(*b->ops[k].request))
                            : merkle::leaf_hash(result_leaf(*b->ops[k].request, results[p][k]));
      });
      for (uint64_t p = 0; p < N; p++) {
        std::vector<Hash32> lvl(leaves.begin() + p * B,
                                leaves.begin() + (p + 1) * B);
        while (lvl.size() > 1) {
          std::vector<Hash32> nx;
          for (size_t i = 0; i < lvl.size(); i += 2) {
            if (i + 1 < lvl.size()) {
              const uint8_t dom = 0x01;
              nx.push_back(hash_concat(
                  {ByteView(&dom, 1), ByteView(lvl[i].data.data(), 32),
                   ByteView(lvl[i + 1].data.data(), 32)}));
            } else {
              nx.push_back(lvl[i]);
            }
          }
          lvl.swap(nx);
        }
        r_root_map[p] = lvl[0];
      }
    }
    for (uint64_t p = 0; p < N; p++)
      std::memcpy(r_roots + 32 * p, r_root_map[p].data.data(), 32);

    // Attestation manifest (restated from Coordinator::try_attest,
    // src/coordinator.cpp:774-832; all N providers present).
    std::vector<AttestLeafRef> manifest;
    std::set<uint64_t> whole;
    for (uint64_t p = 0; p < N; p++) {
      bool all = true;
      for (uint64_t k = 0; k < B; k++) {
        if (!outc[k].satisfied || !outc[k].selected.count(p)) {
          all = false;
          break;
        }
      }
      if (all) whole.insert(p);
    }
    for (uint64_t p : whole) {
      AttestLeafRef ref;
      ref.kind = AttestLeafRef::Kind::whole_batch;
      ref.node = p;
      manifest.push_back(ref);
    }
    for (uint64_t k = 0; k < B; k++) {
      if (!outc[k].satisfied) continue;
      for (uint64_t p : outc[k].selected) {
        if (whole.count(p)) continue;
        AttestLeafRef ref;
        ref.kind = AttestLeafRef::Kind::single;
        ref.node = p;
        ref.op_index = k;
        manifest.push_back(ref);
      }
    }
    for (uint64_t k = 0; k < B; k++) {
      if (outc[k].satisfied) continue;
      AttestLeafRef ref;
      ref.kind = AttestLeafRef::Kind::failure;
      ref.op_index = k;
      manifest.push_back(ref);
    }
    std::map<uint64_t, std::map<uint64_t, InferenceResult>> by_op;
    for (uint64_t k = 0; k < B; k++)
      if (!miss(k))
        for (uint64_t p = 0; p < N; p++) by_op[k][p] = results[p][k];
    std::vector<Bytes> a_leaves(manifest.size());
    parallel_for(manifest.size(), [&](uint64_t i) {
      a_leaves[i] = *attest_leaf_bytes(manifest[i], b->ops, r_root_map, by_op);
    });
    *manifest_len = manifest.size();
    if (!a_leaves.empty()) {
      Hash32 a = merkle::Tree::build(a_leaves).root();
      std::memcpy(a_root, a.data.data(), 32);
    } else {
      std::memset(a_root, 0, 32);
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

// hash_ops (src/messages.cpp:197-202) over n request ops (encodings back to
// back), OpEntry{request_inf, request, no group op, versions[i], statuses[i],
// reasons[i]} (reasons NULL: "").
int ref_hash_ops(const uint8_t* encs, const uint64_t* lens, uint64_t n, const uint64_t* versions,
                 const uint8_t* statuses, const char* const* reasons, uint8_t* out) {
  try {
    std::vector<OpEntry> ops;
    uint64_t off = 0;
    for (uint64_t i = 0; i < n; i++) {
      Decoder d(ByteView(encs + off, lens[i]));
      OpEntry op;
      op.kind = OpKind::request_inf;
      op.request = InferenceRequest::decode(d);
      op.version = versions[i];
      op.status = static_cast<OpStatus>(statuses[i]);
      op.reason = reasons ? std::string(reasons[i]) : std::string();
      ops.push_back(std::move(op));
      off += lens[i];
    }
    Hash32 h = hash_ops(ops);
    std::memcpy(out, h.data.data(), 32);
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

int ref_certify_batch(void* h, uint64_t N, uint64_t f, uint32_t metric, double eps_default,
                      const double* outputs, uint64_t v, uint64_t version,
                      const uint8_t* model_digests, uint64_t view, uint64_t seq, int threads,
                      uint64_t* sel_mask, double* diam, uint8_t* satisfied, int64_t* label,
                      uint8_t* r_roots, uint8_t* a_root, uint64_t* manifest_len) {
  return ref_certify_batch_ex(h, N, f, metric, eps_default, outputs, v, version, model_digests,
                              view, seq, threads, sel_mask, diam, satisfied, label, r_roots,
                              a_root, manifest_len, nullptr);
}

// A mixed PRE-PREPARE op list through the reference: build_result_tree
// (messages.cpp:235-258) per provider and the try_attest manifest
// (coordinator.cpp:735-849, restated above in ref_certify_batch_ex with
// outcomes only for ok request ops) + attest_leaf_bytes. ops: kinds[k] 0 ok
// request (the next encoding), 1 rejected request (next encoding, status
// rejected, reasons[k]), 2 group op (an activate_group op signed here,
// status ok, or rejected when reasons[k] is non-empty). outputs: N x B x v
// provider-major; rows of non-ok ops are ignored. Writes every op's
// OpEntry::encode (entries, entry_lens) and, for rejected ops, the
// FailureRecord::encode (recs, rec_lens), so the GPU path can be fed the
// same bytes; caps are per-op byte capacities.
int ref_certify_slot(const uint8_t* enc, const uint64_t* lens, uint64_t B, const uint8_t* kinds,
                     const char* const* reasons, uint64_t N, uint64_t f, double eps_default,
                     const double* outputs, uint64_t v, uint64_t version,
                     const uint8_t* model_digests, uint8_t* r_roots, uint8_t* a_root,
                     uint64_t* manifest_len, uint8_t* sat_out, uint8_t* entries,
                     uint64_t* entry_lens, uint8_t* recs, uint64_t* rec_lens, uint64_t cap) {
  try {
    std::vector<OpEntry> ops(B);
    KeyPair owner = KeyPair::from_seed(std::array<uint8_t, 32>{42});
    uint64_t off = 0;
    std::string gid;
    for (uint64_t k = 0; k < B; k++) {
      OpEntry& op = ops[k];
      op.version = version;
      if (kinds[k] <= 1) {
        Decoder d(ByteView(enc + off, lens[k]));
        op.kind = OpKind::request_inf;
        op.request = InferenceRequest::decode(d);
        gid = op.request->group_id;
        op.status = kinds[k] == 1 ? OpStatus::rejected : OpStatus::ok;
        if (kinds[k] == 1) op.reason = reasons[k];
      } else {
        Encoder ne;
        ne.u64(k);
        op.kind = OpKind::activate_group;
        op.group_op = make_signed_group_op(owner, ne.take(), OpKind::activate_group, "group-1",
                                           std::nullopt);
        if (reasons[k][0]) {
          op.status = OpStatus::rejected;
          op.reason = reasons[k];
        }
      }
      off += lens[k];
    }
    // per provider results for the ok request ops
    std::vector<std::map<uint64_t, InferenceResult>> results(N);
    std::map<uint64_t, std::map<uint64_t, InferenceResult>> by_op;
    std::map<uint64_t, distance::AgreementOutcome> outc;
    for (uint64_t k = 0; k < B; k++) {
      if (ops[k].kind != OpKind::request_inf || ops[k].status != OpStatus::ok) continue;
      std::map<uint64_t, std::vector<double>> outs;
      for (uint64_t p = 0; p < N; p++) {
        InferenceResult r;
        r.request_id = ops[k].request->request_id;
        r.node_index = p;
        r.group_id = ops[k].request->group_id;
        r.group_version = version;
        const double* o = outputs + (p * B + k) * v;
        r.output.assign(o, o + v);
        r.model_digest = to_h32(model_digests + 32 * p);
        results[p][k] = r;
        by_op[k][p] = r;
        outs[p] = r.output;
      }
      double eps = ops[k].request->epsilon_override ? *ops[k].request->epsilon_override
                                                    : eps_default;
      outc[k] = distance::select_quorum(outs, N, f, distance::Metric::euclidean, eps);
    }
    std::map<uint64_t, Hash32> r_root_map;
    for (uint64_t p = 0; p < N; p++) {
      r_root_map[p] = build_result_tree(0, 1, ops, results[p]).root();
      std::memcpy(r_roots + 32 * p, r_root_map[p].data.data(), 32);
    }
    std::vector<AttestLeafRef> manifest;
    std::set<uint64_t> whole;
    for (uint64_t p = 0; p < N; p++) {
      bool all = true;
      for (const auto& [k, o] : outc)
        if (!o.satisfied || !o.selected.count(p)) {
          all = false;
          break;
        }
      if (all) whole.insert(p);
    }
    for (uint64_t p : whole) {
      AttestLeafRef ref;
      ref.kind = AttestLeafRef::Kind::whole_batch;
      ref.node = p;
      manifest.push_back(ref);
    }
    for (const auto& [k, o] : outc) {
      if (!o.satisfied) continue;
      for (uint64_t p : o.selected) {
        if (whole.count(p)) continue;
        AttestLeafRef ref;
        ref.kind = AttestLeafRef::Kind::single;
        ref.node = p;
        ref.op_index = k;
        manifest.push_back(ref);
      }
    }
    for (uint64_t k = 0; k < B; k++) {
      bool failed = ops[k].status == OpStatus::rejected;
      if (ops[k].kind == OpKind::request_inf && ops[k].status == OpStatus::ok)
        failed = !outc.at(k).satisfied;
      if (!failed) continue;
      AttestLeafRef ref;
      ref.kind = AttestLeafRef::Kind::failure;
      ref.op_index = k;
      manifest.push_back(ref);
    }
    std::vector<Bytes> leaves;
    for (const auto& ref : manifest) leaves.push_back(*attest_leaf_bytes(ref, ops, r_root_map, by_op));
    Hash32 a = merkle::Tree::build(leaves).root();
    std::memcpy(a_root, a.data.data(), 32);
    *manifest_len = manifest.size();
    for (uint64_t k = 0; k < B; k++) {
      sat_out[k] = outc.count(k) && outc.at(k).satisfied ? 1 : 0;
      Encoder e;
      ops[k].encode(e);
      Bytes b = e.take();
      entry_lens[k] = b.size();
      if (b.size() > cap) return -2;
      std::memcpy(entries + k * cap, b.data(), b.size());
      rec_lens[k] = 0;
      if (ops[k].status == OpStatus::rejected) {
        Encoder r;
        failure_record_for(ops[k]).encode(r);
        Bytes rb = r.take();
        if (rb.size() > cap) return -2;
        rec_lens[k] = rb.size();
        std::memcpy(recs + k * cap, rb.data(), rb.size());
      }
    }
    return 0;
  } catch (const std::exception&) {
    return -1;
  }
}

}  // extern "C"
