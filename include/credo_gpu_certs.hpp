// Certificate assembly and verification at batch scale on the B200 path
// (SURVEY §8(f)1): the reference-side bindings for
//
//   assemble_responses : ProxyCore's assemble_response for every op of an
//                        OrderedSlot, with rebuild_committer_trees and the
//                        provider result trees (src/proxy.cpp:28-186)
//   verify_responses   : verify_response / verify_cert / verify_failure over
//                        a response set (src/certificate.cpp:215-347)
//
// Both spend their time re-hashing leaves that stream whole requests
// (result_leaf 0x52, single_attest_leaf 0x53, missing_result_leaf 0x4D:
// 1.2 MB each at ImageNet shape). Those run on the GPU through
// cg_cert_leaf_hashes (one midstate per (request, tag), shared by every
// result of the request); tree levels, auth paths and path folds run through
// cg_merkle_auth_paths / cg_merkle_path_roots. The small leaves (whole-batch
// R roots, failure records, group ops, noops), the signature digests and the
// Ed25519 checks are the reference's own functions on the host. The results
// are the reference's, value for value (oracle/integration_verify.cpp checks
// them against assemble_response / verify_response on run_scenario slots and
// on forged certificates).
#pragma once

#include <algorithm>
#include <atomic>
#include <map>
#include <optional>
#include <set>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#include "credo/certificate.hpp"
#include "credo/coordinator.hpp"
#include "credo/merkle.hpp"
#include "credo/messages.hpp"
#include "credo_gpu_adapters.hpp"

namespace credo::gpu {

// Leaf hashes over requests, computed in one cg_cert_leaf_hashes call per
// (group id, input length) -- the C-ABI batch is uniform in both.
class LeafHasher {
 public:
  enum Kind : uint8_t { result = 1, single = 2, missing = 4 };

  // Registers leaf_hash(result_leaf / single_attest_leaf(req, res)) or
  // leaf_hash(missing_result_leaf(req)) (res unused); returns its index.
  size_t add(const InferenceRequest& req, const InferenceResult* res, Kind kind) {
    Batch& b = batches_[{req.group_id, req.input.size()}];
    // one prefix per distinct request: the same object, or an equal copy
    // (a response set usually carries its request once per response)
    uint32_t k = UINT32_MAX;
    if (auto it = b.index.find(&req); it != b.index.end()) k = it->second;
    else {
      for (uint32_t c : b.by_id[req.request_id])
        if (*b.reqs[c] == req) { k = c; break; }
      if (k == UINT32_MAX) {
        k = (uint32_t)b.reqs.size();
        b.reqs.push_back(&req);
        b.by_id[req.request_id].push_back(k);
      }
      b.index.emplace(&req, k);
    }
    Entry e{k, kind, {}, out_.size()};
    if (kind != missing) {
      Encoder enc;
      res->encode(enc);
      e.enc = enc.take();
    }
    b.entries.push_back(std::move(e));
    out_.emplace_back();
    return out_.size() - 1;
  }

  void run(Context& ctx) {
    for (auto& [key, b] : batches_) {
      const uint32_t B = (uint32_t)b.reqs.size();
      const uint64_t u = key.second;
      std::vector<uint8_t> ids(32 * (size_t)B), has_eps(B), pubs(32 * (size_t)B),
          sigs(64 * (size_t)B), nonces;
      std::vector<double> eps(B), in((size_t)B * u);
      std::vector<uint64_t> nonce_lens(B);
      for (uint32_t k = 0; k < B; k++) {
        const InferenceRequest& r = *b.reqs[k];
        std::memcpy(&ids[32 * (size_t)k], r.request_id.data.data(), 32);
        std::copy(r.input.begin(), r.input.end(), in.begin() + (size_t)k * u);
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
      const uint32_t M = (uint32_t)b.entries.size();
      std::vector<uint32_t> ridx(M);
      std::vector<uint8_t> want(M), enc;
      std::vector<uint64_t> lens(M);
      for (uint32_t m = 0; m < M; m++) {
        ridx[m] = b.entries[m].req;
        want[m] = b.entries[m].kind;
        lens[m] = b.entries[m].enc.size();
        enc.insert(enc.end(), b.entries[m].enc.begin(), b.entries[m].enc.end());
      }
      std::vector<uint8_t> h52(32 * (size_t)M), h53(32 * (size_t)M), h4d(32 * (size_t)M);
      check(ctx.get(), cg_cert_leaf_hashes(ctx.get(), &bt, key.first.data(), key.first.size(), M,
                                           ridx.data(), want.data(), enc.data(), lens.data(),
                                           h52.data(), h53.data(), h4d.data()));
      for (uint32_t m = 0; m < M; m++) {
        const uint8_t* src = b.entries[m].kind == result ? &h52[32 * (size_t)m]
                             : b.entries[m].kind == single ? &h53[32 * (size_t)m]
                                                           : &h4d[32 * (size_t)m];
        std::memcpy(out_[b.entries[m].out].data.data(), src, 32);
      }
    }
    batches_.clear();
  }

  const Hash32& operator[](size_t i) const { return out_[i]; }

 private:
  struct Entry {
    uint32_t req;
    Kind kind;
    Bytes enc;
    size_t out;
  };
  struct Batch {
    std::vector<const InferenceRequest*> reqs;
    std::map<const InferenceRequest*, uint32_t> index;
    std::map<Hash32, std::vector<uint32_t>> by_id;
    std::vector<Entry> entries;
  };
  std::map<std::pair<std::string, size_t>, Batch> batches_;
  std::vector<Hash32> out_;
};

// Host restatement of merkle.cpp's internal fold step (the reference keeps
// internal_hash private, merkle.cpp:14-19): H(0x01 || left || right).
inline Hash32 internal_hash_host(const Hash32& l, const Hash32& r) {
  Bytes b(65);
  b[0] = 0x01;
  std::memcpy(&b[1], l.data.data(), 32);
  std::memcpy(&b[33], r.data.data(), 32);
  return host_hash(b);
}

// get_merkle_root(path, leaf) for many paths from their leaf hashes
// (merkle.cpp:86-93): cg_merkle_path_roots for paths of <= 64 steps (every
// tree that fits in memory), the host fold for longer (forged) ones.
inline std::vector<Hash32> fold_paths(Context& ctx, const std::vector<Hash32>& leaves,
                                      const std::vector<const merkle::AuthPath*>& paths) {
  constexpr size_t kSteps = 64;
  const size_t n = paths.size();
  std::vector<Hash32> roots(n);
  std::vector<size_t> dev;
  for (size_t i = 0; i < n; i++)
    if (paths[i]->siblings.size() <= kSteps) dev.push_back(i);
    else {
      Hash32 h = leaves[i];
      for (const auto& s : paths[i]->siblings)
        h = s.side == merkle::Side::left ? internal_hash_host(s.sibling, h)
                                         : internal_hash_host(h, s.sibling);
      roots[i] = h;
    }
  if (dev.empty()) return roots;
  const size_t c = dev.size();
  std::vector<uint8_t> lh(32 * c), sib(32 * kSteps * c), sides(kSteps * c), out(32 * c);
  std::vector<uint32_t> lens(c);
  for (size_t j = 0; j < c; j++) {
    const auto& p = *paths[dev[j]];
    std::memcpy(&lh[32 * j], leaves[dev[j]].data.data(), 32);
    lens[j] = (uint32_t)p.siblings.size();
    for (size_t s = 0; s < p.siblings.size(); s++) {
      std::memcpy(&sib[32 * (kSteps * j + s)], p.siblings[s].sibling.data.data(), 32);
      sides[kSteps * j + s] = (uint8_t)p.siblings[s].side;
    }
  }
  check(ctx.get(), cg_merkle_path_roots(ctx.get(), lh.data(), sib.data(), sides.data(),
                                        lens.data(), (uint32_t)c, out.data()));
  for (size_t j = 0; j < c; j++) std::memcpy(roots[dev[j]].data.data(), &out[32 * j], 32);
  return roots;
}

// merkle::Tree over precomputed leaf hashes: root and every leaf's path.
// Small trees (a slot's few committers / providers) are folded on the host
// with SHA-NI (65-byte internal nodes); large ones on the GPU.
struct HashTree {
  Hash32 root{};
  std::vector<merkle::AuthPath> paths;
};
inline HashTree build_hash_tree(Context& ctx, const std::vector<Hash32>& leaves) {
  constexpr size_t kSteps = 64, kHostMax = 4096;
  const size_t n = leaves.size();
  HashTree t;
  t.paths.resize(n);
  if (n <= kHostMax) {  // Tree::build + auth_path (merkle.cpp:47-84)
    std::vector<std::vector<Hash32>> lv{leaves};
    while (lv.back().size() > 1) {
      const auto& prev = lv.back();
      std::vector<Hash32> next;
      for (size_t i = 0; i < prev.size(); i += 2)
        next.push_back(i + 1 < prev.size() ? internal_hash_host(prev[i], prev[i + 1]) : prev[i]);
      lv.push_back(std::move(next));
    }
    t.root = lv.back().back();
    for (size_t i = 0; i < n; i++) {
      size_t idx = i;
      for (size_t l = 0; l + 1 < lv.size(); l++) {
        if (idx % 2 == 1) t.paths[i].siblings.push_back({lv[l][idx - 1], merkle::Side::left});
        else if (idx + 1 < lv[l].size())
          t.paths[i].siblings.push_back({lv[l][idx + 1], merkle::Side::right});
        idx /= 2;
      }
    }
    return t;
  }
  std::vector<uint8_t> lh(32 * n), sib(32 * kSteps * n), sides(kSteps * n);
  std::vector<uint64_t> idx(n);
  std::vector<uint32_t> lens(n);
  for (size_t i = 0; i < n; i++) {
    std::memcpy(&lh[32 * i], leaves[i].data.data(), 32);
    idx[i] = i;
  }
  check(ctx.get(), cg_merkle_auth_paths(ctx.get(), lh.data(), n, idx.data(), (uint32_t)n,
                                        sib.data(), sides.data(), lens.data(),
                                        t.root.data.data()));
  for (size_t i = 0; i < n; i++)
    for (uint32_t s = 0; s < lens[i]; s++) {
      merkle::PathStep st;
      std::memcpy(st.sibling.data.data(), &sib[32 * (kSteps * i + s)], 32);
      st.side = sides[kSteps * i + s] ? merkle::Side::right : merkle::Side::left;
      t.paths[i].siblings.push_back(st);
    }
  return t;
}

// ---------------------------------------------------------------- assembly

namespace detail {
// One slot's trees: rebuild_committer_trees (proxy.cpp:28-48) and every
// provider's result tree (build_result_tree, messages.cpp:235-258), leaves
// registered with a LeafHasher shared by all slots of the call.
struct SlotTrees {
  using Ref = std::pair<bool, size_t>;  // (GPU leaf, LeafHasher index) / host leaf index
  struct Committer {
    uint64_t node;
    const CommitMsg* commit;
    std::vector<Ref> leaf;
    HashTree tree;
  };
  std::vector<Committer> cts;
  std::map<uint64_t, std::vector<Ref>> rleaf;
  std::map<uint64_t, HashTree> rtree;
  std::vector<Hash32> host;

  void plan(const OrderedSlot& slot, LeafHasher& lh) {
    const size_t nops = slot.ops.size();
    for (const auto& [c, commit] : slot.commits) {
      Committer ct{c, &commit, {}, {}};
      bool complete = true;
      for (const AttestLeafRef& ref : commit.manifest) {  // attest_leaf_bytes, messages.cpp:315-343
        if (ref.kind == AttestLeafRef::Kind::whole_batch) {
          auto it = slot.r_roots.find(ref.node);
          if (it == slot.r_roots.end()) { complete = false; break; }
          ct.leaf.push_back({false, host.size()});
          host.push_back(merkle::leaf_hash(whole_batch_leaf(it->second)));
        } else if (ref.kind == AttestLeafRef::Kind::single) {
          if (ref.op_index >= nops) { complete = false; break; }
          const OpEntry& op = slot.ops[ref.op_index];
          if (op.kind != OpKind::request_inf) { complete = false; break; }
          auto oit = slot.results_by_op.find(ref.op_index);
          if (oit == slot.results_by_op.end()) { complete = false; break; }
          auto rit = oit->second.find(ref.node);
          if (rit == oit->second.end()) { complete = false; break; }
          ct.leaf.push_back({true, lh.add(*op.request, &rit->second, LeafHasher::single)});
        } else {
          if (ref.op_index >= nops) { complete = false; break; }
          ct.leaf.push_back({false, host.size()});
          host.push_back(merkle::leaf_hash(failure_leaf(failure_record_for(slot.ops[ref.op_index]))));
        }
      }
      if (complete && !ct.leaf.empty()) cts.push_back(std::move(ct));
    }
    std::set<uint64_t> providers;
    for (const auto& [k, per] : slot.results_by_op)
      for (const auto& [p, r] : per) providers.insert(p);
    for (uint64_t p : providers) {
      auto& L = rleaf[p];
      if (slot.ops.empty()) {
        L.push_back({false, host.size()});
        host.push_back(merkle::leaf_hash(noop_leaf(slot.view, slot.seq)));
      }
      for (size_t k = 0; k < nops; k++) {
        const OpEntry& op = slot.ops[k];
        if (op.kind == OpKind::request_inf) {
          const InferenceResult* mine = nullptr;
          if (auto it = slot.results_by_op.find(k); it != slot.results_by_op.end())
            if (auto jt = it->second.find(p); jt != it->second.end()) mine = &jt->second;
          L.push_back({true, lh.add(*op.request, mine,
                                    mine ? LeafHasher::result : LeafHasher::missing)});
        } else {
          L.push_back({false, host.size()});
          host.push_back(merkle::leaf_hash(group_op_leaf(op)));
        }
      }
    }
  }

  void build(Context& ctx, const LeafHasher& lh) {
    auto leaves_of = [&](const std::vector<Ref>& refs) {
      std::vector<Hash32> v;
      for (auto [dev, i] : refs) v.push_back(dev ? lh[i] : host[i]);
      return v;
    };
    for (Committer& ct : cts) ct.tree = build_hash_tree(ctx, leaves_of(ct.leaf));
    for (auto& [p, L] : rleaf) rtree[p] = build_hash_tree(ctx, leaves_of(L));
  }

  // assemble_response's body (proxy.cpp:80-186) with the trees prebuilt
  std::optional<InferenceResponse> respond(const OrderedSlot& slot, size_t op_index,
                                           const ClusterConfig& config) const {
    const uint64_t n = config.n(), f = config.f;
    if (op_index >= slot.ops.size()) return std::nullopt;
    const OpEntry& op = slot.ops[op_index];
    if (op.kind != OpKind::request_inf || !op.request) return std::nullopt;
    InferenceResponse resp;
    resp.request_id = op.request->request_id;
    if (auto oc = slot.outcomes.find(op_index); oc != slot.outcomes.end()) {
      resp.distance = oc->second.descriptor;
      resp.effective_epsilon = oc->second.epsilon;
    }
    if (op.status == OpStatus::ok) {
      auto results_it = slot.results_by_op.find(op_index);
      if (results_it != slot.results_by_op.end()) {
        InferenceCertificate cert;
        cert.view = slot.view;
        cert.seq = slot.seq;
        cert.h_ops = slot.h_ops;
        cert.primary_r_root = slot.primary_r_root;
        cert.pre_prepare_sig = slot.pre_prepare_sig;
        std::vector<InferenceResult> covered;
        for (const auto& [p, result] : results_it->second) {
          auto root_it = slot.r_roots.find(p);
          if (root_it == slot.r_roots.end()) continue;
          std::optional<Signature> order_sig;
          if (p != slot.primary) {
            auto sig_it = slot.prepare_sigs.find(p);
            if (sig_it == slot.prepare_sigs.end()) continue;
            order_sig = sig_it->second;
          }
          std::vector<CertAttestation> atts;
          for (const Committer& ct : cts) {
            // covering_index (proxy.cpp:52-66): the first whole-batch entry
            // for p or single entry for (op, p)
            const auto& man = ct.commit->manifest;
            for (size_t i = 0; i < man.size(); i++) {
              const bool whole = man[i].kind == AttestLeafRef::Kind::whole_batch && man[i].node == p;
              const bool one = man[i].kind == AttestLeafRef::Kind::single && man[i].node == p &&
                               man[i].op_index == op_index;
              if (!whole && !one) continue;
              CertAttestation att;
              att.attestor = ct.node;
              att.kind = man[i].kind;
              att.path = ct.tree.paths[i];
              atts.push_back(std::move(att));
              break;
            }
          }
          if (atts.size() <= f) continue;
          const HashTree& rt = rtree.at(p);
          if (rt.root != root_it->second) continue;
          cert.result_paths[p] = rt.paths[op_index];
          if (order_sig) cert.sigs[p].order_sig = *order_sig;
          for (const CertAttestation& att : atts)
            cert.sigs[att.attestor].commit_sig = slot.commits.at(att.attestor).sig;
          cert.attestations[p] = std::move(atts);
          covered.push_back(result);
        }
        if (covered.size() >= n - f) {
          std::sort(covered.begin(), covered.end(),
                    [](const InferenceResult& a, const InferenceResult& b) {
                      return a.node_index < b.node_index;
                    });
          resp.kind = InferenceResponse::Kind::success;
          resp.results = std::move(covered);
          resp.certificate = std::move(cert);
          return resp;
        }
      }
    }
    FailureCertificate fc;  // certified failure (proxy.cpp:163-184)
    fc.view = slot.view;
    fc.seq = slot.seq;
    fc.h_ops = slot.h_ops;
    fc.primary_r_root = slot.primary_r_root;
    fc.pre_prepare_sig = slot.pre_prepare_sig;
    fc.record = failure_record_for(op);
    for (const Committer& ct : cts) {
      const auto& man = ct.commit->manifest;
      for (size_t i = 0; i < man.size(); i++)
        if (man[i].kind == AttestLeafRef::Kind::failure && man[i].op_index == op_index) {
          FailureCertificate::Attest att;
          att.attestor = ct.node;
          att.path = ct.tree.paths[i];
          att.commit_sig = ct.commit->sig;
          fc.attests.push_back(std::move(att));
          break;
        }
    }
    if (fc.attests.size() <= f) return std::nullopt;
    resp.kind = InferenceResponse::Kind::failure;
    resp.failure = std::move(fc);
    return resp;
  }
};
}  // namespace detail

// assemble_response(slot, k, config) for every op k of every slot
// (proxy.cpp:80-186): the request-streaming leaves of all slots hashed on the
// GPU in one pass, each slot's committer and result trees rebuilt once.
inline std::vector<std::vector<std::optional<InferenceResponse>>> assemble_responses(
    Context& ctx, const std::vector<const OrderedSlot*>& slots, const ClusterConfig& config) {
  LeafHasher lh;
  std::vector<detail::SlotTrees> trees(slots.size());
  for (size_t s = 0; s < slots.size(); s++) trees[s].plan(*slots[s], lh);
  lh.run(ctx);
  std::vector<std::vector<std::optional<InferenceResponse>>> out(slots.size());
  for (size_t s = 0; s < slots.size(); s++) {
    trees[s].build(ctx, lh);
    for (size_t k = 0; k < slots[s]->ops.size(); k++)
      out[s].push_back(trees[s].respond(*slots[s], k, config));
  }
  return out;
}

inline std::vector<std::optional<InferenceResponse>> assemble_responses(
    Context& ctx, const OrderedSlot& slot, const ClusterConfig& config) {
  return assemble_responses(ctx, std::vector<const OrderedSlot*>{&slot}, config)[0];
}

// ------------------------------------------------------------ verification

// verify_response(requests[i], responses[i], config) for every i
// (certificate.cpp:215-347): all leaf hashes and path folds of the whole set
// on the GPU in a few launches, then the reference's checks in its order
// with the signatures verified on the host.
inline std::vector<bool> verify_responses(Context& ctx,
                                          const std::vector<InferenceRequest>& requests,
                                          const std::vector<InferenceResponse>& responses,
                                          const ClusterConfig& config) {
  const size_t R = std::min(requests.size(), responses.size());
  std::vector<bool> ok(R, false);
  const bool cfg_ok = !config.validate();
  const uint64_t n = config.n(), f = config.f;
  LeafHasher lh;
  // per response: leaf indices of its results' R leaves and single leaves
  struct Plan {
    std::vector<size_t> rleaf;                    // per result
    std::vector<std::vector<size_t>> aleaf;       // per result, per attestation (single)
  };
  std::vector<Plan> plan(R);
  auto shaped = [&](size_t i) {  // the checks that need no digest
    const InferenceRequest& req = requests[i];
    const InferenceResponse& resp = responses[i];
    if (resp.request_id != req.request_id) return false;
    if (resp.kind == InferenceResponse::Kind::success) {
      if (!resp.certificate || resp.results.empty()) return false;
      for (size_t j = 1; j < resp.results.size(); j++)
        if (resp.results[j - 1].node_index >= resp.results[j].node_index) return false;
      return resp.results.size() >= n - f;
    }
    return resp.failure.has_value();
  };
  std::vector<bool> live(R);
  for (size_t i = 0; i < R; i++) {
    live[i] = cfg_ok && shaped(i);
    if (!live[i] || responses[i].kind != InferenceResponse::Kind::success) continue;
    const InferenceResponse& resp = responses[i];
    const InferenceCertificate& cert = *resp.certificate;
    for (const InferenceResult& q : resp.results) {
      plan[i].rleaf.push_back(lh.add(requests[i], &q, LeafHasher::result));
      plan[i].aleaf.emplace_back();
      auto ait = cert.attestations.find(q.node_index);
      if (ait == cert.attestations.end()) continue;
      for (const CertAttestation& att : ait->second)
        plan[i].aleaf.back().push_back(att.kind == AttestLeafRef::Kind::whole_batch
                                           ? SIZE_MAX
                                           : lh.add(requests[i], &q, LeafHasher::single));
    }
  }
  lh.run(ctx);
  // result-tree roots m per (response, result) with a path
  std::vector<Hash32> leaves;
  std::vector<const merkle::AuthPath*> paths;
  std::vector<std::vector<std::optional<size_t>>> mix(R);
  for (size_t i = 0; i < R; i++) {
    if (!live[i] || responses[i].kind != InferenceResponse::Kind::success) continue;
    const auto& cert = *responses[i].certificate;
    for (size_t j = 0; j < responses[i].results.size(); j++) {
      auto pit = cert.result_paths.find(responses[i].results[j].node_index);
      if (pit == cert.result_paths.end()) {
        mix[i].push_back(std::nullopt);
        continue;
      }
      mix[i].push_back(leaves.size());
      leaves.push_back(lh[plan[i].rleaf[j]]);
      paths.push_back(&pit->second);
    }
  }
  const std::vector<Hash32> m_roots = fold_paths(ctx, leaves, paths);
  // attestation-tree roots: whole-batch leaves need m; failure leaves
  leaves.clear();
  paths.clear();
  std::vector<std::vector<std::vector<size_t>>> aix(R);
  std::vector<std::vector<size_t>> fix(R);
  for (size_t i = 0; i < R; i++) {
    if (!live[i]) continue;
    const InferenceResponse& resp = responses[i];
    if (resp.kind == InferenceResponse::Kind::success) {
      const auto& cert = *resp.certificate;
      for (size_t j = 0; j < resp.results.size(); j++) {
        aix[i].emplace_back();
        if (!mix[i][j]) continue;
        auto ait = cert.attestations.find(resp.results[j].node_index);
        if (ait == cert.attestations.end()) continue;
        for (size_t a = 0; a < ait->second.size(); a++) {
          const CertAttestation& att = ait->second[a];
          aix[i][j].push_back(leaves.size());
          leaves.push_back(att.kind == AttestLeafRef::Kind::whole_batch
                               ? merkle::leaf_hash(whole_batch_leaf(m_roots[*mix[i][j]]))
                               : lh[plan[i].aleaf[j][a]]);
          paths.push_back(&att.path);
        }
      }
    } else {
      const Hash32 fl = merkle::leaf_hash(failure_leaf(resp.failure->record));
      for (const auto& att : resp.failure->attests) {
        fix[i].push_back(leaves.size());
        leaves.push_back(fl);
        paths.push_back(&att.path);
      }
    }
  }
  const std::vector<Hash32> a_roots = fold_paths(ctx, leaves, paths);

  auto binding = [&](uint64_t view, uint64_t seq, const Hash32& h_ops, const Hash32& r_root,
                     const Signature& sig, Hash32& h_pp) {  // certificate.cpp:195-209
    const uint64_t p = view % n;
    if (!verify(config.nodes[p].public_key, pre_prepare_signing_digest(view, seq, h_ops, r_root),
                sig))
      return false;
    h_pp = pre_prepare_hash_of(view, seq, h_ops, r_root, sig);
    return true;
  };
  auto check_one = [&](size_t i) -> bool {
    if (!live[i]) return false;
    const InferenceRequest& request = requests[i];
    const InferenceResponse& resp = responses[i];
    try {
      if (resp.kind == InferenceResponse::Kind::success) {  // verify_cert
        const auto& cert = *resp.certificate;
        Hash32 h_pp;
        if (!binding(cert.view, cert.seq, cert.h_ops, cert.primary_r_root, cert.pre_prepare_sig,
                     h_pp))
          return false;
        const uint64_t primary = cert.view % n;
        std::set<uint64_t> providers;
        const uint64_t version = resp.results.front().group_version;
        bool good = true;
        for (size_t j = 0; j < resp.results.size() && good; j++) {
          const InferenceResult& q = resp.results[j];
          const uint64_t p = q.node_index;
          if (p >= n || !providers.insert(p).second || q.request_id != request.request_id ||
              q.group_id != request.group_id || q.group_version != version || !mix[i][j]) {
            good = false;
            break;
          }
          const Hash32& m = m_roots[*mix[i][j]];
          if (p == primary) {
            if (m != cert.primary_r_root) { good = false; break; }
          } else {
            auto sit = cert.sigs.find(p);
            if (sit == cert.sigs.end() || !sit->second.order_sig ||
                !verify(config.nodes[p].public_key,
                        prepare_signing_digest(cert.view, cert.seq, h_pp, p, m),
                        *sit->second.order_sig)) {
              good = false;
              break;
            }
          }
          auto ait = cert.attestations.find(p);
          if (ait == cert.attestations.end()) { good = false; break; }
          std::set<uint64_t> attestors;
          for (size_t a = 0; a < ait->second.size(); a++) {
            const CertAttestation& att = ait->second[a];
            if (att.attestor >= n || !attestors.insert(att.attestor).second) { good = false; break; }
            auto sit = cert.sigs.find(att.attestor);
            if (sit == cert.sigs.end() || !sit->second.commit_sig ||
                !verify(config.nodes[att.attestor].public_key,
                        commit_signing_digest(cert.view, cert.seq, h_pp, att.attestor,
                                              a_roots[aix[i][j][a]]),
                        *sit->second.commit_sig)) {
              good = false;
              break;
            }
          }
          if (good && attestors.size() <= f) good = false;
        }
        return good;
      } else {  // verify_failure
        const auto& fc = *resp.failure;
        if (fc.record.request_id != request.request_id || fc.record.group_id != request.group_id)
          return false;
        Hash32 h_pp;
        if (!binding(fc.view, fc.seq, fc.h_ops, fc.primary_r_root, fc.pre_prepare_sig, h_pp))
          return false;
        std::set<uint64_t> attestors;
        bool good = true;
        for (size_t a = 0; a < fc.attests.size(); a++) {
          const auto& att = fc.attests[a];
          if (att.attestor >= n || !attestors.insert(att.attestor).second ||
              !verify(config.nodes[att.attestor].public_key,
                      commit_signing_digest(fc.view, fc.seq, h_pp, att.attestor,
                                            a_roots[fix[i][a]]),
                      att.commit_sig)) {
            good = false;
            break;
          }
        }
        return good && attestors.size() > f;
      }
    } catch (...) {
      return false;
    }
  };
  // the signature checks (libsodium Ed25519, thread-safe) across host threads
  std::vector<uint8_t> okb(R, 0);
  std::atomic<size_t> next{0};
  auto worker = [&] {
    for (size_t i; (i = next.fetch_add(1)) < R;) okb[i] = check_one(i) ? 1 : 0;
  };
  const size_t nt = std::min<size_t>(std::max(1u, std::thread::hardware_concurrency()), (R + 7) / 8);
  std::vector<std::thread> pool;
  for (size_t t = 1; t < nt; t++) pool.emplace_back(worker);
  worker();
  for (auto& t : pool) t.join();
  for (size_t i = 0; i < R; i++) ok[i] = okb[i] != 0;
  return ok;
}

}  // namespace credo::gpu
