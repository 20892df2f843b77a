// TEST INFRASTRUCTURE — certificate assembly and verification at batch scale
// against the UNMODIFIED reference.
//
// For the reference's own harness scenarios (tests/test_harness.cpp:233-296:
// honest, agree_then_execute, corrupt_result beyond / within epsilon) plus a
// C1-shaped and an ImageNet-shaped workload, run_scenario (stock CPU
// executors) produces every node's ordered slots and every certified
// response. Then:
//   * credo::gpu::assemble_responses(slot) must equal assemble_response(slot,
//     k) (proxy.cpp:80-186) for every op k of every slot of every node;
//   * credo::gpu::verify_responses must equal verify_response
//     (certificate.cpp:325-347) on every response and on forged variants of
//     each (flipped output, sibling, side, attestation kind, signature,
//     attestor, record reason, dropped result, altered request).
// The ImageNet-shaped case (1.2 MB requests) also times both sides.
#include <chrono>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "credo/harness.hpp"
#include "credo/proxy.hpp"
#include "credo_gpu_certs.hpp"

using namespace credo;
using namespace credo::harness;
using Clock = std::chrono::steady_clock;

static double secs(Clock::time_point a) {
  return std::chrono::duration<double>(Clock::now() - a).count();
}

// Variants of one response: every one is a forgery the reference rejects
// except drop_result (N - 1 >= N - f results still verify); GPU and
// reference must agree on all of them.
static std::vector<std::pair<std::string, InferenceResponse>> forgeries(const InferenceResponse& r) {
  std::vector<std::pair<std::string, InferenceResponse>> out;
  auto add = [&](const char* name, const std::function<bool(InferenceResponse&)>& mut) {
    InferenceResponse x = r;
    if (mut(x)) out.emplace_back(name, std::move(x));
  };
  add("output", [](InferenceResponse& x) {
    if (x.results.empty() || x.results[0].output.empty()) return false;
    x.results[0].output[0] += 1e-12;
    return true;
  });
  add("sibling", [](InferenceResponse& x) {
    if (!x.certificate) return false;
    for (auto& [p, path] : x.certificate->result_paths)
      if (!path.siblings.empty()) {
        path.siblings[0].sibling.data[5] ^= 1;
        return true;
      }
    return false;
  });
  add("side", [](InferenceResponse& x) {
    if (!x.certificate) return false;
    for (auto& [p, atts] : x.certificate->attestations)
      for (auto& a : atts)
        if (!a.path.siblings.empty()) {
          auto& s = a.path.siblings.back().side;
          s = s == merkle::Side::left ? merkle::Side::right : merkle::Side::left;
          return true;
        }
    return false;
  });
  add("kind", [](InferenceResponse& x) {
    if (!x.certificate) return false;
    for (auto& [p, atts] : x.certificate->attestations)
      if (!atts.empty()) {
        atts[0].kind = atts[0].kind == AttestLeafRef::Kind::whole_batch
                           ? AttestLeafRef::Kind::single
                           : AttestLeafRef::Kind::whole_batch;
        return true;
      }
    return false;
  });
  add("commit_sig", [](InferenceResponse& x) {
    if (x.certificate) {
      for (auto& [node, s] : x.certificate->sigs)
        if (s.commit_sig) {
          (*s.commit_sig)[7] ^= 0x40;
          return true;
        }
      return false;
    }
    if (x.failure && !x.failure->attests.empty()) {
      x.failure->attests[0].commit_sig[3] ^= 1;
      return true;
    }
    return false;
  });
  add("dup_attestor", [](InferenceResponse& x) {
    if (!x.certificate) return false;
    for (auto& [p, atts] : x.certificate->attestations)
      if (atts.size() >= 2) {
        atts[1].attestor = atts[0].attestor;
        return true;
      }
    return false;
  });
  add("drop_result", [](InferenceResponse& x) {
    if (x.results.size() < 2) return false;
    x.results.pop_back();
    return true;
  });
  add("reason", [](InferenceResponse& x) {
    if (!x.failure) return false;
    x.failure->record.reason += "!";
    return true;
  });
  add("primary_root", [](InferenceResponse& x) {
    if (x.certificate) x.certificate->primary_r_root.data[0] ^= 1;
    else if (x.failure) x.failure->primary_r_root.data[0] ^= 1;
    else return false;
    return true;
  });
  return out;
}

int main() {
  gpu::Context ctx(0);
  auto spec_of = [](uint64_t in, uint64_t outd, uint64_t nreq) {  // test_harness.cpp:19-28
    ScenarioSpec spec;
    spec.workload.n_requests = nreq;
    spec.workload.input_dim = in;
    spec.workload.output_dim = outd;
    spec.workload.models_per_group = 4;
    spec.workload.arrival_gap_us = 3'000;
    spec.duration_us = 120'000'000;
    return spec;
  };
  struct Case {
    const char* name;
    ScenarioSpec spec;
    bool timed;
  };
  std::vector<Case> cases;
  cases.push_back({"honest", spec_of(4, 3, 8), false});
  {
    ScenarioSpec s = spec_of(4, 3, 8);
    s.strategy = Coordinator::Strategy::agree_then_execute;
    cases.push_back({"agree_then_execute", s, false});
  }
  {
    ScenarioSpec s = spec_of(4, 3, 8);
    s.faults[2].behavior = FaultSpec::Behavior::corrupt_result;
    s.faults[2].magnitude = 1.0;
    cases.push_back({"corrupt_beyond_eps", s, false});
  }
  {
    ScenarioSpec s = spec_of(4, 3, 8);
    s.faults[2].behavior = FaultSpec::Behavior::corrupt_result;
    s.faults[2].magnitude = 1e-4;
    cases.push_back({"corrupt_within_eps", s, false});
  }
  cases.push_back({"c1_shape", spec_of(3072, 10, 12), false});
  cases.push_back({"imagenet_shape", spec_of(3 * 224 * 224, 10, 32), true});

  int failures = 0;
  for (auto& c : cases) {
    const ScenarioResult r = run_scenario(c.spec);
    // ---- assembly: every op of every slot of every node
    uint64_t slots = 0, ops = 0, succ = 0, fail = 0, none = 0, mism = 0;
    double t_ref_asm = 0, t_gpu_asm = 0;
    std::vector<const OrderedSlot*> all;
    for (const auto& node_slots : r.ordered)
      for (const OrderedSlot& slot : node_slots) all.push_back(&slot);
    slots = all.size();
    auto t0 = Clock::now();
    std::vector<std::vector<std::optional<InferenceResponse>>> ref(all.size());
    for (size_t s = 0; s < all.size(); s++)
      for (size_t k = 0; k < all[s]->ops.size(); k++)
        ref[s].push_back(assemble_response(*all[s], k, r.config));
    t_ref_asm = secs(t0);
    t0 = Clock::now();
    auto got = gpu::assemble_responses(ctx, all, r.config);  // every slot in one pass
    t_gpu_asm = secs(t0);
    {  // and slot by slot, as a proxy does when each slot is ordered
      for (size_t s = 0; s < all.size(); s++)
        if (gpu::assemble_responses(ctx, *all[s], r.config) != ref[s]) mism++;
    }
    for (size_t s = 0; s < all.size(); s++)
      for (size_t k = 0; k < all[s]->ops.size(); k++) {
        ops++;
        if (!ref[s][k]) none++;
        else if (ref[s][k]->kind == InferenceResponse::Kind::success) succ++;
        else fail++;
        if (got[s][k] != ref[s][k]) mism++;
      }
    // ---- verification: certified responses and their forgeries
    std::vector<InferenceRequest> reqs;
    std::vector<InferenceResponse> resps;
    std::vector<std::string> what;
    for (const RequestRecord& rec : r.requests) {
      if (!rec.response) continue;
      reqs.push_back(rec.request);
      resps.push_back(*rec.response);
      what.push_back("genuine");
      for (auto& [name, forged] : forgeries(*rec.response)) {
        reqs.push_back(rec.request);
        resps.push_back(std::move(forged));
        what.push_back(name);
      }
      InferenceRequest other = rec.request;  // the client's request altered
      if (!other.input.empty()) {
        other.input.back() = -other.input.back() + 0.5;
        reqs.push_back(other);
        resps.push_back(*rec.response);
        what.push_back("request");
      }
    }
    t0 = Clock::now();
    std::vector<bool> ref_ok(reqs.size());
    for (size_t i = 0; i < reqs.size(); i++) ref_ok[i] = verify_response(reqs[i], resps[i], r.config);
    const double t_ref_ver = secs(t0);
    t0 = Clock::now();
    std::vector<bool> got_ok = gpu::verify_responses(ctx, reqs, resps, r.config);
    const double t_gpu_ver = secs(t0);
    uint64_t vmism = 0, accepted = 0, genuine = 0, genuine_ok = 0;
    for (size_t i = 0; i < reqs.size(); i++) {
      if (ref_ok[i] != got_ok[i]) {
        vmism++;
        std::printf("  verify mismatch: %s ref %d gpu %d\n", what[i].c_str(), (int)ref_ok[i],
                    (int)got_ok[i]);
      }
      // dropping one of N results still leaves >= N - f valid ones: not a
      // forgery; every other variant must be rejected
      // (nor is an altered request input under a failure certificate:
      // verify_failure binds only the request id and group, certificate.cpp:290-316)
      const bool forgery = what[i] != "drop_result" &&
                           !(what[i] == "request" && resps[i].kind == InferenceResponse::Kind::failure);
      if (forgery || what[i] == "genuine") accepted += ref_ok[i];
      if (what[i] == "genuine") {
        genuine++;
        genuine_ok += ref_ok[i];
      }
    }
    const bool ok = mism == 0 && vmism == 0 && ops > 0 && genuine > 0 && genuine_ok == genuine &&
                    accepted == genuine_ok;
    std::printf("%-20s slots %3lu ops %4lu (success %lu, failure %lu, none %lu) assembly "
                "mismatches %lu | responses %lu (%lu genuine) accepted %lu (genuine + forgeries) verify "
                "mismatches %lu  %s\n",
                c.name, (unsigned long)slots, (unsigned long)ops, (unsigned long)succ,
                (unsigned long)fail, (unsigned long)none, (unsigned long)mism,
                (unsigned long)reqs.size(), (unsigned long)genuine, (unsigned long)accepted,
                (unsigned long)vmism, ok ? "ok" : "FAIL");
    if (c.timed)
      std::printf("timing %s: assemble %lu ops: reference %.3f s, gpu %.3f s | verify %lu "
                  "responses: reference %.3f s, gpu %.3f s\n",
                  c.name, (unsigned long)ops, t_ref_asm, t_gpu_asm, (unsigned long)reqs.size(),
                  t_ref_ver, t_gpu_ver);
    if (!ok) failures++;
  }
  std::printf("integration_verify: %zu scenarios, %d failures\n", cases.size(), failures);
  return failures == 0 ? 0 : 1;
}
