// TEST INFRASTRUCTURE — drop-in demonstration for the headline (CNN group)
// path. Links the UNMODIFIED reference (oracle/_ref/libcredo_ref.so) and the
// product library; uses only reference types and functions on the host side:
//
//   ModelGroup / ModelDescriptor (params["arch"]) + filesystem_fetcher  ->
//   GroupServer::load_group on EVERY listed GPU (one cg_ctx per device, in
//   one process), InferenceRequest objects from make_signed_request, checked
//   by verify_request, submitted through the batch former, dispatched.
//
// Checks: the certificates of all GPUs are bit-identical, and the reference's
// own functions recompute every decision and root from the GPU's outputs
// (distance::select_quorum, build_result_tree, the try_attest manifest and A
// tree via ref_certify_batch_ex).
//
//   integration_cnn <model_dir> <n_models> <batch> <device>...
// model_dir holds m<p>.bin (CNN model files) and m<p>.arch.
#include <cstdio>
#include <fstream>
#include <memory>
#include <random>
#include <string>

#include "credo/crypto.hpp"
#include "credo/domain.hpp"
#include "credo/engine.hpp"
#include "credo_gpu_adapters.hpp"

extern "C" {  // oracle/ref_capi.cpp (the reference's functions behind a C shim)
void* ref_batch_new(const uint8_t* enc, const uint64_t* lens, uint64_t B, uint64_t version);
void ref_batch_free(void* h);
int ref_certify_batch_ex(void* h, uint64_t N, uint64_t f, uint32_t metric, double eps_default,
                         const double* outputs, uint64_t v, uint64_t version,
                         const uint8_t* model_digests, uint64_t view, uint64_t seq, int threads,
                         uint64_t* sel_mask, double* diam, uint8_t* satisfied, int64_t* label,
                         uint8_t* r_roots, uint8_t* a_root, uint64_t* manifest_len,
                         const uint8_t* missing);
}

using namespace credo;

int main(int argc, char** argv) {
  if (argc < 5) {
    std::fprintf(stderr, "usage: %s model_dir n_models batch device...\n", argv[0]);
    return 2;
  }
  const std::string dir = argv[1];
  const uint64_t N = std::stoull(argv[2]), B = std::stoull(argv[3]);
  std::vector<int> devices;
  for (int i = 4; i < argc; i++) devices.push_back(std::atoi(argv[i]));
  const uint64_t f = (N - 1) / 2, u = 3 * 224 * 224, v = 1000;

  ModelFetcher fetch = filesystem_fetcher();
  ModelGroup group;
  group.group_id = "group-0";
  group.version = 1;
  group.status = GroupStatus::active;
  group.distance.metric = distance::Metric::euclidean;
  group.distance.default_epsilon = 0.1;
  std::vector<uint8_t> digests;
  for (uint64_t p = 0; p < N; p++) {
    ModelDescriptor d;
    d.model_url = dir + "/m" + std::to_string(p) + ".bin";
    std::ifstream a(dir + "/m" + std::to_string(p) + ".arch");
    std::getline(a, d.params["arch"]);
    d.input_dim = u;
    d.output_dim = v;
    auto file = fetch(d.model_url);
    if (!file) return 2;
    d.weights_digest = hash(*file);  // the reference's crypto::hash
    digests.insert(digests.end(), d.weights_digest.data.begin(), d.weights_digest.data.end());
    group.models.push_back(d);
  }

  KeyPair client = KeyPair::from_seed(std::array<uint8_t, 32>{9});
  std::mt19937_64 rng(5);
  std::uniform_real_distribution<double> uni(-1.0, 1.0);
  std::vector<InferenceRequest> reqs;
  std::vector<uint8_t> encs;
  std::vector<uint64_t> lens;
  for (uint64_t i = 0; i < B; i++) {
    std::vector<double> x(u);
    for (double& t : x) t = uni(rng);
    Encoder ne;
    ne.u64(i);
    reqs.push_back(make_signed_request(client, ne.take(), "group-0", std::move(x),
                                       i == 3 ? std::optional<double>(0.0) : std::nullopt));
    if (!verify_request(reqs.back())) {
      std::fprintf(stderr, "verify_request failed\n");
      return 2;
    }
    Encoder e;
    reqs.back().encode(e);
    Bytes b = e.take();
    lens.push_back(b.size());
    encs.insert(encs.end(), b.begin(), b.end());
  }

  int mismatches = 0, checks = 0;
  std::vector<gpu::GroupServer::Certified> certs;
  for (int dev : devices) {
    gpu::Context ctx(dev);
    gpu::GroupServer srv(ctx, B, 2000, 4);
    if (auto err = srv.load_group(group, fetch, f)) {
      std::fprintf(stderr, "load_group on device %d: %s\n", dev, err->c_str());
      return 2;
    }
    for (auto& e : srv.submit_many(reqs.data(), reqs.size(), 0))
      if (e) {
        std::fprintf(stderr, "submit: %s\n", e->c_str());
        return 2;
      }
    auto got = srv.dispatch(/*keep_outputs=*/true);
    if (got.size() != 1 || got[0].satisfied.size() != B) {
      std::fprintf(stderr, "expected one batch of %lu\n", (unsigned long)B);
      return 2;
    }
    certs.push_back(std::move(got[0]));
    std::printf("device %d: certified %lu requests, a_root %s\n", dev, (unsigned long)B,
                to_hex(ByteView(certs.back().a_root.data.data(), 8)).c_str());
  }
  // every GPU gives the same certificate
  for (size_t i = 1; i < certs.size(); i++) {
    checks++;
    if (certs[i].a_root != certs[0].a_root || certs[i].r_roots != certs[0].r_roots ||
        certs[i].outputs != certs[0].outputs || certs[i].satisfied != certs[0].satisfied)
      mismatches++;
  }
  // the reference recomputes decisions and roots from the GPU's outputs
  const auto& c = certs[0];
  void* h = ref_batch_new(encs.data(), lens.data(), B, 1);
  std::vector<uint64_t> sel(B);
  std::vector<double> diam(B);
  std::vector<uint8_t> sat(B), rr(32 * N), ar(32);
  std::vector<int64_t> lab(B);
  uint64_t mlen = 0;
  if (ref_certify_batch_ex(h, N, f, 0, 0.1, c.outputs.data(), v, 1, digests.data(), 0, 1, 4,
                           sel.data(), diam.data(), sat.data(), lab.data(), rr.data(), ar.data(),
                           &mlen, nullptr) != 0)
    return 2;
  ref_batch_free(h);
  for (uint64_t k = 0; k < B; k++) {
    checks++;
    if (sel[k] != c.selected[k] || diam[k] != c.diameter[k] || sat[k] != c.satisfied[k] ||
        lab[k] != c.label[k])
      mismatches++;
  }
  for (uint64_t p = 0; p < N; p++) {
    checks++;
    if (std::memcmp(rr.data() + 32 * p, c.r_roots[p].data.data(), 32) != 0) mismatches++;
  }
  checks += 2;
  if (std::memcmp(ar.data(), c.a_root.data.data(), 32) != 0) mismatches++;
  if (mlen != c.manifest_len) mismatches++;
  uint64_t nsat = 0;
  for (auto s : c.satisfied) nsat += s;
  std::printf("integration_cnn: %zu device(s), %lu/%lu satisfied, %d checks, %d mismatches\n",
              devices.size(), (unsigned long)nsat, (unsigned long)B, checks, mismatches);
  return mismatches == 0 ? 0 : 1;
}
