// The batch former in front of the GPU groups: InferenceEngine::submit /
// make_batch / flush_due / flush_version / flush_all / next_flush_deadline
// (proj/src/engine.cpp:166-267) with the reference's semantics -- per live
// (group, version) a FIFO queue with `seen` dedup, a batch released when the
// queue reaches exec_batch_max or when its oldest request has waited
// flush_interval_us, one batch per live version for every submission --
// packing each request, as it is submitted, straight into the pinned
// struct-of-arrays staging of its version's forming batch. A released batch
// is ingested into its group's ring (cg_ingest_batch: framing bytes, H2D,
// request-midstate chains start) and reported as a ready ticket in release
// order; the caller dispatches the tickets (cg_certify_ticket), which is
// where the reference's dispatch_batches hands batches to execute_batch.
//
// verify_request (domain.cpp:204-216): the structural checks (non-empty
// nonce and input, finite non-negative epsilon override, request id ==
// canonical id) run here; the Ed25519 signature check is the caller's (an
// optional host callback), it needs the caller's signature library.
#include <chrono>
#include <condition_variable>
#include <cstdio>
#include <cstdlib>
#include <functional>
#include <map>
#include <set>
#include <thread>

#include "host_sha256.h"
#include "runtime.cuh"

namespace {

using Id = std::array<uint8_t, 32>;

// Persistent pack workers: large submissions copy their inputs into pinned
// staging on several threads (~10 GB/s per thread; a 128 x 1.2 MB burst is
// 154 MB).
class PackPool {
 public:
  explicit PackPool(int n) {
    for (int i = 0; i < n; i++) th_.emplace_back([this] { loop(); });
  }
  ~PackPool() {
    {
      std::lock_guard<std::mutex> lk(mu_);
      stop_ = true;
    }
    cv_.notify_all();
    for (auto& t : th_) t.join();
  }
  int size() const { return (int)th_.size(); }
  // runs fn(i) for i in [0, n) on the workers and the calling thread
  void run(size_t n, const std::function<void(size_t)>& fn) {
    if (th_.empty() || n < 2) {
      for (size_t i = 0; i < n; i++) fn(i);
      return;
    }
    std::unique_lock<std::mutex> lk(mu_);
    fn_ = &fn;
    n_ = n;
    next_ = 0;
    active_ = (int)th_.size();
    gen_++;
    lk.unlock();
    cv_.notify_all();
    for (size_t i; (i = next_.fetch_add(1)) < n;) fn(i);
    lk.lock();
    done_cv_.wait(lk, [&] { return active_ == 0; });
    fn_ = nullptr;
  }

 private:
  void loop() {
    uint64_t seen = 0;
    std::unique_lock<std::mutex> lk(mu_);
    for (;;) {
      cv_.wait(lk, [&] { return stop_ || gen_ != seen; });
      if (stop_) return;
      seen = gen_;
      const std::function<void(size_t)>* fn = fn_;
      const size_t n = n_;
      lk.unlock();
      for (size_t i; (i = next_.fetch_add(1)) < n;) (*fn)(i);
      lk.lock();
      if (--active_ == 0) done_cv_.notify_all();
    }
  }
  std::vector<std::thread> th_;
  std::mutex mu_;
  std::condition_variable cv_, done_cv_;
  const std::function<void(size_t)>* fn_ = nullptr;
  size_t n_ = 0;
  std::atomic<size_t> next_{0};
  int active_ = 0;
  uint64_t gen_ = 0;
  bool stop_ = false;
};

// One forming ExecutionBatch in pinned struct-of-arrays form.
struct Forming {
  uint32_t n = 0;
  std::vector<uint64_t> enq_us;
  PinBuf<uint8_t> ids, pubs, sigs, has_eps, nonces;
  PinBuf<double> inputs, eps;
  PinBuf<uint64_t> nonce_lens, dims;
  std::vector<std::vector<double>> misfit;  // inputs of wrong-dimension requests
  std::vector<const double*> misfit_ptr;
  bool any_misfit = false;
  uint64_t nonce_bytes = 0;
  cudaEvent_t ev = nullptr;  // the ingest's copies out of this staging finished
  ~Forming() {
    if (ev) cudaEventDestroy(ev);
  }
};

struct Version {
  cg_group* g = nullptr;
  int status = CG_GROUP_ACTIVE;
  std::set<Id> seen;
  std::unique_ptr<Forming> cur;
  std::vector<std::unique_ptr<Forming>> pool;      // staging whose ingest was issued
  std::vector<std::unique_ptr<Forming>> released;  // formed, waiting for ring space
};

}  // namespace

struct cg_engine {
  cg_ctx* ctx = nullptr;
  uint64_t max = 0, flush_us = 0;
  std::map<std::string, std::map<uint64_t, Version>> groups;
  std::vector<cg_ready_batch> ready;
  std::unique_ptr<PackPool> pack;
  cg_sig_verify_fn verify = nullptr;
  void* verify_user = nullptr;
  // CREDO_ENGINE_PROFILE=1: host seconds per submit phase, printed at free
  bool prof = std::getenv("CREDO_ENGINE_PROFILE") != nullptr;
  double t_stage = 0, t_pack = 0, t_ingest = 0;
  uint64_t n_submits = 0;
};

namespace {

std::unique_ptr<Forming> take_staging(cg_engine* e, Version& V) {
  for (size_t i = 0; i < V.pool.size(); i++) {
    if (cudaEventQuery(V.pool[i]->ev) == cudaSuccess) {
      auto f = std::move(V.pool[i]);
      V.pool.erase(V.pool.begin() + i);
      return f;
    }
  }
  if (V.pool.size() >= 4) {  // bound the pinned memory: wait for the oldest
    CG_CUDA(cudaEventSynchronize(V.pool.front()->ev));
    auto f = std::move(V.pool.front());
    V.pool.erase(V.pool.begin());
    return f;
  }
  auto f = std::make_unique<Forming>();
  const uint64_t B = e->max, u = V.g->u;
  f->ids.ensure(32 * B);
  f->pubs.ensure(32 * B);
  f->sigs.ensure(64 * B);
  f->has_eps.ensure(B);
  f->eps.ensure(B);
  f->nonce_lens.ensure(B);
  f->dims.ensure(B);
  f->inputs.ensure(B * u);
  f->nonces.ensure(64 * B);
  CG_CUDA(cudaEventCreateWithFlags(&f->ev, cudaEventDisableTiming));
  return f;
}

// Ingest released batches in release order while their group's ring has
// room; each becomes a ready ticket.
void drain_released(cg_engine* e) {
  for (auto& [gid, versions] : e->groups)
    for (auto& [ver, V] : versions)
      while (!V.released.empty()) {
        cg_group* g = V.g;
        IngestSlot& S = *g->slots[g->next_ticket % g->slots.size()];
        if (S.used) break;  // ring full: certify outstanding tickets first
        std::unique_ptr<Forming> f = std::move(V.released.front());
        V.released.erase(V.released.begin());
        cg_request_batch b{};
        b.B = f->n;
        b.u = g->u;
        b.request_ids = f->ids.p;
        b.inputs = f->inputs.p;
        b.inputs_on_device = 0;
        b.has_eps = f->has_eps.p;
        b.eps = f->eps.p;
        b.client_pubs = f->pubs.p;
        b.nonces = f->nonces.p;
        b.nonce_lens = f->nonce_lens.p;
        b.client_sigs = f->sigs.p;
        if (f->any_misfit) {
          b.input_dims = f->dims.p;
          b.misfit_inputs = f->misfit_ptr.data();
        }
        // f->ev fires when the H2D copies out of this staging are done (not
        // after the 35 ms request-midstate chains queued behind them)
        const uint64_t t = ingest(g, &b, f->ev);
        e->ready.push_back(cg_ready_batch{g, ver, t, f->n});
        f->n = 0;
        f->nonce_bytes = 0;
        f->enq_us.clear();
        f->any_misfit = false;
        f->misfit.clear();
        f->misfit_ptr.clear();
        V.pool.push_back(std::move(f));
      }
}

// make_batch (engine.cpp:166-180): the forming batch is released whole (it
// never holds more than exec_batch_max requests).
void release(cg_engine* e, Version& V) {
  if (!V.cur || V.cur->n == 0) return;
  V.released.push_back(std::move(V.cur));
}

int check_request(const cg_request& r) {
  if (r.nonce_len == 0) return CG_SUBMIT_INVALID;
  if (r.input_dim == 0) return CG_SUBMIT_INVALID;
  if (r.has_eps && !(r.eps >= 0.0 && std::isfinite(r.eps))) return CG_SUBMIT_INVALID;
  HostSha256 h;  // canonical_request_id = H(client_pub || 0x1F || nonce)
  h.update(r.client_pub, 32);
  h.u8(0x1F);
  h.update(r.nonce, r.nonce_len);
  uint8_t id[32];
  h.final(id);
  if (std::memcmp(id, r.request_id, 32) != 0) return CG_SUBMIT_INVALID;
  return CG_SUBMIT_OK;
}

}  // namespace

extern "C" {

int cg_engine_create(cg_ctx* ctx, uint64_t exec_batch_max, uint64_t flush_interval_us,
                     int pack_threads, cg_engine** out) {
  if (!out) return CG_EINVAL;
  *out = nullptr;
  return guarded(ctx, [&] {
    if (exec_batch_max < 1) throw InvalidArgument("engine: batch max < 1");
    auto e = std::make_unique<cg_engine>();
    e->ctx = ctx;
    e->max = exec_batch_max;
    e->flush_us = flush_interval_us;
    e->pack = std::make_unique<PackPool>(std::max(0, pack_threads - 1));
    *out = e.release();
    return CG_OK;
  });
}

void cg_engine_free(cg_engine* e) {
  if (!e) return;
  if (e->prof && e->n_submits)
    std::fprintf(stderr, "cg_engine: %lu submits, ms per submit: stage %.3f pack %.3f ingest %.3f\n",
                 (unsigned long)e->n_submits, 1e3 * e->t_stage / e->n_submits,
                 1e3 * e->t_pack / e->n_submits, 1e3 * e->t_ingest / e->n_submits);
  cudaSetDevice(e->ctx->device);
  for (auto& [gid, versions] : e->groups)
    for (auto& [ver, V] : versions)
      for (auto& f : V.pool) cudaEventSynchronize(f->ev);
  delete e;
}

int cg_engine_set_verifier(cg_engine* e, cg_sig_verify_fn fn, void* user) {
  if (!e) return CG_EINVAL;
  e->verify = fn;
  e->verify_user = user;
  return CG_OK;
}

// load_group (engine.cpp:67-97) for a version whose replica set is already
// resident as a cg_group.
int cg_engine_load_group(cg_engine* e, cg_group* g, int status) {
  if (!e || !g) return CG_EINVAL;
  return guarded(e->ctx, [&] {
    if (g->ctx != e->ctx) throw InvalidArgument("group from another context");
    if (e->max > g->maxB) throw InvalidArgument("exec_batch_max exceeds the group's max_batch");
    auto& versions = e->groups[g->gid];
    if (versions.count(g->version)) throw InvalidArgument("version already loaded");
    Version& V = versions[g->version];
    V.g = g;
    V.status = status;
    return CG_OK;
  });
}

// set_status (engine.cpp:99-113): retiring drops the queue.
int cg_engine_set_status(cg_engine* e, const char* group_id, uint64_t group_id_len,
                         uint64_t version, int status) {
  if (!e) return CG_EINVAL;
  return guarded(e->ctx, [&] {
    auto git = e->groups.find(std::string(group_id, group_id_len));
    if (git == e->groups.end()) return CG_OK;
    auto vit = git->second.find(version);
    if (vit == git->second.end()) return CG_OK;
    vit->second.status = status;
    if (status == CG_GROUP_RETIRED && vit->second.cur) {
      vit->second.cur->n = 0;
      vit->second.cur->nonce_bytes = 0;
      vit->second.cur->enq_us.clear();
    }
    return CG_OK;
  });
}

// submit (engine.cpp:182-209) for n requests in order; errors[i] =
// CG_SUBMIT_*. Inputs are packed into pinned staging on the pack threads.
int cg_engine_submit(cg_engine* e, const cg_request* reqs, uint32_t n, uint64_t now_us,
                     int* errors) {
  if (!e || (n && !reqs)) return CG_EINVAL;
  return guarded(e->ctx, [&] {
    using clk = std::chrono::steady_clock;
    const auto t0 = clk::now();
    struct Copy {
      const double* src;
      double* dst;
      uint64_t count;
    };
    std::vector<Copy> copies;
    for (uint32_t i = 0; i < n; i++) {
      const cg_request& r = reqs[i];
      int err = check_request(r);
      if (err == CG_SUBMIT_OK && e->verify) {
        // signing digest H(0x01 || body) on the host, Ed25519 by the caller
        HostSha256 h;
        h.u8(0x01);
        h.update(r.request_id, 32);
        h.bytes(reinterpret_cast<const uint8_t*>(r.group_id), r.group_id_len);
        h.u32((uint32_t)r.input_dim);
        h.f64be(r.input, r.input_dim);
        h.u8(r.has_eps ? 1 : 0);
        if (r.has_eps) {
          uint64_t bits;
          std::memcpy(&bits, &r.eps, 8);
          h.u64(bits);
        }
        h.update(r.client_pub, 32);
        h.bytes(r.nonce, r.nonce_len);
        uint8_t dig[32];
        h.final(dig);
        if (!e->verify(e->verify_user, r.client_pub, dig, r.client_sig)) err = CG_SUBMIT_INVALID;
      }
      if (err == CG_SUBMIT_OK) {
        auto git = e->groups.find(std::string(r.group_id, r.group_id_len));
        if (git == e->groups.end()) {
          err = CG_SUBMIT_UNKNOWN_GROUP;
        } else {
          bool any_live = false;
          Id id;
          std::memcpy(id.data(), r.request_id, 32);
          for (auto& [ver, V] : git->second) {
            if (V.status == CG_GROUP_RETIRED) continue;
            any_live = true;
            if (!V.seen.insert(id).second) continue;  // duplicate, absorbed
            if (!V.cur) V.cur = take_staging(e, V);
            Forming& f = *V.cur;
            const uint32_t k = f.n++;
            f.enq_us.push_back(now_us);
            std::memcpy(f.ids.p + 32 * k, r.request_id, 32);
            std::memcpy(f.pubs.p + 32 * k, r.client_pub, 32);
            std::memcpy(f.sigs.p + 64 * k, r.client_sig, 64);
            f.has_eps.p[k] = r.has_eps ? 1 : 0;
            f.eps.p[k] = r.has_eps ? r.eps : 0.0;
            f.nonce_lens.p[k] = r.nonce_len;
            if (f.nonce_bytes + r.nonce_len > f.nonces.n) {  // grow, keep contents
              PinBuf<uint8_t> bigger;
              bigger.ensure(2 * (f.nonce_bytes + r.nonce_len));
              std::memcpy(bigger.p, f.nonces.p, f.nonce_bytes);
              std::swap(bigger.p, f.nonces.p);
              std::swap(bigger.n, f.nonces.n);
            }
            std::memcpy(f.nonces.p + f.nonce_bytes, r.nonce, r.nonce_len);
            f.nonce_bytes += r.nonce_len;
            f.dims.p[k] = r.input_dim;
            f.misfit.emplace_back();
            if (r.input_dim == V.g->u) {
              copies.push_back(Copy{r.input, f.inputs.p + V.g->u * k, r.input_dim});
            } else {  // misfit: execute_batch will skip it (engine.cpp:286-291)
              f.misfit.back().assign(r.input, r.input + r.input_dim);
              std::memset(f.inputs.p + V.g->u * k, 0, 8 * V.g->u);
              f.any_misfit = true;
            }
            if (f.n >= e->max) release(e, V);
          }
          if (!any_live) err = CG_SUBMIT_RETIRED;
        }
      }
      if (errors) errors[i] = err;
    }
    // the packing copies (1.2 MB per ImageNet request) on the pack threads,
    // before any of these batches is ingested
    const auto t1 = clk::now();
    e->pack->run(copies.size(), [&](size_t i) {
      std::memcpy(copies[i].dst, copies[i].src, 8 * copies[i].count);
    });
    const auto t2 = clk::now();
    for (auto& [gid, versions] : e->groups)
      for (auto& [ver, V] : versions)
        for (auto& f : V.released)
          if (f->any_misfit && f->misfit_ptr.size() != f->n) {
            f->misfit_ptr.resize(f->n);
            for (uint32_t k = 0; k < f->n; k++) f->misfit_ptr[k] = f->misfit[k].data();
          }
    drain_released(e);
    if (e->prof) {
      const auto t3 = clk::now();
      e->t_stage += std::chrono::duration<double>(t1 - t0).count();
      e->t_pack += std::chrono::duration<double>(t2 - t1).count();
      e->t_ingest += std::chrono::duration<double>(t3 - t2).count();
      e->n_submits++;
    }
    return CG_OK;
  });
}

}  // extern "C"

namespace {
template <typename Pred>
int flush_where(cg_engine* e, Pred&& due) {
  return guarded(e->ctx, [&] {
    for (auto& [gid, versions] : e->groups)
      for (auto& [ver, V] : versions)
        if (V.cur && V.cur->n && due(gid, ver, V)) {
          Forming& f = *V.cur;
          if (f.any_misfit) {
            f.misfit_ptr.resize(f.n);
            for (uint32_t k = 0; k < f.n; k++) f.misfit_ptr[k] = f.misfit[k].data();
          }
          release(e, V);
        }
    drain_released(e);
    return CG_OK;
  });
}
}  // namespace

extern "C" {

// flush_due (engine.cpp:211-225): versions whose oldest queued request has
// waited flush_interval_us.
int cg_engine_flush_due(cg_engine* e, uint64_t now_us) {
  if (!e) return CG_EINVAL;
  return flush_where(e, [&](const std::string&, uint64_t, const Version& V) {
    return V.cur->enq_us.front() + e->flush_us <= now_us;
  });
}

// flush_version (engine.cpp:227-241).
int cg_engine_flush_version(cg_engine* e, const char* group_id, uint64_t group_id_len,
                            uint64_t version) {
  if (!e) return CG_EINVAL;
  const std::string want(group_id, group_id_len);
  return flush_where(e, [&](const std::string& gid, uint64_t ver, const Version&) {
    return gid == want && ver == version;
  });
}

// flush_all (engine.cpp:243-254).
int cg_engine_flush_all(cg_engine* e) {
  if (!e) return CG_EINVAL;
  return flush_where(e, [](const std::string&, uint64_t, const Version&) { return true; });
}

// next_flush_deadline (engine.cpp:256-267): *has = 0 when every queue is empty.
int cg_engine_next_flush_deadline(cg_engine* e, uint64_t* deadline, int* has) {
  if (!e || !deadline || !has) return CG_EINVAL;
  *has = 0;
  for (auto& [gid, versions] : e->groups)
    for (auto& [ver, V] : versions) {
      if (!V.cur || V.cur->n == 0) continue;
      const uint64_t due = V.cur->enq_us.front() + e->flush_us;
      if (!*has || due < *deadline) *deadline = due;
      *has = 1;
    }
  return CG_OK;
}

// Batches released so far (ingested, in release order), up to cap; *n_out
// = how many were written; the rest stay queued for the next call. Released
// batches whose group ring was full are ingested here first.
int cg_engine_ready(cg_engine* e, cg_ready_batch* out, uint32_t cap, uint32_t* n_out) {
  if (!e || !n_out) return CG_EINVAL;
  return guarded(e->ctx, [&] {
    drain_released(e);
    const uint32_t n = std::min<uint32_t>(cap, (uint32_t)e->ready.size());
    for (uint32_t i = 0; i < n; i++) out[i] = e->ready[i];
    e->ready.erase(e->ready.begin(), e->ready.begin() + n);
    *n_out = n;
    return CG_OK;
  });
}

// Requests queued in forming batches (not yet released) + released batches
// waiting for ring space.
int cg_engine_pending(cg_engine* e, uint64_t* queued, uint64_t* waiting_batches) {
  if (!e) return CG_EINVAL;
  uint64_t q = 0, w = 0;
  for (auto& [gid, versions] : e->groups)
    for (auto& [ver, V] : versions) {
      if (V.cur) q += V.cur->n;
      w += V.released.size();
    }
  if (queued) *queued = q;
  if (waiting_batches) *waiting_batches = w;
  return CG_OK;
}

}  // extern "C"
