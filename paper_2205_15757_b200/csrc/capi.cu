// The C-ABI (include/credo_gpu.h) and the host-side runtime behind it:
// contexts, device buffers, model residency, the batch former's canonical
// framing bytes, and the per-batch certification pipeline.
//
// Pipeline for one ExecutionBatch (reference: InferenceEngine::execute_batch
// proj/src/engine.cpp:269-306 -> Coordinator::try_prepare's R tree
// proj/src/coordinator.cpp:588-624 -> try_attest proj/src/coordinator.cpp:
// 727-849), all on the device:
//   side stream : request midstates  SHA(0x00||0x52||request)[whole blocks]
//   main stream : N replica forwards -> softmax/top-k -> (join) ->
//                 result-leaf tails -> select_quorum + label -> R roots ->
//                 manifest (+whole/failure A leaves) -> single A leaves ->
//                 A root
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <array>
#include <atomic>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <vector>

#include "../../include/credo_gpu.h"
#include "agree.cuh"
#include "cnn.cuh"
#include "common.cuh"
#include "digest.cuh"
#include "gemm_sm100.cuh"
#include "host_sha256.h"
#include "runtime.cuh"

namespace cg {

static std::atomic<uint64_t> g_launches{0};
thread_local std::atomic<uint64_t>* tl_ctx_launches = nullptr;
uint64_t launch_counter_add(uint64_t n) {
  if (tl_ctx_launches) *tl_ctx_launches += n;
  return g_launches += n;
}

// ------------------------------------------------------------ kernel timers
struct Timers {
  std::mutex mu;
  bool on = false;
  std::vector<cudaEvent_t> pool;
  size_t used = 0;
  std::vector<std::pair<size_t, size_t>> spans[kTimeClasses];  // event indices
  std::vector<size_t> open[kTimeClasses];
  cudaEvent_t take() {
    if (used == pool.size()) {
      cudaEvent_t e;
      CG_CUDA(cudaEventCreate(&e));
      pool.push_back(e);
    }
    return pool[used++];
  }
};
static Timers g_timers;

void timer_begin(cudaStream_t st, int cls) {
  if (!g_timers.on) return;
  std::lock_guard<std::mutex> lk(g_timers.mu);
  size_t i = g_timers.used;
  CG_CUDA(cudaEventRecord(g_timers.take(), st));
  g_timers.open[cls].push_back(i);
}

void timer_end(cudaStream_t st, int cls) {
  if (!g_timers.on) return;
  std::lock_guard<std::mutex> lk(g_timers.mu);
  size_t i = g_timers.used;
  CG_CUDA(cudaEventRecord(g_timers.take(), st));
  size_t b = g_timers.open[cls].back();
  g_timers.open[cls].pop_back();
  g_timers.spans[cls].push_back({b, i});
}

}  // namespace cg

using namespace cg;


namespace {

// SHA-256 of count host messages on the device (one chain job each).
// prefix_byte >= 0 prepends that byte (merkle leaf domain 0x00).
// Enqueue only (results land in ctx->d_out); device_sha256_many waits.
void device_sha256_start(cg_ctx* ctx, const uint8_t* buf, const uint64_t* off,
                         const uint64_t* len, uint64_t count, int prefix_byte) {
  Arena ar;
  std::vector<size_t> pos(count), pre(count);
  const uint8_t pb = (uint8_t)prefix_byte;
  for (uint64_t i = 0; i < count; i++) {
    uint64_t moff = 0;
    if (prefix_byte >= 0) {
      pre[i] = ar.add(&pb, 1, 0);
      moff = 1;
    }
    pos[i] = ar.add(buf + off[i], len[i], moff);
  }
  ctx->d_bytes.ensure(ar.b.size() + 16);
  ctx->d_out.ensure(32 * count);
  ctx->d_jobs.ensure(count);
  std::vector<ChainJob> jobs(count);
  const uint64_t base = (uint64_t)ctx->d_bytes.p;
  for (uint64_t i = 0; i < count; i++) {
    ChainJob& j = jobs[i];
    std::memset(&j, 0, sizeof j);
    uint64_t moff = 0;
    if (prefix_byte >= 0) {
      j.seg[j.nseg++] = ChainSeg{base + pre[i], 0, 1, kSegRaw, 0};
      moff = 1;
    }
    if (len[i]) j.seg[j.nseg++] = ChainSeg{base + pos[i], moff, len[i], kSegRaw, 0};
    j.final_ = 1;
    j.total_len = moff + len[i];
    j.blk_begin = 0;
    j.blk_end = (j.total_len + 9 + 63) / 64;
    j.digest_out = (uint64_t)(ctx->d_out.p + 32 * i);
  }
  CG_CUDA(cudaMemcpyAsync(ctx->d_bytes.p, ar.b.data(), ar.b.size(),
                          cudaMemcpyHostToDevice, ctx->stream));
  CG_CUDA(cudaMemcpyAsync(ctx->d_jobs.p, jobs.data(), count * sizeof(ChainJob),
                          cudaMemcpyHostToDevice, ctx->stream));
  launch_chain_jobs_raw(ctx->d_jobs.p, (uint32_t)count, ctx->stream);
}

void device_sha256_finish(cg_ctx* ctx, uint64_t count, uint8_t* out_host) {
  CG_CUDA(cudaMemcpyAsync(out_host, ctx->d_out.p, 32 * count,
                          cudaMemcpyDeviceToHost, ctx->stream));
  CG_CUDA(cudaStreamSynchronize(ctx->stream));
}

void device_sha256_many(cg_ctx* ctx, const uint8_t* buf, const uint64_t* off,
                        const uint64_t* len, uint64_t count, int prefix_byte,
                        uint8_t* out_host) {
  if (count == 0) return;
  device_sha256_start(ctx, buf, off, len, count, prefix_byte);
  device_sha256_finish(ctx, count, out_host);
}

// load_group's model check (engine.cpp:79-81): SHA-256(file) must equal the
// descriptor's weights digest, checked BEFORE the file is parsed (a tampered
// and malformed file is a digest error, as in the reference). One ~100 MB
// sequential chain for an ImageNet CNN: host SHA-NI (~1.2 GB/s), where the
// reference computes it too.
void check_model_digest(const uint8_t* file, uint64_t len, const uint8_t digest[32]) {
  uint8_t got[32];
  host_sha256(file, len, got);
  if (std::memcmp(got, digest, 32) != 0)
    throw DigestError("model file does not match its weights digest");
}

}  // namespace

extern "C" {

int cg_ctx_create(int device, cg_ctx** out) {
  if (!out) return CG_EINVAL;
  *out = nullptr;
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || device < 0 || device >= ndev)
    return CG_ENOTSUP;
  cudaDeviceProp prop;
  if (cudaGetDeviceProperties(&prop, device) != cudaSuccess) return CG_ECUDA;
  if (prop.major != 10 || prop.minor != 0) return CG_ENOTSUP;  // sm_100a only
  auto* c = new cg_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaStreamCreateWithFlags(&c->side, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_a, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&c->ev_b, cudaEventDisableTiming) != cudaSuccess) {
    delete c;
    return CG_ECUDA;
  }
  *out = c;
  return CG_OK;
}

void cg_ctx_destroy(cg_ctx* ctx) {
  if (!ctx) return;
  cudaSetDevice(ctx->device);
  cudaDeviceSynchronize();
  if (ctx->comm) ncclCommDestroy(ctx->comm);
  if (ctx->own_stream && ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->side) cudaStreamDestroy(ctx->side);
  if (ctx->tail) cudaStreamDestroy(ctx->tail);
  if (ctx->ev_a) cudaEventDestroy(ctx->ev_a);
  if (ctx->ev_b) cudaEventDestroy(ctx->ev_b);
  delete ctx;
}

const char* cg_last_error(const cg_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int cg_ctx_set_stream(cg_ctx* ctx, void* stream) {
  return guarded(ctx, [&] {
    if (ctx->own_stream && ctx->stream) CG_CUDA(cudaStreamDestroy(ctx->stream));
    ctx->stream = (cudaStream_t)stream;
    ctx->own_stream = false;
    return CG_OK;
  });
}

void* cg_ctx_stream(cg_ctx* ctx) { return ctx ? (void*)ctx->stream : nullptr; }

int cg_ctx_synchronize(cg_ctx* ctx) {
  return guarded(ctx, [&] {
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
    CG_CUDA(cudaStreamSynchronize(ctx->side));
    if (ctx->tail) CG_CUDA(cudaStreamSynchronize(ctx->tail));
    return CG_OK;
  });
}

int cg_ctx_join(cg_ctx* ctx) {
  return guarded(ctx, [&] {
    if (ctx->tail) {
      CG_CUDA(cudaEventRecord(ctx->ev_a, ctx->tail));
      CG_CUDA(cudaStreamWaitEvent(ctx->stream, ctx->ev_a, 0));
    }
    join_group_slots(ctx);
    return CG_OK;
  });
}

uint64_t cg_ctx_launch_count(const cg_ctx* ctx) {
  return ctx ? ctx->launches.load() : g_launches.load();
}

int cg_nccl_unique_id(uint8_t out[128]) {
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return CG_ENCCL;
  static_assert(sizeof(id) == 128, "ncclUniqueId size");
  std::memcpy(out, &id, 128);
  return CG_OK;
}

int cg_ctx_init_nccl(cg_ctx* ctx, const uint8_t id[128], int nranks, int rank) {
  return guarded(ctx, [&] {
    if (nranks < 1 || rank < 0 || rank >= nranks) throw InvalidArgument("bad rank/nranks");
    if (ctx->comm) throw InvalidArgument("NCCL already initialised on this context");
    ncclUniqueId uid;
    std::memcpy(&uid, id, 128);
    ncclResult_t r = ncclCommInitRank(&ctx->comm, nranks, uid, rank);
    if (r != ncclSuccess) {
      ctx->comm = nullptr;
      ctx->err = std::string("ncclCommInitRank: ") + ncclGetErrorString(r);
      return CG_ENCCL;
    }
    ctx->rank = rank;
    ctx->nranks = nranks;
    return CG_OK;
  });
}

void cg_timing_enable(int on) {
  std::lock_guard<std::mutex> lk(g_timers.mu);
  g_timers.on = on != 0;
  g_timers.used = 0;
  for (auto& s : g_timers.spans) s.clear();
  for (auto& o : g_timers.open) o.clear();
}

int cg_timing_read(int cls, double* total_ms, uint64_t* launches) {
  if (cls < 0 || cls >= kTimeClasses) return CG_EINVAL;
  std::lock_guard<std::mutex> lk(g_timers.mu);
  double t = 0;
  for (auto& sp : g_timers.spans[cls]) {
    if (cudaEventSynchronize(g_timers.pool[sp.second]) != cudaSuccess) return CG_ECUDA;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, g_timers.pool[sp.first], g_timers.pool[sp.second]) !=
        cudaSuccess)
      return CG_ECUDA;
    t += ms;
  }
  if (total_ms) *total_ms = t;
  if (launches) *launches = g_timers.spans[cls].size();
  return CG_OK;
}

int cg_timing_spans(int cls, double* ms_out, uint64_t cap, uint64_t* count) {
  if (cls < 0 || cls >= kTimeClasses) return CG_EINVAL;
  std::lock_guard<std::mutex> lk(g_timers.mu);
  const auto& sp = g_timers.spans[cls];
  for (size_t i = 0; i < sp.size() && i < cap; i++) {
    if (cudaEventSynchronize(g_timers.pool[sp[i].second]) != cudaSuccess) return CG_ECUDA;
    float ms = 0;
    if (cudaEventElapsedTime(&ms, g_timers.pool[sp[i].first], g_timers.pool[sp[i].second]) !=
        cudaSuccess)
      return CG_ECUDA;
    ms_out[i] = ms;
  }
  if (count) *count = sp.size();
  return CG_OK;
}

double cg_model_flops_per_input(const cg_model* m) {
  if (!m) return 0;
  if (m->kind == 1) return m->cnn->flops_per_image();
  return 2.0 * (double)m->u * (double)m->v;
}

int cg_sha256_batch(cg_ctx* ctx, const uint8_t* buf, const uint64_t* off,
                    const uint64_t* len, uint64_t count, uint8_t* out) {
  return guarded(ctx, [&] {
    device_sha256_many(ctx, buf, off, len, count, -1, out);
    return CG_OK;
  });
}

int cg_leaf_hash_batch(cg_ctx* ctx, const uint8_t* buf, const uint64_t* off,
                       const uint64_t* len, uint64_t count, uint8_t* out) {
  return guarded(ctx, [&] {
    device_sha256_many(ctx, buf, off, len, count, 0x00, out);
    return CG_OK;
  });
}

int cg_merkle_root_batch(cg_ctx* ctx, const uint8_t* leaf_hashes,
                         const uint64_t* n_leaves, uint64_t ntrees,
                         uint8_t* roots) {
  return guarded(ctx, [&] {
    if (ntrees == 0) return CG_OK;
    uint64_t total = 0, mx = 0;
    std::vector<uint64_t> off(ntrees);
    for (uint64_t t = 0; t < ntrees; t++) {
      if (n_leaves[t] == 0) throw InvalidArgument("merkle: empty leaf list");
      off[t] = total;
      total += n_leaves[t];
      mx = std::max(mx, n_leaves[t]);
    }
    ctx->d_bytes.ensure(32 * total);
    ctx->d_out.ensure(32 * ntrees);
    CG_CUDA(cudaMemcpyAsync(ctx->d_bytes.p, leaf_hashes, 32 * total,
                            cudaMemcpyHostToDevice, ctx->stream));
    if (mx <= 8192) {
      ctx->d_u64a.ensure(ntrees);
      ctx->d_u64b.ensure(ntrees);
      CG_CUDA(cudaMemcpyAsync(ctx->d_u64a.p, off.data(), 8 * ntrees,
                              cudaMemcpyHostToDevice, ctx->stream));
      CG_CUDA(cudaMemcpyAsync(ctx->d_u64b.p, n_leaves, 8 * ntrees,
                              cudaMemcpyHostToDevice, ctx->stream));
      launch_merkle_trees(ctx->d_bytes.p, ctx->d_u64a.p, ctx->d_u64b.p, nullptr,
                          (uint32_t)ntrees, mx, ctx->d_out.p, ctx->stream);
    } else {
      DevBuf<uint8_t> scratch;
      scratch.ensure(merkle_big_scratch_bytes(mx));
      for (uint64_t t = 0; t < ntrees; t++)
        launch_merkle_big(ctx->d_bytes.p + 32 * off[t], n_leaves[t], scratch.p,
                          ctx->d_out.p + 32 * t, ctx->stream);
      CG_CUDA(cudaStreamSynchronize(ctx->stream));
    }
    CG_CUDA(cudaMemcpyAsync(roots, ctx->d_out.p, 32 * ntrees,
                            cudaMemcpyDeviceToHost, ctx->stream));
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
    return CG_OK;
  });
}

int cg_select_quorum_batch(cg_ctx* ctx, const double* outs,
                           const uint32_t* present, const double* eps,
                           uint32_t R, uint32_t n, uint32_t f, uint32_t v,
                           uint32_t metric, uint32_t* selected,
                           double* diameter, uint8_t* satisfied,
                           int8_t* status, int64_t* label) {
  return guarded(ctx, [&] {
    if (R == 0) return CG_OK;
    if (n > 20 || n == 0) {
      for (uint32_t r = 0; r < R; r++) {
        if (status) status[r] = -1;
        selected[r] = 0; diameter[r] = 0; satisfied[r] = 0;
        if (label) label[r] = -1;
      }
      throw InvalidArgument("select_quorum: bad n/f or too many results");
    }
    const size_t nv = (size_t)R * n * v;
    ctx->d_f64.ensure(nv);
    ctx->d_f64b.ensure(R);
    ctx->d_u32a.ensure(R);
    ctx->d_u32b.ensure(R);
    ctx->d_u8.ensure(R);
    ctx->d_i8.ensure(R);
    ctx->d_i64.ensure(R);
    DevBuf<double> d_diam;
    d_diam.ensure(R);
    cudaStream_t st = ctx->stream;
    CG_CUDA(cudaMemcpyAsync(ctx->d_f64.p, outs, nv * 8, cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(ctx->d_f64b.p, eps, 8 * (size_t)R, cudaMemcpyHostToDevice, st));
    if (present)
      CG_CUDA(cudaMemcpyAsync(ctx->d_u32a.p, present, 4 * (size_t)R,
                              cudaMemcpyHostToDevice, st));
    if (agree_rows_eligible(R, n, f, v, metric, present))
      launch_agree_rows(ctx->d_f64.p, v, (uint64_t)n * v, ctx->d_f64b.p, R, n, f, v, metric,
                        nullptr, 0, ctx->d_u32b.p, d_diam.p, ctx->d_u8.p, ctx->d_i8.p,
                        label ? ctx->d_i64.p : nullptr, nullptr, st);
    else
      launch_select_quorum(ctx->d_f64.p, v, (uint64_t)n * v,
                           present ? ctx->d_u32a.p : nullptr, ctx->d_f64b.p, R, n,
                           f, v, metric, ctx->d_u32b.p, d_diam.p, ctx->d_u8.p,
                           ctx->d_i8.p, label ? ctx->d_i64.p : nullptr, st);
    std::vector<int8_t> stat(R);
    CG_CUDA(cudaMemcpyAsync(selected, ctx->d_u32b.p, 4 * (size_t)R, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(diameter, d_diam.p, 8 * (size_t)R, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(satisfied, ctx->d_u8.p, (size_t)R, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(stat.data(), ctx->d_i8.p, (size_t)R, cudaMemcpyDeviceToHost, st));
    if (label)
      CG_CUDA(cudaMemcpyAsync(label, ctx->d_i64.p, 8 * (size_t)R, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    bool bad = false;
    for (uint32_t r = 0; r < R; r++) {
      if (status) status[r] = stat[r];
      bad |= stat[r] != 0;
    }
    if (bad) throw InvalidArgument("select_quorum: invalid argument for some request");
    return CG_OK;
  });
}

// Device-resident agreement sweep (C5): everything already in HBM, enqueued
// on the ctx stream without a host sync.
int cg_agree_device(cg_ctx* ctx, const double* outs, uint64_t ps, uint64_t rs,
                    const double* eps, uint32_t R, uint32_t n, uint32_t f, uint32_t v,
                    uint32_t metric, const uint8_t* req_ids, uint64_t version,
                    uint32_t* selected, double* diameter, uint8_t* satisfied, int8_t* status,
                    int64_t* label, uint8_t* label_digest) {
  return guarded(ctx, [&] {
    if (R == 0) return CG_OK;
    if (n == 0 || n > 20) throw InvalidArgument("select_quorum: bad n or too many results");
    if (label_digest && (!label || !req_ids))
      throw InvalidArgument("label digests need label and request id buffers");
    cudaStream_t st = ctx->stream;
    if (agree_rows_eligible(R, n, f, v, metric, nullptr)) {
      launch_agree_rows(outs, ps, rs, eps, R, n, f, v, metric, req_ids, version, selected,
                        diameter, satisfied, status, label, label_digest, st);
    } else {
      launch_select_quorum(outs, ps, rs, nullptr, eps, R, n, f, v, metric, selected, diameter,
                           satisfied, status, label, st);
      if (label_digest) launch_label_digest(req_ids, label, R, version, label_digest, st);
    }
    return CG_OK;
  });
}

int cg_label_digest_batch(cg_ctx* ctx, const uint8_t* req_ids, const int64_t* labels,
                          uint32_t R, uint64_t version, uint8_t* out) {
  return guarded(ctx, [&] {
    if (R == 0) return CG_OK;
    ctx->d_u8.ensure(32 * (size_t)R);
    ctx->d_i64.ensure(R);
    ctx->d_out.ensure(32 * (size_t)R);
    cudaStream_t st = ctx->stream;
    CG_CUDA(cudaMemcpyAsync(ctx->d_u8.p, req_ids, 32 * (size_t)R, cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(ctx->d_i64.p, labels, 8 * (size_t)R, cudaMemcpyHostToDevice, st));
    launch_label_digest(ctx->d_u8.p, ctx->d_i64.p, R, version, ctx->d_out.p, st);
    CG_CUDA(cudaMemcpyAsync(out, ctx->d_out.p, 32 * (size_t)R, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    return CG_OK;
  });
}

// ---------------------------------------------------------------- models
// LinearToyModel::from_file_bytes (proj/src/model.cpp:46-60).
int cg_model_load_linear(cg_ctx* ctx, const uint8_t* file, uint64_t len,
                         const uint8_t digest[32], cg_model** out) {
  return guarded(ctx, [&] {
    *out = nullptr;
    auto rd_u64 = [&](uint64_t& pos) {
      if (pos + 8 > len) throw CodecError("unexpected end of input");
      uint64_t v = 0;
      for (int i = 0; i < 8; i++) v = (v << 8) | file[pos++];
      return v;
    };
    auto rd_u32 = [&](uint64_t& pos) {
      if (pos + 4 > len) throw CodecError("unexpected end of input");
      uint32_t v = 0;
      for (int i = 0; i < 4; i++) v = (v << 8) | file[pos++];
      return v;
    };
    check_model_digest(file, len, digest);
    uint64_t pos = 0;
    uint64_t in = rd_u64(pos), outd = rd_u64(pos);
    if (pos + 1 > len) throw CodecError("unexpected end of input");
    uint8_t sm = file[pos++];
    if (sm > 1) throw CodecError("invalid boolean");
    auto rd_list = [&](std::vector<double>& dst) {
      uint32_t n = rd_u32(pos);
      if ((uint64_t)n * 8 > len - pos) throw CodecError("f64 list count exceeds buffer");
      dst.resize(n);
      for (uint32_t i = 0; i < n; i++) {
        uint64_t bits = rd_u64(pos);
        std::memcpy(&dst[i], &bits, 8);
      }
    };
    std::vector<double> W, b;
    rd_list(W);
    rd_list(b);
    if (pos != len) throw CodecError("trailing bytes after value");
    if (in < 1 || outd < 1 || W.size() != in * outd || b.size() != outd)
      throw CodecError("model file shape mismatch");
    auto m = std::make_unique<cg_model>();
    m->ctx = ctx;
    m->kind = 0;
    m->u = in;
    m->v = outd;
    m->softmax = sm == 1;
    std::memcpy(m->digest, digest, 32);
    m->W.ensure(W.size());
    m->b.ensure(b.size());
    CG_CUDA(cudaMemcpy(m->W.p, W.data(), 8 * W.size(), cudaMemcpyHostToDevice));
    CG_CUDA(cudaMemcpy(m->b.p, b.data(), 8 * b.size(), cudaMemcpyHostToDevice));
    *out = m.release();
    return CG_OK;
  });
}

int cg_model_load_cnn(cg_ctx* ctx, const uint8_t* file, uint64_t len,
                      const uint8_t digest[32], cg_model** out) {
  if (!ctx || !out) return CG_EINVAL;
  *out = nullptr;
  // Host phase -- the ~100 MB digest check (engine.cpp:79, before parsing),
  // the parse and the BN fold -- runs without the context lock, so a model
  // version loaded in the background does not stall certification on this
  // context (C4's mid-stream update).
  std::unique_ptr<CnnModel> cnn;
  int code = CG_OK;
  std::string msg;
  try {
    check_model_digest(file, len, digest);
    cnn = CnnModel::from_file(file, len);
  } catch (const DigestError& e) {
    code = CG_EDIGEST;
    msg = e.what();
  } catch (const std::invalid_argument& e) {
    code = CG_ECODEC;
    msg = e.what();
  } catch (const std::exception& e) {
    code = CG_ECUDA;
    msg = e.what();
  }
  return guarded(ctx, [&] {
    if (code == CG_EDIGEST) throw DigestError(msg);
    if (code == CG_ECODEC) throw CodecError(msg);
    if (code != CG_OK) throw std::runtime_error(msg);
    // weights go up on a private stream: the context's streams keep running
    cudaStream_t up = nullptr;
    CG_CUDA(cudaStreamCreateWithFlags(&up, cudaStreamNonBlocking));
    try {
      cnn->upload(up);
    } catch (...) {
      cudaStreamDestroy(up);
      throw;
    }
    CG_CUDA(cudaStreamSynchronize(up));
    CG_CUDA(cudaStreamDestroy(up));
    auto m = std::make_unique<cg_model>();
    m->ctx = ctx;
    m->kind = 1;
    m->u = cnn->input_dim();
    m->v = cnn->output_dim();
    m->softmax = cnn->softmax();
    std::memcpy(m->digest, digest, 32);
    m->cnn = std::move(cnn);
    *out = m.release();
    return CG_OK;
  });
}

void cg_model_free(cg_model* m) {
  if (!m) return;
  if (m->ctx) cudaSetDevice(m->ctx->device);
  delete m;
}

int cg_model_dims(const cg_model* m, uint64_t* input_dim, uint64_t* output_dim) {
  if (!m) return CG_EINVAL;
  if (input_dim) *input_dim = m->u;
  if (output_dim) *output_dim = m->v;
  return CG_OK;
}

}  // extern "C"

namespace {

// Pre-softmax forward of one replica over B device-resident f64 inputs.
// Linear: f64 into pre64. CNN: f32 logits into pre32.
void replica_forward(cg_model* m, const double* d_in, uint32_t B,
                     double* pre64, float* pre32, cudaStream_t st) {
  if (m->kind == 0) {
    launch_linear_f64(m->W.p, m->b.p, d_in, B, (uint32_t)m->u, (uint32_t)m->v,
                      pre64, st);
  } else {
    m->cnn->forward(d_in, B, pre32, st);
  }
}

}  // namespace

namespace {

// ModelExecutor::run, optionally wrapped by PerturbingExecutor (mag > 0).
int exec_run(cg_ctx* ctx, cg_model* m, const double* in, uint64_t B, uint64_t u,
             double* out, uint64_t v, uint64_t node, double mag) {
  return guarded(ctx, [&] {
    if (!(mag >= 0.0)) throw InvalidArgument("negative magnitude");
    if (!m || m->ctx != ctx) throw InvalidArgument("model from another context");
    if (u != m->u) throw InvalidArgument("model input dimension mismatch");
    if (v != m->v) throw InvalidArgument("model output dimension mismatch");
    if (B == 0) return CG_OK;
    cudaStream_t st = ctx->stream;
    DevBuf<double> d_in, d_pre, d_out, d_topv;
    DevBuf<float> d_pre32;
    DevBuf<uint32_t> d_topi;
    d_in.ensure(B * u);
    d_pre.ensure(B * v);
    d_out.ensure(B * v);
    d_topi.ensure(B);
    d_topv.ensure(B);
    if (m->kind == 1) d_pre32.ensure(B * v);
    CG_CUDA(cudaMemcpyAsync(d_in.p, in, 8 * B * u, cudaMemcpyHostToDevice, st));
    replica_forward(m, d_in.p, (uint32_t)B, d_pre.p, d_pre32.p, st);
    if (m->kind == 0)
      launch_softmax_topk_f64(d_pre.p, v, (uint32_t)B, (uint32_t)v, m->softmax,
                              d_out.p, v, 1, d_topi.p, d_topv.p, st);
    else
      launch_softmax_topk_f32(d_pre32.p, v, (uint32_t)B, (uint32_t)v, m->softmax,
                              d_out.p, v, 1, d_topi.p, d_topv.p, st);
    DevBuf<uint8_t> d_hdr;
    DevBuf<uint32_t> d_mid;
    if (mag != 0.0) {  // model.cpp:85: magnitude 0 returns the inner outputs
      // Seed = u64 node || model digest || u32be count (model.cpp:87-90); the
      // model digest is the descriptor digest verified at load.
      PerturbHdr hdr;
      for (int i = 0; i < 8; i++) hdr.b[i] = (uint8_t)(node >> (56 - 8 * i));
      std::memcpy(hdr.b + 8, m->digest, 32);
      for (int i = 0; i < 4; i++) hdr.b[40 + i] = (uint8_t)((uint32_t)u >> (24 - 8 * i));
      const uint64_t nshared = (44 + 8 * u) / 64;
      if (nshared) {
        d_hdr.ensure(64);
        d_mid.ensure(8 * B);
        CG_CUDA(cudaMemcpyAsync(d_hdr.p, hdr.b, 44, cudaMemcpyHostToDevice, st));
        std::vector<ChainJob> jobs(B);
        for (uint64_t k = 0; k < B; k++) {
          ChainJob& j = jobs[k];
          std::memset(&j, 0, sizeof j);
          j.seg[0] = ChainSeg{(uint64_t)d_hdr.p, 0, 44, kSegRaw, 0};
          j.seg[1] = ChainSeg{(uint64_t)(d_in.p + u * k), 44, 8 * u, kSegF64, 0};
          j.nseg = 2;
          j.total_len = 44 + 8 * u;
          j.blk_end = nshared;
          j.state_out = (uint64_t)(d_mid.p + 8 * k);
        }
        ctx->d_jobs.ensure(B);
        CG_CUDA(cudaMemcpyAsync(ctx->d_jobs.p, jobs.data(), B * sizeof(ChainJob),
                                cudaMemcpyHostToDevice, st));
        launch_chain_jobs(ctx->d_jobs.p, (uint32_t)B, st);
      }
      launch_perturb_tail(d_mid.p, d_in.p, u, hdr, nshared, d_out.p, v, (uint32_t)B,
                          (uint32_t)v, mag, st);
    }
    CG_CUDA(cudaMemcpyAsync(out, d_out.p, 8 * B * v, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    return CG_OK;
  });
}

}  // namespace

extern "C" int cg_exec_run(cg_ctx* ctx, cg_model* m, const double* in,
                           uint64_t B, uint64_t u, double* out, uint64_t v) {
  return exec_run(ctx, m, in, B, u, out, v, 0, 0.0);
}

extern "C" int cg_exec_run_perturbed(cg_ctx* ctx, cg_model* m, const double* in,
                                     uint64_t B, uint64_t u, double* out, uint64_t v,
                                     uint64_t node_index, double magnitude) {
  return exec_run(ctx, m, in, B, u, out, v, node_index, magnitude);
}

// Test hook: iters forwards of one CNN replica over B device-resident random
// inputs; average device ms per forward (CUDA events on the ctx stream).
extern "C" int cg_dbg_forward_bench(cg_ctx* ctx, cg_model* m, uint32_t B, int iters,
                                    double* ms_per_forward) {
  return guarded(ctx, [&] {
    if (!m || m->kind != 1) throw InvalidArgument("cnn model required");
    cudaStream_t st = ctx->stream;
    DevBuf<double> d_in;
    DevBuf<float> d_out;
    d_in.ensure((size_t)B * m->u);
    d_out.ensure((size_t)B * m->v);
    CG_CUDA(cudaMemsetAsync(d_in.p, 0, 8 * (size_t)B * m->u, st));
    m->cnn->reserve(B);
    m->cnn->forward(d_in.p, B, d_out.p, st);  // warm (plan + tensor maps)
    cudaEvent_t e0, e1;
    CG_CUDA(cudaEventCreate(&e0));
    CG_CUDA(cudaEventCreate(&e1));
    CG_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < iters; i++) m->cnn->forward(d_in.p, B, d_out.p, st);
    CG_CUDA(cudaEventRecord(e1, st));
    CG_CUDA(cudaEventSynchronize(e1));
    float ms = 0;
    CG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *ms_per_forward = ms / iters;
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    return CG_OK;
  });
}

namespace cg {

// Each local provider p's outputs += its PerturbingExecutor offsets
// (model.cpp:82-105). The per (p, request) midstates over the shared whole
// blocks of u64 p || weights digest || f64_list(input) were chained at ingest
// on the slot's stream (they depend on the input only); here one thread per
// (request, lane) runs the 1-2 tail blocks. The node index is the provider
// index (the harness builds node i's executor with node_index i).
void perturb_group_outputs(cg_group* g, const IngestSlot& S, double* d_outs, cudaStream_t st) {
  const uint64_t u = g->u, v = g->v;
  const uint32_t nloc = (uint32_t)g->models.size(), B = S.B;
  const uint64_t nshared = (44 + 8 * u) / 64;
  for (uint32_t li = 0; li < nloc; li++) {
    const uint64_t p = g->first + li;
    PerturbHdr hdr;
    for (int i = 0; i < 8; i++) hdr.b[i] = (uint8_t)(p >> (56 - 8 * i));
    std::memcpy(hdr.b + 8, g->digests[p].data(), 32);
    for (int i = 0; i < 4; i++) hdr.b[40 + i] = (uint8_t)((uint32_t)u >> (24 - 8 * i));
    launch_perturb_tail(nshared ? S.d_pmid.p + 8ull * li * B : nullptr, S.d_in_ptr, u, hdr,
                        nshared, d_outs + p * B * v, v, B, (uint32_t)v, g->perturb_mag, st);
  }
}

// cg_ctx_join: the context stream waits for every slot's outstanding work
// (ingest prefix chains of uncertified batches, single leaves + A root of
// certified ones).
void join_group_slots(cg_ctx* ctx) {
  for (cg_group* g : ctx->groups)
    for (auto& sl : g->slots) {
      if (!sl->ever) continue;
      if (sl->used) CG_CUDA(cudaStreamWaitEvent(ctx->stream, sl->ev_prefix, 0));
      if (sl->certified) CG_CUDA(cudaStreamWaitEvent(ctx->stream, sl->ev_done, 0));
    }
}

const IngestSlot& certified_slot(const cg_group* g, uint64_t ticket) {
  const IngestSlot& S = *g->slots[ticket % g->slots.size()];
  if (S.ticket != ticket || !S.certified)
    throw InvalidArgument("ticket not certified or its slot already reused");
  return S;
}

IngestSlot& slot_for(cg_group* g, uint64_t ticket) {
  IngestSlot& s = *g->slots[ticket % g->slots.size()];
  if (!s.used || s.ticket != ticket) throw InvalidArgument("unknown or already certified ticket");
  return s;
}

// InferenceEngine::submit's hot part (engine.cpp:182-209): take the batch,
// build the canonical framing bytes of every leaf it will need, upload, and
// start the request-midstate chains H(0x00||0x52||request)[whole blocks].
uint64_t ingest(cg_group* g, const cg_request_batch* bt, cudaEvent_t staged) {
  const uint32_t B = bt->B, N = g->N;
  const uint64_t u = bt->u, v = g->v;
  if (B == 0) throw InvalidArgument("empty batch");
  if (B > g->maxB) throw InvalidArgument("batch larger than group max_batch");
  if (u != g->u) throw InvalidArgument("request input dimension mismatch");
  const uint64_t ticket = g->next_ticket;
  IngestSlot& S = *g->slots[ticket % g->slots.size()];
  if (S.used) throw InvalidArgument("ingest ring full: certify an outstanding ticket first");
  cudaStream_t st = S.stream;
  if (S.ever) {
    CG_CUDA(cudaEventSynchronize(S.ev_staged));      // pinned staging reusable
    CG_CUDA(cudaStreamWaitEvent(st, S.ev_done, 0));  // device buffers reusable
  }
  Arena ar;
  std::vector<ChainJob> jobs;
  jobs.reserve((size_t)B * (4 + 2 * N + 2 * g->models.size()));
  const uint8_t* gid = (const uint8_t*)g->gid.data();
  const uint32_t gl = (uint32_t)g->gid.size();
  // Per op: an ok inference request (the common case), a request the
  // primary rejected, or a group operation (PRE-PREPARE op list,
  // messages.hpp:106-118). Requests without provider results -- misfits
  // (input dimension != u), rejected requests -- get missing_result_leaf;
  // group ops get group_op_leaf; neither kind has an agreement outcome.
  struct ReqLayout {
    size_t h, h53, h4d, t, h47, f46;
    uint64_t lenH, lenT, P, uk, moff;  // uk: this request's input count; moff: misfit input offset
    uint64_t len47, len46;
    uint8_t kind;
    bool in_mis;   // input read from the misfit buffer (its dimension != u)
    bool noresult; // no provider output: R leaf 0x4D (requests) / 0x47 (group ops)
  };
  std::vector<ReqLayout> rl(B);
  std::vector<size_t> res_off((size_t)B * N), dig_off((size_t)B * N);
  uint64_t lenRes = 0, nonce_pos = 0, misfit_total = 0, entry_pos = 0, rec_pos = 0;
  bool any_miss = false, any_kind = false;
  for (uint32_t k = 0; k < B; k++) {
    const uint8_t* rid = bt->request_ids + 32 * k;
    ReqLayout& L = rl[k];
    L.kind = bt->op_kinds ? bt->op_kinds[k] : CG_OP_REQUEST;
    if (L.kind > CG_OP_GROUP) throw InvalidArgument("unknown op kind");
    any_kind |= L.kind != CG_OP_REQUEST;
    L.uk = L.kind == CG_OP_GROUP ? u : (bt->input_dims ? bt->input_dims[k] : u);
    L.in_mis = L.uk != u;
    L.noresult = L.in_mis || L.kind != CG_OP_REQUEST;
    L.moff = misfit_total;
    if (L.in_mis) {
      if (!bt->misfit_inputs || (L.uk && !bt->misfit_inputs[k]))
        throw InvalidArgument("misfit request without its input");
      misfit_total += L.uk;
    }
    any_miss |= L.noresult;
    L.len47 = L.kind == CG_OP_GROUP ? (bt->op_entry_lens ? bt->op_entry_lens[k] : 0) : 0;
    L.len46 = bt->fail_record_lens ? bt->fail_record_lens[k] : 0;
    if (L.kind == CG_OP_REQUEST && L.len46)
      throw InvalidArgument("a failure record is for rejected ops only");
    if (L.kind == CG_OP_REQUEST_REJECTED && !L.len46)
      throw InvalidArgument("a rejected op needs its failure record");
    if (L.len47) {  // group_op_leaf: 0x00 || 0x47 || OpEntry::encode (messages.cpp:220-225)
      Enc E;
      E.u8(0x00);
      E.u8(0x47);
      E.raw(bt->op_entries + entry_pos, L.len47);
      entry_pos += L.len47;
      L.h47 = ar.add(E.b.data(), E.b.size(), 0);
      L.len47 = E.b.size();
    } else if (L.kind == CG_OP_GROUP) {
      throw InvalidArgument("a group op needs its OpEntry encoding");
    }
    if (L.len46) {  // failure_leaf: 0x00 || 0x46 || FailureRecord::encode (messages.cpp:260-297)
      Enc E;
      E.u8(0x00);
      E.u8(0x46);
      E.raw(bt->fail_records + rec_pos, L.len46);
      rec_pos += L.len46;
      L.f46 = ar.add(E.b.data(), E.b.size(), 0);
      L.len46 = E.b.size();
    }
    Enc H;  // 0x00 (leaf domain) || 0x52 (result leaf) || request body head
    H.u8(0x00);
    H.u8(0x52);
    H.raw(rid, 32);
    H.bytes(gid, gl);
    H.u32((uint32_t)L.uk);
    Enc T;  // request tail after the f64 input list (domain.cpp:144-158)
    bool he = bt->has_eps && bt->has_eps[k];
    T.u8(he ? 1 : 0);
    if (he) T.f64(bt->eps[k]);
    T.raw(bt->client_pubs + 32 * k, 32);
    T.bytes(bt->nonces + nonce_pos, bt->nonce_lens[k]);
    nonce_pos += bt->nonce_lens[k];
    T.raw(bt->client_sigs + 64 * k, 64);
    L.lenH = H.b.size();
    L.lenT = T.b.size();
    L.P = L.lenH + 8 * L.uk + L.lenT;
    L.h = ar.add(H.b.data(), H.b.size(), 0);
    H.b[1] = 0x53;  // single_attest_leaf tag (messages.cpp:283-290)
    L.h53 = ar.add(H.b.data(), H.b.size(), 0);
    H.b[1] = 0x4D;  // missing_result_leaf tag (messages.cpp:213-218)
    L.h4d = (L.noresult && L.kind != CG_OP_GROUP) ? ar.add(H.b.data(), H.b.size(), 0) : 0;
    L.t = ar.add(T.b.data(), T.b.size(), L.lenH + 8 * L.uk);
    for (uint32_t p = 0; p < N; p++) {
      Enc R;  // InferenceResult::encode up to the output list (domain.cpp:218-225)
      R.raw(rid, 32);
      R.u64(p);
      R.bytes(gid, gl);
      R.u64(g->version);
      R.u32((uint32_t)v);
      lenRes = R.b.size();
      res_off[(size_t)k * N + p] = ar.add(R.b.data(), R.b.size(), L.P);
      dig_off[(size_t)k * N + p] = ar.add(g->digests[p].data(), 32, L.P + lenRes + 8 * v);
    }
  }
  S.d_arena.ensure(ar.b.size() + 64);
  S.h_arena.ensure(ar.b.size() + 64);
  std::memcpy(S.h_arena.p, ar.b.data(), ar.b.size());
  const uint64_t A = (uint64_t)S.d_arena.p;
  if (!bt->inputs_on_device) S.d_in.ensure((uint64_t)g->maxB * u);
  S.d_in_ptr = bt->inputs_on_device ? bt->inputs : S.d_in.p;
  S.any_miss = any_miss;
  S.any_kind = any_kind;
  if (!S.d_neg1.p) {
    const int32_t neg1 = -1;
    S.d_neg1.ensure(1);
    CG_CUDA(cudaMemcpy(S.d_neg1.p, &neg1, 4, cudaMemcpyHostToDevice));
  }
  if (any_miss) {
    S.d_misfit.ensure(std::max<uint64_t>(misfit_total, 1));
    S.d_miss.ensure(3 * (uint64_t)g->maxB);  // missing, has-outcome, explicit-failure flags
    S.h_miss.ensure(3 * (uint64_t)g->maxB);
    S.d_fail_pos.ensure(g->maxB);
    for (uint32_t k = 0; k < B; k++) {
      S.h_miss.p[k] = rl[k].noresult ? 1 : 0;
      S.h_miss.p[B + k] = rl[k].kind == CG_OP_REQUEST ? 1 : 0;
      S.h_miss.p[2 * B + k] = rl[k].len46 ? 1 : 0;
      if (rl[k].in_mis && rl[k].uk)  // pageable host source: synchronous, rare
        CG_CUDA(cudaMemcpyAsync(S.d_misfit.p + rl[k].moff, bt->misfit_inputs[k], 8 * rl[k].uk,
                                cudaMemcpyHostToDevice, st));
    }
  }
  const uint64_t MIS = (uint64_t)S.d_misfit.p;
  const uint64_t IN = (uint64_t)S.d_in_ptr;
  const uint64_t OUT = (uint64_t)S.res.d_outs.p;
  auto seg_raw = [](uint64_t ptr, uint64_t off, uint64_t len) {
    return ChainSeg{ptr, off, len, kSegRaw, 0};
  };
  auto seg_f64 = [](uint64_t ptr, uint64_t off, uint64_t len) {
    return ChainSeg{ptr, off, len, kSegF64, 0};
  };
  auto leaf_job = [&](uint32_t k, uint32_t p, size_t head) {
    const ReqLayout& L = rl[k];
    ChainJob j;
    std::memset(&j, 0, sizeof j);
    j.seg[0] = seg_raw(A + head, 0, L.lenH);
    j.seg[1] = seg_f64(L.in_mis ? MIS + 8 * L.moff : IN + 8 * u * k, L.lenH, 8 * L.uk);
    j.seg[2] = seg_raw(A + L.t, L.lenH + 8 * L.uk, L.lenT);
    j.seg[3] = seg_raw(A + res_off[(size_t)k * N + p], L.P, lenRes);
    j.seg[4] = seg_f64(OUT + 8 * v * ((uint64_t)p * B + k), L.P + lenRes, 8 * v);
    j.seg[5] = seg_raw(A + dig_off[(size_t)k * N + p], L.P + lenRes + 8 * v, 32);
    j.nseg = 6;
    j.final_ = 1;
    j.total_len = L.P + lenRes + 8 * v + 32;
    j.blk_end = (j.total_len + 9 + 63) / 64;
    return j;
  };
  // [0, B): request midstates (a misfit's slot is a no-op: its R leaves are
  // whole missing_result_leaf chains, below)
  for (uint32_t k = 0; k < B; k++) {
    const ReqLayout& L = rl[k];
    ChainJob j;
    std::memset(&j, 0, sizeof j);
    j.seg[0] = seg_raw(A + L.h, 0, L.lenH);
    j.seg[1] = seg_f64(IN + 8 * u * k, L.lenH, 8 * u);
    j.seg[2] = seg_raw(A + L.t, L.lenH + 8 * u, L.lenT);
    j.nseg = 3;
    j.total_len = L.P;
    j.blk_end = L.P / 64;
    j.state_out = (uint64_t)(S.d_mid.p + 8 * k);
    if (L.noresult) j.skip_flag = (uint64_t)S.d_neg1.p;
    jobs.push_back(j);
  }
  // ops without provider results: every local provider's R tree holds
  // missing_result_leaf H(0x00||0x4D||request) (misfit / rejected requests)
  // or group_op_leaf H(0x00||0x47||OpEntry) at the op's position
  // (build_result_tree, messages.cpp:235-258)
  if (any_miss)
    for (uint32_t k = 0; k < B; k++) {
      const ReqLayout& L = rl[k];
      if (!L.noresult) continue;
      for (uint32_t li = 0; li < (uint32_t)g->models.size(); li++) {
        const uint32_t p = g->first + li;
        ChainJob j;
        std::memset(&j, 0, sizeof j);
        if (L.kind == CG_OP_GROUP) {
          j.seg[0] = seg_raw(A + L.h47, 0, L.len47);
          j.nseg = 1;
          j.total_len = L.len47;
        } else {
          j.seg[0] = seg_raw(A + L.h4d, 0, L.lenH);
          j.seg[1] = seg_f64(L.in_mis ? MIS + 8 * L.moff : IN + 8 * u * k, L.lenH, 8 * L.uk);
          j.seg[2] = seg_raw(A + L.t, L.lenH + 8 * L.uk, L.lenT);
          j.nseg = 3;
          j.total_len = L.P;
        }
        j.final_ = 1;
        j.blk_end = (j.total_len + 9 + 63) / 64;
        j.digest_out = (uint64_t)(S.res.d_leaf.p + 32 * ((uint64_t)p * B + k));
        jobs.push_back(j);
      }
    }
  // PerturbingExecutor seeds: per (local provider, request) the midstate
  // over the whole blocks of u64 p || weights digest || f64_list(input)
  // (model.cpp:87-90), chained here with the request midstates (same launch)
  const uint32_t nloc = (uint32_t)g->models.size();
  const uint64_t pshared = (44 + 8 * u) / 64;
  S.perturbed = g->perturb_mag != 0.0;
  if (S.perturbed && pshared) {
    S.d_pmid.ensure(8ull * nloc * g->maxB);
    for (uint32_t li = 0; li < nloc; li++)
      for (uint32_t k = 0; k < B; k++) {
        ChainJob j;
        std::memset(&j, 0, sizeof j);
        j.seg[0] = seg_raw((uint64_t)(g->d_phdr.p + 64 * li), 0, 44);
        j.seg[1] = seg_f64(IN + 8 * u * k, 44, 8 * u);
        j.nseg = 2;
        j.total_len = 44 + 8 * u;
        j.blk_end = pshared;
        j.state_out = (uint64_t)(S.d_pmid.p + 8 * ((uint64_t)li * B + k));
        jobs.push_back(j);
      }
  }
  // single attestation leaves H(0x00||0x53||req||res) (messages.cpp:283-290):
  // the manifest kernel decides on device which (request, provider) pairs
  // need one and where it lands; the request part H(0x00||0x53||req) is one
  // midstate per request. Lazy (default): chained after the manifest only for
  // requests that have a single leaf. Speculative (after recent batches had
  // single leaves, g->spec53): chained at ingest with the request midstates,
  // so a faulty stream's 1.2 MB chains are off the certification path.
  S.spec53 = g->spec53 > 0;
  auto push_mid53 = [&] {
    S.off_mid53 = jobs.size();
    for (uint32_t k = 0; k < B; k++) {
      const ReqLayout& L = rl[k];
      ChainJob j;
      std::memset(&j, 0, sizeof j);
      j.seg[0] = seg_raw(A + L.h53, 0, L.lenH);
      j.seg[1] = seg_f64(L.in_mis ? MIS + 8 * L.moff : IN + 8 * u * k, L.lenH, 8 * L.uk);
      j.seg[2] = seg_raw(A + L.t, L.lenH + 8 * L.uk, L.lenT);
      j.nseg = 3;
      j.total_len = L.P;
      j.blk_end = L.P / 64;
      j.state_out = (uint64_t)(S.d_mid53.p + 8 * k);
      if (!S.spec53 || L.noresult) j.skip_flag = (uint64_t)(S.res.d_need53.p + k);
      if (S.spec53 && L.noresult) j.skip_flag = (uint64_t)S.d_neg1.p;
      jobs.push_back(j);
    }
  };
  if (S.spec53) push_mid53();
  const uint64_t n_prefix = jobs.size();
  // result leaves H(0x00||0x52||req||res) from the request midstate
  S.off_leaf = jobs.size();
  for (uint32_t p = 0; p < N; p++)
    for (uint32_t k = 0; k < B; k++) {
      ChainJob j = leaf_job(k, p, rl[k].h);
      j.blk_begin = rl[k].P / 64;
      j.state_in = j.blk_begin ? (uint64_t)(S.d_mid.p + 8 * k) : 0;
      j.digest_out = (uint64_t)(S.res.d_leaf.p + 32 * ((uint64_t)p * B + k));
      if (rl[k].noresult) j.skip_flag = (uint64_t)S.d_neg1.p;  // written at ingest (0x4D / 0x47)
      jobs.push_back(j);
    }
  if (!S.spec53) push_mid53();
  S.off_single = jobs.size();
  for (uint32_t k = 0; k < B; k++)
    for (uint32_t p = 0; p < N; p++) {
      ChainJob j = leaf_job(k, p, rl[k].h53);
      j.blk_begin = rl[k].P / 64;
      j.state_in = j.blk_begin ? (uint64_t)(S.d_mid53.p + 8 * k) : 0;
      j.digest_out = (uint64_t)S.res.d_aleaf.p;
      j.skip_flag = (uint64_t)(S.res.d_single_pos.p + (uint64_t)k * N + p);
      jobs.push_back(j);
    }
  // explicit failure leaves of rejected ops (failure_record_for with the
  // op's reason, messages.cpp:299-312): the manifest decides where they land
  S.n_fail_jobs = 0;
  if (any_miss)
    for (uint32_t k = 0; k < B; k++) {
      const ReqLayout& L = rl[k];
      if (!L.len46) continue;
      ChainJob j;
      std::memset(&j, 0, sizeof j);
      j.seg[0] = seg_raw(A + L.f46, 0, L.len46);
      j.nseg = 1;
      j.final_ = 1;
      j.total_len = L.len46;
      j.blk_end = (L.len46 + 9 + 63) / 64;
      j.digest_out = (uint64_t)S.res.d_aleaf.p;
      j.skip_flag = (uint64_t)(S.d_fail_pos.p + k);
      jobs.push_back(j);
      S.n_fail_jobs++;
    }
  S.h_jobs.ensure(jobs.size());
  S.d_jobs.ensure(jobs.size());
  std::memcpy(S.h_jobs.p, jobs.data(), jobs.size() * sizeof(ChainJob));
  for (uint32_t k = 0; k < B; k++)
    S.h_eps.p[k] = (bt->has_eps && bt->has_eps[k]) ? bt->eps[k] : g->eps_default;
  std::memcpy(S.h_reqids.p, bt->request_ids, 32 * (size_t)B);
  for (uint32_t p = 0; p < N; p++) {
    S.h_tree.p[p] = (uint64_t)p * B;
    S.h_tree.p[N + p] = B;
  }
  CG_CUDA(cudaMemcpyAsync(S.d_arena.p, S.h_arena.p, ar.b.size(), cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemcpyAsync(S.d_jobs.p, S.h_jobs.p, jobs.size() * sizeof(ChainJob),
                          cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemcpyAsync(S.d_eps.p, S.h_eps.p, 8 * (size_t)B, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemcpyAsync(S.d_reqids.p, S.h_reqids.p, 32 * (size_t)B, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaMemcpyAsync(S.d_tree.p, S.h_tree.p, 16 * (size_t)N, cudaMemcpyHostToDevice, st));
  if (any_miss)
    CG_CUDA(cudaMemcpyAsync(S.d_miss.p, S.h_miss.p, 3 * (size_t)B, cudaMemcpyHostToDevice, st));
  if (!bt->inputs_on_device)
    CG_CUDA(cudaMemcpyAsync(S.d_in.p, bt->inputs, 8 * u * B, cudaMemcpyHostToDevice, st));
  CG_CUDA(cudaEventRecord(S.ev_staged, st));
  if (staged) CG_CUDA(cudaEventRecord(staged, st));  // the caller's staging is free again
  launch_chain_jobs(S.d_jobs.p, (uint32_t)n_prefix, st, /*exclusive_sm=*/true);
  CG_CUDA(cudaEventRecord(S.ev_prefix, st));
  S.used = true;
  S.ever = true;
  S.certified = false;
  S.ticket = ticket;
  S.B = B;
  g->next_ticket++;
  return ticket;
}

// execute_batch + try_prepare's R trees + try_attest (engine.cpp:269-306,
// coordinator.cpp:588-624, 727-849). The replica forwards run on the main
// stream; the certification tail (result leaves, R trees, [NCCL exchange],
// select_quorum + label, manifest, A tree) runs on the context's tail stream
// behind the slot's ev_fwd, overlapping the next batch's forwards.
cudaStream_t tail_stream(cg_ctx* ctx) {
  if (!ctx->tail) {
    int lo = 0, hi = 0;
    CG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
    CG_CUDA(cudaStreamCreateWithPriority(&ctx->tail, cudaStreamNonBlocking, hi));
  }
  return ctx->tail;
}

void certify(cg_group* g, uint64_t ticket, const double* precomputed_outputs) {
  IngestSlot& S = slot_for(g, ticket);
  BatchResults& R = S.res;
  cg_ctx* ctx = g->ctx;
  const uint32_t B = S.B, N = g->N;
  const uint64_t v = g->v;
  const uint32_t gl = (uint32_t)g->gid.size();
  cudaStream_t st = ctx->stream;
  cudaStream_t tl = tail_stream(ctx);
  CG_CUDA(cudaStreamWaitEvent(st, S.ev_staged, 0));
  if (precomputed_outputs) {
    // agreement/digest-only mode (C5): N x B x v outputs supplied by the host
    CG_CUDA(cudaMemcpyAsync(R.d_outs.p, precomputed_outputs, 8 * (size_t)N * B * v,
                            cudaMemcpyHostToDevice, st));
  } else {
    // No SM budget: the GEMM launches hand out tiles by cluster launch
    // control, so SMs held by the chain CTAs of other streams are simply
    // not used by the GEMM (gemm_sm100.cu, TileSched).
    const void* prepped = nullptr;
    if (g->same_prep) {  // replica-independent input stage, once per batch
      g->models[0]->cnn->prepare_input(S.d_in_ptr, B, g->d_prep.p, st);
      prepped = g->d_prep.p;
    }
    // Same-architecture CNN replicas: one grouped GEMM launch per layer.
    // (replica-parallel groups: this rank's replicas)
    const uint32_t nloc = (uint32_t)g->models.size(), first = g->first;
    if (g->same_prep && g->group_plan_ok && (!g->gplan || g->gplan->batch() != B)) {
      std::vector<CnnModel*> ms;
      std::vector<float*> lg;
      for (uint32_t li = 0; li < nloc; li++) {
        ms.push_back(g->models[li]->cnn.get());
        lg.push_back(g->d_pre32.p + (uint64_t)li * B * v);
      }
      g->gplan = CnnGroupPlan::build(ms, B, g->d_prep.p, lg);
      g->group_plan_ok = g->gplan != nullptr;
    }
    const bool grouped = g->same_prep && g->gplan && g->gplan->batch() == B;
    if (grouped) {
      g->gplan->run(st);
      bool same_sm = true;
      for (uint32_t li = 1; li < nloc; li++)
        same_sm &= g->models[li]->softmax == g->models[0]->softmax;
      if (same_sm) {  // softmax/top-k of all local rows in one launch
        launch_softmax_topk_f32(g->d_pre32.p, v, nloc * B, (uint32_t)v, g->models[0]->softmax,
                                R.d_outs.p + (uint64_t)first * B * v, v, g->topk,
                                R.d_topi.p + (uint64_t)first * B * g->topk,
                                R.d_topv.p + (uint64_t)first * B * g->topk, st);
      } else {
        for (uint32_t li = 0; li < nloc; li++) {
          const uint64_t p = first + li;
          launch_softmax_topk_f32(g->d_pre32.p + (uint64_t)li * B * v, v, B, (uint32_t)v,
                                  g->models[li]->softmax, R.d_outs.p + p * B * v, v, g->topk,
                                  R.d_topi.p + p * B * g->topk, R.d_topv.p + p * B * g->topk, st);
        }
      }
    }
    static const bool kHeteroStreams = std::getenv("CREDO_NO_HETERO_STREAMS") == nullptr;
    if (!grouped && nloc > 1 && g->all_cnn && kHeteroStreams) {
      if (g->rstreams.size() < nloc) {
        int lo = 0, hi = 0;
        CG_CUDA(cudaDeviceGetStreamPriorityRange(&lo, &hi));
        while (g->rstreams.size() < nloc) {
          cudaStream_t s2;
          CG_CUDA(cudaStreamCreateWithPriority(&s2, cudaStreamNonBlocking, lo));
          g->rstreams.push_back(s2);
        }
        while (g->revs.size() < nloc + 1) {
          cudaEvent_t e;
          CG_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
          g->revs.push_back(e);
        }
      }
      CG_CUDA(cudaEventRecord(g->revs[0], st));
      for (uint32_t li = 0; li < nloc; li++) {
        const uint32_t p = first + li;
        cg_model* m = g->models[li];
        cudaStream_t rs = g->rstreams[li];
        float* lg = g->d_pre32.p + (uint64_t)li * B * v;  // per-replica logits
        CG_CUDA(cudaStreamWaitEvent(rs, g->revs[0], 0));
        m->cnn->forward(S.d_in_ptr, B, lg, rs, prepped);
        launch_softmax_topk_f32(lg, v, B, (uint32_t)v, m->softmax, R.d_outs.p + (uint64_t)p * B * v,
                                v, g->topk, R.d_topi.p + (uint64_t)p * B * g->topk,
                                R.d_topv.p + (uint64_t)p * B * g->topk, rs);
        CG_CUDA(cudaEventRecord(g->revs[1 + li], rs));
      }
      for (uint32_t li = 0; li < nloc; li++) CG_CUDA(cudaStreamWaitEvent(st, g->revs[1 + li], 0));
    }
    const bool concurrent = !grouped && nloc > 1 && g->all_cnn && kHeteroStreams;
    for (uint32_t li = 0; li < nloc && !grouped && !concurrent; li++) {
      const uint32_t p = first + li;  // provider index of local replica li
      cg_model* m = g->models[li];
      double* outs = R.d_outs.p + (uint64_t)p * B * v;
      uint32_t* ti = R.d_topi.p + (uint64_t)p * B * g->topk;
      double* tv = R.d_topv.p + (uint64_t)p * B * g->topk;
      if (m->kind == 1) {
        m->cnn->forward(S.d_in_ptr, B, g->d_pre32.p, st, prepped);
        launch_softmax_topk_f32(g->d_pre32.p, v, B, (uint32_t)v, m->softmax, outs, v,
                                g->topk, ti, tv, st);
      } else {
        replica_forward(m, S.d_in_ptr, B, g->d_pre64.p, g->d_pre32.p, st);
        launch_softmax_topk_f64(g->d_pre64.p, v, B, (uint32_t)v, m->softmax, outs, v,
                                g->topk, ti, tv, st);
      }
    }
  }
  if (S.perturbed && !precomputed_outputs) {
    CG_CUDA(cudaStreamWaitEvent(st, S.ev_prefix, 0));  // seed midstates chained at ingest
    perturb_group_outputs(g, S, R.d_outs.p, st);
  }
  if (g->fault_thr && !precomputed_outputs) {  // OffsetExecutor wraps the perturbing one
    const uint32_t p = g->fault_provider;
    const bool local = p >= g->first && p < g->first + (uint32_t)g->models.size();
    if (local)
      launch_offset_outputs(R.d_outs.p + (uint64_t)p * B * v, S.d_reqids.p, B, (uint32_t)v,
                            g->fault_offset, g->fault_thr, st);
  }
  CG_CUDA(cudaEventRecord(S.ev_fwd, st));
  // ---- the tail, on the tail stream
  CG_CUDA(cudaStreamWaitEvent(tl, S.ev_fwd, 0));
  CG_CUDA(cudaStreamWaitEvent(tl, S.ev_prefix, 0));
  if (g->dist) {
    // This rank serves providers [first, first + nloc) (assigned_models
    // chunking): their result leaves and R roots (try_prepare), then one
    // NCCL all-gather of every provider's outputs and R root over NVLink;
    // agreement and the attestation are then computed on every rank, as
    // every reference node attests.
    const uint32_t first = g->first, nloc = (uint32_t)g->models.size();
    launch_chain_jobs(S.d_jobs.p + S.off_leaf + (uint64_t)first * B, nloc * B, tl,
                      /*exclusive_sm=*/true);
    launch_merkle_trees(R.d_leaf.p, S.d_tree.p + first, S.d_tree.p + N + first, nullptr, nloc, B,
                        R.d_rroots.p + 32 * first, tl);
    timer_begin(tl, kTimeComm);
    ncclResult_t e1, e2, e3;
    e1 = ncclGroupStart();
    e2 = ncclAllGather(R.d_outs.p + (uint64_t)first * B * v, R.d_outs.p, (size_t)nloc * B * v,
                       ncclDouble, ctx->comm, tl);
    e3 = ncclAllGather(R.d_rroots.p + 32 * first, R.d_rroots.p, 32 * (size_t)nloc, ncclUint8,
                       ctx->comm, tl);
    ncclResult_t e4 = ncclGroupEnd();
    timer_end(tl, kTimeComm);
    if (e1 != ncclSuccess || e2 != ncclSuccess || e3 != ncclSuccess || e4 != ncclSuccess)
      throw CudaError(std::string("ncclAllGather: ") + ncclGetErrorString(e4));
  } else {
    launch_chain_jobs(S.d_jobs.p + S.off_leaf, N * B, tl, /*exclusive_sm=*/true);  // result leaves
    launch_merkle_trees(R.d_leaf.p, S.d_tree.p, S.d_tree.p + N, nullptr, N, B, R.d_rroots.p, tl);
  }
  timer_begin(tl, kTimeAgree);
  launch_select_quorum(R.d_outs.p, (uint64_t)B * v, v, nullptr, S.d_eps.p, B, N, g->f,
                       (uint32_t)v, g->metric, R.d_sel.p, R.d_diam.p, R.d_sat.p, R.d_status.p,
                       R.d_label.p, tl);
  // misfits: no provider has an output, so try_attest never runs
  // select_quorum for them (fewer than N-f outputs, coordinator.cpp:759-768)
  if (S.any_miss)
    launch_mark_missing(S.d_miss.p, B, R.d_sel.p, R.d_diam.p, R.d_sat.p, R.d_status.p,
                        R.d_label.p, tl);
  launch_attest_manifest(B, N, R.d_sel.p, R.d_sat.p, R.d_rroots.p, S.d_reqids.p, g->d_gid.p, gl,
                         g->version, R.d_aleaf.p, R.d_single_pos.p, R.d_need53.p, R.d_kinds.p,
                         R.d_mnodes.p, R.d_mops.p, R.d_count.p,
                         S.any_kind ? S.d_miss.p + B : nullptr,
                         S.any_kind ? S.d_miss.p + 2 * (size_t)B : nullptr,
                         S.any_kind ? S.d_fail_pos.p : nullptr, tl);
  timer_end(tl, kTimeAgree);
  // Single attestation leaves re-hash their request (a 1.2 MB chain at
  // ImageNet shape): they run on the slot's own stream, off the shared tail,
  // so a faulty batch delays only its own A root, not the next batches'
  // tails; requests without a single leaf skip their 0x53 midstate chain.
  CG_CUDA(cudaEventRecord(S.ev_man, tl));
  CG_CUDA(cudaStreamWaitEvent(S.stream, S.ev_man, 0));
  if (!S.spec53) launch_chain_jobs(S.d_jobs.p + S.off_mid53, B, S.stream, /*exclusive_sm=*/true);
  launch_chain_jobs(S.d_jobs.p + S.off_single, N * B + S.n_fail_jobs, S.stream);
  launch_merkle_trees(R.d_aleaf.p, nullptr, nullptr, R.d_count.p, 1, (uint64_t)N * B + B + N,
                      R.d_aroot.p, S.stream);
  CG_CUDA(cudaEventRecord(S.ev_done, S.stream));
  S.used = false;
  S.certified = true;
  g->last = &S;
  g->last_B = B;
}

void certify_fetch(cg_group* g, cg_certify_out* o, const IngestSlot* slot) {
  // The readback waits for this batch's own completion only (ev_done), on
  // the context's side stream: on the launch stream it would queue behind
  // every forward enqueued since, and the host would drain the pipeline on
  // each fetch.
  cudaStream_t st = g->ctx->side;
  if (!slot) slot = g->last;
  if (!slot || !slot->certified) throw InvalidArgument("nothing certified yet");
  const uint32_t B = slot->B, N = g->N;
  const uint64_t v = g->v;
  const BatchResults& R = slot->res;
  CG_CUDA(cudaStreamWaitEvent(st, slot->ev_done, 0));
  auto d2h = [&](void* dst, const void* src, size_t n) {
    if (dst) CG_CUDA(cudaMemcpyAsync(dst, src, n, cudaMemcpyDeviceToHost, st));
  };
  std::vector<int8_t> status(B);
  uint32_t count[2] = {0, 0};  // manifest entries, single leaves
  d2h(status.data(), R.d_status.p, B);
  d2h(count, R.d_count.p, 8);
  d2h(o->selected, R.d_sel.p, 4 * (size_t)B);
  d2h(o->diameter, R.d_diam.p, 8 * (size_t)B);
  d2h(o->satisfied, R.d_sat.p, B);
  d2h(o->label, R.d_label.p, 8 * (size_t)B);
  d2h(o->r_roots, R.d_rroots.p, 32 * (size_t)N);
  d2h(o->a_root, R.d_aroot.p, 32);
  d2h(o->leaf_hashes, R.d_leaf.p, 32 * (size_t)N * B);
  d2h(o->outputs, R.d_outs.p, 8 * (size_t)N * B * v);
  d2h(o->topk_idx, R.d_topi.p, 4 * (size_t)N * B * g->topk);
  d2h(o->topk_val, R.d_topv.p, 8 * (size_t)N * B * g->topk);
  CG_CUDA(cudaStreamSynchronize(st));
  if (o->manifest_len) *o->manifest_len = count[0];
  d2h(o->manifest_kind, R.d_kinds.p, count[0]);
  d2h(o->manifest_node, R.d_mnodes.p, 4 * (size_t)count[0]);
  d2h(o->manifest_op, R.d_mops.p, 4 * (size_t)count[0]);
  d2h(o->a_leaf_hashes, R.d_aleaf.p, 32 * (size_t)count[0]);
  // a stream that produces single leaves gets its 0x53 request midstates
  // chained speculatively at ingest for the next ring's worth of batches
  if (count[1]) g->spec53 = 2 * (uint32_t)g->slots.size();
  else if (g->spec53) g->spec53--;
  CG_CUDA(cudaStreamSynchronize(st));
  for (uint32_t k = 0; k < B; k++)
    if (status[k] != 0) throw InvalidArgument("select_quorum: invalid argument");
}

// Shared by cg_group_create (all N replicas local) and cg_group_create_dist
// (this rank's replica only; the N providers are the ctx's NCCL ranks).
int create_group(cg_ctx* ctx, cg_model* const* models, uint32_t nlocal, uint32_t N,
                 const uint8_t* all_digests, bool dist, uint32_t f, uint32_t metric,
                 double default_eps, const char* group_id, uint64_t group_id_len,
                 uint64_t version, uint32_t max_batch, uint32_t topk, cg_group** out) {
  return guarded(ctx, [&] {
    *out = nullptr;
    if (N == 0 || N > 20 || f >= N) throw InvalidArgument("bad n/f");
    if (max_batch == 0) throw InvalidArgument("max_batch must be >= 1");
    if (group_id_len > 100) throw InvalidArgument("group id longer than 100 bytes");
    if (topk == 0) topk = 1;
    auto g = std::make_unique<cg_group>();
    g->ctx = ctx;
    g->N = N;
    g->f = f;
    g->metric = metric;
    g->eps_default = default_eps;
    g->gid.assign(group_id, group_id_len);
    g->version = version;
    g->maxB = max_batch;
    g->topk = topk;
    g->dist = dist;
    g->rank = dist ? (uint32_t)ctx->rank : 0;
    g->first = dist ? g->rank * nlocal : 0;
    if (dist && nlocal * (uint32_t)ctx->nranks != N)
      throw InvalidArgument("replica-parallel group: N must be (replicas per rank) x ranks");
    for (uint32_t p = 0; p < nlocal; p++) {
      if (!models[p] || models[p]->ctx != ctx) throw InvalidArgument("bad model");
      g->models.push_back(models[p]);
    }
    for (uint32_t p = 0; p < N; p++) {
      std::array<uint8_t, 32> d;
      std::memcpy(d.data(), dist ? all_digests + 32 * p : models[p]->digest, 32);
      g->digests.push_back(d);
    }
    for (uint32_t li = 0; dist && li < nlocal; li++)
      if (std::memcmp(g->digests[g->first + li].data(), models[li]->digest, 32) != 0)
        throw InvalidArgument("this rank's models are not providers [rank x k, (rank + 1) x k)");
    g->u = models[0]->u;
    g->v = models[0]->v;
    for (auto* m : g->models)
      if (m->u != g->u || m->v != g->v) throw InvalidArgument("models disagree on dimensions");
    if (g->v > 1024) throw InvalidArgument("output dimension > 1024");
    const uint64_t B = max_batch, v = g->v;
    g->d_pre64.ensure(B * v);
    g->d_pre32.ensure((uint64_t)N * B * v);  // per-replica logits (grouped forward)
    const uint64_t amax = (uint64_t)N * B + B + N;  // manifest entries
    g->d_gid.ensure(g->gid.size() + 1);
    CG_CUDA(cudaMemcpy(g->d_gid.p, g->gid.data(), g->gid.size(), cudaMemcpyHostToDevice));
    g->all_cnn = true;
    for (auto* m : g->models) {
      if (m->kind == 1) m->cnn->reserve(max_batch);
      g->all_cnn = g->all_cnn && m->kind == 1;
    }
    // one shared input stage when every replica consumes the same operand
    // (heterogeneous groups: each replica prepares its own)
    g->same_prep = g->all_cnn;
    for (auto* m : g->models)
      g->same_prep = g->same_prep && m->cnn->prep_kind() == g->models[0]->cnn->prep_kind();
    if (g->same_prep) g->d_prep.ensure(g->models[0]->cnn->prepared_bytes(max_batch));
    // ingest ring: enough batches in flight to hide the request-midstate
    // chains (latency ~ request bytes / 64 compressions, ~30 ms for a C2
    // request) behind the forwards of the batches certified meanwhile
    const int depth = kIngestRing;
    const size_t arena_max = (size_t)B * (512 + 160 * N) + 1024;
    for (int i = 0; i < depth; i++) {
      auto S = std::make_unique<IngestSlot>();
      CG_CUDA(cudaStreamCreateWithFlags(&S->stream, cudaStreamNonBlocking));
      CG_CUDA(cudaEventCreateWithFlags(&S->ev_staged, cudaEventDisableTiming));
      CG_CUDA(cudaEventCreateWithFlags(&S->ev_prefix, cudaEventDisableTiming));
      CG_CUDA(cudaEventCreateWithFlags(&S->ev_done, cudaEventDisableTiming));
      S->d_eps.ensure(B);
      S->d_arena.ensure(arena_max);
      S->d_reqids.ensure(32 * B);
      S->d_jobs.ensure(B * (4 + 2 * N + 2 * nlocal));
      S->d_mid.ensure(8 * B);
      S->d_mid53.ensure(8 * B);
      S->d_tree.ensure(2 * N);
      S->h_arena.ensure(arena_max);
      S->h_reqids.ensure(32 * B);
      S->h_jobs.ensure(B * (4 + 2 * N + 2 * nlocal));
      S->h_eps.ensure(B);
      S->h_tree.ensure(2 * N);
      CG_CUDA(cudaEventCreateWithFlags(&S->ev_fwd, cudaEventDisableTiming));
      CG_CUDA(cudaEventCreateWithFlags(&S->ev_man, cudaEventDisableTiming));
      S->res.d_outs.ensure((uint64_t)N * B * v);
      S->res.d_topi.ensure((uint64_t)N * B * topk);
      S->res.d_topv.ensure((uint64_t)N * B * topk);
      S->res.d_diam.ensure(B);
      S->res.d_sel.ensure(B);
      S->res.d_mnodes.ensure(amax);
      S->res.d_mops.ensure(amax);
      S->res.d_kinds.ensure(amax);
      S->res.d_count.ensure(2);
      S->res.d_leaf.ensure(32 * (uint64_t)N * B);
      S->res.d_rroots.ensure(32 * (uint64_t)N);
      S->res.d_aleaf.ensure(32 * amax);
      S->res.d_aroot.ensure(32);
      S->res.d_sat.ensure(B);
      S->res.d_status.ensure(B);
      S->res.d_label.ensure(B);
      S->res.d_single_pos.ensure((uint64_t)N * B);
      S->res.d_need53.ensure(B);
      g->slots.push_back(std::move(S));
    }
    ctx->groups.push_back(g.get());
    *out = g.release();
    return CG_OK;
  });
}

}  // namespace cg

extern "C" {

int cg_group_create(cg_ctx* ctx, cg_model* const* models, uint32_t N,
                    uint32_t f, uint32_t metric, double default_eps,
                    const char* group_id, uint64_t group_id_len,
                    uint64_t version, uint32_t max_batch, uint32_t topk,
                    cg_group** out) {
  return create_group(ctx, models, N, N, nullptr, false, f, metric, default_eps, group_id,
                      group_id_len, version, max_batch, topk, out);
}

int cg_group_create_dist(cg_ctx* ctx, cg_model* my_model, const uint8_t* all_digests,
                         uint32_t f, uint32_t metric, double default_eps,
                         const char* group_id, uint64_t group_id_len, uint64_t version,
                         uint32_t max_batch, uint32_t topk, cg_group** out) {
  if (!ctx || !ctx->comm) return fail(ctx, CG_EINVAL, "cg_ctx_init_nccl first");
  return create_group(ctx, &my_model, 1, (uint32_t)ctx->nranks, all_digests, true, f, metric,
                      default_eps, group_id, group_id_len, version, max_batch, topk, out);
}

int cg_group_create_dist_multi(cg_ctx* ctx, cg_model* const* my_models, uint32_t nlocal,
                               const uint8_t* all_digests, uint32_t f, uint32_t metric,
                               double default_eps, const char* group_id, uint64_t group_id_len,
                               uint64_t version, uint32_t max_batch, uint32_t topk,
                               cg_group** out) {
  if (!ctx || !ctx->comm) return fail(ctx, CG_EINVAL, "cg_ctx_init_nccl first");
  if (nlocal == 0 || !my_models) return fail(ctx, CG_EINVAL, "no local models");
  return create_group(ctx, my_models, nlocal, nlocal * (uint32_t)ctx->nranks, all_digests, true,
                      f, metric, default_eps, group_id, group_id_len, version, max_batch, topk,
                      out);
}

}  // extern "C"

namespace {
void encode_results_slot(cg_group* g, const IngestSlot* S, uint32_t provider, uint8_t* out,
                         uint64_t cap, uint64_t* len) {
  if (!S || !S->certified) throw InvalidArgument("nothing certified yet");
  if (provider >= g->N) throw InvalidArgument("provider index >= N");
  const uint32_t B = S->B, gl = (uint32_t)g->gid.size();
  const uint64_t v = g->v;
  const uint64_t need = 4 + (uint64_t)B * (88 + gl + 8 * v);
  *len = need;
  if (!out) return;  // size query
  if (cap < need) throw InvalidArgument("output buffer too small");
  cudaStream_t st = g->ctx->stream;
  CG_CUDA(cudaStreamWaitEvent(st, S->ev_done, 0));
  g->ctx->d_bytes.ensure(need);
  Digest32 dg;
  std::memcpy(dg.b, g->digests[provider].data(), 32);
  launch_encode_results(S->d_reqids.p, S->res.d_outs.p + (uint64_t)provider * B * v, B,
                        (uint32_t)v, provider, g->d_gid.p, gl, g->version, dg, g->ctx->d_bytes.p,
                        st);
  CG_CUDA(cudaMemcpyAsync(out, g->ctx->d_bytes.p, need, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

extern "C" {

int cg_group_encode_results(cg_group* g, uint32_t provider, uint8_t* out, uint64_t cap,
                            uint64_t* len) {
  if (!g || !len) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    encode_results_slot(g, g->last, provider, out, cap, len);
    return CG_OK;
  });
}

int cg_group_encode_results_ticket(cg_group* g, uint64_t ticket, uint32_t provider,
                                   uint8_t* out, uint64_t cap, uint64_t* len) {
  if (!g || !len) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    encode_results_slot(g, &certified_slot(g, ticket), provider, out, cap, len);
    return CG_OK;
  });
}

int cg_group_set_perturbation(cg_group* g, double magnitude) {
  if (!g) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    if (!(magnitude >= 0.0)) throw InvalidArgument("negative magnitude");
    for (auto& sl : g->slots)
      if (sl->used) throw InvalidArgument("set the perturbation with no batch ingested ahead");
    cudaStream_t st = g->ctx->stream;
    CG_CUDA(cudaStreamSynchronize(st));  // no certify in flight reads the header
    for (auto& sl : g->slots) CG_CUDA(cudaStreamSynchronize(sl->stream));
    const uint32_t nloc = (uint32_t)g->models.size();
    g->d_phdr.ensure(64ull * nloc);
    std::vector<uint8_t> h(64ull * nloc, 0);
    for (uint32_t li = 0; li < nloc; li++) {
      const uint64_t p = g->first + li;
      uint8_t* b = h.data() + 64ull * li;
      for (int i = 0; i < 8; i++) b[i] = (uint8_t)(p >> (56 - 8 * i));
      std::memcpy(b + 8, g->digests[p].data(), 32);
      for (int i = 0; i < 4; i++) b[40 + i] = (uint8_t)((uint32_t)g->u >> (24 - 8 * i));
    }
    CG_CUDA(cudaMemcpy(g->d_phdr.p, h.data(), h.size(), cudaMemcpyHostToDevice));
    g->perturb_mag = magnitude;
    return CG_OK;
  });
}

int cg_group_set_fault(cg_group* g, uint32_t provider, double offset, double fraction) {
  if (!g) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    if (provider >= g->N) throw InvalidArgument("provider index >= N");
    if (!(fraction >= 0.0 && fraction <= 1.0)) throw InvalidArgument("fraction outside [0, 1]");
    if (!std::isfinite(offset)) throw InvalidArgument("offset must be finite");
    g->fault_provider = provider;
    g->fault_offset = offset;
    g->fault_thr = offset == 0.0 ? 0u : (uint32_t)std::lround(256.0 * fraction);
    return CG_OK;
  });
}

void cg_group_free(cg_group* g) {
  if (!g) return;
  {
    std::lock_guard<std::mutex> lk(g->ctx->mu);
    auto& v = g->ctx->groups;
    v.erase(std::remove(v.begin(), v.end(), g), v.end());
  }
  cudaSetDevice(g->ctx->device);
  cudaStreamSynchronize(g->ctx->stream);
  if (g->ctx->tail) cudaStreamSynchronize(g->ctx->tail);
  for (auto& s : g->slots) cudaStreamSynchronize(s->stream);
  for (cudaStream_t s2 : g->rstreams) {
    cudaStreamSynchronize(s2);
    cudaStreamDestroy(s2);
  }
  for (cudaEvent_t e : g->revs) cudaEventDestroy(e);
  delete g;
}

// verify_request's digests for a batch (domain.cpp:177-216): signing digest
// SHA-256(0x01 || body) -- one 1.2 MB chain per ImageNet request, streamed
// from the f64 input like the result leaves -- and canonical_request_id
// SHA-256(pub || 0x1F || nonce), plus the structural checks. The Ed25519
// check over the digest is the caller's (host) step.
int cg_request_digests(cg_ctx* ctx, const cg_request_batch* bt, const char* group_id,
                       uint64_t group_id_len, uint8_t* signing_digests, uint8_t* canonical_ids,
                       int8_t* status) {
  if (!ctx || !bt) return CG_EINVAL;
  return guarded(ctx, [&] {
    const uint32_t B = bt->B;
    const uint64_t u = bt->u;
    if (B == 0) return CG_OK;
    cudaStream_t st = ctx->stream;
    const double* d_in = bt->inputs;
    if (!bt->inputs_on_device) {
      ctx->d_f64.ensure((size_t)B * u);
      CG_CUDA(cudaMemcpyAsync(ctx->d_f64.p, bt->inputs, 8 * (size_t)B * u,
                              cudaMemcpyHostToDevice, st));
      d_in = ctx->d_f64.p;
    }
    Arena ar;
    struct L {
      size_t h, t, id;
      uint64_t lh, lt, lid;
    };
    std::vector<L> lay(B);
    uint64_t nonce_pos = 0;
    for (uint32_t k = 0; k < B; k++) {
      const uint8_t* nonce = bt->nonces + nonce_pos;
      const uint64_t nl = bt->nonce_lens[k];
      nonce_pos += nl;
      Enc H;  // kRequestSigTag || encode_request_body up to the input list
      H.u8(0x01);
      H.raw(bt->request_ids + 32 * k, 32);
      H.bytes((const uint8_t*)group_id, group_id_len);
      H.u32((uint32_t)u);
      Enc T;
      const bool he = bt->has_eps && bt->has_eps[k];
      T.u8(he ? 1 : 0);
      if (he) T.f64(bt->eps[k]);
      T.raw(bt->client_pubs + 32 * k, 32);
      T.bytes(nonce, nl);
      Enc I;  // canonical_request_id preimage
      I.raw(bt->client_pubs + 32 * k, 32);
      I.u8(0x1F);
      I.raw(nonce, nl);
      L& l = lay[k];
      l.lh = H.b.size();
      l.lt = T.b.size();
      l.lid = I.b.size();
      l.h = ar.add(H.b.data(), l.lh, 0);
      l.t = ar.add(T.b.data(), l.lt, l.lh + 8 * u);
      l.id = ar.add(I.b.data(), l.lid, 0);
      if (status) {
        int8_t s8 = 0;
        if (nl == 0) s8 = 1;
        else if (u == 0) s8 = 2;
        else if (he && !(bt->eps[k] >= 0.0 && std::isfinite(bt->eps[k]))) s8 = 3;
        status[k] = s8;
      }
    }
    ctx->d_bytes.ensure(ar.b.size() + 16);
    ctx->d_out.ensure(64 * (size_t)B);
    ctx->d_jobs.ensure(2 * (size_t)B);
    std::vector<ChainJob> jobs(2 * (size_t)B);
    const uint64_t A = (uint64_t)ctx->d_bytes.p;
    for (uint32_t k = 0; k < B; k++) {
      const L& l = lay[k];
      ChainJob& j = jobs[k];
      std::memset(&j, 0, sizeof j);
      j.seg[0] = ChainSeg{A + l.h, 0, l.lh, kSegRaw, 0};
      j.seg[1] = ChainSeg{(uint64_t)(d_in + u * k), l.lh, 8 * u, kSegF64, 0};
      j.seg[2] = ChainSeg{A + l.t, l.lh + 8 * u, l.lt, kSegRaw, 0};
      j.nseg = 3;
      j.final_ = 1;
      j.total_len = l.lh + 8 * u + l.lt;
      j.blk_end = (j.total_len + 9 + 63) / 64;
      j.digest_out = (uint64_t)(ctx->d_out.p + 32 * k);
      ChainJob& c = jobs[B + k];
      std::memset(&c, 0, sizeof c);
      c.seg[0] = ChainSeg{A + l.id, 0, l.lid, kSegRaw, 0};
      c.nseg = 1;
      c.final_ = 1;
      c.total_len = l.lid;
      c.blk_end = (l.lid + 9 + 63) / 64;
      c.digest_out = (uint64_t)(ctx->d_out.p + 32 * ((size_t)B + k));
    }
    CG_CUDA(cudaMemcpyAsync(ctx->d_bytes.p, ar.b.data(), ar.b.size(), cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(ctx->d_jobs.p, jobs.data(), jobs.size() * sizeof(ChainJob),
                            cudaMemcpyHostToDevice, st));
    launch_chain_jobs(ctx->d_jobs.p, 2 * B, st);
    std::vector<uint8_t> dig(64 * (size_t)B);
    CG_CUDA(cudaMemcpyAsync(dig.data(), ctx->d_out.p, dig.size(), cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    if (signing_digests) std::memcpy(signing_digests, dig.data(), 32 * (size_t)B);
    if (canonical_ids) std::memcpy(canonical_ids, dig.data() + 32 * (size_t)B, 32 * (size_t)B);
    if (status)
      for (uint32_t k = 0; k < B; k++)
        if (status[k] == 0 &&
            std::memcmp(dig.data() + 32 * ((size_t)B + k), bt->request_ids + 32 * k, 32) != 0)
          status[k] = 4;
    return CG_OK;
  });
}

// ------------------------------------------- certificate leaf hashes (verify)
// The leaves a verifier re-hashes (verify_cert, certificate.cpp:235-275) and a
// proxy re-hashes when it rebuilds committer and result trees (proxy.cpp:
// 28-48, :134-141): result_leaf 0x52 / single_attest_leaf 0x53 =
// 0x00 || tag || request || result and missing_result_leaf 0x4D =
// 0x00 || 0x4D || request (messages.cpp:204-218, :283-290). The request part
// is streamed from the f64 input tensor; its whole blocks are hashed once
// per (request, tag) into a midstate that every result of the request
// continues from.
int cg_cert_leaf_hashes(cg_ctx* ctx, const cg_request_batch* bt, const char* group_id,
                        uint64_t group_id_len, uint32_t M, const uint32_t* req_index,
                        const uint8_t* want, const uint8_t* result_enc,
                        const uint64_t* result_lens, uint8_t* leaf52, uint8_t* leaf53,
                        uint8_t* leaf4d) {
  if (!ctx || !bt || (M && (!req_index || !want))) return CG_EINVAL;
  return guarded(ctx, [&] {
    const uint32_t B = bt->B;
    const uint64_t u = bt->u;
    if (M == 0) return CG_OK;
    if (bt->input_dims || bt->op_kinds)
      throw InvalidArgument("cg_cert_leaf_hashes: one input length per batch, request ops only");
    // which (request, tag) prefixes are needed; result byte offsets
    std::vector<uint8_t> need(3 * (size_t)B, 0);  // [tag 0x52 | 0x53 | 0x4D][k]
    std::vector<uint64_t> roff(M);
    uint64_t rpos = 0;
    for (uint32_t m = 0; m < M; m++) {
      const uint32_t k = req_index[m], w = want[m];
      if (k >= B) throw InvalidArgument("cg_cert_leaf_hashes: request index out of range");
      if (w & ~7u) throw InvalidArgument("cg_cert_leaf_hashes: want is a mask of 1 | 2 | 4");
      if (((w & 1) && !leaf52) || ((w & 2) && !leaf53) || ((w & 4) && !leaf4d))
        throw InvalidArgument("cg_cert_leaf_hashes: output for a requested leaf kind is NULL");
      if ((w & 3) && (!result_enc || !result_lens))
        throw InvalidArgument("cg_cert_leaf_hashes: result leaves need result encodings");
      for (int t = 0; t < 3; t++)
        if (w & (1u << t)) need[(size_t)t * B + k] = 1;
      roff[m] = rpos;
      if (result_lens) rpos += result_lens[m];
    }
    cudaStream_t st = ctx->stream;
    const double* d_in = bt->inputs;
    if (!bt->inputs_on_device) {
      ctx->d_f64.ensure((size_t)B * u);
      CG_CUDA(cudaMemcpyAsync(ctx->d_f64.p, bt->inputs, 8 * (size_t)B * u,
                              cudaMemcpyHostToDevice, st));
      d_in = ctx->d_f64.p;
    }
    static const uint8_t kTag[3] = {0x52, 0x53, 0x4D};
    Arena ar;
    std::vector<size_t> h(3 * (size_t)B), t(B);
    std::vector<uint64_t> P(B);
    uint64_t lenH = 0, nonce_pos = 0;
    for (uint32_t k = 0; k < B; k++) {
      Enc H;  // 0x00 || tag || request body up to the input list (domain.cpp:144-158)
      H.u8(0x00);
      H.u8(0x52);
      H.raw(bt->request_ids + 32 * k, 32);
      H.bytes((const uint8_t*)group_id, group_id_len);
      H.u32((uint32_t)u);
      Enc T;
      const bool he = bt->has_eps && bt->has_eps[k];
      T.u8(he ? 1 : 0);
      if (he) T.f64(bt->eps[k]);
      T.raw(bt->client_pubs + 32 * k, 32);
      T.bytes(bt->nonces + nonce_pos, bt->nonce_lens[k]);
      nonce_pos += bt->nonce_lens[k];
      T.raw(bt->client_sigs + 64 * k, 64);
      lenH = H.b.size();
      P[k] = lenH + 8 * u + T.b.size();
      for (int tg = 0; tg < 3; tg++)
        if (need[(size_t)tg * B + k]) {
          H.b[1] = kTag[tg];
          h[(size_t)tg * B + k] = ar.add(H.b.data(), lenH, 0);
        }
      t[k] = ar.add(T.b.data(), T.b.size(), lenH + 8 * u);
    }
    std::vector<size_t> rar(M, 0);
    for (uint32_t m = 0; m < M; m++)
      if ((want[m] & 3) && result_lens[m])
        rar[m] = ar.add(result_enc + roff[m], result_lens[m], P[req_index[m]]);
    // device scratch: digests [0x52: M][0x53: M][0x4D: B], midstates [2][B]
    const size_t dig_bytes = 32 * (2 * (size_t)M + B);
    ctx->d_out.ensure(dig_bytes + 64 * (size_t)B);
    ctx->d_bytes.ensure(ar.b.size() + 16);
    uint8_t* d_dig = ctx->d_out.p;
    uint32_t* d_mid = (uint32_t*)(ctx->d_out.p + dig_bytes);
    const uint64_t A = (uint64_t)ctx->d_bytes.p;
    auto prefix = [&](ChainJob& j, int tg, uint32_t k) {
      std::memset(&j, 0, sizeof j);
      j.seg[0] = ChainSeg{A + h[(size_t)tg * B + k], 0, lenH, kSegRaw, 0};
      j.seg[1] = ChainSeg{(uint64_t)(d_in + u * k), lenH, 8 * u, kSegF64, 0};
      j.seg[2] = ChainSeg{A + t[k], lenH + 8 * u, P[k] - lenH - 8 * u, kSegRaw, 0};
      j.nseg = 3;
      j.total_len = P[k];
    };
    std::vector<ChainJob> mids, fins;
    for (uint32_t k = 0; k < B; k++) {
      for (int tg = 0; tg < 2; tg++)
        if (need[(size_t)tg * B + k] && P[k] >= 64) {
          ChainJob j;
          prefix(j, tg, k);
          j.blk_end = P[k] / 64;
          j.state_out = (uint64_t)(d_mid + 8 * ((size_t)tg * B + k));
          mids.push_back(j);
        }
      if (need[2 * (size_t)B + k]) {  // missing_result_leaf: the request alone
        ChainJob j;
        prefix(j, 2, k);
        j.final_ = 1;
        j.blk_end = (P[k] + 9 + 63) / 64;
        j.digest_out = (uint64_t)(d_dig + 32 * (2 * (size_t)M + k));
        fins.push_back(j);
      }
    }
    for (uint32_t m = 0; m < M; m++)
      for (int tg = 0; tg < 2; tg++) {
        if (!(want[m] & (1u << tg))) continue;
        const uint32_t k = req_index[m];
        ChainJob j;
        prefix(j, tg, k);
        j.seg[3] = ChainSeg{A + rar[m], P[k], result_lens[m], kSegRaw, 0};
        j.nseg = 4;
        j.final_ = 1;
        j.total_len = P[k] + result_lens[m];
        j.blk_begin = P[k] / 64;
        j.blk_end = (j.total_len + 9 + 63) / 64;
        j.state_in = j.blk_begin ? (uint64_t)(d_mid + 8 * ((size_t)tg * B + k)) : 0;
        j.digest_out = (uint64_t)(d_dig + 32 * ((size_t)tg * M + m));
        fins.push_back(j);
      }
    ctx->d_jobs.ensure(mids.size() + fins.size());
    CG_CUDA(cudaMemcpyAsync(ctx->d_bytes.p, ar.b.data(), ar.b.size(), cudaMemcpyHostToDevice, st));
    if (!mids.empty())
      CG_CUDA(cudaMemcpyAsync(ctx->d_jobs.p, mids.data(), mids.size() * sizeof(ChainJob),
                              cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(ctx->d_jobs.p + mids.size(), fins.data(),
                            fins.size() * sizeof(ChainJob), cudaMemcpyHostToDevice, st));
    if (!mids.empty()) launch_chain_jobs(ctx->d_jobs.p, (uint32_t)mids.size(), st);
    launch_chain_jobs(ctx->d_jobs.p + mids.size(), (uint32_t)fins.size(), st);
    std::vector<uint8_t> dig(dig_bytes);
    CG_CUDA(cudaMemcpyAsync(dig.data(), d_dig, dig_bytes, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    for (uint32_t m = 0; m < M; m++) {
      if (want[m] & 1) std::memcpy(leaf52 + 32 * (size_t)m, &dig[32 * (size_t)m], 32);
      if (want[m] & 2) std::memcpy(leaf53 + 32 * (size_t)m, &dig[32 * ((size_t)M + m)], 32);
      if (want[m] & 4)
        std::memcpy(leaf4d + 32 * (size_t)m, &dig[32 * (2 * (size_t)M + req_index[m])], 32);
    }
    return CG_OK;
  });
}

// ---------------------------------------------------- authentication paths
namespace {
void auth_paths_device(cg_ctx* ctx, const uint8_t* d_leaves, uint64_t n, const uint64_t* indices,
                       uint32_t count, uint8_t* siblings, uint8_t* sides, uint32_t* lens,
                       uint8_t* root) {
  if (n == 0) throw InvalidArgument("merkle: empty leaf list");
  for (uint32_t i = 0; i < count; i++)
    if (indices[i] >= n) throw InvalidArgument("merkle: leaf index out of range");
  cudaStream_t st = ctx->stream;
  DevBuf<uint8_t> levels, sib, sd;
  DevBuf<uint64_t> idx;
  DevBuf<uint32_t> ln;
  levels.ensure(32 * merkle_levels_nodes(n));
  const auto off = launch_merkle_levels(d_leaves, n, levels.p, st);
  idx.ensure(count);
  sib.ensure((size_t)count * kMaxPathSteps * 32);
  sd.ensure((size_t)count * kMaxPathSteps);
  ln.ensure(count);
  if (count) {
    CG_CUDA(cudaMemcpyAsync(idx.p, indices, 8 * (size_t)count, cudaMemcpyHostToDevice, st));
    launch_auth_paths(levels.p, off, n, idx.p, count, sib.p, sd.p, ln.p, st);
    CG_CUDA(cudaMemcpyAsync(siblings, sib.p, (size_t)count * kMaxPathSteps * 32,
                            cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaMemcpyAsync(sides, sd.p, (size_t)count * kMaxPathSteps, cudaMemcpyDeviceToHost,
                            st));
    CG_CUDA(cudaMemcpyAsync(lens, ln.p, 4 * (size_t)count, cudaMemcpyDeviceToHost, st));
  }
  if (root)
    CG_CUDA(cudaMemcpyAsync(root, levels.p + 32 * off.back(), 32, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
}
}  // namespace

int cg_merkle_auth_paths(cg_ctx* ctx, const uint8_t* leaf_hashes, uint64_t n,
                         const uint64_t* indices, uint32_t count, uint8_t* siblings,
                         uint8_t* sides, uint32_t* lens, uint8_t* root) {
  return guarded(ctx, [&] {
    DevBuf<uint8_t> leaves;
    leaves.ensure(32 * std::max<uint64_t>(n, 1));
    CG_CUDA(cudaMemcpyAsync(leaves.p, leaf_hashes, 32 * n, cudaMemcpyHostToDevice, ctx->stream));
    auth_paths_device(ctx, leaves.p, n, indices, count, siblings, sides, lens, root);
    return CG_OK;
  });
}

int cg_merkle_path_roots(cg_ctx* ctx, const uint8_t* leaf_hashes, const uint8_t* siblings,
                         const uint8_t* sides, const uint32_t* lens, uint32_t count,
                         uint8_t* roots) {
  return guarded(ctx, [&] {
    if (count == 0) return CG_OK;
    for (uint32_t i = 0; i < count; i++)
      if (lens[i] > (uint32_t)kMaxPathSteps) throw InvalidArgument("merkle: path too long");
    cudaStream_t st = ctx->stream;
    DevBuf<uint8_t> lh, sib, sd, out;
    DevBuf<uint32_t> ln;
    lh.ensure(32 * (size_t)count);
    sib.ensure((size_t)count * kMaxPathSteps * 32);
    sd.ensure((size_t)count * kMaxPathSteps);
    ln.ensure(count);
    out.ensure(32 * (size_t)count);
    CG_CUDA(cudaMemcpyAsync(lh.p, leaf_hashes, 32 * (size_t)count, cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(sib.p, siblings, (size_t)count * kMaxPathSteps * 32,
                            cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(sd.p, sides, (size_t)count * kMaxPathSteps, cudaMemcpyHostToDevice, st));
    CG_CUDA(cudaMemcpyAsync(ln.p, lens, 4 * (size_t)count, cudaMemcpyHostToDevice, st));
    launch_path_roots(lh.p, sib.p, sd.p, ln.p, count, out.p, st);
    CG_CUDA(cudaMemcpyAsync(roots, out.p, 32 * (size_t)count, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    return CG_OK;
  });
}

}  // extern "C"

namespace {
void group_auth_paths(cg_group* g, const IngestSlot* S, uint32_t tree, const uint64_t* indices,
                      uint32_t count, uint8_t* siblings, uint8_t* sides, uint32_t* lens) {
  if (!S || !S->certified) throw InvalidArgument("nothing certified yet");
  const uint32_t B = S->B, N = g->N;
  if (tree > N) throw InvalidArgument("tree index out of range");
  if (g->dist && tree < N && (tree < g->first || tree >= g->first + g->models.size()))
    throw InvalidArgument("replica-parallel group: only this rank's result tree is local");
  const uint8_t* leaves;
  uint64_t n;
  const BatchResults& R = S->res;
  CG_CUDA(cudaStreamWaitEvent(g->ctx->stream, S->ev_done, 0));
  if (tree < N) {  // provider `tree`'s R tree: its B result leaves
    leaves = R.d_leaf.p + 32 * (uint64_t)tree * B;
    n = B;
  } else {  // the attestation tree, manifest order
    uint32_t cnt = 0;
    CG_CUDA(cudaMemcpyAsync(&cnt, R.d_count.p, 4, cudaMemcpyDeviceToHost, g->ctx->stream));
    CG_CUDA(cudaStreamSynchronize(g->ctx->stream));
    leaves = R.d_aleaf.p;
    n = cnt;
  }
  auth_paths_device(g->ctx, leaves, n, indices, count, siblings, sides, lens, nullptr);
}
}  // namespace

extern "C" {

int cg_group_auth_paths(cg_group* g, uint32_t tree, const uint64_t* indices, uint32_t count,
                        uint8_t* siblings, uint8_t* sides, uint32_t* lens) {
  if (!g) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    group_auth_paths(g, g->last, tree, indices, count, siblings, sides, lens);
    return CG_OK;
  });
}

int cg_group_auth_paths_ticket(cg_group* g, uint64_t ticket, uint32_t tree,
                               const uint64_t* indices, uint32_t count, uint8_t* siblings,
                               uint8_t* sides, uint32_t* lens) {
  if (!g) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    group_auth_paths(g, &certified_slot(g, ticket), tree, indices, count, siblings, sides, lens);
    return CG_OK;
  });
}

int cg_ingest_batch(cg_group* g, const cg_request_batch* batch, uint64_t* ticket) {
  if (!g || !batch || !ticket) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    *ticket = ingest(g, batch);
    return CG_OK;
  });
}

int cg_certify_ticket(cg_group* g, uint64_t ticket, cg_certify_out* out) {
  if (!g) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    certify(g, ticket, nullptr);
    if (out) certify_fetch(g, out);
    return CG_OK;
  });
}

int cg_certify_batch(cg_group* g, const cg_request_batch* batch,
                     cg_certify_out* out) {
  if (!g || !batch) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    certify(g, ingest(g, batch), nullptr);
    if (out) certify_fetch(g, out);
    return CG_OK;
  });
}

int cg_certify_outputs(cg_group* g, const cg_request_batch* batch,
                       const double* outputs, cg_certify_out* out) {
  if (!g || !batch || !outputs) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    certify(g, ingest(g, batch), outputs);
    if (out) certify_fetch(g, out);
    return CG_OK;
  });
}

int cg_group_fetch(cg_group* g, cg_certify_out* out) {
  if (!g || !out) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    certify_fetch(g, out);
    return CG_OK;
  });
}

// An empty filler slot (messages.cpp:240-243, coordinator.cpp:776-787):
// R tree = [noop_leaf(view, seq)] for every provider; no outcomes, so every
// provider is whole-batch attested. The four SHA-256 messages run on the
// device like every other digest.
int cg_certify_empty_slot(cg_group* g, uint64_t view, uint64_t seq, cg_certify_out* o) {
  if (!g || !o) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    cg_ctx* ctx = g->ctx;
    const uint32_t N = g->N;
    uint8_t noop[17];
    noop[0] = 0x4E;  // kLeafNoop || u64be view || u64be seq (messages.cpp:227-233)
    for (int i = 0; i < 8; i++) {
      noop[1 + i] = (uint8_t)(view >> (56 - 8 * i));
      noop[9 + i] = (uint8_t)(seq >> (56 - 8 * i));
    }
    uint64_t off = 0, len = 17;
    uint8_t rroot[32], whole[33], aleaf[32];
    device_sha256_many(ctx, noop, &off, &len, 1, 0x00, rroot);  // one-leaf tree: root = leaf hash
    whole[0] = 0x57;  // whole_batch_leaf(R root) (messages.cpp:276-280)
    std::memcpy(whole + 1, rroot, 32);
    len = 33;
    device_sha256_many(ctx, whole, &off, &len, 1, 0x00, aleaf);
    std::vector<uint8_t> leaves(32 * (size_t)N);
    for (uint32_t p = 0; p < N; p++) std::memcpy(leaves.data() + 32 * p, aleaf, 32);
    ctx->d_bytes.ensure(leaves.size());
    ctx->d_out.ensure(32);
    CG_CUDA(cudaMemcpyAsync(ctx->d_bytes.p, leaves.data(), leaves.size(), cudaMemcpyHostToDevice,
                            ctx->stream));
    launch_merkle_trees(ctx->d_bytes.p, nullptr, nullptr, nullptr, 1, N, ctx->d_out.p, ctx->stream,
                        N);
    uint8_t aroot[32];
    CG_CUDA(cudaMemcpyAsync(aroot, ctx->d_out.p, 32, cudaMemcpyDeviceToHost, ctx->stream));
    CG_CUDA(cudaStreamSynchronize(ctx->stream));
    if (o->r_roots)
      for (uint32_t p = 0; p < N; p++) std::memcpy(o->r_roots + 32 * p, rroot, 32);
    if (o->a_root) std::memcpy(o->a_root, aroot, 32);
    if (o->manifest_len) *o->manifest_len = N;
    for (uint32_t p = 0; p < N; p++) {
      if (o->manifest_kind) o->manifest_kind[p] = 0;
      if (o->manifest_node) o->manifest_node[p] = p;
      if (o->manifest_op) o->manifest_op[p] = 0;
      if (o->a_leaf_hashes) std::memcpy(o->a_leaf_hashes + 32 * p, aleaf, 32);
    }
    return CG_OK;
  });
}

int cg_group_fetch_ticket(cg_group* g, uint64_t ticket, cg_certify_out* out) {
  if (!g || !out) return CG_EINVAL;
  return guarded(g->ctx, [&] {
    certify_fetch(g, out, &certified_slot(g, ticket));
    return CG_OK;
  });
}

}  // extern "C"
