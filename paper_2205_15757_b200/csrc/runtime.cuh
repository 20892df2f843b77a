// Host-side runtime behind the C-ABI (include/credo_gpu.h): contexts, device
// and pinned buffers, model residency, the per-group ingest ring and its
// per-batch results. Internal to the library (capi.cu, engine.cu).
#pragma once
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <array>
#include <cstring>
#include <memory>
#include <mutex>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/credo_gpu.h"
#include "cnn.cuh"
#include "common.cuh"
#include "digest.cuh"

namespace cg {

struct CodecError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct DigestError : std::runtime_error {
  using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------- buffers
template <typename T>
struct DevBuf {
  T* p = nullptr;
  size_t n = 0;
  DevBuf() = default;
  DevBuf(const DevBuf&) = delete;
  DevBuf& operator=(const DevBuf&) = delete;
  ~DevBuf() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    n = 0;
  }
  void ensure(size_t count) {
    if (count <= n) return;
    release();
    CG_CUDA(cudaMalloc(&p, std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
};

template <typename T>
struct PinBuf {
  T* p = nullptr;
  size_t n = 0;
  ~PinBuf() {
    if (p) cudaFreeHost(p);
  }
  void ensure(size_t count) {
    if (count <= n) return;
    if (p) cudaFreeHost(p);
    p = nullptr;
    CG_CUDA(cudaMallocHost(&p, std::max<size_t>(count, 1) * sizeof(T)));
    n = count;
  }
};

// ------------------------------------------------------ canonical bytes
// codec.hpp:28-84: u64 BE, u32 BE length prefixes, bool byte, raw fixed.
struct Enc {
  std::vector<uint8_t> b;
  void u8(uint8_t v) { b.push_back(v); }
  void u32(uint32_t v) {
    for (int s = 24; s >= 0; s -= 8) b.push_back((uint8_t)(v >> s));
  }
  void u64(uint64_t v) {
    for (int s = 56; s >= 0; s -= 8) b.push_back((uint8_t)(v >> s));
  }
  void f64(double d) {
    uint64_t v;
    std::memcpy(&v, &d, 8);
    u64(v);
  }
  void raw(const uint8_t* p, size_t n) { b.insert(b.end(), p, p + n); }
  void bytes(const uint8_t* p, size_t n) {
    u32((uint32_t)n);
    raw(p, n);
  }
};

// Host arena for the framing bytes of chain jobs. A raw segment is placed
// at an arena offset congruent to its message offset mod 4 so that every
// whole message word inside it is one aligned 32-bit load on the device.
struct Arena {
  std::vector<uint8_t> b;
  size_t add(const uint8_t* p, size_t n, uint64_t msg_off) {
    while ((b.size() & 3) != (msg_off & 3)) b.push_back(0);
    size_t o = b.size();
    b.insert(b.end(), p, p + n);
    return o;
  }
};

}  // namespace cg

using namespace cg;

constexpr int kIngestRing = CG_INGEST_RING;

// ------------------------------------------------------------------ ctx
struct cg_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  bool own_stream = true;
  cudaStream_t side = nullptr;  // result readback (certify_fetch): waits on one batch only
  cudaEvent_t ev_a = nullptr, ev_b = nullptr;
  std::string err;
  std::mutex mu;
  // scratch for the standalone digest / agreement entry points
  DevBuf<uint8_t> d_bytes, d_out;
  DevBuf<ChainJob> d_jobs;
  DevBuf<double> d_f64;
  DevBuf<uint32_t> d_u32a, d_u32b;
  DevBuf<uint64_t> d_u64a, d_u64b;
  DevBuf<uint8_t> d_u8;
  DevBuf<int8_t> d_i8;
  DevBuf<int64_t> d_i64;
  DevBuf<double> d_f64b;
  // replica-parallel groups: one NCCL communicator over the ranks (one per GPU)
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;
  // certification tails (result leaves, agreement, trees) of every group of
  // this context, in issue order: they overlap the next batch's forwards,
  // and one stream keeps the NCCL exchanges in the same order on all ranks
  cudaStream_t tail = nullptr;
  // groups created on this context (cg_ctx_join drains their slot streams)
  std::vector<cg_group*> groups;
  std::atomic<uint64_t> launches{0};  // kernels launched by this context's calls
};

struct cg_model {
  cg_ctx* ctx = nullptr;
  int kind = 0;  // 0 linear, 1 cnn
  uint64_t u = 0, v = 0;
  bool softmax = false;
  uint8_t digest[32];
  DevBuf<double> W, b;          // linear
  std::unique_ptr<CnnModel> cnn;  // cnn
};

namespace cg {

inline int fail(cg_ctx* ctx, int code, const std::string& msg) {
  if (ctx) ctx->err = msg;
  return code;
}

// The launch counter of the context whose entry point runs on this thread
// (launch_counter_add credits it); set for the duration of a guarded call.
extern thread_local std::atomic<uint64_t>* tl_ctx_launches;
struct LaunchScope {
  std::atomic<uint64_t>* prev;
  explicit LaunchScope(std::atomic<uint64_t>* c) : prev(tl_ctx_launches) { tl_ctx_launches = c; }
  ~LaunchScope() { tl_ctx_launches = prev; }
};

template <typename Fn>
int guarded(cg_ctx* ctx, Fn&& fn) {
  if (!ctx) return CG_EINVAL;
  try {
    std::lock_guard<std::mutex> lk(ctx->mu);
    LaunchScope scope(&ctx->launches);
    ctx->err.clear();
    CG_CUDA(cudaSetDevice(ctx->device));
    return fn();
  } catch (const InvalidArgument& e) {
    return fail(ctx, CG_EINVAL, e.what());
  } catch (const std::invalid_argument& e) {
    return fail(ctx, CG_EINVAL, e.what());
  } catch (const CodecError& e) {
    return fail(ctx, CG_ECODEC, e.what());
  } catch (const DigestError& e) {
    return fail(ctx, CG_EDIGEST, e.what());
  } catch (const CudaError& e) {
    return fail(ctx, CG_ECUDA, e.what());
  } catch (const std::exception& e) {
    return fail(ctx, CG_ECUDA, e.what());
  }
}

}  // namespace cg

// ------------------------------------------------------------------ group
// One in-flight ExecutionBatch: its framing bytes, chain jobs, request
// midstates and (for host inputs) its device copy of the inputs. Ingest runs
// on the slot's own stream so the prefix chains of several batches proceed
// concurrently with each other and with the replica forwards.
// A certified batch's device results; they live in the batch's ingest slot
// until the slot is reused (ring depth later), so the tail of batch i can
// run while batch i+1's forwards write their own slot.
struct BatchResults {
  DevBuf<double> d_outs, d_topv, d_diam;
  DevBuf<uint32_t> d_topi, d_sel, d_mnodes, d_mops, d_count;
  DevBuf<uint8_t> d_leaf, d_rroots, d_aleaf, d_aroot, d_sat, d_kinds;
  DevBuf<int8_t> d_status;
  DevBuf<int64_t> d_label;
  DevBuf<int32_t> d_single_pos, d_need53;
};

struct IngestSlot {
  bool used = false, ever = false, certified = false;
  uint64_t ticket = 0;
  uint32_t B = 0;
  BatchResults res;
  cudaEvent_t ev_fwd = nullptr;  // replica outputs written (main stream)
  const double* d_in_ptr = nullptr;
  DevBuf<double> d_in, d_eps;  // d_in: device copy of host inputs (allocated on first use)
  DevBuf<uint8_t> d_arena, d_reqids;
  // chain jobs: [0, B) request midstates H(0x00||0x52||req), [B, off_leaf)
  // PerturbingExecutor seed midstates, [off_leaf, +N*B) result leaves,
  // [off_mid53, +B) single-attestation request midstates H(0x00||0x53||req)
  // (run only for requests with a single leaf), [off_single, +N*B) the
  // single leaves' tails
  DevBuf<ChainJob> d_jobs;
  uint64_t off_leaf = 0, off_mid53 = 0, off_single = 0;
  bool perturbed = false;
  DevBuf<uint32_t> d_mid, d_mid53, d_pmid;
  DevBuf<uint64_t> d_tree;  // per-provider tree offsets then lengths
  // misfit requests (input dimension != the group's; execute_batch skips
  // them, engine.cpp:286-291): their inputs, flags, and an int32 -1 that the
  // skipped result-leaf jobs point their skip flag at
  bool any_miss = false, any_kind = false;
  DevBuf<double> d_misfit;
  DevBuf<uint8_t> d_miss;        // [B] no result, [B] has outcome, [B] explicit failure
  DevBuf<int32_t> d_neg1, d_fail_pos;
  uint32_t n_fail_jobs = 0;      // explicit failure-leaf jobs after the single leaves
  bool spec53 = false;           // 0x53 request midstates chained at ingest
  PinBuf<uint8_t> h_miss;
  PinBuf<uint8_t> h_arena, h_reqids;
  PinBuf<ChainJob> h_jobs;
  PinBuf<double> h_eps;
  PinBuf<uint64_t> h_tree;
  cudaStream_t stream = nullptr;
  cudaEvent_t ev_staged = nullptr, ev_prefix = nullptr, ev_done = nullptr, ev_man = nullptr;
  ~IngestSlot() {
    if (stream) cudaStreamDestroy(stream);
    if (ev_staged) cudaEventDestroy(ev_staged);
    if (ev_prefix) cudaEventDestroy(ev_prefix);
    if (ev_done) cudaEventDestroy(ev_done);
    if (ev_fwd) cudaEventDestroy(ev_fwd);
    if (ev_man) cudaEventDestroy(ev_man);
  }
};

struct cg_group {
  cg_ctx* ctx = nullptr;
  std::vector<cg_model*> models;          // local replicas (dist: just this rank's)
  std::vector<std::array<uint8_t, 32>> digests;  // weights digest of every provider
  bool dist = false;                      // replica-parallel over the ctx's NCCL ranks
  uint32_t rank = 0;                      // this rank (dist)
  uint32_t first = 0;                     // provider index of local replica 0 (dist: rank x local)
  uint32_t N = 0, f = 0, metric = 0, maxB = 0, topk = 1;
  double eps_default = 0;
  std::string gid;
  uint64_t version = 0;
  uint64_t u = 0, v = 0;
  // forward scratch (main stream); per-batch results live in the slots
  DevBuf<double> d_pre64;
  DevBuf<float> d_pre32;
  DevBuf<uint8_t> d_gid;
  DevBuf<uint8_t> d_prep;  // shared CNN input operand
  IngestSlot* last = nullptr;  // the last certified batch (fetch, paths)
  bool all_cnn = false, same_prep = false;
  bool group_plan_ok = std::getenv("CREDO_NO_GROUP") == nullptr;  // false: per replica
  std::unique_ptr<CnnGroupPlan> gplan;   // grouped per-layer launches
  // heterogeneous CNN groups: each local replica's forward on its own stream
  // (forked from and joined into the main stream) so one model's small
  // layers and tails leave SMs to the others (CREDO_NO_HETERO_STREAMS=1:
  // sequential on the main stream)
  std::vector<cudaStream_t> rstreams;
  std::vector<cudaEvent_t> revs;  // [0] fork, [1 + li] replica li done
  std::vector<std::unique_ptr<IngestSlot>> slots;
  uint64_t next_ticket = 1;
  uint32_t last_B = 0;
  // PerturbingExecutor wrapping of every local replica (harness.cpp:255-258;
  // the harness default perturb_magnitude is 1e-9, harness.hpp:163)
  double perturb_mag = 0;
  DevBuf<uint8_t> d_phdr;     // 64 B per local provider: the seed header
  // OffsetExecutor fault injection (harness.cpp:167-186): provider
  // fault_provider's outputs += fault_offset for requests whose first id
  // byte is < fault_thr (0: no fault)
  uint32_t fault_provider = 0, fault_thr = 0;
  double fault_offset = 0;
  // batches left to ingest with speculative 0x53 midstates (set when a
  // fetched batch had single-attestation leaves)
  uint32_t spec53 = 0;
};

namespace cg {
// capi.cu: the per-batch pipeline
// staged (optional): recorded once the batch's host buffers have been copied
// (before the request-midstate chains), so the caller may reuse them
uint64_t ingest(cg_group* g, const cg_request_batch* bt, cudaEvent_t staged = nullptr);
void certify(cg_group* g, uint64_t ticket, const double* precomputed_outputs);
void certify_fetch(cg_group* g, cg_certify_out* o, const IngestSlot* slot = nullptr);
// the context stream waits for every group slot's outstanding work
void join_group_slots(cg_ctx* ctx);
}  // namespace cg
