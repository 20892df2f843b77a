/* credo_gpu.h — C-ABI of the B200-native hot path of the credo model-group
 * pipeline (arXiv 2205.15757): replica inference, per-request agreement and
 * the SHA-256 certificate digests.
 *
 * Plain C: pointers and sizes only, no C++ or torch types, no exceptions
 * across the boundary. Every entry point returns CG_OK (0) or a CG_E* code;
 * cg_last_error() holds the message. The C++ adapters a maintainer adds on
 * the reference side (CudaExecutor : credo::ModelExecutor, ...) are shown in
 * INTEGRATION.md.
 *
 * Reference interfaces replaced (paths relative to the reference's proj/):
 *   cg_sha256_batch            crypto::hash            include/credo/crypto.hpp:26-30, src/crypto.cpp:22-39
 *   cg_leaf_hash_batch         merkle::leaf_hash       include/credo/merkle.hpp:53, src/merkle.cpp:22-25
 *   cg_merkle_root_batch       merkle::Tree::build     include/credo/merkle.hpp:55-70, src/merkle.cpp:47-67
 *   cg_select_quorum_batch     distance::select_quorum include/credo/distance.hpp:65-67, src/distance.cpp:138-216
 *                              (+ the ensemble_label vote, src/experiments.cpp:99-125)
 *   cg_model_load_linear       LinearToyModel::from_file_bytes + load_group digest check
 *                              include/credo/model.hpp:22-39, src/model.cpp:46-65, src/engine.cpp:67-97
 *   cg_model_load_cnn          (new) ImageNet-class model behind the same seam, keyed by weights_digest
 *   cg_exec_run                ModelExecutor::run      include/credo/model.hpp:41-51, src/model.cpp:67-73
 *   cg_exec_run_perturbed      PerturbingExecutor::run include/credo/model.hpp:60-79, src/model.cpp:75-105
 *   cg_certify_batch           InferenceEngine::execute_batch (src/engine.cpp:269-306) +
 *                              build_result_tree (src/messages.cpp:235-258) + Coordinator::try_attest's
 *                              agreement, manifest and A tree (src/coordinator.cpp:727-849) for one batch
 *   cg_cert_leaf_hashes        the leaf re-hashing inside verify_cert / verify_failure
 *                              (src/certificate.cpp:215-316) and rebuild_committer_trees /
 *                              assemble_response (src/proxy.cpp:28-186): result_leaf,
 *                              single_attest_leaf, missing_result_leaf (src/messages.cpp:204-218,283-290)
 */
#ifndef CREDO_GPU_H
#define CREDO_GPU_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum {
  CG_OK = 0,
  CG_EINVAL = 1,  /* the reference throws std::invalid_argument */
  CG_ECUDA = 2,   /* CUDA runtime / launch failure */
  CG_ENCCL = 3,   /* NCCL failure */
  CG_EDIGEST = 4, /* model file does not hash to its descriptor digest */
  CG_ECODEC = 5,  /* malformed canonical bytes (reference CodecError) */
  CG_ENOTSUP = 6  /* no sm_100a device / not built for this device */
};

/* distance::Metric (include/credo/distance.hpp:23-27) */
enum { CG_EUCLIDEAN = 0, CG_MAX_MINUS_MIN = 1, CG_CHEBYSHEV = 2 };

typedef struct cg_ctx cg_ctx;
typedef struct cg_model cg_model;
typedef struct cg_group cg_group;

/* ---- context ---------------------------------------------------------- */
int cg_ctx_create(int device, cg_ctx** out);
void cg_ctx_destroy(cg_ctx* ctx);
const char* cg_last_error(const cg_ctx* ctx);
/* Make `stream` (a cudaStream_t) the context's launch stream. */
int cg_ctx_set_stream(cg_ctx* ctx, void* stream);
void* cg_ctx_stream(cg_ctx* ctx);
int cg_ctx_synchronize(cg_ctx* ctx);
/* Makes the context stream wait for all work enqueued so far on the
 * context's internal streams: every certification tail (internal tail
 * stream), every certified batch's single-attestation leaves and A root (its
 * ingest slot's stream) and every ingested batch's request-midstate chains. */
int cg_ctx_join(cg_ctx* ctx);

/* Number of kernels this library has launched on the context so far. */
uint64_t cg_ctx_launch_count(const cg_ctx* ctx);

/* ---- digests ------------------------------------------------------------
 * count messages msg i = buf[off[i] .. off[i]+len[i]) (host memory);
 * out: count × 32 bytes. */
int cg_sha256_batch(cg_ctx* ctx, const uint8_t* buf, const uint64_t* off,
                    const uint64_t* len, uint64_t count, uint8_t* out);
/* H(0x00 || leaf_i) for each message. */
int cg_leaf_hash_batch(cg_ctx* ctx, const uint8_t* buf, const uint64_t* off,
                       const uint64_t* len, uint64_t count, uint8_t* out);
/* ntrees Merkle roots over precomputed leaf digests: tree t folds
 * leaf_hashes[first_t .. first_t + n_leaves[t]) where first_t is the running
 * sum of n_leaves. CG_EINVAL for an empty tree (Tree::build throws). */
int cg_merkle_root_batch(cg_ctx* ctx, const uint8_t* leaf_hashes,
                         const uint64_t* n_leaves, uint64_t ntrees,
                         uint8_t* roots);

/* merkle::Tree::auth_path (merkle.cpp:69-84) of `count` leaf indices in the
 * tree over n precomputed leaf hashes; root (may be NULL) = Tree::root().
 * Fixed-stride paths: siblings count x 64 x 32 bytes, sides count x 64
 * (0 = Side::left, 1 = Side::right), lens count (steps, bottom level first).
 * CG_EINVAL for n == 0 (Tree::build throws) or an index >= n
 * (std::out_of_range). */
int cg_merkle_auth_paths(cg_ctx* ctx, const uint8_t* leaf_hashes, uint64_t n,
                         const uint64_t* indices, uint32_t count, uint8_t* siblings,
                         uint8_t* sides, uint32_t* lens, uint8_t* root);
/* merkle::get_merkle_root(path, leaf) (merkle.cpp:86-93) for count paths,
 * each leaf given by its hash leaf_hash(leaf); same path layout. */
int cg_merkle_path_roots(cg_ctx* ctx, const uint8_t* leaf_hashes, const uint8_t* siblings,
                         const uint8_t* sides, const uint32_t* lens, uint32_t count,
                         uint8_t* roots);

/* ---- agreement ----------------------------------------------------------
 * R requests; outs is R × n × v row-major (request, node, lane); row (r, i)
 * is considered only when bit i of present[r] is set (present == NULL: all
 * n present). eps[r] is the request's epsilon (override or group default).
 * Writes selected node mask, diameter, satisfied flag, and (label != NULL)
 * the ensemble label (-1: none). status[r] = -1 where the reference throws
 * std::invalid_argument; the call then returns CG_EINVAL. */
int cg_select_quorum_batch(cg_ctx* ctx, const double* outs,
                           const uint32_t* present, const double* eps,
                           uint32_t R, uint32_t n, uint32_t f, uint32_t v,
                           uint32_t metric, uint32_t* selected,
                           double* diameter, uint8_t* satisfied,
                           int8_t* status, int64_t* label);

/* Device-resident form for large sweeps (C5): every pointer is device
 * memory, the work is enqueued on the context stream and the call returns
 * without synchronising. outs(k, p, t) = outs[p*ps + k*rs + t]; all n
 * results present. label / label_digest may be NULL. label_digest[k] =
 * SHA-256(0x4C || req_ids[k] || u64be version || u64be label[k]) (new; the
 * north star's compact agreed-label digest). */
int cg_agree_device(cg_ctx* ctx, const double* outs, uint64_t ps, uint64_t rs,
                    const double* eps, uint32_t R, uint32_t n, uint32_t f, uint32_t v,
                    uint32_t metric, const uint8_t* req_ids, uint64_t version,
                    uint32_t* selected, double* diameter, uint8_t* satisfied,
                    int8_t* status, int64_t* label, uint8_t* label_digest);
/* The compact label digests alone, host buffers (R × 32 ids, R labels). */
int cg_label_digest_batch(cg_ctx* ctx, const uint8_t* req_ids, const int64_t* labels,
                          uint32_t R, uint64_t version, uint8_t* out);

/* ---- models (executor seam) --------------------------------------------- */
/* LinearToyModel canonical file bytes; digest = descriptor weights_digest.
 * Fails with CG_EDIGEST when SHA-256(file) != digest (src/engine.cpp:79). */
int cg_model_load_linear(cg_ctx* ctx, const uint8_t* file, uint64_t len,
                         const uint8_t digest[32], cg_model** out);
/* CNN model file (format in DESIGN.md §3: canonical header + f32 tensors). */
int cg_model_load_cnn(cg_ctx* ctx, const uint8_t* file, uint64_t len,
                      const uint8_t digest[32], cg_model** out);
void cg_model_free(cg_model* m);
int cg_model_dims(const cg_model* m, uint64_t* input_dim, uint64_t* output_dim);
/* One output row per input row, in order (ModelExecutor::run). Host memory:
 * in is B × u, out is B × v, both f64 row-major. */
int cg_exec_run(cg_ctx* ctx, cg_model* m, const double* in, uint64_t B,
                uint64_t u, double* out, uint64_t v);
/* PerturbingExecutor(inner = cg_exec_run, node_index, magnitude)::run: each
 * output lane gets the node's deterministic offset in [-magnitude,
 * +magnitude] from SHA-256(u64 node || model digest || f64_list(input) ||
 * u64 lane). magnitude 0 = cg_exec_run; negative or NaN -> CG_EINVAL (the
 * reference constructor's std::invalid_argument). */
int cg_exec_run_perturbed(cg_ctx* ctx, cg_model* m, const double* in, uint64_t B,
                          uint64_t u, double* out, uint64_t v,
                          uint64_t node_index, double magnitude);

/* ---- one batch through the whole hot path -------------------------------
 * A model group replica set: models[p] answers for node p (the
 * assigned_models bijection, src/domain.cpp:247-268). */
int cg_group_create(cg_ctx* ctx, cg_model* const* models, uint32_t N,
                    uint32_t f, uint32_t metric, double default_eps,
                    const char* group_id, uint64_t group_id_len,
                    uint64_t version, uint32_t max_batch, uint32_t topk,
                    cg_group** out);
void cg_group_free(cg_group* g);
/* Wrap every local replica in PerturbingExecutor(node_index = provider
 * index, magnitude) (src/model.cpp:75-105, harness wiring
 * src/harness.cpp:255-258; harness default 1e-9, include/credo/harness.hpp:163)
 * for the forwards of later certify calls. 0 (the default) = plain replicas;
 * negative or NaN -> CG_EINVAL. cg_certify_outputs (precomputed outputs) is
 * not affected. The reported top-k is of the unperturbed replica outputs. */
int cg_group_set_perturbation(cg_group* g, double magnitude);
/* Fault injection: wrap provider `provider` in OffsetExecutor(offset) (the
 * corrupt_result fault, src/harness.cpp:167-186, wrapping the perturbing
 * executor as at :255-261) for the requests whose first request-id byte is
 * below round(256 * fraction); fraction 1 = every request (the reference's
 * executor exactly), offset 0 = no fault. Applies to later certify calls. */
int cg_group_set_fault(cg_group* g, uint32_t provider, double offset, double fraction);
/* The wire payload of provider `provider`'s results for the last certified
 * batch, as PREPARE / PRE-PREPARE carry them: encode_results
 * (src/messages.cpp:48-50, used at :376 and :406) = u32be count || B ×
 * InferenceResult::encode (src/domain.cpp:218-225), encoded on the device
 * from the resident f64 outputs. *len = 4 + B·(88 + |group_id| + 8v); with
 * out == NULL only *len is set; cap < *len -> CG_EINVAL. */
int cg_group_encode_results(cg_group* g, uint32_t provider, uint8_t* out, uint64_t cap,
                            uint64_t* len);
/* The same for a named certified ticket (CG_EINVAL when the ticket is not
 * certified or its ingest slot was reused). */
int cg_group_encode_results_ticket(cg_group* g, uint64_t ticket, uint32_t provider,
                                   uint8_t* out, uint64_t cap, uint64_t* len);

/* The ExecutionBatch (include/credo/engine.hpp:29-34) in struct-of-arrays
 * form: the request fields of InferenceRequest (include/credo/domain.hpp:
 * 99-115). inputs is B × u f64; host memory unless inputs_on_device. */
#define CG_INGEST_RING 24

typedef struct {
  uint32_t B;
  uint64_t u;
  const uint8_t* request_ids; /* B × 32 */
  const double* inputs;       /* B × u */
  int inputs_on_device;
  const uint8_t* has_eps;     /* B (NULL: no overrides) */
  const double* eps;          /* B */
  const uint8_t* client_pubs; /* B × 32 */
  const uint8_t* nonces;      /* concatenated nonce bytes */
  const uint64_t* nonce_lens; /* B */
  const uint8_t* client_sigs; /* B × 64 */
  /* Optional (NULL: every request has u inputs). Request k with
   * input_dims[k] != u is a misfit: execute_batch skips it (src/engine.cpp:
   * 286-291), so no provider has a result for it — its R leaf is
   * missing_result_leaf 0x4D (src/messages.cpp:213-218, :246-252), its
   * outcome unsatisfied, its A leaf a failure. Its input_dims[k] doubles are
   * read from misfit_inputs[k] (host); row k of `inputs` is ignored. */
  const uint64_t* input_dims;
  const double* const* misfit_inputs;
  /* Optional slot structure: the batch as a PRE-PREPARE's op list
   * (include/credo/messages.hpp:106-118). op_kinds[k] (NULL: every op an ok
   * request) = CG_OP_REQUEST, CG_OP_REQUEST_REJECTED (status rejected: no
   * result, R leaf missing_result_leaf, no outcome, A leaf = its failure
   * record) or CG_OP_GROUP (a define/activate/retire op: R leaf
   * group_op_leaf 0x47 || op_entries[k], no outcome, an A leaf only if
   * rejected). op_entries: the group ops' OpEntry::encode bytes back to back
   * (op_entry_lens[k], 0 for requests); fail_records: FailureRecord::encode
   * of failure_record_for(op) (messages.cpp:299-312) for every rejected op
   * (fail_record_lens[k], 0 otherwise). A group op's request fields are
   * ignored (zeros, nonce length 0). */
  const uint8_t* op_kinds;
  const uint8_t* op_entries;
  const uint64_t* op_entry_lens;
  const uint8_t* fail_records;
  const uint64_t* fail_record_lens;
} cg_request_batch;

enum { CG_OP_REQUEST = 0, CG_OP_REQUEST_REJECTED = 1, CG_OP_GROUP = 2 };

/* Host-memory results. Optional arrays may be NULL. */
typedef struct {
  uint32_t* selected;     /* B: node mask of the agreed quorum */
  double* diameter;       /* B */
  uint8_t* satisfied;     /* B */
  int64_t* label;         /* B: ensemble label, -1 none */
  uint8_t* r_roots;       /* N × 32: per-provider result-tree roots */
  uint8_t* a_root;        /* 32: attestation-tree root */
  uint64_t* manifest_len; /* 1 */
  uint8_t* manifest_kind; /* optional, ≤ N×B + B: 0 whole, 1 single, 2 failure */
  uint32_t* manifest_node;/* optional */
  uint32_t* manifest_op;  /* optional */
  uint8_t* leaf_hashes;   /* optional N × B × 32 (provider-major) */
  uint8_t* a_leaf_hashes; /* optional ≤ N×B + B × 32 */
  double* outputs;        /* optional N × B × v (provider-major) */
  uint32_t* topk_idx;     /* optional N × B × k */
  double* topk_val;       /* optional N × B × k */
} cg_certify_out;

/* Runs batch → N replica forwards → softmax/top-k → agreement + label →
 * result leaves, R roots, attestation manifest, A leaves, A root. With
 * out == NULL the call only enqueues (results stay on the device; fetch with
 * cg_group_fetch). */
int cg_certify_batch(cg_group* g, const cg_request_batch* batch,
                     cg_certify_out* out);
int cg_group_fetch(cg_group* g, cg_certify_out* out);
/* Results of a certified ticket whose ingest slot has not been reused yet
 * (the ring holds CG_INGEST_RING batches), e.g. to read batch i back while
 * batch i+1's forwards run. */
int cg_group_fetch_ticket(cg_group* g, uint64_t ticket, cg_certify_out* out);
/* The same path split at the reference's own seam: ingest = the hot part of
 * InferenceEngine::submit (src/engine.cpp:182-209) — framing bytes, upload,
 * and the request-midstate SHA-256 chains started on a per-batch stream —
 * and certify = execute_batch + R trees + try_attest for that ticket. Up to
 * CG_INGEST_RING batches may be ingested ahead; tickets are certified in any
 * order. A slot is reused by the CG_INGEST_RING-th ingest after its own, so a
 * certified ticket's results stay fetchable until then. */
int cg_ingest_batch(cg_group* g, const cg_request_batch* batch, uint64_t* ticket);
int cg_certify_ticket(cg_group* g, uint64_t ticket, cg_certify_out* out);
/* Agreement + digest path over precomputed replica outputs (host memory,
 * N × B × v provider-major f64): the C5 sweep and fault-injection entry
 * point (a corrupt replica is just a shifted output row). */
int cg_certify_outputs(cg_group* g, const cg_request_batch* batch,
                       const double* outputs, cg_certify_out* out);
/* An empty filler slot (build_result_tree with no ops, messages.cpp:240-243):
 * every provider's R tree is the single noop_leaf H(0x00||0x4E||u64 view||
 * u64 seq); with no outcomes every provider is whole-batch attested
 * (coordinator.cpp:776-787), so the A tree is N whole-batch leaves. Fills
 * out->r_roots, a_root, manifest_len / kind / node / op, a_leaf_hashes. */
int cg_certify_empty_slot(cg_group* g, uint64_t view, uint64_t seq, cg_certify_out* out);

/* verify_request's digests for a batch (domain.cpp:177-216, :238-241):
 * signing_digests[k] = InferenceRequest::signing_digest() = SHA-256(0x01 ||
 * body), canonical_ids[k] = SHA-256(client_pub || 0x1F || nonce), and
 * status[k] = 0 ok, 1 empty nonce, 2 empty input, 3 bad epsilon override,
 * 4 request id != canonical id. verify_request's last step, Ed25519
 * verify(client_pub, signing_digest, client_sig), stays on the host.
 * Output pointers may be NULL. */
int cg_request_digests(cg_ctx* ctx, const cg_request_batch* batch, const char* group_id,
                       uint64_t group_id_len, uint8_t* signing_digests,
                       uint8_t* canonical_ids, int8_t* status);

/* ---- certificate verification / assembly at batch scale ------------------
 * For M (request, result) pairs over one request batch (uniform input length,
 * request ops only; group_id as in cg_request_digests): want[m] is a mask of
 *   1: leaf_hash(result_leaf(req, res))        -> leaf52 + 32m  (0x52)
 *   2: leaf_hash(single_attest_leaf(req, res)) -> leaf53 + 32m  (0x53)
 *   4: leaf_hash(missing_result_leaf(req))     -> leaf4d + 32m  (0x4D; result unused)
 * with req = request req_index[m] and res = InferenceResult::encode bytes
 * (src/domain.cpp:218-225), result_lens[m] of them, back to back in
 * result_enc (an entry with only bit 4 may have length 0). Each request's
 * 1.2 MB prefix (ImageNet shape) is hashed once per tag as a midstate shared
 * by all of its results. The C++ adapters credo::gpu::verify_responses and
 * credo::gpu::assemble_responses (include/credo_gpu_adapters.hpp) build the
 * reference's verify_response / assemble_response on it. */
int cg_cert_leaf_hashes(cg_ctx* ctx, const cg_request_batch* batch, const char* group_id,
                        uint64_t group_id_len, uint32_t M, const uint32_t* req_index,
                        const uint8_t* want, const uint8_t* result_enc,
                        const uint64_t* result_lens, uint8_t* leaf52, uint8_t* leaf53,
                        uint8_t* leaf4d);

/* ---- the batch former (InferenceEngine, src/engine.cpp:166-267) ----------
 * Per live (group, version): FIFO queue with `seen` dedup; a batch is released
 * when the queue reaches exec_batch_max (submit) or its oldest request has
 * waited flush_interval_us (flush_due), or on demand (flush_version /
 * flush_all); every submission is queued for EVERY live version (one batch
 * per live version, engine.cpp:196-206). Requests are packed into pinned
 * staging as they are submitted; a released batch is ingested into its
 * group (cg_ingest_batch) and reported by cg_engine_ready as a ticket, in
 * release order, for cg_certify_ticket. verify_request's structural checks
 * run in submit; the Ed25519 check is the optional verifier callback's
 * (NULL: the caller verified). */
typedef struct cg_engine cg_engine;
typedef struct { /* one InferenceRequest (include/credo/domain.hpp:99-115) */
  const uint8_t* request_id; /* 32 */
  const char* group_id;
  uint64_t group_id_len;
  const double* input; /* host */
  uint64_t input_dim;
  int has_eps;
  double eps;
  const uint8_t* client_pub; /* 32 */
  const uint8_t* nonce;
  uint64_t nonce_len;
  const uint8_t* client_sig; /* 64 */
} cg_request;
typedef struct {
  cg_group* group;
  uint64_t version;
  uint64_t ticket;
  uint32_t B;
} cg_ready_batch;
/* SubmitOutcome::error (engine.cpp:182-209) */
enum { CG_SUBMIT_OK = 0, CG_SUBMIT_INVALID = 1, CG_SUBMIT_UNKNOWN_GROUP = 2, CG_SUBMIT_RETIRED = 3 };
/* GroupStatus (include/credo/domain.hpp) */
enum { CG_GROUP_DEFINED = 0, CG_GROUP_ACTIVE = 1, CG_GROUP_RETIRED = 2 };
/* Ed25519 verify(pub, signing_digest, sig): nonzero = valid. */
typedef int (*cg_sig_verify_fn)(void* user, const uint8_t pub[32], const uint8_t digest[32],
                                const uint8_t sig[64]);
int cg_engine_create(cg_ctx* ctx, uint64_t exec_batch_max, uint64_t flush_interval_us,
                     int pack_threads, cg_engine** out);
void cg_engine_free(cg_engine* e);
int cg_engine_set_verifier(cg_engine* e, cg_sig_verify_fn fn, void* user);
/* load_group for a version whose replicas are resident as group g
 * (group id and version are g's); status CG_GROUP_*. A second load of the
 * same (group, version) -> CG_EINVAL ("version already loaded"). */
int cg_engine_load_group(cg_engine* e, cg_group* g, int status);
int cg_engine_set_status(cg_engine* e, const char* group_id, uint64_t group_id_len,
                         uint64_t version, int status);
/* n submissions in order at time now_us; errors[i] = CG_SUBMIT_* (may be NULL). */
int cg_engine_submit(cg_engine* e, const cg_request* reqs, uint32_t n, uint64_t now_us,
                     int* errors);
int cg_engine_flush_due(cg_engine* e, uint64_t now_us);
int cg_engine_flush_version(cg_engine* e, const char* group_id, uint64_t group_id_len,
                            uint64_t version);
int cg_engine_flush_all(cg_engine* e);
int cg_engine_next_flush_deadline(cg_engine* e, uint64_t* deadline, int* has);
/* Released, ingested batches in release order (up to cap; *n_out written). A
 * released batch whose group ring is full waits here until tickets of that
 * group are certified. */
int cg_engine_ready(cg_engine* e, cg_ready_batch* out, uint32_t cap, uint32_t* n_out);
int cg_engine_pending(cg_engine* e, uint64_t* queued, uint64_t* waiting_batches);

/* ---- host digests (no device involved) -----------------------------------
 * SHA-256 on the host, x86 SHA extensions when present (the model-file check
 * of load_group, src/engine.cpp:79, runs here: one ~100 MB chain). */
int cg_host_sha256(const uint8_t* data, uint64_t len, uint8_t out[32]);
int cg_host_sha_accelerated(void);

/* One PRE-PREPARE's op list of inference requests for hash_ops
 * (src/messages.cpp:197-202): OpEntry{request_inf, requests[k], version
 * versions[k] (NULL: `version` for all), status statuses[k] (NULL: ok),
 * reason = reasons bytes of reason_lens[k] (NULL: "")}. */
typedef struct {
  const cg_request_batch* requests; /* host inputs */
  const char* group_id;
  uint64_t group_id_len;
  uint64_t version;
  const uint64_t* versions;
  const uint8_t* statuses;
  const char* reasons;
  const uint64_t* reason_lens;
} cg_ops_batch;
/* hash_ops of nslots op lists on up to `threads` host threads (one op list
 * per thread at a time; each is one sequential SHA-256 chain over every
 * request encoding, 1.2 MB per ImageNet request, streamed from the f64
 * inputs without re-serialising). out: nslots x 32. */
int cg_hash_ops_batches(const cg_ops_batch* batches, uint32_t nslots, int threads,
                        uint8_t* out);

/* Certificate assembly for the last certified batch (ProxyCore::
 * assemble_response, proxy.cpp:80-186): auth paths in provider `tree`'s
 * result tree (tree < N; leaf k = request k) or, tree == N, in the
 * attestation tree (leaf i = manifest entry i). Same path layout as
 * cg_merkle_auth_paths. */
int cg_group_auth_paths(cg_group* g, uint32_t tree, const uint64_t* indices, uint32_t count,
                        uint8_t* siblings, uint8_t* sides, uint32_t* lens);
/* The same for a named certified ticket. */
int cg_group_auth_paths_ticket(cg_group* g, uint64_t ticket, uint32_t tree,
                               const uint64_t* indices, uint32_t count, uint8_t* siblings,
                               uint8_t* sides, uint32_t* lens);

/* ---- replica-parallel groups (one model owner's replica per GPU) ---------
 * The SURVEY §8(e) / north-star mapping: rank r of an NCCL communicator is
 * node r of the group and runs only replica r. Every rank ingests the same
 * batch; certify computes rank r's outputs, result leaves and R root, one
 * ncclAllGather over NVLink brings every provider's outputs and R root to
 * every rank, and each rank then runs select_quorum, the label vote and the
 * attestation tree (every reference node attests, coordinator.cpp:727-865).
 * cg_nccl_unique_id on rank 0, broadcast the 128 bytes out of band. */
int cg_nccl_unique_id(uint8_t out[128]);
int cg_ctx_init_nccl(cg_ctx* ctx, const uint8_t id[128], int nranks, int rank);
/* all_digests: nranks x 32 weights digests (provider order); my_model must
 * be provider `rank`'s model. */
int cg_group_create_dist(cg_ctx* ctx, cg_model* my_model, const uint8_t* all_digests,
                         uint32_t f, uint32_t metric, double default_eps,
                         const char* group_id, uint64_t group_id_len, uint64_t version,
                         uint32_t max_batch, uint32_t topk, cg_group** out);
/* k = nlocal replicas per rank (assigned_models chunking): rank r serves
 * providers [r k, (r + 1) k), my_models in that order; N = k x nranks. The
 * local replicas of one architecture run as grouped launches; the
 * all-gather moves k providers' outputs and R roots per rank. */
int cg_group_create_dist_multi(cg_ctx* ctx, cg_model* const* my_models, uint32_t nlocal,
                               const uint8_t* all_digests, uint32_t f, uint32_t metric,
                               double default_eps, const char* group_id, uint64_t group_id_len,
                               uint64_t version, uint32_t max_batch, uint32_t topk,
                               cg_group** out);

/* ---- measurement hooks ----------------------------------------------------
 * Per-kernel-class device time from CUDA events recorded on each launching
 * stream (0 conv GEMM, 1 SHA-256 chains, 2 agreement + trees, 3 CNN
 * auxiliary kernels, 4 NCCL exchange). Enabling resets the counters. */
void cg_timing_enable(int on);
int cg_timing_read(int cls, double* total_ms, uint64_t* launches);
/* The individual launch durations of a class in launch order (up to cap). */
int cg_timing_spans(int cls, double* ms_out, uint64_t cap, uint64_t* count);
/* Algorithmic FLOPs of one forward of one input (2 x MACs). */
double cg_model_flops_per_input(const cg_model* m);
/* C5 synthetic sweep input, generated on the device: per
 * request k a centre U(0,1)^v, each replica p = centre + U(-a, a) per lane
 * with a = eps/(8 sqrt(v)) (honest euclidean spread ~eps/10), and with
 * probability shift_frac a replica shifted by 3 eps/sqrt(v) on every lane
 * (euclidean distance ~3 eps: the accuracy_experiment "beyond" shift). outs(k, p, t) = outs[p*R*v + k*v + t]; req_ids R × 32. */
int cg_synth_outputs(cg_ctx* ctx, uint64_t seed, uint32_t R, uint32_t n, uint32_t v,
                     double eps, double shift_frac, double* outs, uint8_t* req_ids);

/* ---- test hooks (not on the certified path) -----------------------------
 * One tcgen05 conv-GEMM launch on host buffers (bf16 as uint16 bits). */
int cg_dbg_conv_gemm(cg_ctx* ctx, const uint16_t* A, int rowsA,
                     const uint16_t* B, int N, int Kc, int ntaps,
                     const int* tap_off, const float* bias,
                     const uint16_t* residual, int relu, int row_mode, int H,
                     int W, int M, int rows_out, int out_f32, int BN, void* out,
                     int max_ctas);
/* The same on SM pairs (cta_group::2: 256 x 256 tiles, each CTA holding
 * half of the weight tile; BN = 256 only). */
int cg_dbg_conv_gemm_pair(cg_ctx* ctx, const uint16_t* A, int rowsA, const uint16_t* B, int N,
                          int Kc, int ntaps, const int* tap_off, const float* bias,
                          const uint16_t* residual, int relu, int row_mode, int H, int W, int M,
                          int rows_out, int out_f32, int BN, void* out, int max_ctas);
/* The same in halo mode (one (BM + 2*halo_lo)-row box per channel block
 * feeds all 9 taps from shared memory). */
int cg_dbg_conv_gemm_halo(cg_ctx* ctx, const uint16_t* A, int rowsA, const uint16_t* B, int N,
                          int Kc, int ntaps, const int* tap_off, const float* bias, int relu,
                          int row_mode, int H, int W, int M, int rows_out, int BN, void* out,
                          int halo_lo);
/* Halo mode on SM pairs (cta_group::2, 256-row tiles; BN = 128 only). */
int cg_dbg_conv_gemm_halo_pair(cg_ctx* ctx, const uint16_t* A, int rowsA, const uint16_t* B,
                               int N, int Kc, int ntaps, const int* tap_off, const float* bias,
                               int relu, int row_mode, int H, int W, int M, int rows_out, int BN,
                               void* out, int halo_lo);

#ifdef __cplusplus
}
#endif
#endif /* CREDO_GPU_H */
