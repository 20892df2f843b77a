/* TEST INFRASTRUCTURE — the CPU oracle. Only tests/, __graft_entry__.smoke()
 * and bench.py's cpu_baseline/reference legs may load this. It is a plain-C
 * restatement of the reference's hot-path algorithms (each function cites the
 * reference file:line it follows) and is pinned against the compiled
 * reference (oracle/_ref) through tests/golden/ fixtures. */
#ifndef CREDO_ORACLE_H
#define CREDO_ORACLE_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct {
  uint32_t h[8];
  uint64_t total;
  uint8_t buf[64];
  uint32_t nbuf;
} oc_sha256_ctx;

void oc_sha256_init(oc_sha256_ctx* c);
void oc_sha256_update(oc_sha256_ctx* c, const uint8_t* p, uint64_t n);
void oc_sha256_final(oc_sha256_ctx* c, uint8_t out[32]);
void oc_sha256(const uint8_t* p, uint64_t n, uint8_t out[32]);
/* Compression-function state after absorbing `nblocks` whole blocks. */
void oc_sha256_midstate(const uint8_t* p, uint64_t nblocks, uint32_t out[8]);

/* Canonical encodings (codec.hpp:28-84; domain.cpp:144-158, 218-225). Return
 * the encoded length; write only when out != NULL. */
uint64_t oc_request_encode(const uint8_t req_id[32], const char* gid,
                           uint64_t gid_len, const double* input, uint64_t u,
                           int has_eps, double eps, const uint8_t pub[32],
                           const uint8_t* nonce, uint64_t nonce_len,
                           const uint8_t sig[64], uint8_t* out);
uint64_t oc_result_encode(const uint8_t req_id[32], uint64_t node,
                          const char* gid, uint64_t gid_len, uint64_t version,
                          const double* output, uint64_t v,
                          const uint8_t model_digest[32], uint8_t* out);

/* merkle.cpp:22-25 leaf hash H(0x00 || leaf). */
void oc_leaf_hash(const uint8_t* leaf, uint64_t n, uint8_t out[32]);
/* H(0x00 || 0x52 || req || res) — leaf_hash(result_leaf) (messages.cpp:204-211). */
void oc_result_leaf_hash(const uint8_t* req, uint64_t req_len,
                         const uint8_t* res, uint64_t res_len, uint8_t out[32]);
/* H(0x00 || tag || a || b) generic two-part leaf (single 0x53, missing 0x4D). */
void oc_tagged_leaf_hash(uint8_t tag, const uint8_t* a, uint64_t na,
                         const uint8_t* b, uint64_t nb, uint8_t out[32]);
/* Tree::build fold (merkle.cpp:47-67) over precomputed leaf hashes. */
int oc_merkle_root(const uint8_t* leaf_hashes, uint64_t n, uint8_t out[32]);

/* distance::select_quorum (distance.cpp:138-216). outs m×v row-major;
 * node_idx ascending. Returns 0, or -1 where the reference throws
 * std::invalid_argument. selected_mask uses node ids as bit positions. */
int oc_select_quorum(const double* outs, const uint64_t* node_idx, uint64_t m,
                     uint64_t v, uint64_t n, uint64_t f, uint32_t metric,
                     double eps, uint64_t* selected_mask, double* diam,
                     int* satisfied);
double oc_delta(uint32_t metric, const double* x, const double* y, uint64_t v);

/* experiments.cpp:99-101 argmax (first maximum). */
uint64_t oc_argmax(const double* v, uint64_t n);
/* experiments.cpp:106-125 ensemble_label over outs rows in mask. -1: none. */
int64_t oc_ensemble_label(const double* outs, uint64_t m, uint64_t v,
                          uint64_t mask, uint64_t f);
/* Top-k (new; no reference equivalent): k largest, ties to lower index,
 * consistent with oc_argmax for k = 1. */
void oc_topk(const double* v, uint64_t n, uint32_t k, uint32_t* idx,
             double* val);

/* LinearToyModel::run (model.cpp:12-36), fp64 sequential, no contraction. */
void oc_linear_run(const double* W, const double* b, uint64_t u, uint64_t v,
                   int softmax, const double* x, double* y);
/* The softmax tail of model.cpp:26-34 applied in place. */
void oc_softmax(double* y, uint64_t v);
/* PerturbingExecutor::run (model.cpp:82-105) for one request, in place on
 * its v outputs: lane offset from SHA(u64 node || model_digest ||
 * f64_list(input) || u64 lane), first 8 digest bytes -> U[-mag, +mag].
 * mag == 0 leaves y unchanged (model.cpp:85). */
void oc_perturb(uint64_t node, const uint8_t model_digest[32], const double* x,
                uint64_t u, double* y, uint64_t v, double mag);

/* Coordinator::try_attest manifest (coordinator.cpp:774-832) for a batch of
 * B request ops with all N providers present. kinds: 0 whole_batch,
 * 1 single, 2 failure. Returns the manifest length. */
uint64_t oc_attest_manifest(uint64_t B, uint64_t N, const uint64_t* sel_mask,
                            const uint8_t* satisfied, uint8_t* kinds,
                            uint64_t* nodes, uint64_t* ops);
/* FailureRecord encoding (messages.cpp:262-267) with tag 0x46 prepended. */
uint64_t oc_failure_leaf(const uint8_t req_id[32], const char* gid,
                         uint64_t gid_len, uint64_t version, const char* reason,
                         uint64_t reason_len, uint8_t* out);

/* Compact agreed-label digest (new, north star / SURVEY §8(d) C5 "D2"):
 * SHA-256(0x4C || req_id[32] || u64be version || u64be label). */
void oc_label_digest(const uint8_t req_id[32], uint64_t version, int64_t label,
                     uint8_t out[32]);
/* C5 batch: outs(k, p, t) = outs[p*R*v + k*v + t], all n present; per
 * request select_quorum + ensemble_label + label digest (NULL ids: none).
 * Returns 0 or -1 (invalid arguments, as select_quorum). */
int oc_agree_batch(const double* outs, uint64_t R, uint64_t n, uint64_t f,
                   uint64_t v, uint32_t metric, const double* eps,
                   const uint8_t* req_ids, uint64_t version, uint64_t* sel,
                   double* diam, uint8_t* sat, int64_t* label, uint8_t* digest);

#ifdef __cplusplus
}
#endif
#endif
