// Host launchers for agree.cu.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg {

void launch_select_quorum(const double* outs, uint64_t ps, uint64_t rs,
                          const uint32_t* present, const double* eps,
                          uint32_t R, uint32_t n, uint32_t f, uint32_t v,
                          uint32_t metric, uint32_t* selected, double* diameter,
                          uint8_t* satisfied, int8_t* status, int64_t* label,
                          cudaStream_t st);
// Throughput form of select_quorum + ensemble_label (+ optional compact
// label digests) for large all-present batches with n <= 8 (C5 sweep).
constexpr uint32_t kAgreeRowsMinBatch = 4096;
bool agree_rows_eligible(uint32_t R, uint32_t n, uint32_t f, uint32_t v, uint32_t metric,
                         const uint32_t* present);
void launch_agree_rows(const double* outs, uint64_t ps, uint64_t rs, const double* eps,
                       uint32_t R, uint32_t n, uint32_t f, uint32_t v, uint32_t metric,
                       const uint8_t* req_ids, uint64_t version, uint32_t* selected,
                       double* diameter, uint8_t* satisfied, int8_t* status, int64_t* label,
                       uint8_t* digest, cudaStream_t st);
void launch_label_digest(const uint8_t* req_ids, const int64_t* label, uint32_t R,
                         uint64_t version, uint8_t* out, cudaStream_t st);
void launch_attest_manifest(uint32_t B, uint32_t N, const uint32_t* sel,
                            const uint8_t* sat, const uint8_t* r_roots,
                            const uint8_t* req_ids, const uint8_t* gid,
                            uint32_t gid_len, uint64_t version,
                            uint8_t* a_leaves, int32_t* single_pos, int32_t* need53,
                            uint8_t* kinds, uint32_t* m_nodes, uint32_t* m_ops,
                            uint32_t* count, const uint8_t* has_outcome,
                            const uint8_t* explicit_fail, int32_t* fail_pos, cudaStream_t st);
void launch_mark_missing(const uint8_t* miss, uint32_t B, uint32_t* sel, double* diam,
                         uint8_t* sat, int8_t* status, int64_t* label, cudaStream_t st);
void launch_softmax_topk_f32(const float* in, uint64_t in_ld, uint32_t rows,
                             uint32_t v, int do_softmax, double* out,
                             uint64_t out_ld, uint32_t k, uint32_t* topi,
                             double* topv, cudaStream_t st);
void launch_softmax_topk_f64(const double* in, uint64_t in_ld, uint32_t rows,
                             uint32_t v, int do_softmax, double* out,
                             uint64_t out_ld, uint32_t k, uint32_t* topi,
                             double* topv, cudaStream_t st);
void launch_linear_f64(const double* W, const double* b, const double* X,
                       uint32_t B, uint32_t u, uint32_t v, double* Y,
                       cudaStream_t st);

}  // namespace cg
