// Host launchers for the digest kernels (digest.cu).
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>

#include <vector>

#include "sha256.cuh"

namespace cg {

constexpr int kChainExclusiveSmem = 120 * 1024;
constexpr int kChainExclusiveThreads = 128;
void launch_chain_jobs(const ChainJob* d_jobs, uint32_t n, cudaStream_t st,
                       bool exclusive_sm = false);
// Jobs whose messages are plain bytes (no f64 segment, no skip flag).
void launch_chain_jobs_raw(const ChainJob* d_jobs, uint32_t n, cudaStream_t st);
// ntrees trees; tree t = leaves [off[t], off[t]+len[t]) or count_dev[t].
void launch_merkle_trees(const uint8_t* d_leaves, const uint64_t* d_off,
                         const uint64_t* d_len, const uint32_t* d_count,
                         uint32_t ntrees, uint64_t max_leaves, uint8_t* d_roots,
                         cudaStream_t st, uint64_t n_const = 0);
size_t merkle_big_scratch_bytes(uint64_t n);
void launch_merkle_big(const uint8_t* d_leaves, uint64_t n, uint8_t* d_scratch,
                       uint8_t* d_root, cudaStream_t st);

// Authentication paths (merkle.cpp:69-93). Paths are fixed-stride:
// kMaxPathSteps slots of a 32-byte sibling, a side byte (0 = Side::left,
// 1 = Side::right) per slot, and a step count.
constexpr int kMaxPathSteps = 64;
struct PathLevels {
  uint64_t n;
  int nlevels;
  uint64_t off[kMaxPathSteps + 1];
};
uint64_t merkle_levels_nodes(uint64_t n);
std::vector<uint64_t> launch_merkle_levels(const uint8_t* d_leaves, uint64_t n,
                                           uint8_t* d_levels, cudaStream_t st);
void launch_auth_paths(const uint8_t* d_levels, const std::vector<uint64_t>& off, uint64_t n,
                       const uint64_t* d_idx, uint32_t count, uint8_t* d_sib, uint8_t* d_sides,
                       uint32_t* d_lens, cudaStream_t st);
void launch_path_roots(const uint8_t* d_leaf_hashes, const uint8_t* d_sib, const uint8_t* d_sides,
                       const uint32_t* d_lens, uint32_t count, uint8_t* d_roots,
                       cudaStream_t st);

// encode_results (proj/src/messages.cpp:48-50) of one provider's B results
// into d_dst (4 + B * (88 + gl + 8v) bytes).
struct Digest32 {
  uint8_t b[32];
};
void launch_encode_results(const uint8_t* d_reqids, const double* d_outs, uint32_t B, uint32_t v,
                           uint64_t node, const uint8_t* d_gid, uint32_t gl, uint64_t version,
                           const Digest32& model_digest, uint8_t* d_dst, cudaStream_t st);

// PerturbingExecutor (proj/src/model.cpp:82-105): the 44-byte seed header
// (u64 node || model_digest || u32be input count), the B midstates over the
// first nshared = (44 + 8u) / 64 blocks, then one thread per (request, lane).
struct PerturbHdr {
  uint8_t b[44];
};
void launch_perturb_tail(const uint32_t* d_mid, const double* d_in, uint64_t u,
                         const PerturbHdr& hdr, uint64_t nshared, double* d_out,
                         uint64_t ldo, uint32_t B, uint32_t v, double mag,
                         cudaStream_t st);

// OffsetExecutor (harness.cpp:167-186) on one provider's B x v outputs for
// the requests whose first id byte is < thr (256 = all).
void launch_offset_outputs(double* d_out, const uint8_t* d_reqids, uint32_t B, uint32_t v,
                           double offset, uint32_t thr, cudaStream_t st);

}  // namespace cg
