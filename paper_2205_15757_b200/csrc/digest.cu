// Certificate-digest kernels: SHA-256 chain jobs (request midstates, result
// leaves, single-attestation leaves, flat message batches) and Merkle roots.
//
// Reference: crypto::hash (proj/src/crypto.cpp:22-39), merkle::leaf_hash /
// Tree::build (proj/src/merkle.cpp:14-67), leaf constructions
// (proj/src/messages.cpp:204-341).
#include "digest.cuh"

#include <vector>
#include "sha256.cuh"

namespace cg {

// One thread per job. Latency-bound by design: a job is a Merkle-Damgard
// chain, so parallelism comes from the number of jobs (requests × providers),
// never from splitting a message. 32 jobs per warp, 2 warps per CTA keeps
// chains spread over many SMs (each chain runs at the single-warp issue rate).
__global__ void __launch_bounds__(128) chain_jobs_kernel(const ChainJob* jobs,
                                                        uint32_t n) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  const ChainJob& j = jobs[t];
  uint64_t digest_out = j.digest_out;
  if (j.skip_flag) {  // slot assigned on device (single attestation leaves)
    int32_t pos = *reinterpret_cast<const int32_t*>(j.skip_flag);
    if (pos < 0) return;
    digest_out += 32ull * (uint32_t)pos;
  }
  run_chain_job(j, digest_out);
}

// Flat byte messages (no f64 segment): the raw-segment fast run.
__global__ void __launch_bounds__(64) chain_jobs_raw_kernel(const ChainJob* jobs, uint32_t n) {
  uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= n) return;
  run_chain_job<CG_CHAIN_LOOP, true>(jobs[t], jobs[t].digest_out);
}

void launch_chain_jobs_raw(const ChainJob* d_jobs, uint32_t n, cudaStream_t st) {
  if (n == 0) return;
  chain_jobs_raw_kernel<<<(unsigned)ceil_div(n, 64), 64, 0, st>>>(d_jobs, n);
  CG_CHECK_LAUNCH();
}

void launch_chain_jobs(const ChainJob* d_jobs, uint32_t n, cudaStream_t st,
                       bool exclusive_sm) {
  if (n == 0) return;
  // exclusive launches: one warp per SMSP of a reserved SM (128 chains/CTA)
  const int tpb = exclusive_sm ? kChainExclusiveThreads : 64;
  // exclusive_sm: claim (unused) shared memory so the CTA can never share an
  // SM with a persistent GEMM CTA (~200 KB); long chains then run on their
  // own SMs instead of slowing one statically scheduled GEMM CTA.
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    CG_CUDA(cudaFuncSetAttribute(chain_jobs_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 kChainExclusiveSmem));
  });
  timer_begin(st, kTimeChain);
  chain_jobs_kernel<<<(unsigned)ceil_div(n, tpb), tpb, exclusive_sm ? kChainExclusiveSmem : 0,
                      st>>>(d_jobs, n);
  CG_CHECK_LAUNCH();
  timer_end(st, kTimeChain);
}

// ---------------------------------------------------------------------------
// Merkle roots. One CTA per tree; the level array lives in shared memory.
// Tree t has leaves leaf[off[t] .. off[t]+len[t]) (32-byte digests), or a
// device-resident count when count_dev != nullptr (the A tree, whose size the
// attestation manifest decides on device).
constexpr int kMerkleSmemLeaves = 8192;

__global__ void __launch_bounds__(256) merkle_tree_kernel(
    const uint8_t* __restrict__ leaves, const uint64_t* __restrict__ off,
    const uint64_t* __restrict__ len, const uint32_t* __restrict__ count_dev,
    uint64_t n_const, uint8_t* __restrict__ roots) {
  extern __shared__ __align__(16) uint8_t sm[];  // (n/2 + 1) × 32 bytes
  const uint32_t t = blockIdx.x;
  uint64_t n = count_dev ? count_dev[t] : (len ? len[t] : n_const);
  const uint8_t* L = leaves + 32 * (off ? off[t] : 0);
  uint8_t* out = roots + 32 * t;
  if (n == 0) {  // Tree::build throws on an empty list; the caller checks.
    if (threadIdx.x < 8) reinterpret_cast<uint32_t*>(out)[threadIdx.x] = 0;
    return;
  }
  if (n == 1) {
    if (threadIdx.x < 8)
      reinterpret_cast<uint32_t*>(out)[threadIdx.x] =
          reinterpret_cast<const uint32_t*>(L)[threadIdx.x];
    return;
  }
  // level 1 from global leaves
  uint64_t m = (n + 1) / 2;
  for (uint64_t i = threadIdx.x; i < m; i += blockDim.x) {
    if (2 * i + 1 < n) {
      sha256_internal_node(L + 64 * i, L + 64 * i + 32, sm + 32 * i);
    } else {
      const uint4* src = reinterpret_cast<const uint4*>(L + 64 * i);
      uint4* dst = reinterpret_cast<uint4*>(sm + 32 * i);
      dst[0] = src[0];
      dst[1] = src[1];
    }
  }
  __syncthreads();
  n = m;
  while (n > 1) {
    m = (n + 1) / 2;
    // in-place: node i reads 2i, 2i+1 and writes i; i <= 2i so process in
    // two phases to avoid read-after-overwrite races.
    uint4 tmp[2];
    bool have = false;
    uint64_t i = threadIdx.x;
    // each thread handles at most m/blockDim.x nodes; stage via registers
    for (uint64_t base = 0; base < m; base += blockDim.x) {
      i = base + threadIdx.x;
      have = i < m;
      if (have) {
        if (2 * i + 1 < n) {
          uint8_t h[32];
          sha256_internal_node(sm + 64 * i, sm + 64 * i + 32, h);
          tmp[0] = reinterpret_cast<uint4*>(h)[0];
          tmp[1] = reinterpret_cast<uint4*>(h)[1];
        } else {
          tmp[0] = reinterpret_cast<uint4*>(sm + 64 * i)[0];
          tmp[1] = reinterpret_cast<uint4*>(sm + 64 * i)[1];
        }
      }
      __syncthreads();
      if (have) {
        reinterpret_cast<uint4*>(sm + 32 * i)[0] = tmp[0];
        reinterpret_cast<uint4*>(sm + 32 * i)[1] = tmp[1];
      }
      __syncthreads();
    }
    n = m;
  }
  if (threadIdx.x < 8)
    reinterpret_cast<uint32_t*>(out)[threadIdx.x] =
        reinterpret_cast<const uint32_t*>(sm)[threadIdx.x];
}

// One Merkle level in global memory for trees too big for one CTA.
__global__ void merkle_level_kernel(const uint8_t* __restrict__ in, uint64_t n,
                                    uint8_t* __restrict__ out) {
  uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint64_t m = (n + 1) / 2;
  if (i >= m) return;
  if (2 * i + 1 < n) {
    sha256_internal_node(in + 64 * i, in + 64 * i + 32, out + 32 * i);
  } else {
    const uint4* s = reinterpret_cast<const uint4*>(in + 64 * i);
    uint4* d = reinterpret_cast<uint4*>(out + 32 * i);
    d[0] = s[0];
    d[1] = s[1];
  }
}

void launch_merkle_trees(const uint8_t* d_leaves, const uint64_t* d_off,
                         const uint64_t* d_len, const uint32_t* d_count,
                         uint32_t ntrees, uint64_t max_leaves, uint8_t* d_roots,
                         cudaStream_t st, uint64_t n_const) {
  if (ntrees == 0) return;
  if (max_leaves > kMerkleSmemLeaves)
    throw InvalidArgument("merkle_tree: too many leaves for one CTA");
  size_t smem = 32 * ((max_leaves + 1) / 2 + 1);
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    CG_CUDA(cudaFuncSetAttribute(merkle_tree_kernel,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize,
                                 32 * (kMerkleSmemLeaves / 2 + 1)));
  });
  merkle_tree_kernel<<<ntrees, 256, smem, st>>>(d_leaves, d_off, d_len,
                                                d_count, n_const, d_roots);
  CG_CHECK_LAUNCH();
}

size_t merkle_big_scratch_bytes(uint64_t n) { return 2 * 32 * ((n + 1) / 2 + 1); }

void launch_merkle_big(const uint8_t* d_leaves, uint64_t n, uint8_t* d_scratch,
                       uint8_t* d_root, cudaStream_t st) {
  if (n == 0) throw InvalidArgument("merkle: empty leaf list");
  uint8_t* bufs[2] = {d_scratch, d_scratch + 32 * ((n + 1) / 2 + 1)};
  const uint8_t* in = d_leaves;
  int which = 0;
  while (n > kMerkleSmemLeaves) {
    uint64_t m = (n + 1) / 2;
    merkle_level_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(in, n, bufs[which]);
    CG_CHECK_LAUNCH();
    in = bufs[which];
    which ^= 1;
    n = m;
  }
  launch_merkle_trees(in, nullptr, nullptr, nullptr, 1, n, d_root, st, n);
}

// ------------------------------------------------------ authentication paths
// Tree::build's level arrays in global memory (level 0 = the leaf hashes),
// then Tree::auth_path (merkle.cpp:69-84) for many indices at once, and
// get_merkle_root (merkle.cpp:86-93) for many (leaf hash, path) pairs: one
// thread per path, 2 compressions per step. kMaxPathSteps covers 2^64 leaves.
std::vector<uint64_t> launch_merkle_levels(const uint8_t* d_leaves, uint64_t n,
                                           uint8_t* d_levels, cudaStream_t st) {
  if (n == 0) throw InvalidArgument("merkle: empty leaf list");
  std::vector<uint64_t> off{0};
  CG_CUDA(cudaMemcpyAsync(d_levels, d_leaves, 32 * n, cudaMemcpyDeviceToDevice, st));
  uint64_t cur = 0;
  while (n > 1) {
    const uint64_t m = (n + 1) / 2;
    merkle_level_kernel<<<(unsigned)ceil_div(m, 256), 256, 0, st>>>(d_levels + 32 * cur, n,
                                                                      d_levels + 32 * (cur + n));
    CG_CHECK_LAUNCH();
    cur += n;
    off.push_back(cur);
    n = m;
  }
  return off;  // level l starts at node off[l]; the root is the last node
}

uint64_t merkle_levels_nodes(uint64_t n) {
  uint64_t t = 0;
  while (n > 1) {
    t += n;
    n = (n + 1) / 2;
  }
  return t + 1;
}

__global__ void auth_path_kernel(const uint8_t* __restrict__ levels, PathLevels lv,
                                 const uint64_t* __restrict__ idx, uint32_t count,
                                 uint8_t* __restrict__ sib, uint8_t* __restrict__ sides,
                                 uint32_t* __restrict__ lens) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  uint64_t i = idx[t];
  uint32_t k = 0;
  uint64_t n = lv.n;
  for (int l = 0; l + 1 < lv.nlevels; l++) {
    const uint8_t* level = levels + 32 * lv.off[l];
    const uint8_t* s = nullptr;
    uint8_t side = 0;
    if (i & 1) {
      s = level + 32 * (i - 1);
      side = 0;  // Side::left
    } else if (i + 1 < n) {
      s = level + 32 * (i + 1);
      side = 1;  // Side::right
    }
    if (s) {
      const uint4* src = reinterpret_cast<const uint4*>(s);
      uint4* dst = reinterpret_cast<uint4*>(sib + ((uint64_t)t * kMaxPathSteps + k) * 32);
      dst[0] = src[0];
      dst[1] = src[1];
      sides[(uint64_t)t * kMaxPathSteps + k] = side;
      k++;
    }
    i >>= 1;
    n = (n + 1) / 2;
  }
  lens[t] = k;
}

__global__ void path_root_kernel(const uint8_t* __restrict__ leaf_hashes,
                                 const uint8_t* __restrict__ sib,
                                 const uint8_t* __restrict__ sides,
                                 const uint32_t* __restrict__ lens, uint32_t count,
                                 uint8_t* __restrict__ roots) {
  const uint32_t t = blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= count) return;
  __align__(16) uint8_t h[32];
  reinterpret_cast<uint4*>(h)[0] = reinterpret_cast<const uint4*>(leaf_hashes + 32ull * t)[0];
  reinterpret_cast<uint4*>(h)[1] = reinterpret_cast<const uint4*>(leaf_hashes + 32ull * t)[1];
  const uint32_t k = lens[t] < kMaxPathSteps ? lens[t] : kMaxPathSteps;
  for (uint32_t s = 0; s < k; s++) {
    const uint8_t* sb = sib + ((uint64_t)t * kMaxPathSteps + s) * 32;
    __align__(16) uint8_t o[32];
    if (sides[(uint64_t)t * kMaxPathSteps + s] == 0) sha256_internal_node(sb, h, o);
    else sha256_internal_node(h, sb, o);
    reinterpret_cast<uint4*>(h)[0] = reinterpret_cast<uint4*>(o)[0];
    reinterpret_cast<uint4*>(h)[1] = reinterpret_cast<uint4*>(o)[1];
  }
  reinterpret_cast<uint4*>(roots + 32ull * t)[0] = reinterpret_cast<uint4*>(h)[0];
  reinterpret_cast<uint4*>(roots + 32ull * t)[1] = reinterpret_cast<uint4*>(h)[1];
}

void launch_auth_paths(const uint8_t* d_levels, const std::vector<uint64_t>& off, uint64_t n,
                       const uint64_t* d_idx, uint32_t count, uint8_t* d_sib, uint8_t* d_sides,
                       uint32_t* d_lens, cudaStream_t st) {
  if (count == 0) return;
  PathLevels lv{};
  lv.n = n;
  lv.nlevels = (int)off.size();
  if (lv.nlevels > kMaxPathSteps + 1) throw InvalidArgument("merkle: tree too deep");
  for (size_t l = 0; l < off.size(); l++) lv.off[l] = off[l];
  auth_path_kernel<<<(unsigned)ceil_div(count, 128), 128, 0, st>>>(d_levels, lv, d_idx, count,
                                                                   d_sib, d_sides, d_lens);
  CG_CHECK_LAUNCH();
}

void launch_path_roots(const uint8_t* d_leaf_hashes, const uint8_t* d_sib, const uint8_t* d_sides,
                       const uint32_t* d_lens, uint32_t count, uint8_t* d_roots,
                       cudaStream_t st) {
  if (count == 0) return;
  path_root_kernel<<<(unsigned)ceil_div(count, 128), 128, 0, st>>>(d_leaf_hashes, d_sib, d_sides,
                                                                   d_lens, count, d_roots);
  CG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// PerturbingExecutor lane offsets (proj/src/model.cpp:82-105). Message per
// (request i, lane) = hdr(44: u64 node || model_digest || u32 count) ||
// f64_list body(8u) || u64 lane. The first nshared whole blocks are common
// to every lane of a request and were absorbed by a chain job into mid[i];
// each thread here finishes one (request, lane): the last P mod 64 prefix
// bytes, the lane, FIPS padding (1-2 blocks), then applies the offset to
// out[i][lane] with explicitly rounded f64 ops (no FMA contraction), in the
// reference's order: unit = raw / (2^64 - 1); out += (2 unit - 1) * mag.
__global__ void __launch_bounds__(128) perturb_tail_kernel(
    const uint32_t* __restrict__ mid, const double* __restrict__ in, uint64_t u,
    PerturbHdr hdr, uint64_t nshared, double* __restrict__ out, uint64_t ldo,
    uint32_t B, uint32_t v, double mag) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (uint64_t)B * v) return;
  const uint32_t i = (uint32_t)(t / v);
  const uint64_t lane = t % v;
  uint32_t s[8];
  if (nshared) {
#pragma unroll
    for (int k = 0; k < 8; k++) s[k] = mid[8ull * i + k];
  } else {
    sha256_iv(s);
  }
  const double* x = in + (uint64_t)i * u;
  const uint64_t P = 44 + 8 * u, total = P + 8;
  const uint64_t nblk = (total + 9 + 63) / 64;
  for (uint64_t blk = nshared; blk < nblk; blk++) {
    uint32_t w[16];
    for (int q = 0; q < 16; q++) {
      uint32_t word = 0;
      for (int b = 0; b < 4; b++) {
        const uint64_t pos = blk * 64 + 4 * q + b;
        uint32_t byte;
        if (pos < 44) {
          byte = hdr.b[pos];
        } else if (pos < P) {
          const uint64_t r = pos - 44;
          const uint64_t bits = __double_as_longlong(__ldg(x + (r >> 3)));
          byte = (uint32_t)(bits >> (56 - 8 * (r & 7))) & 0xffu;
        } else if (pos < total) {
          byte = (uint32_t)(lane >> (56 - 8 * (pos - P))) & 0xffu;
        } else if (pos == total) {
          byte = 0x80u;
        } else if (pos >= nblk * 64 - 8) {
          byte = (uint32_t)((total * 8) >> (56 - 8 * (pos - (nblk * 64 - 8)))) & 0xffu;
        } else {
          byte = 0;
        }
        word = (word << 8) | byte;
      }
      w[q] = word;
    }
    sha256_compress<true>(s, w);
  }
  const uint64_t raw = ((uint64_t)s[0] << 32) | s[1];
  const double unit = __ddiv_rn(__ull2double_rn(raw), 18446744073709551615.0);
  const double off = __dmul_rn(__dsub_rn(__dmul_rn(2.0, unit), 1.0), mag);
  double* y = out + (uint64_t)i * ldo + lane;
  *y = __dadd_rn(*y, off);
}

void launch_perturb_tail(const uint32_t* d_mid, const double* d_in, uint64_t u,
                         const PerturbHdr& hdr, uint64_t nshared, double* d_out,
                         uint64_t ldo, uint32_t B, uint32_t v, double mag,
                         cudaStream_t st) {
  const uint64_t n = (uint64_t)B * v;
  if (n == 0) return;
  perturb_tail_kernel<<<(unsigned)ceil_div(n, 128), 128, 0, st>>>(d_mid, d_in, u, hdr, nshared,
                                                                d_out, ldo, B, v, mag);
  CG_CHECK_LAUNCH();
}

// OffsetExecutor (proj/src/harness.cpp:167-186, the corrupt_result fault):
// every output lane of the faulty node += offset, applied after the
// PerturbingExecutor it wraps (harness.cpp:255-261). Fault injection for a
// fraction of requests: request k is hit when its first request-id byte is
// below `thr` (thr = 256: every request, exactly the reference's executor).
__global__ void offset_outputs_kernel(double* __restrict__ out, const uint8_t* __restrict__ reqids,
                                      uint32_t B, uint32_t v, double offset, uint32_t thr) {
  const uint64_t i = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= (uint64_t)B * v) return;
  const uint32_t k = (uint32_t)(i / v);
  if ((uint32_t)reqids[32ull * k] < thr) out[i] = __dadd_rn(out[i], offset);
}

void launch_offset_outputs(double* d_out, const uint8_t* d_reqids, uint32_t B, uint32_t v,
                           double offset, uint32_t thr, cudaStream_t st) {
  const uint64_t n = (uint64_t)B * v;
  if (n == 0 || thr == 0) return;
  offset_outputs_kernel<<<(unsigned)ceil_div(n, 256), 256, 0, st>>>(d_out, d_reqids, B, v, offset,
                                                                    thr);
  CG_CHECK_LAUNCH();
}

// ---------------------------------------------------------------------------
// encode_results (proj/src/messages.cpp:48-50): u32be count || per result
// InferenceResult::encode (proj/src/domain.cpp:218-225) = request_id[32] ||
// u64 node || str(group) || u64 version || f64_list(output) || digest[32],
// all big-endian. Fixed stride 88 + gl + 8v per result; one CTA per result,
// threads stride the output doubles (byte stores: the f64 list starts at an
// arbitrary offset).
__global__ void __launch_bounds__(128) encode_results_kernel(
    const uint8_t* __restrict__ reqids, const double* __restrict__ outs, uint32_t B, uint32_t v,
    uint64_t node, const uint8_t* __restrict__ gid, uint32_t gl, uint64_t version,
    Digest32 model_digest, uint8_t* __restrict__ dst) {
  const uint32_t k = blockIdx.x;
  const uint64_t stride = 88ull + gl + 8ull * v;
  uint8_t* o = dst + 4 + stride * k;
  if (k == 0 && threadIdx.x < 4) dst[threadIdx.x] = (uint8_t)(B >> (24 - 8 * threadIdx.x));
  const uint32_t hdr = 32 + 8 + 4 + gl + 8 + 4;  // bytes before the doubles
  for (uint32_t t = threadIdx.x; t < hdr; t += blockDim.x) {
    uint8_t b;
    if (t < 32) b = reqids[32ull * k + t];
    else if (t < 40) b = (uint8_t)(node >> (56 - 8 * (t - 32)));
    else if (t < 44) b = (uint8_t)(gl >> (24 - 8 * (t - 40)));
    else if (t < 44 + gl) b = gid[t - 44];
    else if (t < 52 + gl) b = (uint8_t)(version >> (56 - 8 * (t - 44 - gl)));
    else b = (uint8_t)(v >> (24 - 8 * (t - 52 - gl)));
    o[t] = b;
  }
  const double* y = outs + (uint64_t)k * v;
  uint8_t* od = o + hdr;
  for (uint32_t i = threadIdx.x; i < v; i += blockDim.x) {
    const uint64_t bits = __double_as_longlong(y[i]);
#pragma unroll
    for (int q = 0; q < 8; q++) od[8ull * i + q] = (uint8_t)(bits >> (56 - 8 * q));
  }
  if (threadIdx.x < 32) od[8ull * v + threadIdx.x] = model_digest.b[threadIdx.x];
}

void launch_encode_results(const uint8_t* d_reqids, const double* d_outs, uint32_t B, uint32_t v,
                           uint64_t node, const uint8_t* d_gid, uint32_t gl, uint64_t version,
                           const Digest32& model_digest, uint8_t* d_dst, cudaStream_t st) {
  if (B == 0) return;
  encode_results_kernel<<<B, 128, 0, st>>>(d_reqids, d_outs, B, v, node, d_gid, gl, version,
                                           model_digest, d_dst);
  CG_CHECK_LAUNCH();
}

}  // namespace cg
