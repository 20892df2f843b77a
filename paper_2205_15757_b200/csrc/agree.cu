// Agreement, label vote, attestation manifest, softmax/top-k and the fp64
// LinearToyModel executor.
//
// Reference semantics (bit-exact targets):
//   distance::delta / select_quorum   proj/src/distance.cpp:70-216
//   argmax / ensemble_label           proj/src/experiments.cpp:99-125
//   try_attest manifest               proj/src/coordinator.cpp:774-832
//   LinearToyModel::run               proj/src/model.cpp:12-36
// Every fp64 reduction that the reference performs sequentially is kept
// sequential (and un-fused: __dmul_rn/__dadd_rn) so decisions match bit for
// bit; parallelism comes from requests, pairs and subsets instead.
#include "agree.cuh"
#include "sha256.cuh"

namespace cg {

struct Cand {
  uint32_t valid, size, mask;
  double diam;
};

// better(a, b) of distance.cpp:128-134 on subset masks (positions ascend
// with node ids, so the sorted-tuple order is decided by the lowest bit of
// the symmetric difference).
__device__ __forceinline__ bool cand_better(const Cand& a, const Cand& b) {
  if (!a.valid) return false;
  if (!b.valid) return true;
  if (a.size != b.size) return a.size > b.size;
  if (a.diam != b.diam) return a.diam < b.diam;
  uint32_t d = a.mask ^ b.mask;
  return d && (a.mask & (d & (0u - d)));
}

__device__ __forceinline__ Cand shfl_cand(const Cand& c, int src) {
  Cand o;
  o.valid = __shfl_sync(0xffffffffu, c.valid, src);
  o.size = __shfl_sync(0xffffffffu, c.size, src);
  o.mask = __shfl_sync(0xffffffffu, c.mask, src);
  o.diam = __shfl_sync(0xffffffffu, c.diam, src);
  return o;
}

constexpr int kQThreads = 128;
constexpr int kMaxM = 20;
constexpr int kQChunk = 64;                                            // lanes per smem chunk
constexpr int kQPairsPerThread = (kMaxM * (kMaxM - 1) / 2 + kQThreads - 1) / kQThreads;
constexpr int kQPrefetch = (kMaxM * kQChunk + kQThreads - 1) / kQThreads;

// metric 1 (max_minus_min) is defined on scalars only: |x0 - y0|
__device__ __forceinline__ double rows_first(const double* outs, const uint32_t* nodes, int i,
                                             uint64_t ps, uint32_t k, uint64_t rs) {
  return __ldg(outs + nodes[i] * ps + k * rs);
}

// One CTA per request. outs(k, p, i) = outs[p*ps + k*rs + i].
__global__ void __launch_bounds__(kQThreads) select_quorum_kernel(
    const double* __restrict__ outs, uint64_t ps, uint64_t rs,
    const uint32_t* __restrict__ present, const double* __restrict__ eps,
    uint32_t R, uint32_t n, uint32_t f, uint32_t v, uint32_t metric,
    uint32_t* __restrict__ selected, double* __restrict__ diameter,
    uint8_t* __restrict__ satisfied, int8_t* __restrict__ status,
    int64_t* __restrict__ label) {
  __shared__ double dist[kMaxM * kMaxM];
  __shared__ uint32_t nodes[kMaxM];
  __shared__ Cand warp_best[kQThreads / 32];
  __shared__ int s_m, s_bad;
  __shared__ uint32_t s_arg[kMaxM];
  __shared__ double s_argv[kMaxM];
  const uint32_t k = blockIdx.x;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    uint32_t pm = present ? present[k] : ((n >= 32) ? 0xffffffffu : ((1u << n) - 1));
    int m = 0, bad = 0;
    // select_quorum argument checks (distance.cpp:141-165)
    if (n == 0 || f >= n) bad = 1;
    if (n < 32 && (pm >> n)) bad = 1;  // node index out of range
    if (v == 0) bad = 1;               // empty result vector
    for (uint32_t i = 0; i < 32; i++)
      if (pm >> i & 1) {
        if (m < kMaxM) nodes[m] = i;
        m++;
      }
    if (!bad && (uint32_t)m < n - f) bad = 1;  // fewer than N-f present
    if (m > kMaxM) bad = 1;                    // too many results
    if (!bad && m >= 2 && metric == 1 && v != 1) bad = 1;  // scalar metric
    if (!bad && m >= 2 && metric > 2) bad = 1;             // unknown metric
    s_m = m;
    s_bad = bad;
  }
  __syncthreads();
  if (s_bad) {
    if (tid == 0) {
      status[k] = -1;
      selected[k] = 0;
      diameter[k] = 0.0;
      satisfied[k] = 0;
      if (label) label[k] = -1;
    }
    return;
  }
  const int m = s_m;
  const uint32_t need = n - f;
  // Pairwise distances once (distance.cpp:167-174) plus every row's argmax
  // (experiments.cpp:99-101), in one pass: the m rows stream through shared
  // memory in chunks of kQChunk lanes (coalesced loads, next chunk prefetched
  // into registers), one thread per pair keeps its sequential un-fused sum,
  // threads m.. of the last warp scan rows for the first maximum.
  extern __shared__ double q_rows[];  // 2 buffers x m rows x (kQChunk + 1)
  const int npairs = m * (m - 1) / 2;
  const int stride = kQChunk + 1;     // +1: rows land on distinct banks
  int pi[kQPairsPerThread], pj[kQPairsPerThread];
  double acc[kQPairsPerThread];
#pragma unroll
  for (int q = 0; q < kQPairsPerThread; q++) {
    const int pr = tid + q * kQThreads;
    int i = 0, rem = pr < npairs ? pr : 0;
    while (rem >= m - 1 - i) { rem -= m - 1 - i; i++; }
    pi[q] = i;
    pj[q] = i + 1 + rem;
    acc[q] = 0.0;
  }
  const int arow = tid - (kQThreads - 32);  // argmax row of this thread (last warp)
  double abv = 0.0;
  uint32_t abi = 0;
  if (arow >= 0 && arow < m) abv = __ldg(outs + nodes[arow] * ps + k * rs);
  const int per = (m * kQChunk + kQThreads - 1) / kQThreads;  // prefetch slots
  double pf[kQPrefetch];
  auto fetch = [&](uint32_t c0) {
#pragma unroll
    for (int q = 0; q < kQPrefetch; q++) {
      const int e = tid + q * kQThreads;
      if (q < per && e < m * kQChunk) {
        const int r = e / kQChunk, t = e % kQChunk;
        pf[q] = (c0 + t < v) ? __ldg(outs + nodes[r] * ps + k * rs + c0 + t) : 0.0;
      }
    }
  };
  auto stash = [&](int buf) {
#pragma unroll
    for (int q = 0; q < kQPrefetch; q++) {
      const int e = tid + q * kQThreads;
      if (q < per && e < m * kQChunk)
        q_rows[(buf * m + e / kQChunk) * stride + e % kQChunk] = pf[q];
    }
  };
  fetch(0);
  stash(0);
  __syncthreads();
  int buf = 0;
  for (uint32_t c0 = 0; c0 < v; c0 += kQChunk) {
    const bool more = c0 + kQChunk < v;
    if (more) fetch(c0 + kQChunk);
    const int len = (int)min((uint32_t)kQChunk, v - c0);
    const double* rows = q_rows + buf * m * stride;
#pragma unroll
    for (int q = 0; q < kQPairsPerThread; q++) {
      if (tid + q * kQThreads >= npairs) continue;
      const double* x = rows + pi[q] * stride;
      const double* y = rows + pj[q] * stride;
      double a = acc[q];
      if (metric == 0) {
        for (int t = 0; t < len; t++) {
          const double d = __dsub_rn(x[t], y[t]);
          a = __dadd_rn(a, __dmul_rn(d, d));
        }
      } else {
        for (int t = 0; t < len; t++) {
          const double d = fabs(__dsub_rn(x[t], y[t]));
          a = (a < d) ? d : a;
        }
      }
      acc[q] = a;
    }
    if (arow >= 0 && arow < m) {
      const double* x = rows + arow * stride;
      for (int t = 0; t < len; t++)
        if (abv < x[t]) {  // std::max_element: first maximum
          abv = x[t];
          abi = c0 + t;
        }
    }
    if (more) stash(buf ^ 1);
    __syncthreads();
    buf ^= 1;
  }
#pragma unroll
  for (int q = 0; q < kQPairsPerThread; q++) {
    if (tid + q * kQThreads >= npairs) continue;
    double d = acc[q];
    if (metric == 0) d = __dsqrt_rn(d);
    else if (metric == 1) d = fabs(__dsub_rn(rows_first(outs, nodes, pi[q], ps, k, rs),
                                             rows_first(outs, nodes, pj[q], ps, k, rs)));
    dist[pi[q] * kMaxM + pj[q]] = d;
    dist[pj[q] * kMaxM + pi[q]] = d;
  }
  if (arow >= 0 && arow < m) {
    s_arg[arow] = abi;
    s_argv[arow] = abv;
  }
  __syncthreads();
  // exhaustive subset scan (distance.cpp:178-205), masks striped over threads
  const double e = eps[k];
  Cand best{0, 0, 0, 0.0};
  const uint32_t limit = 1u << m;
  for (uint32_t mask = 1 + tid; mask < limit; mask += kQThreads) {
    uint32_t size = __popc(mask);
    if (size < need) continue;
    double dm = 0.0;
    bool ok = true;
    for (int i = 0; i < m && ok; i++) {
      if (!(mask >> i & 1)) continue;
      for (int j = i + 1; j < m; j++) {
        if (!(mask >> j & 1)) continue;
        double x = dist[i * kMaxM + j];
        dm = (dm < x) ? x : dm;
        if (dm > e) { ok = false; break; }
      }
    }
    if (!ok) continue;
    Cand c{1, size, mask, dm};
    if (cand_better(c, best)) best = c;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    Cand other = shfl_cand(best, lane ^ o);
    if (cand_better(other, best)) best = other;
  }
  if (lane == 0) warp_best[warp] = best;
  __syncthreads();
  if (tid == 0) {
    for (int w = 1; w < kQThreads / 32; w++)
      if (cand_better(warp_best[w], best)) best = warp_best[w];
    warp_best[0] = best;
    uint32_t sel = 0;
    if (best.valid)
      for (int i = 0; i < m; i++)
        if (best.mask >> i & 1) sel |= 1u << nodes[i];
    status[k] = 0;
    selected[k] = sel;
    diameter[k] = best.valid ? best.diam : 0.0;
    satisfied[k] = best.valid ? 1 : 0;
  }
  if (!label) return;
  __syncthreads();
  // ensemble_label (experiments.cpp:106-125) over the selected members:
  // argmax per member (first maximum), votes > f, highest confidence wins.
  best = warp_best[0];
  if (!best.valid) {
    if (tid == 0) label[k] = -1;
    return;
  }
  __syncthreads();
  if (tid == 0) {
    int64_t win = -1;
    double win_conf = -1.0;
    // labels ascending; count and max confidence per label
    for (int i = 0; i < m; i++) {
      if (!(best.mask >> i & 1)) continue;
      uint32_t l = s_arg[i];
      bool seen_before = false;
      for (int q = 0; q < i; q++)
        if ((best.mask >> q & 1) && s_arg[q] == l) seen_before = true;
      if (seen_before) continue;
      uint32_t cnt = 0;
      double conf = 0.0;
      for (int q = 0; q < m; q++)
        if ((best.mask >> q & 1) && s_arg[q] == l) {
          cnt++;
          conf = (conf < s_argv[q]) ? s_argv[q] : conf;
        }
      if (cnt <= f) continue;
      // ascending label scan with strict >: a smaller label wins ties
      if (conf > win_conf || (conf == win_conf && win >= 0 && (int64_t)l < win)) {
        win = l;
        win_conf = conf;
      }
    }
    label[k] = win;
  }
}

void launch_select_quorum(const double* outs, uint64_t ps, uint64_t rs,
                          const uint32_t* present, const double* eps,
                          uint32_t R, uint32_t n, uint32_t f, uint32_t v,
                          uint32_t metric, uint32_t* selected, double* diameter,
                          uint8_t* satisfied, int8_t* status, int64_t* label,
                          cudaStream_t st) {
  if (R == 0) return;
  const size_t smem = 2ull * kMaxM * (kQChunk + 1) * sizeof(double);
  select_quorum_kernel<<<R, kQThreads, smem, st>>>(outs, ps, rs, present, eps, R,
                                                n, f, v, metric, selected,
                                                diameter, satisfied, status,
                                                label);
  CG_CHECK_LAUNCH();
}

// ------------------------------------------- agreement, throughput form (C5)
// One thread per request, for large batches with all M <= 8 results present:
// the thread streams its M rows once (16-byte loads, each row sequential so
// every sector is consumed whole) and keeps all M(M-1)/2 pair accumulators,
// the per-row argmax and the running state in registers. The sums stay
// sequential and un-fused per pair, so distances equal distance.cpp:70-117
// bit for bit; the subset search visits sizes M, M-1, ... and stops at the
// first size with a valid subset, which is the same winner as the exhaustive
// scan of distance.cpp:178-205 (size is the first criterion). Optional
// epilogue: the compact label digest (sha256_label_digest) per request.
template <int M>
__device__ __forceinline__ void agree_step(const double (&x)[M], uint32_t t, int metric,
                                           double (&acc)[M * (M - 1) / 2], double (&bv)[M],
                                           uint32_t (&bi)[M]) {
  int p = 0;
#pragma unroll
  for (int i = 0; i < M; i++)
#pragma unroll
    for (int j = i + 1; j < M; j++, p++) {
      double d = __dsub_rn(x[i], x[j]);
      if (metric == 0) {
        acc[p] = __dadd_rn(acc[p], __dmul_rn(d, d));
      } else {
        d = fabs(d);
        acc[p] = (acc[p] < d) ? d : acc[p];
      }
    }
#pragma unroll
  for (int i = 0; i < M; i++)
    if (bv[i] < x[i]) {  // std::max_element: first maximum
      bv[i] = x[i];
      bi[i] = t;
    }
}

__device__ __forceinline__ double ld_stream(const double* p) {
  double v;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(v) : "l"(p));
  return v;
}
// 256-bit load (sm_100): one whole 32-byte sector per lane, so a warp's 32
// strided rows cost 32 L1 wavefronts per 1 KB instead of per 512 B.
__device__ __forceinline__ void ld_stream4(const double* p, double& a, double& b, double& c,
                                           double& d) {
  asm volatile("ld.global.nc.L1::no_allocate.v4.f64 {%0, %1, %2, %3}, [%4];"
               : "=d"(a), "=d"(b), "=d"(c), "=d"(d) : "l"(p));
}
__device__ __forceinline__ double2 ld_stream2(const double* p) {
  double2 v;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0, %1}, [%2];"
               : "=d"(v.x), "=d"(v.y) : "l"(p));
  return v;
}

template <int M>
__global__ void __launch_bounds__(128) agree_rows_kernel(
    const double* __restrict__ outs, uint64_t ps, uint64_t rs, const double* __restrict__ eps,
    uint32_t R, uint32_t f, uint32_t v, int metric, int vec,
    const uint8_t* __restrict__ req_ids, uint64_t version, uint32_t* __restrict__ selected,
    double* __restrict__ diameter, uint8_t* __restrict__ satisfied,
    int8_t* __restrict__ status, int64_t* __restrict__ label, uint8_t* __restrict__ digest) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= R) return;
  constexpr int P = M * (M - 1) / 2;
  const double* row = outs + (uint64_t)k * rs;
  double acc[P], bv[M];
  uint32_t bi[M];
#pragma unroll
  for (int p = 0; p < P; p++) acc[p] = 0.0;
#pragma unroll
  for (int i = 0; i < M; i++) {
    bv[i] = __ldg(row + i * ps);
    bi[i] = 0;
  }
  uint32_t t = 0;
  if (vec >= 2) {  // 4 lanes per trip: M 32-byte (or 2M 16-byte) loads in flight
#pragma unroll 1
    for (; t + 4 <= v; t += 4) {
      double q[4][M];
#pragma unroll
      for (int i = 0; i < M; i++) {
        if (vec == 4) {
          ld_stream4(row + i * ps + t, q[0][i], q[1][i], q[2][i], q[3][i]);
        } else {
          double2 a = ld_stream2(row + i * ps + t), b = ld_stream2(row + i * ps + t + 2);
          q[0][i] = a.x;
          q[1][i] = a.y;
          q[2][i] = b.x;
          q[3][i] = b.y;
        }
      }
#pragma unroll
      for (int e = 0; e < 4; e++) agree_step<M>(q[e], t + e, metric, acc, bv, bi);
    }
  }
#pragma unroll 1
  for (; t < v; t++) {
    double x[M];
#pragma unroll
    for (int i = 0; i < M; i++) x[i] = ld_stream(row + i * ps + t);
    agree_step<M>(x, t, metric, acc, bv, bi);
  }
  if (metric == 0) {
#pragma unroll
    for (int p = 0; p < P; p++) acc[p] = __dsqrt_rn(acc[p]);
  }
  // subset search, sizes descending (need = n - f with n = M)
  const double e = eps[k];
  const int need = M - (int)f;
  Cand best{0, 0, 0, 0.0};
  for (int s = M; s >= need && !best.valid; s--) {
    // the size-s subsets in increasing order (Gosper's next combination)
#pragma unroll 1
    for (uint32_t mask = (1u << s) - 1; mask < (1u << M);) {
      const uint32_t cur = mask;
      {
        const uint32_t c = mask & (0u - mask), r = mask + c;
        mask = (((r ^ mask) >> 2) >> (__ffs(c) - 1)) | r;
      }
      double dm = 0.0;
      bool ok = true;
      int p = 0;
#pragma unroll
      for (int i = 0; i < M; i++)
#pragma unroll
        for (int j = i + 1; j < M; j++, p++)
          if (ok && (cur >> i & 1) && (cur >> j & 1)) {
            dm = (dm < acc[p]) ? acc[p] : dm;
            if (dm > e) ok = false;
          }
      if (!ok) continue;
      Cand c{1, (uint32_t)s, cur, dm};
      if (cand_better(c, best)) best = c;
    }
  }
  status[k] = 0;
  selected[k] = best.valid ? best.mask : 0;
  diameter[k] = best.valid ? best.diam : 0.0;
  satisfied[k] = best.valid ? 1 : 0;
  int64_t win = -1;
  if (best.valid) {  // ensemble_label over the quorum members
    double win_conf = -1.0;
#pragma unroll
    for (int i = 0; i < M; i++) {
      if (!(best.mask >> i & 1)) continue;
      const uint32_t l = bi[i];
      bool seen = false;
#pragma unroll
      for (int q = 0; q < i; q++)
        if ((best.mask >> q & 1) && bi[q] == l) seen = true;
      if (seen) continue;
      uint32_t cnt = 0;
      double conf = 0.0;
#pragma unroll
      for (int q = 0; q < M; q++)
        if ((best.mask >> q & 1) && bi[q] == l) {
          cnt++;
          conf = (conf < bv[q]) ? bv[q] : conf;
        }
      if (cnt <= f) continue;
      if (conf > win_conf || (conf == win_conf && win >= 0 && (int64_t)l < win)) {
        win = l;
        win_conf = conf;
      }
    }
  }
  if (label) label[k] = win;
  if (digest) sha256_label_digest(req_ids + 32ull * k, version, win, digest + 32ull * k);
}

bool agree_rows_eligible(uint32_t R, uint32_t n, uint32_t f, uint32_t v, uint32_t metric,
                         const uint32_t* present) {
  return present == nullptr && n >= 2 && n <= 8 && f < n && v >= 1 &&
         (metric == 0 || metric == 2) && R >= kAgreeRowsMinBatch;
}

void launch_agree_rows(const double* outs, uint64_t ps, uint64_t rs, const double* eps,
                       uint32_t R, uint32_t n, uint32_t f, uint32_t v, uint32_t metric,
                       const uint8_t* req_ids, uint64_t version, uint32_t* selected,
                       double* diameter, uint8_t* satisfied, int8_t* status, int64_t* label,
                       uint8_t* digest, cudaStream_t st) {
  if (R == 0) return;
  // widest row load every row start allows (32 B, 16 B, else scalar)
  const int vec = ((ps | rs) % 4 == 0 && (uintptr_t)outs % 32 == 0)   ? 4
                  : ((ps | rs) % 2 == 0 && (uintptr_t)outs % 16 == 0) ? 2
                                                                      : 1;
  const unsigned grid = (unsigned)ceil_div(R, 128);
#define CG_AGREE(MM)                                                                    \
  case MM:                                                                              \
    agree_rows_kernel<MM><<<grid, 128, 0, st>>>(outs, ps, rs, eps, R, f, v, (int)metric, \
                                                vec, req_ids, version, selected,       \
                                                diameter, satisfied, status, label,     \
                                                digest);                                \
    break;
  switch (n) {
    CG_AGREE(2) CG_AGREE(3) CG_AGREE(4) CG_AGREE(5) CG_AGREE(6) CG_AGREE(7) CG_AGREE(8)
    default: throw InvalidArgument("agree_rows: n out of range");
  }
#undef CG_AGREE
  CG_CHECK_LAUNCH();
}

// Compact label digests alone (labels already on the device).
__global__ void label_digest_kernel(const uint8_t* __restrict__ req_ids,
                                    const int64_t* __restrict__ label, uint32_t R,
                                    uint64_t version, uint8_t* __restrict__ out) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k < R) sha256_label_digest(req_ids + 32ull * k, version, label[k], out + 32ull * k);
}

void launch_label_digest(const uint8_t* req_ids, const int64_t* label, uint32_t R,
                         uint64_t version, uint8_t* out, cudaStream_t st) {
  if (R == 0) return;
  label_digest_kernel<<<(unsigned)ceil_div(R, 128), 128, 0, st>>>(req_ids, label, R, version,
                                                                  out);
  CG_CHECK_LAUNCH();
}

// ----------------------------------------------------- attestation manifest
// Single CTA. Manifest order (coordinator.cpp:774-832): whole_batch leaves
// by node, then single leaves by (op, node), then failure leaves by op.
// Whole-batch and failure leaf hashes are written here; single leaves are
// long chains (the full request is re-hashed under tag 0x53), so this kernel
// only assigns their manifest slots (single_pos) for the chain-job kernel.

__device__ void sha256_local(const uint8_t* m, uint32_t len, uint8_t* out) {
  uint32_t s[8], w[16];
  sha256_iv(s);
  uint32_t nblk = (len + 9 + 63) / 64;
  for (uint32_t b = 0; b < nblk; b++) {
    for (int i = 0; i < 16; i++) {
      uint32_t x = 0;
      for (int t = 0; t < 4; t++) {
        uint32_t pos = b * 64 + 4 * i + t, byte = 0;
        if (pos < len) byte = m[pos];
        else if (pos == len) byte = 0x80;
        else if (pos >= nblk * 64 - 8) byte = (uint32_t)((uint64_t)len * 8 >> (56 - 8 * (pos - (nblk * 64 - 8)))) & 0xff;
        x = (x << 8) | byte;
      }
      w[i] = x;
    }
    sha256_compress(s, w);
  }
  store_digest(s, out);
}

constexpr int kManThreads = 1024;

__global__ void __launch_bounds__(kManThreads) attest_manifest_kernel(
    uint32_t B, uint32_t N, const uint32_t* __restrict__ sel,
    const uint8_t* __restrict__ sat, const uint8_t* __restrict__ r_roots,
    const uint8_t* __restrict__ req_ids, const uint8_t* __restrict__ gid,
    uint32_t gid_len, uint64_t version, uint8_t* __restrict__ a_leaves,
    int32_t* __restrict__ single_pos, int32_t* __restrict__ need53,
    uint8_t* __restrict__ kinds, uint32_t* __restrict__ m_nodes, uint32_t* __restrict__ m_ops,
    uint32_t* __restrict__ count, const uint8_t* __restrict__ has_outcome,
    const uint8_t* __restrict__ explicit_fail, int32_t* __restrict__ fail_pos) {
  // has_outcome == NULL: every op is an ok inference request (an outcome,
  // coordinator.cpp:738-771); ops without one (rejected requests, group
  // ops) neither restrict whole-batch attestation nor get single leaves,
  // and fail only with their explicit record (messages.cpp:299-312).
  auto outcome = [&](uint32_t k) { return has_outcome ? has_outcome[k] != 0 : true; };
  auto explicit_f = [&](uint32_t k) { return explicit_fail ? explicit_fail[k] != 0 : false; };
  __shared__ uint32_t s_whole;
  __shared__ uint32_t s_scan[kManThreads];
  __shared__ uint32_t s_carry_single, s_carry_fail;
  const int tid = threadIdx.x;
  if (tid == 0) { s_whole = 0xffffffffu; s_carry_single = 0; s_carry_fail = 0; }
  __syncthreads();
  uint32_t acc = 0xffffffffu;
  for (uint32_t k = tid; k < B; k += kManThreads)
    if (outcome(k)) acc &= sat[k] ? sel[k] : 0u;
  atomicAnd(&s_whole, acc);
  __syncthreads();
  const uint32_t all_nodes = (N >= 32) ? 0xffffffffu : ((1u << N) - 1);
  const uint32_t whole = (B ? s_whole : 0u) & all_nodes;
  const uint32_t nwhole = __popc(whole);
  // whole-batch leaves: H(0x00 || 0x57 || R root of node p)
  if (tid < 32 && (whole >> tid & 1)) {
    uint32_t pos = __popc(whole & ((1u << tid) - 1));
    sha256_tagged_digest_leaf(0x57, r_roots + 32 * tid, a_leaves + 32 * pos);
    kinds[pos] = 0;
    m_nodes[pos] = tid;
    m_ops[pos] = 0;
  }
  // total singles for the failure offset
  uint32_t local = 0;
  for (uint32_t k = tid; k < B; k += kManThreads)
    if (outcome(k) && sat[k]) local += __popc(sel[k] & ~whole);
  s_scan[tid] = local;
  __syncthreads();
  if (tid == 0) {
    uint32_t t = 0;
    for (int i = 0; i < kManThreads; i++) t += s_scan[i];
    s_carry_fail = t;
  }
  __syncthreads();
  const uint32_t nsingle = s_carry_fail;
  // ordered passes over chunks of kManThreads ops
  for (uint32_t base = 0; base < B; base += kManThreads) {
    uint32_t k = base + tid;
    uint32_t ns = 0, nf = 0;
    if (k < B) {
      if (outcome(k)) {
        if (sat[k]) ns = __popc(sel[k] & ~whole);
        else nf = 1;
      } else if (explicit_f(k)) {
        nf = 1;
      }
    }
    // exclusive scan of (ns | nf<<16) — B and N small enough for 16 bits
    s_scan[tid] = ns | (nf << 16);
    __syncthreads();
    for (int o = 1; o < kManThreads; o <<= 1) {
      uint32_t x = (tid >= o) ? s_scan[tid - o] : 0;
      __syncthreads();
      s_scan[tid] += x;
      __syncthreads();
    }
    uint32_t incl = s_scan[tid];
    uint32_t ex = incl - (ns | (nf << 16));
    uint32_t spos = nwhole + s_carry_single + (ex & 0xffff);
    uint32_t fpos = nwhole + nsingle + s_carry_fail - nsingle + (ex >> 16);
    if (k < B) {
      for (uint32_t p = 0; p < N; p++) single_pos[k * N + p] = -1;
      // request k's single leaves H(0x00||0x53||req||res) share one request
      // midstate, computed only when k has at least one single leaf
      if (need53) need53[k] = (outcome(k) && sat[k] && (sel[k] & ~whole)) ? 0 : -1;
      if (fail_pos) fail_pos[k] = -1;
      if (!outcome(k)) {
        if (explicit_f(k)) {  // the op's own FailureRecord: a chain job hashes it there
          fail_pos[k] = (int32_t)fpos;
          kinds[fpos] = 2;
          m_nodes[fpos] = 0;
          m_ops[fpos] = k;
        }
      } else if (sat[k]) {
        uint32_t sm = sel[k] & ~whole;
        for (uint32_t p = 0; p < N; p++)
          if (sm >> p & 1) {
            single_pos[k * N + p] = (int32_t)spos;
            kinds[spos] = 1;
            m_nodes[spos] = p;
            m_ops[spos] = k;
            spos++;
          }
      } else {
        // failure leaf: 0x00 || 0x46 || FailureRecord (messages.cpp:260-297)
        uint8_t msg[192];
        uint32_t L = 0;
        msg[L++] = 0x00;
        msg[L++] = 0x46;
        for (int i = 0; i < 32; i++) msg[L++] = req_ids[32 * k + i];
        msg[L++] = (uint8_t)(gid_len >> 24); msg[L++] = (uint8_t)(gid_len >> 16);
        msg[L++] = (uint8_t)(gid_len >> 8);  msg[L++] = (uint8_t)gid_len;
        for (uint32_t i = 0; i < gid_len && L < 150; i++) msg[L++] = gid[i];
        for (int i = 0; i < 8; i++) msg[L++] = (uint8_t)(version >> (56 - 8 * i));
        const char reason[] = "quorum unsatisfied";
        const uint32_t rl = sizeof(reason) - 1;
        msg[L++] = 0; msg[L++] = 0; msg[L++] = 0; msg[L++] = (uint8_t)rl;
        for (uint32_t i = 0; i < rl; i++) msg[L++] = (uint8_t)reason[i];
        sha256_local(msg, L, a_leaves + 32 * fpos);
        kinds[fpos] = 2;
        m_nodes[fpos] = 0;
        m_ops[fpos] = k;
      }
    }
    __syncthreads();
    if (tid == kManThreads - 1) {
      s_carry_single += incl & 0xffff;
      s_carry_fail += incl >> 16;
    }
    __syncthreads();
  }
  if (tid == 0) {
    count[0] = nwhole + nsingle + (s_carry_fail - nsingle);
    count[1] = nsingle;
  }
}

void launch_attest_manifest(uint32_t B, uint32_t N, const uint32_t* sel,
                            const uint8_t* sat, const uint8_t* r_roots,
                            const uint8_t* req_ids, const uint8_t* gid,
                            uint32_t gid_len, uint64_t version,
                            uint8_t* a_leaves, int32_t* single_pos, int32_t* need53,
                            uint8_t* kinds, uint32_t* m_nodes, uint32_t* m_ops,
                            uint32_t* count, const uint8_t* has_outcome,
                            const uint8_t* explicit_fail, int32_t* fail_pos, cudaStream_t st) {
  if (gid_len > 100) throw InvalidArgument("group id too long for failure leaf");
  attest_manifest_kernel<<<1, kManThreads, 0, st>>>(
      B, N, sel, sat, r_roots, req_ids, gid, gid_len, version, a_leaves,
      single_pos, need53, kinds, m_nodes, m_ops, count, has_outcome, explicit_fail, fail_pos);
  CG_CHECK_LAUNCH();
}

// Requests without any provider output (misfits): outcome unsatisfied with
// an empty quorum, no label (coordinator.cpp:759-773: select_quorum only
// runs with >= N-f outputs).
__global__ void mark_missing_kernel(const uint8_t* __restrict__ miss, uint32_t B,
                                    uint32_t* sel, double* diam, uint8_t* sat, int8_t* status,
                                    int64_t* label) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= B || !miss[k]) return;
  sel[k] = 0;
  diam[k] = 0.0;
  sat[k] = 0;
  status[k] = 0;
  if (label) label[k] = -1;
}

void launch_mark_missing(const uint8_t* miss, uint32_t B, uint32_t* sel, double* diam,
                         uint8_t* sat, int8_t* status, int64_t* label, cudaStream_t st) {
  if (B == 0) return;
  mark_missing_kernel<<<(unsigned)ceil_div(B, 128), 128, 0, st>>>(miss, B, sel, diam, sat, status,
                                                                 label);
  CG_CHECK_LAUNCH();
}

// ---------------------------------------------------------- softmax/top-k
// One warp per row: peak = first max, exp(x - peak) lane-parallel, the sum
// taken sequentially by lane 0 in lane order (model.cpp:26-34 sums in index
// order), then division. Top-k over the probabilities: k largest, ties to
// the lower index (consistent with argmax/std::max_element).
constexpr int kSmWarps = 4;
constexpr int kSmMaxV = 1024;

template <typename Tin>
__global__ void __launch_bounds__(32 * kSmWarps) softmax_topk_kernel(
    const Tin* __restrict__ in, uint64_t in_ld, uint32_t rows, uint32_t v,
    int do_softmax, double* __restrict__ out, uint64_t out_ld, uint32_t k,
    uint32_t* __restrict__ topi, double* __restrict__ topv) {
  __shared__ double buf[kSmWarps][kSmMaxV];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const uint32_t row = blockIdx.x * kSmWarps + w;
  if (row >= rows) return;
  const Tin* x = in + row * in_ld;
  double* b = buf[w];
  double peak = -INFINITY;
  for (uint32_t i = lane; i < v; i += 32) {
    double t = (double)x[i];
    b[i] = t;
    peak = (peak < t) ? t : peak;
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) {
    double p2 = __shfl_xor_sync(0xffffffffu, peak, o);
    peak = (peak < p2) ? p2 : peak;
  }
  if (do_softmax) {
    for (uint32_t i = lane; i < v; i += 32) b[i] = exp(__dsub_rn(b[i], peak));
    __syncwarp();
    double sum = 0.0;
    if (lane == 0)
      for (uint32_t i = 0; i < v; i++) sum = __dadd_rn(sum, b[i]);
    sum = __shfl_sync(0xffffffffu, sum, 0);
    for (uint32_t i = lane; i < v; i += 32) b[i] = __ddiv_rn(b[i], sum);
    __syncwarp();
  }
  double* o = out + row * out_ld;
  for (uint32_t i = lane; i < v; i += 32) o[i] = b[i];
  // top-k: lane-local candidates then warp arg-reduce, k rounds
  uint32_t taken = 0;  // bit t: element lane + 32 t already chosen
  for (uint32_t r = 0; r < k; r++) {
    double bv = 0.0;
    uint32_t bi = 0xffffffffu;
    for (uint32_t t = 0; lane + 32 * t < v && t < 32; t++) {
      if (taken >> t & 1) continue;
      double y = b[lane + 32 * t];
      if (bi == 0xffffffffu || bv < y) { bv = y; bi = lane + 32 * t; }
    }
#pragma unroll
    for (int s = 16; s > 0; s >>= 1) {
      double ov = __shfl_xor_sync(0xffffffffu, bv, s);
      uint32_t oi = __shfl_xor_sync(0xffffffffu, bi, s);
      bool take = (oi != 0xffffffffu) &&
                  (bi == 0xffffffffu || bv < ov || (!(ov < bv) && oi < bi));
      if (take) { bv = ov; bi = oi; }
    }
    if (bi != 0xffffffffu && (bi & 31) == (uint32_t)lane) taken |= 1u << (bi >> 5);
    if (lane == 0) {
      topi[row * k + r] = bi;
      topv[row * k + r] = bv;
    }
  }
}

void launch_softmax_topk_f32(const float* in, uint64_t in_ld, uint32_t rows,
                             uint32_t v, int do_softmax, double* out,
                             uint64_t out_ld, uint32_t k, uint32_t* topi,
                             double* topv, cudaStream_t st) {
  if (v > kSmMaxV) throw InvalidArgument("softmax: output dim > 1024");
  softmax_topk_kernel<float><<<(unsigned)ceil_div(rows, kSmWarps), 32 * kSmWarps, 0, st>>>(
      in, in_ld, rows, v, do_softmax, out, out_ld, k, topi, topv);
  CG_CHECK_LAUNCH();
}

void launch_softmax_topk_f64(const double* in, uint64_t in_ld, uint32_t rows,
                             uint32_t v, int do_softmax, double* out,
                             uint64_t out_ld, uint32_t k, uint32_t* topi,
                             double* topv, cudaStream_t st) {
  if (v > kSmMaxV) throw InvalidArgument("softmax: output dim > 1024");
  softmax_topk_kernel<double><<<(unsigned)ceil_div(rows, kSmWarps), 32 * kSmWarps, 0, st>>>(
      in, in_ld, rows, v, do_softmax, out, out_ld, k, topi, topv);
  CG_CHECK_LAUNCH();
}

// ------------------------------------------------ LinearToyModel (fp64)
// y[row] = b[row] + sum_col W[row,col] * x[col], accumulated in column order
// without fused multiply-add (model.cpp:20-25 on x86-64 SSE2). One thread
// per (input, row); a warp covers 32 rows of one input so x is broadcast.
__global__ void __launch_bounds__(128) linear_f64_kernel(
    const double* __restrict__ W, const double* __restrict__ bias,
    const double* __restrict__ X, uint32_t B, uint32_t u, uint32_t v,
    double* __restrict__ Y) {
  uint64_t t = (uint64_t)blockIdx.x * blockDim.x + threadIdx.x;
  uint32_t rows_pad = (v + 31) / 32 * 32;
  uint32_t i = (uint32_t)(t / rows_pad), row = (uint32_t)(t % rows_pad);
  if (i >= B || row >= v) return;
  const double* w = W + (uint64_t)row * u;
  const double* x = X + (uint64_t)i * u;
  double acc = bias[row];
#pragma unroll 8
  for (uint32_t c = 0; c < u; c++) acc = __dadd_rn(acc, __dmul_rn(__ldg(w + c), __ldg(x + c)));
  Y[(uint64_t)i * v + row] = acc;
}

void launch_linear_f64(const double* W, const double* b, const double* X,
                       uint32_t B, uint32_t u, uint32_t v, double* Y,
                       cudaStream_t st) {
  uint64_t total = (uint64_t)B * ((v + 31) / 32 * 32);
  linear_f64_kernel<<<(unsigned)ceil_div(total, 128), 128, 0, st>>>(W, b, X, B, u, v, Y);
  CG_CHECK_LAUNCH();
}

}  // namespace cg
