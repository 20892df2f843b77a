// Test hooks (cg_dbg_*): run one kernel in isolation on host buffers so the
// parity tests can check it against a plain fp32 reference. Not part of the
// certified hot path; declared in include/credo_gpu.h under "test hooks".
#include <cuda_bf16.h>

#include <vector>

#include "../../include/credo_gpu.h"
#include "common.cuh"
#include "gemm_sm100.cuh"
#include "sha256.cuh"

using namespace cg;

// Cycles per SHA-256 block for one warp of 32 chains: mode 0 = unrolled
// compression only (registers), 1 = rolled compression only, 2..4 = the
// chain engine over an f64 segment with run_chain_job<mode - 2>; +8 = all
// lanes read the same stream (coalesced).
__global__ void sha_bench_kernel(int mode, uint64_t nblocks, const double* buf,
                                 uint64_t per_thread_doubles, long long* cycles,
                                 uint32_t* sink) {
  uint32_t s[8], w[16];
  sha256_iv(s);
  for (int i = 0; i < 16; i++) w[i] = threadIdx.x * 16 + i;
  const uint64_t lane_off = (mode & 8) ? 0 : threadIdx.x * per_thread_doubles;
  mode &= 7;  // +16 (host): 128 threads = one warp per SMSP
  long long t0 = clock64();
  if (mode == 0) {
    for (uint64_t b = 0; b < nblocks; b++) {
      sha256_compress<false>(s, w);
      w[0] ^= s[0];
    }
  } else if (mode == 1) {
    for (uint64_t b = 0; b < nblocks; b++) {
      sha256_compress<true>(s, w);
      w[0] ^= s[0];
    }
  } else {
    ChainJob j;
    memset(&j, 0, sizeof j);
    j.seg[0] = ChainSeg{(uint64_t)(buf + lane_off), 1, nblocks * 64, kSegF64, 0};
    j.nseg = 1;
    j.total_len = nblocks * 64 + 1;
    j.blk_begin = 1;
    j.blk_end = nblocks;
    j.state_out = (uint64_t)(sink + 128 + 8 * threadIdx.x);
    if (mode == 2) run_chain_job<0>(j, 0);
    else if (mode == 3) run_chain_job<1>(j, 0);
    else run_chain_job<2>(j, 0);
    s[0] = (uint32_t)j.blk_end;
  }
  long long t1 = clock64();
  if (threadIdx.x == 0) *cycles = t1 - t0;
  uint32_t acc = 0;
  for (int i = 0; i < 8; i++) acc ^= s[i];
  sink[threadIdx.x] = acc;
}

extern "C" int cg_dbg_sha_bench(cg_ctx* ctx, int mode, uint64_t nblocks,
                                double* cycles_per_block) {
  try {
    cudaStream_t st = (cudaStream_t)cg_ctx_stream(ctx);
    double* buf = nullptr;
    long long* cyc = nullptr;
    uint32_t* sink = nullptr;
    uint64_t per = nblocks * 8 + 16;
    CG_CUDA(cudaMalloc(&buf, 128 * per * 8));
    CG_CUDA(cudaMemset(buf, 1, 128 * per * 8));
    CG_CUDA(cudaMalloc(&cyc, 8));
    CG_CUDA(cudaMalloc(&sink, 4 * (128 + 8 * 128)));
    sha_bench_kernel<<<1, (mode & 16) ? 128 : 32, 0, st>>>(mode & 15, nblocks, buf, per, cyc, sink);
    CG_CHECK_LAUNCH();
    long long c = 0;
    CG_CUDA(cudaMemcpyAsync(&c, cyc, 8, cudaMemcpyDeviceToHost, st));
    CG_CUDA(cudaStreamSynchronize(st));
    *cycles_per_block = (double)c / (double)nblocks;
    cudaFree(buf);
    cudaFree(cyc);
    cudaFree(sink);
    return CG_OK;
  } catch (const std::exception&) {
    return CG_ECUDA;
  }
}

// Timing + CTA-0 event trace of one halo-mode 3x3 conv (B images of H x H,
// C -> N channels) over a padded grid of device-resident operands.
extern "C" int cg_dbg_halo_trace2(cg_ctx* ctx, int B, int H, int C, int N, int BN, int pair,
                                  long long* trace_host, double* us);
extern "C" int cg_dbg_halo_trace(cg_ctx* ctx, int B, int H, int C, int N, int BN,
                                 long long* trace_host, double* us) {
  return cg_dbg_halo_trace2(ctx, B, H, C, N, BN, 0, trace_host, us);
}
extern "C" int cg_dbg_halo_trace2(cg_ctx* ctx, int B, int H, int C, int N, int BN, int pair,
                                  long long* trace_host, double* us) {
  try {
    cudaStream_t st = (cudaStream_t)cg_ctx_stream(ctx);
    const int Hp = H + 1, rows = B * Hp * Hp;  // shared-border grid pitch
    void *dA, *dB, *dbias, *dout;
    long long* dtr;
    CG_CUDA(cudaMalloc(&dA, (size_t)rows * C * 2));
    CG_CUDA(cudaMalloc(&dB, (size_t)N * 9 * C * 2));
    CG_CUDA(cudaMalloc(&dbias, (size_t)N * 4));
    CG_CUDA(cudaMalloc(&dout, (size_t)B * H * H * N * 2));
    CG_CUDA(cudaMalloc(&dtr, 16 * 64 * 8));
    CG_CUDA(cudaMemset(dA, 0x11, (size_t)rows * C * 2));
    CG_CUDA(cudaMemset(dB, 0x11, (size_t)N * 9 * C * 2));
    CG_CUDA(cudaMemset(dbias, 0, (size_t)N * 4));
    CG_CUDA(cudaMemset(dtr, 0, 16 * 64 * 8));
    Operand oa, ob;
    make_operand(oa, dA, rows, C, 128 + 2 * (Hp + 1));
    make_operand(ob, dB, N, 9 * C, pair ? BN / 2 : BN);
    ConvGemmArgs a{};
    a.pair = pair;
    a.M = rows;
    a.N = N;
    a.Kc = C;
    a.ntaps = 9;
    for (int dr = 0; dr < 3; dr++)
      for (int ds = 0; ds < 3; ds++) a.tap_off[dr * 3 + ds] = (dr - 1) * Hp + (ds - 1);
    a.bias = (const float*)dbias;
    a.out = dout;
    a.ld_out = N;
    a.relu = 1;
    a.row_mode = kRowPadToCompact;
    a.H = H;
    a.W = H;
    a.rows_out = B * H * H;
    a.halo_lo = Hp + 1;
    launch_conv_gemm(oa, ob, a, BN, st);  // warm
    cudaEvent_t e0, e1;
    CG_CUDA(cudaEventCreate(&e0));
    CG_CUDA(cudaEventCreate(&e1));
    CG_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < 5; i++) launch_conv_gemm(oa, ob, a, BN, st);
    CG_CUDA(cudaEventRecord(e1, st));
    a.trace = dtr;
    launch_conv_gemm(oa, ob, a, BN, st);
    CG_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    CG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *us = 1000.0 * ms / 5;
    CG_CUDA(cudaMemcpy(trace_host, dtr, 16 * 64 * 8, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dbias);
    cudaFree(dout);
    cudaFree(dtr);
    return CG_OK;
  } catch (const std::exception&) {
    return CG_ECUDA;
  }
}

// Timing + CTA-0 event trace of one 1x1 conv GEMM shape on device-resident
// random operands (no host copies in the timed launch).
extern "C" int cg_dbg_gemm_trace_mode(cg_ctx* ctx, int M, int N, int K, int BN, int residual,
                                      int row_mode, int H, long long* trace_host, double* us);

extern "C" int cg_dbg_gemm_trace(cg_ctx* ctx, int M, int N, int K, int BN, int residual,
                                 long long* trace_host, double* us) {
  return cg_dbg_gemm_trace_mode(ctx, M, N, K, BN, residual, 0, 0, trace_host, us);
}

// The same with a row remap (row_mode, H = W): M compact rows in, the output
// sized for the mode (e.g. CompactToPad writes the padded grid interior).
extern "C" int cg_dbg_gemm_trace_mode(cg_ctx* ctx, int M, int N, int K, int BN, int residual,
                                      int row_mode, int H, long long* trace_host, double* us) {
  try {
    cudaStream_t st = (cudaStream_t)cg_ctx_stream(ctx);
    void *dA, *dB, *dbias, *dres = nullptr, *dout;
    long long* dtr;
    CG_CUDA(cudaMalloc(&dA, (size_t)M * K * 2));
    CG_CUDA(cudaMalloc(&dB, (size_t)N * K * 2));
    CG_CUDA(cudaMalloc(&dbias, (size_t)N * 4));
    const size_t out_rows = row_mode == kRowCompactToPad
                                ? (size_t)(M / (H * H)) * (H + 1) * (H + 1) + H + 2
                                : (size_t)M;
    CG_CUDA(cudaMalloc(&dout, out_rows * N * 2));
    CG_CUDA(cudaMalloc(&dtr, 16 * 64 * 8));
    CG_CUDA(cudaMemset(dA, 0x11, (size_t)M * K * 2));
    CG_CUDA(cudaMemset(dB, 0x11, (size_t)N * K * 2));
    CG_CUDA(cudaMemset(dbias, 0, (size_t)N * 4));
    CG_CUDA(cudaMemset(dtr, 0, 16 * 64 * 8));
    if (residual) {
      CG_CUDA(cudaMalloc(&dres, (size_t)M * N * 2));
      CG_CUDA(cudaMemset(dres, 0x11, (size_t)M * N * 2));
    }
    Operand oa, ob;
    const int pair = (residual >> 1) & 1;
    residual &= 1;
    make_operand(oa, dA, M, K, 128);
    make_operand(ob, dB, N, K, pair ? BN / 2 : BN);
    ConvGemmArgs a{};
    a.pair = pair;
    a.M = M;
    a.N = N;
    a.Kc = K;
    a.ntaps = 1;
    a.bias = (const float*)dbias;
    a.residual = (const __nv_bfloat16*)dres;
    a.ld_res = N;
    a.out = dout;
    a.ld_out = N;
    a.relu = 1;
    a.rows_out = (int)out_rows;
    a.row_mode = row_mode;
    a.H = H;
    a.W = H;
    launch_conv_gemm(oa, ob, a, BN, st);  // warm
    cudaEvent_t e0, e1;
    CG_CUDA(cudaEventCreate(&e0));
    CG_CUDA(cudaEventCreate(&e1));
    CG_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < 5; i++) launch_conv_gemm(oa, ob, a, BN, st);
    CG_CUDA(cudaEventRecord(e1, st));
    a.trace = dtr;
    launch_conv_gemm(oa, ob, a, BN, st);
    CG_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    CG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *us = 1000.0 * ms / 5;
    CG_CUDA(cudaMemcpy(trace_host, dtr, 16 * 64 * 8, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dbias);
    cudaFree(dout);
    cudaFree(dtr);
    if (dres) cudaFree(dres);
    return CG_OK;
  } catch (const std::exception&) {
    return CG_ECUDA;
  }
}

static int dbg_conv_gemm(cg_ctx* ctx, const uint16_t* A, int rowsA, const uint16_t* B, int N,
                         int Kc, int ntaps, const int* tap_off, const float* bias,
                         const uint16_t* residual, int relu, int row_mode, int H, int W, int M,
                         int rows_out, int out_f32, int BN, void* out, int max_ctas, int halo_lo,
                         int pair = 0);

extern "C" int cg_dbg_conv_gemm(cg_ctx* ctx, const uint16_t* A, int rowsA,
                                const uint16_t* B, int N, int Kc, int ntaps,
                                const int* tap_off, const float* bias,
                                const uint16_t* residual, int relu, int row_mode,
                                int H, int W, int M, int rows_out, int out_f32,
                                int BN, void* out, int max_ctas) {
  return dbg_conv_gemm(ctx, A, rowsA, B, N, Kc, ntaps, tap_off, bias, residual, relu, row_mode,
                       H, W, M, rows_out, out_f32, BN, out, max_ctas, 0);
}

extern "C" int cg_dbg_conv_gemm_halo(cg_ctx* ctx, const uint16_t* A, int rowsA,
                                     const uint16_t* B, int N, int Kc, int ntaps,
                                     const int* tap_off, const float* bias, int relu,
                                     int row_mode, int H, int W, int M, int rows_out, int BN,
                                     void* out, int halo_lo) {
  return dbg_conv_gemm(ctx, A, rowsA, B, N, Kc, ntaps, tap_off, bias, nullptr, relu, row_mode, H,
                       W, M, rows_out, 0, BN, out, 0, halo_lo);
}

extern "C" int cg_dbg_conv_gemm_pair(cg_ctx* ctx, const uint16_t* A, int rowsA,
                                     const uint16_t* B, int N, int Kc, int ntaps,
                                     const int* tap_off, const float* bias,
                                     const uint16_t* residual, int relu, int row_mode, int H,
                                     int W, int M, int rows_out, int out_f32, int BN, void* out,
                                     int max_ctas) {
  return dbg_conv_gemm(ctx, A, rowsA, B, N, Kc, ntaps, tap_off, bias, residual, relu, row_mode,
                       H, W, M, rows_out, out_f32, BN, out, max_ctas, 0, 1);
}

extern "C" int cg_dbg_conv_gemm_halo_pair(cg_ctx* ctx, const uint16_t* A, int rowsA,
                                          const uint16_t* B, int N, int Kc, int ntaps,
                                          const int* tap_off, const float* bias, int relu,
                                          int row_mode, int H, int W, int M, int rows_out,
                                          int BN, void* out, int halo_lo) {
  return dbg_conv_gemm(ctx, A, rowsA, B, N, Kc, ntaps, tap_off, bias, nullptr, relu, row_mode, H,
                       W, M, rows_out, 0, BN, out, 0, halo_lo, 1);
}

static int dbg_conv_gemm(cg_ctx* ctx, const uint16_t* A, int rowsA, const uint16_t* B, int N,
                         int Kc, int ntaps, const int* tap_off, const float* bias,
                         const uint16_t* residual, int relu, int row_mode, int H, int W, int M,
                         int rows_out, int out_f32, int BN, void* out, int max_ctas, int halo_lo,
                         int pair) {
  try {
    cudaStream_t st = (cudaStream_t)cg_ctx_stream(ctx);
    void *dA, *dB, *dbias, *dres = nullptr, *dout;
    size_t outsz = (size_t)rows_out * N * (out_f32 ? 4 : 2);
    CG_CUDA(cudaMalloc(&dA, (size_t)rowsA * Kc * 2));
    CG_CUDA(cudaMalloc(&dB, (size_t)N * ntaps * Kc * 2));
    CG_CUDA(cudaMalloc(&dbias, (size_t)N * 4));
    CG_CUDA(cudaMalloc(&dout, outsz));
    CG_CUDA(cudaMemset(dout, 0, outsz));
    CG_CUDA(cudaMemcpy(dA, A, (size_t)rowsA * Kc * 2, cudaMemcpyHostToDevice));
    CG_CUDA(cudaMemcpy(dB, B, (size_t)N * ntaps * Kc * 2, cudaMemcpyHostToDevice));
    CG_CUDA(cudaMemcpy(dbias, bias, (size_t)N * 4, cudaMemcpyHostToDevice));
    if (residual) {
      CG_CUDA(cudaMalloc(&dres, (size_t)rows_out * N * 2));
      CG_CUDA(cudaMemcpy(dres, residual, (size_t)rows_out * N * 2, cudaMemcpyHostToDevice));
    }
    Operand oa, ob;
    // halos wider than one 256-row box: stacked boxes (ConvGemmArgs::halo_sub)
    int hsub = 1, hbox = 128 + 2 * halo_lo;
    if (halo_lo > 0 && hbox > 256) halo_boxes(halo_lo, hsub, hbox);
    make_operand(oa, dA, rowsA, Kc, hbox);
    make_operand(ob, dB, N, ntaps * Kc, pair ? BN / 2 : BN);
    ConvGemmArgs a{};
    a.M = M;
    a.N = N;
    a.Kc = Kc;
    a.ntaps = ntaps;
    a.pair = pair;
    for (int t = 0; t < ntaps; t++) a.tap_off[t] = tap_off[t];
    a.bias = (const float*)dbias;
    a.residual = (const __nv_bfloat16*)dres;
    a.ld_res = N;
    a.out = dout;
    a.ld_out = N;
    a.out_f32 = out_f32;
    a.relu = relu;
    a.row_mode = row_mode;
    a.H = H;
    a.W = W;
    a.rows_out = rows_out;
    a.halo_lo = halo_lo;
    a.halo_sub = hsub;
    a.halo_box = hbox;
    launch_conv_gemm(oa, ob, a, BN, st, max_ctas);
    CG_CUDA(cudaStreamSynchronize(st));
    CG_CUDA(cudaMemcpy(out, dout, outsz, cudaMemcpyDeviceToHost));
    cudaFree(dA);
    cudaFree(dB);
    cudaFree(dbias);
    cudaFree(dout);
    if (dres) cudaFree(dres);
    return CG_OK;
  } catch (const std::exception& e) {
    return CG_ECUDA;
  }
}

// ------------------------------------------------- C5 synthetic generator
namespace {
__device__ __forceinline__ uint64_t mix64(uint64_t z) {  // splitmix64 finaliser
  z += 0x9e3779b97f4a7c15ull;
  z = (z ^ (z >> 30)) * 0xbf58476d1ce4e5b9ull;
  z = (z ^ (z >> 27)) * 0x94d049bb133111ebull;
  return z ^ (z >> 31);
}
__device__ __forceinline__ double unit(uint64_t h) {  // [0, 1)
  return (double)(h >> 11) * (1.0 / 9007199254740992.0);
}
__global__ void synth_outputs_kernel(uint64_t seed, uint32_t R, uint32_t n, uint32_t v,
                                     double eps, double shift_frac, double* outs) {
  const uint64_t total = (uint64_t)R * v;
  const double jit = eps / (8.0 * sqrt((double)v));  // honest euclidean spread ~ eps/10
  for (uint64_t e = blockIdx.x * (uint64_t)blockDim.x + threadIdx.x; e < total;
       e += (uint64_t)gridDim.x * blockDim.x) {
    const uint64_t k = e / v, t = e % v;
    const double c = unit(mix64(seed ^ mix64(k * 0x100000001b3ull + t)));
    for (uint32_t p = 0; p < n; p++) {
      const uint64_t hk = mix64(seed + 0x51ull + mix64(k * 64 + p));
      const double shift = unit(hk) < shift_frac ? 3.0 * eps / sqrt((double)v) : 0.0;
      const double j = (unit(mix64(hk ^ (t * 0x9e3779b97f4a7c15ull))) * 2.0 - 1.0) * jit;
      outs[(uint64_t)p * total + e] = c + j + shift;
    }
  }
}
__global__ void synth_ids_kernel(uint64_t seed, uint32_t R, uint8_t* ids) {
  const uint32_t k = blockIdx.x * blockDim.x + threadIdx.x;
  if (k >= R) return;
  uint64_t* o = reinterpret_cast<uint64_t*>(ids + 32ull * k);
  for (int i = 0; i < 4; i++) o[i] = mix64(seed * 31 + k * 4ull + i);
}
}  // namespace

extern "C" int cg_synth_outputs(cg_ctx* ctx, uint64_t seed, uint32_t R, uint32_t n, uint32_t v,
                                double eps, double shift_frac, double* outs, uint8_t* req_ids) {
  try {
    cudaStream_t st = (cudaStream_t)cg_ctx_stream(ctx);
    if (R == 0) return CG_OK;
    synth_outputs_kernel<<<148 * 8, 256, 0, st>>>(seed, R, n, v, eps, shift_frac, outs);
    CG_CHECK_LAUNCH();
    if (req_ids) {
      synth_ids_kernel<<<(unsigned)ceil_div(R, 128), 128, 0, st>>>(seed, R, req_ids);
      CG_CHECK_LAUNCH();
    }
    return CG_OK;
  } catch (const std::exception&) {
    return CG_ECUDA;
  }
}

extern "C" int cg_dbg_mma_rate(cg_ctx* ctx, int N, int iters, int ctas, int two_acc,
                               double* cycles_per_mma) {
  try {
    *cycles_per_mma = mma_rate_bench(N, iters, ctas, two_acc, (cudaStream_t)cg_ctx_stream(ctx));
    return CG_OK;
  } catch (const std::exception&) {
    return CG_ECUDA;
  }
}

// Timing + CTA-0 event trace of the s2d stem GEMM (conv1 of a ResNet at
// S x S input: 16 taps of K = 16 over the Gs x Gs space-to-depth grid, 64
// outputs on the same grid) for `reps` grouped replicas of B images.
extern "C" int cg_dbg_s2d_trace(cg_ctx* ctx, int B, int S, int reps, long long* trace_host,
                                double* us) {
  try {
    cudaStream_t st = (cudaStream_t)cg_ctx_stream(ctx);
    const int Gs = (S + 6) / 2, rows = B * Gs * Gs;
    if (reps < 1 || reps > kMaxGroup) return CG_EINVAL;
    void *dA[kMaxGroup], *dB, *dbias, *dout[kMaxGroup];
    long long* dtr;
    CG_CUDA(cudaMalloc(&dB, (size_t)16 * 64 * 16 * 2));
    CG_CUDA(cudaMalloc(&dbias, 64 * 4));
    CG_CUDA(cudaMalloc(&dtr, 16 * 64 * 8));
    CG_CUDA(cudaMemset(dB, 0x11, (size_t)16 * 64 * 16 * 2));
    CG_CUDA(cudaMemset(dbias, 0, 64 * 4));
    CG_CUDA(cudaMemset(dtr, 0, 16 * 64 * 8));
    Operand oa[kMaxGroup], ob;
    make_operand_s2d_b(ob, dB, 16 * 64);
    ConvGemmGroup g;
    g.n = reps;
    for (int r = 0; r < reps; r++) {
      CG_CUDA(cudaMalloc(&dA[r], (size_t)rows * 32));
      CG_CUDA(cudaMalloc(&dout[r], (size_t)rows * 64 * 2));
      CG_CUDA(cudaMemset(dA[r], 0x11, (size_t)rows * 32));
      make_operand_s2d_a(oa[r], dA[r], rows, 128 + Gs + 3);
      g.A[r] = &oa[r];
      g.B[r] = &ob;
      g.bias[r] = (const float*)dbias;
      g.residual[r] = nullptr;
      g.out[r] = dout[r];
    }
    ConvGemmArgs a{};
    a.M = rows;
    a.N = 64;
    a.Kc = 16;
    a.ntaps = 16;
    a.ld_out = 64;
    a.relu = 1;
    a.row_mode = kRowIdentity;
    a.H = a.W = S / 2;
    a.rows_out = rows;
    a.s2d = 1;
    a.gh = a.gw = Gs;
    PreparedGemm p;
    prepare_conv_gemm(p, g, a, 64);
    launch_prepared(p, st);  // warm
    cudaEvent_t e0, e1;
    CG_CUDA(cudaEventCreate(&e0));
    CG_CUDA(cudaEventCreate(&e1));
    CG_CUDA(cudaEventRecord(e0, st));
    for (int i = 0; i < 5; i++) launch_prepared(p, st);
    CG_CUDA(cudaEventRecord(e1, st));
    PreparedGemm pt = p;
    pt.args.trace = dtr;
    launch_prepared(pt, st);
    CG_CUDA(cudaStreamSynchronize(st));
    float ms = 0;
    CG_CUDA(cudaEventElapsedTime(&ms, e0, e1));
    *us = 1000.0 * ms / 5;
    CG_CUDA(cudaMemcpy(trace_host, dtr, 16 * 64 * 8, cudaMemcpyDeviceToHost));
    for (int r = 0; r < reps; r++) {
      cudaFree(dA[r]);
      cudaFree(dout[r]);
    }
    cudaFree(dB);
    cudaFree(dbias);
    cudaFree(dtr);
    return CG_OK;
  } catch (const std::exception&) {
    return CG_ECUDA;
  }
}
