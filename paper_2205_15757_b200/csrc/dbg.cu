// Test hooks (cg_dbg_*): run one kernel in isolation on host buffers so the
// parity tests can check it against a plain fp32 reference. Not part of the
// certified hot path; declared in include/credo_gpu.h under "test hooks".
#include <cuda_bf16.h>

#include <vector>

#include "../../include/credo_gpu.h"
#include "common.cuh"
#include "gemm_sm100.cuh"

using namespace cg;

extern "C" int cg_dbg_conv_gemm(cg_ctx* ctx, const uint16_t* A, int rowsA,
                                const uint16_t* B, int N, int Kc, int ntaps,
                                const int* tap_off, const float* bias,
                                const uint16_t* residual, int relu, int row_mode,
                                int H, int W, int M, int rows_out, int out_f32,
                                int BN, void* out, int max_ctas) {
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
    make_operand(oa, dA, rowsA, Kc, 128);
    make_operand(ob, dB, N, ntaps * Kc, BN);
    ConvGemmArgs a{};
    a.M = M;
    a.N = N;
    a.Kc = Kc;
    a.ntaps = ntaps;
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
