// Persistent, warp-specialised tcgen05 implicit-GEMM convolution (sm_100a).
//
// CTA = 6 warps: w0 TMA producer (one lane), w1 TMEM owner + MMA issuer (one
// lane), w2-w5 epilogue (TMEM lane quarters). Operands stream through a
// STAGES-deep smem ring (128B-swizzled TMA boxes, mbarrier full/empty);
// accumulators are double-buffered in TMEM (2 x BN fp32 columns) so the
// epilogue of tile i overlaps the MMAs of tile i+1.
#include <cuda.h>

#include "common.cuh"
#include "gemm_sm100.cuh"

namespace cg {
namespace {

constexpr int BM = 128, BK = 64, kThreads = 192;
constexpr int A_BYTES = BM * BK * 2;

__device__ __forceinline__ uint32_t su32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* b, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(su32(b)), "r"(count));
}
__device__ __forceinline__ void mbar_expect_tx(uint64_t* b, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su32(b)),
               "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_arrive(uint64_t* b) {
  asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(su32(b)) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* tm, uint64_t* bar,
                                            void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(tm), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tc_fence_before() {
  asm volatile("tcgen05.fence::before_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void tc_fence_after() {
  asm volatile("tcgen05.fence::after_thread_sync;" ::: "memory");
}
__device__ __forceinline__ void umma_commit(uint64_t* b) {
  asm volatile(
      "tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];" ::"r"(
          su32(b))
      : "memory");
}
__device__ __forceinline__ void umma_bf16(uint32_t d, uint64_t a, uint64_t b,
                                          uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
// K-major, 128B-swizzled operand tile: 8-row atoms of 1024 B (SBO), version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  uint64_t addr = su32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}
__device__ __forceinline__ void tmem_ld32(uint32_t taddr, uint32_t (&v)[32]) {
  asm volatile(
      "tcgen05.ld.sync.aligned.32x32b.x32.b32 "
      "{%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15,"
      "%16,%17,%18,%19,%20,%21,%22,%23,%24,%25,%26,%27,%28,%29,%30,%31}, [%32];"
      : "=r"(v[0]), "=r"(v[1]), "=r"(v[2]), "=r"(v[3]), "=r"(v[4]), "=r"(v[5]),
        "=r"(v[6]), "=r"(v[7]), "=r"(v[8]), "=r"(v[9]), "=r"(v[10]), "=r"(v[11]),
        "=r"(v[12]), "=r"(v[13]), "=r"(v[14]), "=r"(v[15]), "=r"(v[16]),
        "=r"(v[17]), "=r"(v[18]), "=r"(v[19]), "=r"(v[20]), "=r"(v[21]),
        "=r"(v[22]), "=r"(v[23]), "=r"(v[24]), "=r"(v[25]), "=r"(v[26]),
        "=r"(v[27]), "=r"(v[28]), "=r"(v[29]), "=r"(v[30]), "=r"(v[31])
      : "r"(taddr));
  asm volatile("tcgen05.wait::ld.sync.aligned;" ::: "memory");
}

__device__ __forceinline__ int remap_row(int M, int rows_out, int mode, int H,
                                         int W, int m) {
  if (m >= M) return -1;
  if (mode == kRowIdentity) return m < rows_out ? m : -1;
  const int Wp = W + 2, HpWp = (H + 2) * Wp;
  if (mode == kRowPadToCompact) {
    int img = m / HpWp, rem = m - img * HpWp;
    int hp = rem / Wp, wp = rem - hp * Wp;
    if (hp < 1 || hp > H || wp < 1 || wp > W) return -1;
    return (img * H + hp - 1) * W + wp - 1;
  }
  const int HW = H * W;
  int img = m / HW, rem = m - img * HW;
  int h = rem / W, w = rem - h * W;
  return img * HpWp + (h + 1) * Wp + w + 1;
}

template <int BN, int STAGES>
__global__ void __launch_bounds__(kThreads, 1)
    conv_gemm_kernel(const __grid_constant__ CUtensorMap tmA,
                     const __grid_constant__ CUtensorMap tmB,
                     const ConvGemmArgs a) {
  constexpr int B_BYTES = BN * BK * 2;
  constexpr uint32_t TMEM_COLS = 2 * BN;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(smem_raw) + 1023) & ~uintptr_t(1023));
  uint8_t* sA = smem;
  uint8_t* sB = smem + STAGES * A_BYTES;
  uint64_t* full = reinterpret_cast<uint64_t*>(sB + STAGES * B_BYTES);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(tempty + 2);
  int* s_tap = reinterpret_cast<int*>(tmem_slot + 4);

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_n = (a.N + BN - 1) / BN, num_m = (a.M + BM - 1) / BM;
  const int tiles = num_m * num_n;
  const int kpt = a.Kc / BK, num_k = a.ntaps * kpt;

  if (warp == 0 && lane == 0) {
#pragma unroll
    for (int i = 0; i < 9; i++) s_tap[i] = a.tap_off[i];
  }
  if (warp == 0 && lane == 0) {
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmA) : "memory");
    asm volatile("prefetch.tensormap [%0];" ::"l"(&tmB) : "memory");
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; s++) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], 4);
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tmem_slot)),
                 "r"(TMEM_COLS)
                 : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        const int m0 = (t / num_n) * BM, n0 = (t % num_n) * BN;
        for (int kb = 0; kb < num_k; kb++) {
          const int tap = kb / kpt, cb = kb - tap * kpt;
          mbar_wait(&empty[stage], phase ^ 1);
          mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
          tma_load_2d(&tmA, &full[stage], sA + stage * A_BYTES, cb * BK,
                      m0 + s_tap[tap]);
          tma_load_2d(&tmB, &full[stage], sB + stage * B_BYTES, kb * BK, n0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    if (lane == 0) {  // ---------------- MMA issuer
      // kind::f16 instruction descriptor: D f32, A/B bf16, K-major, M=128, N=BN
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0, acc = 0;
      uint32_t phase = 0, acc_phase = 0;
      for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN;
        for (int kb = 0; kb < num_k; kb++) {
          mbar_wait(&full[stage], phase);
          tc_fence_after();
          const uint64_t ad = smem_desc_sw128(sA + stage * A_BYTES);
          const uint64_t bd = smem_desc_sw128(sB + stage * B_BYTES);
#pragma unroll
          for (int k = 0; k < BK / 16; k++)  // UMMA_K = 16 (32 bytes)
            umma_bf16(d, ad + 2 * k, bd + 2 * k, idesc, (kb | k) != 0);
          umma_commit(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit(&tfull[acc]);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else {  // ------------------------------ epilogue (warps 2..5)
    const int q = warp & 3;  // TMEM lane quarter this warp may access
    int acc = 0;
    uint32_t acc_phase = 0;
    for (int t = blockIdx.x; t < tiles; t += gridDim.x) {
      const int m0 = (t / num_n) * BM, n0 = (t % num_n) * BN;
      mbar_wait(&tfull[acc], acc_phase);
      tc_fence_after();
      const int m = m0 + q * 32 + lane;
      const int orow = remap_row(a.M, a.rows_out, a.row_mode, a.H, a.W, m);
#pragma unroll 1
      for (int c = 0; c < BN / 32; c++) {
        uint32_t v[32];
        tmem_ld32(tmem + ((uint32_t)(q * 32) << 16) + acc * BN + c * 32, v);
        const int n = n0 + c * 32;
        if (orow < 0 || n >= a.N) continue;
        float x[32];
        const float* bp = a.bias + n;
#pragma unroll
        for (int j = 0; j < 32; j++)
          x[j] = __uint_as_float(v[j]) + ((n + j < a.N) ? __ldg(bp + j) : 0.f);
        if (a.residual) {
          const uint4* rp = reinterpret_cast<const uint4*>(
              a.residual + (size_t)orow * a.ld_res + n);
#pragma unroll
          for (int j = 0; j < 4; j++) {
            uint4 r4 = __ldg(rp + j);
            const __nv_bfloat162* r2 = reinterpret_cast<const __nv_bfloat162*>(&r4);
#pragma unroll
            for (int e = 0; e < 4; e++) {
              float2 f = __bfloat1622float2(r2[e]);
              x[8 * j + 2 * e] += f.x;
              x[8 * j + 2 * e + 1] += f.y;
            }
          }
        }
        if (a.relu) {
#pragma unroll
          for (int j = 0; j < 32; j++) x[j] = fmaxf(x[j], 0.f);
        }
        if (a.out_f32) {
          float* op = reinterpret_cast<float*>(a.out) + (size_t)orow * a.ld_out + n;
          if (n + 32 <= a.N) {
#pragma unroll
            for (int j = 0; j < 8; j++)
              reinterpret_cast<float4*>(op)[j] =
                  make_float4(x[4 * j], x[4 * j + 1], x[4 * j + 2], x[4 * j + 3]);
          } else {
#pragma unroll
            for (int j = 0; j < 32; j++)
              if (n + j < a.N) op[j] = x[j];
          }
        } else {
          __nv_bfloat16* op =
              reinterpret_cast<__nv_bfloat16*>(a.out) + (size_t)orow * a.ld_out + n;
          uint4 o4[4];
          __nv_bfloat162* o2 = reinterpret_cast<__nv_bfloat162*>(o4);
#pragma unroll
          for (int j = 0; j < 16; j++) o2[j] = __floats2bfloat162_rn(x[2 * j], x[2 * j + 1]);
#pragma unroll
          for (int j = 0; j < 4; j++) reinterpret_cast<uint4*>(op)[j] = o4[j];
        }
      }
      tc_fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&tempty[acc]);
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
  }
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                 "r"(TMEM_COLS)
                 : "memory");
  }
}

using EncodeFn = CUresult (*)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*,
                              const cuuint64_t*, const cuuint64_t*, const cuuint32_t*,
                              const cuuint32_t*, CUtensorMapInterleave,
                              CUtensorMapSwizzle, CUtensorMapL2promotion,
                              CUtensorMapFloatOOBfill);

EncodeFn get_encode() {
  static EncodeFn fn = nullptr;
  if (!fn) {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    CG_CUDA(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q));
    if (!p || q != cudaDriverEntryPointSuccess)
      throw CudaError("cuTensorMapEncodeTiled unavailable");
    fn = reinterpret_cast<EncodeFn>(p);
  }
  return fn;
}

template <int BN, int STAGES>
constexpr int smem_bytes() {
  return STAGES * (A_BYTES + BN * BK * 2) + 2 * STAGES * 8 + 4 * 8 + 16 + 64 + 1024;
}

template <int BN, int STAGES>
void launch_t(const Operand& A, const Operand& B, const ConvGemmArgs& a,
              cudaStream_t st, int max_ctas) {
  static bool attr = false;
  constexpr int smem = smem_bytes<BN, STAGES>();
  if (!attr) {
    CG_CUDA(cudaFuncSetAttribute(conv_gemm_kernel<BN, STAGES>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    attr = true;
  }
  int tiles = ((a.M + BM - 1) / BM) * ((a.N + BN - 1) / BN);
  int grid = tiles < kNumSMs ? tiles : kNumSMs;
  if (max_ctas > 0 && grid > max_ctas) grid = max_ctas;
  timer_begin(st, kTimeGemm);
  conv_gemm_kernel<BN, STAGES><<<grid, kThreads, smem, st>>>(A.map, B.map, a);
  CG_CHECK_LAUNCH();
  timer_end(st, kTimeGemm);
}

}  // namespace

void make_operand(Operand& op, const void* ptr, int rows, int cols, int box_rows) {
  if (cols % 64 != 0) throw InvalidArgument("operand K must be a multiple of 64");
  if (reinterpret_cast<uintptr_t>(ptr) % 16) throw InvalidArgument("operand misaligned");
  cuuint64_t dims[2] = {(cuuint64_t)cols, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)cols * 2};
  cuuint32_t box[2] = {64, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&op.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                            const_cast<void*>(ptr), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_128B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("cuTensorMapEncodeTiled failed: " + std::to_string((int)r));
  op.ptr = ptr;
  op.rows = rows;
  op.cols = cols;
  op.box_rows = box_rows;
}

void launch_conv_gemm(const Operand& A, const Operand& B, const ConvGemmArgs& a,
                      int BN, cudaStream_t st, int max_ctas) {
  if (a.Kc % 64 || a.ntaps < 1 || a.ntaps > 9) throw InvalidArgument("conv_gemm: bad K");
  if (A.box_rows != BM || B.box_rows != BN) throw InvalidArgument("conv_gemm: box mismatch");
  if (!a.out_f32 && (a.N % 32)) throw InvalidArgument("conv_gemm: bf16 out needs N%32==0");
  switch (BN) {
    case 64: launch_t<64, 8>(A, B, a, st, max_ctas); break;
    case 128: launch_t<128, 6>(A, B, a, st, max_ctas); break;
    case 256: launch_t<256, 4>(A, B, a, st, max_ctas); break;
    default: throw InvalidArgument("conv_gemm: BN must be 64, 128 or 256");
  }
}

}  // namespace cg
