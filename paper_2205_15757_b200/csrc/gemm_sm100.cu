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

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

namespace cg {
namespace {

// warps: 0 TMA producer, 1 MMA issuer, 2-9 epilogue, 10 residual loader
constexpr int BM = 128, BK = 64, kThreads = 352;
constexpr int kEpiWarps = 8, kStgLd = 36;        // staging row stride (floats)
constexpr int A_BYTES = BM * BK * 2;
constexpr int kHaloBytes = 256 * BK * 2;  // largest halo box (BM + 2*halo_lo <= 256 rows)
// wide-halo slot rows (stacked boxes): 3x3 convs up to 224 pixels wide
// (BM + 2 * (W + 2) = 580 at W = 224 on the shared-border grid: 3 boxes of
// 200 rows)
constexpr int kWideHaloRows = 600;
constexpr int kWideHaloRows128 = 368;  // 128-wide tiles (streamed weights): up to 112 pixels
// s2d stem: one box per dy pair, BM + gw + 3 <= 256 rows of 32 bytes (16 channels)
constexpr int kS2DSlot = 256 * 32;
#ifndef CG_RES_COLS
#define CG_RES_COLS 64
#endif
#ifndef CG_DIRECT_REMAP
#define CG_DIRECT_REMAP 1
#endif
constexpr bool kDirectRemap = CG_DIRECT_REMAP != 0;  // thread-per-row remapped epilogue

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
#ifndef CG_MBAR_SUSPEND_NS
#define CG_MBAR_SUSPEND_NS 0  // 0: hardware default try_wait window (no hint)
#endif
__device__ __forceinline__ void mbar_wait(uint64_t* b, uint32_t parity) {
#if CG_MBAR_SUSPEND_NS > 0
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity), "r"(CG_MBAR_SUSPEND_NS)
      : "memory");
#else
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity)
      : "memory");
#endif
}
// The same wait with a suspend-time hint: the warp sleeps in the barrier
// until the phase completes (or the hint elapses) instead of re-polling, so
// an epilogue warp waiting for its next accumulator takes no issue slots
// from the warps of its SM sub-partition that are still draining theirs.
__device__ __forceinline__ void mbar_wait_sleep(uint64_t* b, uint32_t parity) {
  asm volatile(
      "{\n\t.reg .pred p;\n"
      "WAIT_%=:\n\t"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n\t"
      "@!p bra WAIT_%=;\n}" ::"r"(su32(b)),
      "r"(parity), "r"(100000)
      : "memory");
}
// n / d for a kernel-uniform divisor by multiply-high (n, d < 2^31): the
// tile -> (replica, row block, column block) split runs once per tile in
// every warp role, and a generic integer division is ~20 instructions.
struct FastDiv {
  uint32_t d, m, l;
  __device__ __forceinline__ void init(uint32_t d_) {
    d = d_;
    l = 0;
    while ((1u << l) < d && l < 31) l++;
    m = (uint32_t)((((1ull << l) - d) << 32) / d + 1);
  }
  __device__ __forceinline__ uint32_t div(uint32_t n) const { return (__umulhi(n, m) + n) >> l; }
};
__device__ __forceinline__ void tma_load_2d(const CUtensorMap* tm, uint64_t* bar,
                                            void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(tm), "r"(su32(bar)), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void tma_load_3d(const CUtensorMap* tm, uint64_t* bar, void* dst, int x,
                                            int y, int z) {
  asm volatile(
      "cp.async.bulk.tensor.3d.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4, %5}], [%2];" ::"r"(su32(dst)),
      "l"(tm), "r"(su32(bar)), "r"(x), "r"(y), "r"(z)
      : "memory");
}
__device__ __forceinline__ void sts_f32(uint32_t addr, float v) {
  asm volatile("st.shared.f32 [%0], %1;" ::"r"(addr), "f"(v) : "memory");
}
__device__ __forceinline__ float lds_f32(uint32_t addr) {
  float v;
  asm volatile("ld.shared.f32 %0, [%1];" : "=f"(v) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void sts_v4(uint32_t addr, uint32_t x, uint32_t y, uint32_t z,
                                       uint32_t w) {
  asm volatile("st.shared.v4.u32 [%0], {%1, %2, %3, %4};" ::"r"(addr), "r"(x), "r"(y), "r"(z),
               "r"(w)
               : "memory");
}
__device__ __forceinline__ float4 lds_f4(uint32_t addr) {
  float4 v;
  asm volatile("ld.shared.v4.f32 {%0, %1, %2, %3}, [%4];"
               : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ uint2 lds_u2(uint32_t addr) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(addr) : "memory");
  return v;
}
__device__ __forceinline__ void stg_u2(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1, %2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}
__device__ __forceinline__ uint4 lds_u4(uint32_t addr) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w)
               : "r"(addr)
               : "memory");
  return v;
}
__device__ __forceinline__ void stg_u4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1, %2, %3, %4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void stg_f4(void* p, float4 v) {
  asm volatile("st.global.v4.f32 [%0], {%1, %2, %3, %4};" ::"l"(p), "f"(v.x), "f"(v.y),
               "f"(v.z), "f"(v.w)
               : "memory");
}
// ---- SM-pair (cta_group::2) helpers
__device__ __forceinline__ uint32_t cluster_rank() {
  uint32_t r;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(r));
  return r;
}
// shared::cluster address of the same smem offset in CTA `rank` of the cluster
__device__ __forceinline__ uint32_t mapa_cluster(const void* p, uint32_t rank) {
  uint32_t r;
  asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(r) : "r"(su32(p)), "r"(rank));
  return r;
}
__device__ __forceinline__ void mbar_arrive_cluster(uint32_t cluster_addr) {
  asm volatile("mbarrier.arrive.release.cluster.shared::cluster.b64 _, [%0];" ::"r"(cluster_addr)
               : "memory");
}
__device__ __forceinline__ void cluster_sync_all() {
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
}
// TMA into this CTA's smem, completion counted on the pair leader's mbarrier
__device__ __forceinline__ void tma_load_2d_pair(const CUtensorMap* tm, uint32_t bar_cluster,
                                                 void* dst, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.cta_group::2.shared::cluster.global.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%3, %4}], [%2];" ::"r"(su32(dst)),
      "l"(tm), "r"(bar_cluster), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void umma_commit_pair(uint64_t* b) {  // both CTAs' barrier
  asm volatile(
      "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;" ::"r"(su32(b)), "h"((uint16_t)3)
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair(uint32_t d, uint64_t a, uint64_t b,
                                               uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
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
// Warp-collective forms: every lane of the warp executes them, one lane
// (elect.sync) issues the tcgen05 instruction.
// Four MMAs under one elect: descriptors a + 2j, b + bstep * j (j = 0..3),
// the first accumulating when accum != 0, the rest always. One elect and
// one set of uniform-register moves per 4 MMAs instead of per MMA (the MMA
// warp's issue overhead bounds the N = 64 layers): a k-block's 4 K = 16
// slices (bstep 2) or the s2d stem's 4 dx taps (+32 B rows of A, +2 KB tap
// tiles of B).
template <int BSTEP>
__device__ __forceinline__ void umma_bf16_x4_w(uint32_t d, uint64_t a, uint64_t b, uint32_t idesc,
                                               uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 a1, a2, a3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "add.s64 a1, %1, 2;\n\tadd.s64 a2, %1, 4;\n\tadd.s64 a3, %1, 6;\n\t"
      "add.s64 b1, %2, %5;\n\tadd.s64 b2, %2, %6;\n\tadd.s64 b3, %2, %7;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a1, b1, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a2, b2, %3, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], a3, b3, %3, 1;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum), "n"(BSTEP), "n"(2 * BSTEP), "n"(3 * BSTEP));
}

// The same 4 taps for two accumulators (d0 with A a0, d1 with A a1, shared
// B), interleaved so that no MMA waits on the previous one's accumulation:
// a K = 16, N = 64 MMA is shorter than the accumulate latency, so back-to-
// back MMAs into one accumulator run at the latency, not the tensor rate.
template <int BSTEP>
__device__ __forceinline__ void umma_bf16_x4x2_w(uint32_t d0, uint32_t d1, uint64_t a0,
                                                 uint64_t a1, uint64_t b, uint32_t idesc,
                                                 uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t.reg .b64 x1, x2, x3, y1, y2, y3, b1, b2, b3;\n\t"
      "setp.ne.b32 p, %6, 0;\n\t"
      "add.s64 x1, %2, 2;\n\tadd.s64 x2, %2, 4;\n\tadd.s64 x3, %2, 6;\n\t"
      "add.s64 y1, %3, 2;\n\tadd.s64 y2, %3, 4;\n\tadd.s64 y3, %3, 6;\n\t"
      "add.s64 b1, %4, %7;\n\tadd.s64 b2, %4, %8;\n\tadd.s64 b3, %4, %9;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], %2, %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], %3, %4, %5, p;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x1, b1, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], y1, b1, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x2, b2, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], y2, b2, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%0], x3, b3, %5, 1;\n\t"
      "@e tcgen05.mma.cta_group::1.kind::f16 [%1], y3, b3, %5, 1;\n}" ::"r"(d0),
      "r"(d1), "l"(a0), "l"(a1), "l"(b), "r"(idesc), "r"(accum), "n"(BSTEP), "n"(2 * BSTEP),
      "n"(3 * BSTEP));
}
// bf16x2 pack of (lo, hi) with the ReLU folded into the conversion
// (cvt.rn.relu: negative -> 0 in the same instruction; lo in the low half)
__device__ __forceinline__ uint32_t pack_bf16x2_relu(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.relu.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  uint32_t d;
  asm("cvt.rn.bf16x2.f32 %0, %1, %2;" : "=r"(d) : "f"(hi), "f"(lo));
  return d;
}
// x[0..31] += the bf16 residual of 16-byte chunks J0..J0+3 of this lane's
// 128-byte row (128B-swizzled residual box row at rbase; row % 8 == lane % 8)
template <int J0>
__device__ __forceinline__ void add_res_row(float* x, uint32_t rbase, int lane) {
#pragma unroll
  for (int j = 0; j < 4; j++) {
    const uint4 rv = lds_u4(rbase + (uint32_t)((((J0 + j) ^ (lane & 7))) << 4));
    const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
    for (int e = 0; e < 4; e++) {
      x[8 * j + 2 * e] += __uint_as_float(w[e] << 16);
      x[8 * j + 2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
    }
  }
}
// ReLU / ReLU6 / none + bf16 pack of 2n floats
template <int N2>
__device__ __forceinline__ void act_pack(const float* x, uint32_t* o, int relu) {
  if (relu == 1) {
#pragma unroll
    for (int j = 0; j < N2; j++) o[j] = pack_bf16x2_relu(x[2 * j], x[2 * j + 1]);
  } else if (relu == 2) {
#pragma unroll
    for (int j = 0; j < N2; j++)
      o[j] = pack_bf16x2_relu(fminf(x[2 * j], 6.f), fminf(x[2 * j + 1], 6.f));
  } else {
#pragma unroll
    for (int j = 0; j < N2; j++) o[j] = pack_bf16x2(x[2 * j], x[2 * j + 1]);
  }
}
__device__ __forceinline__ void umma_commit_w(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n}" ::"r"(
          su32(b))
      : "memory");
}
__device__ __forceinline__ void umma_bf16_pair_w(uint32_t d, uint64_t a, uint64_t b,
                                                 uint32_t idesc, uint32_t accum) {
  asm volatile(
      "{\n\t.reg .pred p, e;\n\t"
      "setp.ne.b32 p, %4, 0;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(d),
      "l"(a), "l"(b), "r"(idesc), "r"(accum));
}
__device__ __forceinline__ void umma_commit_pair_w(uint64_t* b) {
  asm volatile(
      "{\n\t.reg .pred e;\n\t"
      "elect.sync _|e, 0xffffffff;\n\t"
      "@e tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
      " [%0], %1;\n}" ::"r"(su32(b)), "h"((uint16_t)3)
      : "memory");
}
// K-major, 128B-swizzled operand tile: 8-row atoms of 1024 B (SBO), version 1.
__device__ __forceinline__ uint64_t smem_desc_sw128(const void* p) {
  uint64_t addr = su32(p);
  return ((addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}
// The same tile starting at an arbitrary 128-byte row of a TMA-written halo
// (halo mode). Measured on B200: the UMMA read applies the 128B swizzle on
// absolute smem address bits, exactly like the TMA write, so the start
// address alone selects the row and the base-offset field [49,52) stays 0
// (setting it to (addr >> 7) & 7 reads the wrong rows).
__device__ __forceinline__ uint64_t smem_desc_sw128_row(uint32_t addr, int) {
  return (((uint64_t)addr >> 4) & 0x3FFFull) | (1ull << 16) | (64ull << 32) | (1ull << 46) |
         (2ull << 61);
}
// K-major operand with 32-byte rows (K = 16 bf16) under the 32B swizzle (the
// s2d stem): 8-row atoms of 256 B (SBO), layout type 6. Like the 128B halo
// mode, the start address may sit at any 32-byte row of a TMA-written box:
// the swizzle follows absolute smem address bits.
__device__ __forceinline__ uint64_t smem_desc_sw32_row(uint32_t addr) {
  return (((uint64_t)addr >> 4) & 0x3FFFull) | (1ull << 16) | ((uint64_t)(256 >> 4) << 32) |
         (1ull << 46) | (6ull << 61);
}
// tcgen05.ld without the wait (the registers are valid after tmem_ld_wait).
__device__ __forceinline__ void tmem_ld32_issue(uint32_t taddr, uint32_t (&v)[32]) {
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
}
// Waits for outstanding tcgen05.ld; the "+r" operands keep the compiler from
// reading v[] before the wait.
__device__ __forceinline__ void tmem_ld_wait(uint32_t (&v)[32]) {
  asm volatile("tcgen05.wait::ld.sync.aligned;"
               : "+r"(v[0]), "+r"(v[1]), "+r"(v[2]), "+r"(v[3]), "+r"(v[4]), "+r"(v[5]),
                 "+r"(v[6]), "+r"(v[7]), "+r"(v[8]), "+r"(v[9]), "+r"(v[10]), "+r"(v[11]),
                 "+r"(v[12]), "+r"(v[13]), "+r"(v[14]), "+r"(v[15]), "+r"(v[16]),
                 "+r"(v[17]), "+r"(v[18]), "+r"(v[19]), "+r"(v[20]), "+r"(v[21]),
                 "+r"(v[22]), "+r"(v[23]), "+r"(v[24]), "+r"(v[25]), "+r"(v[26]),
                 "+r"(v[27]), "+r"(v[28]), "+r"(v[29]), "+r"(v[30]), "+r"(v[31])
               :
               : "memory");
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

// TMA bulk store of a [32 rows x 32 cols] bf16 box from (64B-swizzled) smem.
__device__ __forceinline__ void tma_store_2d(const CUtensorMap* tm, uint32_t src, int x, int y) {
  asm volatile(
      "cp.async.bulk.tensor.2d.global.shared::cta.bulk_group [%0, {%2, %3}], [%1];" ::"l"(tm),
      "r"(src), "r"(x), "r"(y)
      : "memory");
}
__device__ __forceinline__ void bulk_commit() {
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}
template <int N>
__device__ __forceinline__ void bulk_wait_read() {  // <= N groups still reading smem
  asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(N) : "memory");
}
__device__ __forceinline__ void bulk_wait_all() {
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}
__device__ __forceinline__ void fence_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
// 16-byte chunk j of 64-byte row r under the 64B TMA swizzle (addr bits
// [4,6) ^= bits [7,9)).
__device__ __forceinline__ uint32_t sw64(int r, int j) {
  return (uint32_t)(r * 64 + 16 * (j ^ ((r >> 1) & 3)));
}

// Output row of GEMM row m under ConvGemmArgs::row_mode (-1: not stored),
// the mode's two divisors as multiply-high divisions set up once per thread
// (the epilogue maps one row per thread per tile).
// Zero-bordered pixel grid with shared borders: each grid row is W pixels
// plus one zero column (the right border of a row is the left border of the
// next), each image H + 1 grid rows of which row 0 is zero (the bottom
// border of the image above). Pixel (n, h, w) sits at grid row
// n (H+1)(W+1) + (h+1)(W+1) + w; the 3x3 taps are shifts by
// (dr-1)(W+1) + (ds-1); index -1 (top-left of image 0) and the rows past the
// last image are TMA out-of-bounds zeros. (H+1)(W+1) rows per image instead
// of (H+2)(W+2): 21 % fewer MMA rows at 7x7.
struct RowRemap {
  FastDiv d1, d2;
  int mode, M, rows_out, H, W, Bn;
  __device__ __forceinline__ void init(const ConvGemmArgs& a) {
    mode = a.row_mode;
    M = a.M;
    rows_out = a.rows_out;
    H = a.H;
    W = a.W;
    Bn = 0;
    switch (mode) {
      case kRowGridToCompact:
      case kRowGridToPad: d1.init(a.gh * a.gw); d2.init(a.gw); break;
      case kRowPhaseGridToCompact:
      case kRowPadToCompact:
      case kRowPadToPad: d1.init((H + 1) * (W + 1)); d2.init(W + 1); break;
      case kRowCompactToPhasePad:
      case kRowCompactToPad:
        d1.init(H * W);
        d2.init(W);
        Bn = M / (H * W);
        break;
      default: d1.init(1); d2.init(1);
    }
  }
  __device__ __forceinline__ int map(int m) const {
    if (m >= M) return -1;
    if (mode == kRowIdentity) return m < rows_out ? m : -1;
    const int n = (int)d1.div(m), rem = m - n * (int)d1.d;
    const int i = (int)d2.div(rem), j = rem - i * (int)d2.d;
    switch (mode) {
      case kRowGridToCompact:
      case kRowPhaseGridToCompact: return (i < H && j < W) ? (n * H + i) * W + j : -1;
      case kRowGridToPad:  // -> the shared-border grid's interior
        return (i < H && j < W) ? (n * (H + 1) + i + 1) * (W + 1) + j : -1;
      case kRowCompactToPhasePad: {
        const int h = i + 1, w = j + 1, Hq = (H + 2) >> 1, Wq = (W + 2) >> 1;
        return ((((h & 1) * 2 + (w & 1)) * Bn + n) * Hq + (h >> 1)) * Wq + (w >> 1);
      }
      case kRowPadToCompact:
      case kRowPadToPad:
        if (i < 1 || j >= W) return -1;
        return mode == kRowPadToPad ? m : (n * H + i - 1) * W + j;
      default: return (n * (H + 1) + i + 1) * (W + 1) + j;  // compact -> shared-border grid
    }
  }
};

// ------------------------------------------------------------ tile scheduler
// The work of a launch is `units` runs of T consecutive tiles.
//  * static (a.sched == 0: SM-pair launches, tests that force a small grid):
//    a persistent grid, CTA (pair) b takes units b, b + G, b + 2G, ...
//  * CLC (a.sched == 1, the default): one CTA per unit. A running CTA takes
//    its own unit, then keeps cancelling not-yet-launched CTAs of its grid
//    with Blackwell cluster launch control (clusterlaunchcontrol.try_cancel)
//    and runs their units instead. A CTA that cannot get an SM -- because the
//    SHA-256 chain kernels of the ingest streams hold it -- never runs: the
//    resident CTAs take its work, so no tile ever waits behind another
//    kernel, and the grid needs no SM budget guessed on the host.
// One cancel request is in flight per CTA (issued by the TMA producer when it
// starts a unit); its 16-byte response lands in a ring slot whose mbarrier
// every consumer warp waits on, and every warp that walks the tile sequence
// releases the slot (cempty counts those warps).
constexpr int kClcSlots = 8;
struct TileSched {
  int tiles, T, step;
  bool clc;
  uint32_t resp, cfull, cempty;  // shared::cta addresses of slot 0
  int unit = 0, k = 0, nu = 0, t = 0;
  __device__ __forceinline__ void issue(int q) const {
    const int slot = q % kClcSlots, use = q / kClcSlots;
    const uint32_t e = cempty + 8 * slot, f = cfull + 8 * slot;
    if (use >= 1) {
      asm volatile(
          "{\n\t.reg .pred p;\n"
          "CLCE_%=:\n\t"
          "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
          "@!p bra CLCE_%=;\n}" ::"r"(e), "r"((uint32_t)((use - 1) & 1))
          : "memory");
    }
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], 16;" ::"r"(f) : "memory");
    asm volatile(
        "clusterlaunchcontrol.try_cancel.async.shared::cta.mbarrier::complete_tx::bytes.b128"
        " [%0], [%1];" ::"r"(resp + 16 * slot), "r"(f)
        : "memory");
  }
  // Response q: true and the cancelled CTA's unit, or false (grid exhausted).
  __device__ __forceinline__ bool take(int q, int& u, bool arrive) const {
    const int slot = q % kClcSlots, use = q / kClcSlots;
    const uint32_t f = cfull + 8 * slot;
    asm volatile(
        "{\n\t.reg .pred p;\n"
        "CLCF_%=:\n\t"
        "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t"
        "@!p bra CLCF_%=;\n}" ::"r"(f), "r"((uint32_t)(use & 1))
        : "memory");
    uint32_t ok, x;
    asm volatile(
        "{\n\t.reg .b128 rr;\n\t.reg .pred p;\n\t"
        "ld.shared.b128 rr, [%2];\n\t"
        "clusterlaunchcontrol.query_cancel.is_canceled.pred.b128 p, rr;\n\t"
        "selp.u32 %0, 1, 0, p;\n\t"
        "clusterlaunchcontrol.query_cancel.get_first_ctaid::x.b32.b128 %1, rr;\n}"
        : "=r"(ok), "=r"(x)
        : "r"(resp + 16 * slot)
        : "memory");
    __syncwarp(__activemask());
    if (arrive)
      asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(cempty + 8 * slot) : "memory");
    u = (int)x;
    return ok != 0;
  }
  __device__ __forceinline__ bool first(int first_unit, bool issuer) {
    unit = first_unit;
    k = 0;
    nu = 1;
    t = unit * T;
    if (t >= tiles) return false;
    if (clc && issuer) issue(0);
    return true;
  }
  // arrive: this thread releases response slots for its warp (lane 0)
  __device__ __forceinline__ bool next(bool issuer, bool arrive) {
    if (++k < T && t + 1 < tiles) {
      t++;
      return true;
    }
    if (!clc) {
      unit += step;
      k = 0;
      t = unit * T;
      return t < tiles;
    }
    const int q = nu - 1;
    int u;
    if (!take(q, u, arrive)) return false;
    unit = u;
    nu++;
    k = 0;
    t = unit * T;
    if (issuer) issue(q + 1);
    return true;
  }
};

#define CG_TRACE(slot, i)                                             \
  do {                                                                \
    if (a.trace && blockIdx.x == 0 && (i) < 64 && (lane == 0))        \
      a.trace[(slot) * 64 + (i)] = clock64();                         \
  } while (0)

// PAIR: an SM pair (cluster of 2, cta_group::2) computes 256-row tiles: each
// CTA loads its 128 rows of A (or its 128-row halo) and half of the weight
// tile (BN/2 rows) with cta_group::2 TMA that completes on the leader's
// barrier; the leader issues M=256 MMAs over both CTAs' shared memory and
// commits to both CTAs' barriers; each CTA's epilogue drains its own TMEM
// half and the peer releases the accumulator on the leader's barrier.
// Per SM and 128x256 output this halves the weight bytes written to and read
// from shared memory (the bound of the BN=256 mainloop).
// Floats of epilogue staging per epilogue warp: 32 x kStgLd for the f32 /
// remapped-row staging paths, 1024 (2 x 2 KB) for the TMA-store path only,
// 0 for halo variants whose remapped bf16 rows go out by direct stores. The
// launcher picks the reduced variants only for outputs that fit them; the
// freed shared memory buys mainloop stages / halo slots.
template <int BN, int STAGES, int kResSlots, int HALO, int RESB, int PAIR, int HROWS = 256>
constexpr int stg_floats() {
  if (HROWS > 256) return 0;  // wide halos: remapped rows, staging-free direct stores
  if (!PAIR && BN == 256 && STAGES == 2 && kResSlots == 12) return 1024;  // residual: 6 boxes
  // staging blocks are 1024-aligned (5 KB >= the generic path's 32 x 36
  // floats) for the 128B-swizzled 32 x 64 bulk stores of the block path
  if (PAIR || kResSlots) return 1280;
  if (HALO == 0 && ((BN == 256 && STAGES == 4) || (BN == 128 && STAGES == 6) ||
                    (BN == 64 && STAGES == 8)))
    return 1024;
  if ((BN == 256 && STAGES == 4 && HALO == 2) || (BN == 128 && STAGES == 8 && HALO == 2) ||
      (BN == 64 && STAGES == 8 && HALO == 4) || (BN == 64 && RESB == 9 && HALO == 4))
    return 0;
  // 64-wide tiles: one 32 x 128 B staging block per warp, 1024-aligned for
  // the 128B-swizzled bulk store (the s2d stem: 4 KB exactly)
  if (BN == 64 && RESB == 4 && HALO == 12) return 1024;
  return 1280;
}

template <int BN, int STAGES, int kResSlots, int HALO, int RESB, int PAIR, int S2D = 0,
          int A2S = 0, int HROWS = 256>
__global__ void __launch_bounds__(kThreads, 1)
    conv_gemm_kernel(const __grid_constant__ GemmGroupParams gp, const ConvGemmArgs a) {
  // A2S (strided second segment): A slots hold up to 4 boxes of 56 rows
  constexpr int kASlot = A2S ? 4 * 56 * 128 : A_BYTES;
  static_assert(!A2S || (HALO == 0 && RESB == 0 && !PAIR && !S2D), "strided A2: plain GEMMs");
  // 4-stage 256-wide streamed GEMMs: epilogue staging sized for the
  // TMA-store path only (2 x 2 KB per warp; the launcher picks them for bf16
  // outputs, which take the TMA-store or the staging-free direct-store
  // epilogue), which frees the fourth stage
  constexpr int kStgWarp = stg_floats<BN, STAGES, kResSlots, HALO, RESB, PAIR, HROWS>();
  static_assert(!PAIR || (RESB == 0 && (HALO == 0 || kResSlots == 0)), "pair: streamed weights");
  static_assert(!S2D || (BN == 64 && RESB == 4 && HALO > 0 && !PAIR), "s2d stem layout");
  // s2d stem: a ring slot holds one dy box (2 planes x (BM + 3) rows x 16 B)
  // halo slot: HROWS rows of 128 B (wide halos: several stacked boxes)
  constexpr int kHaloB = HROWS * BK * 2;
  constexpr int kHaloSlot = S2D ? kS2DSlot : kHaloB;
  constexpr int B_BYTES = (PAIR ? BN / 2 : BN) * BK * 2;  // this CTA's weight tile
  // s2d stem: 256-row tiles of two 128-row sub-tiles (2 accumulators each)
  constexpr int kSubTiles = S2D ? 2 : 1;
  constexpr uint32_t TMEM_COLS = 2 * BN * kSubTiles;
  // BN = 64 (2 chunks of 32 columns): the two epilogue warp groups take
  // alternate tiles whole; wider tiles split their chunks between the groups.
  // An accumulator is released (tempty) by exactly the warps that drained it.
  constexpr bool kTileSplit = BN == 64 && !S2D;  // s2d: group h drains sub-tile h
  constexpr int kDrainWarps = kTileSplit ? kEpiWarps / 2 : kEpiWarps;
  // epilogue block path: whole 64-column blocks per warp (see the epilogue)
  constexpr int kCPT = BN / 32, kC0S = (kTileSplit || S2D) ? 1 : 2;
  constexpr bool kBlockPath = !PAIR && stg_floats<BN, STAGES, kResSlots, HALO, RESB, PAIR, HROWS>() >=
                                           1024 && ((kC0S == 1 && kCPT == 2) || kC0S == 2);
  // residual ring: 128-row boxes of kResCols columns (64: 128-byte rows, SW128;
  // half the TMA row requests of 32-column SW64 boxes) in kResSlots x 8 KB
  constexpr int kResCols = CG_RES_COLS;
  constexpr int kResBox = 128 * kResCols * 2;
  constexpr int kRS = kResSlots > 0 ? kResSlots * 8192 / kResBox : 1;
  extern __shared__ uint8_t smem_raw[];
  // 1024-aligned regions first: operand ring (128B swizzle), residual ring and
  // output staging (64B swizzle), then barriers.
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + (HALO > 0 ? HALO * kHaloSlot : STAGES * kASlot);
  uint8_t* s_res = sB + (RESB > STAGES ? RESB : STAGES) * B_BYTES;  // residual ring (SW64)
  float* s_epi = reinterpret_cast<float*>(s_res + kResSlots * 8192);  // 36 KB
  uint64_t* full = reinterpret_cast<uint64_t*>(s_epi + kEpiWarps * kStgWarp);
  uint64_t* empty = full + STAGES;
  uint64_t* tfull = empty + STAGES;
  uint64_t* tempty = tfull + 2;
  uint64_t* rfull = tempty + 2;
  uint64_t* rempty = rfull + (kResSlots > 0 ? kResSlots : 1);
  uint64_t* hfull = rempty + (kResSlots > 0 ? kResSlots : 1);  // halo ring
  uint64_t* hempty = hfull + (HALO > 0 ? HALO : 1);
  uint32_t* tmem_slot = reinterpret_cast<uint32_t*>(hempty + (HALO > 0 ? HALO : 1));
  int* s_tap = reinterpret_cast<int*>(tmem_slot + 4);
  // CLC response ring (16 B aligned) and its full/empty barriers
  uint8_t* clc_base = reinterpret_cast<uint8_t*>(
      (reinterpret_cast<uintptr_t>(s_tap + 9) + 15) & ~uintptr_t(15));
  uint64_t* cfull = reinterpret_cast<uint64_t*>(clc_base + 16 * kClcSlots);
  uint64_t* cempty = cfull + kClcSlots;
  // identity rows + bf16 out: thread-per-row epilogue, TMA bulk stores
  const bool tma_out = a.row_mode == kRowIdentity && !a.out_f32;
  const bool res_tma = kResSlots > 0 && gp.residual[0] != nullptr && tma_out;

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int num_n = (a.N + BN - 1) / BN, num_m = (a.M + BM - 1) / BM;
  // tile order t -> (m block, replica r, n block): the replicas' tiles of one
  // row block run back to back, so an operand they share (the conv1 im2col
  // of the batch) is read from HBM once and from L2 by the other replicas
  // pair: a tile is 256 rows (this CTA's 128-row half at crank * 128)
  const uint32_t crank = PAIR ? cluster_rank() : 0;
  constexpr int BMT = (PAIR || S2D) ? 2 * BM : BM;
  const int num_mt = (a.M + BMT - 1) / BMT;
  const int tiles = num_mt * num_n * gp.n;
  const int first_unit = PAIR ? (int)(blockIdx.x >> 1) : (int)blockIdx.x;
  const int kpt = S2D ? 4 : a.Kc / BK;  // s2d: kpt = the 4 dy boxes
  const int num_k1 = a.ntaps * kpt, num_k = num_k1 + a.kc2 / BK;  // + second K segment
  (void)num_m;
  // one halo: halo_sub stacked boxes of hbox rows (one box when halo_sub <= 1)
  const int hsub = a.halo_sub > 1 ? a.halo_sub : 1;
  const int hbox = hsub > 1 ? a.halo_box : BM + 2 * a.halo_lo;
  auto load_halo = [&](const CUtensorMap* map, uint64_t* bar, uint8_t* dst, int x, int y) {
    mbar_expect_tx(bar, hsub * hbox * BK * 2);
    for (int j = 0; j < hsub; j++) tma_load_2d(map, bar, dst + j * hbox * BK * 2, x, y + j * hbox);
  };
  static_assert(HROWS == 256 || (!PAIR && !S2D), "wide halos: single-SM, non-stem");
  FastDiv div_outer, div_n;  // per_r (RESB) or per_m, and num_n
  div_outer.init(RESB > 0 ? num_mt * num_n : gp.n * num_n);
  div_n.init(num_n);
  auto coords = [&](int t, int& r, int& m0, int& n0) {
    if constexpr (RESB > 0) {
      // resident weights: replica-major, so a CTA's consecutive tiles (and
      // the units it steals, which follow launch order) rarely switch replica
      r = (int)div_outer.div(t);
      const int rem = t - r * (int)div_outer.d, mb = (int)div_n.div(rem);
      m0 = mb * BMT + (int)crank * BM;
      n0 = (rem - mb * num_n) * BN;
    } else {
      const int mb = (int)div_outer.div(t), rem = t - mb * (int)div_outer.d;
      r = (int)div_n.div(rem);
      m0 = mb * BMT + (int)crank * BM;
      n0 = (rem - r * num_n) * BN;
    }
  };

  if (warp == 0 && lane == 0) {
#pragma unroll
    for (int i = 0; i < 9; i++) s_tap[i] = a.tap_off[i];
  }
  if (warp == 0 && lane == 0) {
    for (int r = 0; r < gp.n; r++) {
      asm volatile("prefetch.tensormap [%0];" ::"l"(&gp.A[r]) : "memory");
      asm volatile("prefetch.tensormap [%0];" ::"l"(&gp.B[r]) : "memory");
      if (a.kc2) asm volatile("prefetch.tensormap [%0];" ::"l"(&gp.A2[r]) : "memory");
      if (tma_out) asm volatile("prefetch.tensormap [%0];" ::"l"(&gp.O[r]) : "memory");
      if (res_tma) asm volatile("prefetch.tensormap [%0];" ::"l"(&gp.R[r]) : "memory");
    }
    for (int s = 0; s < STAGES; s++) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
    }
    for (int s = 0; s < 2; s++) {
      mbar_init(&tfull[s], 1);
      mbar_init(&tempty[s], kDrainWarps * (PAIR ? 2 : 1));  // pair: both CTAs' epilogues
    }
    for (int s = 0; s < kResSlots; s++) {
      mbar_init(&rfull[s], 1);
      // block path: a box is one warp group's 64-column block (4 warps);
      // chunk path: 4 warps x the box's 32-column chunks
      mbar_init(&rempty[s], kBlockPath ? 4 : 4 * (kResCols / 32));
    }
    for (int s = 0; s < HALO; s++) {
      mbar_init(&hfull[s], 1);
      mbar_init(&hempty[s], 1);
    }
    // CLC slots are released by the producer, the MMA warp, the 8 epilogue
    // warps and (when it streams a residual) the residual loader
    for (int s = 0; s < kClcSlots; s++) {
      mbar_init(&cfull[s], 1);
      mbar_init(&cempty[s], 2 + kEpiWarps + (res_tma ? 1 : 0));
    }
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    if constexpr (PAIR) {
      asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
    } else {
      asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                       su32(tmem_slot)),
                   "r"(TMEM_COLS)
                   : "memory");
      asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
    }
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();  // peer barriers initialised before any remote arrive
  else __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tmem_slot;
  TileSched sched;
  sched.tiles = tiles;
  sched.T = a.sched ? a.tile_unit : 1;
  sched.step = PAIR ? (int)(gridDim.x >> 1) : (int)gridDim.x;
  sched.clc = !PAIR && a.sched != 0;
  sched.resp = su32(clc_base);
  sched.cfull = su32(cfull);
  sched.cempty = su32(cempty);
  // Programmatic dependent launch: the setup above (barriers, TMEM, tensor
  // map prefetch) overlapped the previous launch's tail; wait for that grid
  // and its memory before reading activations or writing outputs, and let
  // the next launch's CTAs take SMs as this grid's CTAs retire.
  asm volatile("griddepcontrol.wait;" ::: "memory");
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");

  if (warp == 0) {
    if (lane == 0) {  // ---------------- TMA producer
      int stage = 0;
      uint32_t phase = 0;
      int ti = 0;
      int hs = 0;
      uint32_t hphase = 0;
      int wr = -1, wl = 0;  // RESB: replica whose weights are resident, loads so far
      for (bool ok = sched.first(first_unit, true); ok; ok = sched.next(true, true), ti++) {
        const int t = sched.t;
        int r, m0, n0;
        coords(t, r, m0, n0);
        CG_TRACE(0, ti);
        if constexpr (RESB > 0) {
          // resident weights (one n block): all RESB tiles of B are loaded
          // when the replica changes (full[0] / empty[0] are the weight
          // barriers: the MMA warp releases the old set before a reload);
          // per tile only the halo boxes stream
          if (r != wr) {
            if (wl > 0) mbar_wait(&empty[0], (uint32_t)((wl - 1) & 1));
            mbar_expect_tx(&full[0], RESB * B_BYTES);
            if constexpr (S2D) {  // 16 taps x 64 rows x 32 B, 256-row boxes
              for (int j = 0; j < RESB * B_BYTES / 8192; j++)
                tma_load_2d(&gp.B[r], &full[0], sB + j * 8192, 0, j * 256);
            } else {
              for (int j = 0; j < RESB; j++)
                tma_load_2d(&gp.B[r], &full[0], sB + j * B_BYTES, j * BK, n0);
            }
            wr = r;
            wl++;
          }
          if constexpr (S2D) {
            // per dy pair (or per dy), one box per sub-tile: BM + gw + 3
            // (or BM + 3) rows
            const int step = a.s2d_step == 1 ? 1 : 2;
            const int nbox = step == 1 && a.s2d_ndy > 0 ? a.s2d_ndy : 4 / step;
            const int brows = BM + (step - 1) * a.gw + 3;
            for (int h = 0; h < nbox; h++)
              for (int sub = 0; sub < kSubTiles; sub++) {
                mbar_wait(&hempty[hs], hphase ^ 1);
                mbar_expect_tx(&hfull[hs], brows * 32);
                tma_load_2d(&gp.A[r], &hfull[hs], sA + hs * kHaloSlot, 0,
                            m0 + sub * BM + step * h * a.gw);
                if (++hs == HALO) { hs = 0; hphase ^= 1; }
              }
            continue;
          }
          for (int cb = 0; cb < kpt; cb++) {
            mbar_wait(&hempty[hs], hphase ^ 1);
            load_halo(&gp.A[r], &hfull[hs], sA + hs * kHaloB, cb * BK, m0 - a.halo_lo);
            if (++hs == HALO) { hs = 0; hphase ^= 1; }
          }
          continue;
        }
        if constexpr (PAIR && HALO > 0) {
          // both CTAs load their halves; all completions land on the
          // leader's barriers, which expect both CTAs' bytes
          const int hrows = BM + 2 * a.halo_lo;
          for (int cb = 0; cb < kpt; cb++) {
            mbar_wait(&hempty[hs], hphase ^ 1);
            if (crank == 0) mbar_expect_tx(&hfull[hs], 2 * hrows * BK * 2);
            tma_load_2d_pair(&gp.A[r], mapa_cluster(&hfull[hs], 0), sA + hs * kHaloB, cb * BK,
                             m0 - a.halo_lo);
            if (++hs == HALO) { hs = 0; hphase ^= 1; }
            for (int tap = 0; tap < a.ntaps; tap++) {
              mbar_wait(&empty[stage], phase ^ 1);
              if (crank == 0) mbar_expect_tx(&full[stage], 2 * B_BYTES);
              tma_load_2d_pair(&gp.B[r], mapa_cluster(&full[stage], 0), sB + stage * B_BYTES,
                               (tap * kpt + cb) * BK, n0 + (int)crank * (BN / 2));
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          }
          continue;
        }
        if constexpr (HALO > 0) {
          // per channel block: one halo box, then the 9 taps' weight tiles
          for (int cb = 0; cb < kpt; cb++) {
            mbar_wait(&hempty[hs], hphase ^ 1);
            load_halo(&gp.A[r], &hfull[hs], sA + hs * kHaloB, cb * BK, m0 - a.halo_lo);
            if (++hs == HALO) { hs = 0; hphase ^= 1; }
            for (int tap = 0; tap < a.ntaps; tap++) {
              mbar_wait(&empty[stage], phase ^ 1);
              mbar_expect_tx(&full[stage], B_BYTES);
              tma_load_2d(&gp.B[r], &full[stage], sB + stage * B_BYTES, (tap * kpt + cb) * BK,
                          n0);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
          }
          continue;
        }
        if constexpr (PAIR) {
          // this CTA's 128 rows of A and half of the weight tile, completing
          // on the leader's barrier (which expects both CTAs' bytes)
          for (int kb = 0; kb < num_k; kb++) {
            const int tap = kb / kpt, cb = kb - tap * kpt;
            mbar_wait(&empty[stage], phase ^ 1);
            if (kb == 0) CG_TRACE(1, ti);
            uint32_t fb = mapa_cluster(&full[stage], 0);
            if (crank == 0) mbar_expect_tx(&full[stage], 2 * (A_BYTES + B_BYTES));
            tma_load_2d_pair(&gp.A[r], fb, sA + stage * A_BYTES, cb * BK, m0 + s_tap[tap]);
            tma_load_2d_pair(&gp.B[r], fb, sB + stage * B_BYTES, kb * BK,
                             n0 + (int)crank * (BN / 2));
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          continue;
        }
        for (int kb = 0; kb < num_k; kb++) {
          const int tap = kb / kpt, cb = kb - tap * kpt;
          mbar_wait(&empty[stage], phase ^ 1);
          if (kb == 0) CG_TRACE(1, ti);
          if (A2S && kb >= num_k1) {
            // strided second segment: the output rows covering [m0, m0 + 128)
            const int rows_box = a.a2_rpb * a.a2_wo, r0 = m0 / a.a2_wo;
            const int nbox = (m0 - r0 * a.a2_wo + BM + rows_box - 1) / rows_box;
            mbar_expect_tx(&full[stage], nbox * rows_box * 128 + B_BYTES);
            for (int j = 0; j < nbox; j++)
              tma_load_3d(&gp.A2[r], &full[stage], sA + stage * kASlot + j * rows_box * 128,
                          (kb - num_k1) * BK, 0, r0 + j * a.a2_rpb);
          } else {
            mbar_expect_tx(&full[stage], A_BYTES + B_BYTES);
            if (kb < num_k1)
              tma_load_2d(&gp.A[r], &full[stage], sA + stage * kASlot, cb * BK,
                          m0 + s_tap[tap]);
            else  // second K segment: the same rows of the A2 operand
              tma_load_2d(&gp.A2[r], &full[stage], sA + stage * kASlot, (kb - num_k1) * BK, m0);
          }
          tma_load_2d(&gp.B[r], &full[stage], sB + stage * B_BYTES, kb * BK, n0);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
      }
    }
  } else if (warp == 1) {
    // ---------------- MMA issuer: the whole warp runs the loop (warp-uniform
    // control flow keeps descriptors in uniform registers); one elected lane
    // issues each tcgen05 instruction
    if (crank == 0) {
      // kind::f16 instruction descriptor: D f32, A/B bf16, K-major, M=128, N=BN
      const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) |
                             ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(BM >> 4) << 24);
      int stage = 0, acc = 0, hs = 0;
      uint32_t phase = 0, acc_phase = 0, hphase = 0;
      int ti = 0;
      int mr = -1, ml = 0;  // RESB: replica of the resident weights, sets consumed
      for (bool ok = sched.first(first_unit, false); ok;
           ok = sched.next(false, lane == 0), ti++) {
        mbar_wait(&tempty[acc], acc_phase ^ 1);
        CG_TRACE(2, ti);
        tc_fence_after();
        const uint32_t d = tmem + acc * BN * kSubTiles;
        if constexpr (RESB > 0) {
          int r_, m0_, n0_;
          coords(sched.t, r_, m0_, n0_);
          if (r_ != mr) {
            if (ml > 0) umma_commit_w(&empty[0]);  // old weights free once the MMAs drain
            mbar_wait(&full[0], (uint32_t)(ml & 1));
            tc_fence_after();
            mr = r_;
            ml++;
          }
          if constexpr (S2D) {
            // 16 taps (dy, dx): A = the dy box from row dx, B = the tap's [64][16]
            const uint32_t sA_u = su32(sA), sB_u = su32(sB);
            // per dy pair: both sub-tiles' boxes (ring slots hs, hs + 1), the
            // two accumulators' MMAs interleaved
            static_assert(kSubTiles == 2 && HALO % 2 == 0, "s2d: sub-tile box pairs");
            const int step = a.s2d_step == 1 ? 1 : 2;
            const int nbox = step == 1 && a.s2d_ndy > 0 ? a.s2d_ndy : 4 / step;
            for (int h = 0; h < nbox; h++) {
              mbar_wait(&hfull[hs], hphase);
              mbar_wait(&hfull[hs + 1], hphase);
              if (h == 0) CG_TRACE(3, ti);
              tc_fence_after();
              const uint32_t hb0 = sA_u + (uint32_t)(hs * kHaloSlot), hb1 = hb0 + kHaloSlot;
              for (int j = 0; j < step; j++) {  // dy = step * h + j: rows j * gw on of each box
                const int dy = step * h + j;
                const uint32_t ro = (uint32_t)(j * a.gw * 32);
                umma_bf16_x4x2_w<2048 / 16>(d, d + BN, smem_desc_sw32_row(hb0 + ro),
                                            smem_desc_sw32_row(hb1 + ro),
                                            smem_desc_sw32_row(sB_u + (uint32_t)(dy * 4 * 2048)),
                                            idesc, dy != 0);
              }
              umma_commit_w(&hempty[hs]);
              umma_commit_w(&hempty[hs + 1]);
              hs += 2;
              if (hs == HALO) { hs = 0; hphase ^= 1; }
            }
            umma_commit_w(&tfull[acc]);
            CG_TRACE(4, ti);
            if (++acc == 2) { acc = 0; acc_phase ^= 1; }
            continue;
          }
          // 9 taps unrolled: tap offsets come from the kernel parameters and
          // every descriptor is uniform arithmetic (no per-MMA register moves)
          const uint32_t sA_u = su32(sA), sB_u = su32(sB);
          for (int cb = 0; cb < kpt; cb++) {
            mbar_wait(&hfull[hs], hphase);
            if (cb == 0) CG_TRACE(3, ti);
            tc_fence_after();
            const uint32_t hbase = sA_u + (uint32_t)(hs * kHaloB + a.halo_lo * 128);
#pragma unroll
            for (int tap = 0; tap < 9; tap++) {
              const uint64_t ad = smem_desc_sw128_row(hbase + (uint32_t)(a.tap_off[tap] * 128), 0);
              const uint64_t bd =
                  smem_desc_sw128_row(sB_u + (uint32_t)((tap * kpt + cb) * B_BYTES), 0);
              umma_bf16_x4_w<2>(d, ad, bd, idesc, (cb | tap) != 0);
            }
            umma_commit_w(&hempty[hs]);
            if (++hs == HALO) { hs = 0; hphase ^= 1; }
          }
          umma_commit_w(&tfull[acc]);
          CG_TRACE(4, ti);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
        if constexpr (PAIR && HALO == 0) {
          // leader: both CTAs' A rows and weight halves landed; M=256 MMAs
          const uint32_t idesc2 = (1u << 4) | (1u << 7) | (1u << 10) |
                                  ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
          const uint64_t ad0 = smem_desc_sw128(sA), bd0 = smem_desc_sw128(sB);
          for (int kb = 0; kb < num_k; kb++) {
            mbar_wait(&full[stage], phase);
            if (kb == 0) CG_TRACE(3, ti);
            tc_fence_after();
            const uint64_t ad = ad0 + (uint64_t)((stage * A_BYTES) >> 4);
            const uint64_t bd = bd0 + (uint64_t)((stage * B_BYTES) >> 4);
#pragma unroll
            for (int k = 0; k < BK / 16; k++)
              umma_bf16_pair_w(d, ad + 2 * k, bd + 2 * k, idesc2, (kb | k) != 0);
            umma_commit_pair_w(&empty[stage]);
            if (++stage == STAGES) { stage = 0; phase ^= 1; }
          }
          umma_commit_pair_w(&tfull[acc]);
          CG_TRACE(4, ti);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
        if constexpr (PAIR) {
          // leader: wait for both CTAs' halo and weight halves, M=256 MMAs
          const uint32_t idesc2 = (1u << 4) | (1u << 7) | (1u << 10) |
                                  ((uint32_t)(BN >> 3) << 17) | ((uint32_t)(256 >> 4) << 24);
          const uint32_t sA_u = su32(sA), sB_u = su32(sB);
          for (int cb = 0; cb < kpt; cb++) {
            mbar_wait(&hfull[hs], hphase);
            tc_fence_after();
            const uint32_t hbase = sA_u + (uint32_t)(hs * kHaloB + a.halo_lo * 128);
#pragma unroll
            for (int tap = 0; tap < 9; tap++) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint64_t ad = smem_desc_sw128_row(hbase + (uint32_t)(a.tap_off[tap] * 128), 0);
              const uint64_t bd = smem_desc_sw128_row(sB_u + (uint32_t)(stage * B_BYTES), 0);
#pragma unroll
              for (int k = 0; k < BK / 16; k++)
                umma_bf16_pair_w(d, ad + 2 * k, bd + 2 * k, idesc2, (cb | tap | k) != 0);
              umma_commit_pair_w(&empty[stage]);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            umma_commit_pair_w(&hempty[hs]);
            if (++hs == HALO) { hs = 0; hphase ^= 1; }
          }
          umma_commit_pair_w(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
        if constexpr (HALO > 0) {
          const uint32_t sA_u = su32(sA), sB_u = su32(sB);
          for (int cb = 0; cb < kpt; cb++) {
            mbar_wait(&hfull[hs], hphase);
            tc_fence_after();
            const uint32_t hbase = sA_u + (uint32_t)(hs * kHaloB + a.halo_lo * 128);
#pragma unroll
            for (int tap = 0; tap < 9; tap++) {
              mbar_wait(&full[stage], phase);
              tc_fence_after();
              const uint64_t ad = smem_desc_sw128_row(hbase + (uint32_t)(a.tap_off[tap] * 128), 0);
              const uint64_t bd = smem_desc_sw128_row(sB_u + (uint32_t)(stage * B_BYTES), 0);
              umma_bf16_x4_w<2>(d, ad, bd, idesc, (cb | tap) != 0);
              umma_commit_w(&empty[stage]);
              if (++stage == STAGES) { stage = 0; phase ^= 1; }
            }
            umma_commit_w(&hempty[hs]);
            if (++hs == HALO) { hs = 0; hphase ^= 1; }
          }
          umma_commit_w(&tfull[acc]);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
        const uint64_t ad0 = smem_desc_sw128(sA), bd0 = smem_desc_sw128(sB);
        uint32_t a2_off = 0;  // strided second segment: the tile's row in its first box
        if constexpr (A2S) {
          int r_, m0_, n0_;
          coords(sched.t, r_, m0_, n0_);
          a2_off = (uint32_t)(m0_ % a.a2_wo) * (128 >> 4);
        }
        for (int kb = 0; kb < num_k; kb++) {
          mbar_wait(&full[stage], phase);
          if (kb == 0) CG_TRACE(3, ti);
          tc_fence_after();
          // stage offsets added to the 14-bit start-address field (uniform adds)
          const uint64_t ad = ad0 + (uint64_t)((stage * kASlot) >> 4) +
                              (A2S && kb >= num_k1 ? a2_off : 0u);
          const uint64_t bd = bd0 + (uint64_t)((stage * B_BYTES) >> 4);
          umma_bf16_x4_w<2>(d, ad, bd, idesc, kb != 0);  // 4 x UMMA_K = 16
          umma_commit_w(&empty[stage]);
          if (++stage == STAGES) { stage = 0; phase ^= 1; }
        }
        umma_commit_w(&tfull[acc]);
        CG_TRACE(4, ti);
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
      }
    }
  } else if (warp == 10) {
    // ---------------- residual loader: streams [128 x 32] residual chunks
    // through the ring in epilogue order, as far ahead as the slots allow.
    if (res_tma && lane == 0) {
      int g = 0;
      for (bool ok = sched.first(first_unit, false); ok; ok = sched.next(false, true)) {
        int r, m0, n0;
        coords(sched.t, r, m0, n0);
        for (int c = 0; c < BN / kResCols; c++, g++) {
          const int slot = g % kRS;
          if (g >= kRS) mbar_wait(&rempty[slot], ((g / kRS) - 1) & 1);
          mbar_expect_tx(&rfull[slot], kResBox);
          tma_load_2d(&gp.R[r], &rfull[slot], s_res + slot * kResBox, n0 + c * kResCols, m0);
        }
      }
    }
  } else {  // ------------------------------ epilogue (warps 2..9)
    // Warp w owns TMEM lanes [32q, 32q+32), q = w % 4 (= tile rows), and the
    // 32-column chunks c with c % 2 == h, h = (w - 2) / 4. Two paths:
    //  * identity rows, bf16 out (tma_out): thread = row, see below;
    //  * remapped rows / f32 out: (1) lane = row: tcgen05.ld -> a private
    //    32x36 fp32 smem tile; (2) lane = (row group, 8-column group): bias,
    //    ReLU, pack, 16-byte stores covering 8 rows x 64 B per instruction.
    const int q = warp & 3, h = (warp - 2) >> 2;
    const uint32_t stg_a = su32(s_epi + (warp - 2) * kStgWarp);
    const int rr8 = lane >> 2, cg8 = lane & 3;
    constexpr int CPT = BN / 32;  // 32-column chunks per tile
    // BN = 64 (2 chunks): the two warp groups take alternate tiles whole
    // (both TMEM accumulators drained concurrently) instead of one chunk
    // each of the same tile; wider tiles split chunks between the groups.
    // s2d stem (256-row tiles): group h drains sub-tile h, both chunks.
    constexpr int C0S = (kTileSplit || S2D) ? 1 : 2;  // chunk stride of one warp
    RowRemap rowmap;
    rowmap.init(a);
    int tile_i = 0, acc = 0;
    int stage_seq = 0;  // staging buffer sequence across all of this warp's chunks
    uint32_t acc_phase = 0;
    for (bool ok = sched.first(first_unit, false); ok;
         ok = sched.next(false, lane == 0), tile_i++) {
      const int t = sched.t;
      if (kTileSplit && (tile_i & 1) != h) {
        // the other group drains (and releases) this accumulator. Arriving
        // here as well would let this group, running ahead on its own odd
        // tiles, complete the NEXT phase of tempty[acc] while the other
        // group still reads the accumulator.
        if (++acc == 2) { acc = 0; acc_phase ^= 1; }
        continue;
      }
      const int c_first = (kTileSplit || S2D) ? 0 : h;
      int r_, m0, n0;
      coords(t, r_, m0, n0);
      if (S2D) m0 += h * BM;  // this group's sub-tile
      const float* bias_r = gp.bias[r_];
      const __nv_bfloat16* res_r = gp.residual[r_];
      void* out_r = gp.out[r_];
      const int my_orow =
          rowmap.map(m0 + q * 32 + lane);

      mbar_wait_sleep(&tfull[acc], acc_phase);
      if (warp == 2) CG_TRACE(5, tile_i);
      tc_fence_after();
      // TMEM reads are software-pipelined: chunk c+2's tcgen05.ld is in flight
      // while chunk c is biased, stored and written out.
      const uint32_t trow =
          tmem + ((uint32_t)(q * 32) << 16) + acc * BN * kSubTiles + (S2D ? h * BN : 0);
      uint32_t v[32];
      // 64-column blocks drained whole by one warp (the staging-free halo
      // variants never take these paths): both 32-column TMEM loads of a
      // block in flight together, one 32 x 128 B staging buffer (rows
      // XOR-swizzled in 16-byte units, the TMA 128B pattern).
      //  * identity rows, 64-wide tiles: one fence and ONE bulk store;
      //  * remapped rows (any width; group h takes blocks h, h + 2, ...):
      //    read back 4 rows x 128 B per instruction (8 lanes a row), so each
      //    16-byte store instruction writes 4 whole 128-byte row segments
      //    instead of 32 rows' 16-byte pieces.
      constexpr bool kWhole = C0S == 1 && CPT == 2;
      if constexpr (kBlockPath) {
        static_assert((kStgWarp * 4) % 1024 == 0, "block path: 1024-aligned staging");
        static_assert(kResSlots == 0 || kResCols == 64, "block path: 64-column residual boxes");
        const bool remap_fast = !tma_out && kDirectRemap && !a.out_f32 && !res_r;
        if ((tma_out && (res_tma || !res_r)) || remap_fast) {
          constexpr int kBlk = BN / 64, kBStep = kWhole ? 1 : 2;
#pragma unroll 1
          for (int b = kWhole ? 0 : h; b < kBlk; b += kBStep) {
            const uint32_t tb = trow + (uint32_t)(b * 64);
            const int nb = n0 + b * 64;
            uint32_t w[32];
            tmem_ld32_issue(tb, v);
            tmem_ld32_issue(tb + 32, w);
            tmem_ld_wait(v);
            tmem_ld_wait(w);
            if (S2D && warp == 2) CG_TRACE(1, tile_i);  // dbg: TMEM loads landed
            if (b + kBStep >= kBlk) {  // this warp's last block: hand TMEM back early
              tc_fence_before();
              __syncwarp();
              if (lane == 0) mbar_arrive(&tempty[acc]);
            }
            // residual: box gq of this CTA's ring is block b of this tile
            // (128 rows x 64 columns, 128B swizzle); this warp's 32 rows
            uint32_t rbase = 0;
            int rslot = 0;
            if (res_tma) {
              const int gq = tile_i * kBlk + b;
              rslot = gq % kRS;
              mbar_wait(&rfull[rslot], (gq / kRS) & 1);
              rbase = su32(s_res + rslot * kResBox) + (uint32_t)((q * 32 + lane) * 128);
            }
            uint32_t o[32];
            float x[32];
#pragma unroll
            for (int j = 0; j < 8; j++) {
              const float4 b4 = nb < a.N
                                    ? __ldg(reinterpret_cast<const float4*>(bias_r + nb) + j)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
              x[4 * j] = __uint_as_float(v[4 * j]) + b4.x;
              x[4 * j + 1] = __uint_as_float(v[4 * j + 1]) + b4.y;
              x[4 * j + 2] = __uint_as_float(v[4 * j + 2]) + b4.z;
              x[4 * j + 3] = __uint_as_float(v[4 * j + 3]) + b4.w;
            }
            if (res_tma) add_res_row<0>(x, rbase, lane);
            act_pack<16>(x, o, a.relu);
#pragma unroll
            for (int j = 0; j < 8; j++) {
              const float4 b4 = nb + 32 < a.N
                                    ? __ldg(reinterpret_cast<const float4*>(bias_r + nb + 32) + j)
                                    : make_float4(0.f, 0.f, 0.f, 0.f);
              x[4 * j] = __uint_as_float(w[4 * j]) + b4.x;
              x[4 * j + 1] = __uint_as_float(w[4 * j + 1]) + b4.y;
              x[4 * j + 2] = __uint_as_float(w[4 * j + 2]) + b4.z;
              x[4 * j + 3] = __uint_as_float(w[4 * j + 3]) + b4.w;
            }
            if (res_tma) {
              add_res_row<4>(x, rbase, lane);
              __syncwarp();
              if (lane == 0) mbar_arrive(&rempty[rslot]);
            }
            act_pack<16>(x, o + 16, a.relu);
            if (!remap_fast && lane == 0) bulk_wait_read<0>();  // last store read its buffer
            __syncwarp();
#pragma unroll
            for (int j = 0; j < 8; j++)
              sts_v4(stg_a + (uint32_t)(lane * 128 + ((j ^ (lane & 7)) << 4)), o[4 * j],
                     o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
            if (remap_fast) {
              __syncwarp();
              const int ch = lane & 7, n = nb + ch * 8;
#pragma unroll
              for (int it = 0; it < 8; it++) {
                const int row = it * 4 + (lane >> 3);
                const uint4 val =
                    lds_u4(stg_a + (uint32_t)(row * 128 + ((ch ^ (row & 7)) << 4)));
                const int orow = __shfl_sync(0xffffffffu, my_orow, row);
                if (orow >= 0 && n < a.N)
                  stg_u4(reinterpret_cast<__nv_bfloat16*>(out_r) + (size_t)orow * a.ld_out + n,
                         val);
              }
              __syncwarp();  // staging read back before the next block rewrites it
            } else {
              fence_async_smem();
              __syncwarp();
              if (lane == 0) {
                tma_store_2d(&gp.O64[r_], stg_a, nb, m0 + q * 32);
                bulk_commit();
              }
            }
          }
          if (warp == 2) CG_TRACE(6, tile_i);
          if (warp == 9) CG_TRACE(7, tile_i);
          CG_TRACE(8 + warp - 2, tile_i);
          if (++acc == 2) { acc = 0; acc_phase ^= 1; }
          continue;
        }
      }
      if (c_first < CPT) tmem_ld32_issue(trow + c_first * 32, v);
#pragma unroll 1
      for (int c = c_first; c < CPT; c += C0S) {
        const int g = tile_i * CPT + c;
        tmem_ld_wait(v);
        if (S2D && warp == 2 && c == c_first) CG_TRACE(1, tile_i);  // dbg: first TMEM load landed
        if (c + C0S >= CPT) {  // this warp's last chunk: hand TMEM back early
          tc_fence_before();
          __syncwarp();
          if (lane == 0) {
            if (PAIR && crank == 1) mbar_arrive_cluster(mapa_cluster(&tempty[acc], 0));
            else mbar_arrive(&tempty[acc]);
          }
        }
        if (tma_out) {
          // thread = row: bias (+ residual row from the 64B-swizzled ring) +
          // ReLU + bf16 in registers, 4 swizzled 16-byte smem stores, one TMA
          // bulk store of the warp's 32 x 32 box. Two staging buffers per
          // warp; the older bulk store must have finished reading its buffer.
          const int n = n0 + c * 32;
          float x[32];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const float4 b4 = __ldg(reinterpret_cast<const float4*>(bias_r + n) + j);
            x[4 * j] = __uint_as_float(v[4 * j]) + b4.x;
            x[4 * j + 1] = __uint_as_float(v[4 * j + 1]) + b4.y;
            x[4 * j + 2] = __uint_as_float(v[4 * j + 2]) + b4.z;
            x[4 * j + 3] = __uint_as_float(v[4 * j + 3]) + b4.w;
          }
          if (c + C0S < CPT) tmem_ld32_issue(trow + (c + C0S) * 32, v);
          if (res_tma) {
            // box gq of this CTA's residual stream holds chunk c's columns
            const int gq = tile_i * (BN / kResCols) + c / (kResCols / 32);
            const int slot = gq % kRS;
            mbar_wait(&rfull[slot], (gq / kRS) & 1);
            const uint32_t rb = su32(s_res + slot * kResBox + q * 32 * kResCols * 2);
#pragma unroll
            for (int j = 0; j < 4; j++) {
              const uint4 rv =
                  lds_u4(rb + (kResCols == 64 ? (uint32_t)(lane * 128 +
                                                           16 * ((((c & 1) * 4) + j) ^ (lane & 7)))
                                              : sw64(lane, j)));
              const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
              for (int e = 0; e < 4; e++) {
                x[8 * j + 2 * e] += __uint_as_float(w[e] << 16);
                x[8 * j + 2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
              }
            }
            __syncwarp();
            if (lane == 0) mbar_arrive(&rempty[slot]);
          }
          uint32_t o[16];
          act_pack<16>(x, o, a.relu);  // ReLU / ReLU6 + bf16 pack
          const int buf = stage_seq++ & 1;  // this warp's chunks alternate buffers
          const uint32_t sb = stg_a + buf * 2048;
          if (lane == 0) bulk_wait_read<1>();
          __syncwarp();
#pragma unroll
          for (int j = 0; j < 4; j++)
            sts_v4(sb + sw64(lane, j), o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]);
          fence_async_smem();
          __syncwarp();
          if (lane == 0) {
            tma_store_2d(&gp.O[r_], sb, n, m0 + q * 32);
            bulk_commit();
          }
          continue;
        }
        if (kDirectRemap && !a.out_f32 && !res_r) {
          // remapped rows, bf16 out, no residual (the 3x3 / 1x1 grid layers):
          // thread = row; bias + activation + pack in registers, then the
          // row's 64 bytes go straight to its remapped output row
          const int n = n0 + c * 32;
          float x[32];
#pragma unroll
          for (int j = 0; j < 8; j++) {
            const float4 b4 = n + 4 * j < a.N
                                  ? __ldg(reinterpret_cast<const float4*>(bias_r + n) + j)
                                  : make_float4(0.f, 0.f, 0.f, 0.f);
            x[4 * j] = __uint_as_float(v[4 * j]) + b4.x;
            x[4 * j + 1] = __uint_as_float(v[4 * j + 1]) + b4.y;
            x[4 * j + 2] = __uint_as_float(v[4 * j + 2]) + b4.z;
            x[4 * j + 3] = __uint_as_float(v[4 * j + 3]) + b4.w;
          }
          if (c + C0S < CPT) tmem_ld32_issue(trow + (c + C0S) * 32, v);
          uint32_t o[16];
          act_pack<16>(x, o, a.relu);  // ReLU / ReLU6 + bf16 pack
          if (my_orow >= 0 && n < a.N) {
            __nv_bfloat16* dst = reinterpret_cast<__nv_bfloat16*>(out_r) +
                                 (size_t)my_orow * a.ld_out + n;
#pragma unroll
            for (int j = 0; j < 4; j++)
              stg_u4(dst + 8 * j, make_uint4(o[4 * j], o[4 * j + 1], o[4 * j + 2], o[4 * j + 3]));
          }
          continue;
        }
#pragma unroll
        for (int j = 0; j < 8; j++)
          sts_v4(stg_a + 4 * (lane * kStgLd + 4 * j), v[4 * j], v[4 * j + 1], v[4 * j + 2],
                 v[4 * j + 3]);
        __syncwarp();
        if (c + C0S < CPT) tmem_ld32_issue(trow + (c + C0S) * 32, v);
        // phase 2: lane = (row rr8 of 8, 8-column group cg8 of 4): 16-byte
        // stores, each warp store instruction covers 8 rows x 64 B.
        const int n = n0 + c * 32 + cg8 * 8;
        const bool col_ok = n < a.N;
        float b8[8];
        if (col_ok) {
          const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias_r + n));
          const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias_r + n + 4));
          b8[0] = b0.x; b8[1] = b0.y; b8[2] = b0.z; b8[3] = b0.w;
          b8[4] = b1.x; b8[5] = b1.y; b8[6] = b1.z; b8[7] = b1.w;
        } else {
#pragma unroll
          for (int e = 0; e < 8; e++) b8[e] = 0.f;
        }
#pragma unroll 2
        for (int it = 0; it < 4; it++) {
          const int r = it * 8 + rr8;
          const int orow = __shfl_sync(0xffffffffu, my_orow, r);
          const bool ok = orow >= 0 && col_ok;
          const float4 p0 = lds_f4(stg_a + 4 * (r * kStgLd + cg8 * 8));
          const float4 p1 = lds_f4(stg_a + 4 * (r * kStgLd + cg8 * 8 + 4));
          float x[8] = {p0.x + b8[0], p0.y + b8[1], p0.z + b8[2], p0.w + b8[3],
                        p1.x + b8[4], p1.y + b8[5], p1.z + b8[6], p1.w + b8[7]};
          if (res_r) {
            uint4 rv = make_uint4(0, 0, 0, 0);
            if (ok) rv = __ldg(reinterpret_cast<const uint4*>(res_r + (size_t)orow * a.ld_res + n));
            const uint32_t w[4] = {rv.x, rv.y, rv.z, rv.w};
#pragma unroll
            for (int e = 0; e < 4; e++) {
              x[2 * e] += __uint_as_float(w[e] << 16);
              x[2 * e + 1] += __uint_as_float(w[e] & 0xffff0000u);
            }
          }
          if (a.relu) {
            const float hi = a.relu == 2 ? 6.f : INFINITY;
#pragma unroll
            for (int e = 0; e < 8; e++) x[e] = fminf(fmaxf(x[e], 0.f), hi);
          }
          if (ok) {
            if (a.out_f32) {
              float* op = reinterpret_cast<float*>(out_r) + (size_t)orow * a.ld_out + n;
              stg_f4(op, make_float4(x[0], x[1], x[2], x[3]));
              stg_f4(op + 4, make_float4(x[4], x[5], x[6], x[7]));
            } else {
              uint32_t o[4];
#pragma unroll
              for (int e = 0; e < 4; e++) {
                __nv_bfloat162 t = __floats2bfloat162_rn(x[2 * e], x[2 * e + 1]);
                o[e] = *reinterpret_cast<uint32_t*>(&t);
              }
              stg_u4(reinterpret_cast<__nv_bfloat16*>(out_r) + (size_t)orow * a.ld_out + n,
                     make_uint4(o[0], o[1], o[2], o[3]));
            }
          }
        }
        __syncwarp();
      }
      if (warp == 2) CG_TRACE(6, tile_i);
      if (warp == 9) CG_TRACE(7, tile_i);
      CG_TRACE(8 + warp - 2, tile_i);  // every epilogue warp's end (trace buffers: 16 x 64)
      if (++acc == 2) { acc = 0; acc_phase ^= 1; }
    }
    if (tma_out && lane == 0) bulk_wait_all();  // this warp's stores read their staging
  }
  tc_fence_before();
  if (PAIR) cluster_sync_all();  // both CTAs done with the pair's TMEM
  else __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    if constexpr (PAIR)
      asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem),
                   "r"(TMEM_COLS)
                   : "memory");
    else
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

template <int BN, int STAGES, int kResSlots, int HALO, int RESB, int PAIR = 0, int S2D = 0,
          int A2S = 0, int HROWS = 256>
constexpr int smem_bytes() {
  return 1024 +
         (HALO > 0 ? HALO * (S2D ? kS2DSlot : HROWS * BK * 2)
                   : STAGES * (A2S ? 4 * 56 * 128 : A_BYTES)) +
         (RESB > STAGES ? RESB : STAGES) * (PAIR ? BN / 2 : BN) * BK * 2 +
         kResSlots * 8192 +
         kEpiWarps * 4 * stg_floats<BN, STAGES, kResSlots, HALO, RESB, PAIR, HROWS>() +
         8 * (2 * STAGES + 4 + 2 * (kResSlots > 0 ? kResSlots : 1) + 2 * (HALO > 0 ? HALO : 1)) +
         16 + 48 + 16 + 32 * kClcSlots;
}

// env CREDO_NO_PDL: plain stream serialisation between GEMM launches (A/B)
const int g_pdl = std::getenv("CREDO_NO_PDL") == nullptr ? 1 : 0;
// env CREDO_NO_CLC: static persistent grids (A/B); CREDO_CLC_UNIT_NS: target
// work per scheduling unit
const bool g_clc = std::getenv("CREDO_NO_CLC") == nullptr;
// env CREDO_NO_STG4=1: 3 stages for every streamed 256-wide GEMM (A/B)
const bool g_stg4 = std::getenv("CREDO_NO_STG4") == nullptr;
// env CREDO_HALO_STAGED=1: remapped halo convs keep epilogue staging (the
// staged 128-byte-row store path) instead of a deeper halo ring (A/B)
const bool g_halo_deep = std::getenv("CREDO_HALO_STAGED") == nullptr;
const double g_unit_ns = std::getenv("CREDO_CLC_UNIT_NS") ? std::atof(std::getenv("CREDO_CLC_UNIT_NS"))
                                                          : 1500.0;

// Tiles per CLC unit: enough work per unit (~g_unit_ns at ~8 TFLOP/s per SM)
// to hide one cancel round trip, while leaving >= 3 units per SM so CTAs that
// start late (SMs freed by other kernels) still balance the load.
int tiles_per_unit(const ConvGemmArgs& a, int BN, int tiles) {
  const double tile_flops = 2.0 * BM * BN * ((double)a.Kc * a.ntaps + a.kc2);
  const double tile_ns = tile_flops / 8.0e3;  // 8 TFLOP/s per SM = 8e3 FLOP/ns
  int T = (int)std::ceil(g_unit_ns / std::max(tile_ns, 1.0));
  T = std::min(T, std::max(1, tiles / (3 * kNumSMs)));
  return std::max(T, 1);
}

template <int BN, int STAGES, int RS, int HALO = 0, int RESB = 0, int PAIR = 0, int S2D = 0,
          int A2S = 0, int HROWS = 256>
void launch_t(const PreparedGemm& p, cudaStream_t st, int max_ctas) {
  constexpr int smem = smem_bytes<BN, STAGES, RS, HALO, RESB, PAIR, S2D, A2S, HROWS>();
  static_assert(smem <= 232448, "smem budget");
  static std::atomic<uint64_t> attr{0};
  once_per_device(attr, [] {
    CG_CUDA(cudaFuncSetAttribute(conv_gemm_kernel<BN, STAGES, RS, HALO, RESB, PAIR, S2D, A2S, HROWS>,
                                 cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
  });
  ConvGemmArgs a = p.args;
  constexpr int kTileRows = S2D ? 2 * BM : BM;  // the s2d stem's 256-row tiles
  const int tiles = ((a.M + kTileRows - 1) / kTileRows) * ((a.N + BN - 1) / BN) * p.gp.n;
  int grid;
  if (!PAIR && g_clc && max_ctas <= 0) {
    a.sched = 1;
    a.tile_unit = tiles_per_unit(a, BN, tiles);
    grid = (tiles + a.tile_unit - 1) / a.tile_unit;
  } else {
    a.sched = 0;
    a.tile_unit = 1;
    grid = std::min(tiles, max_ctas > 0 ? max_ctas : kNumSMs);
  }
  timer_begin(st, kTimeGemm);
  if constexpr (PAIR) {
    // SM pairs (static scheduler): a cluster of 2 CTAs per 256-row tile
    const int pair_tiles = ((a.M + 2 * BM - 1) / (2 * BM)) * ((a.N + BN - 1) / BN) * p.gp.n;
    int g2 = std::min(2 * pair_tiles, kNumSMs);
    if (max_ctas > 0) g2 = std::min(g2, max_ctas - (max_ctas & 1));
    if (g2 < 2) throw InvalidArgument("conv_gemm: an SM pair needs 2 CTAs");
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)g2);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute attr2[2];
    attr2[0].id = cudaLaunchAttributeClusterDimension;
    attr2[0].val.clusterDim.x = 2;
    attr2[0].val.clusterDim.y = 1;
    attr2[0].val.clusterDim.z = 1;
    attr2[1].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr2[1].val.programmaticStreamSerializationAllowed = g_pdl;
    cfg.attrs = attr2;
    cfg.numAttrs = 2;
    CG_CUDA(cudaLaunchKernelEx(&cfg, conv_gemm_kernel<BN, STAGES, RS, HALO, RESB, PAIR>, p.gp, a));
    launch_counter_add(1);
  } else {
    // programmatic dependent launch (the kernel waits on griddepcontrol)
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3((unsigned)grid);
    cfg.blockDim = dim3(kThreads);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = st;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    at[0].val.programmaticStreamSerializationAllowed = g_pdl;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    CG_CUDA(cudaLaunchKernelEx(&cfg, conv_gemm_kernel<BN, STAGES, RS, HALO, RESB, PAIR, S2D, A2S, HROWS>,
                               p.gp, a));
    launch_counter_add(1);
  }
  timer_end(st, kTimeGemm);
}

}  // namespace

// ---------------------------------------------------- MMA rate microbench
// One elected thread per CTA issues `iters` x 4 back-to-back kind::f16 MMAs
// (M=128, N, K=16, both operands in shared memory) into one or two TMEM
// accumulators; cycles per MMA = the issue/dispatch rate the conv kernels
// can reach at best for that N (tools/mma_rate.py).
template <int N>
__global__ void __launch_bounds__(128, 1) mma_rate_kernel(int iters, int two_acc,
                                                          long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  // two_acc 3 / 4: rotate over nbuf distinct A and B tiles (1 / 2 accumulators)
  const int nbuf = two_acc >= 3 ? (N == 64 ? 8 : 4) : 1;
  uint8_t* sA = smem;
  uint8_t* sB = smem + nbuf * A_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + nbuf * N * BK * 2);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tslot)), "r"(512) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  __syncthreads();
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (warp == 1 && lane == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(BM >> 4) << 24);
    const uint64_t ad = smem_desc_sw128(sA), bd = smem_desc_sw128(sB);
    long long t0 = clock64();
    if (two_acc == 5) {
      // the s2d stem's pattern: SW32 K = 16 rows, A at 4 row shifts (+32 B),
      // 16 B tap tiles of 64 x 32 B, one accumulator
      const uint64_t a32 = smem_desc_sw32_row(su32(sA)), b32 = smem_desc_sw32_row(su32(sB));
      for (int i = 0; i < iters; i++)
#pragma unroll
        for (int k = 0; k < 4; k++)
          umma_bf16(tmem, a32 + 2 * k + 2 * 4 * (i & 1), b32 + 128 * (4 * (i & 3) + k), idesc,
                    (i | k) != 0);
      iters *= 1;  // 4 MMAs per iteration, as the other modes
    } else
    for (int i = 0; i < iters; i++) {
      const bool alt = (two_acc == 1 || two_acc == 4) && (i & 1);
      const uint32_t d = tmem + (alt ? 256u : 0u);
      const int bi = (i >> (two_acc == 4 ? 1 : 0)) % nbuf;
      const uint64_t a_i = ad + (uint64_t)((bi * A_BYTES) >> 4);
      const uint64_t b_i = bd + (uint64_t)((bi * N * BK * 2) >> 4);
#pragma unroll
      for (int k = 0; k < 4; k++) umma_bf16(d, a_i + 2 * k, b_i + 2 * k, idesc, (i | k) != 0);
    }
    umma_commit(bar);
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  tc_fence_before();
  __syncthreads();
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(512)
                 : "memory");
  }
}

// The same on an SM pair: cluster of 2 CTAs, TMEM allocated with
// cta_group::2, the leader issues M = 256 MMAs over both CTAs' operands and
// commits to both CTAs' barriers.
template <int N>
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(128, 1)
    mma_rate_pair_kernel(int iters, long long* cycles) {
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024 - (su32(smem_raw) & 1023)) & 1023);
  uint8_t* sA = smem;
  uint8_t* sB = smem + A_BYTES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(sB + (N / 2) * BK * 2);
  uint32_t* tslot = reinterpret_cast<uint32_t*>(bar + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  uint32_t rank;
  asm volatile("mov.u32 %0, %%cluster_ctarank;" : "=r"(rank));
  if (threadIdx.x == 0) {
    mbar_init(bar, 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  }
  if (warp == 1) {
    asm volatile("tcgen05.alloc.cta_group::2.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(
                     su32(tslot)), "r"(256) : "memory");
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::2.sync.aligned;" ::: "memory");
  }
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
  tc_fence_after();
  const uint32_t tmem = *tslot;
  if (rank == 0 && warp == 1 && lane == 0) {
    const uint32_t idesc = (1u << 4) | (1u << 7) | (1u << 10) | ((uint32_t)(N >> 3) << 17) |
                           ((uint32_t)(256 >> 4) << 24);
    const uint64_t ad = smem_desc_sw128(sA), bd = smem_desc_sw128(sB);
    long long t0 = clock64();
    for (int i = 0; i < iters; i++) {
#pragma unroll
      for (int k = 0; k < 4; k++) {
        asm volatile(
            "{\n\t.reg .pred p;\n\tsetp.ne.b32 p, %4, 0;\n\t"
            "tcgen05.mma.cta_group::2.kind::f16 [%0], %1, %2, %3, p;\n}" ::"r"(tmem),
            "l"(ad + 2 * k), "l"(bd + 2 * k), "r"(idesc), "r"((uint32_t)((i | k) != 0)));
      }
    }
    asm volatile(
        "tcgen05.commit.cta_group::2.mbarrier::arrive::one.shared::cluster.multicast::cluster.b64"
        " [%0], %1;" ::"r"(su32(bar)), "h"((uint16_t)3) : "memory");
    mbar_wait(bar, 0);
    long long t1 = clock64();
    if (blockIdx.x == 0) *cycles = t1 - t0;
  }
  if (rank == 1 && warp == 1 && lane == 0) mbar_wait(bar, 0);
  tc_fence_before();
  asm volatile("barrier.cluster.arrive.release.aligned;\n\tbarrier.cluster.wait.acquire.aligned;"
               ::: "memory");
  if (warp == 1) {
    tc_fence_after();
    asm volatile("tcgen05.dealloc.cta_group::2.sync.aligned.b32 %0, %1;" ::"r"(tmem), "r"(256)
                 : "memory");
  }
}

double mma_rate_pair_bench(int N, int iters, int ctas, cudaStream_t st) {
  long long* d = nullptr;
  CG_CUDA(cudaMalloc(&d, 8));
  const int smem = 1024 + A_BYTES + (N / 2) * BK * 2 + 64;
  auto run = [&](auto kern) {
    CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<ctas, 128, smem, st>>>(iters, d);
    CG_CHECK_LAUNCH();
  };
  if (N == 64) run(mma_rate_pair_kernel<64>);
  else if (N == 128) run(mma_rate_pair_kernel<128>);
  else run(mma_rate_pair_kernel<256>);
  long long c = 0;
  CG_CUDA(cudaMemcpyAsync(&c, d, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d);
  return (double)c / (4.0 * iters);
}

double mma_rate_bench(int N, int iters, int ctas, int two_acc, cudaStream_t st) {
  if (two_acc == 2) return mma_rate_pair_bench(N, iters, ctas, st);
  long long* d = nullptr;
  CG_CUDA(cudaMalloc(&d, 8));
  const int nbuf = two_acc >= 3 ? (N == 64 ? 8 : 4) : 1;
  if (two_acc == 5 && N != 64) throw InvalidArgument("mma_rate: the s2d pattern is N = 64");
  if (N == 256 && nbuf > 1) throw InvalidArgument("mma_rate: rotating buffers for N <= 128");
  const int smem = 1024 + nbuf * (A_BYTES + N * BK * 2) + 64;
  auto run = [&](auto kern) {
    CG_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, smem));
    kern<<<ctas, 128, smem, st>>>(iters, two_acc, d);
    CG_CHECK_LAUNCH();
  };
  if (N == 64) run(mma_rate_kernel<64>);
  else if (N == 128) run(mma_rate_kernel<128>);
  else run(mma_rate_kernel<256>);
  long long c = 0;
  CG_CUDA(cudaMemcpyAsync(&c, d, 8, cudaMemcpyDeviceToHost, st));
  CG_CUDA(cudaStreamSynchronize(st));
  cudaFree(d);
  return (double)c / (4.0 * iters);
}


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

void make_operand_s2_view(Operand& op, const void* x, int B, int H, int C, int rpb) {
  if (reinterpret_cast<uintptr_t>(x) % 16 || C % 64 || H % 2)
    throw InvalidArgument("strided view: misaligned or odd shape");
  const int Wo = H / 2;
  cuuint64_t dims[3] = {(cuuint64_t)C, (cuuint64_t)Wo, (cuuint64_t)B * Wo};
  cuuint64_t strides[2] = {(cuuint64_t)2 * C * 2, (cuuint64_t)2 * H * C * 2};
  cuuint32_t box[3] = {64, (cuuint32_t)Wo, (cuuint32_t)rpb};
  cuuint32_t estr[3] = {1, 1, 1};
  CUresult r = get_encode()(&op.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 3, const_cast<void*>(x),
                            dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("strided view tensor map failed: " + std::to_string((int)r));
  op.ptr = x;
  op.rows = B * Wo * Wo;
  op.cols = C;
  op.box_rows = Wo * rpb;
}

// [rows, 16] bf16 (32-byte rows) with the 32B swizzle: the s2d stem's
// image (box_rows-row boxes) and weights (256-row boxes).
static void make_operand_k16(Operand& op, const void* ptr, int rows, int box_rows) {
  if (reinterpret_cast<uintptr_t>(ptr) % 16) throw InvalidArgument("operand misaligned");
  cuuint64_t dims[2] = {16, (cuuint64_t)rows};
  cuuint64_t strides[1] = {32};
  cuuint32_t box[2] = {16, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&op.map, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2,
                            const_cast<void*>(ptr), dims, strides, box, estr,
                            CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_32B,
                            CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("s2d tensor map failed: " + std::to_string((int)r));
  op.ptr = ptr;
  op.rows = rows;
  op.cols = 16;
  op.box_rows = box_rows;
}
void make_operand_s2d_a(Operand& op, const void* ptr, int rows, int box_rows) {
  make_operand_k16(op, ptr, rows, box_rows);
}
void make_operand_s2d_b(Operand& op, const void* ptr, int rows) {
  make_operand_k16(op, ptr, rows, 256);
}

// [rows, ld] bf16 map with a 32-column box and the 64B swizzle (64-byte box
// rows): the residual ring (128-row box) and the output stage (32-row box).
static void map64(CUtensorMap& m, const void* p, int ld, int rows, int box_rows) {
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {32, (cuuint32_t)box_rows};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_64B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("epilogue tensor map failed");
}

// [rows, ld] bf16 map with a 64-column x 32-row box, 128B swizzle: a warp's
// whole 32 x 64 output block of a 64-wide tile in one bulk store.
static void map_out128(CUtensorMap& m, const void* p, int ld, int rows) {
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, 32};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("epilogue tensor map failed");
}

// [rows, ld] bf16 map with a 64-column x 128-row box, 128B swizzle: the
// residual ring's boxes.
static void map128_res(CUtensorMap& m, const void* p, int ld, int rows) {
  cuuint64_t dims[2] = {(cuuint64_t)ld, (cuuint64_t)rows};
  cuuint64_t strides[1] = {(cuuint64_t)ld * 2};
  cuuint32_t box[2] = {64, 128};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = get_encode()(&m, CU_TENSOR_MAP_DATA_TYPE_BFLOAT16, 2, const_cast<void*>(p), dims,
                            strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE,
                            CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) throw CudaError("residual tensor map failed");
}

void prepare_conv_gemm(PreparedGemm& p, const ConvGemmGroup& g, const ConvGemmArgs& a, int BN) {
  if (a.s2d) {
    if (a.s2d_ndy < 0 || a.s2d_ndy > 4 || (a.s2d_ndy && a.s2d_step != 1))
      throw InvalidArgument("conv_gemm: s2d_ndy is for one box per kernel row");
    if (BN != 64 || a.N != 64 || a.Kc != 16 || a.ntaps != 16 || a.halo_lo || a.pair ||
        (a.row_mode != kRowGridToCompact && a.row_mode != kRowIdentity &&
         a.row_mode != kRowGridToPad) || a.out_f32 ||
        a.gw < 4 || a.gh < 4)
      throw InvalidArgument("conv_gemm: s2d stem is 64 outputs, 16 taps of K = 16, grid rows");
    for (int r = 0; r < g.n; r++)
      if (g.A[r]->box_rows != BM + (a.s2d_step == 1 ? 0 : a.gw) + 3 || g.A[r]->box_rows > 256 ||
          g.B[r]->box_rows != 256 ||
          g.residual[r])
        throw InvalidArgument("conv_gemm: s2d stem operand mismatch");
  } else if (a.Kc % 64 || a.ntaps < 1 || a.ntaps > 9) {
    throw InvalidArgument("conv_gemm: bad K");
  }
  if (a.kc2 && (a.kc2 % 64 || a.ntaps != 1 || a.halo_lo || a.pair || a.s2d))
    throw InvalidArgument("conv_gemm: a second K segment is for 1x1 streamed GEMMs");
  if (!a.out_f32 && (a.N % 32)) throw InvalidArgument("conv_gemm: bf16 out needs N%32==0");
  if (a.out_f32 && (a.N % 8)) throw InvalidArgument("conv_gemm: f32 out needs N%8==0");
  if (g.n < 1 || g.n > kMaxGroup) throw InvalidArgument("conv_gemm: group size 1..4");
  if (BN != 64 && BN != 128 && BN != 256) throw InvalidArgument("conv_gemm: BN 64/128/256");
  const bool tma_out = a.row_mode == kRowIdentity && !a.out_f32;
  std::memset(&p.gp, 0, sizeof p.gp);
  p.gp.n = g.n;
  const int hsub = a.halo_sub > 1 ? a.halo_sub : 1;
  if (a.halo_lo < 0 || (hsub == 1 && BM + 2 * a.halo_lo > 256) ||
      (hsub > 1 && (a.pair || a.halo_box % 8 || a.halo_box > 256 ||
                    hsub * a.halo_box < BM + 2 * a.halo_lo || !wide_halo_fits(BN, a))))
    throw InvalidArgument("conv_gemm: halo too wide");
  if (a.halo_lo > 0 && a.ntaps != 9) throw InvalidArgument("conv_gemm: halo needs 9 taps");
  for (int t = 0; a.halo_lo > 0 && t < a.ntaps; t++)
    if (a.tap_off[t] < -a.halo_lo || a.tap_off[t] > a.halo_lo)
      throw InvalidArgument("conv_gemm: tap outside the halo");
  for (int r = 0; r < g.n; r++) {
    if (!a.s2d &&
        (g.A[r]->box_rows != (hsub > 1 ? a.halo_box : BM + 2 * a.halo_lo) ||
         g.B[r]->box_rows != (a.pair ? BN / 2 : BN)))
      throw InvalidArgument("conv_gemm: box mismatch");
    if ((g.residual[r] != nullptr) != (g.residual[0] != nullptr))
      throw InvalidArgument("conv_gemm: residual on some replicas only");
    p.gp.A[r] = g.A[r]->map;
    if (a.kc2) {
      if (!g.A2[r] || g.A2[r]->cols != a.kc2 ||
          g.A2[r]->box_rows != (a.a2_wo ? a.a2_wo * a.a2_rpb : BM))
        throw InvalidArgument("conv_gemm: second K segment operand mismatch");
      if (a.a2_wo && (a.a2_wo * a.a2_rpb != 56 || a.kc2 % 64))
        throw InvalidArgument("conv_gemm: strided A2 boxes are 56 rows");
      p.gp.A2[r] = g.A2[r]->map;
    }
    p.gp.B[r] = g.B[r]->map;
    p.gp.bias[r] = g.bias[r];
    p.gp.residual[r] = g.residual[r];
    p.gp.out[r] = g.out[r];
    if (tma_out) {
      if (a.ld_out % 8 || reinterpret_cast<uintptr_t>(g.out[r]) % 16)
        throw InvalidArgument("conv_gemm: output must be 16B aligned");
      // 64-wide tiles without a residual: the kernel's one-store-per-warp path
      map64(p.gp.O[r], g.out[r], a.ld_out, a.rows_out, 32);
      if (!a.pair) map_out128(p.gp.O64[r], g.out[r], a.ld_out, a.rows_out);
      if (g.residual[r]) {
        if (a.ld_res % 8 || reinterpret_cast<uintptr_t>(g.residual[r]) % 16)
          throw InvalidArgument("conv_gemm: residual must be 16B aligned");
        if (CG_RES_COLS == 64) map128_res(p.gp.R[r], g.residual[r], a.ld_res, a.rows_out);
        else map64(p.gp.R[r], g.residual[r], a.ld_res, a.rows_out, 128);
      }
    }
  }
  p.args = a;
  p.BN = BN;
  // Residual layers are 1x1 with small K: trade mainloop stages for a deep
  // residual ring so the epilogue streams at HBM rate.
  p.res = g.residual[0] != nullptr && tma_out;
}

void halo_boxes(int halo_lo, int& sub, int& box) {
  const int rows = BM + 2 * halo_lo;
  sub = (rows + 255) / 256;
  box = ((rows + sub - 1) / sub + 7) / 8 * 8;
  if (box > 256) box = 256, sub = (rows + 255) / 256 + 1;
}

bool wide_halo_fits(int BN, const ConvGemmArgs& a) {
  int sub, box;
  halo_boxes(a.halo_lo, sub, box);
  if (a.ntaps != 9 || a.pair || a.out_f32) return false;
  if (BN == 64) return a.N <= 64 && a.Kc == 64 && sub * box <= kWideHaloRows;  // resident B
  return BN == 128 && sub * box <= kWideHaloRows128;
}

void launch_prepared(const PreparedGemm& p, cudaStream_t st, int max_ctas) {
  if (p.args.a2_wo) {  // strided second segment (the stride-2 shortcut, no gather)
    if (p.BN != 256 || p.res) throw InvalidArgument("conv_gemm: strided A2 is for BN = 256");
    launch_t<256, 3, 0, 0, 0, 0, 0, 1>(p, st, max_ctas);
    return;
  }
  if (p.args.s2d) {  // 12 dy-pair boxes (6 tiles) in flight, 16 taps' weights resident
    launch_t<64, 1, 0, 12, 4, 0, 1>(p, st, max_ctas);
    return;
  }
  if (p.args.pair) {
    if (p.args.halo_lo > 0) {
      if (p.BN != 128 || p.res)
        throw InvalidArgument("conv_gemm: halo SM pairs only for 128-wide tiles");
      launch_t<128, 7, 0, 2, 0, 1>(p, st, max_ctas);
      return;
    }
    if (p.BN != 256) throw InvalidArgument("conv_gemm: SM pairs only for 256-wide tiles");
    if (p.res) launch_t<256, 3, 10, 0, 0, 1>(p, st, max_ctas);
    else launch_t<256, 5, 0, 0, 0, 1>(p, st, max_ctas);
    return;
  }
  if (p.args.halo_lo > 0) {
    if (p.res) throw InvalidArgument("conv_gemm: halo mode has no residual ring");
    if (p.args.halo_sub > 1) {
      // wide halos (stacked boxes): remapped bf16 rows, staging-free epilogue
      if (p.args.out_f32 || p.args.row_mode == kRowIdentity || !kDirectRemap)
        throw InvalidArgument("conv_gemm: wide halos write remapped bf16 rows");
      if (wide_halo_fits(p.BN, p.args)) {
        if (p.BN == 64) launch_t<64, 1, 0, 2, 9, 0, 0, 0, kWideHaloRows>(p, st, max_ctas);
        else launch_t<128, 8, 0, 2, 0, 0, 0, 0, kWideHaloRows128>(p, st, max_ctas);
        return;
      }
      throw InvalidArgument("conv_gemm: no wide-halo variant for this shape");
    }
    // small weight sets (one n block, 9 x 64-channel taps): keep B resident
    if (p.BN == 64 && p.args.N <= 64 && p.args.Kc == 64 && p.args.ntaps == 9 &&
        std::getenv("CREDO_NO_RESB") == nullptr) {
      if (!p.args.out_f32 && p.args.row_mode != kRowIdentity && kDirectRemap && g_stg4 &&
          g_halo_deep)
        launch_t<64, 1, 0, 4, 9>(p, st, max_ctas);  // no staging: a 4th halo slot
      else
        launch_t<64, 1, 0, 3, 9>(p, st, max_ctas);
      return;
    }
    // remapped bf16 rows leave the epilogue staging unused: deeper halo rings
    const bool deep_halo = !p.args.out_f32 && p.args.row_mode != kRowIdentity && kDirectRemap &&
                           g_stg4 && g_halo_deep;
    switch (p.BN) {
      case 64:
        if (deep_halo) launch_t<64, 8, 0, 4>(p, st, max_ctas);
        else launch_t<64, 8, 0, 3>(p, st, max_ctas);
        return;
      case 128:
        if (deep_halo) launch_t<128, 8, 0, 2>(p, st, max_ctas);
        else launch_t<128, 6, 0, 2>(p, st, max_ctas);
        return;
      case 256:
        if (deep_halo) launch_t<256, 4, 0, 2>(p, st, max_ctas);
        else launch_t<256, 3, 0, 2>(p, st, max_ctas);
        return;
      default: throw InvalidArgument("conv_gemm: BN must be 64, 128 or 256");
    }
  }
  // Residual layers share shared memory between mainloop stages and the
  // residual ring: short K (< 8 k-blocks per tile) is epilogue-bound and
  // wants the deep ring; long K starves a 2-stage mainloop (measured: ResNet
  // stage-4 c3, K = 512: 60 -> 46 us with 3 stages and a 2-box ring).
#ifndef CG_RES_DEEPK
#define CG_RES_DEEPK 1
#endif
  const bool deep_k = CG_RES_DEEPK && p.args.Kc * p.args.ntaps >= 8 * BK;
  switch (p.BN * 2 + (p.res ? 1 : 0)) {
    case 128:  // (p.BN * 2 + residual); bf16 out: one more stage in the freed staging
      if (!p.args.out_f32 && (p.args.row_mode == kRowIdentity || kDirectRemap) && g_stg4)
        launch_t<64, 8, 0>(p, st, max_ctas);
      else
        launch_t<64, 7, 0>(p, st, max_ctas);
      break;
    case 129:
      if (deep_k) launch_t<64, 5, 6>(p, st, max_ctas);
      else launch_t<64, 4, 10>(p, st, max_ctas);
      break;
    case 256:
      if (!p.args.out_f32 && (p.args.row_mode == kRowIdentity || kDirectRemap) && g_stg4)
        launch_t<128, 6, 0>(p, st, max_ctas);
      else
        launch_t<128, 5, 0>(p, st, max_ctas);
      break;
    case 257:
      if (deep_k) launch_t<128, 4, 6>(p, st, max_ctas);
      else launch_t<128, 3, 10>(p, st, max_ctas);
      break;
    case 512:  // bf16 out through the TMA-store or direct-store epilogue: room for 4 stages
      if (!p.args.out_f32 && (p.args.row_mode == kRowIdentity || kDirectRemap) && g_stg4)
        launch_t<256, 4, 0>(p, st, max_ctas);
      else
        launch_t<256, 3, 0>(p, st, max_ctas);
      break;
    case 513:
      if (deep_k) launch_t<256, 3, 4>(p, st, max_ctas);
      else if (p.args.row_mode == kRowIdentity && !p.args.out_f32 && g_stg4)
        launch_t<256, 2, 12>(p, st, max_ctas);  // TMA-store staging only: a deeper ring
      else launch_t<256, 2, 10>(p, st, max_ctas);
      break;
    default: throw InvalidArgument("conv_gemm: BN must be 64, 128 or 256");
  }
}

void launch_conv_gemm(const Operand& A, const Operand& B, const ConvGemmArgs& a, int BN,
                      cudaStream_t st, int max_ctas) {
  ConvGemmGroup g;
  g.n = 1;
  g.A[0] = &A;
  g.B[0] = &B;
  g.bias[0] = a.bias;
  g.residual[0] = a.residual;
  g.out[0] = a.out;
  PreparedGemm p;
  prepare_conv_gemm(p, g, a, BN);
  launch_prepared(p, st, max_ctas);
}

}  // namespace cg
