// tcgen05 implicit-GEMM convolution for sm_100a.
//
//   D[m, n] = epi( sum_t sum_kb A[m + tap_off[t], kb] * B[n, t*Kc + kb] )
//
// A: bf16 activations, NHWC rows (row = pixel, K = channels, Kc % 64 == 0).
//    A 3x3/stride-1 convolution runs over the zero-bordered ("padded") pixel
//    grid so tap t is a constant row shift; TMA zero-fills rows outside the
//    tensor. 1x1 convolutions and explicit im2col operands have one tap.
// B: bf16 weights, [N, ntaps*Kc] K-major (BN folded).
// epi: + bias[n] (+ residual) (ReLU) -> bf16 (or f32) with a row remap
//    (identity / padded-grid -> compact / compact -> padded-grid interior).
#pragma once
#include <cuda.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace cg {

enum RowMode : int {
  kRowIdentity = 0,     // out row = m
  kRowPadToCompact = 1, // m on the (H+2)x(W+2) grid; interior -> compact row
  kRowCompactToPad = 2, // m compact; written to the interior of the padded grid
  kRowPadToPad = 3,     // m on the padded grid; interior rows written in place
                        // (the zero border of the output grid is never touched)
  // Phase-split grid for stride-2 3x3 convs: the zero-bordered grid stored
  // as 4 planes (row parity a, column parity b), plane ab holding padded
  // pixels (2i+a, 2j+b), so the stride-2 3x3 becomes 9 constant row shifts
  // (plane base + p*Wq + q) instead of a gather.
  kRowCompactToPhasePad = 4,  // m compact (H x W) -> phase-split padded grid
  kRowPhaseGridToCompact = 5, // m on an (H+1) x (W+1) plane-00 grid -> compact
                              // H x W (H, W = output dims)
  kRowGridToCompact = 6,      // m on a per-image gh x gw grid -> compact H x W
                              // (rows with i >= H or j >= W are not stored)
  kRowGridToPad = 7,          // m on a per-image gh x gw grid -> the interior
                              // of the shared-border (H+1) x (W+1) grid
};

struct ConvGemmArgs {
  int M;           // GEMM rows (A row space)
  int N;           // output channels
  int Kc;          // channels per tap (multiple of 64)
  int ntaps;       // 1 or 9
  int tap_off[9];  // row shift per tap
  const float* bias;                 // [N]
  const __nv_bfloat16* residual;     // [rows_out, ld_res] or null
  int ld_res;
  void* out;                         // bf16 or f32 [rows_out, ld_out]
  int ld_out;
  int out_f32;
  int relu;        // 0 none, 1 ReLU, 2 ReLU6
  int row_mode;
  int H, W;                          // unpadded spatial dims (row remap)
  int rows_out;                      // valid output rows (identity mode)
  long long* trace;                  // debug: CTA-0 event timestamps or null
  // Halo mode (3x3 taps = row shifts within [-halo_lo, +halo_lo]): per
  // channel block ONE TMA box of BM + 2*halo_lo rows feeds all 9 taps from
  // shared memory (each tap's MMA reads it at its row offset), instead of
  // one BM-row box per tap. 0 = off. The A operand's box must then have
  // BM + 2*halo_lo (<= 256) rows.
  int halo_lo;
  // Wide halo (BM + 2*halo_lo > 256 rows, e.g. 3x3 convs at 112 / 224
  // pixels): the halo arrives as halo_sub TMA boxes of the operand's
  // box_rows rows each, stacked in one shared-memory slot. 0 / 1 = one box.
  int halo_sub, halo_box;  // halo_box: rows per box (a multiple of 8)
  int pair;  // 1: SM-pair (cta_group::2) 256-row tiles, B operand box = BN/2 rows
  // Tile scheduler, set by the launcher: 0 = static persistent stride, 1 =
  // cluster launch control (one CTA per unit of tile_unit tiles; resident
  // CTAs cancel pending ones and take their units).
  int sched;
  int tile_unit;
  // Space-to-depth stem (s2d = 1): the 7x7/2 conv1 as a 4x4 stride-1 conv
  // over the 2x2 space-to-depth image (12 channels padded to 16: 32-byte
  // rows, 32B swizzle): per tile 2 row boxes (dy pairs) of BM + gw + 3 <=
  // 256 rows, 16 taps (dy, dx) of one K = 16 MMA each at row shift
  // dy * gw + dx, the 16 taps' weights resident ([tap][N][16]).
  // Rows live on a per-image gh x gw grid (row_mode kRowGridToCompact).
  int s2d;
  int gh, gw;
  // s2d boxes: 0 / 2 = one box per dy pair (BM + gw + 3 rows <= 256), 1 = one
  // box per dy (BM + 3 rows; grids wider than 125 columns, e.g. a 3x3 conv
  // over a 16-channel 224-pixel image as a 4x4 with zero fourth taps)
  int s2d_step;
  int s2d_ndy;  // s2d_step 1: kernel rows with non-zero taps (0 = all 4)
  // Second K segment (1x1 convs only): k-blocks Kc/64 .. Kc/64 + kc2/64 - 1
  // read A from the A2 operand (same rows) against weight columns Kc ..
  // Kc + kc2 - 1 -- a bottleneck's c3 and its projection shortcut (ds) as one
  // GEMM over [t2 | x] x [W3 | Wds]^T, no shortcut tensor in HBM. 0 = off.
  int kc2;
  // Strided second segment (a2_wo > 0): the A2 operand is x[2h, 2w] read in
  // place through a 3-D tensor map (channels, w' stepping 2 pixels, output
  // rows stepping 2 input rows) in boxes of a2_rpb output rows of a2_wo
  // pixels (a2_rpb * a2_wo = 56 rows, 7 KB, 1024-aligned in the stage), the
  // MMA reading the tile's 128 rows from its offset in the first box -- the
  // stride-2 shortcut without a gather pass. 0 = A2 is a compact operand.
  int a2_wo, a2_rpb;
};

// One encoded operand (tensor map over a row-major bf16 [rows, cols] matrix
// with a 64 x box_rows box and 128B swizzle).
struct Operand {
  CUtensorMap map;
  const void* ptr = nullptr;
  int rows = 0, cols = 0, box_rows = 0;
};

void make_operand(Operand& op, const void* ptr, int rows, int cols, int box_rows);
// x[2h, 2w] of an NHWC [B, H, H, C] bf16 tensor as a 3-D map (C, H/2 w',
// B*H/2 output rows), box 64 x (H/2) x rpb, 128B swizzle (ConvGemmArgs::a2_wo)
void make_operand_s2_view(Operand& op, const void* x, int B, int H, int C, int rpb);
// s2d stem operands: A = [rows, 16] bf16 image, box 16 x box_rows; B =
// [16 * N, 16] bf16 weights in [tap][N][16] order, box 16 x 256; 32B swizzle.
void make_operand_s2d_a(Operand& op, const void* ptr, int rows, int box_rows);
void make_operand_s2d_b(Operand& op, const void* ptr, int rows);

// One launch over up to kMaxGroup replicas: the same GEMM shape on each
// replica's own activations/weights (tiles are replica-major), so small
// layers of a model group fill the GPU in one wave-balanced launch.
constexpr int kMaxGroup = 4;
struct ConvGemmGroup {
  int n = 0;
  const Operand* A[kMaxGroup];
  const Operand* A2[kMaxGroup] = {};  // second K segment (ConvGemmArgs::kc2)
  const Operand* B[kMaxGroup];
  const float* bias[kMaxGroup];
  const __nv_bfloat16* residual[kMaxGroup];
  void* out[kMaxGroup];
};

// Kernel parameters of a grouped launch (all tensor maps pre-encoded).
struct GemmGroupParams {
  CUtensorMap A[kMaxGroup], B[kMaxGroup], R[kMaxGroup], O[kMaxGroup], A2[kMaxGroup];
  CUtensorMap O64[kMaxGroup];  // output, 64-column x 32-row boxes (128B swizzle)
  const float* bias[kMaxGroup];
  const __nv_bfloat16* residual[kMaxGroup];
  void* out[kMaxGroup];
  int n;
};

struct PreparedGemm {
  GemmGroupParams gp;
  ConvGemmArgs args;
  int BN = 128;
  bool res = false;
};

// Encodes every tensor map of a (grouped) launch once; launch_prepared then
// costs one kernel launch (plans cache PreparedGemm per layer).
void prepare_conv_gemm(PreparedGemm& p, const ConvGemmGroup& g, const ConvGemmArgs& a, int BN);
void launch_prepared(const PreparedGemm& p, cudaStream_t st, int max_ctas = 0);
// Whether a wide halo (ConvGemmArgs::halo_sub > 1) has a kernel variant for
// this tile width and shape (else the 3x3 streams its 9 taps).
bool wide_halo_fits(int BN, const ConvGemmArgs& a);
// The stacked boxes of a halo of BM + 2 * halo_lo rows: sub boxes of box rows
// (<= 256, a multiple of 8 so every box starts on a swizzle-atom boundary).
void halo_boxes(int halo_lo, int& sub, int& box);

// Cycles per M=128 x N x K=16 SS-mode MMA issued back to back (microbench).
double mma_rate_bench(int N, int iters, int ctas, int two_acc, cudaStream_t st);

// Launches the warp-specialised kernel; BN in {64, 128, 256}. max_ctas > 0
// forces the static persistent scheduler on at most that many CTAs (tests);
// otherwise tiles are handed out by cluster launch control.
void launch_conv_gemm(const Operand& A, const Operand& B, const ConvGemmArgs& a,
                      int BN, cudaStream_t st, int max_ctas = 0);

}  // namespace cg
