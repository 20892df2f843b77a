// ResNet (bottleneck, torchvision v1.5 layout) forward on the tcgen05
// implicit-GEMM kernel. Activations are NHWC bf16; every convolution is one
// conv_gemm launch with BN folded into the weights and bias/ReLU/residual
// fused into the epilogue:
//   1x1 conv           -> GEMM over compact pixel rows
//   3x3 conv, stride 1 -> 9 row-shifted taps over a zero-bordered grid that
//                         the preceding 1x1 conv writes directly (no im2col)
//   3x3, stride 2      -> c1 writes its zero-bordered grid phase split (4
//                         parity planes), so the 3x3 is 9 row shifts over
//                         the planes (no im2col); 1x1/2 downsample: gather
//   conv1 7x7/2        -> fused f64->bf16 im2col of the request input
//   fc                 -> GEMM with f32 logits out
#include <cuda_bf16.h>

#include <cmath>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <stdexcept>

#include "cnn.cuh"
#include "common.cuh"
#include "gemm_sm100.cuh"

namespace cg {
namespace {

using bf16 = __nv_bfloat16;

// ------------------------------------------------------------------ kernels
// Pass 1 of the conv1 operand: f64 CHW -> bf16 NHWC4 on a grid padded by 3
// (channel 3 and the border are zero). Coalesced on both sides: adjacent
// threads read adjacent doubles of each channel plane and write 8 B each.
__global__ void chw_to_nhwc4_pad3_kernel(const double* __restrict__ in, int B, int S,
                                         uint2* __restrict__ out) {
  const int Sp = S + 6;
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)B * Sp * Sp) return;
  int n = (int)(t / ((size_t)Sp * Sp)), rem = (int)(t - (size_t)n * Sp * Sp);
  int hp = rem / Sp, wp = rem - hp * Sp;
  int h = hp - 3, w = wp - 3;
  const bool inside = h >= 0 && h < S && w >= 0 && w < S;
  __align__(8) bf16 b[4];
#pragma unroll
  for (int k = 0; k < 3; k++)  // one f64 -> bf16 rounding, as the direct im2col
    b[k] = __double2bfloat16(inside ? __ldg(in + (((size_t)n * 3 + k) * S + h) * S + w) : 0.0);
  b[3] = __float2bfloat16(0.f);
  out[t] = *reinterpret_cast<uint2*>(b);
}

// The s2d stem operand (default): f64 CHW -> the 2x2 space-to-depth image
// of the input padded by 3 (S + 6 = 2 Gs), channel (py*2 + px)*3 + c holding
// padded pixel (2Y + py, 2X + px) channel c, 12 channels padded to 16:
// [B * Gs * Gs][16] bf16, one 32-byte K = 16 row per pixel
// (ConvGemmArgs::s2d). One thread per s2d pixel; one f64 -> bf16 rounding,
// as the im2col path.
__global__ void chw_to_s2d16_kernel(const double* __restrict__ in, int B, int S,
                                    uint4* __restrict__ out) {
  const int Gs = (S + 6) / 2;
  const size_t npix = (size_t)B * Gs * Gs;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= npix) return;
  const int n = (int)(t / ((size_t)Gs * Gs)), rem = (int)(t - (size_t)n * Gs * Gs);
  const int Y = rem / Gs, X = rem - Y * Gs;
  __align__(16) bf16 v[16];
#pragma unroll
  for (int q = 0; q < 4; q++) {
    const int h = 2 * Y + (q >> 1) - 3, w = 2 * X + (q & 1) - 3;
    const bool inside = h >= 0 && h < S && w >= 0 && w < S;
#pragma unroll
    for (int c = 0; c < 3; c++)
      v[q * 3 + c] =
          __double2bfloat16(inside ? __ldg(in + (((size_t)n * 3 + c) * S + h) * S + w) : 0.0);
  }
#pragma unroll
  for (int k = 12; k < 16; k++) v[k] = __float2bfloat16(0.f);
  out[2 * t] = *reinterpret_cast<const uint4*>(v);
  out[2 * t + 1] = *reinterpret_cast<const uint4*>(v + 8);
}

// Pass 2: [B*Ho*Wo, 192] im2col from the padded NHWC4 grid (K = (dr*7+ds)*3+c,
// zero beyond 147). A warp builds 32 consecutive output rows: lane = row,
// taps loaded as 8-byte pixels (adjacent lanes read pixels 16 B apart), the
// row assembled 16 B at a time in a padded smem tile (row stride 25 x 16 B,
// conflict-free), then written out as one contiguous 12 KB block.
constexpr int kIm2colWarps = 3;
__global__ void __launch_bounds__(32 * kIm2colWarps) conv1_im2col_nhwc4_kernel(
    const uint2* __restrict__ px, int B, int S, int Ho, bf16* __restrict__ out) {
  __shared__ uint4 tile[kIm2colWarps][32 * 25];
  const int Sp = S + 6, lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const size_t rows = (size_t)B * Ho * Ho;
  const size_t row0 = ((size_t)blockIdx.x * kIm2colWarps + w) * 32;
  if (row0 >= rows) return;
  const size_t row = row0 + lane;
  const bool valid = row < rows;
  int n = 0, ho = 0, wo = 0;
  if (valid) {
    n = (int)(row / (Ho * Ho));
    int rem = (int)(row - (size_t)n * Ho * Ho);
    ho = rem / Ho;
    wo = rem - ho * Ho;
  }
  const uint2* base = px + ((size_t)n * Sp + 2 * ho) * Sp + 2 * wo;
  uint4* my = &tile[w][lane * 25];
  uint32_t buf[4] = {0, 0, 0, 0};  // 8 bf16 = one 16-byte chunk
  int fill = 0, chunk = 0;
  auto put = [&](uint32_t bf16_bits) {  // append one bf16
    if (fill & 1) buf[fill >> 1] |= bf16_bits << 16;
    else buf[fill >> 1] = bf16_bits;
    if (++fill == 8) {
      my[chunk++] = make_uint4(buf[0], buf[1], buf[2], buf[3]);
      fill = 0;
    }
  };
  // fully unrolled: every put() position is a compile-time constant, so the
  // 8-value staging buffer stays in registers
#pragma unroll
  for (int dr = 0; dr < 7; dr++) {
#pragma unroll
    for (int ds = 0; ds < 7; ds++) {
      uint2 p = valid ? __ldg(base + dr * Sp + ds) : make_uint2(0, 0);
      put(p.x & 0xffffu);
      put(p.x >> 16);
      put(p.y & 0xffffu);
    }
  }
#pragma unroll
  for (int k = 147; k < 192; k++) put(0);  // K 147 -> 192
  __syncwarp();
  const size_t nrow = rows - row0 < 32 ? rows - row0 : 32;
  uint4* dst = reinterpret_cast<uint4*>(out + row0 * 192);
  for (int i = lane; i < (int)nrow * 24; i += 32) dst[i] = tile[w][(i / 24) * 25 + i % 24];
}

// 3x3/2 max pool, pad 1 (torch pads with -inf). A thread owns two
// horizontally adjacent outputs x 8 channels: their windows share a column,
// so 15 loads instead of 18; packed bf16x2 max (exact, like fmaxf on the
// widened values).
// The input is H x H pixels stored with a row pitch of P pixels and Gh rows
// per image (P = Gh = H: compact; the s2d stem's output grid: Gs x Gs).
__global__ void maxpool3s2_kernel(const bf16* __restrict__ in, int B, int H, int C, int P,
                                  int Gh, bf16* __restrict__ out) {
  const int Ho = (H + 1) / 2, chunks = C / 8, Wq = (Ho + 1) / 2;
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t pq = t / chunks;
  int ch = (int)(t - pq * chunks);
  if (pq >= (size_t)B * Ho * Wq) return;
  int n = (int)(pq / (Ho * Wq)), rem = (int)(pq - (size_t)n * Ho * Wq);
  int ho = rem / Wq, j = rem - ho * Wq;
  const __nv_bfloat162 ninf = __float2bfloat162_rn(-INFINITY);
  __align__(16) __nv_bfloat162 m0[4] = {ninf, ninf, ninf, ninf};
  __align__(16) __nv_bfloat162 m1[4] = {ninf, ninf, ninf, ninf};
#pragma unroll
  for (int dr = 0; dr < 3; dr++) {
    const int h = 2 * ho - 1 + dr;
    if (h < 0 || h >= H) continue;
    const bf16* row = in + ((size_t)n * Gh + h) * P * C + ch * 8;
    uint4 qs[5];  // the row's 5 column loads in flight together (clamped addresses)
#pragma unroll
    for (int dc = 0; dc < 5; dc++)
      qs[dc] = __ldg(reinterpret_cast<const uint4*>(
          row + (size_t)min(max(4 * j - 1 + dc, 0), H - 1) * C));
#pragma unroll
    for (int dc = 0; dc < 5; dc++) {
      const int w = 4 * j - 1 + dc;
      if (w < 0 || w >= H) continue;
      const uint4 q = qs[dc];
      const __nv_bfloat162* e = reinterpret_cast<const __nv_bfloat162*>(&q);
#pragma unroll
      for (int k = 0; k < 4; k++) {
        if (dc <= 2) m0[k] = __hmax2(m0[k], e[k]);
        if (dc >= 2) m1[k] = __hmax2(m1[k], e[k]);
      }
    }
  }
  const int wo = 2 * j;
  bf16* o = out + (((size_t)n * Ho + ho) * Ho + wo) * C + ch * 8;
  *reinterpret_cast<uint4*>(o) = *reinterpret_cast<uint4*>(m0);
  if (wo + 1 < Ho) *reinterpret_cast<uint4*>(o + C) = *reinterpret_cast<uint4*>(m1);
}

// Stride-2 1x1 operand: [B*Ho*Wo, C] = in[n, 2ho, 2wo, :].
__global__ void gather_s2_1x1_kernel(const bf16* __restrict__ in, int B, int H, int C,
                                     bf16* __restrict__ out) {
  const int Ho = H / 2, chunks = C / 8;
  size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  size_t row = t / chunks;
  int ch = (int)(t - row * chunks);
  if (row >= (size_t)B * Ho * Ho) return;
  int n = (int)(row / (Ho * Ho)), rem = (int)(row - (size_t)n * Ho * Ho);
  int ho = rem / Ho, wo = rem - ho * Ho;
  *reinterpret_cast<uint4*>(out + row * C + ch * 8) = __ldg(reinterpret_cast<const uint4*>(
      in + (((size_t)n * H + 2 * ho) * H + 2 * wo) * C + ch * 8));
}

// Global average pool [B, HW, C] -> [B, C]. A CTA owns (image, 256
// channels): 32 lanes x 8 channels, 8 warps striding the pixels, then a
// fixed-order smem reduction over the warps (deterministic, batch-invariant).
__global__ void __launch_bounds__(256) avgpool_kernel(const bf16* __restrict__ in, int B, int HW,
                                                      int C, bf16* __restrict__ out) {
  __shared__ float part[8][32][9];
  const int lane = threadIdx.x & 31, w = threadIdx.x >> 5;
  const int groups = C / 256, n = blockIdx.x / groups, cg = blockIdx.x - n * groups;
  const int c0 = cg * 256 + lane * 8;
  float s[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  for (int p = w; p < HW; p += 8) {
    uint4 q = __ldg(reinterpret_cast<const uint4*>(in + ((size_t)n * HW + p) * C + c0));
    const bf16* e = reinterpret_cast<const bf16*>(&q);
#pragma unroll
    for (int j = 0; j < 8; j++) s[j] += __bfloat162float(e[j]);
  }
#pragma unroll
  for (int j = 0; j < 8; j++) part[w][lane][j] = s[j];
  __syncthreads();
  if (w == 0) {
    float t[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    for (int g = 0; g < 8; g++)
#pragma unroll
      for (int j = 0; j < 8; j++) t[j] += part[g][lane][j];
    __align__(16) bf16 o[8];
    const float inv = 1.0f / (float)HW;
#pragma unroll
    for (int j = 0; j < 8; j++) o[j] = __float2bfloat16(t[j] * inv);
    *reinterpret_cast<uint4*>(out + (size_t)n * C + c0) = *reinterpret_cast<uint4*>(o);
  }
}

unsigned grid_for(size_t threads, int tpb = 256) { return (unsigned)ceil_div(threads, tpb); }

// -------------------------------------------------------- model file parse
// Canonical CNN model file, all big-endian:
//   str "credo.cnn.v1" | str arch | u64 input_dim | u64 output_dim |
//   bool softmax | u32 n | n × { str name | u32 ndim | u64 dim[ndim] |
//   u32 count | count × f32 }
struct HostTensor {
  std::vector<int64_t> dims;
  std::vector<float> v;
};

struct Reader {
  const uint8_t* p;
  uint64_t n, pos = 0;
  void need(uint64_t k) {
    if (n - pos < k) throw std::invalid_argument("cnn file: unexpected end of input");
  }
  uint64_t u64() {
    need(8);
    uint64_t v = 0;
    for (int i = 0; i < 8; i++) v = (v << 8) | p[pos++];
    return v;
  }
  uint32_t u32() {
    need(4);
    uint32_t v = 0;
    for (int i = 0; i < 4; i++) v = (v << 8) | p[pos++];
    return v;
  }
  std::string str() {
    uint32_t l = u32();
    need(l);
    std::string s(reinterpret_cast<const char*>(p + pos), l);
    pos += l;
    return s;
  }
};

uint16_t f2bf_bits(float f) {
  bf16 b = __float2bfloat16(f);  // host conversion, round-to-nearest-even
  uint16_t u;
  std::memcpy(&u, &b, 2);
  return u;
}

struct ConvW {
  int cin = 0, cout = 0, k = 1, stride = 1;
  int Kc = 0, ntaps = 1;        // GEMM K per tap and taps (Ktot = Kc * ntaps)
  std::vector<uint16_t> hw;     // [cout][Ktot] bf16 bits, folded
  std::vector<float> hb;        // [cout]
  bf16* w = nullptr;
  float* b = nullptr;
  Operand opB;
  int BN = 128;
};

struct Block {
  ConvW c1, c2, c3, ds;
  ConvW c3ds;  // has_ds: [W3 | Wds] with b3 + bds, c3 + shortcut as one GEMM
  bool has_ds = false;
  int width = 0, stride = 1, H_in = 0, H_out = 0, cin = 0, cout = 0;
};

// Tile width: minimise waves x BN / eff(BN), where eff reflects that a
// 128 x 64 tile is shared-memory-bandwidth bound (A is re-read per 64
// columns) while 128 x 256 streams A once per 256 columns. Ties -> wider.
int kSmallKMaxBN = 256;  // env CREDO_SMALLK_BN overrides (tuning)
// ResNet stem: the s2d conv (default) or CREDO_NO_S2D=1, the im2col (K = 192)
const bool kUseS2D = std::getenv("CREDO_NO_S2D") == nullptr;
// VGG-16's conv1_1 as the s2d-mode GEMM over a 16-channel grid
// (CREDO_NO_VGG_GRID16=1: the K = 64 im2col operand, A/B)
const bool kVggGrid16 = std::getenv("CREDO_NO_VGG_GRID16") == nullptr;
// 3x3 convs wider than one halo box (VGG-16 at 224 / 112 pixels) through
// stacked halo boxes (CREDO_NO_WIDE_HALO=1: the 9 taps stream, A/B)
const bool kWideHalo = std::getenv("CREDO_NO_WIDE_HALO") == nullptr;
constexpr int kWideHaloRows = 600;  // = gemm_sm100.cu's slot rows
// c3 + projection shortcut as one GEMM over concatenated K (or
// CREDO_NO_FUSE_DS=1: the shortcut GEMM's output read back as a residual)
const bool kFuseDs = std::getenv("CREDO_NO_FUSE_DS") == nullptr;
// the fused stride-2 shortcut reads x[2h, 2w] in place through a strided
// tensor map (or CREDO_NO_A2VIEW=1: a gather pass first)
const bool kA2View = std::getenv("CREDO_NO_A2VIEW") == nullptr;
constexpr int kS2DMaxS = 2 * (256 - 128 - 3) - 6;  // a dy-pair box (128 + Gs + 3 rows) fits 256
const bool kUseHalo = std::getenv("CREDO_NO_HALO") == nullptr;  // A/B switch for measurements

int pick_bn(int rows, int N, int replicas = 1) {
  int best = 64;
  double best_cost = 1e30;
  for (int bn : {256, 128, 64}) {
    if (bn > N && bn != 64) continue;
    long tiles = (long)replicas * ((rows + 127) / 128) * ((N + bn - 1) / bn);
    long waves = (tiles + kNumSMs - 1) / kNumSMs;
    double eff = bn == 256 ? 1.0 : (bn == 128 ? 0.9 : 0.6);
    double cost = (double)waves * bn / eff;
    if (cost < best_cost * 0.999) { best_cost = cost; best = bn; }
  }
  return best;
}

class ResNet final : public CnnModel {
 public:
  ResNet(std::string arch, std::vector<int> layers, uint64_t in_dim, uint64_t out_dim,
         bool sm, std::map<std::string, HostTensor>& T)
      : arch_(std::move(arch)), in_dim_(in_dim), out_dim_(out_dim), softmax_(sm) {
    S_ = (int)std::lround(std::sqrt((double)in_dim / 3.0));
    if ((uint64_t)3 * S_ * S_ != in_dim || S_ % 32 != 0)
      throw std::invalid_argument("cnn file: input_dim must be 3*S*S with S % 32 == 0");
    // conv1 + bn1: the s2d stem (16 taps of K = 16) or K = 147 padded to 192
    s2d_ = kUseS2D && S_ <= kS2DMaxS;
    if (s2d_) fold_s2d(conv1_, T, "conv1.weight", "bn1");
    else fold(conv1_, T, "conv1.weight", "bn1", 7, 2, 192);
    flops_ = 2.0 * (S_ / 2) * (S_ / 2) * 64 * 147;
    int H = S_ / 4, cin = 64;
    const int widths[4] = {64, 128, 256, 512};
    for (int L = 0; L < 4; L++) {
      for (int i = 0; i < layers[L]; i++) {
        Block b;
        std::string pre = "layer" + std::to_string(L + 1) + "." + std::to_string(i) + ".";
        b.width = widths[L];
        b.cin = cin;
        b.cout = 4 * b.width;
        b.stride = (i == 0 && L > 0) ? 2 : 1;
        b.H_in = H;
        b.H_out = H / b.stride;
        fold(b.c1, T, pre + "conv1.weight", pre + "bn1", 1, 1, 0);
        fold(b.c2, T, pre + "conv2.weight", pre + "bn2", 3, b.stride, 0);
        fold(b.c3, T, pre + "conv3.weight", pre + "bn3", 1, 1, 0);
        b.has_ds = T.count(pre + "downsample.0.weight") > 0;
        if (b.has_ds) {
          fold(b.ds, T, pre + "downsample.0.weight", pre + "downsample.1", 1, b.stride, 0);
          fuse_shortcut(b);
        }
        if (b.c1.cin != cin || b.c3.cout != b.cout || b.c2.cin != b.width)
          throw std::invalid_argument("cnn file: unexpected block shapes at " + pre);
        double ho2 = (double)b.H_out * b.H_out;
        flops_ += 2.0 * ((double)H * H * b.cin * b.width + ho2 * 9 * b.width * b.width +
                         ho2 * b.width * b.cout + (b.has_ds ? ho2 * b.cin * b.cout : 0));
        blocks_.push_back(std::move(b));
        cin = 4 * widths[L];
        H = blocks_.back().H_out;
      }
    }
    H_last_ = H;
    // fc
    auto& fw = get(T, "fc.weight", {(int64_t)out_dim, (int64_t)cin});
    auto& fb = get(T, "fc.bias", {(int64_t)out_dim});
    fc_.cin = cin;
    fc_.cout = (int)out_dim;
    fc_.Kc = cin;
    fc_.hw.resize((size_t)out_dim * cin);
    for (size_t i = 0; i < fc_.hw.size(); i++) fc_.hw[i] = f2bf_bits(fw.v[i]);
    fc_.hb = fb.v;
    flops_ += 2.0 * cin * out_dim;
  }

  ~ResNet() override {
    for (ConvW* c : all_convs()) {
      if (c->w) cudaFree(c->w);
      if (c->b) cudaFree(c->b);
    }
    for (void* p : bufs_) cudaFree(p);
  }

  void upload(cudaStream_t st) override {
    for (ConvW* c : all_convs()) {
      CG_CUDA(cudaMalloc(&c->w, c->hw.size() * 2));
      CG_CUDA(cudaMalloc(&c->b, c->hb.size() * 4));
      CG_CUDA(cudaMemcpyAsync(c->w, c->hw.data(), c->hw.size() * 2, cudaMemcpyHostToDevice, st));
      CG_CUDA(cudaMemcpyAsync(c->b, c->hb.data(), c->hb.size() * 4, cudaMemcpyHostToDevice, st));
    }
    CG_CUDA(cudaStreamSynchronize(st));
    for (ConvW* c : all_convs()) {
      std::vector<uint16_t>().swap(c->hw);
    }
  }

  void reserve(uint32_t maxB) override {
    if (maxB <= maxB_) return;
    for (void* p : bufs_) cudaFree(p);
    bufs_.clear();
    plans_.clear();
    maxB_ = maxB;
    const size_t B = maxB;
    const int H1 = S_ / 2, H2 = S_ / 4;
    auto alloc = [&](size_t elems) {
      void* p = nullptr;
      CG_CUDA(cudaMalloc(&p, std::max<size_t>(elems, 8) * 2));
      CG_CUDA(cudaMemset(p, 0, std::max<size_t>(elems, 8) * 2));
      bufs_.push_back(p);
      return reinterpret_cast<bf16*>(p);
    };
    xcol_ = alloc(B * H1 * H1 * 192);
    nhwc4_ = alloc(B * (S_ + 6) * (S_ + 6) * 4);
    c1out_ = alloc(B * (size_t)((S_ + 6) / 2) * ((S_ + 6) / 2) * 64);  // s2d grid >= H1 x H1
    size_t act = 0, t2 = 0, dsz = 0, g1 = 0;
    for (auto& b : blocks_) {
      act = std::max(act, B * b.H_out * b.H_out * b.cout);
      act = std::max(act, B * b.H_in * b.H_in * b.cin);
      t2 = std::max(t2, B * b.H_out * b.H_out * b.width);
      if (b.has_ds) dsz = std::max(dsz, B * b.H_out * b.H_out * b.cout);
      if (b.stride == 2) g1 = std::max(g1, B * b.H_out * b.H_out * b.cin);
      auto key = std::make_pair(b.H_in, b.width);
      if (!pads_.count(key)) pads_[key] = nullptr;
    }
    act_[0] = alloc(std::max(act, B * H2 * H2 * 64));
    act_[1] = alloc(act);
    t2_ = alloc(t2);
    ds_ = alloc(dsz);
    g1_ = alloc(g1);
    for (auto& kv : pads_) {
      size_t Hp = kv.first.first + 2;
      kv.second = alloc(B * Hp * Hp * kv.first.second);
    }
    pooled_ = alloc(B * fc_.cin);
  }

  size_t prepared_bytes(uint32_t B) const override {
    const size_t Gs = (S_ + 6) / 2;
    return s2d_ ? (size_t)B * Gs * Gs * 32 : (size_t)B * (S_ / 2) * (S_ / 2) * 192 * 2;
  }
  std::string prep_kind() const override {
    return (s2d_ ? "s2d16/" : "im2col7x7s2k192/") + std::to_string(S_);
  }

  void prepare_input(const double* d_in, uint32_t B, void* prepped, cudaStream_t st) override {
    const int H1 = S_ / 2, Sp = S_ + 6;
    if (B > maxB_) reserve(B);
    timer_begin(st, kTimeAux);
    if (s2d_) {  // one pass: f64 CHW -> the padded s2d image
      chw_to_s2d16_kernel<<<grid_for((size_t)B * (Sp / 2) * (Sp / 2)), 256, 0, st>>>(
          d_in, B, S_, reinterpret_cast<uint4*>(prepped));
      CG_CHECK_LAUNCH();
      timer_end(st, kTimeAux);
      return;
    }
    // two coalesced passes: f64 CHW -> bf16 NHWC4 (pad 3), then im2col
    chw_to_nhwc4_pad3_kernel<<<grid_for((size_t)B * Sp * Sp), 256, 0, st>>>(
        d_in, B, S_, reinterpret_cast<uint2*>(nhwc4_));
    CG_CHECK_LAUNCH();
    size_t rows = (size_t)B * H1 * H1;
    conv1_im2col_nhwc4_kernel<<<(unsigned)ceil_div(rows, 32 * kIm2colWarps), 32 * kIm2colWarps,
                                0, st>>>(reinterpret_cast<const uint2*>(nhwc4_), B, S_, H1,
                                         reinterpret_cast<bf16*>(prepped));
    CG_CHECK_LAUNCH();
    timer_end(st, kTimeAux);
  }

  void forward(const double* d_in, uint32_t B, float* logits, cudaStream_t st,
               const void* prepped) override {
    if (B > maxB_) reserve(B);
    const bf16* x0 = reinterpret_cast<const bf16*>(prepped);
    if (!x0) {
      prepare_input(d_in, B, xcol_, st);
      x0 = xcol_;
    }
    Plan& p = plan_for(B, x0, logits);
    for (auto& s : p.steps) s(st);
  }

  uint64_t input_dim() const override { return in_dim_; }
  uint64_t output_dim() const override { return out_dim_; }
  bool softmax() const override { return softmax_; }
  std::string arch() const override { return arch_; }
  double flops_per_image() const override { return flops_; }
  int image_size() const { return S_; }
  size_t num_blocks() const { return blocks_.size(); }

  // One launch of the forward, described per replica (nothing launched):
  // a GEMM (shape + this replica's operands) or an auxiliary kernel.
  struct GemmDesc {
    ConvW* c = nullptr;
    const bf16* A = nullptr;
    int rowsA = 0, M = 0, Kc = 0, ntaps = 1, taps[9] = {0};
    const bf16* res = nullptr;
    int ldres = 0;
    void* out = nullptr;
    int ldout = 0, out_f32 = 0, relu = 0, mode = 0, H = 0, rows_out = 0;
    int halo_lo = 0;  // > 0: 3x3 taps fed from one halo box per channel block
    int s2d = 0, gh = 0, gw = 0;  // the s2d stem (ConvGemmArgs::s2d)
    int s2d_step = 0, s2d_ndy = 0;  // ConvGemmArgs::s2d_step / s2d_ndy
    const bf16* A2 = nullptr;     // second K segment operand (ConvGemmArgs::kc2)
    int kc2 = 0;
    int a2_b = 0, a2_h = 0, a2_rpb = 0;  // A2 = x[2h, 2w] of [a2_b, a2_h, a2_h, kc2] in place
  };
  struct Op {
    bool gemm = false;
    GemmDesc g;
    std::function<void(cudaStream_t)> aux;
  };

  // The forward as a list of launches (csrc/cnn.cu header comment).
  std::vector<Op> ops(uint32_t B, const void* x0, float* logits) {
    std::vector<Op> L;
    auto gemm = [&](ConvW& c, const bf16* A, int rowsA, int M, int Kc, int ntaps,
                    const int* taps, const bf16* residual, int ldres, void* out, int ldout,
                    int out_f32, int relu, int mode, int H, int rows_out) {
      Op o;
      o.gemm = true;
      GemmDesc& g = o.g;
      g.c = &c;
      g.A = A;
      g.rowsA = rowsA;
      g.M = M;
      g.Kc = Kc;
      g.ntaps = ntaps;
      for (int t = 0; t < ntaps; t++) g.taps[t] = taps[t];
      g.res = residual;
      g.ldres = ldres;
      g.out = out;
      g.ldout = ldout;
      g.out_f32 = out_f32;
      g.relu = relu;
      g.mode = mode;
      g.H = H;
      g.rows_out = rows_out;
      L.push_back(std::move(o));
    };
    auto aux = [&](std::function<void(cudaStream_t)> f) {
      Op o;
      o.aux = [f](cudaStream_t st) {
        timer_begin(st, kTimeAux);
        f(st);
        timer_end(st, kTimeAux);
      };
      L.push_back(std::move(o));
    };
    const int H1 = S_ / 2;
    const int zero = 0;
    // conv1 (s2d stem or im2col operand) -> c1out, then maxpool -> act_[0]
    if (s2d_) {
      const int Gs = (S_ + 6) / 2;
      // output stays on the Gs x Gs grid (identity rows: TMA-store epilogue;
      // the max pool reads the H1 x H1 interior of each image's grid)
      gemm(conv1_, reinterpret_cast<const bf16*>(x0), B * Gs * Gs, B * Gs * Gs, 16, 1, &zero,
           nullptr, 0, c1out_, 64, 0, 1, kRowIdentity, H1, B * Gs * Gs);
      L.back().g.ntaps = 16;  // taps (dy, dx) are implicit in the s2d mode
      L.back().g.s2d = 1;
      L.back().g.gh = L.back().g.gw = Gs;
    } else {
      gemm(conv1_, reinterpret_cast<const bf16*>(x0), B * H1 * H1, B * H1 * H1, conv1_.Kc, 1,
           &zero, nullptr, 0, c1out_, 64, 0, 1, kRowIdentity, 0, B * H1 * H1);
    }
    {
      bf16* in = c1out_;
      bf16* out = act_[0];
      const int P = s2d_ ? (S_ + 6) / 2 : H1;  // conv1 output pitch / rows per image
      aux([in, out, B, H1, P](cudaStream_t st) {
        const size_t Ho = (H1 + 1) / 2;
        size_t th = (size_t)B * Ho * ((Ho + 1) / 2) * (64 / 8);
        maxpool3s2_kernel<<<grid_for(th), 256, 0, st>>>(in, B, H1, 64, P, P, out);
        CG_CHECK_LAUNCH();
      });
    }
    int cur = 0;
    for (auto& b : blocks_) {
      bf16* X = act_[cur];
      bf16* Y = act_[cur ^ 1];
      const int Hi = b.H_in, Ho = b.H_out, Hp = Hi + 2;
      const int G = Hi + 1;  // shared-border grid pitch (remap_row, gemm_sm100.cu)
      bf16* P = pads_.at({Hi, b.width});
      if (b.stride == 1) {
        // c1: 1x1 -> interior of the zero-bordered grid
        gemm(b.c1, X, B * Hi * Hi, B * Hi * Hi, b.c1.Kc, 1, &zero, nullptr, 0, P, b.width, 0, 1,
             kRowCompactToPad, Hi, B * G * G);
        // c2: 3x3 as 9 row shifts of the padded grid
        int taps[9];
        for (int dr = 0; dr < 3; dr++)
          for (int ds = 0; ds < 3; ds++) taps[dr * 3 + ds] = (dr - 1) * G + (ds - 1);
        gemm(b.c2, P, B * G * G, B * G * G, b.c2.Kc, 9, taps, nullptr, 0, t2_, b.width, 0,
             1, kRowPadToCompact, Hi, B * Ho * Ho);
        // halo mode: the 9 taps read one (128 + 2*(G+1))-row box per
        // channel block from shared memory (4.7-7x less operand traffic)
        if (kUseHalo && 128 + 2 * (G + 1) <= 256) L.back().g.halo_lo = G + 1;
      } else {
        // Stride 2: c1 writes the phase split of its zero-bordered grid; the
        // stride-2 3x3 is then 9 row shifts (plane base + p*Wq + q) over an
        // (Ho+1)^2 plane-00 grid.
        gemm(b.c1, X, B * Hi * Hi, B * Hi * Hi, b.c1.Kc, 1, &zero, nullptr, 0, P, b.width, 0, 1,
             kRowCompactToPhasePad, Hi, B * Hp * Hp);
        const int Wq = Ho + 1, plane = B * Wq * Wq;
        int taps[9];
        for (int dr = 0; dr < 3; dr++)
          for (int ds = 0; ds < 3; ds++)
            taps[dr * 3 + ds] = ((dr & 1) * 2 + (ds & 1)) * plane + (dr >> 1) * Wq + (ds >> 1);
        gemm(b.c2, P, 4 * plane, plane, b.c2.Kc, 9, taps, nullptr, 0, t2_, b.width, 0, 1,
             kRowPhaseGridToCompact, Ho, B * Ho * Ho);
      }
      // identity / downsample (stride 2: the decimated input X[2h, 2w])
      const bf16* ident = X;
      if (b.has_ds && kFuseDs) {
        // c3 + shortcut: K over t2's width channels, then the (decimated) x
        const bf16* dsin = X;
        const bool view = b.stride == 2 && kA2View && Ho <= 56 && 56 % Ho == 0;
        if (b.stride == 2 && !view) {
          bf16* G1 = g1_;
          const int C = b.cin;
          aux([X, G1, B, Hi, C](cudaStream_t st) {
            size_t th = (size_t)B * (Hi / 2) * (Hi / 2) * (C / 8);
            gather_s2_1x1_kernel<<<grid_for(th), 256, 0, st>>>(X, B, Hi, C, G1);
            CG_CHECK_LAUNCH();
          });
          dsin = G1;
        }
        gemm(b.c3ds, t2_, B * Ho * Ho, B * Ho * Ho, b.c3ds.Kc, 1, &zero, nullptr, 0, Y, b.cout,
             0, 1, kRowIdentity, 0, B * Ho * Ho);
        L.back().g.A2 = dsin;
        L.back().g.kc2 = b.ds.Kc;
        if (view) {
          L.back().g.a2_b = (int)B;
          L.back().g.a2_h = Hi;
          L.back().g.a2_rpb = 56 / Ho;
        }
        cur ^= 1;
        continue;
      }
      if (b.has_ds) {
        const bf16* dsin = X;
        if (b.stride == 2) {
          bf16* G1 = g1_;
          const int C = b.cin;
          aux([X, G1, B, Hi, C](cudaStream_t st) {
            size_t th = (size_t)B * (Hi / 2) * (Hi / 2) * (C / 8);
            gather_s2_1x1_kernel<<<grid_for(th), 256, 0, st>>>(X, B, Hi, C, G1);
            CG_CHECK_LAUNCH();
          });
          dsin = G1;
        }
        gemm(b.ds, dsin, B * Ho * Ho, B * Ho * Ho, b.ds.Kc, 1, &zero, nullptr, 0, ds_, b.cout,
             0, 0, kRowIdentity, 0, B * Ho * Ho);
        ident = ds_;
      }
      // c3: 1x1 + residual + ReLU
      gemm(b.c3, t2_, B * Ho * Ho, B * Ho * Ho, b.c3.Kc, 1, &zero, ident, b.cout, Y, b.cout, 0,
           1, kRowIdentity, 0, B * Ho * Ho);
      cur ^= 1;
    }
    {
      bf16* in = act_[cur];
      bf16* out = pooled_;
      int HW = H_last_ * H_last_, C = fc_.cin;
      aux([in, out, B, HW, C](cudaStream_t st) {
        avgpool_kernel<<<(unsigned)(B * (C / 256)), 256, 0, st>>>(in, B, HW, C, out);
        CG_CHECK_LAUNCH();
      });
    }
    gemm(fc_, pooled_, B, B, fc_.Kc, 1, &zero, nullptr, 0, logits, (int)out_dim_, 1, 0,
         kRowIdentity, 0, B);
    return L;
  }

 private:
  struct Plan {
    const void* x0 = nullptr;
    float* logits = nullptr;
    std::vector<std::function<void(cudaStream_t)>> steps;
  };

  static HostTensor& get(std::map<std::string, HostTensor>& T, const std::string& name,
                         std::vector<int64_t> dims) {
    auto it = T.find(name);
    if (it == T.end()) throw std::invalid_argument("cnn file: missing tensor " + name);
    if (!dims.empty() && it->second.dims != dims)
      throw std::invalid_argument("cnn file: bad shape for " + name);
    return it->second;
  }

  // Folds eval-mode BatchNorm into the preceding conv (torch BN eps 1e-5):
  // w' = w * g / sqrt(var + eps), b' = beta - mean * g / sqrt(var + eps).
  // Weight layout [cout][(dr*k + ds)*cin + c], zero-padded to Kpad.
  void fold(ConvW& c, std::map<std::string, HostTensor>& T, const std::string& wname,
            const std::string& bn, int k, int stride, int Kpad) {
    auto it = T.find(wname);
    if (it == T.end()) throw std::invalid_argument("cnn file: missing tensor " + wname);
    const HostTensor& W = it->second;
    if (W.dims.size() != 4 || W.dims[2] != k || W.dims[3] != k)
      throw std::invalid_argument("cnn file: bad conv shape " + wname);
    c.cout = (int)W.dims[0];
    c.cin = (int)W.dims[1];
    c.k = k;
    c.stride = stride;
    const int64_t co = c.cout;
    auto& g = get(T, bn + ".weight", {co});
    auto& be = get(T, bn + ".bias", {co});
    auto& mu = get(T, bn + ".running_mean", {co});
    auto& var = get(T, bn + ".running_var", {co});
    const int K = k * k * c.cin;
    const int Ktot = Kpad ? Kpad : K;
    if (!Kpad && c.cin % 64) throw std::invalid_argument("cnn file: channels % 64 != 0");
    c.ntaps = (k == 3 && !Kpad) ? 9 : 1;
    c.Kc = (c.ntaps == 9) ? c.cin : Ktot;
    c.hw.assign((size_t)c.cout * Ktot, 0);
    c.hb.resize(c.cout);
    for (int o = 0; o < c.cout; o++) {
      double s = (double)g.v[o] / std::sqrt((double)var.v[o] + 1e-5);
      c.hb[o] = (float)((double)be.v[o] - (double)mu.v[o] * s);
      for (int ci = 0; ci < c.cin; ci++)
        for (int dr = 0; dr < k; dr++)
          for (int ds = 0; ds < k; ds++) {
            float w = W.v[(((size_t)o * c.cin + ci) * k + dr) * k + ds];
            c.hw[(size_t)o * Ktot + (dr * k + ds) * c.cin + ci] = f2bf_bits((float)(w * s));
          }
    }
  }

  // conv1 (7x7/2, pad 3) as a 4x4 stride-1 conv over the 2x2 space-to-depth
  // image: tap (dy, dx), s2d channel (py*2 + px)*3 + c is kernel position
  // (2 dy + py, 2 dx + px) channel c (zero at kernel row / column 7). Layout
  // [tap][cout][16] (K = 16 per tap), the resident weight tile of the s2d
  // GEMM mode.
  void fold_s2d(ConvW& c, std::map<std::string, HostTensor>& T, const std::string& wname,
                const std::string& bn) {
    fold(c, T, wname, bn, 7, 2, 147);  // [cout][(dr*7 + ds)*3 + ci]
    if (c.cin != 3 || c.cout != 64) throw std::invalid_argument("cnn file: stem must be 3 -> 64");
    std::vector<uint16_t> w((size_t)16 * 64 * 16, 0);
    for (int o = 0; o < 64; o++)
      for (int tap = 0; tap < 16; tap++)
        for (int ch = 0; ch < 12; ch++) {
          const int dy = tap / 4, dx = tap % 4, q = ch / 3, ci = ch % 3;
          const int dr = 2 * dy + (q >> 1), ds = 2 * dx + (q & 1);
          if (dr > 6 || ds > 6) continue;
          w[((size_t)tap * 64 + o) * 16 + ch] =
              c.hw[(size_t)o * 147 + (dr * 7 + ds) * 3 + ci];
        }
    c.hw.swap(w);
    c.Kc = 16;
    c.ntaps = 16;
  }

  // relu(bn3(conv3(t2)) + bn_ds(conv_ds(x))) = relu([t2 | x] [W3 | Wds]^T +
  // b3 + bds): the bottleneck's last conv and its projection shortcut as
  // one GEMM whose K runs over t2's channels, then x's (ConvGemmArgs::kc2),
  // both folded with their BatchNorms; one fp32 accumulation instead of a
  // bf16 shortcut tensor written and read back.
  static void fuse_shortcut(Block& b) {
    const ConvW &c3 = b.c3, &ds = b.ds;
    if (c3.cout != ds.cout || c3.ntaps != 1 || ds.ntaps != 1)
      throw std::invalid_argument("cnn file: shortcut does not match conv3");
    ConvW& f = b.c3ds;
    f.cin = c3.Kc + ds.Kc;
    f.cout = c3.cout;
    f.k = 1;
    f.stride = 1;
    f.Kc = c3.Kc;  // first segment; the second (ds.Kc) goes in GemmDesc::kc2
    f.ntaps = 1;
    const int K = c3.Kc + ds.Kc;
    f.hw.assign((size_t)f.cout * K, 0);
    f.hb.resize(f.cout);
    for (int o = 0; o < f.cout; o++) {
      std::copy(c3.hw.begin() + (size_t)o * c3.Kc, c3.hw.begin() + (size_t)(o + 1) * c3.Kc,
                f.hw.begin() + (size_t)o * K);
      std::copy(ds.hw.begin() + (size_t)o * ds.Kc, ds.hw.begin() + (size_t)(o + 1) * ds.Kc,
                f.hw.begin() + (size_t)o * K + c3.Kc);
      f.hb[o] = c3.hb[o] + ds.hb[o];
    }
  }

  std::vector<ConvW*> all_convs() {
    std::vector<ConvW*> v{&conv1_, &fc_};
    for (auto& b : blocks_) {
      v.push_back(&b.c1);
      v.push_back(&b.c2);
      v.push_back(&b.c3);
      if (b.has_ds) {
        v.push_back(&b.ds);
        v.push_back(&b.c3ds);
      }
    }
    return v;
  }

  Plan& plan_for(uint32_t B, const void* x0, float* logits) {
    auto it = plans_.find(B);
    if (it != plans_.end() && it->second.x0 == x0 && it->second.logits == logits)
      return it->second;
    Plan& p = plans_[B];
    p = Plan{};
    p.x0 = x0;
    p.logits = logits;
    for (Op& o : ops(B, x0, logits)) {
      if (o.gemm) p.steps.push_back(make_gemm_step({&o.g}));
      else p.steps.push_back(std::move(o.aux));
    }
    return p;
  }

 public:
  // One (grouped) GEMM launch over R replicas' descriptors of the same layer:
  // tensor maps encoded once here, the returned step just launches.
  static std::function<void(cudaStream_t)> make_gemm_step(const std::vector<const GemmDesc*>& ds) {
    const GemmDesc& d0 = *ds[0];
    const int R = (int)ds.size();
    int BN = pick_bn(d0.M, d0.c->cout, R);
    if (const char* e = std::getenv("CREDO_SMALLK_BN")) kSmallKMaxBN = std::atoi(e);
    if (d0.Kc * d0.ntaps <= 128 && BN > kSmallKMaxBN) BN = kSmallKMaxBN;
    std::vector<Operand> A(R), Bm(R), A2(R);
    ConvGemmGroup g;
    g.n = R;
    if (d0.s2d) BN = 64;
    if (d0.a2_rpb) BN = 256;  // the strided-A2 kernel variant is BN = 256
    // wide halos (BM + 2 * halo_lo > 256 rows): stacked boxes of <= 256
    // rows when a kernel variant fits this shape, else the taps stream
    int halo_lo = d0.halo_lo, halo_sub = 1, hbox = 128 + 2 * halo_lo;
    if (halo_lo > 0 && 128 + 2 * halo_lo > 256) {
      ConvGemmArgs t{};
      t.N = d0.c->cout;
      t.Kc = d0.Kc;
      t.ntaps = d0.ntaps;
      t.halo_lo = halo_lo;
      t.out_f32 = d0.out_f32;
      halo_boxes(halo_lo, halo_sub, hbox);
      if (!kWideHalo || !wide_halo_fits(BN, t)) halo_lo = 0, halo_sub = 1, hbox = 128;
    }
    for (int r = 0; r < R; r++) {
      const GemmDesc& d = *ds[r];
      if (d.s2d) {
        make_operand_s2d_a(A[r], d.A, d.rowsA, 128 + (d.s2d_step == 1 ? 0 : d.gw) + 3);
        make_operand_s2d_b(Bm[r], d.c->w, 16 * d.c->cout);
      } else {
        make_operand(A[r], d.A, d.rowsA, d.Kc, hbox);
        make_operand(Bm[r], d.c->w, d.c->cout, d.Kc * d.ntaps + d.kc2, BN);
        if (d.kc2) {
          if (d.a2_rpb) make_operand_s2_view(A2[r], d.A2, d.a2_b, d.a2_h, d.kc2, d.a2_rpb);
          else make_operand(A2[r], d.A2, d.rowsA, d.kc2, 128);
          g.A2[r] = &A2[r];
        }
      }
      g.A[r] = &A[r];
      g.B[r] = &Bm[r];
      g.bias[r] = d.c->b;
      g.residual[r] = d.res;
      g.out[r] = d.out;
    }
    ConvGemmArgs a{};
    a.M = d0.M;
    a.N = d0.c->cout;
    a.Kc = d0.Kc;
    a.ntaps = d0.ntaps;
    for (int t = 0; t < d0.ntaps && t < 9; t++) a.tap_off[t] = d0.taps[t];
    a.ld_res = d0.ldres;
    a.ld_out = d0.ldout;
    a.out_f32 = d0.out_f32;
    a.relu = d0.relu;
    a.row_mode = d0.mode;
    a.H = d0.H;
    a.W = d0.H;
    a.rows_out = d0.rows_out;
    a.halo_lo = halo_lo;
    a.halo_sub = halo_sub;
    a.halo_box = hbox;
    a.s2d = d0.s2d;
    a.s2d_step = d0.s2d_step;
    a.s2d_ndy = d0.s2d_ndy;
    a.kc2 = d0.kc2;
    a.a2_wo = d0.a2_rpb ? d0.a2_h / 2 : 0;
    a.a2_rpb = d0.a2_rpb;
    a.gh = d0.gh;
    a.gw = d0.gw;
    auto p = std::make_shared<PreparedGemm>();
    prepare_conv_gemm(*p, g, a, BN);
    return [p](cudaStream_t st) { launch_prepared(*p, st); };
  }

 private:
  std::string arch_;
  uint64_t in_dim_, out_dim_;
  bool softmax_;
  int S_ = 224, H_last_ = 7;
  double flops_ = 0;
  ConvW conv1_, fc_;
  std::vector<Block> blocks_;
  uint32_t maxB_ = 0;
  std::vector<void*> bufs_;
  bool s2d_ = false;  // the s2d stem (kUseS2D, image size within kS2DMaxS)
  bf16 *xcol_ = nullptr, *nhwc4_ = nullptr, *c1out_ = nullptr, *act_[2] = {nullptr, nullptr}, *t2_ = nullptr,
       *ds_ = nullptr, *g1_ = nullptr, *pooled_ = nullptr;
  std::map<std::pair<int, int>, bf16*> pads_;
  std::map<uint32_t, Plan> plans_;
};

// ------------------------------------------------ VGG-16 and MobileNetV2
// The heterogeneous-group architectures (BASELINE configs[2]), on the same
// tcgen05 conv GEMM. Channel counts are padded to multiples of 64 with zero
// weights (zero bias), so padded channels carry exact zeros end to end.

// 3x3 im2col straight from the f64 CHW request input: [B*Ho*Ho, 64] bf16,
// K = (dr*3 + ds)*3 + c for the 27 real taps, zero beyond (pad 1).
__global__ void im2col3x3_f64_kernel(const double* __restrict__ in, int B, int S, int stride,
                                     int Ho, bf16* __restrict__ out) {
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t row = t >> 3;
  const int chunk = (int)(t & 7);
  if (row >= (size_t)B * Ho * Ho) return;
  const int n = (int)(row / ((size_t)Ho * Ho)), rem = (int)(row - (size_t)n * Ho * Ho);
  const int ho = rem / Ho, wo = rem - ho * Ho;
  __align__(16) bf16 o[8];
#pragma unroll
  for (int j = 0; j < 8; j++) {
    const int k = chunk * 8 + j;
    double x = 0.0;
    if (k < 27) {
      const int tap = k / 3, c = k - tap * 3, dr = tap / 3, ds = tap - dr * 3;
      const int h = ho * stride - 1 + dr, w = wo * stride - 1 + ds;
      if (h >= 0 && h < S && w >= 0 && w < S) x = __ldg(in + (((size_t)n * 3 + c) * S + h) * S + w);
    }
    o[j] = __double2bfloat16(x);
  }
  *reinterpret_cast<uint4*>(out + row * 64 + chunk * 8) = *reinterpret_cast<uint4*>(o);
}

// The same operand, one CTA per output image row (n, ho): the 3 input rows
// x 3 planes it needs are read once, coalesced along w, rounded f64 ->
// bf16 (the same single rounding) into shared memory with a zero column on
// each side, then every (pixel, 16-byte K chunk) of the row is assembled
// from shared memory and stored coalesced (consecutive threads, consecutive
// 16-byte pieces of the [rows, 64] operand).
constexpr int kIm2colMaxS = 512;
__global__ void __launch_bounds__(256) im2col3x3_f64_rows_kernel(const double* __restrict__ in,
                                                                 int B, int S, int stride,
                                                                 int Ho, bf16* __restrict__ out) {
  __shared__ bf16 sm[9][kIm2colMaxS + 2];  // [c * 3 + dr][w + 1]
  const int n = blockIdx.x / Ho, ho = blockIdx.x - n * Ho;
  for (int i = threadIdx.x; i < 9 * (S + 2); i += blockDim.x) {
    const int rr = i / (S + 2), wp = i - rr * (S + 2);
    const int c = rr / 3, dr = rr - c * 3, h = ho * stride - 1 + dr, w = wp - 1;
    double x = 0.0;
    if (h >= 0 && h < S && w >= 0 && w < S) x = __ldg(in + (((size_t)n * 3 + c) * S + h) * S + w);
    sm[rr][wp] = __double2bfloat16(x);
  }
  __syncthreads();
  uint4* o = reinterpret_cast<uint4*>(out + ((size_t)n * Ho + ho) * Ho * 64);
  for (int i = threadIdx.x; i < Ho * 8; i += blockDim.x) {
    const int wo = i >> 3, chunk = i & 7;
    uint4 v = make_uint4(0, 0, 0, 0);
    if (chunk < 4) {
      __align__(16) bf16 e[8];
#pragma unroll
      for (int j = 0; j < 8; j++) {
        const int k = chunk * 8 + j;  // K = (dr * 3 + ds) * 3 + c
        bf16 x = __float2bfloat16(0.f);
        if (k < 27) {
          const int tap = k / 3, c = k - tap * 3, dr = tap / 3, ds = tap - dr * 3;
          x = sm[c * 3 + dr][wo * stride + ds];
        }
        e[j] = x;
      }
      v = *reinterpret_cast<const uint4*>(e);
    }
    o[i] = v;
  }
}

// VGG-16's conv1_1 operand: f64 CHW -> a zero-bordered [B][S+3][S+3][16]
// bf16 grid, pixel (i, j) at grid (i+1, j+1), channels 3..15 zero (one
// rounding f64 -> bf16). The 3x3 conv then runs as the s2d-mode GEMM: a 4x4
// with zero fourth taps, one K = 16 MMA per tap (ConvGemmArgs::s2d_step 1).
__global__ void chw_to_grid16_kernel(const double* __restrict__ in, int B, int S,
                                     uint4* __restrict__ out) {
  const int G = S + 3;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= (size_t)B * G * G) return;
  const int n = (int)(t / ((size_t)G * G)), rem = (int)(t - (size_t)n * G * G);
  const int i = rem / G - 1, j = rem - (rem / G) * G - 1;
  __align__(16) bf16 e[16];
#pragma unroll
  for (int c = 0; c < 16; c++) e[c] = __float2bfloat16(0.f);
  if (i >= 0 && i < S && j >= 0 && j < S) {
#pragma unroll
    for (int c = 0; c < 3; c++)
      e[c] = __double2bfloat16(__ldg(in + (((size_t)n * 3 + c) * S + i) * S + j));
  }
  out[2 * t] = reinterpret_cast<const uint4*>(e)[0];
  out[2 * t + 1] = reinterpret_cast<const uint4*>(e)[1];
}

// 2x2/2 max pool, compact NHWC in; out compact, or the interior of a
// zero-bordered (H/2+2)^2 grid when padded_out.
__global__ void maxpool2x2_kernel(const bf16* __restrict__ in, int B, int H, int C,
                                  int padded_out, bf16* __restrict__ out) {
  const int Ho = H / 2, chunks = C / 8;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t pix = t / chunks;
  const int ch = (int)(t - pix * chunks);
  if (pix >= (size_t)B * Ho * Ho) return;
  const int n = (int)(pix / (Ho * Ho)), rem = (int)(pix - (size_t)n * Ho * Ho);
  const int ho = rem / Ho, wo = rem - ho * Ho;
  float m[8];
#pragma unroll
  for (int j = 0; j < 8; j++) m[j] = -INFINITY;
#pragma unroll
  for (int d = 0; d < 4; d++) {
    const int h = 2 * ho + (d >> 1), w = 2 * wo + (d & 1);
    const uint4 q =
        __ldg(reinterpret_cast<const uint4*>(in + (((size_t)n * H + h) * H + w) * C + ch * 8));
    const bf16* e = reinterpret_cast<const bf16*>(&q);
#pragma unroll
    for (int j = 0; j < 8; j++) m[j] = fmaxf(m[j], __bfloat162float(e[j]));
  }
  __align__(16) bf16 o[8];
#pragma unroll
  for (int j = 0; j < 8; j++) o[j] = __float2bfloat16(m[j]);
  // padded: the next conv's shared-border grid (pitch Ho + 1, remap_row)
  const size_t orow = padded_out ? ((size_t)n * (Ho + 1) + ho + 1) * (Ho + 1) + wo : pix;
  *reinterpret_cast<uint4*>(out + orow * C + ch * 8) = *reinterpret_cast<uint4*>(o);
}

// Depthwise 3x3 (pad 1, stride 1/2) + folded-BN bias + ReLU6, NHWC bf16,
// f32 weights [9][C] tap-major; thread = (output pixel, 8 channels).
// Depthwise 3x3 (pad 1) + bias + ReLU6 on NHWC bf16. A thread owns 8
// channels of P horizontally adjacent outputs: each input column is loaded
// once for all the outputs whose windows cover it, and a kernel row's 3 x 8
// weights are loaded once for all P outputs (per output: 9 x 16 B input +
// 9 x 32 B weight loads at P = 1, about a third of that at P = 4). The tap
// order of every output's FMA chain is unchanged (rows, then columns).
template <int STRIDE, int P>
__global__ void __launch_bounds__(256) dw3x3_kernel(const bf16* __restrict__ in, int B, int H,
                                                    int C, const float* __restrict__ w,
                                                    const float* __restrict__ bias,
                                                    bf16* __restrict__ out) {
  const int Ho = (H - 1) / STRIDE + 1, chunks = C / 8, Wg = (Ho + P - 1) / P;
  const size_t t = (size_t)blockIdx.x * blockDim.x + threadIdx.x;
  const size_t grp = t / chunks;
  const int ch = (int)(t - grp * chunks);
  if (grp >= (size_t)B * Ho * Wg) return;
  const int n = (int)(grp / ((size_t)Ho * Wg)), rem = (int)(grp - (size_t)n * Ho * Wg);
  const int ho = rem / Wg, wo0 = (rem - ho * Wg) * P;
  const int c0 = ch * 8;
  float acc[P][8];
  {
    const float4 b0 = __ldg(reinterpret_cast<const float4*>(bias + c0));
    const float4 b1 = __ldg(reinterpret_cast<const float4*>(bias + c0 + 4));
    const float bv[8] = {b0.x, b0.y, b0.z, b0.w, b1.x, b1.y, b1.z, b1.w};
#pragma unroll
    for (int p = 0; p < P; p++)
#pragma unroll
      for (int j = 0; j < 8; j++) acc[p][j] = bv[j];
  }
  constexpr int NCOL = (P - 1) * STRIDE + 3;  // input columns covering the P windows
  const int x0 = wo0 * STRIDE - 1;
#pragma unroll
  for (int dr = 0; dr < 3; dr++) {
    const int h = ho * STRIDE - 1 + dr;
    if (h < 0 || h >= H) continue;
    float wr[3][8];
#pragma unroll
    for (int ds = 0; ds < 3; ds++) {
      const float4 w0 = __ldg(reinterpret_cast<const float4*>(w + (dr * 3 + ds) * C + c0));
      const float4 w1 = __ldg(reinterpret_cast<const float4*>(w + (dr * 3 + ds) * C + c0 + 4));
      wr[ds][0] = w0.x; wr[ds][1] = w0.y; wr[ds][2] = w0.z; wr[ds][3] = w0.w;
      wr[ds][4] = w1.x; wr[ds][5] = w1.y; wr[ds][6] = w1.z; wr[ds][7] = w1.w;
    }
    const bf16* row = in + ((size_t)n * H + h) * H * C + c0;
    // all of the row's column loads first (clamped addresses, zero outside):
    // NCOL independent 16-byte loads in flight per thread
    uint4 qs[NCOL];
#pragma unroll
    for (int col = 0; col < NCOL; col++) {
      const int x = min(max(x0 + col, 0), H - 1);
      qs[col] = __ldg(reinterpret_cast<const uint4*>(row + (size_t)x * C));
    }
#pragma unroll
    for (int col = 0; col < NCOL; col++) {
      const int x = x0 + col;
      if (x < 0 || x >= H) continue;
      const bf16* e = reinterpret_cast<const bf16*>(&qs[col]);
      float v[8];
#pragma unroll
      for (int j = 0; j < 8; j++) v[j] = __bfloat162float(e[j]);
#pragma unroll
      for (int p = 0; p < P; p++) {
        const int ds = col - p * STRIDE;  // this column's tap in output p's window
        if (ds < 0 || ds > 2) continue;
#pragma unroll
        for (int j = 0; j < 8; j++) acc[p][j] = fmaf(v[j], wr[ds][j], acc[p][j]);
      }
    }
  }
#pragma unroll
  for (int p = 0; p < P; p++) {
    if (wo0 + p >= Ho) break;
    __align__(16) bf16 o[8];
#pragma unroll
    for (int j = 0; j < 8; j++) o[j] = __float2bfloat16(fminf(fmaxf(acc[p][j], 0.f), 6.f));
    *reinterpret_cast<uint4*>(out + (((size_t)n * Ho + ho) * Ho + wo0 + p) * C + c0) =
        *reinterpret_cast<uint4*>(o);
  }
}
// outputs per thread (A/B: CREDO_DW_P = 1, 2 or 4)
const int kDwP = std::getenv("CREDO_DW_P") ? std::atoi(std::getenv("CREDO_DW_P")) : 4;
template <int STRIDE>
void launch_dw3x3(const bf16* in, int B, int H, int C, const float* w, const float* b, bf16* out,
                  cudaStream_t st) {
  const int Ho = (H - 1) / STRIDE + 1;
  auto go = [&](auto kern, int P) {
    const size_t th = (size_t)B * Ho * ((Ho + P - 1) / P) * (C / 8);
    kern<<<grid_for(th), 256, 0, st>>>(in, B, H, C, w, b, out);
  };
  if (kDwP == 1) go(dw3x3_kernel<STRIDE, 1>, 1);
  else if (kDwP == 4) go(dw3x3_kernel<STRIDE, 4>, 4);
  else go(dw3x3_kernel<STRIDE, 2>, 2);
}

int pad64(int c) { return (c + 63) / 64 * 64; }

HostTensor& tensor(std::map<std::string, HostTensor>& T, const std::string& name,
                   std::vector<int64_t> dims) {
  auto it = T.find(name);
  if (it == T.end()) throw std::invalid_argument("cnn file: missing tensor " + name);
  if (!dims.empty() && it->second.dims != dims)
    throw std::invalid_argument("cnn file: bad shape for " + name);
  return it->second;
}

// Per-output-channel scale/shift of an eval BatchNorm (eps 1e-5), or the
// conv/linear bias (bn empty), or zero.
void affine(std::map<std::string, HostTensor>& T, const std::string& bn, const std::string& bias,
            int cout, std::vector<double>& scale, std::vector<double>& shift) {
  scale.assign(cout, 1.0);
  shift.assign(cout, 0.0);
  if (!bn.empty()) {
    const int64_t co = cout;
    auto& g = tensor(T, bn + ".weight", {co});
    auto& be = tensor(T, bn + ".bias", {co});
    auto& mu = tensor(T, bn + ".running_mean", {co});
    auto& var = tensor(T, bn + ".running_var", {co});
    for (int o = 0; o < cout; o++) {
      scale[o] = (double)g.v[o] / std::sqrt((double)var.v[o] + 1e-5);
      shift[o] = (double)be.v[o] - (double)mu.v[o] * scale[o];
    }
  } else if (!bias.empty()) {
    auto& b = tensor(T, bias, {(int64_t)cout});
    for (int o = 0; o < cout; o++) shift[o] = b.v[o];
  }
}

// A conv (k x k) or linear layer (k == 0) as GEMM weights [cout_p][K]:
//   Kim2col > 0 : one tap, K = Kim2col, column (dr*k+ds)*cin + c
//   k == 3      : 9 taps over a padded grid, column tap*cin_p + c
//   k == 1 / 0  : one tap, column c (hwc: linear input in (h, w, c) order
//                 from torch's (c, h, w) flatten, hwc = {C, H, W})
void load_gemm_layer(ConvW& c, std::map<std::string, HostTensor>& T, const std::string& wname,
                     const std::string& bn, const std::string& bias, int k, int stride,
                     int Kim2col, const int* hwc = nullptr, bool pad_out = true) {
  auto it = T.find(wname);
  if (it == T.end()) throw std::invalid_argument("cnn file: missing tensor " + wname);
  const HostTensor& W = it->second;
  const int kk = k == 0 ? 1 : k;
  if ((k == 0 && W.dims.size() != 2) ||
      (k > 0 && (W.dims.size() != 4 || W.dims[2] != k || W.dims[3] != k)))
    throw std::invalid_argument("cnn file: bad layer shape " + wname);
  c.cout = (int)W.dims[0];
  c.cin = (int)W.dims[1];
  c.k = kk;
  c.stride = stride;
  const int cout_p = pad_out ? pad64(c.cout) : c.cout, cin_p = pad64(c.cin);
  c.ntaps = (k == 3 && !Kim2col) ? 9 : 1;
  c.Kc = Kim2col ? Kim2col : cin_p;
  const int Ktot = c.Kc * c.ntaps;
  std::vector<double> sc, sh;
  affine(T, bn, bias, c.cout, sc, sh);
  c.hw.assign((size_t)cout_p * Ktot, 0);
  c.hb.assign(cout_p, 0.f);
  for (int o = 0; o < c.cout; o++) {
    c.hb[o] = (float)sh[o];
    for (int ci = 0; ci < c.cin; ci++)
      for (int dr = 0; dr < kk; dr++)
        for (int ds = 0; ds < kk; ds++) {
          const float w = W.v[(((size_t)o * c.cin + ci) * kk + dr) * kk + ds];
          size_t col;
          if (Kim2col) col = (size_t)(dr * kk + ds) * c.cin + ci;
          else if (c.ntaps == 9) col = (size_t)(dr * 3 + ds) * cin_p + ci;
          else if (hwc) {  // torch flatten index ci = (ch * H + h) * W + w
            const int C = hwc[0], H = hwc[1], Wd = hwc[2];
            const int ch = ci / (H * Wd), r = ci - ch * H * Wd, h = r / Wd, x = r - h * Wd;
            col = ((size_t)h * Wd + x) * C + ch;
          } else col = ci;
          c.hw[(size_t)o * Ktot + col] = f2bf_bits((float)(w * sc[o]));
        }
  }
  c.cout = cout_p;  // the GEMM's N (padded)
}

struct DwW {
  int C = 0, stride = 1;  // C padded
  std::vector<float> hw, hb;
  float *w = nullptr, *b = nullptr;
};

void load_dw(DwW& d, std::map<std::string, HostTensor>& T, const std::string& wname,
             const std::string& bn, int stride) {
  auto& W = tensor(T, wname, {});
  if (W.dims.size() != 4 || W.dims[1] != 1 || W.dims[2] != 3 || W.dims[3] != 3)
    throw std::invalid_argument("cnn file: bad depthwise shape " + wname);
  const int C = (int)W.dims[0];
  d.C = pad64(C);
  d.stride = stride;
  std::vector<double> sc, sh;
  affine(T, bn, "", C, sc, sh);
  d.hw.assign((size_t)9 * d.C, 0.f);
  d.hb.assign(d.C, 0.f);
  for (int c = 0; c < C; c++) {
    d.hb[c] = (float)sh[c];
    for (int tap = 0; tap < 9; tap++) d.hw[(size_t)tap * d.C + c] = (float)(W.v[c * 9 + tap] * sc[c]);
  }
}

// Shared plumbing of the sequential nets: device buffers, the cached launch
// plan per (batch, input, logits), upload of GEMM and depthwise weights.
class SeqNet : public CnnModel {
 public:
  SeqNet(std::string arch, uint64_t in_dim, uint64_t out_dim, bool sm)
      : arch_(std::move(arch)), in_dim_(in_dim), out_dim_(out_dim), softmax_(sm) {
    S_ = (int)std::lround(std::sqrt((double)in_dim / 3.0));
    if ((uint64_t)3 * S_ * S_ != in_dim || S_ % 32 != 0)
      throw std::invalid_argument("cnn file: input_dim must be 3*S*S with S % 32 == 0");
  }
  ~SeqNet() override {
    for (ConvW* c : gemms_) {
      if (c->w) cudaFree(c->w);
      if (c->b) cudaFree(c->b);
    }
    for (DwW* d : dws_) {
      if (d->w) cudaFree(d->w);
      if (d->b) cudaFree(d->b);
    }
    for (void* p : bufs_) cudaFree(p);
  }
  void upload(cudaStream_t st) override {
    for (ConvW* c : gemms_) {
      CG_CUDA(cudaMalloc(&c->w, c->hw.size() * 2));
      CG_CUDA(cudaMalloc(&c->b, c->hb.size() * 4));
      CG_CUDA(cudaMemcpyAsync(c->w, c->hw.data(), c->hw.size() * 2, cudaMemcpyHostToDevice, st));
      CG_CUDA(cudaMemcpyAsync(c->b, c->hb.data(), c->hb.size() * 4, cudaMemcpyHostToDevice, st));
    }
    for (DwW* d : dws_) {
      CG_CUDA(cudaMalloc(&d->w, d->hw.size() * 4));
      CG_CUDA(cudaMalloc(&d->b, d->hb.size() * 4));
      CG_CUDA(cudaMemcpyAsync(d->w, d->hw.data(), d->hw.size() * 4, cudaMemcpyHostToDevice, st));
      CG_CUDA(cudaMemcpyAsync(d->b, d->hb.data(), d->hb.size() * 4, cudaMemcpyHostToDevice, st));
    }
    CG_CUDA(cudaStreamSynchronize(st));
    for (ConvW* c : gemms_) std::vector<uint16_t>().swap(c->hw);
  }
  void reserve(uint32_t maxB) override {
    if (maxB <= maxB_) return;
    for (void* p : bufs_) cudaFree(p);
    bufs_.clear();
    plans_.clear();
    maxB_ = maxB;
    alloc_buffers(maxB);
  }
  size_t prepared_bytes(uint32_t B) const override {
    if (grid16_) return (size_t)B * (S_ + 3) * (S_ + 3) * 32;
    return (size_t)B * rows0_ * 64 * 2;
  }
  std::string prep_kind() const override {
    if (grid16_) return "grid16/" + std::to_string(S_);
    return "im2col3x3s" + std::to_string(stride0_) + "k64/" + std::to_string(S_);
  }
  void prepare_input(const double* d_in, uint32_t B, void* prepped, cudaStream_t st) override {
    if (B > maxB_) reserve(B);
    timer_begin(st, kTimeAux);
    if (grid16_) {
      const size_t px = (size_t)B * (S_ + 3) * (S_ + 3);
      chw_to_grid16_kernel<<<grid_for(px), 256, 0, st>>>(d_in, (int)B, S_,
                                                         reinterpret_cast<uint4*>(prepped));
      CG_CHECK_LAUNCH();
      timer_end(st, kTimeAux);
      return;
    }
    const int Ho = S_ / stride0_;
    if (S_ <= kIm2colMaxS && std::getenv("CREDO_IM2COL_OLD") == nullptr) {
      im2col3x3_f64_rows_kernel<<<(unsigned)(B * Ho), 256, 0, st>>>(
          d_in, (int)B, S_, stride0_, Ho, reinterpret_cast<bf16*>(prepped));
    } else {
      im2col3x3_f64_kernel<<<grid_for((size_t)B * Ho * Ho * 8), 256, 0, st>>>(
          d_in, (int)B, S_, stride0_, Ho, reinterpret_cast<bf16*>(prepped));
    }
    CG_CHECK_LAUNCH();
    timer_end(st, kTimeAux);
  }
  void forward(const double* d_in, uint32_t B, float* logits, cudaStream_t st,
               const void* prepped) override {
    if (B > maxB_) reserve(B);
    const void* x0 = prepped;
    if (!x0) {
      prepare_input(d_in, B, xcol_, st);
      x0 = xcol_;
    }
    auto it = plans_.find(B);
    if (it == plans_.end() || it->second.x0 != x0 || it->second.logits != logits) {
      Plan& p = plans_[B];
      p = Plan{};
      p.x0 = x0;
      p.logits = logits;
      for (ResNet::Op& o : ops(B, reinterpret_cast<const bf16*>(x0), logits)) {
        if (o.gemm) p.steps.push_back(ResNet::make_gemm_step({&o.g}));
        else p.steps.push_back(std::move(o.aux));
      }
      it = plans_.find(B);
    }
    for (auto& s : it->second.steps) s(st);
  }
  uint64_t input_dim() const override { return in_dim_; }
  uint64_t output_dim() const override { return out_dim_; }
  bool softmax() const override { return softmax_; }
  std::string arch() const override { return arch_; }
  double flops_per_image() const override { return flops_; }

 protected:
  struct Plan {
    const void* x0 = nullptr;
    float* logits = nullptr;
    std::vector<std::function<void(cudaStream_t)>> steps;
  };
  virtual void alloc_buffers(uint32_t B) = 0;
  virtual std::vector<ResNet::Op> ops(uint32_t B, const bf16* x0, float* logits) = 0;

  bf16* alloc(size_t elems) {
    void* p = nullptr;
    CG_CUDA(cudaMalloc(&p, std::max<size_t>(elems, 8) * 2));
    CG_CUDA(cudaMemset(p, 0, std::max<size_t>(elems, 8) * 2));
    bufs_.push_back(p);
    return reinterpret_cast<bf16*>(p);
  }
  static void push_gemm(std::vector<ResNet::Op>& L, ConvW& c, const bf16* A, int rowsA, int M,
                        const int* taps, const bf16* res, int ldres, void* out, int ldout,
                        int out_f32, int act, int mode, int H, int rows_out) {
    ResNet::Op o;
    o.gemm = true;
    ResNet::GemmDesc& g = o.g;
    g.c = &c;
    g.A = A;
    g.rowsA = rowsA;
    g.M = M;
    g.Kc = c.Kc;
    g.ntaps = c.ntaps;
    for (int t = 0; t < c.ntaps && t < 9; t++) g.taps[t] = taps ? taps[t] : 0;  // s2d: 16, implicit
    g.res = res;
    g.ldres = ldres;
    g.out = out;
    g.ldout = ldout;
    g.out_f32 = out_f32;
    g.relu = act;
    g.mode = mode;
    g.H = H;
    g.rows_out = rows_out;
    L.push_back(std::move(o));
  }
  static void push_aux(std::vector<ResNet::Op>& L, std::function<void(cudaStream_t)> f) {
    ResNet::Op o;
    o.aux = [f](cudaStream_t st) {
      timer_begin(st, kTimeAux);
      f(st);
      timer_end(st, kTimeAux);
    };
    L.push_back(std::move(o));
  }

  std::string arch_;
  uint64_t in_dim_, out_dim_;
  bool softmax_;
  int S_ = 224, stride0_ = 1;
  size_t rows0_ = 0;  // conv0 output pixels per image
  bool grid16_ = false;  // conv0 as the s2d-mode GEMM over a 16-channel grid (VGG-16)
  double flops_ = 0;
  std::vector<ConvW*> gemms_;
  std::vector<DwW*> dws_;
  uint32_t maxB_ = 0;
  std::vector<void*> bufs_;
  bf16* xcol_ = nullptr;
  std::map<uint32_t, Plan> plans_;
};

// torchvision vgg16 (no BN): 13 3x3 convs (ReLU) in 5 stages with 2x2 max
// pools, then 3 linear layers. conv0 from an im2col of the input; every
// other 3x3 conv runs 9 row-shifted taps over a zero-bordered grid written
// in place by its producer (PadToPad) or by the pool kernel.
class Vgg16 final : public SeqNet {
 public:
  Vgg16(uint64_t in_dim, uint64_t out_dim, bool sm, std::map<std::string, HostTensor>& T)
      : SeqNet("vgg16", in_dim, out_dim, sm) {
    const int cfg[] = {64, 64, 0, 128, 128, 0, 256, 256, 256, 0, 512, 512, 512, 0,
                       512, 512, 512, 0};
    int idx = 0, H = S_, cin = 3;
    for (int v : cfg) {
      if (v == 0) {
        pool_after_.back() = true;
        H /= 2;
        idx += 1;
        continue;
      }
      convs_.emplace_back();
      ConvW& c = convs_.back();
      const std::string pre = "features." + std::to_string(idx);
      load_gemm_layer(c, T, pre + ".weight", "", pre + ".bias", 3, 1, convs_.size() == 1 ? 64 : 0);
      if (c.cin != cin) throw std::invalid_argument("cnn file: unexpected vgg16 shapes");
      flops_ += 2.0 * H * H * 9.0 * cin * v;
      Hs_.push_back(H);
      pool_after_.push_back(false);
      cin = v;
      idx += 2;
    }
    H_last_ = H;
    const int hwc[3] = {cin, H, H};
    const int fc_in = cin * H * H;
    load_gemm_layer(fc_[0], T, "classifier.0.weight", "", "classifier.0.bias", 0, 1, 0, hwc);
    load_gemm_layer(fc_[1], T, "classifier.3.weight", "", "classifier.3.bias", 0, 1, 0);
    load_gemm_layer(fc_[2], T, "classifier.6.weight", "", "classifier.6.bias", 0, 1, 0, nullptr,
                    false);
    if (fc_[0].cin != fc_in || fc_[2].cout != (int)out_dim)
      throw std::invalid_argument("cnn file: unexpected vgg16 classifier shapes");
    flops_ += 2.0 * ((double)fc_in * 4096 + 4096.0 * 4096 + 4096.0 * out_dim);
    for (auto& c : convs_) gemms_.push_back(&c);
    for (auto& c : fc_) gemms_.push_back(&c);
    stride0_ = 1;
    rows0_ = (size_t)S_ * S_;
    // conv1_1 as a 4x4 s2d-mode GEMM over the 16-channel grid: tap (dy, dx)
    // = kernel position (dr, ds) = (dy, dx) for dy, dx < 3, zero otherwise;
    // [tap][cout][16] like the ResNet stem's resident weight tile
    ConvW& c0 = convs_[0];
    grid16_ = kVggGrid16 && S_ + 3 <= 4096 && c0.cout == 64;
    if (grid16_) {
      std::vector<uint16_t> w((size_t)16 * 64 * 16, 0);
      for (int o = 0; o < 64; o++)
        for (int dr = 0; dr < 3; dr++)
          for (int ds = 0; ds < 3; ds++)
            for (int ci = 0; ci < 3; ci++)
              w[((size_t)(dr * 4 + ds) * 64 + o) * 16 + ci] =
                  c0.hw[(size_t)o * c0.Kc + (dr * 3 + ds) * 3 + ci];
      c0.hw.swap(w);
      c0.Kc = 16;
      c0.ntaps = 16;
    }
  }

 protected:
  void alloc_buffers(uint32_t B) override {
    xcol_ = alloc((size_t)B * rows0_ * 64);
    pads_.assign(convs_.size(), nullptr);
    compact_.assign(convs_.size(), nullptr);
    for (size_t i = 0; i < convs_.size(); i++) {
      const size_t H = Hs_[i], C = convs_[i].cout, Hp = H + 2;
      // output grid of conv i: padded (consumed by conv i+1) or compact (pool)
      if (pool_after_[i]) compact_[i] = alloc((size_t)B * H * H * C);
      else pads_[i] = alloc((size_t)B * Hp * Hp * C);
    }
    // pool outputs feed the next conv's padded grid (or the classifier)
    pool_out_.assign(convs_.size(), nullptr);
    for (size_t i = 0; i < convs_.size(); i++)
      if (pool_after_[i]) {
        const size_t Ho = Hs_[i] / 2, C = convs_[i].cout;
        pool_out_[i] = alloc(i + 1 < convs_.size() ? (size_t)B * (Ho + 2) * (Ho + 2) * C
                                                   : (size_t)B * Ho * Ho * C);
      }
    fcbuf_[0] = alloc((size_t)B * 4096);
    fcbuf_[1] = alloc((size_t)B * 4096);
  }
  std::vector<ResNet::Op> ops(uint32_t B, const bf16* x0, float* logits) override {
    std::vector<ResNet::Op> L;
    const int b = (int)B;
    const bf16* in = x0;  // conv0: im2col rows; later: a padded grid
    for (size_t i = 0; i < convs_.size(); i++) {
      ConvW& c = convs_[i];
      const int H = Hs_[i], G = H + 1, rows_pad = b * G * G;  // shared-border grid
      void* out = pool_after_[i] ? (void*)compact_[i] : (void*)pads_[i];
      if (i == 0 && grid16_) {
        // the s2d-mode GEMM over the 16-channel grid, rows remapped into
        // conv1_2's shared-border grid (or compact rows before a pool)
        const int Gg = H + 3;
        push_gemm(L, c, in, b * Gg * Gg, b * Gg * Gg, nullptr, nullptr, 0, out, c.cout, 0, 1,
                  pool_after_[i] ? kRowGridToCompact : kRowGridToPad, H, b * H * H);
        L.back().g.Kc = 16;
        L.back().g.ntaps = 16;
        L.back().g.s2d = 1;
        L.back().g.s2d_step = 1;
        L.back().g.s2d_ndy = 3;  // the 3x3's fourth kernel row is all zero: skipped
        L.back().g.gh = L.back().g.gw = Gg;
      } else if (i == 0) {
        push_gemm(L, c, in, b * H * H, b * H * H, nullptr, nullptr, 0, out, c.cout, 0, 1,
                  pool_after_[i] ? kRowIdentity : kRowCompactToPad, H, b * H * H);
      } else {
        int taps[9];
        for (int dr = 0; dr < 3; dr++)
          for (int ds = 0; ds < 3; ds++) taps[dr * 3 + ds] = (dr - 1) * G + (ds - 1);
        push_gemm(L, c, in, rows_pad, rows_pad, taps, nullptr, 0, out, c.cout, 0, 1,
                  pool_after_[i] ? kRowPadToCompact : kRowPadToPad, H, b * H * H);
        // wider than one halo box: stacked boxes (make_gemm_step checks a
        // kernel variant fits, else the taps stream)
        if (kUseHalo && 128 + 2 * (G + 1) <= kWideHaloRows) L.back().g.halo_lo = G + 1;
      }
      if (pool_after_[i]) {
        const bf16* src = compact_[i];
        bf16* dst = pool_out_[i];
        const int C = c.cout, padded = i + 1 < convs_.size();
        push_aux(L, [src, dst, b, H, C, padded](cudaStream_t st) {
          size_t th = (size_t)b * (H / 2) * (H / 2) * (C / 8);
          maxpool2x2_kernel<<<grid_for(th), 256, 0, st>>>(src, b, H, C, padded, dst);
          CG_CHECK_LAUNCH();
        });
        in = dst;
      } else {
        in = pads_[i];
      }
    }
    // classifier: (h, w, c) flatten matches the permuted fc0 columns
    push_gemm(L, fc_[0], in, b, b, nullptr, nullptr, 0, fcbuf_[0], 4096, 0, 1, kRowIdentity, 0, b);
    push_gemm(L, fc_[1], fcbuf_[0], b, b, nullptr, nullptr, 0, fcbuf_[1], 4096, 0, 1,
              kRowIdentity, 0, b);
    push_gemm(L, fc_[2], fcbuf_[1], b, b, nullptr, nullptr, 0, logits, (int)out_dim_, 1, 0,
              kRowIdentity, 0, b);
    return L;
  }

 private:
  std::vector<ConvW> convs_;
  std::vector<int> Hs_;
  std::vector<bool> pool_after_;
  ConvW fc_[3];
  int H_last_ = 7;
  std::vector<bf16*> pads_, compact_, pool_out_;
  bf16* fcbuf_[2] = {nullptr, nullptr};
};

// torchvision mobilenet_v2: conv0 3x3/2 (ReLU6), 17 inverted residual
// blocks (1x1 expand ReLU6 -> depthwise 3x3 ReLU6 -> 1x1 linear project,
// + identity when stride 1 and cin == cout), 1x1 to 1280 (ReLU6), global
// average pool, linear. Expand/project/head are GEMMs (residual fused into
// the project epilogue); the depthwise conv is a CUDA-core NHWC kernel.
class MobileNetV2 final : public SeqNet {
 public:
  MobileNetV2(uint64_t in_dim, uint64_t out_dim, bool sm, std::map<std::string, HostTensor>& T)
      : SeqNet("mobilenet_v2", in_dim, out_dim, sm) {
    stride0_ = 2;
    int H = S_ / 2;
    rows0_ = (size_t)H * H;
    load_gemm_layer(conv0_, T, "features.0.0.weight", "features.0.1", "", 3, 2, 64);
    flops_ += 2.0 * H * H * 27 * 32;
    const int setting[7][4] = {{1, 16, 1, 1}, {6, 24, 2, 2}, {6, 32, 3, 2}, {6, 64, 4, 2},
                               {6, 96, 3, 1}, {6, 160, 3, 2}, {6, 320, 1, 1}};
    int cin = 32, f = 1;
    blocks_.reserve(17);
    for (auto& s : setting)
      for (int i = 0; i < s[2]; i++, f++) {
        blocks_.emplace_back();
        Blk& b = blocks_.back();
        const int stride = i == 0 ? s[3] : 1, hidden = cin * s[0];
        const std::string pre = "features." + std::to_string(f) + ".conv.";
        b.expand = s[0] != 1;
        int k = 0;
        if (b.expand) {
          load_gemm_layer(b.pw1, T, pre + "0.0.weight", pre + "0.1", "", 1, 1, 0);
          flops_ += 2.0 * H * H * cin * hidden;
          k = 1;
        }
        load_dw(b.dw, T, pre + std::to_string(k) + ".0.weight", pre + std::to_string(k) + ".1",
                stride);
        const int Ho = (H - 1) / stride + 1;
        flops_ += 2.0 * Ho * Ho * 9 * hidden;
        load_gemm_layer(b.pw2, T, pre + std::to_string(k + 1) + ".weight",
                        pre + std::to_string(k + 2), "", 1, 1, 0);
        flops_ += 2.0 * Ho * Ho * hidden * s[1];
        b.H = H;
        b.Ho = Ho;
        b.cin = pad64(cin);
        b.hidden = pad64(hidden);
        b.cout = pad64(s[1]);
        b.residual = stride == 1 && cin == s[1];
        if (b.dw.C != b.hidden || b.pw2.cout != b.cout)
          throw std::invalid_argument("cnn file: unexpected mobilenet_v2 shapes at " + pre);
        cin = s[1];
        H = Ho;
      }
    load_gemm_layer(head_, T, "features.18.0.weight", "features.18.1", "", 1, 1, 0);
    flops_ += 2.0 * H * H * cin * 1280;
    load_gemm_layer(fc_, T, "classifier.1.weight", "", "classifier.1.bias", 0, 1, 0, nullptr,
                    false);
    if (fc_.cout != (int)out_dim) throw std::invalid_argument("cnn file: bad classifier");
    flops_ += 2.0 * 1280.0 * out_dim;
    H_last_ = H;
    gemms_.push_back(&conv0_);
    for (auto& b : blocks_) {
      if (b.expand) gemms_.push_back(&b.pw1);
      gemms_.push_back(&b.pw2);
      dws_.push_back(&b.dw);
    }
    gemms_.push_back(&head_);
    gemms_.push_back(&fc_);
  }

 protected:
  void alloc_buffers(uint32_t B) override {
    xcol_ = alloc((size_t)B * rows0_ * 64);
    size_t act = (size_t)B * rows0_ * conv0_.cout, hid = 0;
    for (auto& b : blocks_) {
      act = std::max(act, (size_t)B * b.Ho * b.Ho * b.cout);
      hid = std::max(hid, (size_t)B * b.H * b.H * b.hidden);
    }
    act_[0] = alloc(act);
    act_[1] = alloc(act);
    e_ = alloc(hid);
    d_ = alloc(hid);
    head_out_ = alloc((size_t)B * H_last_ * H_last_ * 1280);
    pooled_ = alloc((size_t)B * 1280);
  }
  std::vector<ResNet::Op> ops(uint32_t B, const bf16* x0, float* logits) override {
    std::vector<ResNet::Op> L;
    const int b = (int)B;
    const int H0 = S_ / 2;
    push_gemm(L, conv0_, x0, b * H0 * H0, b * H0 * H0, nullptr, nullptr, 0, act_[0],
              conv0_.cout, 0, 2, kRowIdentity, 0, b * H0 * H0);
    int cur = 0;
    for (auto& k : blocks_) {
      bf16* X = act_[cur];
      bf16* Y = act_[cur ^ 1];
      const bf16* dwin = X;
      if (k.expand) {
        push_gemm(L, k.pw1, X, b * k.H * k.H, b * k.H * k.H, nullptr, nullptr, 0, e_, k.hidden,
                  0, 2, kRowIdentity, 0, b * k.H * k.H);
        dwin = e_;
      }
      {
        const DwW* dw = &k.dw;
        bf16* D = d_;
        const int H = k.H, C = k.hidden, s = k.dw.stride, Ho = k.Ho;
        push_aux(L, [dwin, dw, D, b, H, C, s](cudaStream_t st) {
          if (s == 1) launch_dw3x3<1>(dwin, b, H, C, dw->w, dw->b, D, st);
          else launch_dw3x3<2>(dwin, b, H, C, dw->w, dw->b, D, st);
          CG_CHECK_LAUNCH();
        });
      }
      push_gemm(L, k.pw2, d_, b * k.Ho * k.Ho, b * k.Ho * k.Ho, nullptr,
                k.residual ? X : nullptr, k.residual ? k.cout : 0, Y, k.cout, 0, 0,
                kRowIdentity, 0, b * k.Ho * k.Ho);
      cur ^= 1;
    }
    const int HW = H_last_ * H_last_;
    push_gemm(L, head_, act_[cur], b * HW, b * HW, nullptr, nullptr, 0, head_out_, 1280, 0, 2,
              kRowIdentity, 0, b * HW);
    {
      bf16* in = head_out_;
      bf16* out = pooled_;
      push_aux(L, [in, out, b, HW](cudaStream_t st) {
        avgpool_kernel<<<(unsigned)(b * (1280 / 256)), 256, 0, st>>>(in, b, HW, 1280, out);
        CG_CHECK_LAUNCH();
      });
    }
    push_gemm(L, fc_, pooled_, b, b, nullptr, nullptr, 0, logits, (int)out_dim_, 1, 0,
              kRowIdentity, 0, b);
    return L;
  }

 private:
  struct Blk {
    ConvW pw1, pw2;
    DwW dw;
    bool expand = false, residual = false;
    int H = 0, Ho = 0, cin = 0, hidden = 0, cout = 0;
  };
  ConvW conv0_, head_, fc_;
  std::vector<Blk> blocks_;
  int H_last_ = 7;
  bf16 *act_[2] = {nullptr, nullptr}, *e_ = nullptr, *d_ = nullptr, *head_out_ = nullptr,
       *pooled_ = nullptr;
};

class ResNetGroupPlan final : public CnnGroupPlan {
 public:
  uint32_t B = 0;
  std::vector<std::function<void(cudaStream_t)>> steps;
  void run(cudaStream_t st) override {
    for (auto& f : steps) f(st);
  }
  uint32_t batch() const override { return B; }
};

}  // namespace

std::unique_ptr<CnnGroupPlan> CnnGroupPlan::build(const std::vector<CnnModel*>& models,
                                                  uint32_t B, const void* prepped,
                                                  const std::vector<float*>& logits) {
  if (models.size() < 2 || models.size() > (size_t)kMaxGroup) return nullptr;
  std::vector<ResNet*> rs;
  for (CnnModel* m : models) {
    auto* r = dynamic_cast<ResNet*>(m);
    if (!r) return nullptr;
    rs.push_back(r);
  }
  for (ResNet* r : rs)
    if (r->arch() != rs[0]->arch() || r->image_size() != rs[0]->image_size() ||
        r->num_blocks() != rs[0]->num_blocks() || r->output_dim() != rs[0]->output_dim())
      return nullptr;
  std::vector<std::vector<ResNet::Op>> ops;
  for (size_t i = 0; i < rs.size(); i++) {
    rs[i]->reserve(B);
    ops.push_back(rs[i]->ops(B, prepped, logits[i]));
  }
  auto plan = std::make_unique<ResNetGroupPlan>();
  plan->B = B;
  for (size_t k = 0; k < ops[0].size(); k++) {
    if (ops[0][k].gemm) {
      std::vector<const ResNet::GemmDesc*> ds;
      for (auto& o : ops) ds.push_back(&o[k].g);
      plan->steps.push_back(ResNet::make_gemm_step(ds));
    } else {
      std::vector<std::function<void(cudaStream_t)>> fs;
      for (auto& o : ops) fs.push_back(o[k].aux);
      plan->steps.push_back([fs](cudaStream_t st) {
        for (auto& f : fs) f(st);
      });
    }
  }
  return plan;
}

std::unique_ptr<CnnModel> CnnModel::from_file(const uint8_t* file, uint64_t len) {
  Reader r{file, len};
  if (r.str() != "credo.cnn.v1") throw std::invalid_argument("cnn file: bad magic");
  std::string arch = r.str();
  uint64_t in_dim = r.u64(), out_dim = r.u64();
  r.need(1);
  uint8_t sm = file[r.pos++];
  if (sm > 1) throw std::invalid_argument("cnn file: invalid boolean");
  uint32_t n = r.u32();
  std::map<std::string, HostTensor> T;
  for (uint32_t i = 0; i < n; i++) {
    std::string name = r.str();
    HostTensor t;
    uint32_t nd = r.u32();
    if (nd > 8) throw std::invalid_argument("cnn file: too many dims");
    uint64_t count = 1;
    for (uint32_t d = 0; d < nd; d++) {
      t.dims.push_back((int64_t)r.u64());
      count *= (uint64_t)t.dims.back();
    }
    uint32_t c = r.u32();
    if (c != count) throw std::invalid_argument("cnn file: count/shape mismatch");
    r.need(4ull * c);
    t.v.resize(c);
    const uint8_t* src = file + r.pos;  // f32 big-endian, bounds checked above
    for (uint32_t k = 0; k < c; k++) {
      uint32_t b;
      std::memcpy(&b, src + 4ull * k, 4);
      b = __builtin_bswap32(b);
      std::memcpy(&t.v[k], &b, 4);
    }
    r.pos += 4ull * c;
    T[name] = std::move(t);
  }
  if (r.pos != len) throw std::invalid_argument("cnn file: trailing bytes after value");
  std::vector<int> layers;
  if (arch == "resnet50") layers = {3, 4, 6, 3};
  else if (arch == "resnet101") layers = {3, 4, 23, 3};
  else if (arch == "resnet152") layers = {3, 8, 36, 3};
  else if (arch == "vgg16") return std::make_unique<Vgg16>(in_dim, out_dim, sm == 1, T);
  else if (arch == "mobilenet_v2")
    return std::make_unique<MobileNetV2>(in_dim, out_dim, sm == 1, T);
  else throw std::invalid_argument("cnn file: unsupported arch " + arch);
  return std::make_unique<ResNet>(arch, layers, in_dim, out_dim, sm == 1, T);
}

}  // namespace cg
