// SHA-256 on sm_100a: the compression function and the "segmented message"
// chain engine used for every certificate digest.
//
// Reference semantics: crypto::hash / hash_concat (reference
// proj/src/crypto.cpp:22-39, libsodium SHA-256) and merkle::leaf_hash /
// internal_hash (proj/src/merkle.cpp:14-25). A certificate leaf such as
// result_leaf (proj/src/messages.cpp:204-211) is never materialised: the
// canonical big-endian bytes (proj/include/credo/codec.hpp:28-84) are
// streamed straight out of the request's f64 input tensor and the replica's
// f64 output tensor, with the few framing bytes (ids, lengths, keys, nonce,
// signature) coming from a small host-built arena.
#pragma once
#include <stdint.h>

#include "common.cuh"

namespace cg {

// One contiguous piece of a message. kind == kSegRaw: `len` raw bytes at
// device address `ptr`. kind == kSegF64: the canonical big-endian encoding
// of len/8 doubles stored natively (little-endian) at `ptr`.
enum : uint32_t { kSegRaw = 0, kSegF64 = 1 };
constexpr int kMaxSegs = 8;

struct ChainSeg {
  uint64_t ptr;
  uint64_t msg_off;  // absolute offset of the segment inside the message
  uint64_t len;
  uint32_t kind;
  uint32_t pad_;
};

// A run of SHA-256 compressions over blocks [blk_begin, blk_end) of one
// message. Non-final jobs store the chaining value (a midstate shared by all
// providers of a request); final jobs append the FIPS 180-4 padding, so
// blk_end = ceil((total_len + 9) / 64), and write the 32-byte digest.
struct ChainJob {
  ChainSeg seg[kMaxSegs];
  uint32_t nseg;
  uint32_t final_;
  uint64_t total_len;
  uint64_t blk_begin, blk_end;
  uint64_t state_in;    // device uint32[8] or 0 for the IV
  uint64_t state_out;   // device uint32[8] or 0
  uint64_t digest_out;  // device uint8[32] or 0
  uint64_t skip_flag;   // device int32*: skip when < 0, else digest slot
};

__device__ __forceinline__ uint32_t rotr32(uint32_t x, int n) {
  return __funnelshift_r(x, x, n);
}
__device__ __forceinline__ uint32_t bswap32(uint32_t x) {
  return __byte_perm(x, 0, 0x0123);
}

__device__ __forceinline__ void sha256_iv(uint32_t s[8]) {
  s[0] = 0x6a09e667u; s[1] = 0xbb67ae85u; s[2] = 0x3c6ef372u;
  s[3] = 0xa54ff53au; s[4] = 0x510e527fu; s[5] = 0x9b05688cu;
  s[6] = 0x1f83d9abu; s[7] = 0x5be0cd19u;
}

static __constant__ uint32_t kSha256K[64] = {
    0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u,
    0x923f82a4u, 0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u,
    0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u,
    0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
    0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u,
    0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u,
    0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
    0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
    0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au,
    0x5b9cca4fu, 0x682e6ff3u, 0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u,
    0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};

// Measured on B200 (tools/shabench.py): a round is ALU-pipe bound (~21
// SHF/LOP3/IADD3 at half rate per SMSP = ~42 cycles). Moving the additions,
// shifts or a rotation onto the FMA pipe as IMADs made it slower (longer
// dependent chains), so rounds stay on the ALU pipe.
// One FIPS 180-4 round; i is the round index within its 16-round group so
// the rolling 16-word schedule window indices are compile-time constants.
template <int i, bool kSched>
__device__ __forceinline__ void sha256_round(uint32_t& a, uint32_t& b, uint32_t& c,
                                             uint32_t& d, uint32_t& e, uint32_t& f,
                                             uint32_t& g, uint32_t& h, uint32_t w[16],
                                             uint32_t k) {
  if (kSched) {
    uint32_t x = w[(i + 1) & 15], y = w[(i + 14) & 15];
    uint32_t s0 = rotr32(x, 7) ^ rotr32(x, 18) ^ (x >> 3);
    uint32_t s1 = rotr32(y, 17) ^ rotr32(y, 19) ^ (y >> 10);
    w[i & 15] += s0 + w[(i + 9) & 15] + s1;
  }
  const uint32_t S1 = rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25);
  const uint32_t ch = (e & f) ^ (~e & g);
  const uint32_t S0 = rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22);
  const uint32_t maj = (a & b) | (c & (a | b));
  const uint32_t t1 = h + S1 + ch + k + w[i & 15];
  h = g; g = f; f = e; e = d + t1;
  d = c; c = b; b = a; a = t1 + S0 + maj;
}

#define CG_SHA_R(n) \
  sha256_round<n, kSched>(a, b, c, d, e, f, g, h, w, kSha256K[r + n]);
template <bool kSched>
__device__ __forceinline__ void sha256_16rounds(uint32_t& a, uint32_t& b, uint32_t& c,
                                                uint32_t& d, uint32_t& e, uint32_t& f,
                                                uint32_t& g, uint32_t& h, uint32_t w[16],
                                                int r) {
  CG_SHA_R(0) CG_SHA_R(1) CG_SHA_R(2) CG_SHA_R(3) CG_SHA_R(4) CG_SHA_R(5)
  CG_SHA_R(6) CG_SHA_R(7) CG_SHA_R(8) CG_SHA_R(9) CG_SHA_R(10) CG_SHA_R(11)
  CG_SHA_R(12) CG_SHA_R(13) CG_SHA_R(14) CG_SHA_R(15)
}
#undef CG_SHA_R

// FIPS 180-4 compression of one block into s. kRolled == false: all 64
// rounds unrolled with immediate constants (~1.5k instructions; used by the
// short digests). kRolled == true: rounds 16-63 as a 3-trip loop over one
// 16-round body with K from constant memory (~1/3 the code, so a chain loop
// stays resident in the SMSP's instruction cache).
template <bool kRolled = false>
__device__ __forceinline__ void sha256_compress(uint32_t s[8], uint32_t w[16]) {
  uint32_t a = s[0], b = s[1], c = s[2], d = s[3];
  uint32_t e = s[4], f = s[5], g = s[6], h = s[7];
  if (!kRolled) {
    constexpr uint32_t KI[64] = {
        0x428a2f98u, 0x71374491u, 0xb5c0fbcfu, 0xe9b5dba5u, 0x3956c25bu, 0x59f111f1u,
        0x923f82a4u, 0xab1c5ed5u, 0xd807aa98u, 0x12835b01u, 0x243185beu, 0x550c7dc3u,
        0x72be5d74u, 0x80deb1feu, 0x9bdc06a7u, 0xc19bf174u, 0xe49b69c1u, 0xefbe4786u,
        0x0fc19dc6u, 0x240ca1ccu, 0x2de92c6fu, 0x4a7484aau, 0x5cb0a9dcu, 0x76f988dau,
        0x983e5152u, 0xa831c66du, 0xb00327c8u, 0xbf597fc7u, 0xc6e00bf3u, 0xd5a79147u,
        0x06ca6351u, 0x14292967u, 0x27b70a85u, 0x2e1b2138u, 0x4d2c6dfcu, 0x53380d13u,
        0x650a7354u, 0x766a0abbu, 0x81c2c92eu, 0x92722c85u, 0xa2bfe8a1u, 0xa81a664bu,
        0xc24b8b70u, 0xc76c51a3u, 0xd192e819u, 0xd6990624u, 0xf40e3585u, 0x106aa070u,
        0x19a4c116u, 0x1e376c08u, 0x2748774cu, 0x34b0bcb5u, 0x391c0cb3u, 0x4ed8aa4au,
        0x5b9cca4fu, 0x682e6ff3u, 0x748f82eeu, 0x78a5636fu, 0x84c87814u, 0x8cc70208u,
        0x90befffau, 0xa4506cebu, 0xbef9a3f7u, 0xc67178f2u};
#pragma unroll
    for (int i = 0; i < 64; i++) {
      if (i >= 16) {
        uint32_t x = w[(i - 15) & 15], y = w[(i - 2) & 15];
        uint32_t s0 = rotr32(x, 7) ^ rotr32(x, 18) ^ (x >> 3);
        uint32_t s1 = rotr32(y, 17) ^ rotr32(y, 19) ^ (y >> 10);
        w[i & 15] += s0 + w[(i - 7) & 15] + s1;
      }
      uint32_t t1 = h + (rotr32(e, 6) ^ rotr32(e, 11) ^ rotr32(e, 25)) +
                    ((e & f) ^ (~e & g)) + KI[i] + w[i & 15];
      uint32_t t2 = (rotr32(a, 2) ^ rotr32(a, 13) ^ rotr32(a, 22)) +
                    ((a & b) | (c & (a | b)));
      h = g; g = f; f = e; e = d + t1;
      d = c; c = b; b = a; a = t1 + t2;
    }
  } else {
    sha256_16rounds<false>(a, b, c, d, e, f, g, h, w, 0);
#pragma unroll 1
    for (int r = 16; r < 64; r += 16) sha256_16rounds<true>(a, b, c, d, e, f, g, h, w, r);
  }
  s[0] += a; s[1] += b; s[2] += c; s[3] += d;
  s[4] += e; s[5] += f; s[6] += g; s[7] += h;
}

__device__ __forceinline__ void store_digest(const uint32_t s[8], uint8_t* out) {
  // out is 4-byte aligned in every caller.
  uint32_t* o = reinterpret_cast<uint32_t*>(out);
#pragma unroll
  for (int i = 0; i < 8; i++) o[i] = bswap32(s[i]);
}

// Big-endian stream word k of an f64 segment: double k/2, high half first.
__device__ __forceinline__ uint32_t f64_stream_word(const double* p, uint64_t k) {
  uint64_t bits = __double_as_longlong(__ldg(p + (k >> 1)));
  return (k & 1) ? (uint32_t)bits : (uint32_t)(bits >> 32);
}

// Byte `pos` of the (padded) message, generic slow path.
__device__ __forceinline__ uint32_t msg_byte(const ChainJob& j, uint64_t pos,
                                             uint64_t nblk_total) {
  if (pos < j.total_len) {
    for (uint32_t s = 0; s < j.nseg; s++) {
      const ChainSeg& g = j.seg[s];
      if (pos >= g.msg_off && pos < g.msg_off + g.len) {
        uint64_t q = pos - g.msg_off;
        if (g.kind == kSegRaw)
          return __ldg(reinterpret_cast<const uint8_t*>(g.ptr) + q);
        uint64_t bits = __double_as_longlong(
            __ldg(reinterpret_cast<const double*>(g.ptr) + (q >> 3)));
        return (uint32_t)(bits >> (56 - 8 * (q & 7))) & 0xffu;
      }
    }
    return 0;  // unreachable for well-formed jobs
  }
  if (pos == j.total_len) return 0x80u;
  uint64_t len_pos = nblk_total * 64 - 8;
  if (pos >= len_pos) {
    uint64_t bits = j.total_len * 8;
    return (uint32_t)(bits >> (56 - 8 * (pos - len_pos))) & 0xffu;
  }
  return 0;
}

// Word at message offset pos (pos % 4 == 0): one load when the word sits
// inside one segment, else byte assembly (segment edges and padding).
__device__ __forceinline__ uint32_t msg_word(const ChainJob& j, uint64_t pos,
                                             uint64_t nblk_total) {
  if (pos + 4 <= j.total_len) {
    for (uint32_t s = 0; s < j.nseg; s++) {
      const ChainSeg& g = j.seg[s];
      if (pos >= g.msg_off && pos + 4 <= g.msg_off + g.len) {
        uint64_t q = pos - g.msg_off;
        if (g.kind == kSegRaw) {
          uint64_t addr = g.ptr + q;
          if ((addr & 3) == 0)
            return bswap32(__ldg(reinterpret_cast<const uint32_t*>(addr)));
          break;
        }
        const double* p = reinterpret_cast<const double*>(g.ptr);
        uint64_t k = q >> 2;
        uint32_t r = (uint32_t)(q & 3);
        uint32_t hi = f64_stream_word(p, k);
        if (r == 0) return hi;
        uint32_t lo = f64_stream_word(p, k + 1);
        return __funnelshift_l(lo, hi, 8 * r);
      }
    }
  }
  uint32_t w = 0;
#pragma unroll
  for (int t = 0; t < 4; t++) w = (w << 8) | msg_byte(j, pos + t, nblk_total);
  return w;
}

__device__ __forceinline__ void load_block_slow(const ChainJob& j, uint64_t blk,
                                                uint64_t nblk_total,
                                                uint32_t w[16]) {
#pragma unroll
  for (int i = 0; i < 16; i++) w[i] = msg_word(j, blk * 64 + 4 * i, nblk_total);
}

// Fast path: a block lying wholly inside one f64 segment. The 64 message
// bytes are 16 big-endian words funnel-shifted out of 9 consecutive doubles
// (8 when the block happens to be 8-byte aligned in the stream).
struct F64Window {
  uint64_t v[9];
};

__device__ __forceinline__ void f64_window_load(const double* base,
                                                uint64_t d0, uint64_t dmax,
                                                F64Window& win) {
#pragma unroll
  for (int t = 0; t < 9; t++) {
    uint64_t d = d0 + t;
    d = d < dmax ? d : dmax;  // clamp: the 9th double may be past the end
    win.v[t] = __double_as_longlong(__ldg(base + d));
  }
}

__device__ __forceinline__ void f64_window_words(const F64Window& win,
                                                 uint32_t o, uint32_t w[16]) {
  // Stream words of the window: S[2t] = hi(v[t]), S[2t+1] = lo(v[t]).
  // Block word i = bytes [o + 4i, o + 4i + 4) of the window, o in [0, 8).
  uint32_t S[18];
#pragma unroll
  for (int t = 0; t < 9; t++) {
    S[2 * t] = (uint32_t)(win.v[t] >> 32);
    S[2 * t + 1] = (uint32_t)win.v[t];
  }
  const uint32_t r8 = 8 * (o & 3);
  if (o >= 4) {
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = __funnelshift_l(S[i + 2], S[i + 1], r8);
  } else {
#pragma unroll
    for (int i = 0; i < 16; i++) w[i] = __funnelshift_l(S[i + 1], S[i], r8);
  }
}

// Runs one job in the calling thread. kLoop selects the fast-run code shape
// (cycles per block on B200, tools/shabench.py): 0 = two unrolled
// compressions per trip (~4.9k: the 48 KB loop misses the SMSP instruction
// cache), 1 = one rolled compression per trip with window rotation (~3.3k,
// default), 2 = one unrolled compression per trip (~3.4k).
#ifndef CG_CHAIN_LOOP
#define CG_CHAIN_LOOP 1
#endif
template <int kLoop = CG_CHAIN_LOOP, bool kRawFast = false>
__device__ __forceinline__ void run_chain_job(const ChainJob& j,
                                              uint64_t digest_out) {
  constexpr bool kRolled = kLoop == 1;
  uint32_t s[8];
  if (j.state_in) {
    const uint32_t* si = reinterpret_cast<const uint32_t*>(j.state_in);
#pragma unroll
    for (int i = 0; i < 8; i++) s[i] = si[i];
  } else {
    sha256_iv(s);
  }
  const uint64_t nblk_total = j.final_ ? (j.total_len + 9 + 63) / 64 : j.blk_end;

  // The fast run: the f64 segment covering the most whole blocks of
  // [blk_begin, blk_end); those blocks skip the generic word assembly.
  uint64_t run_b = j.blk_end, run_e = j.blk_end;
  int fs = -1;
  for (uint32_t t = 0; t < j.nseg; t++) {
    const ChainSeg& g = j.seg[t];
    if (g.kind != kSegF64) continue;
    uint64_t b0 = (g.msg_off + 63) / 64;
    uint64_t b1 = (g.msg_off + g.len) / 64;
    b0 = b0 > j.blk_begin ? b0 : j.blk_begin;
    b1 = b1 < j.blk_end ? b1 : j.blk_end;
    if (b1 > b0 && (fs < 0 || b1 - b0 > run_e - run_b)) {
      fs = (int)t;
      run_b = b0;
      run_e = b1;
    }
  }
  // kRawFast (flat byte messages: cg_sha256_batch, model-file digests): with
  // no f64 segment, the raw segment covering the most whole blocks runs with
  // 16 word loads per block (word-aligned: Arena places a segment at an
  // address congruent to its message offset mod 4), issued one block ahead.
  int rs = -1;
  if (kRawFast && fs < 0) {
    for (uint32_t t = 0; t < j.nseg; t++) {
      const ChainSeg& g = j.seg[t];
      if (g.kind != kSegRaw || ((g.ptr - g.msg_off) & 3)) continue;
      uint64_t b0 = (g.msg_off + 63) / 64;
      uint64_t b1 = (g.msg_off + g.len) / 64;
      b0 = b0 > j.blk_begin ? b0 : j.blk_begin;
      b1 = b1 < j.blk_end ? b1 : j.blk_end;
      if (b1 > b0 && (rs < 0 || b1 - b0 > run_e - run_b)) {
        rs = (int)t;
        run_b = b0;
        run_e = b1;
      }
    }
  }
  uint32_t w[16];
  uint64_t blk = j.blk_begin;
#pragma unroll 1
  for (; blk < run_b; blk++) {
    load_block_slow(j, blk, nblk_total, w);
    sha256_compress<kRolled>(s, w);
  }
  if (kRawFast && rs >= 0) {
    const ChainSeg& g = j.seg[rs];
    const uint32_t* p = reinterpret_cast<const uint32_t*>(g.ptr + run_b * 64 - g.msg_off);
    const uint64_t n = run_e - run_b;
    uint32_t nx[16];
#pragma unroll
    for (int q = 0; q < 16; q++) nx[q] = __ldg(p + q);
#pragma unroll 1
    for (uint64_t i = 0; i < n; i++) {
#pragma unroll
      for (int q = 0; q < 16; q++) w[q] = bswap32(nx[q]);
      if (i + 1 < n) {
#pragma unroll
        for (int q = 0; q < 16; q++) nx[q] = __ldg(p + 16 * (i + 1) + q);
      }
      sha256_compress<kRolled>(s, w);
    }
    blk = run_e;
  } else if (run_e > run_b) {
    const ChainSeg& g = j.seg[fs];
    const double* base = reinterpret_cast<const double*>(g.ptr);
    const uint64_t dmax = g.len / 8 - 1;
    // byte offset of block `blk` inside the stream: q = 64*blk - msg_off
    const uint64_t q0 = run_b * 64 - g.msg_off;
    const uint32_t o = (uint32_t)(q0 & 7);
    uint64_t d = q0 >> 3;  // first double of block run_b
    F64Window A, Bw;
    f64_window_load(base, d, dmax, A);
    f64_window_load(base, d + 8, dmax, Bw);
    uint64_t n = run_e - run_b;
    uint64_t i = 0;
    if (kLoop == 0) {
#pragma unroll 1
      for (; i + 2 <= n; i += 2) {
        f64_window_words(A, o, w);
        f64_window_load(base, d + 8 * (i + 2), dmax, A);
        sha256_compress<kRolled>(s, w);
        f64_window_words(Bw, o, w);
        f64_window_load(base, d + 8 * (i + 3), dmax, Bw);
        sha256_compress<kRolled>(s, w);
      }
      if (i < n) {
        f64_window_words(A, o, w);
        sha256_compress<kRolled>(s, w);
      }
    } else {
#pragma unroll 1
      for (; i < n; i++) {
        f64_window_words(A, o, w);
        A = Bw;
        f64_window_load(base, d + 8 * (i + 2), dmax, Bw);
        sha256_compress<kRolled>(s, w);
      }
    }
    blk = run_e;
  }
#pragma unroll 1
  for (; blk < nblk_total; blk++) {
    load_block_slow(j, blk, nblk_total, w);
    sha256_compress<kRolled>(s, w);
  }
  if (j.state_out) {
    uint32_t* so = reinterpret_cast<uint32_t*>(j.state_out);
#pragma unroll
    for (int i = 0; i < 8; i++) so[i] = s[i];
  }
  if (j.final_ && digest_out) store_digest(s, reinterpret_cast<uint8_t*>(digest_out));
}

// H(0x01 || L || R) for two 32-byte digests (merkle.cpp:14-19): 65 bytes,
// two blocks.
__device__ __forceinline__ void sha256_internal_node(const uint8_t* L,
                                                     const uint8_t* R,
                                                     uint8_t* out) {
  const uint32_t* l = reinterpret_cast<const uint32_t*>(L);
  const uint32_t* r = reinterpret_cast<const uint32_t*>(R);
  uint32_t lw[8], rw[8];
#pragma unroll
  for (int i = 0; i < 8; i++) { lw[i] = bswap32(l[i]); rw[i] = bswap32(r[i]); }
  uint32_t w[16], s[8];
  sha256_iv(s);
  w[0] = 0x01000000u | (lw[0] >> 8);
#pragma unroll
  for (int i = 1; i < 8; i++) w[i] = (lw[i - 1] << 24) | (lw[i] >> 8);
  w[8] = (lw[7] << 24) | (rw[0] >> 8);
#pragma unroll
  for (int i = 9; i < 16; i++) w[i] = (rw[i - 9] << 24) | (rw[i - 8] >> 8);
  sha256_compress(s, w);
  w[0] = (rw[7] << 24) | 0x00800000u;
#pragma unroll
  for (int i = 1; i < 15; i++) w[i] = 0;
  w[15] = 65 * 8;
  sha256_compress(s, w);
  store_digest(s, out);
}

// H(0x00 || tag || d) for a 32-byte digest d (whole-batch A leaf,
// messages.cpp:276-281 under merkle.cpp:22-25): 34 bytes, one block.
__device__ __forceinline__ void sha256_tagged_digest_leaf(uint8_t tag,
                                                          const uint8_t* D,
                                                          uint8_t* out) {
  const uint32_t* dp = reinterpret_cast<const uint32_t*>(D);
  uint32_t dw[8];
#pragma unroll
  for (int i = 0; i < 8; i++) dw[i] = bswap32(dp[i]);
  uint32_t w[16], s[8];
  sha256_iv(s);
  w[0] = ((uint32_t)tag << 16) | (dw[0] >> 16);
#pragma unroll
  for (int i = 1; i < 8; i++) w[i] = (dw[i - 1] << 16) | (dw[i] >> 16);
  w[8] = (dw[7] << 16) | 0x8000u;
#pragma unroll
  for (int i = 9; i < 15; i++) w[i] = 0;
  w[15] = 34 * 8;
  sha256_compress(s, w);
  store_digest(s, out);
}

// Compact agreed-label digest (SURVEY §8(d) C5 "D2"; new, no reference
// equivalent, composed like the reference's leaves from Encoder fields):
// SHA-256(0x4C || request_id[32] || u64be version || u64be label), label -1
// = no agreed label. 49 bytes: one block.
constexpr uint8_t kLabelDigestTag = 0x4C;
__device__ __forceinline__ void sha256_label_digest(const uint8_t* rid, uint64_t version,
                                                    int64_t label, uint8_t* out) {
  const uint32_t* rp = reinterpret_cast<const uint32_t*>(rid);  // 4-byte aligned
  uint32_t r[8];
#pragma unroll
  for (int i = 0; i < 8; i++) r[i] = bswap32(rp[i]);
  const uint32_t vh = (uint32_t)(version >> 32), vl = (uint32_t)version;
  const uint64_t lu = (uint64_t)label;
  const uint32_t lh = (uint32_t)(lu >> 32), ll = (uint32_t)lu;
  uint32_t w[16], s[8];
  sha256_iv(s);
  w[0] = ((uint32_t)kLabelDigestTag << 24) | (r[0] >> 8);
#pragma unroll
  for (int i = 1; i < 8; i++) w[i] = (r[i - 1] << 24) | (r[i] >> 8);
  w[8] = (r[7] << 24) | (vh >> 8);
  w[9] = (vh << 24) | (vl >> 8);
  w[10] = (vl << 24) | (lh >> 8);
  w[11] = (lh << 24) | (ll >> 8);
  w[12] = (ll << 24) | 0x00800000u;
  w[13] = 0;
  w[14] = 0;
  w[15] = 49 * 8;
  sha256_compress(s, w);
  store_digest(s, out);
}

}  // namespace cg
