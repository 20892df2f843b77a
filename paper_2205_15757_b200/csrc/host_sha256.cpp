// Host SHA-256 for the digests the reference computes on the host and that
// are single sequential chains too long for one GPU thread:
//   * the model-file check of InferenceEngine::load_group (proj/src/
//     engine.cpp:79): SHA-256 over a ~100 MB CNN file;
//   * hash_ops (proj/src/messages.cpp:197-202): H(0x4F || list(OpEntry)) over
//     a PRE-PREPARE's ops, which embed every request encoding (1.2 MB each at
//     ImageNet shape): one 154 MB chain per 128-request slot.
// Compression uses the x86 SHA extensions (SHA-NI) when the CPU has them,
// else a portable scalar round function (same digests). The f64 request
// inputs are streamed big-endian through a small staging buffer, so no
// request encoding is ever materialised.
#include <immintrin.h>
#include <cpuid.h>

#include <algorithm>
#include <atomic>
#include <cstring>
#include <stdexcept>
#include <string>
#include <thread>
#include <vector>

#include "../../include/credo_gpu.h"
#include "host_sha256.h"

namespace cg {
namespace {

const uint32_t kK[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1, 0x923f82a4,
    0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3, 0x72be5d74, 0x80deb1fe,
    0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786, 0x0fc19dc6, 0x240ca1cc, 0x2de92c6f,
    0x4a7484aa, 0x5cb0a9dc, 0x76f988da, 0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7,
    0xc6e00bf3, 0xd5a79147, 0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc,
    0x53380d13, 0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070, 0x19a4c116,
    0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a, 0x5b9cca4f, 0x682e6ff3,
    0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208, 0x90befffa, 0xa4506ceb, 0xbef9a3f7,
    0xc67178f2};

inline uint32_t rotr(uint32_t x, int n) { return (x >> n) | (x << (32 - n)); }

void compress_scalar(uint32_t st[8], const uint8_t* p, size_t nblocks) {
  for (; nblocks; nblocks--, p += 64) {
    uint32_t w[64];
    for (int i = 0; i < 16; i++)
      w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 |
             (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
    for (int i = 16; i < 64; i++) {
      const uint32_t s0 = rotr(w[i - 15], 7) ^ rotr(w[i - 15], 18) ^ (w[i - 15] >> 3);
      const uint32_t s1 = rotr(w[i - 2], 17) ^ rotr(w[i - 2], 19) ^ (w[i - 2] >> 10);
      w[i] = w[i - 16] + s0 + w[i - 7] + s1;
    }
    uint32_t a = st[0], b = st[1], c = st[2], d = st[3], e = st[4], f = st[5], g = st[6],
             h = st[7];
    for (int i = 0; i < 64; i++) {
      const uint32_t t1 = h + (rotr(e, 6) ^ rotr(e, 11) ^ rotr(e, 25)) + ((e & f) ^ (~e & g)) +
                          kK[i] + w[i];
      const uint32_t t2 = (rotr(a, 2) ^ rotr(a, 13) ^ rotr(a, 22)) + ((a & b) ^ (a & c) ^ (b & c));
      h = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
    }
    st[0] += a; st[1] += b; st[2] += c; st[3] += d;
    st[4] += e; st[5] += f; st[6] += g; st[7] += h;
  }
}

// SHA-NI: the state lives as (ABEF, CDGH); each sha256rnds2 runs two rounds,
// sha256msg1/msg2 extend the message schedule four words at a time.
__attribute__((target("sha,sse4.1,ssse3"))) void compress_shani(uint32_t st[8], const uint8_t* p,
                                                                size_t nblocks) {
  const __m128i kMask = _mm_set_epi64x(0x0c0d0e0f08090a0bULL, 0x0405060700010203ULL);
  __m128i tmp = _mm_loadu_si128(reinterpret_cast<const __m128i*>(st));
  __m128i s1 = _mm_loadu_si128(reinterpret_cast<const __m128i*>(st + 4));
  tmp = _mm_shuffle_epi32(tmp, 0xB1);   // CDAB
  s1 = _mm_shuffle_epi32(s1, 0x1B);     // EFGH
  __m128i s0 = _mm_alignr_epi8(tmp, s1, 8);  // ABEF
  s1 = _mm_blend_epi16(s1, tmp, 0xF0);       // CDGH
  for (; nblocks; nblocks--, p += 64) {
    const __m128i abef = s0, cdgh = s1;
    __m128i w[4];
#define CG_SHANI_GROUP(g)                                                                      \
  {                                                                                            \
    if ((g) < 4) {                                                                             \
      w[(g)&3] = _mm_shuffle_epi8(_mm_loadu_si128(reinterpret_cast<const __m128i*>(p + 16 * (g))), \
                                  kMask);                                                      \
    } else {                                                                                   \
      const __m128i t7 = _mm_alignr_epi8(w[((g)-1) & 3], w[((g)-2) & 3], 4);                  \
      w[(g)&3] = _mm_sha256msg2_epu32(                                                         \
          _mm_add_epi32(_mm_sha256msg1_epu32(w[(g)&3], w[((g)-3) & 3]), t7), w[((g)-1) & 3]);  \
    }                                                                                          \
    __m128i m = _mm_add_epi32(w[(g)&3], _mm_loadu_si128(reinterpret_cast<const __m128i*>(kK + 4 * (g)))); \
    s1 = _mm_sha256rnds2_epu32(s1, s0, m);                                                     \
    m = _mm_shuffle_epi32(m, 0x0E);                                                            \
    s0 = _mm_sha256rnds2_epu32(s0, s1, m);                                                     \
  }
    CG_SHANI_GROUP(0) CG_SHANI_GROUP(1) CG_SHANI_GROUP(2) CG_SHANI_GROUP(3)
    CG_SHANI_GROUP(4) CG_SHANI_GROUP(5) CG_SHANI_GROUP(6) CG_SHANI_GROUP(7)
    CG_SHANI_GROUP(8) CG_SHANI_GROUP(9) CG_SHANI_GROUP(10) CG_SHANI_GROUP(11)
    CG_SHANI_GROUP(12) CG_SHANI_GROUP(13) CG_SHANI_GROUP(14) CG_SHANI_GROUP(15)
#undef CG_SHANI_GROUP
    s0 = _mm_add_epi32(s0, abef);
    s1 = _mm_add_epi32(s1, cdgh);
  }
  tmp = _mm_shuffle_epi32(s0, 0x1B);          // FEBA
  s1 = _mm_shuffle_epi32(s1, 0xB1);           // DCHG
  s0 = _mm_blend_epi16(tmp, s1, 0xF0);        // DCBA
  s1 = _mm_alignr_epi8(s1, tmp, 8);           // ABEF -> HGFE
  _mm_storeu_si128(reinterpret_cast<__m128i*>(st), s0);
  _mm_storeu_si128(reinterpret_cast<__m128i*>(st + 4), s1);
}

bool cpu_has_shani() {
  unsigned a, b, c, d;
  if (!__get_cpuid_count(7, 0, &a, &b, &c, &d)) return false;
  const bool sha = (b >> 29) & 1;
  if (!__get_cpuid(1, &a, &b, &c, &d)) return false;
  const bool sse41 = (c >> 19) & 1, ssse3 = (c >> 9) & 1;
  return sha && sse41 && ssse3;
}

using CompressFn = void (*)(uint32_t*, const uint8_t*, size_t);
const CompressFn g_compress = (std::getenv("CREDO_HOST_SHA_SCALAR") == nullptr && cpu_has_shani())
                                  ? compress_shani
                                  : compress_scalar;

}  // namespace

bool host_sha256_accelerated() { return g_compress == compress_shani; }

HostSha256::HostSha256() {
  static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372, 0xa54ff53a,
                                 0x510e527f, 0x9b05688c, 0x1f83d9ab, 0x5be0cd19};
  std::memcpy(h, iv, sizeof h);
}

void HostSha256::update(const uint8_t* p, size_t len) {
  total += len;
  if (n) {
    const size_t take = std::min(len, (size_t)64 - n);
    std::memcpy(buf + n, p, take);
    n += take;
    p += take;
    len -= take;
    if (n < 64) return;
    g_compress(h, buf, 1);
    n = 0;
  }
  const size_t whole = len / 64;
  if (whole) g_compress(h, p, whole);
  p += 64 * whole;
  len -= 64 * whole;
  std::memcpy(buf, p, len);
  n = len;
}

void HostSha256::u8(uint8_t v) { update(&v, 1); }
void HostSha256::u32(uint32_t v) {
  const uint8_t b[4] = {(uint8_t)(v >> 24), (uint8_t)(v >> 16), (uint8_t)(v >> 8), (uint8_t)v};
  update(b, 4);
}
void HostSha256::u64(uint64_t v) {
  uint8_t b[8];
  for (int i = 0; i < 8; i++) b[i] = (uint8_t)(v >> (56 - 8 * i));
  update(b, 8);
}
void HostSha256::bytes(const uint8_t* p, size_t len) {
  u32((uint32_t)len);
  update(p, len);
}

// Codec f64 values (codec.hpp: IEEE-754 bits, big-endian) straight from the
// host f64 array, 4 KB at a time.
void HostSha256::f64be(const double* x, size_t count) {
  uint64_t stage[512];
  while (count) {
    const size_t c = std::min(count, (size_t)512);
    for (size_t i = 0; i < c; i++) {
      uint64_t b;
      std::memcpy(&b, x + i, 8);
      stage[i] = __builtin_bswap64(b);
    }
    update(reinterpret_cast<const uint8_t*>(stage), 8 * c);
    x += c;
    count -= c;
  }
}

void HostSha256::final(uint8_t out[32]) {
  const uint64_t bits = total * 8;
  uint8_t pad[72] = {0x80};
  const size_t padlen = (n < 56 ? 56 - n : 120 - n);
  update(pad, padlen);
  uint8_t lb[8];
  for (int i = 0; i < 8; i++) lb[i] = (uint8_t)(bits >> (56 - 8 * i));
  update(lb, 8);
  for (int i = 0; i < 8; i++) {
    out[4 * i] = (uint8_t)(h[i] >> 24);
    out[4 * i + 1] = (uint8_t)(h[i] >> 16);
    out[4 * i + 2] = (uint8_t)(h[i] >> 8);
    out[4 * i + 3] = (uint8_t)h[i];
  }
}

void host_sha256(const uint8_t* p, size_t len, uint8_t out[32]) {
  HostSha256 s;
  s.update(p, len);
  s.final(out);
}

}  // namespace cg

using namespace cg;

namespace {

// hash_ops (messages.cpp:197-202) over an all-request op list:
// 0x4F || u32 count || per op OpEntry::encode (messages.cpp:161-169) =
//   u8 kind (request_inf = 0) || bool 1 || InferenceRequest::encode
//   (domain.cpp:144-158) || bool 0 (no group op) || u64 version ||
//   u8 status || str reason.
void hash_ops_one(const cg_ops_batch& ob, uint8_t out[32]) {
  const cg_request_batch& b = *ob.requests;
  HostSha256 s;
  s.u8(0x4F);
  s.u32(b.B);
  uint64_t npos = 0, rpos = 0;
  for (uint32_t k = 0; k < b.B; k++) {
    s.u8(0);  // OpKind::request_inf
    s.u8(1);  // optional<InferenceRequest> present
    s.update(b.request_ids + 32 * k, 32);
    s.bytes(reinterpret_cast<const uint8_t*>(ob.group_id), ob.group_id_len);
    s.u32((uint32_t)b.u);
    s.f64be(b.inputs + b.u * k, b.u);
    const bool he = b.has_eps && b.has_eps[k];
    s.u8(he ? 1 : 0);
    if (he) {
      uint64_t bits;
      std::memcpy(&bits, &b.eps[k], 8);
      s.u64(bits);
    }
    s.update(b.client_pubs + 32 * k, 32);
    s.bytes(b.nonces + npos, b.nonce_lens[k]);
    npos += b.nonce_lens[k];
    s.update(b.client_sigs + 64 * k, 64);
    s.u8(0);  // optional<GroupOp> absent
    s.u64(ob.versions ? ob.versions[k] : ob.version);
    s.u8(ob.statuses ? ob.statuses[k] : 0);
    const uint64_t rl = ob.reason_lens ? ob.reason_lens[k] : 0;
    s.bytes(ob.reasons ? reinterpret_cast<const uint8_t*>(ob.reasons) + rpos : nullptr, rl);
    rpos += rl;
  }
  s.final(out);
}

}  // namespace

extern "C" {

int cg_host_sha256(const uint8_t* data, uint64_t len, uint8_t out[32]) {
  if ((!data && len) || !out) return CG_EINVAL;
  host_sha256(data, len, out);
  return CG_OK;
}

int cg_host_sha_accelerated(void) { return host_sha256_accelerated() ? 1 : 0; }

int cg_hash_ops_batches(const cg_ops_batch* batches, uint32_t nslots, int threads,
                        uint8_t* out) {
  if (!batches || !out) return CG_EINVAL;
  for (uint32_t i = 0; i < nslots; i++) {
    const cg_request_batch* b = batches[i].requests;
    if (!b || b->inputs_on_device || (b->B && (!b->inputs || !b->request_ids ||
                                                !b->client_pubs || !b->client_sigs ||
                                                !b->nonce_lens)))
      return CG_EINVAL;
  }
  const int nt = std::max(1, std::min<int>(threads > 0 ? threads : 1, (int)nslots));
  std::atomic<uint32_t> next{0};
  auto work = [&] {
    for (uint32_t i; (i = next.fetch_add(1)) < nslots;) hash_ops_one(batches[i], out + 32 * i);
  };
  if (nt == 1) {
    work();
  } else {
    std::vector<std::thread> pool;
    for (int t = 0; t < nt; t++) pool.emplace_back(work);
    for (auto& t : pool) t.join();
  }
  return CG_OK;
}

}  // extern "C"
