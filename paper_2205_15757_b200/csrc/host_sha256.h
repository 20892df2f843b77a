// Host SHA-256 (SHA-NI when available): the model-file check and hash_ops.
#pragma once
#include <stddef.h>
#include <stdint.h>

namespace cg {

struct HostSha256 {
  uint32_t h[8];
  uint8_t buf[64];
  size_t n = 0;
  uint64_t total = 0;
  HostSha256();
  void update(const uint8_t* p, size_t len);
  void u8(uint8_t v);
  void u32(uint32_t v);
  void u64(uint64_t v);
  void bytes(const uint8_t* p, size_t len);  // u32be length || bytes (codec.hpp)
  void f64be(const double* x, size_t count);  // IEEE bits, big-endian
  void final(uint8_t out[32]);
};

void host_sha256(const uint8_t* p, size_t len, uint8_t out[32]);
bool host_sha256_accelerated();

}  // namespace cg
