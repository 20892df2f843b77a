/* Test-infrastructure shim (oracle only): the four crypto_hash_sha256*
 * entry points on top of OpenSSL's SHA-256 (SHA-NI on x86). Digests are
 * identical to libsodium's; only speed differs (23 MB/s
 * for the shipped libsodium vs ~1.25 GB/s here). */
#include <openssl/sha.h>
#include <string.h>

#include "sodium.h"

/* OpenSSL's SHA256_CTX is {h[8], Nl, Nh, data[16], num, md_len} = 112 B,
 * larger than the 104-byte libsodium state, so keep the chaining value in
 * state->state and re-create a SHA256_CTX around it for each update. */

static void load_ctx(SHA256_CTX* c, const crypto_hash_sha256_state* s) {
  memset(c, 0, sizeof(*c));
  for (int i = 0; i < 8; i++) c->h[i] = s->state[i];
  uint64_t bits = s->count; /* total bits processed so far (incl. buffered) */
  c->Nl = (unsigned int)(bits & 0xffffffffu);
  c->Nh = (unsigned int)(bits >> 32);
  unsigned int buffered = (unsigned int)((bits >> 3) & 63);
  memcpy(c->data, s->buf, buffered);
  c->num = buffered;
  c->md_len = SHA256_DIGEST_LENGTH;
}

static void store_ctx(crypto_hash_sha256_state* s, const SHA256_CTX* c) {
  for (int i = 0; i < 8; i++) s->state[i] = c->h[i];
  s->count = ((uint64_t)c->Nh << 32) | c->Nl;
  memcpy(s->buf, c->data, c->num);
}

int crypto_hash_sha256_init(crypto_hash_sha256_state* state) {
  SHA256_CTX c;
  SHA256_Init(&c);
  store_ctx(state, &c);
  return 0;
}

int crypto_hash_sha256_update(crypto_hash_sha256_state* state,
                              const unsigned char* in,
                              unsigned long long inlen) {
  SHA256_CTX c;
  load_ctx(&c, state);
  SHA256_Update(&c, in, (size_t)inlen);
  store_ctx(state, &c);
  return 0;
}

int crypto_hash_sha256_final(crypto_hash_sha256_state* state,
                             unsigned char* out) {
  SHA256_CTX c;
  load_ctx(&c, state);
  SHA256_Final(out, &c);
  return 0;
}

int crypto_hash_sha256(unsigned char* out, const unsigned char* in,
                       unsigned long long inlen) {
  SHA256(in, (size_t)inlen, out);
  return 0;
}
