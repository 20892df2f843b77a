/* Test-infrastructure shim (oracle only). Declares the eleven libsodium
 * entry points the reference calls (reference proj/src/crypto.cpp:22-83).
 * SHA-256 is served by OpenSSL (sodium_sha_openssl.c); Ed25519 comes from
 * the libsodium 26.2.0 shared object that ships inside the image (pyzmq).
 * The state layout matches libsodium's crypto_hash_sha256_state (104 bytes).
 */
#ifndef CREDO_ORACLE_SODIUM_SHIM_H
#define CREDO_ORACLE_SODIUM_SHIM_H
#include <stddef.h>
#include <stdint.h>
#ifdef __cplusplus
extern "C" {
#endif

typedef struct crypto_hash_sha256_state {
  uint32_t state[8];
  uint64_t count;
  uint8_t buf[64];
} crypto_hash_sha256_state;

int sodium_init(void);
int crypto_hash_sha256(unsigned char* out, const unsigned char* in,
                       unsigned long long inlen);
int crypto_hash_sha256_init(crypto_hash_sha256_state* state);
int crypto_hash_sha256_update(crypto_hash_sha256_state* state,
                              const unsigned char* in,
                              unsigned long long inlen);
int crypto_hash_sha256_final(crypto_hash_sha256_state* state,
                             unsigned char* out);
int crypto_sign_keypair(unsigned char* pk, unsigned char* sk);
int crypto_sign_seed_keypair(unsigned char* pk, unsigned char* sk,
                             const unsigned char* seed);
int crypto_sign_detached(unsigned char* sig, unsigned long long* siglen_p,
                         const unsigned char* m, unsigned long long mlen,
                         const unsigned char* sk);
int crypto_sign_verify_detached(const unsigned char* sig,
                                const unsigned char* m,
                                unsigned long long mlen,
                                const unsigned char* pk);
int crypto_sign_ed25519_sk_to_pk(unsigned char* pk, const unsigned char* sk);

#ifdef __cplusplus
}
#endif
#endif
