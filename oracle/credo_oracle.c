/* TEST INFRASTRUCTURE — CPU oracle (plain C restatement). See credo_oracle.h.
 * Compiled with -ffp-contract=off so a*b+c is never fused, matching the
 * reference's x86-64 SSE2 build (CMakeLists.txt:35, no -march). */
#include "credo_oracle.h"

#include <math.h>
#include <stdlib.h>
#include <string.h>

/* ---------------------------------------------------------------- SHA-256
 * FIPS 180-4; the reference delegates to libsodium (crypto.cpp:22-39). */
static const uint32_t K256[64] = {
    0x428a2f98, 0x71374491, 0xb5c0fbcf, 0xe9b5dba5, 0x3956c25b, 0x59f111f1,
    0x923f82a4, 0xab1c5ed5, 0xd807aa98, 0x12835b01, 0x243185be, 0x550c7dc3,
    0x72be5d74, 0x80deb1fe, 0x9bdc06a7, 0xc19bf174, 0xe49b69c1, 0xefbe4786,
    0x0fc19dc6, 0x240ca1cc, 0x2de92c6f, 0x4a7484aa, 0x5cb0a9dc, 0x76f988da,
    0x983e5152, 0xa831c66d, 0xb00327c8, 0xbf597fc7, 0xc6e00bf3, 0xd5a79147,
    0x06ca6351, 0x14292967, 0x27b70a85, 0x2e1b2138, 0x4d2c6dfc, 0x53380d13,
    0x650a7354, 0x766a0abb, 0x81c2c92e, 0x92722c85, 0xa2bfe8a1, 0xa81a664b,
    0xc24b8b70, 0xc76c51a3, 0xd192e819, 0xd6990624, 0xf40e3585, 0x106aa070,
    0x19a4c116, 0x1e376c08, 0x2748774c, 0x34b0bcb5, 0x391c0cb3, 0x4ed8aa4a,
    0x5b9cca4f, 0x682e6ff3, 0x748f82ee, 0x78a5636f, 0x84c87814, 0x8cc70208,
    0x90befffa, 0xa4506ceb, 0xbef9a3f7, 0xc67178f2};

#define ROR(x, n) (((x) >> (n)) | ((x) << (32 - (n))))

static void compress(uint32_t h[8], const uint8_t* p) {
  uint32_t w[64];
  for (int i = 0; i < 16; i++)
    w[i] = (uint32_t)p[4 * i] << 24 | (uint32_t)p[4 * i + 1] << 16 |
           (uint32_t)p[4 * i + 2] << 8 | p[4 * i + 3];
  for (int i = 16; i < 64; i++) {
    uint32_t s0 = ROR(w[i - 15], 7) ^ ROR(w[i - 15], 18) ^ (w[i - 15] >> 3);
    uint32_t s1 = ROR(w[i - 2], 17) ^ ROR(w[i - 2], 19) ^ (w[i - 2] >> 10);
    w[i] = w[i - 16] + s0 + w[i - 7] + s1;
  }
  uint32_t a = h[0], b = h[1], c = h[2], d = h[3], e = h[4], f = h[5],
           g = h[6], hh = h[7];
  for (int i = 0; i < 64; i++) {
    uint32_t t1 = hh + (ROR(e, 6) ^ ROR(e, 11) ^ ROR(e, 25)) +
                  ((e & f) ^ (~e & g)) + K256[i] + w[i];
    uint32_t t2 = (ROR(a, 2) ^ ROR(a, 13) ^ ROR(a, 22)) +
                  ((a & b) ^ (a & c) ^ (b & c));
    hh = g; g = f; f = e; e = d + t1; d = c; c = b; b = a; a = t1 + t2;
  }
  h[0] += a; h[1] += b; h[2] += c; h[3] += d;
  h[4] += e; h[5] += f; h[6] += g; h[7] += hh;
}

void oc_sha256_init(oc_sha256_ctx* c) {
  static const uint32_t iv[8] = {0x6a09e667, 0xbb67ae85, 0x3c6ef372,
                                 0xa54ff53a, 0x510e527f, 0x9b05688c,
                                 0x1f83d9ab, 0x5be0cd19};
  memcpy(c->h, iv, sizeof iv);
  c->total = 0;
  c->nbuf = 0;
}

void oc_sha256_update(oc_sha256_ctx* c, const uint8_t* p, uint64_t n) {
  c->total += n;
  while (n) {
    if (c->nbuf == 0 && n >= 64) {
      compress(c->h, p);
      p += 64;
      n -= 64;
      continue;
    }
    uint32_t take = 64 - c->nbuf;
    if (take > n) take = (uint32_t)n;
    memcpy(c->buf + c->nbuf, p, take);
    c->nbuf += take;
    p += take;
    n -= take;
    if (c->nbuf == 64) {
      compress(c->h, c->buf);
      c->nbuf = 0;
    }
  }
}

void oc_sha256_final(oc_sha256_ctx* c, uint8_t out[32]) {
  uint64_t bits = c->total * 8;
  uint8_t pad = 0x80;
  uint64_t total = c->total;
  oc_sha256_update(c, &pad, 1);
  uint8_t z = 0;
  while (c->nbuf != 56) oc_sha256_update(c, &z, 1);
  uint8_t len[8];
  for (int i = 0; i < 8; i++) len[i] = (uint8_t)(bits >> (56 - 8 * i));
  oc_sha256_update(c, len, 8);
  (void)total;
  for (int i = 0; i < 8; i++) {
    out[4 * i] = (uint8_t)(c->h[i] >> 24);
    out[4 * i + 1] = (uint8_t)(c->h[i] >> 16);
    out[4 * i + 2] = (uint8_t)(c->h[i] >> 8);
    out[4 * i + 3] = (uint8_t)c->h[i];
  }
}

void oc_sha256(const uint8_t* p, uint64_t n, uint8_t out[32]) {
  oc_sha256_ctx c;
  oc_sha256_init(&c);
  oc_sha256_update(&c, p, n);
  oc_sha256_final(&c, out);
}

void oc_sha256_midstate(const uint8_t* p, uint64_t nblocks, uint32_t out[8]) {
  oc_sha256_ctx c;
  oc_sha256_init(&c);
  for (uint64_t i = 0; i < nblocks; i++) compress(c.h, p + 64 * i);
  memcpy(out, c.h, 32);
}

/* ------------------------------------------------------------ encodings
 * codec.hpp:28-84: u64/f64 8-byte BE, u32 BE length prefixes, bool byte. */
typedef struct {
  uint8_t* out;
  uint64_t n;
} enc_t;

static void put(enc_t* e, const void* p, uint64_t n) {
  if (e->out) memcpy(e->out + e->n, p, n);
  e->n += n;
}
static void put_u8(enc_t* e, uint8_t v) { put(e, &v, 1); }
static void put_u32(enc_t* e, uint32_t v) {
  uint8_t b[4] = {(uint8_t)(v >> 24), (uint8_t)(v >> 16), (uint8_t)(v >> 8),
                  (uint8_t)v};
  put(e, b, 4);
}
static void put_u64(enc_t* e, uint64_t v) {
  uint8_t b[8];
  for (int i = 0; i < 8; i++) b[i] = (uint8_t)(v >> (56 - 8 * i));
  put(e, b, 8);
}
static void put_f64(enc_t* e, double d) {
  uint64_t v;
  memcpy(&v, &d, 8);
  put_u64(e, v);
}
static void put_bytes(enc_t* e, const void* p, uint64_t n) {
  put_u32(e, (uint32_t)n);
  put(e, p, n);
}

/* InferenceRequest::encode = encode_request_body + sig (domain.cpp:144-158). */
uint64_t oc_request_encode(const uint8_t req_id[32], const char* gid,
                           uint64_t gid_len, const double* input, uint64_t u,
                           int has_eps, double eps, const uint8_t pub[32],
                           const uint8_t* nonce, uint64_t nonce_len,
                           const uint8_t sig[64], uint8_t* out) {
  enc_t e = {out, 0};
  put(&e, req_id, 32);
  put_bytes(&e, gid, gid_len);
  put_u32(&e, (uint32_t)u);
  for (uint64_t i = 0; i < u; i++) put_f64(&e, input[i]);
  put_u8(&e, has_eps ? 1 : 0);
  if (has_eps) put_f64(&e, eps);
  put(&e, pub, 32);
  put_bytes(&e, nonce, nonce_len);
  put(&e, sig, 64);
  return e.n;
}

/* InferenceResult::encode (domain.cpp:218-225). */
uint64_t oc_result_encode(const uint8_t req_id[32], uint64_t node,
                          const char* gid, uint64_t gid_len, uint64_t version,
                          const double* output, uint64_t v,
                          const uint8_t model_digest[32], uint8_t* out) {
  enc_t e = {out, 0};
  put(&e, req_id, 32);
  put_u64(&e, node);
  put_bytes(&e, gid, gid_len);
  put_u64(&e, version);
  put_u32(&e, (uint32_t)v);
  for (uint64_t i = 0; i < v; i++) put_f64(&e, output[i]);
  put(&e, model_digest, 32);
  return e.n;
}

/* FailureRecord::encode behind tag 0x46 (messages.cpp:260-266, 292-297). */
uint64_t oc_failure_leaf(const uint8_t req_id[32], const char* gid,
                         uint64_t gid_len, uint64_t version, const char* reason,
                         uint64_t reason_len, uint8_t* out) {
  enc_t e = {out, 0};
  put_u8(&e, 0x46);
  put(&e, req_id, 32);
  put_bytes(&e, gid, gid_len);
  put_u64(&e, version);
  put_bytes(&e, reason, reason_len);
  return e.n;
}

/* -------------------------------------------------------------- merkle */
void oc_leaf_hash(const uint8_t* leaf, uint64_t n, uint8_t out[32]) {
  oc_sha256_ctx c;
  uint8_t dom = 0x00;
  oc_sha256_init(&c);
  oc_sha256_update(&c, &dom, 1);
  oc_sha256_update(&c, leaf, n);
  oc_sha256_final(&c, out);
}

void oc_tagged_leaf_hash(uint8_t tag, const uint8_t* a, uint64_t na,
                         const uint8_t* b, uint64_t nb, uint8_t out[32]) {
  oc_sha256_ctx c;
  uint8_t pre[2] = {0x00, tag};
  oc_sha256_init(&c);
  oc_sha256_update(&c, pre, 2);
  oc_sha256_update(&c, a, na);
  if (nb) oc_sha256_update(&c, b, nb);
  oc_sha256_final(&c, out);
}

void oc_result_leaf_hash(const uint8_t* req, uint64_t req_len,
                         const uint8_t* res, uint64_t res_len, uint8_t out[32]) {
  oc_tagged_leaf_hash(0x52, req, req_len, res, res_len, out);
}

/* Tree::build level fold (merkle.cpp:47-67; internal node merkle.cpp:14-19). */
int oc_merkle_root(const uint8_t* leaf_hashes, uint64_t n, uint8_t out[32]) {
  if (n == 0) return -1;
  uint8_t* lvl = (uint8_t*)malloc(32 * n);
  memcpy(lvl, leaf_hashes, 32 * n);
  while (n > 1) {
    uint64_t m = 0;
    for (uint64_t i = 0; i < n; i += 2) {
      if (i + 1 < n) {
        uint8_t buf[65];
        buf[0] = 0x01;
        memcpy(buf + 1, lvl + 32 * i, 32);
        memcpy(buf + 33, lvl + 32 * (i + 1), 32);
        oc_sha256(buf, 65, lvl + 32 * m);
      } else {
        memmove(lvl + 32 * m, lvl + 32 * i, 32); /* unpaired node promoted */
      }
      m++;
    }
    n = m;
  }
  memcpy(out, lvl, 32);
  free(lvl);
  return 0;
}

/* ------------------------------------------------------------ agreement
 * distance.cpp:70-103. */
double oc_delta(uint32_t metric, const double* x, const double* y, uint64_t v) {
  if (metric == 0) {
    double acc = 0.0;
    for (uint64_t i = 0; i < v; i++) {
      double d = x[i] - y[i];
      acc += d * d;
    }
    return sqrt(acc);
  }
  if (metric == 1) return fabs(x[0] - y[0]);
  double worst = 0.0;
  for (uint64_t i = 0; i < v; i++) {
    double d = fabs(x[i] - y[i]);
    worst = (worst < d) ? d : worst; /* std::max(worst, d) */
  }
  return worst;
}

/* select_quorum (distance.cpp:138-216): exhaustive mask scan; order = size
 * desc, diameter asc, sorted index tuple asc (better(), :128-134). */
int oc_select_quorum(const double* outs, const uint64_t* node_idx, uint64_t m,
                     uint64_t v, uint64_t n, uint64_t f, uint32_t metric,
                     double eps, uint64_t* selected_mask, double* diam,
                     int* satisfied) {
  if (n == 0 || f >= n) return -1;
  const uint64_t need = n - f;
  if (m < need) return -1;
  for (uint64_t i = 0; i < m; i++)
    if (node_idx[i] >= n || v == 0) return -1;
  if (m > 20) return -1;
  /* max_minus_min throws on vectors, but only when delta runs (m >= 2,
   * distance.cpp:87-91 inside the pair loop at :170-175) */
  if (metric == 1 && v != 1 && m >= 2) return -1;
  double* dist = (double*)calloc(m * m, sizeof(double));
  for (uint64_t i = 0; i < m; i++)
    for (uint64_t j = i + 1; j < m; j++)
      dist[i * m + j] = dist[j * m + i] =
          oc_delta(metric, outs + i * v, outs + j * v, v);
  int have = 0;
  uint64_t best_mask = 0, best_size = 0;
  double best_diam = 0.0;
  for (uint64_t mask = 1; mask < (1ull << m); mask++) {
    uint64_t size = (uint64_t)__builtin_popcountll(mask);
    if (size < need) continue;
    double d = 0.0;
    int ok = 1;
    for (uint64_t i = 0; i < m && ok; i++) {
      if (!(mask >> i & 1)) continue;
      for (uint64_t j = i + 1; j < m; j++) {
        if (!(mask >> j & 1)) continue;
        double x = dist[i * m + j];
        d = (d < x) ? x : d;
        if (d > eps) {
          ok = 0;
          break;
        }
      }
    }
    if (!ok) continue;
    int wins;
    if (!have) {
      wins = 1;
    } else if (size != best_size) {
      wins = size > best_size;
    } else if (d != best_diam) {
      wins = d < best_diam;
    } else {
      /* sorted tuples compare lexicographically: the lowest differing
       * position decides, and the tuple holding it is smaller. */
      uint64_t diff = mask ^ best_mask;
      wins = diff && ((mask & (diff & (~diff + 1))) != 0);
    }
    if (wins) {
      have = 1;
      best_mask = mask;
      best_size = size;
      best_diam = d;
    }
  }
  free(dist);
  uint64_t sel = 0;
  if (have)
    for (uint64_t i = 0; i < m; i++)
      if (best_mask >> i & 1) sel |= 1ull << node_idx[i];
  *selected_mask = sel;
  *diam = have ? best_diam : 0.0;
  *satisfied = have;
  return 0;
}

uint64_t oc_argmax(const double* v, uint64_t n) {
  uint64_t best = 0;
  for (uint64_t i = 1; i < n; i++)
    if (v[best] < v[i]) best = i; /* std::max_element: first maximum */
  return best;
}

int64_t oc_ensemble_label(const double* outs, uint64_t m, uint64_t v,
                          uint64_t mask, uint64_t f) {
  /* votes keyed by label, iterated ascending (std::map, :108-123). */
  uint64_t* cnt = (uint64_t*)calloc(v, sizeof(uint64_t));
  double* conf = (double*)malloc(v * sizeof(double));
  for (uint64_t i = 0; i < v; i++) conf[i] = 0.0; /* value-initialised pair */
  for (uint64_t i = 0; i < m; i++) {
    if (!(mask >> i & 1)) continue;
    const double* row = outs + i * v;
    uint64_t l = oc_argmax(row, v);
    cnt[l]++;
    conf[l] = (conf[l] < row[l]) ? row[l] : conf[l];
  }
  int64_t best = -1;
  double best_conf = -1.0;
  for (uint64_t l = 0; l < v; l++) {
    if (cnt[l] == 0 || cnt[l] <= f) continue;
    if (conf[l] > best_conf) {
      best = (int64_t)l;
      best_conf = conf[l];
    }
  }
  free(cnt);
  free(conf);
  return best;
}

void oc_topk(const double* v, uint64_t n, uint32_t k, uint32_t* idx,
             double* val) {
  for (uint32_t s = 0; s < k; s++) {
    int64_t best = -1;
    for (uint64_t i = 0; i < n; i++) {
      int taken = 0;
      for (uint32_t t = 0; t < s; t++)
        if (idx[t] == i) taken = 1;
      if (taken) continue;
      if (best < 0 || v[best] < v[i]) best = (int64_t)i;
    }
    idx[s] = (uint32_t)best;
    val[s] = v[best];
  }
}

/* ---------------------------------------------------------- model path */
void oc_softmax(double* y, uint64_t v) {
  double peak = y[0];
  for (uint64_t i = 1; i < v; i++) peak = (peak < y[i]) ? y[i] : peak;
  double sum = 0.0;
  for (uint64_t i = 0; i < v; i++) {
    y[i] = exp(y[i] - peak);
    sum += y[i];
  }
  for (uint64_t i = 0; i < v; i++) y[i] /= sum;
}

void oc_linear_run(const double* W, const double* b, uint64_t u, uint64_t v,
                   int softmax, const double* x, double* y) {
  for (uint64_t row = 0; row < v; row++) {
    double acc = b[row];
    const double* w = W + row * u;
    for (uint64_t col = 0; col < u; col++) acc += w[col] * x[col];
    y[row] = acc;
  }
  if (softmax) oc_softmax(y, v);
}

/* PerturbingExecutor::run (model.cpp:82-105). The seed encoder is
 * u64 node || hash(model_digest) || f64_list(input) (codec.hpp:32-71: u32be
 * count, then big-endian doubles); each lane appends u64 lane and hashes. */
void oc_perturb(uint64_t node, const uint8_t model_digest[32], const double* x,
                uint64_t u, double* y, uint64_t v, double mag) {
  if (mag == 0.0) return;
  uint8_t hdr[44];
  for (int i = 0; i < 8; i++) hdr[i] = (uint8_t)(node >> (56 - 8 * i));
  memcpy(hdr + 8, model_digest, 32);
  for (int i = 0; i < 4; i++) hdr[40 + i] = (uint8_t)((uint32_t)u >> (24 - 8 * i));
  oc_sha256_ctx seed;
  oc_sha256_init(&seed);
  oc_sha256_update(&seed, hdr, 44);
  for (uint64_t k = 0; k < u; k++) {
    uint64_t bits;
    uint8_t be[8];
    memcpy(&bits, x + k, 8);
    for (int i = 0; i < 8; i++) be[i] = (uint8_t)(bits >> (56 - 8 * i));
    oc_sha256_update(&seed, be, 8);
  }
  for (uint64_t lane = 0; lane < v; lane++) {
    oc_sha256_ctx c = seed;
    uint8_t lb[8], h[32];
    for (int i = 0; i < 8; i++) lb[i] = (uint8_t)(lane >> (56 - 8 * i));
    oc_sha256_update(&c, lb, 8);
    oc_sha256_final(&c, h);
    uint64_t raw = 0;
    for (int b = 0; b < 8; b++) raw = (raw << 8) | h[b];
    double unit = (double)raw / 18446744073709551615.0;
    y[lane] += (2.0 * unit - 1.0) * mag;
  }
}

/* -------------------------------------------------------- attestation */
uint64_t oc_attest_manifest(uint64_t B, uint64_t N, const uint64_t* sel_mask,
                            const uint8_t* satisfied, uint8_t* kinds,
                            uint64_t* nodes, uint64_t* ops) {
  uint64_t whole = 0, cnt = 0;
  for (uint64_t p = 0; p < N; p++) {
    int all = 1;
    for (uint64_t k = 0; k < B; k++)
      if (!satisfied[k] || !(sel_mask[k] >> p & 1)) { all = 0; break; }
    if (all) whole |= 1ull << p;
  }
  for (uint64_t p = 0; p < N; p++)
    if (whole >> p & 1) { kinds[cnt] = 0; nodes[cnt] = p; ops[cnt] = 0; cnt++; }
  for (uint64_t k = 0; k < B; k++) {
    if (!satisfied[k]) continue;
    for (uint64_t p = 0; p < N; p++) {
      if (!(sel_mask[k] >> p & 1) || (whole >> p & 1)) continue;
      kinds[cnt] = 1; nodes[cnt] = p; ops[cnt] = k; cnt++;
    }
  }
  for (uint64_t k = 0; k < B; k++)
    if (!satisfied[k]) { kinds[cnt] = 2; nodes[cnt] = 0; ops[cnt] = k; cnt++; }
  return cnt;
}

/* ------------------------------------------------------ C5 agreement sweep */
void oc_label_digest(const uint8_t req_id[32], uint64_t version, int64_t label,
                     uint8_t out[32]) {
  uint8_t m[49];
  m[0] = 0x4C;
  memcpy(m + 1, req_id, 32);
  for (int i = 0; i < 8; i++) m[33 + i] = (uint8_t)(version >> (56 - 8 * i));
  const uint64_t l = (uint64_t)label;
  for (int i = 0; i < 8; i++) m[41 + i] = (uint8_t)(l >> (56 - 8 * i));
  oc_sha256(m, sizeof m, out);
}

int oc_agree_batch(const double* outs, uint64_t R, uint64_t n, uint64_t f,
                   uint64_t v, uint32_t metric, const double* eps,
                   const uint8_t* req_ids, uint64_t version, uint64_t* sel,
                   double* diam, uint8_t* sat, int64_t* label, uint8_t* digest) {
  double* rows = (double*)malloc(n * v * sizeof(double));
  uint64_t idx[64];
  int rc = 0;
  for (uint64_t i = 0; i < n && i < 64; i++) idx[i] = i;
  for (uint64_t k = 0; k < R && rc == 0; k++) {
    for (uint64_t p = 0; p < n; p++)
      memcpy(rows + p * v, outs + p * R * v + k * v, v * sizeof(double));
    int s = 0;
    if (oc_select_quorum(rows, idx, n, v, n, f, metric, eps[k], &sel[k], &diam[k], &s) != 0) {
      rc = -1;
      break;
    }
    sat[k] = (uint8_t)s;
    label[k] = s ? oc_ensemble_label(rows, n, v, sel[k], f) : -1;
    if (req_ids && digest) oc_label_digest(req_ids + 32 * k, version, label[k], digest + 32 * k);
  }
  free(rows);
  return rc;
}
