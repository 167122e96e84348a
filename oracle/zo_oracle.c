/*
 * oracle/zo_oracle.c -- TEST INFRASTRUCTURE ONLY.
 *
 * CPU restatement of the reference's direction-stream and digest arithmetic,
 * used by tests/, __graft_entry__.smoke() and bench.py's cpu_baseline leg as
 * the CHECKER.  Nothing in paper_2605_28760_b200/ links or calls this file.
 *
 * What it restates (reference = /root/reference/pkg/src/zoserve):
 *   fnv1a64            numerics.py:60-89   (_fnv1a_nb / _fnv1a_py)
 *   zo_oracle_key      numerics.py:156-158 (StreamKey.generator: entropy list
 *                      -> numpy SeedSequence -> Philox key; numpy 2.3.5
 *                      numpy/random/bit_generator.pyx SeedSequence.mix_entropy
 *                      / generate_state, Philox(seed_seq) -> key = 2 x u64)
 *   zo_oracle_gaussian numerics.py:161-168 (Generator.standard_normal =
 *                      numpy/random/src/distributions/distributions.c
 *                      random_standard_normal: 256-layer ziggurat over
 *                      Philox4x64-10 u64s, counter starting at 0 and
 *                      incremented before each 4-word block)
 *
 * The libm calls (log1p, exp) are the SAME glibc functions numpy calls, so
 * this restatement matches numpy by construction; the product's device
 * sampler carries its own glibc-equivalent log1p (csrc/zo_glibc_math.cuh).
 *
 * Pinned against: live numpy 2.3.5 in the build container and the golden
 * vectors under tests/golden/streams.json (tests/golden/make_golden.py).
 */
#include <math.h>
#include <stdint.h>
#include <string.h>

#include "ziggurat_tables.h"

#define FNV_PRIME 0x100000001B3ULL

uint64_t zo_oracle_fnv1a64(const uint8_t* buf, uint64_t n, uint64_t h) {
  for (uint64_t i = 0; i < n; ++i) h = (h ^ (uint64_t)buf[i]) * FNV_PRIME;
  return h;
}

/* ---- numpy SeedSequence (pool_size 4, uint32 arithmetic) ---- */
#define SS_INIT_A 0x43b0d7e5u
#define SS_MULT_A 0x931e8875u
#define SS_INIT_B 0x8b51f9ddu
#define SS_MULT_B 0x58f38dedu
#define SS_MIX_L 0xca01f9ddu
#define SS_MIX_R 0x4973f715u

static uint32_t ss_hashmix(uint32_t v, uint32_t* hc) {
  v ^= *hc;
  *hc *= SS_MULT_A;
  v *= *hc;
  v ^= v >> 16;
  return v;
}
static uint32_t ss_mix(uint32_t x, uint32_t y) {
  uint32_t r = SS_MIX_L * x - SS_MIX_R * y;
  r ^= r >> 16;
  return r;
}
static int ss_words(uint64_t v, uint32_t* out) {
  /* numpy _int_to_uint32_array: 0 -> [0], else little-endian 32-bit words */
  int n = 0;
  if (v == 0) { out[n++] = 0; return n; }
  while (v) { out[n++] = (uint32_t)(v & 0xffffffffu); v >>= 32; }
  return n;
}

void zo_oracle_key(uint64_t seed, uint64_t step, uint64_t lid_hash, uint64_t role,
                   uint64_t key_out[2]) {
  uint32_t ent[8];
  int n = 0;
  n += ss_words(seed, ent + n);
  n += ss_words(step, ent + n);
  n += ss_words(lid_hash, ent + n);
  n += ss_words(role, ent + n);
  uint32_t pool[4];
  uint32_t hc = SS_INIT_A;
  for (int i = 0; i < 4; ++i) pool[i] = ss_hashmix(i < n ? ent[i] : 0u, &hc);
  for (int s = 0; s < 4; ++s)
    for (int d = 0; d < 4; ++d)
      if (s != d) pool[d] = ss_mix(pool[d], ss_hashmix(pool[s], &hc));
  for (int s = 4; s < n; ++s)
    for (int d = 0; d < 4; ++d) pool[d] = ss_mix(pool[d], ss_hashmix(ent[s], &hc));
  uint32_t w[4];
  uint32_t hb = SS_INIT_B;
  for (int i = 0; i < 4; ++i) {
    uint32_t v = pool[i] ^ hb;
    hb *= SS_MULT_B;
    v *= hb;
    v ^= v >> 16;
    w[i] = v;
  }
  key_out[0] = (uint64_t)w[0] | ((uint64_t)w[1] << 32);
  key_out[1] = (uint64_t)w[2] | ((uint64_t)w[3] << 32);
}

/* ---- Philox4x64-10 ---- */
static inline uint64_t mulhilo(uint64_t a, uint64_t b, uint64_t* hi) {
  __uint128_t p = (__uint128_t)a * b;
  *hi = (uint64_t)(p >> 64);
  return (uint64_t)p;
}

void zo_oracle_philox_block(const uint64_t key_in[2], uint64_t block, uint64_t out[4]) {
  /* block = 0-based block index; numpy's counter value is block + 1 */
  uint64_t c[4] = {block + 1, 0, 0, 0};
  if (c[0] == 0) c[1] = 1;
  uint64_t k0 = key_in[0], k1 = key_in[1];
  for (int r = 0; r < 10; ++r) {
    uint64_t hi0, hi1;
    uint64_t lo0 = mulhilo(0xD2E7470EE14C6C93ULL, c[0], &hi0);
    uint64_t lo1 = mulhilo(0xCA5A826395121157ULL, c[2], &hi1);
    uint64_t n0 = hi1 ^ c[1] ^ k0, n2 = hi0 ^ c[3] ^ k1;
    c[0] = n0; c[1] = lo1; c[2] = n2; c[3] = lo0;
    k0 += 0x9E3779B97F4A7C15ULL;
    k1 += 0xBB67AE8584CAA73BULL;
  }
  memcpy(out, c, sizeof(c));
}

typedef struct {
  uint64_t key[2];
  uint64_t pos; /* next u64 position */
  uint64_t buf[4];
  uint64_t buf_block;
} stream_t;

static uint64_t next_u64(stream_t* s) {
  uint64_t blk = s->pos >> 2;
  if (blk != s->buf_block) {
    zo_oracle_philox_block(s->key, blk, s->buf);
    s->buf_block = blk;
  }
  return s->buf[s->pos++ & 3];
}
static double next_double(stream_t* s) {
  return (double)(next_u64(s) >> 11) * (1.0 / 9007199254740992.0);
}

static const double ZIG_R = 3.6541528853610088;
static const double ZIG_INV_R = 0.27366123732975828;

static double std_normal(stream_t* s) {
  for (;;) {
    uint64_t r = next_u64(s);
    int idx = (int)(r & 0xff);
    r >>= 8;
    int sign = (int)(r & 1);
    uint64_t rabs = (r >> 1) & 0x000fffffffffffffULL;
    double x = (double)rabs * zo_zig_wi[idx];
    if (sign) x = -x;
    if (rabs < zo_zig_ki[idx]) return x;
    if (idx == 0) {
      for (;;) {
        double xx = -ZIG_INV_R * log1p(-next_double(s));
        double yy = -log1p(-next_double(s));
        if (yy + yy > xx * xx)
          return ((rabs >> 8) & 1) ? -(ZIG_R + xx) : ZIG_R + xx;
      }
    } else {
      double lhs = (zo_zig_fi[idx - 1] - zo_zig_fi[idx]) * next_double(s) + zo_zig_fi[idx];
      if (lhs < exp(-0.5 * x * x)) return x;
    }
  }
}

/* Fill out[0..n) with the stream's standard normals (row-major fill order is
 * the caller's reshape).  Returns the number of u64 consumed. */
uint64_t zo_oracle_gaussian(const uint64_t key[2], uint64_t n, double* out) {
  stream_t s;
  s.key[0] = key[0]; s.key[1] = key[1];
  s.pos = 0; s.buf_block = ~0ULL;
  for (uint64_t i = 0; i < n; ++i) out[i] = std_normal(&s);
  return s.pos;
}

/* Same, starting the attempt chain at u64 position `start` (speculative parse
 * used to test the device chunk splice); writes up to n samples, returns the
 * position after the last consumed u64. */
uint64_t zo_oracle_gaussian_from(const uint64_t key[2], uint64_t start, uint64_t n, double* out) {
  stream_t s;
  s.key[0] = key[0]; s.key[1] = key[1];
  s.pos = start; s.buf_block = ~0ULL;
  for (uint64_t i = 0; i < n; ++i) out[i] = std_normal(&s);
  return s.pos;
}
