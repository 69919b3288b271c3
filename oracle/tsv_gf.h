/*
 * tsv_gf.h -- GF(2^64) arithmetic and the counter PRNG of the oracle
 * (TEST INFRASTRUCTURE ONLY; see tsv_oracle.c).  Static inline so the
 * multi-threaded restatement (tsv_oracle_big.c) inlines them.
 */
#ifndef TSV_ORACLE_GF_H
#define TSV_ORACLE_GF_H
#include <stdint.h>
#if defined(__PCLMUL__)
#include <wmmintrin.h>
#endif

/* 64x64 -> 128 carry-less product (gf.hpp:55-78). */
static inline void clmul(uint64_t a, uint64_t b, uint64_t *hi, uint64_t *lo) {
#if defined(__PCLMUL__)
  __m128i p = _mm_clmulepi64_si128(_mm_set_epi64x(0, (long long)a),
                                   _mm_set_epi64x(0, (long long)b), 0);
  *lo = (uint64_t)_mm_cvtsi128_si64(p);
  *hi = (uint64_t)_mm_cvtsi128_si64(_mm_unpackhi_epi64(p, p));
#else
  uint64_t h = 0, l = 0;
  for (int i = 0; i < 64; ++i) {
    if (!((b >> i) & 1)) continue;
    l ^= a << i;
    if (i) h ^= a >> (64 - i);
  }
  *hi = h;
  *lo = l;
#endif
}

/* Product in GF(2^64): fold the high word twice through 0x1b (gf.hpp:95-105). */
static inline uint64_t gf_mul(uint64_t a, uint64_t b) {
  uint64_t hi, lo, h1, l1, h2, l2;
  clmul(a, b, &hi, &lo);
  clmul(hi, 0x1bull, &h1, &l1);
  clmul(h1, 0x1bull, &h2, &l2);
  (void)h2;
  return lo ^ l1 ^ l2;
}

/* Bit-serial long-division product, independent of tsvo_gf_mul (mirrors the
 * reference's own test oracle idea, test_gf.cpp:16-45). */
static inline uint64_t gf_mul_slow(uint64_t a, uint64_t b) {
  uint64_t r = 0;
  for (int i = 63; i >= 0; --i) {
    uint64_t top = r >> 63;
    r <<= 1;
    if (top) r ^= 0x1bull;
    if ((b >> i) & 1) r ^= a;
  }
  return r;
}

static inline uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

/* gf.hpp:135-143 */
static inline uint64_t draw64(uint64_t seed, uint64_t role, uint64_t a, uint64_t b,
                     uint64_t c) {
  uint64_t h = seed + 0x9e3779b97f4a7c15ull;
  h = mix64(h ^ (role * 0xff51afd7ed558ccdull));
  h = mix64(h ^ (a + 0xc2b2ae3d27d4eb4full));
  h = mix64(h ^ (b + 0x165667b19e3779f9ull));
  h = mix64(h ^ (c + 0x27d4eb2f165667c5ull));
  return h;
}

/* gf.hpp:147-153 (64-bit word: re-mix until nonzero). */
static inline uint64_t draw_nonzero(uint64_t seed, uint64_t role, uint64_t a,
                           uint64_t b, uint64_t c) {
  uint64_t h = draw64(seed, role, a, b, c);
  while (h == 0) h = mix64(h + 0x9e3779b97f4a7c15ull);
  return h;
}

enum { ROLE_SHADE_V = 1, ROLE_SHADE_W = 2, ROLE_EDGE_Y = 3 };

#endif
