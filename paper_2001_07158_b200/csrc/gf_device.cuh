// gf_device.cuh -- GF(2^64) arithmetic and position-addressed draws on sm_100a.
//
// Field: GF(2)[x] / (x^64 + x^4 + x^3 + x + 1), the reference's b = 64 field
// (/root/reference/proj/core/include/tsieve/gf.hpp:37-42).  Addition is XOR.
// Blackwell has no carry-less multiply instruction, so the 64x64 -> 128
// carry-less product is emulated on the integer pipes.  Every variant below
// returns the same field element as gf::mul<uint64_t> (gf.hpp:85-106); the
// engine picks one by measurement (tsv_bench_gf / DESIGN.md).
//
//  * clmul32_holes: 32x32 -> 64 via integer multiplies of operands masked to
//    every 4th bit ("holes"): each IMAD.WIDE sums at most 8 one-bit products
//    per output position, which fits in the 3 spare bits above it, so the
//    parity bit of each position is the carry-less result.  16 IMAD.WIDE on
//    the FMA pipe + LOP3 masking on the ALU pipe.
//  * clmul64 = one Karatsuba level over clmul32 (3 products, not 4).
//  * gf_reduce folds the high word: h*x^64 == h*(x^4+x^3+x+1), twice.
//  * gf_mul_serial: bit-serial reference, used only by the self-test kernel.
#pragma once
#include <cstdint>

namespace tsv {

struct u128 {
  uint64_t lo, hi;
};

__device__ __forceinline__ uint64_t clmul32_holes(uint32_t a, uint32_t b) {
  const uint32_t m0 = 0x11111111u, m1 = 0x22222222u, m2 = 0x44444444u,
                 m3 = 0x88888888u;
  const uint32_t a0 = a & m0, a1 = a & m1, a2 = a & m2, a3 = a & m3;
  const uint32_t b0 = b & m0, b1 = b & m1, b2 = b & m2, b3 = b & m3;
#define TSV_P(x, y) ((uint64_t)(x) * (uint64_t)(y))
  // Output class r collects the products whose mask classes sum to r mod 4.
  const uint64_t c0 = TSV_P(a0, b0) ^ TSV_P(a1, b3) ^ TSV_P(a2, b2) ^ TSV_P(a3, b1);
  const uint64_t c1 = TSV_P(a0, b1) ^ TSV_P(a1, b0) ^ TSV_P(a2, b3) ^ TSV_P(a3, b2);
  const uint64_t c2 = TSV_P(a0, b2) ^ TSV_P(a1, b1) ^ TSV_P(a2, b0) ^ TSV_P(a3, b3);
  const uint64_t c3 = TSV_P(a0, b3) ^ TSV_P(a1, b2) ^ TSV_P(a2, b1) ^ TSV_P(a3, b0);
#undef TSV_P
  return (c0 & 0x1111111111111111ull) | (c1 & 0x2222222222222222ull) |
         (c2 & 0x4444444444444444ull) | (c3 & 0x8888888888888888ull);
}

// 64x64 -> 128 carry-less product, one Karatsuba level.
__device__ __forceinline__ u128 clmul64(uint64_t a, uint64_t b) {
  const uint32_t al = (uint32_t)a, ah = (uint32_t)(a >> 32);
  const uint32_t bl = (uint32_t)b, bh = (uint32_t)(b >> 32);
  const uint64_t L = clmul32_holes(al, bl);
  const uint64_t H = clmul32_holes(ah, bh);
  const uint64_t M = clmul32_holes(al ^ ah, bl ^ bh) ^ L ^ H;
  u128 r;
  r.lo = L ^ (M << 32);
  r.hi = H ^ (M >> 32);
  return r;
}

// Reduce a 128-bit carry-less product modulo x^64 + x^4 + x^3 + x + 1.
__device__ __forceinline__ uint64_t gf_reduce(u128 p) {
  const uint64_t h = p.hi;
  const uint64_t over = (h >> 63) ^ (h >> 61) ^ (h >> 60);
  return p.lo ^ h ^ (h << 1) ^ (h << 3) ^ (h << 4) ^ over ^ (over << 1) ^
         (over << 3) ^ (over << 4);
}

__device__ __forceinline__ uint64_t gf_mul(uint64_t a, uint64_t b) {
  return gf_reduce(clmul64(a, b));
}

__device__ __forceinline__ u128 u128_xor(u128 a, u128 b) {
  return {a.lo ^ b.lo, a.hi ^ b.hi};
}

// Bit-serial product (Horner over the bits of b); independent check path.
__device__ __forceinline__ uint64_t gf_mul_serial(uint64_t a, uint64_t b) {
  uint64_t r = 0;
  for (int i = 63; i >= 0; --i) {
    const uint64_t top = r >> 63;
    r = (r << 1) ^ (top ? 0x1bull : 0ull);
    if ((b >> i) & 1) r ^= a;
  }
  return r;
}

// ---- counter PRNG: gf.hpp:111-153 (splitmix64 finalizer rounds) ----------

__host__ __device__ __forceinline__ uint64_t mix64(uint64_t x) {
  x ^= x >> 30;
  x *= 0xbf58476d1ce4e5b9ull;
  x ^= x >> 27;
  x *= 0x94d049bb133111ebull;
  x ^= x >> 31;
  return x;
}

enum : uint64_t { kRoleShadeV = 1, kRoleShadeW = 2, kRoleEdgeY = 3 };

// First two rounds of draw64 depend only on (seed, role): hoisted per launch.
__host__ __device__ __forceinline__ uint64_t draw_prefix(uint64_t seed,
                                                         uint64_t role) {
  uint64_t h = seed + 0x9e3779b97f4a7c15ull;
  return mix64(h ^ (role * 0xff51afd7ed558ccdull));
}

__host__ __device__ __forceinline__ uint64_t draw_nonzero_from(uint64_t pre,
                                                               uint64_t a,
                                                               uint64_t b,
                                                               uint64_t c) {
  uint64_t h = mix64(pre ^ (a + 0xc2b2ae3d27d4eb4full));
  h = mix64(h ^ (b + 0x165667b19e3779f9ull));
  h = mix64(h ^ (c + 0x27d4eb2f165667c5ull));
  while (h == 0) h = mix64(h + 0x9e3779b97f4a7c15ull);
  return h;
}

__host__ __device__ __forceinline__ uint64_t draw_nonzero(uint64_t seed,
                                                          uint64_t role,
                                                          uint64_t a,
                                                          uint64_t b,
                                                          uint64_t c) {
  return draw_nonzero_from(draw_prefix(seed, role), a, b, c);
}

// Round 3 of a y draw: the c = 0 round and the (seed, role) prefix are fixed
// per (level, launch); only the edge id varies.  yb = b + const for level l-1.
__device__ __forceinline__ uint64_t draw_edge_y(uint64_t pre, uint64_t yb,
                                                uint32_t edge) {
  uint64_t h = mix64(pre ^ ((uint64_t)edge + 0xc2b2ae3d27d4eb4full));
  h = mix64(h ^ yb);
  h = mix64(h ^ 0x27d4eb2f165667c5ull);  // c = 0
  while (h == 0) h = mix64(h + 0x9e3779b97f4a7c15ull);
  return h;
}

}  // namespace tsv
