// gf_device.cuh -- GF(2^64) arithmetic and position-addressed draws on sm_100a.
//
// Field: GF(2)[x] / (x^64 + x^4 + x^3 + x + 1), the reference's b = 64 field
// (/root/reference/proj/core/include/tsieve/gf.hpp:37-42).  Addition is XOR.
// Blackwell has no carry-less multiply instruction, so products are emulated
// on the integer pipes.  Every routine returns the same field element as
// gf::mul<uint64_t> (gf.hpp:85-106); the engine picks by measurement
// (tsv_gf_bench, DESIGN.md section "GF(2^64) multiply"):
//
//  * gf_mul_kara  -- general product.  32x32 -> 64 carry-less products come
//    from integer multiplies of operands masked to every 4th bit ("holes"):
//    each mul.wide sums at most 8 one-bit products per output position, which
//    fits below the next position of the same residue class, so bit p of the
//    integer product is the carry-less bit p for its class.  Classes are XORed
//    unmasked through one Karatsuba level and masked once at the end.
//  * gf_mul_school -- same, schoolbook (4 sub-products, no operand sums).
//  * GfTable -- product by a WARP-UNIFORM multiplier y: 16 tables of the 16
//    multiples c * x^(4i) * y (fully reduced, 2 KB in shared memory, built
//    cooperatively by the warp), then 16 nibble lookups per product.  Each
//    table spans the 32 banks exactly once, so lookups are conflict-free.
//  * gf_mul_serial -- bit-serial reference for the self-test kernel.
#pragma once
#include <cstdint>
#include <utility>

namespace tsv {

struct u128 {
  uint64_t lo, hi;
};

__device__ __forceinline__ uint64_t wmul(uint32_t a, uint32_t b) {
  uint64_t r;
  asm("mul.wide.u32 %0, %1, %2;" : "=l"(r) : "r"(a), "r"(b));
  return r;
}

__device__ __forceinline__ uint32_t lo32(uint64_t x) { return static_cast<uint32_t>(x); }
__device__ __forceinline__ uint32_t hi32(uint64_t x) { return static_cast<uint32_t>(x >> 32); }
__device__ __forceinline__ uint64_t pack(uint32_t lo, uint32_t hi) {
  return (static_cast<uint64_t>(hi) << 32) | lo;
}

struct Split4 {
  uint32_t c[4];
};

__device__ __forceinline__ Split4 split4(uint32_t a) {
  Split4 s;
  s.c[0] = a & 0x11111111u;
  s.c[1] = a & 0x22222222u;
  s.c[2] = a & 0x44444444u;
  s.c[3] = a & 0x88888888u;
  return s;
}

// Class-r raw product (unmasked): XOR over i of a_i * b_{(r-i) mod 4}.
template <int R>
__device__ __forceinline__ uint64_t class_prod(const Split4& a, const Split4& b) {
  return wmul(a.c[0], b.c[R & 3]) ^ wmul(a.c[1], b.c[(R + 3) & 3]) ^
         wmul(a.c[2], b.c[(R + 2) & 3]) ^ wmul(a.c[3], b.c[(R + 1) & 3]);
}

__device__ __forceinline__ uint64_t mask_class(uint64_t c0, uint64_t c1, uint64_t c2,
                                               uint64_t c3) {
  return (c0 & 0x1111111111111111ull) | (c1 & 0x2222222222222222ull) |
         (c2 & 0x4444444444444444ull) | (c3 & 0x8888888888888888ull);
}

// Karatsuba over 32-bit halves with deferred class masking.
__device__ __forceinline__ u128 clmul64_kara(uint64_t a, uint64_t b) {
  const Split4 al = split4(lo32(a)), ah = split4(hi32(a)), am = split4(lo32(a) ^ hi32(a));
  const Split4 bl = split4(lo32(b)), bh = split4(hi32(b)), bm = split4(lo32(b) ^ hi32(b));
  uint64_t lo[4], hi[4];
#define TSV_KCLASS(R)                                          \
  {                                                            \
    const uint64_t L = class_prod<R>(al, bl);                  \
    const uint64_t H = class_prod<R>(ah, bh);                  \
    const uint64_t M = class_prod<R>(am, bm) ^ L ^ H;          \
    lo[R] = L ^ (M << 32);                                     \
    hi[R] = H ^ (M >> 32);                                     \
  }
  TSV_KCLASS(0) TSV_KCLASS(1) TSV_KCLASS(2) TSV_KCLASS(3)
#undef TSV_KCLASS
  return {mask_class(lo[0], lo[1], lo[2], lo[3]), mask_class(hi[0], hi[1], hi[2], hi[3])};
}

// Operand pre-split for Karatsuba (lo, hi, lo^hi halves, 4 classes each):
// a multiplier reused across products (z_head along a head's runs) is split
// once and cached.
struct KSplit {
  Split4 l, h, m;
};

__device__ __forceinline__ KSplit ksplit(uint64_t a) {
  return {split4(lo32(a)), split4(hi32(a)), split4(lo32(a) ^ hi32(a))};
}

__device__ __forceinline__ u128 clmul64_kara_s(const KSplit& A, const KSplit& B) {
  uint64_t lo[4], hi[4];
#define TSV_KSCLASS(R)                                         \
  {                                                            \
    const uint64_t L = class_prod<R>(A.l, B.l);                \
    const uint64_t H = class_prod<R>(A.h, B.h);                \
    const uint64_t M = class_prod<R>(A.m, B.m) ^ L ^ H;        \
    lo[R] = L ^ (M << 32);                                     \
    hi[R] = H ^ (M >> 32);                                     \
  }
  TSV_KSCLASS(0) TSV_KSCLASS(1) TSV_KSCLASS(2) TSV_KSCLASS(3)
#undef TSV_KSCLASS
  return {mask_class(lo[0], lo[1], lo[2], lo[3]), mask_class(hi[0], hi[1], hi[2], hi[3])};
}

// Sums of carry-less products in raw Karatsuba class form: the class
// products L, H, M of every term are XORed as they come and combined, masked
// (mask_class) and reduced ONCE for the whole sum -- all three steps are
// linear over XOR.  For sums of several products (the z map's
// S[T] = XOR_j z_j * U[T - {j}]) this saves the per-product combine and mask.
struct ClassAcc {
  uint64_t L[4], H[4], M[4];
};

__device__ __forceinline__ void class_zero(ClassAcc& c) {
#pragma unroll
  for (int r = 0; r < 4; ++r) c.L[r] = c.H[r] = c.M[r] = 0;
}

__device__ __forceinline__ void class_acc(const KSplit& A, const KSplit& B, ClassAcc& c) {
  c.L[0] ^= class_prod<0>(A.l, B.l);
  c.L[1] ^= class_prod<1>(A.l, B.l);
  c.L[2] ^= class_prod<2>(A.l, B.l);
  c.L[3] ^= class_prod<3>(A.l, B.l);
  c.H[0] ^= class_prod<0>(A.h, B.h);
  c.H[1] ^= class_prod<1>(A.h, B.h);
  c.H[2] ^= class_prod<2>(A.h, B.h);
  c.H[3] ^= class_prod<3>(A.h, B.h);
  c.M[0] ^= class_prod<0>(A.m, B.m);
  c.M[1] ^= class_prod<1>(A.m, B.m);
  c.M[2] ^= class_prod<2>(A.m, B.m);
  c.M[3] ^= class_prod<3>(A.m, B.m);
}

__device__ __forceinline__ u128 class_finish(const ClassAcc& c) {
  uint64_t lo[4], hi[4];
#pragma unroll
  for (int r = 0; r < 4; ++r) {
    const uint64_t M = c.M[r] ^ c.L[r] ^ c.H[r];
    lo[r] = c.L[r] ^ (M << 32);
    hi[r] = c.H[r] ^ (M >> 32);
  }
  return {mask_class(lo[0], lo[1], lo[2], lo[3]), mask_class(hi[0], hi[1], hi[2], hi[3])};
}

// Schoolbook over 32-bit halves with deferred class masking.
__device__ __forceinline__ u128 clmul64_school(uint64_t a, uint64_t b) {
  const Split4 al = split4(lo32(a)), ah = split4(hi32(a));
  const Split4 bl = split4(lo32(b)), bh = split4(hi32(b));
  uint64_t lo[4], hi[4];
#define TSV_SCLASS(R)                                                  \
  {                                                                    \
    const uint64_t L = class_prod<R>(al, bl);                          \
    const uint64_t H = class_prod<R>(ah, bh);                          \
    const uint64_t M = class_prod<R>(al, bh) ^ class_prod<R>(ah, bl);  \
    lo[R] = L ^ (M << 32);                                             \
    hi[R] = H ^ (M >> 32);                                             \
  }
  TSV_SCLASS(0) TSV_SCLASS(1) TSV_SCLASS(2) TSV_SCLASS(3)
#undef TSV_SCLASS
  return {mask_class(lo[0], lo[1], lo[2], lo[3]), mask_class(hi[0], hi[1], hi[2], hi[3])};
}

// ---- period-5 holes: class sums accumulate inside the multiplier ----------
//
// With operands masked to every 5th bit, a 32x32 product has at most
// min(p+1, 63-p) <= 31 one-bit products at position p once all 5 products of
// an output class are SUMMED, which fits the 5-bit field: the class sum is
// one chain of mul.wide with accumulate (no XORs).  The single exception is
// p = 31 with x = y = 0xffffffff (32 products): its field wraps to 0 (right
// parity) and carries one unit into p = 36, which the correction undoes.

__device__ __forceinline__ uint64_t wmad(uint32_t a, uint32_t b, uint64_t c) {
  uint64_t r;
  asm("mad.wide.u32 %0, %1, %2, %3;" : "=l"(r) : "r"(a), "r"(b), "l"(c));
  return r;
}

struct Split5 {
  uint32_t c[5];
};

__device__ __forceinline__ Split5 split5(uint32_t a) {
  return {{a & 0x42108421u, a & 0x84210842u, a & 0x08421084u, a & 0x10842108u,
           a & 0x21084210u}};
}

// 32x32 -> 64 carry-less product (masked), period-5 holes.
__device__ __forceinline__ uint64_t clmul32_p5(const Split5& x, const Split5& y, bool full) {
  uint64_t c[5];
#pragma unroll
  for (int r = 0; r < 5; ++r) {
    uint64_t s = wmul(x.c[0], y.c[r]);
#pragma unroll
    for (int i = 1; i < 5; ++i) s = wmad(x.c[i], y.c[(r - i + 5) % 5], s);
    c[r] = s;
  }
  if (full) c[1] ^= 1ull << 36;
  return (c[0] & 0x1084210842108421ull) | (c[1] & 0x2108421084210842ull) |
         (c[2] & 0x4210842108421084ull) | (c[3] & 0x8421084210842108ull) |
         (c[4] & 0x0842108421084210ull);
}

struct KSplit5 {
  Split5 l, h, m;
  bool fl, fh, fm;  // operand half is all ones
};

__device__ __forceinline__ KSplit5 ksplit5(uint64_t a) {
  const uint32_t l = lo32(a), h = hi32(a), m = l ^ h;
  return {split5(l), split5(h), split5(m), l == 0xffffffffu, h == 0xffffffffu,
          m == 0xffffffffu};
}

__device__ __forceinline__ u128 clmul64_p5(const KSplit5& A, const KSplit5& B) {
  const uint64_t L = clmul32_p5(A.l, B.l, A.fl && B.fl);
  const uint64_t H = clmul32_p5(A.h, B.h, A.fh && B.fh);
  const uint64_t M = clmul32_p5(A.m, B.m, A.fm && B.fm) ^ L ^ H;
  return {L ^ (M << 32), H ^ (M >> 32)};
}

// Shifts issued on the FMA pipe (IMAD.SHL / IMAD.HI) instead of the ALU pipe,
// which the carry-less XOR network already saturates.
__device__ __forceinline__ uint32_t shl_f(uint32_t x, uint32_t pow2) {
  uint32_t r;
  asm("mul.lo.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(pow2));
  return r;
}
__device__ __forceinline__ uint32_t shr_f(uint32_t x, uint32_t pow2_32ms) {
  uint32_t r;
  asm("mul.hi.u32 %0, %1, %2;" : "=r"(r) : "r"(x), "r"(pow2_32ms));
  return r;
}

// Reduce a 128-bit carry-less product modulo x^64 + x^4 + x^3 + x + 1:
// h * x^64 == h * (x^4 + x^3 + x + 1), folded twice.  Written on 32-bit
// halves so every shift is a multiply (FMA pipe) and every combine an XOR.
__device__ __forceinline__ uint64_t gf_reduce(u128 p) {
  const uint32_t hl = lo32(p.hi), hh = hi32(p.hi);
  const uint32_t over = shr_f(hh, 2u) ^ shr_f(hh, 8u) ^ shr_f(hh, 16u);  // bits 63,61,60
  const uint32_t lo = lo32(p.lo) ^ hl ^ shl_f(hl, 2u) ^ shl_f(hl, 8u) ^ shl_f(hl, 16u) ^ over ^
                      shl_f(over, 2u) ^ shl_f(over, 8u) ^ shl_f(over, 16u);
  const uint32_t hi = hi32(p.lo) ^ hh ^ shl_f(hh, 2u) ^ shl_f(hh, 8u) ^ shl_f(hh, 16u) ^
                      shr_f(hl, 2u) ^ shr_f(hl, 8u) ^ shr_f(hl, 16u);
  return pack(lo, hi);
}

__device__ __forceinline__ uint64_t gf_mul_kara(uint64_t a, uint64_t b) {
  return gf_reduce(clmul64_kara(a, b));
}
__device__ __forceinline__ uint64_t gf_mul_p5(uint64_t a, uint64_t b) {
  return gf_reduce(clmul64_p5(ksplit5(a), ksplit5(b)));
}
__device__ __forceinline__ uint64_t gf_mul_presplit5(const KSplit5& a, uint64_t b) {
  return gf_reduce(clmul64_p5(a, ksplit5(b)));
}
__device__ __forceinline__ uint64_t gf_mul_presplit(const KSplit& a, uint64_t b) {
  return gf_reduce(clmul64_kara_s(a, ksplit(b)));
}
__device__ __forceinline__ uint64_t gf_mul_school(uint64_t a, uint64_t b) {
  return gf_reduce(clmul64_school(a, b));
}

// Production general multiply (selected by tsv_gf_bench measurements).
__device__ __forceinline__ uint64_t gf_mul(uint64_t a, uint64_t b) {
  return gf_mul_kara(a, b);
}

// a * x in the field.
__device__ __forceinline__ uint64_t gf_mulx(uint64_t a) {
  return (a << 1) ^ ((a >> 63) * 0x1bull);
}

// a * x^s, 0 <= s <= 60, in one fold (the overflow has <= 60 bits).
__device__ __forceinline__ uint64_t gf_mul_xpow(uint64_t a, int s) {
  if (s == 0) return a;
  const uint64_t h = a >> (64 - s);
  return (a << s) ^ h ^ (h << 1) ^ (h << 3) ^ (h << 4);
}

// Bit-serial product (Horner over the bits of b); independent check path.
__device__ __forceinline__ uint64_t gf_mul_serial(uint64_t a, uint64_t b) {
  uint64_t r = 0;
  for (int i = 63; i >= 0; --i) {
    r = gf_mulx(r);
    if ((b >> i) & 1) r ^= a;
  }
  return r;
}

// ---- products by a warp-uniform multiplier --------------------------------

// tab: 256 u64 in shared memory, private to one warp.  build() must be called
// by all 32 lanes of the warp with the same y; mul() by any lane afterwards.
struct GfTable {
  // Window i (the 16 multiples c * x^(4i) * y) starts at byte 136*i: the
  // 8-byte pad per window spreads the build's stores over all banks (two
  // wavefronts per 8-byte store instead of sixteen) at no instruction cost,
  // and a window's 16 entries still span 128 contiguous bytes, so lookups
  // stay conflict-free.  Table footprint: kWords u64, a multiple of 256
  // bytes so that consecutive tables stay 256-byte aligned.
  static constexpr int kWinBytes = 136;
  static constexpr int kWords = (16 * kWinBytes + 255) / 256 * 256 / 8;
  uint64_t* tab;

  template <int OFF>
  __device__ __forceinline__ static void sts(uint32_t addr, uint64_t v) {
    asm volatile("st.shared.u64 [%0+%1], %2;" ::"r"(addr), "n"(OFF), "l"(v) : "memory");
  }

  // Lane L writes entries 8*(L&1) .. 8*(L&1)+7 of window i = L>>1, i.e.
  // the 64 bytes at offset 136*i + 64*(L&1): c * x^(4i) * y for
  // c = 8*(L&1) + e, e < 8.  Branch-free (the window shift is a clamped PTX
  // shift) and stored as 8-byte stores.
  __device__ __forceinline__ void build(uint64_t y, int lane) {
    const uint32_t s = 4u * static_cast<uint32_t>(lane >> 1);
    uint64_t h, lo;
    asm("shr.b64 %0, %1, %2;" : "=l"(h) : "l"(y), "r"(64u - s));  // 0 when s == 0
    asm("shl.b64 %0, %1, %2;" : "=l"(lo) : "l"(y), "r"(s));
    const uint64_t B0 = lo ^ h ^ (h << 1) ^ (h << 3) ^ (h << 4);  // y * x^s (s <= 60)
    const uint64_t B1 = gf_mulx(B0), B2 = gf_mulx(B1);
    const uint64_t base = (lane & 1) ? gf_mulx(B2) : 0ull;
    const uint32_t a = static_cast<uint32_t>(__cvta_generic_to_shared(tab)) +
                       kWinBytes * static_cast<uint32_t>(lane >> 1) + 64u * (lane & 1);
    sts<0>(a, base);
    sts<8>(a, base ^ B0);
    sts<16>(a, base ^ B1);
    sts<24>(a, base ^ B1 ^ B0);
    sts<32>(a, base ^ B2);
    sts<40>(a, base ^ B2 ^ B0);
    sts<48>(a, base ^ B2 ^ B1);
    sts<56>(a, base ^ B2 ^ B1 ^ B0);
  }

  // Lookups: nibble j of s, scaled by 8, is placed into the low byte of the
  // table's shared-memory address with one byte permute (the table is
  // 256-byte aligned); the window offset j*136 rides in the load immediate.
  template <int OFF>
  __device__ __forceinline__ static uint64_t lds(uint32_t addr) {
    uint64_t v;
    asm volatile("ld.shared.u64 %0, [%1+%2];" : "=l"(v) : "r"(addr), "n"(OFF));
    return v;
  }

  template <int WIN>
  __device__ __forceinline__ static uint64_t word8(uint32_t w, uint32_t base) {
    const uint32_t e = shl_f(w, 8u) & 0x78787878u;          // nibbles 0,2,4,6 (x8)
    const uint32_t o = shr_f(w, 0x80000000u) & 0x78787878u; // nibbles 1,3,5,7 (x8)
    uint64_t a = lds<(WIN + 0) * kWinBytes>(__byte_perm(e, base, 0x7650)) ^
                 lds<(WIN + 1) * kWinBytes>(__byte_perm(o, base, 0x7650));
    a ^= lds<(WIN + 2) * kWinBytes>(__byte_perm(e, base, 0x7651)) ^
         lds<(WIN + 3) * kWinBytes>(__byte_perm(o, base, 0x7651));
    a ^= lds<(WIN + 4) * kWinBytes>(__byte_perm(e, base, 0x7652)) ^
         lds<(WIN + 5) * kWinBytes>(__byte_perm(o, base, 0x7652));
    a ^= lds<(WIN + 6) * kWinBytes>(__byte_perm(e, base, 0x7653)) ^
         lds<(WIN + 7) * kWinBytes>(__byte_perm(o, base, 0x7653));
    return a;
  }

  __device__ __forceinline__ uint64_t mul(uint64_t s) const {
    const uint32_t base = static_cast<uint32_t>(__cvta_generic_to_shared(tab));
    return word8<0>(lo32(s), base) ^ word8<8>(hi32(s), base);
  }
};

// ---- products by a PER-LANE multiplier reused for several products ---------
//
// LaneTable: every lane keeps the 16 multiples c * y (c a polynomial of
// degree < 4, fully reduced) of ITS OWN multiplier y in shared memory, laid
// out [c][lane] (4 KB per warp, 4 KB aligned): a lane's entries live in its
// own bank pair whatever c is, so the 16 nibble lookups of a product never
// conflict, and the table is private to the lane (no warp barrier).  A
// product is x * y = XOR_w T[x_w] * X^(4w): the two nibbles at the same
// position of x's 32-bit halves are paired (word-aligned, free) and the 8
// pairs combined by Horner steps of 4 bits on a 128-bit accumulator.  No
// integer multiplies: 16 LDS.64 and ~100 ALU instructions per product
// against 48 quarter-rate IMAD.WIDE and ~120 ALU for the holes product; the
// build (3 doublings, 11 XORs, 15 stores) is paid once per multiplier.
struct LaneTable {
  uint32_t base;  // shared address of T[0][lane]; bits 8..11 are zero
  uint32_t brep;  // byte 1 of base in all four bytes

  // tab_saddr: shared-space address of the warp's 4 KB table (4 KB aligned)
  __device__ __forceinline__ void init(uint32_t tab_saddr, int lane) {
    base = tab_saddr + 8u * static_cast<uint32_t>(lane);
    brep = ((base >> 8) & 0xffu) * 0x01010101u;
    asm volatile("st.shared.v2.u32 [%0], {%1, %1};" ::"r"(base), "r"(0u) : "memory");
  }

  template <int C>
  __device__ __forceinline__ void sts(uint64_t v) const {
    asm volatile("st.shared.v2.u32 [%0+%1], {%2, %3};" ::"r"(base), "n"(C * 256), "r"(lo32(v)),
                 "r"(hi32(v))
                 : "memory");
  }

  __device__ __forceinline__ void build(uint64_t y) const {
    const uint64_t y2 = gf_mulx(y), y4 = gf_mulx(y2), y8 = gf_mulx(y4);
    const uint64_t y3 = y ^ y2, y5 = y ^ y4, y6 = y2 ^ y4, y7 = y3 ^ y4;
    sts<1>(y);
    sts<2>(y2);
    sts<3>(y3);
    sts<4>(y4);
    sts<5>(y5);
    sts<6>(y6);
    sts<7>(y7);
    sts<8>(y8);
    sts<9>(y ^ y8);
    sts<10>(y2 ^ y8);
    sts<11>(y3 ^ y8);
    sts<12>(y4 ^ y8);
    sts<13>(y5 ^ y8);
    sts<14>(y6 ^ y8);
    sts<15>(y7 ^ y8);
  }

  // T[nibble in byte B of m]: m's bytes are nibbles OR'ed with brep, so one
  // byte permute forms the address base + 256 * nibble.  `gen` is a token of
  // the last build (orders the loads after it for the compiler).
  template <int B>
  __device__ __forceinline__ void look(uint32_t m, uint32_t gen, uint32_t& lo, uint32_t& hi) const {
    const uint32_t addr = __byte_perm(m, base, 0x7604 | (B << 4));
    asm("ld.shared.v2.u32 {%0, %1}, [%2]; // %3" : "=r"(lo), "=r"(hi) : "r"(addr), "r"(gen));
  }

  // 128-bit carry-less x * y (y's multiples reduced, so < 2^124)
  __device__ __forceinline__ u128 clmul(uint64_t x, uint32_t gen) const {
    const uint32_t xl = lo32(x), xh = hi32(x);
    // nibbles r = 0,2,4,6 (e*) and 1,3,5,7 (o*) of each half, one per byte
    const uint32_t el = (xl & 0x0f0f0f0fu) | brep, ol = ((xl >> 4) & 0x0f0f0f0fu) | brep;
    const uint32_t eh = (xh & 0x0f0f0f0fu) | brep, oh = ((xh >> 4) & 0x0f0f0f0fu) | brep;
    uint32_t w0, w1, w2, w3 = 0;
#define TSV_LT_STEP(FIRST, ML, MH, B)                                   \
  {                                                                     \
    uint32_t a0, a1, b0, b1;                                            \
    look<B>(ML, gen, a0, a1);                                           \
    look<B>(MH, gen, b0, b1);                                           \
    if (FIRST) {                                                        \
      w0 = a0;                                                          \
      w1 = a1 ^ b0;                                                     \
      w2 = b1;                                                          \
    } else {                                                            \
      w3 = __funnelshift_l(w2, w3, 4);                                  \
      w2 = __funnelshift_l(w1, w2, 4) ^ b1;                             \
      w1 = __funnelshift_l(w0, w1, 4) ^ a1 ^ b0;                        \
      w0 = (w0 << 4) ^ a0;                                              \
    }                                                                   \
  }
    TSV_LT_STEP(true, ol, oh, 3)   // nibble 7 of each half
    TSV_LT_STEP(false, el, eh, 3)  // 6
    TSV_LT_STEP(false, ol, oh, 2)  // 5
    TSV_LT_STEP(false, el, eh, 2)  // 4
    TSV_LT_STEP(false, ol, oh, 1)  // 3
    TSV_LT_STEP(false, el, eh, 1)  // 2
    TSV_LT_STEP(false, ol, oh, 0)  // 1
    TSV_LT_STEP(false, el, eh, 0)  // 0
#undef TSV_LT_STEP
    return {pack(w0, w1), pack(w2, w3)};
  }
};

// Reduction of a LaneTable::clmul product: it is below 2^124 (reduced
// multiples shifted by at most 60 bits), so the high word has no bit above
// 59 and one fold by x^4 + x^3 + x + 1 finishes it.
__device__ __forceinline__ uint64_t gf_reduce124(u128 p) {
  const uint64_t h = p.hi;
  return p.lo ^ h ^ (h << 1) ^ (h << 3) ^ (h << 4);
}

// Reduction of a 128-bit carry-less product with ALU shifts only.
__device__ __forceinline__ uint64_t gf_reduce_shift(u128 p) {
  const uint64_t h = p.hi;
  const uint64_t over = (h >> 60) ^ (h >> 61) ^ (h >> 63);
  const uint64_t f1 = h ^ (h << 1) ^ (h << 3) ^ (h << 4);
  return p.lo ^ f1 ^ over ^ (over << 1) ^ (over << 3) ^ (over << 4);
}

// ---- host field arithmetic (a handful of products per evaluation) -------

// GF(2^64) product mod x^64 + x^4 + x^3 + x + 1, bit-serial (gf.hpp:55-65, 85-106).
inline uint64_t gf_mul_host(uint64_t a, uint64_t b) {
  uint64_t r = 0;
  for (int i = 0; i < 64; ++i) {
    if ((b >> i) & 1ull) r ^= a;
    a = (a << 1) ^ ((a >> 63) ? 0x1bull : 0ull);
  }
  return r;
}

// a^(2^64 - 2) = a^-1 (a != 0).
inline uint64_t gf_inv_host(uint64_t a) {
  uint64_t r = 1, sq = a;
  for (int i = 1; i < 64; ++i) {  // exponent bits 1..63 are set, bit 0 is not
    sq = gf_mul_host(sq, sq);
    r = gf_mul_host(r, sq);
  }
  return r;
}

// Determinant of the row-major k x k matrix m (Gaussian elimination; in
// characteristic 2 it equals the permanent).
inline uint64_t gf_det_host(const uint64_t* m, int k) {
  uint64_t a[32 * 32];
  for (int i = 0; i < k * k; ++i) a[i] = m[i];
  uint64_t det = 1;
  for (int c = 0; c < k; ++c) {
    int p = c;
    while (p < k && a[p * k + c] == 0) ++p;
    if (p == k) return 0;
    if (p != c)
      for (int j = 0; j < k; ++j) std::swap(a[p * k + j], a[c * k + j]);
    det = gf_mul_host(det, a[c * k + c]);
    const uint64_t inv = gf_inv_host(a[c * k + c]);
    for (int r = c + 1; r < k; ++r) {
      const uint64_t f = gf_mul_host(a[r * k + c], inv);
      if (f)
        for (int j = c; j < k; ++j) a[r * k + j] ^= gf_mul_host(f, a[c * k + j]);
    }
  }
  return det;
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
__host__ __device__ __forceinline__ uint64_t draw_prefix(uint64_t seed, uint64_t role) {
  uint64_t h = seed + 0x9e3779b97f4a7c15ull;
  return mix64(h ^ (role * 0xff51afd7ed558ccdull));
}

__host__ __device__ __forceinline__ uint64_t draw_nonzero_from(uint64_t pre, uint64_t a,
                                                               uint64_t b, uint64_t c) {
  uint64_t h = mix64(pre ^ (a + 0xc2b2ae3d27d4eb4full));
  h = mix64(h ^ (b + 0x165667b19e3779f9ull));
  h = mix64(h ^ (c + 0x27d4eb2f165667c5ull));
  while (h == 0) h = mix64(h + 0x9e3779b97f4a7c15ull);
  return h;
}

__host__ __device__ __forceinline__ uint64_t draw_nonzero(uint64_t seed, uint64_t role,
                                                          uint64_t a, uint64_t b, uint64_t c) {
  return draw_nonzero_from(draw_prefix(seed, role), a, b, c);
}

// y(e, l-1) = draw_nonzero(seed, edge_y, e, l-1, 0) with the (seed, role)
// prefix hoisted; yb = (l-1) + the round-3 constant.
__device__ __forceinline__ uint64_t draw_edge_y(uint64_t pre, uint64_t yb, uint32_t edge) {
  uint64_t h = mix64(pre ^ (static_cast<uint64_t>(edge) + 0xc2b2ae3d27d4eb4full));
  h = mix64(h ^ yb);
  h = mix64(h ^ 0x27d4eb2f165667c5ull);  // c = 0
  while (h == 0) h = mix64(h + 0x9e3779b97f4a7c15ull);
  return h;
}

}  // namespace tsv
