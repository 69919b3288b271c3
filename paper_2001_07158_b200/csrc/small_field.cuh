// small_field.cuh -- GF(2^b) arithmetic for b in {8, 16, 32} (gf.hpp:36-42,
// 85-97, 147-153), shared by the temporal point form (small_field.cu) and the
// static / junction projection sieve (static_kernels.cu).  Values travel in
// uint64_t words with the high bits zero; fmul / fdraw_y pick the 64-bit
// product and draw for BITS == 64, so one kernel template serves every width.
#pragma once

#include <cstdint>

#include "gf_device.cuh"

namespace tsv {

template <typename Word>
struct SmallField;
template <>
struct SmallField<uint8_t> {
  static constexpr int kBits = 8;
  static constexpr uint64_t kLow = 0x1b;  // x^8 + x^4 + x^3 + x + 1
};
template <>
struct SmallField<uint16_t> {
  static constexpr int kBits = 16;
  static constexpr uint64_t kLow = 0x2b;  // x^16 + x^5 + x^3 + x + 1
};
template <>
struct SmallField<uint32_t> {
  static constexpr int kBits = 32;
  static constexpr uint64_t kLow = 0x8d;  // x^32 + x^7 + x^3 + x^2 + 1
};

// gf::mul<Word> for b <= 32 (gf.hpp:85-97): the 64-bit carry-less product
// (the holes product of gf_device.cuh on 32-bit operands), overflow bits
// scanned from the top and cleared with shifted copies of the modulus.
template <typename Word>
__device__ __forceinline__ Word smul(Word a, Word b) {
  constexpr int nb = SmallField<Word>::kBits;
  constexpr uint64_t poly = (uint64_t{1} << nb) | SmallField<Word>::kLow;
  const Split4 sa = split4(a), sb = split4(b);
  uint64_t p = mask_class(class_prod<0>(sa, sb), class_prod<1>(sa, sb), class_prod<2>(sa, sb),
                          class_prod<3>(sa, sb));
#pragma unroll
  for (int bit = 2 * nb - 2; bit >= nb; --bit)
    if ((p >> bit) & 1ull) p ^= poly << (bit - nb);
  return static_cast<Word>(p);
}

// draw_nonzero<Word> (gf.hpp:147-153) with the (seed, role) rounds hoisted:
// the 64-bit draw truncated to b bits, re-mixed while the truncation is zero
template <typename Word>
__device__ __forceinline__ Word sdraw(uint64_t pre, uint64_t a, uint64_t b, uint64_t c) {
  uint64_t h = mix64(pre ^ (a + 0xc2b2ae3d27d4eb4full));
  h = mix64(h ^ (b + 0x165667b19e3779f9ull));
  h = mix64(h ^ (c + 0x27d4eb2f165667c5ull));
  while (static_cast<Word>(h) == 0) h = mix64(h + 0x9e3779b97f4a7c15ull);
  return static_cast<Word>(h);
}

template <int BITS>
struct WordOf;
template <>
struct WordOf<8> { using type = uint8_t; };
template <>
struct WordOf<16> { using type = uint16_t; };
template <>
struct WordOf<32> { using type = uint32_t; };

// product in GF(2^BITS) of two words holding field elements
template <int BITS>
__device__ __forceinline__ uint64_t fmul(uint64_t a, uint64_t b) {
  if constexpr (BITS == 64) {
    return gf_mul(a, b);
  } else {
    using W = typename WordOf<BITS>::type;
    return static_cast<uint64_t>(smul<W>(static_cast<W>(a), static_cast<W>(b)));
  }
}

// y(e, level) = draw_nonzero<Word>(seed, role, e, level, 0); yb is the 64-bit
// path's hoisted (level + round-2 constant) of draw_edge_y
template <int BITS>
__device__ __forceinline__ uint64_t fdraw_y(uint64_t pre, uint64_t yb, uint64_t level,
                                            uint32_t edge) {
  if constexpr (BITS == 64) {
    return draw_edge_y(pre, yb, edge);
  } else {
    using W = typename WordOf<BITS>::type;
    return static_cast<uint64_t>(sdraw<W>(pre, static_cast<uint64_t>(edge), level, 0));
  }
}

}  // namespace tsv
