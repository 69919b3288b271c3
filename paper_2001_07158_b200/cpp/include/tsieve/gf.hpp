// tsieve/gf.hpp -- host-side field arithmetic and counter-based draws.
//
// API of /root/reference/proj/core/include/tsieve/gf.hpp (add :47-50,
// mul<Word> :85-106, Role :111-119, draw64 :135-143, draw_nonzero :147-153,
// SeededStream :157-170), re-implemented.  The sieve itself never runs these
// on the host: the device copies live in csrc/gf_device.cuh.  They exist here
// so host code written against the reference keeps compiling and produces
// the same values.
#pragma once

#include <cstdint>
#include <type_traits>

namespace tsieve::gf {

template <typename Word>
concept FieldWord = std::is_same_v<Word, std::uint8_t> || std::is_same_v<Word, std::uint16_t> ||
                    std::is_same_v<Word, std::uint32_t> || std::is_same_v<Word, std::uint64_t>;

template <FieldWord Word>
inline constexpr int field_bits = static_cast<int>(sizeof(Word)) * 8;

// Low word of the irreducible modulus (the x^b term is implicit).
template <FieldWord Word>
inline constexpr Word modulus_low = static_cast<Word>(
    sizeof(Word) == 1 ? 0x1b : sizeof(Word) == 2 ? 0x2b : sizeof(Word) == 4 ? 0x8d : 0x1b);

template <FieldWord Word>
constexpr Word add(Word a, Word b) {
  return static_cast<Word>(a ^ b);
}

// Product by shift-and-reduce (Horner over the bits of b).
template <FieldWord Word>
constexpr Word mul(Word a, Word b) {
  constexpr int nb = field_bits<Word>;
  Word r = 0;
  for (int i = nb - 1; i >= 0; --i) {
    const bool top = (r >> (nb - 1)) & 1;
    r = static_cast<Word>(r << 1);
    if (top) r ^= modulus_low<Word>;
    if ((b >> i) & 1) r ^= a;
  }
  return r;
}

enum class Role : std::uint64_t {
  shade_v = 1,
  shade_w = 2,
  edge_y = 3,
  edge_y2 = 4,
  label_z = 5,
  stream = 6,
  walk = 7,
};

namespace detail {
constexpr std::uint64_t finalize(std::uint64_t x) {
  x = (x ^ (x >> 30)) * 0xbf58476d1ce4e5b9ull;
  x = (x ^ (x >> 27)) * 0x94d049bb133111ebull;
  return x ^ (x >> 31);
}
}  // namespace detail

constexpr std::uint64_t draw64(std::uint64_t seed, Role role, std::uint64_t a, std::uint64_t b,
                               std::uint64_t c) {
  std::uint64_t h = detail::finalize((seed + 0x9e3779b97f4a7c15ull) ^
                                     (static_cast<std::uint64_t>(role) * 0xff51afd7ed558ccdull));
  h = detail::finalize(h ^ (a + 0xc2b2ae3d27d4eb4full));
  h = detail::finalize(h ^ (b + 0x165667b19e3779f9ull));
  return detail::finalize(h ^ (c + 0x27d4eb2f165667c5ull));
}

template <FieldWord Word>
constexpr Word draw_nonzero(std::uint64_t seed, Role role, std::uint64_t a, std::uint64_t b,
                            std::uint64_t c) {
  std::uint64_t h = draw64(seed, role, a, b, c);
  while (static_cast<Word>(h) == 0) h = detail::finalize(h + 0x9e3779b97f4a7c15ull);
  return static_cast<Word>(h);
}

struct SeededStream {
  std::uint64_t seed = 0;
  std::uint64_t pos = 0;
  template <FieldWord Word>
  Word next_nonzero() {
    return draw_nonzero<Word>(seed, Role::stream, pos++, 0, 0);
  }
  template <FieldWord Word>
  Word nonzero_at(std::uint64_t i) const {
    return draw_nonzero<Word>(seed, Role::stream, i, 0, 0);
  }
};

}  // namespace tsieve::gf
