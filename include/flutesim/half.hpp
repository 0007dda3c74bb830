// flute-b200 — IEEE binary16 host numerics.
//
// Drop-in for the reference's half.hpp (reference: proj/include/flutesim/
// half.hpp:14-93): same type and function names, same semantics (RNE
// narrowing, overflow to signed infinity, exact subnormals, quiet NaNs with
// the top payload bits kept; exact widening; f16 add via binary32).  On the
// device the same arithmetic is done by native __half / HMUL2 instructions; the
// host keeps this software form for packing, table building and the API.
#pragma once

#include <bit>
#include <cstdint>

namespace flutesim {

struct Half {
  std::uint16_t bits = 0;

  static constexpr Half from_bits(std::uint16_t b) { return Half{b}; }
  constexpr std::uint16_t to_bits() const { return bits; }

  friend constexpr bool operator==(Half a, Half b) { return a.bits == b.bits; }
  friend constexpr bool operator!=(Half a, Half b) { return a.bits != b.bits; }
};

namespace detail {
// v / 2^sh rounded to nearest, ties to even; sh >= 1.
constexpr std::uint32_t round_shift_even(std::uint32_t v, int sh) {
  if (sh >= 32) return 0;
  const std::uint32_t q = v >> sh;
  const std::uint32_t rem = v & ((1u << sh) - 1u);
  const std::uint32_t half = 1u << (sh - 1);
  return q + ((rem > half || (rem == half && (q & 1u))) ? 1u : 0u);
}
}  // namespace detail

constexpr std::uint16_t f32_bits_to_f16_bits(std::uint32_t u) {
  const auto s = static_cast<std::uint16_t>((u >> 16) & 0x8000u);
  const std::uint32_t a = u & 0x7FFFFFFFu;
  if (a > 0x7F800000u) {  // NaN: force quiet, keep the top payload bits
    return static_cast<std::uint16_t>(s | 0x7E00u | ((a & 0x7FFFFFu) >> 13));
  }
  if (a == 0x7F800000u) return static_cast<std::uint16_t>(s | 0x7C00u);
  const int biased = static_cast<int>(a >> 23);
  if (biased == 0) return s;  // binary32 zero/subnormal: below half's reach
  const std::uint32_t sig = (a & 0x7FFFFFu) | 0x800000u;
  const int e = biased - 127;
  if (e >= -14) {
    const std::uint32_t r = detail::round_shift_even(sig, 13);  // [1024, 2048]
    const std::uint32_t h = (static_cast<std::uint32_t>(e + 15) << 10) + (r - 1024u);
    return static_cast<std::uint16_t>(s | (h >= 0x7C00u ? 0x7C00u : h));
  }
  // Subnormal half (quantum 2^-24); a carry to 1024 is the smallest normal.
  return static_cast<std::uint16_t>(s | detail::round_shift_even(sig, 13 + (-14 - e)));
}

constexpr std::uint32_t f16_bits_to_f32_bits(std::uint16_t h) {
  const std::uint32_t s = static_cast<std::uint32_t>(h & 0x8000u) << 16;
  const std::uint32_t e = (h >> 10) & 0x1Fu;
  const std::uint32_t m = h & 0x3FFu;
  if (e == 0x1Fu) return s | 0x7F800000u | (m << 13);
  if (e != 0) return s | ((e + 112u) << 23) | (m << 13);
  if (m == 0) return s;
  // Subnormal: the leading one sits at bit (w-1); renormalise.
  const int w = std::bit_width(m);
  return s | (static_cast<std::uint32_t>(w + 102) << 23) | ((m << (24 - w)) & 0x7FFFFFu);
}

inline Half f32_to_f16(float x) {
  return Half::from_bits(f32_bits_to_f16_bits(std::bit_cast<std::uint32_t>(x)));
}

inline float f16_to_f32(Half h) { return std::bit_cast<float>(f16_bits_to_f32_bits(h.bits)); }

// Binary32 sum rounded back to binary16 (the reference's partial-sum rule).
inline Half f16_add(Half a, Half b) { return f32_to_f16(f16_to_f32(a) + f16_to_f32(b)); }

}  // namespace flutesim
