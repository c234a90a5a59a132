// quake/bitcore.hpp (drop-in) — word carrier, float layout and bit helpers.
//
// Source-compatible with the reference's core/include/quake/bitcore.hpp
// (:26-82, paths relative to /root/reference/proj/): the same names, types and
// values, so code written against the reference compiles unchanged with
// -I <repo>/include/quake_b200. These are host-side reinterpretations with
// no arithmetic of their own; every QuAKE evaluation runs on the GPU (see
// quake/kernels.hpp).
#ifndef QUAKE_B200_QUAKE_BITCORE_HPP_
#define QUAKE_B200_QUAKE_BITCORE_HPP_

#include <bit>
#include <cstdint>

namespace quake {

// Raw IEEE-754 binary32 bit pattern (bitcore.hpp:26).
using Word32 = std::uint32_t;

// Exponent width, mantissa width and exponent bias of a binary format
// (bitcore.hpp:32-53). Coefficient derivation takes any format; the kernels
// assemble 32-bit words.
struct FpFormat {
  int exponent_bits;
  int mantissa_bits;
  int bias;

  static constexpr FpFormat single() { return FpFormat{8, 23, 127}; }
  constexpr bool standard_bias() const { return bias == (1 << (exponent_bits - 1)) - 1; }
  constexpr Word32 mantissa_mask() const { return (Word32{1} << mantissa_bits) - Word32{1}; }
  constexpr Word32 sign_exponent_mask() const { return ~mantissa_mask(); }
  constexpr Word32 unit_exponent_bits() const {
    return static_cast<Word32>(bias) << mantissa_bits;  // the word of 1.0
  }
};

inline constexpr FpFormat kSingle = FpFormat::single();

// binary32 field masks (bitcore.hpp:59-61).
inline constexpr Word32 kMantissaMask = kSingle.mantissa_mask();            // 0x007FFFFF
inline constexpr Word32 kSignExponentMask = kSingle.sign_exponent_mask();   // 0xFF800000
inline constexpr Word32 kUnitExponentBits = kSingle.unit_exponent_bits();   // 0x3F800000
static_assert(kMantissaMask == 0x007FFFFFu && kSignExponentMask == 0xFF800000u &&
              kUnitExponentBits == 0x3F800000u);

// Bit reinterpretation, both directions exact (NaN payloads kept).
inline Word32 float_bits_as_int(float x) { return std::bit_cast<Word32>(x); }
inline float int_bits_as_float(Word32 w) { return std::bit_cast<float>(w); }

// Value conversion toward zero; the argument must fit int32 (bitcore.hpp:75-77).
inline std::int32_t convert_to_int(float x) { return static_cast<std::int32_t>(x); }

inline Word32 extract_mantissa_field(Word32 w, const FpFormat& fmt = kSingle) {
  return w & fmt.mantissa_mask();
}

}  // namespace quake

#endif  // QUAKE_B200_QUAKE_BITCORE_HPP_
