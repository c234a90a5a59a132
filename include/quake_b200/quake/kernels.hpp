// quake/kernels.hpp (drop-in) — QuAKE exponential kernels on the GPU.
//
// Source-compatible with the reference's core/include/quake/kernels.hpp
// (:26-171, paths relative to /root/reference/proj/): same namespace, types,
// signatures and default arguments, implemented over the C-ABI in
// quake_b200.h (libquake_b200.so). Compile reference callers with
// -I <repo>/include/quake_b200 and link -lquake_b200.
//
//  * coefficient derivation: the reference's fp64 formulas, bit-identical,
//    for any FpFormat (kernels.cpp:25-87);
//  * buffer operators: the sm_100a kernels (host, pinned or device spans);
//  * scalar forms quake()/quake2(): one element through the same kernels via
//    a per-thread pinned mailbox (one small launch per call; batch through
//    the buffer forms for throughput).
// Preconditions throw std::invalid_argument with the reference's messages;
// CUDA failures throw std::runtime_error.
#ifndef QUAKE_B200_QUAKE_KERNELS_HPP_
#define QUAKE_B200_QUAKE_KERNELS_HPP_

#include <cmath>
#include <numbers>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>

#include "../../quake_b200.h"
#include "bitcore.hpp"
#include "buffer.hpp"

namespace quake {

inline constexpr double kCenteringBias = 0.0436;  // kernels.hpp:29

struct AffineCoeffs {  // kernels.hpp:39-46
  float c0;
  float c1;
  float input_scale;  // p
  float input_shift;  // q
  bool bias_applied;
};

struct QuadCoeffs {  // kernels.hpp:60-76
  float a0;
  float a1;
  float a2;
  static constexpr QuadCoeffs continuity() { return {1.0f / 3.0f, 0.0f, 2.0f / 3.0f}; }
  static constexpr QuadCoeffs minimax() { return {0.33f, -0.017f, 0.68f}; }
  constexpr bool is_continuity_default() const {
    return a0 == 1.0f / 3.0f && a1 == 0.0f && a2 == 2.0f / 3.0f;
  }
};

struct ClampRange {  // kernels.hpp:81-84
  float lo;
  float hi;
};

namespace b200_detail {

inline void check(qk_status s) {
  if (s == QK_OK) return;
  if (qk_is_invalid_argument(s)) throw std::invalid_argument(qk_last_error());
  throw std::runtime_error(std::string("quake_b200: ") + qk_last_error());
}
inline qk_affine_coeffs to_c(const AffineCoeffs& c) {
  return {c.c0, c.c1, c.input_scale, c.input_shift, c.bias_applied ? 1 : 0};
}
inline AffineCoeffs from_c(const qk_affine_coeffs& c) {
  return {c.c0, c.c1, c.input_scale, c.input_shift, c.bias_applied != 0};
}
inline qk_quad_coeffs to_c(const QuadCoeffs& a) { return {a.a0, a.a1, a.a2}; }
inline qk_clamp_range to_c(const ClampRange& r) { return {r.lo, r.hi}; }
inline qk_fp_format to_c(const FpFormat& f) { return {f.exponent_bits, f.mantissa_bits, f.bias}; }
inline int32_t bias_arg(std::optional<bool> b) { return b.has_value() ? (*b ? 1 : 0) : -1; }

}  // namespace b200_detail

// ---- coefficient derivation (kernels.hpp:47-93, kernels.cpp:25-87) ----
inline AffineCoeffs coeffs_for(float p, float q, const FpFormat& fmt = kSingle,
                               bool centering_bias = false) {
  const qk_fp_format f = b200_detail::to_c(fmt);
  qk_affine_coeffs c;
  b200_detail::check(qk_coeffs_for_format(p, q, &f, centering_bias ? 1 : 0, &c));
  return b200_detail::from_c(c);
}
inline AffineCoeffs natural_exp_coeffs(bool centering_bias = true) {
  return b200_detail::from_c(qk_natural_exp_coeffs(centering_bias ? 1 : 0));
}
inline AffineCoeffs base2_coeffs(bool centering_bias = false) {
  return b200_detail::from_c(qk_base2_coeffs(centering_bias ? 1 : 0));
}
inline AffineCoeffs negated_natural_exp_coeffs(bool centering_bias = true) {
  return b200_detail::from_c(qk_negated_natural_exp_coeffs(centering_bias ? 1 : 0));
}
inline ClampRange default_clamp(float p, float q, const FpFormat& fmt = kSingle) {
  const qk_fp_format f = b200_detail::to_c(fmt);
  qk_clamp_range r;
  b200_detail::check(qk_default_clamp_format(p, q, &f, &r));
  return {r.lo, r.hi};
}
inline ClampRange clamp_for(const AffineCoeffs& c) {
  const qk_affine_coeffs cc = b200_detail::to_c(c);
  const qk_clamp_range r = qk_clamp_for(&cc);
  return {r.lo, r.hi};
}

// ---- scalar forms (kernels.hpp:141-155, kernels.cpp:92-96), GPU-evaluated ----
inline float quake(float x, const AffineCoeffs& c, const ClampRange& r) {
  const qk_affine_coeffs cc = b200_detail::to_c(c);
  const qk_clamp_range rr = b200_detail::to_c(r);
  float y = 0.0f;
  b200_detail::check(qk_quake(x, &cc, &rr, &y));
  return y;
}
inline float quake2(float x, const AffineCoeffs& c, const QuadCoeffs& a, const ClampRange& r) {
  const qk_affine_coeffs cc = b200_detail::to_c(c);
  const qk_quad_coeffs aa = b200_detail::to_c(a);
  const qk_clamp_range rr = b200_detail::to_c(r);
  float y = 0.0f;
  b200_detail::check(qk_quake2(x, &cc, &aa, &rr, &y));
  return y;
}
inline float quake(float x, const AffineCoeffs& c) { return quake(x, c, clamp_for(c)); }
inline float quake2(float x, const AffineCoeffs& c, const QuadCoeffs& a = QuadCoeffs::continuity()) {
  return quake2(x, c, a, clamp_for(c));
}

// ---- buffer operators (kernels.hpp:163-171, kernels.cpp:95-136) ----
inline void quake_buffer(std::span<const float> xs, std::span<float> out, const AffineCoeffs& c,
                         const ClampRange& r) {
  const qk_affine_coeffs cc = b200_detail::to_c(c);
  const qk_clamp_range rr = b200_detail::to_c(r);
  b200_detail::check(qk_quake_buffer(xs.data(), xs.size(), out.data(), out.size(), &cc, &rr));
}
inline void quake2_buffer(std::span<const float> xs, std::span<float> out, const AffineCoeffs& c,
                          const QuadCoeffs& a, const ClampRange& r) {
  const qk_affine_coeffs cc = b200_detail::to_c(c);
  const qk_quad_coeffs aa = b200_detail::to_c(a);
  const qk_clamp_range rr = b200_detail::to_c(r);
  b200_detail::check(
      qk_quake2_buffer(xs.data(), xs.size(), out.data(), out.size(), &cc, &aa, &rr));
}
inline NumericBuffer quake_buffer(std::span<const float> xs, const AffineCoeffs& c,
                                  const ClampRange& r) {
  NumericBuffer out(xs.size());
  quake_buffer(xs, out, c, r);
  return out;
}
inline NumericBuffer quake2_buffer(std::span<const float> xs, const AffineCoeffs& c,
                                   const QuadCoeffs& a, const ClampRange& r) {
  NumericBuffer out(xs.size());
  quake2_buffer(xs, out, c, a, r);
  return out;
}

}  // namespace quake

#endif  // QUAKE_B200_QUAKE_KERNELS_HPP_
