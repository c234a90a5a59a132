// quake_b200/quake.hpp — C++ drop-in for the reference's quake:: operator API.
//
// Same namespace, types and signatures as the reference headers
// core/include/quake/kernels.hpp (:39-171) and core/include/quake/nonlin.hpp
// (:32-97) (paths relative to /root/reference/proj/), implemented over the
// C-ABI in quake_b200.h: a caller that included "quake/kernels.hpp" and
// "quake/nonlin.hpp" includes this header instead and links
// libquake_b200.so. Preconditions throw std::invalid_argument with the
// reference's messages; CUDA failures throw std::runtime_error. Every
// operator — scalar forms included — runs on the GPU; there is no CPU path.
#ifndef QUAKE_B200_QUAKE_HPP_
#define QUAKE_B200_QUAKE_HPP_

#include <cstddef>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>
#include <vector>

#include "../quake_b200.h"

namespace quake {

using NumericBuffer = std::vector<float>;  // buffer.hpp:27

enum class KernelChoice { Exact = QK_EXACT, Quake = QK_QUAKE, Quake2 = QK_QUAKE2 };

struct AffineCoeffs {  // kernels.hpp:39-46
  float c0;
  float c1;
  float input_scale;
  float input_shift;
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

struct SoftmaxParams {  // nonlin.hpp:43-49
  float temperature = 1.0f;
  std::optional<bool> centering_bias;
  QuadCoeffs quad = QuadCoeffs::continuity();
};

struct GeluConstants {  // nonlin.hpp:55-62
  float kappa;
  float root2_over_pi;
  float fused_scale;
  float inverse_kappa;
  static GeluConstants defaults() {
    const qk_gelu_constants g = qk_gelu_constants_defaults();
    return {g.kappa, g.root2_over_pi, g.fused_scale, g.inverse_kappa};
  }
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
inline int32_t bias_arg(std::optional<bool> b) { return b.has_value() ? (*b ? 1 : 0) : -1; }
inline qk_softmax_params to_c(const SoftmaxParams& p) {
  return {p.temperature, bias_arg(p.centering_bias), to_c(p.quad)};
}

}  // namespace b200_detail

inline constexpr double kCenteringBias = 0.0436;  // kernels.hpp:29

inline const char* kernel_name(KernelChoice k) {
  return qk_kernel_name(static_cast<qk_kernel>(k));
}
inline bool resolve_centering_bias(KernelChoice k, std::optional<bool> requested) {
  return qk_resolve_centering_bias(static_cast<qk_kernel>(k), b200_detail::bias_arg(requested)) != 0;
}

// ---- kernels.hpp:47-93 coefficient derivation (FpFormat: single only) ----
inline AffineCoeffs coeffs_for(float p, float q, bool centering_bias = false) {
  qk_affine_coeffs c;
  b200_detail::check(qk_coeffs_for(p, q, centering_bias ? 1 : 0, &c));
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
inline ClampRange default_clamp(float p, float q) {
  qk_clamp_range r;
  b200_detail::check(qk_default_clamp(p, q, &r));
  return {r.lo, r.hi};
}
inline ClampRange clamp_for(const AffineCoeffs& c) {
  const qk_affine_coeffs cc = b200_detail::to_c(c);
  const qk_clamp_range r = qk_clamp_for(&cc);
  return {r.lo, r.hi};
}

// ---- kernels.hpp:163-171 buffer operators ----
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

// ---- kernels.hpp:141-155, kernels.cpp:92-96 scalar forms (GPU-evaluated) ----
inline float quake(float x, const AffineCoeffs& c, const ClampRange& r) {
  float y = 0.0f;
  quake_buffer(std::span<const float>(&x, 1), std::span<float>(&y, 1), c, r);
  return y;
}
inline float quake2(float x, const AffineCoeffs& c, const QuadCoeffs& a, const ClampRange& r) {
  float y = 0.0f;
  quake2_buffer(std::span<const float>(&x, 1), std::span<float>(&y, 1), c, a, r);
  return y;
}
inline float quake(float x, const AffineCoeffs& c) { return quake(x, c, clamp_for(c)); }
inline float quake2(float x, const AffineCoeffs& c, const QuadCoeffs& a = QuadCoeffs::continuity()) {
  return quake2(x, c, a, clamp_for(c));
}

// ---- nonlin.hpp:70-97 ----
inline void softmax_row(std::span<const float> v, const SoftmaxParams& params, KernelChoice kernel,
                        std::span<float> out) {
  const qk_softmax_params p = b200_detail::to_c(params);
  b200_detail::check(qk_softmax_row(v.data(), v.size(), &p, static_cast<qk_kernel>(kernel),
                                    out.data(), out.size()));
}
inline NumericBuffer softmax_row(std::span<const float> v, const SoftmaxParams& params,
                                 KernelChoice kernel) {
  NumericBuffer out(v.size());
  softmax_row(v, params, kernel, out);
  return out;
}
inline void softmax_rows(std::span<const float> matrix, std::size_t cols,
                         const SoftmaxParams& params, KernelChoice kernel, std::span<float> out) {
  const qk_softmax_params p = b200_detail::to_c(params);
  b200_detail::check(qk_softmax_rows(matrix.data(), matrix.size(), cols, &p,
                                     static_cast<qk_kernel>(kernel), out.data(), out.size()));
}
inline NumericBuffer softmax_rows(std::span<const float> matrix, std::size_t cols,
                                  const SoftmaxParams& params, KernelChoice kernel) {
  NumericBuffer out(matrix.size());
  softmax_rows(matrix, cols, params, kernel, out);
  return out;
}
inline void logistic_buffer(std::span<const float> xs, std::span<float> out, KernelChoice kernel,
                            std::optional<bool> centering_bias = std::nullopt) {
  b200_detail::check(qk_logistic_buffer(xs.data(), xs.size(), out.data(), out.size(),
                                        static_cast<qk_kernel>(kernel),
                                        b200_detail::bias_arg(centering_bias)));
}
inline float logistic(float x, KernelChoice kernel,
                      std::optional<bool> centering_bias = std::nullopt) {
  float y = 0.0f;
  logistic_buffer(std::span<const float>(&x, 1), std::span<float>(&y, 1), kernel, centering_bias);
  return y;
}
inline void gelu_buffer(std::span<const float> xs, std::span<float> out, KernelChoice kernel,
                        std::optional<bool> centering_bias = std::nullopt) {
  b200_detail::check(qk_gelu_buffer(xs.data(), xs.size(), out.data(), out.size(),
                                    static_cast<qk_kernel>(kernel),
                                    b200_detail::bias_arg(centering_bias)));
}
inline float gelu(float x, KernelChoice kernel, std::optional<bool> centering_bias = std::nullopt) {
  float y = 0.0f;
  gelu_buffer(std::span<const float>(&x, 1), std::span<float>(&y, 1), kernel, centering_bias);
  return y;
}

}  // namespace quake

#endif  // QUAKE_B200_QUAKE_HPP_
