// quake/nonlin.hpp (drop-in) — softmax, logistic and GELU on the GPU.
//
// Source-compatible with the reference's core/include/quake/nonlin.hpp
// (:28-97, paths relative to /root/reference/proj/), implemented over the
// C-ABI in quake_b200.h. Softmax keeps the reference's contract: every row
// is validated before anything is written to `out` (nonlin.cpp:176-180),
// and results do not depend on how rows are partitioned across GPUs.
#ifndef QUAKE_B200_QUAKE_NONLIN_HPP_
#define QUAKE_B200_QUAKE_NONLIN_HPP_

#include <cstddef>
#include <optional>
#include <span>

#include "buffer.hpp"
#include "kernels.hpp"

namespace quake {

enum class KernelChoice { Exact = QK_EXACT, Quake = QK_QUAKE, Quake2 = QK_QUAKE2 };  // :32

inline const char* kernel_name(KernelChoice k) {  // nonlin.cpp:120-130
  return qk_kernel_name(static_cast<qk_kernel>(k));
}
inline bool resolve_centering_bias(KernelChoice k, std::optional<bool> requested) {  // :39-41
  return qk_resolve_centering_bias(static_cast<qk_kernel>(k),
                                   b200_detail::bias_arg(requested)) != 0;
}

struct SoftmaxParams {  // :43-49
  float temperature = 1.0f;
  std::optional<bool> centering_bias;
  QuadCoeffs quad = QuadCoeffs::continuity();
};

struct GeluConstants {  // :55-62, nonlin.cpp:132-141
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
inline qk_softmax_params to_c(const SoftmaxParams& p) {
  return {p.temperature, bias_arg(p.centering_bias), to_c(p.quad)};
}
}  // namespace b200_detail

// ---- softmax (:70-81, nonlin.cpp:143-189) ----
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

// ---- logistic (:83-88, nonlin.cpp:198-243) ----
inline float logistic(float x, KernelChoice kernel,
                      std::optional<bool> centering_bias = std::nullopt) {
  float y = 0.0f;
  b200_detail::check(qk_logistic(x, static_cast<qk_kernel>(kernel),
                                 b200_detail::bias_arg(centering_bias), &y));
  return y;
}
inline void logistic_buffer(std::span<const float> xs, std::span<float> out, KernelChoice kernel,
                            std::optional<bool> centering_bias = std::nullopt) {
  b200_detail::check(qk_logistic_buffer(xs.data(), xs.size(), out.data(), out.size(),
                                        static_cast<qk_kernel>(kernel),
                                        b200_detail::bias_arg(centering_bias)));
}

// ---- GELU (:90-97, nonlin.cpp:248-330) ----
inline float gelu(float x, KernelChoice kernel, std::optional<bool> centering_bias = std::nullopt) {
  float y = 0.0f;
  b200_detail::check(qk_gelu(x, static_cast<qk_kernel>(kernel),
                             b200_detail::bias_arg(centering_bias), &y));
  return y;
}
inline void gelu_buffer(std::span<const float> xs, std::span<float> out, KernelChoice kernel,
                        std::optional<bool> centering_bias = std::nullopt) {
  b200_detail::check(qk_gelu_buffer(xs.data(), xs.size(), out.data(), out.size(),
                                    static_cast<qk_kernel>(kernel),
                                    b200_detail::bias_arg(centering_bias)));
}

}  // namespace quake

#endif  // QUAKE_B200_QUAKE_NONLIN_HPP_
