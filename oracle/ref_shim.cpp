// TEST INFRASTRUCTURE ONLY — extern "C" wrappers around the reference
// library, compiled in place from /root/reference/proj/core/src by
// oracle/Makefile into oracle/_ref/libquake_ref.so. Used by tests/ (to pin
// the C restatement and to generate tests/golden/), and by bench.py's
// cpu_baseline and --impl reference legs (the reference's own CPU path,
// timed on the host cores). Never linked into the product library.
//
// Each wrapper calls exactly one public reference entry point:
//   kernels.hpp:163-171 quake_buffer / quake2_buffer
//   nonlin.hpp:70-97    softmax_row(s), logistic_buffer, gelu_buffer
//   kernels.hpp:47-51, 86-88   coeffs_for / clamp_for / default_clamp
//   oracle.hpp:28-42    exact_* ground truth
//   bench.hpp:74-83     fusion_ablation (checksums pin the unfused restatement)
//   lab.hpp:70-125      sweep_error, quad_max_rel_err, grid_search_quad,
//                       continuity_probe, bias_reoptimize (pin the GPU lab)
#include <cstring>
#include <optional>
#include <span>
#include <stdexcept>
#include <string>

#include <random>

#include "quake/bench.hpp"
#include "quake/kernels.hpp"
#include "quake/lab.hpp"
#include "quake/nonlin.hpp"
#include "quake/oracle.hpp"
#include "quake/parallel.hpp"

namespace {

thread_local std::string g_last_error;

quake::KernelChoice kernel_of(int k) {
  switch (k) {
    case 1: return quake::KernelChoice::Quake;
    case 2: return quake::KernelChoice::Quake2;
    default: return quake::KernelChoice::Exact;
  }
}

std::optional<bool> bias_of(int b) {
  if (b < 0) return std::nullopt;
  return b != 0;
}

template <typename Fn>
int guarded(Fn&& fn) {
  try {
    fn();
    return 0;
  } catch (const std::invalid_argument& e) {
    g_last_error = e.what();
    return 1;
  } catch (const std::exception& e) {
    g_last_error = e.what();
    return 2;
  }
}

}  // namespace

extern "C" {

const char* ref_last_error() { return g_last_error.c_str(); }

unsigned ref_effective_threads() { return quake::effective_threads(); }

int ref_coeffs_for(float p, float q, int bias, float* c0, float* c1) {
  return guarded([&] {
    const quake::AffineCoeffs c = quake::coeffs_for(p, q, quake::kSingle, bias != 0);
    *c0 = c.c0;
    *c1 = c.c1;
  });
}

int ref_default_clamp(float p, float q, float* lo, float* hi) {
  return guarded([&] {
    const quake::ClampRange r = quake::default_clamp(p, q);
    *lo = r.lo;
    *hi = r.hi;
  });
}

void ref_clamp_for(float c0, float c1, float* lo, float* hi) {
  quake::AffineCoeffs c{c0, c1, 0.0f, 0.0f, false};
  const quake::ClampRange r = quake::clamp_for(c);
  *lo = r.lo;
  *hi = r.hi;
}

void ref_named_coeffs(int which, int bias, float* c0, float* c1) {
  // 0 natural, 1 base2, 2 negated natural (kernels.cpp:42-54)
  quake::AffineCoeffs c = which == 0   ? quake::natural_exp_coeffs(bias != 0)
                          : which == 1 ? quake::base2_coeffs(bias != 0)
                                       : quake::negated_natural_exp_coeffs(bias != 0);
  *c0 = c.c0;
  *c1 = c.c1;
}

float ref_quake(float x, float c0, float c1, float lo, float hi) {
  quake::AffineCoeffs c{c0, c1, 0.0f, 0.0f, false};
  return quake::quake(x, c, quake::ClampRange{lo, hi});
}

float ref_quake2(float x, float c0, float c1, float a0, float a1, float a2, float lo,
                 float hi) {
  quake::AffineCoeffs c{c0, c1, 0.0f, 0.0f, false};
  return quake::quake2(x, c, quake::QuadCoeffs{a0, a1, a2}, quake::ClampRange{lo, hi});
}

int ref_quake_buffer(const float* xs, size_t n, float* out, float c0, float c1, float lo,
                     float hi) {
  return guarded([&] {
    quake::AffineCoeffs c{c0, c1, 0.0f, 0.0f, false};
    quake::quake_buffer(std::span<const float>(xs, n), std::span<float>(out, n), c,
                        quake::ClampRange{lo, hi});
  });
}

int ref_quake2_buffer(const float* xs, size_t n, float* out, float c0, float c1, float a0,
                      float a1, float a2, float lo, float hi) {
  return guarded([&] {
    quake::AffineCoeffs c{c0, c1, 0.0f, 0.0f, false};
    quake::quake2_buffer(std::span<const float>(xs, n), std::span<float>(out, n), c,
                         quake::QuadCoeffs{a0, a1, a2}, quake::ClampRange{lo, hi});
  });
}

int ref_logistic_buffer(const float* xs, size_t n, float* out, int kernel, int bias) {
  return guarded([&] {
    quake::logistic_buffer(std::span<const float>(xs, n), std::span<float>(out, n),
                           kernel_of(kernel), bias_of(bias));
  });
}

int ref_gelu_buffer(const float* xs, size_t n, float* out, int kernel, int bias) {
  return guarded([&] {
    quake::gelu_buffer(std::span<const float>(xs, n), std::span<float>(out, n),
                       kernel_of(kernel), bias_of(bias));
  });
}

float ref_logistic(float x, int kernel, int bias) {
  return quake::logistic(x, kernel_of(kernel), bias_of(bias));
}

float ref_gelu(float x, int kernel, int bias) {
  return quake::gelu(x, kernel_of(kernel), bias_of(bias));
}

int ref_softmax_rows(const float* m, size_t n, size_t cols, float temperature, int bias,
                     float a0, float a1, float a2, int kernel, float* out, size_t out_n) {
  return guarded([&] {
    quake::SoftmaxParams p;
    p.temperature = temperature;
    p.centering_bias = bias_of(bias);
    p.quad = quake::QuadCoeffs{a0, a1, a2};
    quake::softmax_rows(std::span<const float>(m, n), cols, p, kernel_of(kernel),
                        std::span<float>(out, out_n));
  });
}

int ref_softmax_row(const float* v, size_t n, float temperature, int bias, float a0,
                    float a1, float a2, int kernel, float* out, size_t out_n) {
  return guarded([&] {
    quake::SoftmaxParams p;
    p.temperature = temperature;
    p.centering_bias = bias_of(bias);
    p.quad = quake::QuadCoeffs{a0, a1, a2};
    quake::softmax_row(std::span<const float>(v, n), p, kernel_of(kernel),
                       std::span<float>(out, out_n));
  });
}

void ref_gelu_constants(float* kappa, float* r2pi, float* fused_scale, float* inverse_kappa) {
  const quake::GeluConstants g = quake::GeluConstants::defaults();
  *kappa = g.kappa;
  *r2pi = g.root2_over_pi;
  *fused_scale = g.fused_scale;
  *inverse_kappa = g.inverse_kappa;
}

double ref_exact_exp(double x) { return quake::oracle::exact_exp(x); }
double ref_exact_logistic(double x) { return quake::oracle::exact_logistic(x); }
double ref_exact_gelu_tanh(double x) { return quake::oracle::exact_gelu_tanh(x); }

int ref_exact_softmax(const float* v, size_t n, double t, double* out) {
  return guarded([&] {
    quake::oracle::exact_softmax(std::span<const float>(v, n), t, std::span<double>(out, n));
  });
}

// The reference bench's input generator (bench.cpp:48-60 input_range,
// :341-348 fill_inputs): mt19937_64(seed), uniform float in the workload's
// range; workload 0 softmax_matrix, 1 gelu_vector, 2 exp_vector, 3 logistic_vector.
void ref_bench_inputs(int workload, size_t count, uint64_t seed, float* out) {
  static const float lo[] = {-8.0f, -6.0f, -20.0f, -12.0f};
  static const float hi[] = {8.0f, 6.0f, 20.0f, 12.0f};
  std::mt19937_64 rng(seed);
  std::uniform_real_distribution<float> dist(lo[workload], hi[workload]);
  for (size_t i = 0; i < count; ++i) out[i] = dist(rng);
}

// bench.cpp:425-513 fusion_ablation: the checksums (sum of outputs in
// double) of the fused and unfused passes and their max relative divergence.
int ref_fusion_ablation(int workload, int kernel, size_t rows, size_t cols, size_t n,
                        float temperature, uint64_t seed, double* fused_checksum,
                        double* unfused_checksum, double* divergence) {
  return guarded([&] {
    quake::bench::BenchConfig cfg;
    cfg.workload = workload == 0 ? quake::bench::Workload::SoftmaxMatrix
                                 : quake::bench::Workload::GeluVector;
    cfg.rows = rows;
    cfg.cols = cols;
    cfg.n = n;
    cfg.kernel = kernel_of(kernel);
    cfg.temperature = temperature;
    cfg.seed = seed;
    const quake::bench::AblationReport r = quake::bench::fusion_ablation(cfg);
    *fused_checksum = r.fused.checksum;
    *unfused_checksum = r.unfused.checksum;
    *divergence = r.max_rel_divergence;
  });
}

namespace {
quake::lab::ExpConfig exp_config(int kind, int natural, int bias, float a0, float a1, float a2) {
  quake::lab::ExpConfig c;
  c.kind = kernel_of(kind);
  c.natural_base = natural != 0;
  c.centering_bias = bias != 0;
  c.quad = quake::QuadCoeffs{a0, a1, a2};
  return c;
}
}  // namespace

int ref_sweep_error(int kind, int natural, int bias, float a0, float a1, float a2, float lo,
                    float hi, uint64_t uniform_samples, uint32_t period_stride,
                    uint64_t* samples, double* max_rel, double* mean_rel, float* argmax) {
  return guarded([&] {
    quake::lab::SweepSpec spec{lo, hi, uniform_samples, period_stride};
    const quake::lab::ErrorReport r =
        quake::lab::sweep_error(exp_config(kind, natural, bias, a0, a1, a2), spec);
    *samples = r.samples;
    *max_rel = r.max_rel_err;
    *mean_rel = r.mean_rel_err;
    *argmax = r.argmax_input;
  });
}

double ref_quad_max_rel_err(double a0, double a1, double a2, size_t intervals) {
  return quake::lab::quad_max_rel_err(a0, a1, a2, intervals);
}

int ref_grid_search_quad(const double* axes /* 9: lo, hi, step x3 */, float* best,
                         double* best_err, uint64_t* points) {
  return guarded([&] {
    quake::lab::GridSpec g;
    g.a0 = {axes[0], axes[1], axes[2]};
    g.a1 = {axes[3], axes[4], axes[5]};
    g.a2 = {axes[6], axes[7], axes[8]};
    const quake::lab::GridSearchResult r = quake::lab::grid_search_quad(g);
    best[0] = r.best.a0;
    best[1] = r.best.a1;
    best[2] = r.best.a2;
    *best_err = r.best_max_rel_err;
    *points = r.points_searched;
  });
}

int ref_continuity_probe(int kind, int natural, int bias, float a0, float a1, float a2,
                         int k_lo, int k_hi, double* worst, float* at) {
  return guarded([&] {
    const quake::lab::ContinuityReport r = quake::lab::continuity_probe(
        exp_config(kind, natural, bias, a0, a1, a2), k_lo, k_hi);
    *worst = r.worst_jump;
    *at = r.at;
  });
}

int ref_bias_reoptimize(int kind, int natural, int bias, float a0, float a1, float a2,
                        double beta_lo, double beta_hi, float* beta, double* max_rel,
                        int* near) {
  return guarded([&] {
    const quake::lab::BiasSearchResult r = quake::lab::bias_reoptimize(
        exp_config(kind, natural, bias, a0, a1, a2), beta_lo, beta_hi);
    *beta = r.beta;
    *max_rel = r.max_rel_err;
    *near = r.near_reference_bias ? 1 : 0;
  });
}

}  // extern "C"
