/*
 * quake_b200_lab.h — GPU accuracy lab.
 *
 * The reference's numerical lab (core/include/quake/lab.hpp:30-125,
 * core/src/lab.cpp) evaluated on the sm_100a device functions of the
 * product kernels, so every approximation it measures is the GPU's own
 * (bit-identical to the reference's). Same configuration structs, error
 * messages and result semantics as the reference; in addition,
 * qk_sweep_exhaustive walks EVERY binary32 input of a range — full fp32
 * resolution, which the reference's CPU sweep samples — and checks
 * monotonicity across consecutive floats and positivity on the way.
 *
 * Determinism: per-block partials are combined in index order; maxima keep
 * the first (lowest-index) input attaining them, as lab.cpp:86-107 does.
 * Ground truth is exp / exp2 in binary64 on the device (CUDA libdevice,
 * <= 1 ulp of binary64; the reference uses the host libm).
 */
#ifndef QUAKE_B200_LAB_H_
#define QUAKE_B200_LAB_H_

#include "quake_b200.h"

#ifdef __cplusplus
extern "C" {
#endif

/* lab.hpp:30-44 ExpConfig: kernel, base, centering bias, quadratic. */
typedef struct {
  qk_kernel kind;          /* QK_EXACT, QK_QUAKE or QK_QUAKE2 */
  int32_t natural_base;    /* 1: e^x (input scale log2e); 0: 2^x (scale 1) */
  int32_t centering_bias;  /* c1 carries the 0.0436 centering offset */
  qk_quad_coeffs quad;     /* QK_QUAKE2 refinement (continuity default) */
} qk_exp_config;

/* lab.hpp:46-55 SweepSpec */
typedef struct {
  float lo, hi;
  uint64_t uniform_samples; /* uniform grid over [lo, hi] (>= 10^4) */
  uint32_t period_stride;   /* stride of the walk over one mantissa period; 0 = off */
} qk_sweep_spec;

/* lab.hpp:57-66 ErrorReport */
typedef struct {
  float lo, hi;
  uint64_t samples;
  double max_rel_err;
  double mean_rel_err;
  float argmax_input;
} qk_error_report;

/* Every binary32 x in [lo, hi] (both zeros included), increasing order. */
typedef struct {
  float lo, hi;
  uint64_t samples;
  double max_rel_err;
  double mean_rel_err;
  float argmax_input;
  uint64_t monotonic_violations; /* consecutive x < x' with y(x) > y(x') */
  float first_violation;         /* the x of the first violating pair (NaN if none) */
  uint64_t non_positive;         /* y <= 0 or y not finite */
  float first_non_positive;      /* NaN if none */
} qk_exhaustive_report;

/* lab.hpp:105-108 ContinuityReport */
typedef struct {
  double worst_jump;
  float at;
} qk_continuity_report;

/* lab.hpp:72-95 grid search */
typedef struct {
  double lo, hi, step;
} qk_grid_axis;
typedef struct {
  qk_grid_axis a0, a1, a2;
} qk_grid_spec;
typedef struct {
  qk_quad_coeffs best;
  double best_max_rel_err;
  double step_a0, step_a1, step_a2;
  uint64_t points_searched;
} qk_grid_result;

/* lab.hpp:115-121 BiasSearchResult */
typedef struct {
  float beta;
  double max_rel_err;
  int32_t near_reference_bias; /* |beta - 0.0436| <= 0.0035 */
} qk_bias_result;

/* The lab's default specs: lab.hpp:46-55, 80-84. */
qk_sweep_spec qk_sweep_spec_defaults(void);
qk_grid_spec qk_grid_spec_defaults(void);

/* ExpConfig::coeffs / clamp (lab.cpp:121-129). */
qk_status qk_lab_coeffs(const qk_exp_config* cfg, qk_affine_coeffs* c, qk_clamp_range* r);
/* lab.cpp:150-200 sweep_error: uniform grid + one exhaustive mantissa period. */
qk_status qk_sweep_error(const qk_exp_config* cfg, const qk_sweep_spec* spec,
                         qk_error_report* out);
/* Every binary32 in [lo, hi]: error band, monotonicity, positivity. lo/hi
 * must lie inside the kernel's clamp range (QuAKE kinds). */
qk_status qk_sweep_exhaustive(const qk_exp_config* cfg, float lo, float hi,
                              qk_exhaustive_report* out);
/* lab.cpp:281-328 continuity_probe over exponent steps k in [k_lo, k_hi]. */
qk_status qk_continuity_probe(const qk_exp_config* cfg, int32_t k_lo, int32_t k_hi,
                              qk_continuity_report* out);
/* lab.cpp:209-219 quad_max_rel_err (intervals + 1 points over [1, 2]). */
qk_status qk_quad_max_rel_err(double a0, double a1, double a2, uint64_t intervals, double* out);
/* lab.cpp:221-279 grid_search_quad (coarse 512, best 2048 at 2^16, winner at 2^20). */
qk_status qk_grid_search_quad(const qk_grid_spec* spec, qk_grid_result* out);
/* lab.cpp:330-410 bias_reoptimize (golden section over [beta_lo, beta_hi]). */
qk_status qk_bias_reoptimize(const qk_exp_config* cfg, double beta_lo, double beta_hi,
                             qk_bias_result* out);

#ifdef __cplusplus
}  /* extern "C" */
#endif

#endif /* QUAKE_B200_LAB_H_ */
