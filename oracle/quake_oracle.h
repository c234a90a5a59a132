/*
 * TEST INFRASTRUCTURE ONLY — CPU oracle for the QuAKE hot path.
 *
 * This is a plain-C restatement of the reference's arithmetic, used as the
 * parity checker by tests/, __graft_entry__.smoke() and bench.py's
 * cpu_baseline / --impl reference legs. The product path (the CUDA library
 * in paper_2412_00408_b200/) never links, loads or calls anything here.
 *
 * Every function cites the reference file:line it restates; paths are
 * relative to /root/reference/proj/. Parity is pinned two ways:
 *   - against the reference compiled in place (oracle/_ref, see Makefile),
 *   - against the golden vectors in tests/golden/ (generated from oracle/_ref
 *     by tests/golden/make_golden.py) and the reference tests' in-test
 *     known answers (test_kernels.cpp, test_nonlin.cpp).
 *
 * Build: gcc -O2 -std=c11 -ffp-contract=off (no -march): the reference's
 * Release build has no FMA contraction, so neither may this.
 */
#ifndef QUAKE_ORACLE_H_
#define QUAKE_ORACLE_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum { OR_EXACT = 0, OR_QUAKE = 1, OR_QUAKE2 = 2 };
/* Unfused ablation variants of the bench passes (bench.cpp:137-166 softmax,
 * :212-233 GELU): the affine transform is computed explicitly and fed to
 * the plain natural / negated-natural exponential kernel. Softmax and GELU
 * only; the centering bias resolves as for the base kernel. */
enum { OR_QUAKE_UNFUSED = 5, OR_QUAKE2_UNFUSED = 6 };

/* Status codes (match include/quake_b200.h's qk_status for the shared cases). */
enum {
  OR_OK = 0,
  OR_ERR_SIZE_MISMATCH = 1,
  OR_ERR_NOT_DIVISIBLE = 2,
  OR_ERR_BAD_TEMPERATURE = 3,
  OR_ERR_EMPTY_ROW = 4,
  OR_ERR_NON_FINITE = 5,
  OR_ERR_ZERO_SLOPE = 6
};

/* kernels.cpp:25-40 (coeffs_for); kernels.cpp:61-87 (solve_clamp / clamp_for). */
int or_coeffs_for(float p, float q, int centering_bias, float* c0, float* c1);
void or_clamp_for(float c0, float c1, float* lo, float* hi);
int or_default_clamp(float p, float q, float* lo, float* hi);

/* kernels.hpp:97-136 scalar bodies. */
float or_quake(float x, float c0, float c1, float lo, float hi);
float or_quake2(float x, float c0, float c1, float a0, float a1, float a2,
                float lo, float hi);

/* kernels.cpp:95-136 buffer forms. */
void or_quake_buffer(const float* xs, float* out, size_t n, float c0, float c1,
                     float lo, float hi);
void or_quake2_buffer(const float* xs, float* out, size_t n, float c0, float c1,
                      float a0, float a1, float a2, float lo, float hi);

/* nonlin.cpp:210-243 (logistic_buffer); bias < 0 selects the per-kernel default. */
void or_logistic_buffer(const float* xs, float* out, size_t n, int kernel, int bias);
/* nonlin.cpp:292-330 (gelu_buffer). */
void or_gelu_buffer(const float* xs, float* out, size_t n, int kernel, int bias);

/* nonlin.cpp:162-189 (softmax_rows). sum_mode 0 = the reference's sequential
 * fp32 row sum (nonlin.cpp:63-67); sum_mode 1 = fp64 row sum, the restatement
 * SURVEY.md F5/H3 uses for vocab-length rows. Returns OR_* status; on error
 * `out` is untouched (nonlin.cpp:176-180). */
int or_softmax_rows(const float* m, size_t n, size_t cols, float temperature,
                    int bias, float a0, float a1, float a2, int kernel,
                    int sum_mode, float* out);

/* Same arithmetic as or_softmax_rows (QuAKE kernels only), but each row is
 * summed in the declared order of the GPU kernels (paper_2412_00408_b200/
 * csrc/softmax.cu): the row (in chunks of `width` consecutive elements) is
 * cut into `cluster` slices — `balanced`: the first nchunks % cluster slices
 * get one extra chunk; else `slice` chunks each, the last short; slice 0 =
 * one slice. Lane l of `lanes` adds the elements of chunks l, l+lanes, ... of
 * its slice in index order; lanes combine by butterfly (xor 16..1 inside a
 * warp, then over warp results zero-padded to a power of two); slice
 * partials are added sequentially in slice order. Only the reference's
 * sequential fp32 sum (nonlin.cpp:63-67) is replaced. */
int or_softmax_rows_ordered(const float* m, size_t n, size_t cols, float temperature,
                            int bias, float a0, float a1, float a2, int kernel,
                            int width, int lanes, int cluster, long long slice,
                            int balanced, float* out);

/* Per-row scalars of the fused softmax (nonlin.cpp:85-93), exposed so tests
 * can pin the device's fp64 derivation. */
void or_softmax_row_scalars(float m, float temperature, int bias, float* c0,
                            float* c1, float* v_min);

/* nonlin.cpp:132-141 GeluConstants::defaults and the fused exp kernel
 * coefficients (nonlin.cpp:248-264). */
void or_gelu_constants(float* kappa, float* root2_over_pi, float* fused_scale,
                       float* inverse_kappa);

/* oracle.cpp:30-61 fp64 ground truth. */
double or_exact_exp(double x);
double or_exact_logistic(double x);
double or_exact_gelu_tanh(double x);
double or_exact_gelu_sigmoid(double x);
int or_exact_softmax(const float* v, size_t n, double temperature, double* out);

/* Exhaustive sweep support: recompute op(bits = start .. start+count-1) on
 * `threads` pthreads and compare bit-for-bit with `got` (the GPU's output for
 * the same bit patterns). op: 0 quake_buffer, 1 quake2_buffer (continuity),
 * 2 logistic_buffer, 3 gelu_buffer; for ops 0/1 the coefficients are the
 * natural-exp ones with `bias`, clamp from clamp_for. Returns the number of
 * mismatches; *first_bad receives the first mismatching bit pattern. */
uint64_t or_sweep_compare(int op, int kernel, int bias, uint64_t start, uint64_t count,
                          const float* got, int threads, uint64_t* first_bad);

/* Exhaustive check helpers used by the CPU test-suite: returns the number of
 * fp32 values t in [3, 6] for which the reciprocal-multiply + FMA correction
 * (the device's y/3) differs from the IEEE quotient t/3. */
uint64_t or_check_div3_replacement(void);

#ifdef __cplusplus
}
#endif

#endif /* QUAKE_ORACLE_H_ */
