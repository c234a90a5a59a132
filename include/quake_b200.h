/*
 * quake_b200.h — C-ABI of the B200-native QuAKE hot path.
 *
 * Plain C: POD structs, raw pointers, sizes, int status codes. No C++ or
 * torch types cross this boundary; exceptions never do. Implemented by
 * paper_2412_00408_b200/libquake_b200.so (sm_100a kernels + C++ host layer).
 *
 * Each entry point replaces one public function of the reference library
 * (paths relative to /root/reference/proj/). Three families:
 *
 *  1. Coefficient derivation (host-only scalar math, bit-identical to the
 *     reference's fp64 derivations).
 *  2. Host-span operators `qk_<op>(...)`: the drop-in for the reference's
 *     std::span overloads. Synchronous; same preconditions, same error
 *     categories and messages; on error `out` is left untouched (softmax
 *     validates every row before anything is written back, nonlin.cpp:176-
 *     180). Inputs may be pageable, pinned or device memory; work is sharded
 *     across the devices set by qk_set_devices() (default: current device).
 *  3. Device operators `qk_<op>_device(...)`: stream-ordered launches on
 *     device pointers, no allocation and no synchronisation — what an
 *     application with data already in HBM calls.
 *
 * KernelChoice values 0..2 match the reference enum (nonlin.hpp:32);
 * QK_EXPF and QK_FAST_EXP are GPU-only comparison kernels of identical
 * structure (CUDA expf / __expf in place of the QuAKE bit trick);
 * QK_QUAKE_UNFUSED / QK_QUAKE2_UNFUSED are the fusion-ablation variants of
 * the reference bench (softmax and gelu only).
 */
#ifndef QUAKE_B200_H_
#define QUAKE_B200_H_

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

#define QK_ABI_VERSION 3

typedef struct CUstream_st* qk_stream; /* == cudaStream_t; NULL = legacy default stream */

typedef enum {
  QK_OK = 0,
  /* 1..99: the reference's std::invalid_argument cases */
  QK_ERR_SIZE_MISMATCH = 1,   /* "<op>: output size mismatch" (kernels.cpp:97-99, ...) */
  QK_ERR_NOT_DIVISIBLE = 2,   /* "softmax_rows: length not divisible by cols" (nonlin.cpp:165-168) */
  QK_ERR_BAD_TEMPERATURE = 3, /* "<op>: temperature must be positive" (nonlin.cpp:148-150, 172-174) */
  QK_ERR_EMPTY_ROW = 4,       /* "softmax: empty row" (nonlin.cpp:44-46) */
  QK_ERR_NON_FINITE = 5,      /* "softmax: non-finite input" (nonlin.cpp:49-51) */
  QK_ERR_ZERO_SLOPE = 6,      /* "coeffs_for: input scale p must be non-zero" (kernels.cpp:27-29) */
  QK_ERR_BAD_ARGUMENT = 7,    /* null pointer / unknown kernel choice / unsupported size */
  /* 100+: runtime failures (no reference analogue) */
  QK_ERR_CUDA = 100,
  QK_ERR_NO_DEVICE = 101
} qk_status;

typedef enum {
  QK_EXACT = 0,   /* reference KernelChoice::Exact (libm-style expf / tanhf) */
  QK_QUAKE = 1,   /* KernelChoice::Quake  — first-order bit-trick exp */
  QK_QUAKE2 = 2,  /* KernelChoice::Quake2 — second-order mantissa refinement */
  QK_EXPF = 3,    /* comparison: QuAKE structure with CUDA expf */
  QK_FAST_EXP = 4,/* comparison: QuAKE structure with __expf */
  /* fusion ablation (bench.cpp:137-166, 212-233; softmax and gelu only): the
   * affine transform (t*(x - m), resp. fused_scale*x*(1/kappa + x*x)) is
   * computed explicitly and fed to the plain natural / negated-natural
   * QuAKE kernel instead of being folded into c0/c1. */
  QK_QUAKE_UNFUSED = 5,
  QK_QUAKE2_UNFUSED = 6
} qk_kernel;

/* kernels.hpp:39-46 AffineCoeffs */
typedef struct {
  float c0;
  float c1;
  float input_scale; /* p */
  float input_shift; /* q */
  int32_t bias_applied;
} qk_affine_coeffs;

/* kernels.hpp:60-76 QuadCoeffs */
typedef struct {
  float a0, a1, a2;
} qk_quad_coeffs;

/* kernels.hpp:81-84 ClampRange */
typedef struct {
  float lo, hi;
} qk_clamp_range;

/* nonlin.hpp:43-49 SoftmaxParams; centering_bias: -1 = unset (per-kernel
 * default, nonlin.hpp:39-41), 0 = off, 1 = on. */
typedef struct {
  float temperature;
  int32_t centering_bias;
  qk_quad_coeffs quad;
} qk_softmax_params;

/* bitcore.hpp:32-53 FpFormat (layout of a binary floating-point format) */
typedef struct {
  int32_t exponent_bits, mantissa_bits, bias;
} qk_fp_format;

/* nonlin.hpp:55-62 GeluConstants */
typedef struct {
  float kappa, root2_over_pi, fused_scale, inverse_kappa;
} qk_gelu_constants;

/* Softmax launch plan (introspection; the reduction geometry that fixes the
 * summation order, see softmax.cu). */
typedef struct {
  int32_t variant; /* 2 smem(+cluster), 3 global 3-sweep,
                      4 persistent TMA pipeline (+cluster),
                      6 long-row pipeline (one stage, prefix refilled early),
                      7 scalar-lane pipeline (cols % 4 != 0),
                      9 one thread per row (<= 16 cols; lanes = 1: sequential sum),
                      10 one thread per row through an smem tile (lanes = 1),
                      11 G lanes per row (lanes = G, vpt = chunks per lane),
                      13 row spans through smem, row-relative float4 chunks, G lanes
                         (unaligned 17-32 cols, misaligned bases),
                      14 per-agent TMA rings of row spans, scalar lanes (unaligned
                         33-28000 cols; lanes = G lanes per row with vpt elements each,
                         or vpt = 0: three sweeps by an agent of lanes/32 warps;
                         stages = buffers per ring);
                      0, 1, 5, 8, 12: retired variants (numbers reserved) */
  int32_t width;   /* elements per chunk: 4 when cols % 4 == 0, else 1 (any address) */
  int32_t lanes;   /* partial-sum lanes per CTA */
  int32_t cluster; /* CTAs per row */
  int64_t slice;   /* chunks per CTA slice (0 = whole row) */
  int32_t threads; /* CTA size */
  int32_t vpt;     /* warp variants: chunks per lane */
  int64_t smem;    /* dynamic smem bytes per CTA */
  int32_t stages;  /* variants 4-7: row slices staged per CTA */
  int32_t balanced;/* 1: CTA r's slice is q (+1 for r < nchunks % cluster) chunks;
                      0: `slice` chunks per CTA, the last one short */
  int32_t resident;/* variants 4-7: clusters resident at once on this device (0 = unknown) */
} qk_softmax_plan_info;

/* ---- library ---- */
int qk_abi_version(void);
const char* qk_last_error(void);        /* message of the last failure on this thread */
int qk_is_invalid_argument(qk_status s);/* 1 for the std::invalid_argument family */
qk_status qk_device_count(int* count);
/* Devices the host-span operators shard over (rows / 16-byte element
 * ranges, no collectives). n = 0 restores the default (current device). */
qk_status qk_set_devices(const int* devices, int n);
/* As qk_set_devices, but a device may be listed several times: each entry is
 * one shard with its own workspace and host thread. Lets one GPU run the
 * 2/4/8-way split of the multi-GPU driver (tests; outputs do not depend on
 * the split). */
qk_status qk_set_device_shards(const int* devices, int n);
/* Number of shards (entries) and their devices. */
int qk_get_devices(int* devices, int cap);
/* Frees the cached device workspace of the host-span path. */
void qk_release_workspace(void);
/* Device workspace one host-span shard may hold, in bytes (0 = automatic: 90%
 * of free HBM). Shards whose host-side spans exceed it stream through rings
 * of 64 MiB chunk buffers, softmax with a validation pass first. */
void qk_set_workspace_limit(size_t bytes);
/* Overlapped write-back of qk_softmax_rows with pinned host spans on both
 * sides: `threads` host threads test the shard for non-finite values from its
 * last element backwards while the device validates the uploaded chunks from
 * the front; once the two fronts meet, every row is validated (the
 * reference's validate-before-write order, nonlin.cpp:176-180) and the
 * download runs under the rest of the upload. The host threads test exponent
 * bits only; every output value comes from the kernels. threads < 0:
 * automatic (host CPUs, at most 16; QK_HOST_SCAN in the environment
 * overrides), 0: off (the device validates alone). Used for shards of at
 * least `min_bytes` (default 64 MiB). */
void qk_set_host_validation(int32_t threads, size_t min_bytes);
/* Softmax planner knobs (the QK_SM_* measurement options, read from the
 * environment once at first use): set `name` to `value`, or unset it when
 * `clear` != 0; name = NULL clears every option. Plans are cached per
 * (device, cols, kernel, options). QK_ERR_BAD_ARGUMENT for an unknown name. */
qk_status qk_set_plan_override(const char* name, int32_t value, int32_t clear);

/* ---- 1. coefficient derivation (kernels.cpp:25-87, nonlin.cpp:132-141) ---- */
qk_status qk_coeffs_for(float p, float q, int32_t centering_bias, qk_affine_coeffs* out);
qk_affine_coeffs qk_natural_exp_coeffs(int32_t centering_bias);
qk_affine_coeffs qk_base2_coeffs(int32_t centering_bias);
qk_affine_coeffs qk_negated_natural_exp_coeffs(int32_t centering_bias);
qk_status qk_default_clamp(float p, float q, qk_clamp_range* out);
/* kernels.cpp:25-40 / :74-82 with an explicit format (kernels.hpp:50-51, 89):
 * scale 2^mantissa_bits, exponent bias `bias`. NULL = binary32. */
qk_status qk_coeffs_for_format(float p, float q, const qk_fp_format* fmt, int32_t centering_bias,
                               qk_affine_coeffs* out);
qk_status qk_default_clamp_format(float p, float q, const qk_fp_format* fmt, qk_clamp_range* out);
qk_clamp_range qk_clamp_for(const qk_affine_coeffs* c);
qk_quad_coeffs qk_quad_continuity(void);
qk_quad_coeffs qk_quad_minimax(void);
int qk_quad_is_continuity_default(const qk_quad_coeffs* a);
qk_gelu_constants qk_gelu_constants_defaults(void);
int32_t qk_resolve_centering_bias(qk_kernel k, int32_t requested);
const char* qk_kernel_name(qk_kernel k);
/* Launch geometry (and hence summation order) of softmax rows of `cols`
 * columns for `kernel` on the current device. It depends on cols, kernel
 * and device only: rows at any address get the same order (`aligned16` is
 * ignored since ABI 3). */
qk_status qk_softmax_plan(size_t cols, int32_t aligned16, qk_kernel kernel,
                          qk_softmax_plan_info* out);

/* ---- 2. host-span operators (drop-ins for the std::span overloads) ---- */
/* kernels.hpp:163-164 / kernels.cpp:95-107 quake_buffer */
qk_status qk_quake_buffer(const float* xs, size_t n, float* out, size_t out_n,
                          const qk_affine_coeffs* c, const qk_clamp_range* r);
/* kernels.hpp:165-167 / kernels.cpp:109-136 quake2_buffer */
qk_status qk_quake2_buffer(const float* xs, size_t n, float* out, size_t out_n,
                           const qk_affine_coeffs* c, const qk_quad_coeffs* a,
                           const qk_clamp_range* r);
/* nonlin.hpp:86-88 / nonlin.cpp:210-243 logistic_buffer */
qk_status qk_logistic_buffer(const float* xs, size_t n, float* out, size_t out_n, qk_kernel k,
                             int32_t centering_bias);
/* nonlin.hpp:95-97 / nonlin.cpp:292-330 gelu_buffer */
qk_status qk_gelu_buffer(const float* xs, size_t n, float* out, size_t out_n, qk_kernel k,
                         int32_t centering_bias);
/* nonlin.hpp:77-79 / nonlin.cpp:162-189 softmax_rows */
qk_status qk_softmax_rows(const float* matrix, size_t n, size_t cols,
                          const qk_softmax_params* params, qk_kernel k, float* out,
                          size_t out_n);
/* nonlin.hpp:70-71 / nonlin.cpp:143-153 softmax_row */
qk_status qk_softmax_row(const float* v, size_t n, const qk_softmax_params* params, qk_kernel k,
                         float* out, size_t out_n);
/* exp comparison (bench.cpp:236-258 make_exp_pass analogue): QK_EXACT/QK_EXPF
 * = expf, QK_FAST_EXP = __expf, QK_QUAKE/QK_QUAKE2 = natural-exp QuAKE with
 * the per-kernel default bias. */
qk_status qk_exp_buffer(const float* xs, size_t n, float* out, size_t out_n, qk_kernel k);

/* Scalar forms: kernels.hpp:141-155 quake / quake2, nonlin.cpp:198-208
 * logistic, nonlin.cpp:277-290 gelu. One element through the same GPU
 * kernels (a per-thread pinned mailbox and one small launch on the first
 * configured device); bit-identical to the buffer forms. */
qk_status qk_quake(float x, const qk_affine_coeffs* c, const qk_clamp_range* r, float* y);
qk_status qk_quake2(float x, const qk_affine_coeffs* c, const qk_quad_coeffs* a,
                    const qk_clamp_range* r, float* y);
qk_status qk_logistic(float x, qk_kernel k, int32_t centering_bias, float* y);
qk_status qk_gelu(float x, qk_kernel k, int32_t centering_bias, float* y);

/* ---- 3. device operators (stream-ordered, device pointers, no sync) ---- */
qk_status qk_quake_buffer_device(const float* xs, float* out, size_t n,
                                 const qk_affine_coeffs* c, const qk_clamp_range* r,
                                 qk_stream stream);
qk_status qk_quake2_buffer_device(const float* xs, float* out, size_t n,
                                  const qk_affine_coeffs* c, const qk_quad_coeffs* a,
                                  const qk_clamp_range* r, qk_stream stream);
qk_status qk_logistic_buffer_device(const float* xs, float* out, size_t n, qk_kernel k,
                                    int32_t centering_bias, qk_stream stream);
qk_status qk_gelu_buffer_device(const float* xs, float* out, size_t n, qk_kernel k,
                                int32_t centering_bias, qk_stream stream);
qk_status qk_exp_buffer_device(const float* xs, float* out, size_t n, qk_kernel k,
                               qk_stream stream);
/* Row softmax on device memory. Shape/temperature are validated on the host
 * before launch; non-finite inputs are detected inside the kernel's max pass
 * and reported by OR-ing 1 into *d_flags (device word, may be NULL). Unlike
 * the host-span form, `out` may already be written when that happens. */
qk_status qk_softmax_rows_device(const float* matrix, size_t n, size_t cols,
                                 const qk_softmax_params* params, qk_kernel k, float* out,
                                 uint32_t* d_flags, qk_stream stream);

#ifdef __cplusplus
}
#endif

#endif /* QUAKE_B200_H_ */
