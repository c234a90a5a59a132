/*
 * TEST INFRASTRUCTURE ONLY — plain-C restatement of the QuAKE hot path.
 * See quake_oracle.h for the contract. Paths cited are relative to
 * /root/reference/proj/. Compile with -ffp-contract=off and no -march.
 */
#include "quake_oracle.h"

#include <math.h>
#include <pthread.h>
#include <string.h>

/* std::numbers::log2e / ln2 / pi as exact binary64 literals. */
static const double kLog2e = 0x1.71547652b82fep+0;
static const double kLn2 = 0x1.62e42fefa39efp-1;
static const double kPi = 0x1.921fb54442d18p+1;
/* kernels.hpp:29 kCenteringBias. */
static const double kCenteringBias = 0.0436;
/* kernels.cpp:63-64 interior exponent margins. */
static const double kLowExponentEdge = 1.01;
static const double kHighExponentEdge = 254.99;
/* 2^23: std::ldexp(1.0, mantissa_bits) (kernels.cpp:30). */
static const double kScale = 8388608.0;

/* bitcore.hpp:57-59 masks. */
#define MANTISSA_MASK 0x007FFFFFu
#define SIGN_EXPONENT_MASK 0xFF800000u
#define UNIT_EXPONENT_BITS 0x3F800000u

/* bitcore.hpp:67-70 bit casts. */
static inline uint32_t f2u(float x) { uint32_t w; memcpy(&w, &x, 4); return w; }
static inline float u2f(uint32_t w) { float x; memcpy(&x, &w, 4); return x; }

/* bitcore.hpp:75-77 convert_to_int: static_cast<int32_t>(float), which the
 * reference's x86-64 build lowers to cvttss2si / cvttps2dq. Those return the
 * "integer indefinite" 0x80000000 for NaN and out-of-range inputs; spelled
 * out here so the C stays well defined. */
static inline uint32_t trunc_word(float z) {
  if (!(z >= -2147483648.0f && z < 2147483648.0f)) return 0x80000000u;
  return (uint32_t)(int32_t)z;
}

/* kernels.hpp:97-103 detail::saturate — NaN falls through to hi. */
static inline float saturate(float x, float lo, float hi) {
  const float t = x < lo ? lo : x;
  return t <= hi ? t : hi;
}

/* kernels.hpp:105-108 detail::quake_body. */
static inline float quake_body(float x, float c0, float c1) {
  const float z = c0 * x + c1;
  return u2f(trunc_word(z));
}

/* kernels.hpp:73-75 QuadCoeffs::is_continuity_default. */
static inline int is_continuity(float a0, float a1, float a2) {
  return a0 == 1.0f / 3.0f && a1 == 0.0f && a2 == 2.0f / 3.0f;
}

/* kernels.hpp:123-136 detail::quake2_body with refine_default (:111) or the
 * plain-association refine_general branch (:115-121, FP_FAST_FMAF unset). */
static inline float quake2_body(float x, float c0, float c1, int general,
                                float a0, float a1, float a2) {
  const float z = c0 * x + c1;
  const uint32_t zw = trunc_word(z);
  const float am = u2f((zw & MANTISSA_MASK) | UNIT_EXPONENT_BITS);
  float ym;
  if (!general) {
    ym = (am * am + 2.0f) / 3.0f;
  } else {
    ym = a0 * am * am + a1 * am + a2;
  }
  const uint32_t yw = (zw & SIGN_EXPONENT_MASK) + f2u(ym) - UNIT_EXPONENT_BITS;
  return u2f(yw);
}

int or_coeffs_for(float p, float q, int centering_bias, float* c0, float* c1) {
  /* kernels.cpp:25-40 */
  if (p == 0.0f) return OR_ERR_ZERO_SLOPE;
  const double beta = centering_bias ? kCenteringBias : 0.0;
  *c0 = (float)(kScale * (double)p);
  *c1 = (float)(kScale * ((double)127 + (double)q - beta));
  return OR_OK;
}

static void solve_clamp(double c0, double c1, float* lo, float* hi) {
  /* kernels.cpp:64-70 */
  double a = (kLowExponentEdge * kScale - c1) / c0;
  double b = (kHighExponentEdge * kScale - c1) / c0;
  if (a > b) { const double t = a; a = b; b = t; }
  *lo = (float)a;
  *hi = (float)b;
}

void or_clamp_for(float c0, float c1, float* lo, float* hi) {
  /* kernels.cpp:84-87 */
  solve_clamp((double)c0, (double)c1, lo, hi);
}

int or_default_clamp(float p, float q, float* lo, float* hi) {
  /* kernels.cpp:74-82 */
  if (p == 0.0f) return OR_ERR_ZERO_SLOPE;
  solve_clamp(kScale * (double)p, kScale * ((double)127 + (double)q), lo, hi);
  return OR_OK;
}

float or_quake(float x, float c0, float c1, float lo, float hi) {
  return quake_body(saturate(x, lo, hi), c0, c1); /* kernels.hpp:141-143 */
}

float or_quake2(float x, float c0, float c1, float a0, float a1, float a2,
                float lo, float hi) {
  /* kernels.hpp:146-155 */
  return quake2_body(saturate(x, lo, hi), c0, c1, !is_continuity(a0, a1, a2),
                     a0, a1, a2);
}

void or_quake_buffer(const float* xs, float* out, size_t n, float c0, float c1,
                     float lo, float hi) {
  /* kernels.cpp:95-107 */
  for (size_t i = 0; i < n; ++i) out[i] = quake_body(saturate(xs[i], lo, hi), c0, c1);
}

void or_quake2_buffer(const float* xs, float* out, size_t n, float c0, float c1,
                      float a0, float a1, float a2, float lo, float hi) {
  /* kernels.cpp:109-136: coefficient-set dispatch hoisted out of the loop. */
  const int general = !is_continuity(a0, a1, a2);
  for (size_t i = 0; i < n; ++i) {
    out[i] = quake2_body(saturate(xs[i], lo, hi), c0, c1, general, a0, a1, a2);
  }
}

static int is_unfused(int kernel) {
  return kernel == OR_QUAKE_UNFUSED || kernel == OR_QUAKE2_UNFUSED;
}
/* the exponential body an (un)fused kernel id uses: OR_QUAKE or OR_QUAKE2 */
static int body_of(int kernel) {
  return kernel == OR_QUAKE_UNFUSED ? OR_QUAKE : kernel == OR_QUAKE2_UNFUSED ? OR_QUAKE2 : kernel;
}

/* nonlin.hpp:39-41 resolve_centering_bias (unfused ids resolve as their body). */
static int resolve_bias(int kernel, int requested) {
  return requested < 0 ? (body_of(kernel) == OR_QUAKE) : (requested != 0);
}

void or_logistic_buffer(const float* xs, float* out, size_t n, int kernel, int bias) {
  /* nonlin.cpp:210-243 */
  if (kernel == OR_EXACT) {
    for (size_t i = 0; i < n; ++i) out[i] = 1.0f / (1.0f + expf(-xs[i]));
    return;
  }
  /* nonlin.cpp:35-41 negated_exp_kernel: -log2e slope, clamp from coefficients. */
  float c0, c1, lo, hi;
  or_coeffs_for((float)(-kLog2e), 0.0f, resolve_bias(kernel, bias), &c0, &c1);
  or_clamp_for(c0, c1, &lo, &hi);
  for (size_t i = 0; i < n; ++i) {
    const float u = saturate(xs[i], lo, hi);
    const float e = kernel == OR_QUAKE ? quake_body(u, c0, c1)
                                       : quake2_body(u, c0, c1, 0, 0.f, 0.f, 0.f);
    out[i] = 1.0f / (1.0f + e);
  }
}

void or_gelu_constants(float* kappa, float* root2_over_pi, float* fused_scale,
                       float* inverse_kappa) {
  /* nonlin.cpp:132-141 GeluConstants::defaults */
  const double k = 0.044715;
  const double r = sqrt(2.0 / kPi);
  *kappa = (float)k;
  *root2_over_pi = (float)r;
  *fused_scale = (float)(2.0 * k * r);
  *inverse_kappa = (float)(1.0 / k);
}

void or_gelu_buffer(const float* xs, float* out, size_t n, int kernel, int bias) {
  /* nonlin.cpp:292-330 */
  float kappa, r2pi, fs, ik;
  or_gelu_constants(&kappa, &r2pi, &fs, &ik);
  if (kernel == OR_EXACT) {
    for (size_t i = 0; i < n; ++i) {
      const float x = xs[i];
      out[i] = 0.5f * x * (1.0f + tanhf(r2pi * (x + kappa * x * x * x)));
    }
    return;
  }
  float c0, c1, lo, hi;
  if (is_unfused(kernel)) {
    /* bench.cpp:212-233: w = fused_scale*x*(inverse_kappa + x*x) computed
     * explicitly, fed to the e^-x kernel (negated natural coefficients). */
    or_coeffs_for((float)(-kLog2e), 0.0f, resolve_bias(kernel, bias), &c0, &c1);
    or_clamp_for(c0, c1, &lo, &hi);
    for (size_t i = 0; i < n; ++i) {
      const float x = xs[i];
      const float w = fs * x * (ik + x * x);
      const float s = saturate(w, lo, hi);
      const float e = body_of(kernel) == OR_QUAKE ? quake_body(s, c0, c1)
                                                  : quake2_body(s, c0, c1, 0, 0.f, 0.f, 0.f);
      out[i] = x / (1.0f + e);
    }
    return;
  }
  /* nonlin.cpp:248-264 gelu_exp_kernel: slope -log2e * fused_scale. */
  or_coeffs_for((float)(-kLog2e * (double)fs), 0.0f, resolve_bias(kernel, bias), &c0, &c1);
  or_clamp_for(c0, c1, &lo, &hi);
  for (size_t i = 0; i < n; ++i) {
    const float x = xs[i];
    const float u = x * (x * x + ik); /* nonlin.cpp:266-273, plain branch */
    const float s = saturate(u, lo, hi);
    const float e = kernel == OR_QUAKE ? quake_body(s, c0, c1)
                                       : quake2_body(s, c0, c1, 0, 0.f, 0.f, 0.f);
    out[i] = x / (1.0f + e);
  }
}

void or_softmax_row_scalars(float m, float temperature, int bias, float* c0,
                            float* c1, float* v_min) {
  /* nonlin.cpp:85-93 */
  const double beta = bias ? kCenteringBias : 0.0;
  *c0 = (float)(kScale * (double)temperature * kLog2e);
  *c1 = (float)(kScale * ((double)127 - beta) - (double)(*c0) * (double)m);
  *v_min = (float)((double)m - 126.0 * kLn2 / (double)temperature);
}

/* nonlin.cpp:43-55 row_max_checked (emptiness is checked by the callers). */
static int row_max_checked(const float* v, size_t n, float* m_out) {
  float m = v[0];
  for (size_t i = 0; i < n; ++i) {
    const float x = v[i];
    if (!isfinite(x)) return OR_ERR_NON_FINITE;
    m = x > m ? x : m;
  }
  *m_out = m;
  return OR_OK;
}

/* Per-row exponential of the QuAKE softmax kernels. Fused (nonlin.cpp:
 * 85-116): c0/c1 carry temperature and row max, inputs clamped below at
 * v_min. Unfused (bench.cpp:137-166): tmp = t*(x - m) explicitly, saturated
 * to the natural-exp clamp range, plain natural-exp body. */
typedef struct {
  int body, general, unfused;
  float c0, c1, v_min, a0, a1, a2;
  float m, t, lo, hi;
} row_exp_ctx;

static row_exp_ctx row_exp_setup(float m, float t, int kernel, int bias_req, float a0, float a1,
                                 float a2) {
  row_exp_ctx c;
  c.body = body_of(kernel);
  c.unfused = is_unfused(kernel);
  c.general = c.unfused ? 0 : !is_continuity(a0, a1, a2);
  c.a0 = a0;
  c.a1 = a1;
  c.a2 = a2;
  c.m = m;
  c.t = t;
  if (c.unfused) {
    or_coeffs_for((float)kLog2e, 0.0f, resolve_bias(kernel, bias_req), &c.c0, &c.c1);
    or_clamp_for(c.c0, c.c1, &c.lo, &c.hi);
    c.v_min = 0.0f;
  } else {
    or_softmax_row_scalars(m, t, resolve_bias(kernel, bias_req), &c.c0, &c.c1, &c.v_min);
    c.lo = c.hi = 0.0f;
  }
  return c;
}

static float row_exp_elem(const row_exp_ctx* c, float x) {
  float u;
  if (c->unfused) {
    const float tmp = c->t * (x - c->m);
    u = saturate(tmp, c->lo, c->hi);
  } else {
    u = x > c->v_min ? x : c->v_min;
  }
  return c->body == OR_QUAKE ? quake_body(u, c->c0, c->c1)
                             : quake2_body(u, c->c0, c->c1, c->general, c->a0, c->a1, c->a2);
}

/* nonlin.cpp:59-116 softmax_row_with + softmax_row_unchecked. */
static void softmax_row_unchecked(const float* v, size_t n, float m, float t,
                                  int bias_req, float a0, float a1, float a2,
                                  int kernel, int sum_mode, float* out) {
  if (kernel == OR_EXACT) {
    float fsum = 0.0f;
    double dsum = 0.0;
    for (size_t i = 0; i < n; ++i) {
      const float y = expf(t * (v[i] - m));
      out[i] = y;
      fsum += y;
      dsum += (double)y;
    }
    const float sum = sum_mode ? (float)dsum : fsum;
    for (size_t i = 0; i < n; ++i) out[i] /= sum;
    return;
  }
  const row_exp_ctx ctx = row_exp_setup(m, t, kernel, bias_req, a0, a1, a2);
  float fsum = 0.0f;
  double dsum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    const float y = row_exp_elem(&ctx, v[i]);
    out[i] = y;
    fsum += y;
    dsum += (double)y;
  }
  const float sum = sum_mode ? (float)dsum : fsum;
  for (size_t i = 0; i < n; ++i) out[i] /= sum;
}

int or_softmax_rows(const float* mat, size_t n, size_t cols, float temperature,
                    int bias, float a0, float a1, float a2, int kernel,
                    int sum_mode, float* out) {
  /* nonlin.cpp:162-189: shape, then temperature, then every row max, all
   * before the first write. */
  if (cols == 0 || n % cols != 0) return OR_ERR_NOT_DIVISIBLE;
  if (!(temperature > 0.0f)) return OR_ERR_BAD_TEMPERATURE;
  const size_t rows = n / cols;
  for (size_t r = 0; r < rows; ++r) {
    float m = 0.0f;
    const int st = row_max_checked(mat + r * cols, cols, &m);
    if (st != OR_OK) return st;
  }
  for (size_t r = 0; r < rows; ++r) {
    float m = 0.0f;
    row_max_checked(mat + r * cols, cols, &m);
    softmax_row_unchecked(mat + r * cols, cols, m, temperature, bias, a0, a1, a2,
                          kernel, sum_mode, out + r * cols);
  }
  return OR_OK;
}

/* Block tree of the GPU kernels over `lanes` thread partials (lanes = 32 for
 * the warp kernels, else a multiple of 32): butterfly with xor masks
 * 16,8,4,2,1 inside each warp; then lane 0's value of each warp, padded with
 * +0.0 up to the next power of two P, butterfly with masks P/2..1; returns
 * element 0 (every lane ends equal since fp addition commutes). */
static float block_tree_sum(float* p, int lanes) {
  float tmp[1024];
  const int w = lanes < 32 ? lanes : 32;
  for (int o = w / 2; o > 0; o >>= 1) {
    for (int l = 0; l < lanes; ++l) tmp[l] = p[l] + p[l ^ o];
    memcpy(p, tmp, sizeof(float) * (size_t)lanes);
  }
  if (lanes <= 32) return p[0];
  const int nw = lanes / 32;
  int P = 1;
  while (P < nw) P <<= 1;
  float wv[32];
  for (int i = 0; i < P; ++i) wv[i] = i < nw ? p[32 * i] : 0.0f;
  for (int o = P / 2; o > 0; o >>= 1) {
    float t2[32];
    for (int i = 0; i < P; ++i) t2[i] = wv[i] + wv[i ^ o];
    memcpy(wv, t2, sizeof(float) * (size_t)P);
  }
  return wv[0];
}

int or_softmax_rows_ordered(const float* mat, size_t n, size_t cols, float temperature,
                            int bias_req, float a0, float a1, float a2, int kernel,
                            int width, int lanes, int cluster, long long slice,
                            int balanced, float* out) {
  if (cols == 0 || n % cols != 0) return OR_ERR_NOT_DIVISIBLE;
  if (!(temperature > 0.0f)) return OR_ERR_BAD_TEMPERATURE;
  if (kernel == OR_EXACT || lanes > 1024 || lanes < 1) return OR_ERR_SIZE_MISMATCH;
  const size_t rows = n / cols;
  for (size_t r = 0; r < rows; ++r) {
    float m = 0.0f;
    const int st = row_max_checked(mat + r * cols, cols, &m);
    if (st != OR_OK) return st;
  }
  /* chunks of `width` consecutive elements; with cols % width != 0 the last
     chunk is partial and adds only its valid elements (kSpan, width 4) */
  const long long nchunks = (long long)((cols + (size_t)width - 1) / (size_t)width);
  if (slice <= 0) { slice = nchunks; cluster = 1; balanced = 0; }
  float part[1024];
  for (size_t r = 0; r < rows; ++r) {
    const float* v = mat + r * cols;
    float* y = out + r * cols;
    float m = 0.0f;
    row_max_checked(v, cols, &m);
    const row_exp_ctx ctx = row_exp_setup(m, temperature, kernel, bias_req, a0, a1, a2);
    for (size_t i = 0; i < cols; ++i) y[i] = row_exp_elem(&ctx, v[i]);
    float S = 0.0f;
    const long long q = nchunks / cluster, rem = nchunks % cluster;
    for (int c = 0; c < cluster; ++c) {
      long long b, cnt;
      if (balanced) {  /* rank c: q (+1 for the first rem ranks) chunks */
        b = (long long)c * q + (c < rem ? c : rem);
        cnt = q + (c < rem ? 1 : 0);
      } else {         /* rank c: `slice` chunks, the last one short */
        b = (long long)c * slice;
        cnt = nchunks - b;
        if (cnt > slice) cnt = slice;
        if (cnt < 0) cnt = 0;
      }
      for (int l = 0; l < lanes; ++l) {
        float s = 0.0f;
        for (long long j = l; j < cnt; j += lanes) {
          for (int e = 0; e < width; ++e) {
            const size_t idx = (size_t)((b + j) * width + e);
            if (idx < cols) s = s + y[idx];
          }
        }
        part[l] = s;
      }
      const float cs = block_tree_sum(part, lanes);
      S = c == 0 ? cs : S + cs;
    }
    for (size_t i = 0; i < cols; ++i) y[i] = y[i] / S;
  }
  return OR_OK;
}

/* oracle.cpp:30-61 */
double or_exact_exp(double x) { return exp(x); }
double or_exact_logistic(double x) { return 1.0 / (1.0 + exp(-x)); }
double or_exact_gelu_tanh(double x) {
  const double r = sqrt(2.0 / kPi);
  return 0.5 * x * (1.0 + tanh(r * (x + 0.044715 * x * x * x)));
}
double or_exact_gelu_sigmoid(double x) {
  const double k = 0.044715;
  const double r = sqrt(2.0 / kPi);
  const double arg = 2.0 * k * r * x * (1.0 / k + x * x);
  return x * or_exact_logistic(arg);
}
int or_exact_softmax(const float* v, size_t n, double temperature, double* out) {
  if (n == 0) return OR_ERR_EMPTY_ROW;
  double m = v[0];
  for (size_t i = 1; i < n; ++i) m = (double)v[i] > m ? (double)v[i] : m;
  double sum = 0.0;
  for (size_t i = 0; i < n; ++i) {
    out[i] = exp(temperature * ((double)v[i] - m));
    sum += out[i];
  }
  for (size_t i = 0; i < n; ++i) out[i] /= sum;
  return OR_OK;
}

uint64_t or_check_div3_replacement(void) {
  /* The device replaces (am*am + 2) / 3 by q = t*r3, q += fma(fma(-3,q,t), r3)
   * (Markstein correction with r3 = RN(1/3)). t = RN(RN(am^2) + 2) lies in
   * [3, 6]; check every binary32 value there against the IEEE quotient. */
  const float r3 = 1.0f / 3.0f;
  uint64_t bad = 0;
  for (uint32_t w = f2u(3.0f); w <= f2u(6.0f); ++w) {
    const float t = u2f(w);
    const float q0 = t * r3;
    const float res = fmaf(-3.0f, q0, t);
    const float q1 = fmaf(res, r3, q0);
    if (f2u(q1) != f2u(t / 3.0f)) ++bad;
  }
  return bad;
}

typedef struct {
  int op, kernel, bias;
  uint64_t start, count;
  const float* got;
  uint64_t bad, first_bad;
} sweep_job;

static void* sweep_worker(void* arg) {
  sweep_job* j = (sweep_job*)arg;
  enum { B = 4096 };
  float xs[B], ys[B];
  float c0 = 0, c1 = 0, lo = 0, hi = 0;
  if (j->op <= 1) {
    or_coeffs_for((float)kLog2e, 0.0f, j->bias, &c0, &c1);
    or_clamp_for(c0, c1, &lo, &hi);
  }
  j->bad = 0;
  j->first_bad = UINT64_MAX;
  for (uint64_t off = 0; off < j->count; off += B) {
    const uint64_t n = j->count - off < B ? j->count - off : B;
    for (uint64_t i = 0; i < n; ++i) xs[i] = u2f((uint32_t)(j->start + off + i));
    switch (j->op) {
      case 0: or_quake_buffer(xs, ys, n, c0, c1, lo, hi); break;
      case 1: or_quake2_buffer(xs, ys, n, c0, c1, 1.0f / 3.0f, 0.0f, 2.0f / 3.0f, lo, hi); break;
      case 2: or_logistic_buffer(xs, ys, n, j->kernel, j->bias); break;
      default: or_gelu_buffer(xs, ys, n, j->kernel, j->bias); break;
    }
    for (uint64_t i = 0; i < n; ++i) {
      if (f2u(ys[i]) != f2u(j->got[off + i])) {
        if (j->bad == 0) j->first_bad = j->start + off + i;
        ++j->bad;
      }
    }
  }
  return NULL;
}

uint64_t or_sweep_compare(int op, int kernel, int bias, uint64_t start, uint64_t count,
                          const float* got, int threads, uint64_t* first_bad) {
  if (threads < 1) threads = 1;
  if (threads > 256) threads = 256;
  pthread_t tid[256];
  sweep_job jobs[256];
  const uint64_t per = (count + (uint64_t)threads - 1) / (uint64_t)threads;
  int used = 0;
  for (int t = 0; t < threads; ++t) {
    const uint64_t b = (uint64_t)t * per;
    if (b >= count) break;
    jobs[t] = (sweep_job){op, kernel, bias, start + b, count - b < per ? count - b : per,
                          got + b, 0, 0};
    pthread_create(&tid[t], NULL, sweep_worker, &jobs[t]);
    ++used;
  }
  uint64_t bad = 0, fb = UINT64_MAX;
  for (int t = 0; t < used; ++t) {
    pthread_join(tid[t], NULL);
    bad += jobs[t].bad;
    if (jobs[t].bad && jobs[t].first_bad < fb) fb = jobs[t].first_bad;
  }
  if (first_bad) *first_bad = fb;
  return bad;
}
