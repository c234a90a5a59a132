// GPU accuracy lab (reference core/src/lab.cpp).
//
// Every approximation is produced by the product's own device functions
// (numerics.cuh: saturate, quake_body, quake2_body — bit-identical to the
// reference), the ground truth by binary64 exp / exp2 on the device. Sweeps
// are split into contiguous index blocks; each block reduces its elements in
// a fixed tree and the host folds the block partials in index order, so a
// report is a deterministic function of the inputs (lab.cpp:86-107 keeps
// the same "first index attaining the maximum" rule).
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <limits>
#include <numeric>
#include <string>
#include <vector>

#include "internal.h"
#include "numerics.cuh"
#include "quake_b200_lab.h"

namespace qk {
namespace {

constexpr double kLog2e = 0x1.71547652b82fep+0;
constexpr double kCenteringBias = 0.0436;  // kernels.hpp:29
constexpr double kScale = 8388608.0;       // 2^23
constexpr uint32_t kBias = 127;
constexpr int kLabThreads = 256;
constexpr uint64_t kNone = ~0ull;

// lab.cpp:36-74 Evaluator, device side.
struct LabEval {
  int kind;     // 0 exact, 1 quake, 2 quake2
  int natural;  // e^x vs 2^x
  int general;  // quake2 with a non-continuity quad (refine_general)
  float c0, c1, lo, hi, a0, a1, a2;
};

__device__ __forceinline__ float lab_approx(const LabEval& e, float x) {
  const float u = saturate(x, e.lo, e.hi);
  if (e.kind == 1) return quake_body(u, e.c0, e.c1);
  if (e.general) return quake2_body<true>(u, e.c0, e.c1, e.a0, e.a1, e.a2);
  return quake2_body<false>(u, e.c0, e.c1, 0.f, 0.f, 0.f);
}

__device__ __forceinline__ double lab_truth(const LabEval& e, float x) {
  return e.natural ? exp(static_cast<double>(x)) : exp2(static_cast<double>(x));
}

__device__ __forceinline__ double lab_eval(const LabEval& e, float x) {
  return e.kind == 0 ? lab_truth(e, x) : static_cast<double>(lab_approx(e, x));
}

// Inputs of one sweep, by index (lab.cpp:170-196).
struct LabInputs {
  int mode;           // 0 uniform grid, 1 mantissa-period walk, 2 every binary32
  double lo, step;    // mode 0: x_i = float(lo + step*i)
  uint64_t w0;        // mode 1: w = double(w0 + i*stride), x = (w - c1)/c0
  uint32_t stride;
  double c0, c1, wlo, whi;
  uint32_t key0;      // mode 2: ordered key of the first input
};

__device__ __forceinline__ float from_key(uint32_t k) {
  // ordered key -> binary32: keys increase with the value, -0 just below +0
  const uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  return __uint_as_float(b);
}

__device__ __forceinline__ float lab_input(const LabInputs& in, uint64_t i) {
  if (in.mode == 0) {
    return __double2float_rn(__dadd_rn(in.lo, __dmul_rn(in.step, static_cast<double>(i))));
  }
  if (in.mode == 1) {
    const double w = static_cast<double>(in.w0 + i * in.stride);
    const double x = __ddiv_rn(__dsub_rn(w, in.c1), in.c0);
    if (x < in.wlo || x > in.whi) return __int_as_float(0x7FC00000);  // skipped (NaN)
    return __double2float_rn(x);
  }
  return from_key(in.key0 + static_cast<uint32_t>(i));
}

struct LabPartial {
  double max_rel;   // -1: no sample
  uint64_t arg;     // index of the first maximum
  double sum;
  uint64_t n;
  uint64_t viol, first_viol;
  uint64_t nonpos, first_nonpos;
};

__device__ __forceinline__ void lab_combine(LabPartial& a, const LabPartial& b) {
  if (b.max_rel > a.max_rel || (b.max_rel == a.max_rel && b.arg < a.arg)) {
    a.max_rel = b.max_rel;
    a.arg = b.arg;
  }
  a.sum += b.sum;
  a.n += b.n;
  a.viol += b.viol;
  a.first_viol = b.first_viol < a.first_viol ? b.first_viol : a.first_viol;
  a.nonpos += b.nonpos;
  a.first_nonpos = b.first_nonpos < a.first_nonpos ? b.first_nonpos : a.first_nonpos;
}

// Block b covers indices [b*chunk, min(count, (b+1)*chunk)); thread t takes
// every T-th of them in increasing order; then a fixed shared-memory tree.
template <bool kProps>
__global__ void __launch_bounds__(kLabThreads) lab_sweep_kernel(LabEval e, LabInputs in,
                                                                uint64_t count, uint64_t chunk,
                                                                LabPartial* out) {
  __shared__ LabPartial sh[kLabThreads];
  LabPartial p{-1.0, kNone, 0.0, 0, 0, kNone, 0, kNone};
  const uint64_t begin = static_cast<uint64_t>(blockIdx.x) * chunk;
  const uint64_t end = begin + chunk < count ? begin + chunk : count;
  for (uint64_t i = begin + threadIdx.x; i < end; i += kLabThreads) {
    const float x = lab_input(in, i);
    if (x != x) continue;
    const double approx = lab_eval(e, x);
    const double exact = lab_truth(e, x);
    const double rel = fabs(approx - exact) / exact;
    if (rel > p.max_rel) {
      p.max_rel = rel;
      p.arg = i;
    }
    p.sum += rel;
    ++p.n;
    if constexpr (kProps) {
      if (!(approx > 0.0) || !isfinite(approx)) {
        ++p.nonpos;
        if (p.first_nonpos == kNone) p.first_nonpos = i;
      }
      if (i + 1 < count) {
        const double next = lab_eval(e, lab_input(in, i + 1));
        if (approx > next) {
          ++p.viol;
          if (p.first_viol == kNone) p.first_viol = i;
        }
      }
    }
  }
  sh[threadIdx.x] = p;
  __syncthreads();
  for (int o = kLabThreads / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) lab_combine(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  if (threadIdx.x == 0) out[blockIdx.x] = sh[0];
}

// lab.cpp:300-309 value_of_word, per exponent step k (one thread each).
__global__ void lab_continuity_kernel(LabEval e, int k_lo, int nk, double* jump) {
  const int j = blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nk) return;
  auto value_of_word = [&](uint32_t zw) -> double {
    if (e.kind == 1) return static_cast<double>(__uint_as_float(zw));
    const uint32_t ab = (zw & kMantissaMask) | kUnitExponentBits;
    const float am = __uint_as_float(ab);
    const float ym = e.general ? refine_general(am, e.a0, e.a1, e.a2) : refine_default(am);
    return static_cast<double>(__uint_as_float((zw & 0xFF800000u) + __float_as_uint(ym) -
                                               kUnitExponentBits));
  };
  const uint32_t boundary = static_cast<uint32_t>(static_cast<int>(kBias) + k_lo + j) << 23;
  const double at = value_of_word(boundary);
  const double below = value_of_word(boundary - 1u);
  jump[j] = fabs(at - below) / at;
}

// lab.cpp:209-219 quad_max_rel_err for points [i0, i1) of one coefficient
// triple; returns the maximum in the block (order-independent).
__device__ double quad_rel_at(double a0, double a1, double a2, uint64_t i, uint64_t intervals) {
  const double am = __dadd_rn(1.0, __ddiv_rn(static_cast<double>(i), static_cast<double>(intervals)));
  const double poly = __dadd_rn(__dmul_rn(__dadd_rn(__dmul_rn(a0, am), a1), am), a2);
  const double exact = exp2(__dsub_rn(am, 1.0));
  return __ddiv_rn(fabs(__dsub_rn(poly, exact)), exact);
}

__device__ __forceinline__ double block_max(double v, double* sh) {
  sh[threadIdx.x] = v;
  __syncthreads();
  for (int o = blockDim.x / 2; o > 0; o >>= 1) {
    if (static_cast<int>(threadIdx.x) < o) sh[threadIdx.x] = fmax(sh[threadIdx.x], sh[threadIdx.x + o]);
    __syncthreads();
  }
  return sh[0];
}

// Coarse pass: one thread per grid point (lab.cpp:239-245).
__global__ void lab_grid_coarse(qk_grid_spec g, uint64_t n1, uint64_t n2, uint64_t total,
                                uint64_t intervals, double* out) {
  const uint64_t flat = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x;
  if (flat >= total) return;
  const uint64_t i2 = flat % n2, i1 = (flat / n2) % n1, i0 = flat / (n1 * n2);
  const double a0 = __dadd_rn(g.a0.lo, __dmul_rn(g.a0.step, static_cast<double>(i0)));
  const double a1 = __dadd_rn(g.a1.lo, __dmul_rn(g.a1.step, static_cast<double>(i1)));
  const double a2 = __dadd_rn(g.a2.lo, __dmul_rn(g.a2.step, static_cast<double>(i2)));
  double worst = 0.0;
  for (uint64_t i = 0; i <= intervals; ++i) {
    const double r = quad_rel_at(a0, a1, a2, i, intervals);
    if (r > worst) worst = r;
  }
  out[flat] = worst;
}

// One block per coefficient triple (fine re-evaluation, lab.cpp:258-266),
// or many blocks over one triple (intervals split): partial maxima.
__global__ void __launch_bounds__(kLabThreads) lab_quad_blocks(const double* coeffs, int per_triple,
                                                               uint64_t intervals, double* out) {
  __shared__ double sh[kLabThreads];
  const int t = blockIdx.x / per_triple, part = blockIdx.x % per_triple;
  const double a0 = coeffs[3 * t], a1 = coeffs[3 * t + 1], a2 = coeffs[3 * t + 2];
  const uint64_t npts = intervals + 1;
  const uint64_t chunk = (npts + per_triple - 1) / per_triple;
  const uint64_t b = static_cast<uint64_t>(part) * chunk;
  const uint64_t e = b + chunk < npts ? b + chunk : npts;
  double worst = 0.0;
  for (uint64_t i = b + threadIdx.x; i < e; i += kLabThreads) {
    const double r = quad_rel_at(a0, a1, a2, i, intervals);
    if (r > worst) worst = r;
  }
  const double m = block_max(worst, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = m;
}

// bias_reoptimize objective (lab.cpp:340-376): worst relative error over
// x_i = float(period*i/(N-1)), i <= N-1, for one (c0, c1, clamp).
__global__ void __launch_bounds__(kLabThreads) lab_bias_objective(LabEval e, double period,
                                                                  uint64_t n, double* out) {
  __shared__ double sh[kLabThreads];
  double worst = 0.0;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * kLabThreads + threadIdx.x; i < n;
       i += static_cast<uint64_t>(gridDim.x) * kLabThreads) {
    const float x = __double2float_rn(
        __ddiv_rn(__dmul_rn(period, static_cast<double>(i)), static_cast<double>(n - 1)));
    const double ref = lab_truth(e, x);
    const double approx = static_cast<double>(lab_approx(e, x));
    const double rel = fabs(approx - ref) / ref;
    if (rel > worst) worst = rel;
  }
  const double m = block_max(worst, sh);
  if (threadIdx.x == 0) out[blockIdx.x] = m;
}

// ---- host side ----------------------------------------------------------

struct DevBuf {
  void* p = nullptr;
  ~DevBuf() {
    if (p) cudaFree(p);
  }
};

qk_status cuda_err(cudaError_t e, const char* where) {
  return set_error(QK_ERR_CUDA, std::string(where) + ": " + cudaGetErrorString(e));
}

bool valid_kind(qk_kernel k) { return k == QK_EXACT || k == QK_QUAKE || k == QK_QUAKE2; }

bool is_continuity(const qk_quad_coeffs& a) {
  return a.a0 == 1.0f / 3.0f && a.a1 == 0.0f && a.a2 == 2.0f / 3.0f;
}

// lab.cpp:121-129 + Evaluator construction (lab.cpp:44-52)
qk_status make_eval(const qk_exp_config* cfg, LabEval* e, qk_affine_coeffs* c,
                    qk_clamp_range* r) {
  if (!cfg || !valid_kind(cfg->kind)) return set_error(QK_ERR_BAD_ARGUMENT, "lab: unknown kernel choice");
  const float p = cfg->natural_base ? static_cast<float>(kLog2e) : 1.0f;
  qk_affine_coeffs cc{};
  qk_status s = qk_coeffs_for(p, 0.0f, cfg->centering_bias ? 1 : 0, &cc);
  if (s != QK_OK) return s;
  const qk_clamp_range rr = qk_clamp_for(&cc);
  e->kind = cfg->kind == QK_EXACT ? 0 : (cfg->kind == QK_QUAKE ? 1 : 2);
  e->natural = cfg->natural_base ? 1 : 0;
  e->general = (cfg->kind == QK_QUAKE2 && !is_continuity(cfg->quad)) ? 1 : 0;
  e->c0 = cc.c0;
  e->c1 = cc.c1;
  e->lo = rr.lo;
  e->hi = rr.hi;
  e->a0 = cfg->quad.a0;
  e->a1 = cfg->quad.a1;
  e->a2 = cfg->quad.a2;
  if (c) *c = cc;
  if (r) *r = rr;
  return QK_OK;
}

// Run one sweep and fold the block partials in index order.
template <bool kProps>
qk_status run_sweep(const LabEval& e, const LabInputs& in, uint64_t count, LabPartial* total) {
  if (count == 0) return QK_OK;
  const uint64_t max_blocks = 148ull * 16;
  uint64_t chunk = (count + max_blocks - 1) / max_blocks;
  chunk = std::max<uint64_t>(chunk, kLabThreads);
  const uint64_t blocks = (count + chunk - 1) / chunk;
  DevBuf d;
  cudaError_t ce = cudaMalloc(&d.p, blocks * sizeof(LabPartial));
  if (ce != cudaSuccess) return cuda_err(ce, "lab: cudaMalloc");
  lab_sweep_kernel<kProps><<<static_cast<unsigned>(blocks), kLabThreads>>>(
      e, in, count, chunk, static_cast<LabPartial*>(d.p));
  if ((ce = cudaGetLastError()) != cudaSuccess) return cuda_err(ce, "lab: sweep launch");
  std::vector<LabPartial> h(blocks);
  ce = cudaMemcpy(h.data(), d.p, blocks * sizeof(LabPartial), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_err(ce, "lab: sweep");
  for (const LabPartial& b : h) {  // lab.cpp:100-106: strict > keeps the earlier chunk
    if (b.max_rel > total->max_rel) {
      total->max_rel = b.max_rel;
      total->arg = b.arg;
    }
    total->sum += b.sum;
    total->n += b.n;
    total->viol += b.viol;
    if (total->first_viol == kNone) total->first_viol = b.first_viol;
    total->nonpos += b.nonpos;
    if (total->first_nonpos == kNone) total->first_nonpos = b.first_nonpos;
  }
  return QK_OK;
}

uint32_t key_of(float f) {
  uint32_t b;
  std::memcpy(&b, &f, 4);
  return (b & 0x80000000u) ? ~b : (b | 0x80000000u);
}

float float_of_key(uint32_t k) {
  const uint32_t b = (k & 0x80000000u) ? (k & 0x7FFFFFFFu) : ~k;
  float f;
  std::memcpy(&f, &b, 4);
  return f;
}

// Host restatement of the device input map (for reporting argmax inputs).
float host_input(const LabInputs& in, uint64_t i) {
  if (in.mode == 0) return static_cast<float>(in.lo + in.step * static_cast<double>(i));
  if (in.mode == 1) {
    const double w = static_cast<double>(in.w0 + i * in.stride);
    return static_cast<float>((w - in.c1) / in.c0);
  }
  return float_of_key(in.key0 + static_cast<uint32_t>(i));
}

qk_status quad_max(const std::vector<double>& triples, int per_triple, uint64_t intervals,
                   std::vector<double>* maxima) {
  const size_t nt = triples.size() / 3;
  DevBuf dc, dout;
  cudaError_t ce = cudaMalloc(&dc.p, triples.size() * sizeof(double));
  if (ce == cudaSuccess) ce = cudaMalloc(&dout.p, nt * per_triple * sizeof(double));
  if (ce != cudaSuccess) return cuda_err(ce, "lab: cudaMalloc");
  ce = cudaMemcpy(dc.p, triples.data(), triples.size() * sizeof(double), cudaMemcpyHostToDevice);
  if (ce != cudaSuccess) return cuda_err(ce, "lab: copy");
  lab_quad_blocks<<<static_cast<unsigned>(nt * per_triple), kLabThreads>>>(
      static_cast<const double*>(dc.p), per_triple, intervals, static_cast<double*>(dout.p));
  if ((ce = cudaGetLastError()) != cudaSuccess) return cuda_err(ce, "lab: quad launch");
  std::vector<double> parts(nt * per_triple);
  ce = cudaMemcpy(parts.data(), dout.p, parts.size() * sizeof(double), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_err(ce, "lab: quad");
  maxima->assign(nt, 0.0);
  for (size_t t = 0; t < nt; ++t) {
    for (int k = 0; k < per_triple; ++k) (*maxima)[t] = std::max((*maxima)[t], parts[t * per_triple + k]);
  }
  return QK_OK;
}

size_t axis_points(const qk_grid_axis& a) {  // lab.cpp:202-205
  if (a.step <= 0.0 || a.hi < a.lo) return 0;
  return static_cast<size_t>(std::floor((a.hi - a.lo) / a.step + 0.5)) + 1;
}

double axis_at(const qk_grid_axis& a, size_t i) { return a.lo + a.step * static_cast<double>(i); }

}  // namespace
}  // namespace qk

using namespace qk;

extern "C" {

qk_sweep_spec qk_sweep_spec_defaults(void) { return qk_sweep_spec{-80.0f, 80.0f, 1ull << 22, 1}; }

qk_grid_spec qk_grid_spec_defaults(void) {
  return qk_grid_spec{{0.30, 0.36, 0.001}, {-0.05, 0.02, 0.001}, {0.64, 0.72, 0.001}};
}

qk_status qk_lab_coeffs(const qk_exp_config* cfg, qk_affine_coeffs* c, qk_clamp_range* r) {
  LabEval e;
  return make_eval(cfg, &e, c, r);
}

qk_status qk_sweep_error(const qk_exp_config* cfg, const qk_sweep_spec* spec,
                         qk_error_report* out) {
  if (!spec || !out) return set_error(QK_ERR_BAD_ARGUMENT, "sweep_error: null pointer");
  // lab.cpp:151-163, same order and messages
  if (!(spec->lo < spec->hi)) return set_error(QK_ERR_BAD_ARGUMENT, "sweep_error: range is empty");
  if (spec->uniform_samples < 10000) {
    return set_error(QK_ERR_BAD_ARGUMENT, "sweep_error: need at least 10^4 samples");
  }
  LabEval e;
  qk_affine_coeffs c;
  qk_clamp_range r;
  qk_status s = make_eval(cfg, &e, &c, &r);
  if (s != QK_OK) return s;
  if (cfg->kind != QK_EXACT && (spec->lo < r.lo || spec->hi > r.hi)) {
    return set_error(QK_ERR_BAD_ARGUMENT, "sweep_error: range exceeds clamp bounds");
  }
  LabPartial total{-1.0, kNone, 0.0, 0, 0, kNone, 0, kNone};
  LabInputs uni{};
  uni.mode = 0;
  uni.lo = spec->lo;
  uni.step = (static_cast<double>(spec->hi) - uni.lo) / static_cast<double>(spec->uniform_samples - 1);
  if ((s = run_sweep<false>(e, uni, spec->uniform_samples, &total)) != QK_OK) return s;
  const LabPartial after_uniform = total;
  LabInputs per{};
  if (cfg->kind != QK_EXACT && spec->period_stride > 0) {  // lab.cpp:180-196
    per.mode = 1;
    per.w0 = static_cast<uint64_t>(kBias) << 23;
    per.stride = spec->period_stride;
    per.c0 = c.c0;
    per.c1 = c.c1;
    per.wlo = spec->lo;
    per.whi = spec->hi;
    const uint64_t span = 1ull << 23;
    const uint64_t count = (span + spec->period_stride - 1) / spec->period_stride;
    if ((s = run_sweep<false>(e, per, count, &total)) != QK_OK) return s;
  }
  out->lo = spec->lo;
  out->hi = spec->hi;
  out->samples = total.n;
  out->max_rel_err = total.max_rel < 0.0 ? 0.0 : total.max_rel;
  out->mean_rel_err = total.n == 0 ? 0.0 : total.sum / static_cast<double>(total.n);
  if (total.arg == kNone) {
    out->argmax_input = 0.0f;
  } else {
    const bool from_period = total.max_rel > after_uniform.max_rel;
    out->argmax_input = host_input(from_period ? per : uni, total.arg);
  }
  return QK_OK;
}

qk_status qk_sweep_exhaustive(const qk_exp_config* cfg, float lo, float hi,
                              qk_exhaustive_report* out) {
  if (!out) return set_error(QK_ERR_BAD_ARGUMENT, "sweep_exhaustive: null pointer");
  if (!(lo <= hi)) return set_error(QK_ERR_BAD_ARGUMENT, "sweep_exhaustive: range is empty");
  LabEval e;
  qk_clamp_range r;
  qk_status s = make_eval(cfg, &e, nullptr, &r);
  if (s != QK_OK) return s;
  if (cfg->kind != QK_EXACT && (lo < r.lo || hi > r.hi)) {
    return set_error(QK_ERR_BAD_ARGUMENT, "sweep_exhaustive: range exceeds clamp bounds");
  }
  LabInputs in{};
  in.mode = 2;
  in.key0 = key_of(lo);
  const uint64_t count = static_cast<uint64_t>(key_of(hi)) - in.key0 + 1;
  LabPartial total{-1.0, kNone, 0.0, 0, 0, kNone, 0, kNone};
  if ((s = run_sweep<true>(e, in, count, &total)) != QK_OK) return s;
  const float nan = std::numeric_limits<float>::quiet_NaN();
  out->lo = lo;
  out->hi = hi;
  out->samples = total.n;
  out->max_rel_err = total.max_rel < 0.0 ? 0.0 : total.max_rel;
  out->mean_rel_err = total.n == 0 ? 0.0 : total.sum / static_cast<double>(total.n);
  out->argmax_input = total.arg == kNone ? 0.0f : host_input(in, total.arg);
  out->monotonic_violations = total.viol;
  out->first_violation = total.first_viol == kNone ? nan : host_input(in, total.first_viol);
  out->non_positive = total.nonpos;
  out->first_non_positive = total.first_nonpos == kNone ? nan : host_input(in, total.first_nonpos);
  return QK_OK;
}

qk_status qk_continuity_probe(const qk_exp_config* cfg, int32_t k_lo, int32_t k_hi,
                              qk_continuity_report* out) {
  if (!cfg || !out) return set_error(QK_ERR_BAD_ARGUMENT, "continuity_probe: null pointer");
  *out = qk_continuity_report{0.0, 0.0f};
  if (cfg->kind == QK_EXACT) return QK_OK;  // lab.cpp:282
  // lab.cpp:283-293, same order and messages
  if (k_hi < k_lo) return set_error(QK_ERR_BAD_ARGUMENT, "continuity_probe: empty range");
  if (static_cast<int>(kBias) + k_lo < 2 || static_cast<int>(kBias) + k_hi > 254) {
    return set_error(QK_ERR_BAD_ARGUMENT, "continuity_probe: range exceeds the normal band");
  }
  LabEval e;
  qk_status s = make_eval(cfg, &e, nullptr, nullptr);
  if (s != QK_OK) return s;
  if (e.c0 <= 0.0f) {
    return set_error(QK_ERR_BAD_ARGUMENT, "continuity_probe: requires a positive input scale");
  }
  const int nk = k_hi - k_lo + 1;
  DevBuf d;
  cudaError_t ce = cudaMalloc(&d.p, nk * sizeof(double));
  if (ce != cudaSuccess) return cuda_err(ce, "lab: cudaMalloc");
  lab_continuity_kernel<<<(nk + 127) / 128, 128>>>(e, k_lo, nk, static_cast<double*>(d.p));
  if ((ce = cudaGetLastError()) != cudaSuccess) return cuda_err(ce, "lab: continuity launch");
  std::vector<double> jump(nk);
  ce = cudaMemcpy(jump.data(), d.p, nk * sizeof(double), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_err(ce, "lab: continuity");
  for (int j = 0; j < nk; ++j) {  // lab.cpp:316-325
    if (jump[j] > out->worst_jump) {
      out->worst_jump = jump[j];
      const uint32_t boundary = static_cast<uint32_t>(static_cast<int>(kBias) + k_lo + j) << 23;
      out->at = static_cast<float>((static_cast<double>(boundary) - static_cast<double>(e.c1)) /
                                   static_cast<double>(e.c0));
    }
  }
  return QK_OK;
}

qk_status qk_quad_max_rel_err(double a0, double a1, double a2, uint64_t intervals, double* out) {
  if (!out) return set_error(QK_ERR_BAD_ARGUMENT, "quad_max_rel_err: null pointer");
  if (intervals == 0) return set_error(QK_ERR_BAD_ARGUMENT, "quad_max_rel_err: zero intervals");
  const int parts = static_cast<int>(std::min<uint64_t>(1024, (intervals + 1 + 4095) / 4096));
  std::vector<double> m;
  qk_status s = quad_max({a0, a1, a2}, std::max(parts, 1), intervals, &m);
  if (s != QK_OK) return s;
  *out = m[0];
  return QK_OK;
}

qk_status qk_grid_search_quad(const qk_grid_spec* spec, qk_grid_result* out) {
  if (!spec || !out) return set_error(QK_ERR_BAD_ARGUMENT, "grid_search_quad: null pointer");
  const size_t n0 = axis_points(spec->a0), n1 = axis_points(spec->a1), n2 = axis_points(spec->a2);
  if (n0 == 0 || n1 == 0 || n2 == 0) {
    return set_error(QK_ERR_BAD_ARGUMENT, "grid_search_quad: empty grid");
  }
  const size_t total = n0 * n1 * n2;
  auto coeffs_at = [&](size_t flat) {
    const size_t i2 = flat % n2, i1 = (flat / n2) % n1, i0 = flat / (n1 * n2);
    return std::vector<double>{axis_at(spec->a0, i0), axis_at(spec->a1, i1),
                               axis_at(spec->a2, i2)};
  };
  // coarse pass (lab.cpp:239-245) on the device
  DevBuf d;
  cudaError_t ce = cudaMalloc(&d.p, total * sizeof(double));
  if (ce != cudaSuccess) return cuda_err(ce, "lab: cudaMalloc");
  lab_grid_coarse<<<static_cast<unsigned>((total + 127) / 128), 128>>>(
      *spec, n1, n2, total, 512, static_cast<double*>(d.p));
  if ((ce = cudaGetLastError()) != cudaSuccess) return cuda_err(ce, "lab: grid launch");
  std::vector<double> coarse(total);
  ce = cudaMemcpy(coarse.data(), d.p, total * sizeof(double), cudaMemcpyDeviceToHost);
  if (ce != cudaSuccess) return cuda_err(ce, "lab: grid");
  // best candidates (lab.cpp:247-254)
  const size_t keep = std::min<size_t>(total, 2048);
  std::vector<size_t> order(total);
  std::iota(order.begin(), order.end(), size_t{0});
  std::partial_sort(order.begin(), order.begin() + static_cast<std::ptrdiff_t>(keep), order.end(),
                    [&](size_t l, size_t r) {
                      if (coarse[l] != coarse[r]) return coarse[l] < coarse[r];
                      return l < r;
                    });
  // fine re-evaluation at 2^16 intervals (lab.cpp:256-266)
  std::vector<double> triples;
  triples.reserve(keep * 3);
  for (size_t k = 0; k < keep; ++k) {
    const auto a = coeffs_at(order[k]);
    triples.insert(triples.end(), a.begin(), a.end());
  }
  std::vector<double> fine;
  qk_status s = quad_max(triples, 4, 1u << 16, &fine);
  if (s != QK_OK) return s;
  size_t best_index = order[0];
  double best_err = std::numeric_limits<double>::infinity();
  for (size_t k = 0; k < keep; ++k) {
    if (fine[k] < best_err || (fine[k] == best_err && order[k] < best_index)) {
      best_err = fine[k];
      best_index = order[k];
    }
  }
  const auto a = coeffs_at(best_index);
  out->best = qk_quad_coeffs{static_cast<float>(a[0]), static_cast<float>(a[1]),
                             static_cast<float>(a[2])};
  // independent dense re-sweep of the winner (lab.cpp:274)
  if ((s = qk_quad_max_rel_err(a[0], a[1], a[2], 1u << 20, &out->best_max_rel_err)) != QK_OK) {
    return s;
  }
  out->step_a0 = spec->a0.step;
  out->step_a1 = spec->a1.step;
  out->step_a2 = spec->a2.step;
  out->points_searched = total;
  return QK_OK;
}

qk_status qk_bias_reoptimize(const qk_exp_config* cfg, double beta_lo, double beta_hi,
                             qk_bias_result* out) {
  if (!cfg || !out) return set_error(QK_ERR_BAD_ARGUMENT, "bias_reoptimize: null pointer");
  if (cfg->kind == QK_EXACT) {  // lab.cpp:332-338, same order and messages
    return set_error(QK_ERR_BAD_ARGUMENT, "bias_reoptimize: nothing to optimize for exact");
  }
  if (!(beta_lo < beta_hi)) {
    return set_error(QK_ERR_BAD_ARGUMENT, "bias_reoptimize: empty search interval");
  }
  LabEval base;
  qk_status s = make_eval(cfg, &base, nullptr, nullptr);
  if (s != QK_OK) return s;
  const double p = cfg->natural_base ? static_cast<double>(static_cast<float>(kLog2e)) : 1.0;
  const double period = 1.0 / p;
  constexpr uint64_t kSamples = (1u << 19) + 1;
  constexpr int kBlocks = 148 * 4;
  DevBuf d;
  cudaError_t ce = cudaMalloc(&d.p, kBlocks * sizeof(double));
  if (ce != cudaSuccess) return cuda_err(ce, "lab: cudaMalloc");
  std::vector<double> h(kBlocks);
  qk_status st = QK_OK;
  auto objective = [&](double beta) -> double {  // lab.cpp:353-376
    LabEval e = base;
    qk_affine_coeffs c{};
    c.c0 = static_cast<float>(kScale * p);
    c.c1 = static_cast<float>(kScale * (static_cast<double>(kBias) - beta));
    c.input_scale = static_cast<float>(p);
    c.input_shift = 0.0f;
    c.bias_applied = beta != 0.0;
    const qk_clamp_range r = qk_clamp_for(&c);
    e.c0 = c.c0;
    e.c1 = c.c1;
    e.lo = r.lo;
    e.hi = r.hi;
    lab_bias_objective<<<kBlocks, kLabThreads>>>(e, period, kSamples, static_cast<double*>(d.p));
    cudaError_t err = cudaGetLastError();
    if (err == cudaSuccess) {
      err = cudaMemcpy(h.data(), d.p, kBlocks * sizeof(double), cudaMemcpyDeviceToHost);
    }
    if (err != cudaSuccess) {
      st = cuda_err(err, "lab: bias objective");
      return 0.0;
    }
    return *std::max_element(h.begin(), h.end());
  };
  constexpr double kGolden = 0.6180339887498949;  // lab.cpp:378-399
  double a = beta_lo, b = beta_hi;
  double x1 = b - kGolden * (b - a);
  double x2 = a + kGolden * (b - a);
  double f1 = objective(x1);
  double f2 = objective(x2);
  while (st == QK_OK && b - a > 1e-6) {
    if (f1 <= f2) {
      b = x2;
      x2 = x1;
      f2 = f1;
      x1 = b - kGolden * (b - a);
      f1 = objective(x1);
    } else {
      a = x1;
      x1 = x2;
      f1 = f2;
      x2 = a + kGolden * (b - a);
      f2 = objective(x2);
    }
  }
  const double beta = 0.5 * (a + b);
  out->beta = static_cast<float>(beta);
  out->max_rel_err = objective(beta);
  out->near_reference_bias = std::abs(beta - kCenteringBias) <= 0.0035 ? 1 : 0;
  return st;
}

}  // extern "C"
