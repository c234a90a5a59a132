// Elementwise QuAKE kernels for sm_100a: exp (K1/K2), logistic (K3),
// GELU (K4) and the expf / __expf comparison kernels (K7/K8) of identical
// structure.
//
// Design (HBM-bound: 8 algorithmic bytes per element):
//  * one wave of contiguous tiles (non-persistent grid; see ew_vec_kernel),
//  * 128-bit coalesced ld.global.cs / st.global.cs (streaming: every byte is
//    touched exactly once, so keep it from displacing L2),
//  * U float4 loads in flight per thread before any compute (MLP),
//  * per-element arithmetic from numerics.cuh — bit-exact restatements of the
//    reference's no-FMA operation sequence.
// Reference paths cited relative to /root/reference/proj/.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>

#include "internal.h"
#include "numerics.cuh"

namespace qk {
namespace {

constexpr int kThreads = 256;

template <bool X86>
__device__ __forceinline__ float sat(float x, const EwParams& p) {
  return X86 ? saturate(x, p.lo, p.hi) : saturate_fast(x, p.lo, p.hi);
}

template <EwOp OP, bool X86>
__device__ __forceinline__ float apply(float x, const EwParams& p) {
  if constexpr (OP == EwOp::kQuake) {
    // kernels.cpp:103-104 (X86: the caller's clamp may be NaN or unbounded;
    // keep the literal select chain and the x86 conversion there)
    return quake_body<X86>(sat<X86>(x, p), p.c0, p.c1);
  } else if constexpr (OP == EwOp::kQuake2) {
    // kernels.cpp:118-124
    return quake2_body<false, X86>(sat<X86>(x, p), p.c0, p.c1, 0.f, 0.f, 0.f);
  } else if constexpr (OP == EwOp::kQuake2General) {
    // kernels.cpp:126-134
    return quake2_body<true, X86>(sat<X86>(x, p), p.c0, p.c1, p.a0, p.a1, p.a2);
  } else if constexpr (OP == EwOp::kExpExpf) {
    return expf(x);
  } else if constexpr (OP == EwOp::kExpFast) {
    return __expf(x);
  } else if constexpr (OP == EwOp::kLogisticQuake) {
    // nonlin.cpp:229-231: 1 / (1 + e). __frcp_rn is the correctly rounded
    // reciprocal, i.e. exactly IEEE 1.0f / d.
    const float e = quake_body(saturate_fast(x, p.lo, p.hi), p.c0, p.c1);
    return __frcp_rn(__fadd_rn(1.0f, e));
  } else if constexpr (OP == EwOp::kLogisticQuake2) {
    // nonlin.cpp:237-240
    const float e = quake2_body<false>(saturate_fast(x, p.lo, p.hi), p.c0, p.c1, 0.f, 0.f, 0.f);
    return __frcp_rn(__fadd_rn(1.0f, e));
  } else if constexpr (OP == EwOp::kLogisticExpf) {
    // nonlin.cpp:219: 1.0f / (1.0f + std::exp(-x))
    return __frcp_rn(__fadd_rn(1.0f, expf(-x)));
  } else if constexpr (OP == EwOp::kLogisticFast) {
    return __frcp_rn(__fadd_rn(1.0f, __expf(-x)));
  } else if constexpr (OP == EwOp::kGeluQuake || OP == EwOp::kGeluQuake2) {
    // nonlin.cpp:266-273 gelu_inner (plain branch): u = x * (x*x + 1/kappa),
    // then nonlin.cpp:314-317 / 324-327: x / (1 + quake(saturate(u))).
    const float u = __fmul_rn(x, __fadd_rn(__fmul_rn(x, x), p.k0));
    const float s = saturate_fast(u, p.lo, p.hi);
    const float e = OP == EwOp::kGeluQuake
                        ? quake_body(s, p.c0, p.c1)
                        : quake2_body<false>(s, p.c0, p.c1, 0.f, 0.f, 0.f);
    // 1 + e is finite and >= 1, so the quotient is NaN only for NaN x, where
    // SSE's divss returns x quieted (payload kept).
    const float y = __fdiv_rn(x, __fadd_rn(1.0f, e));
    return y != y ? x86_quiet(x) : y;
  } else if constexpr (OP == EwOp::kGeluQuakeUnfused || OP == EwOp::kGeluQuake2Unfused) {
    // bench.cpp:212-233 (ablation): w = fused_scale*x*(inverse_kappa + x*x)
    // computed explicitly (k1 = fused_scale), then x / (1 + e^-w) with the
    // negated natural-exp coefficients in c0/c1.
    const float w = __fmul_rn(__fmul_rn(p.k1, x), __fadd_rn(p.k0, __fmul_rn(x, x)));
    const float s = saturate_fast(w, p.lo, p.hi);
    const float e = OP == EwOp::kGeluQuakeUnfused
                        ? quake_body(s, p.c0, p.c1)
                        : quake2_body<false>(s, p.c0, p.c1, 0.f, 0.f, 0.f);
    const float y = __fdiv_rn(x, __fadd_rn(1.0f, e));
    return y != y ? x86_quiet(x) : y;
  } else if constexpr (OP == EwOp::kGeluTanh) {
    // nonlin.cpp:302-304: 0.5f*x*(1 + tanh(r2pi*(x + kappa*x*x*x)))
    const float cube = __fmul_rn(__fmul_rn(__fmul_rn(p.k1, x), x), x);
    const float th = tanhf(__fmul_rn(p.k2, __fadd_rn(x, cube)));
    return __fmul_rn(__fmul_rn(0.5f, x), __fadd_rn(1.0f, th));
  } else if constexpr (OP == EwOp::kGeluExpf || OP == EwOp::kGeluFast) {
    // Same sigmoid structure as the QuAKE GELU with the exponential swapped;
    // c0 carries -fused_scale.
    const float u = __fmul_rn(x, __fadd_rn(__fmul_rn(x, x), p.k0));
    const float a = __fmul_rn(p.c0, u);
    const float e = OP == EwOp::kGeluExpf ? expf(a) : __expf(a);
    return __fdiv_rn(x, __fadd_rn(1.0f, e));
  } else {
    return x;
  }
}

// Two elements of the QuAKE ops with the paired FMUL2/FFMA2 sequences of
// numerics.cuh (bit-identical to apply<OP>); other ops go element-wise.
// The guard records the range the paired fast divisions saw; apply4 tests it
// once per float4 and the caller recomputes a refused float4 with apply.
template <EwOp OP, bool X86>
__device__ __forceinline__ void apply2(float& a, float& b, const EwParams& p, DivGuard& g) {
  if constexpr (X86 || !(OP == EwOp::kQuake || OP == EwOp::kQuake2 ||
                         OP == EwOp::kQuake2General || OP == EwOp::kLogisticQuake ||
                         OP == EwOp::kLogisticQuake2 || OP == EwOp::kGeluQuake ||
                         OP == EwOp::kGeluQuake2 || OP == EwOp::kGeluQuakeUnfused ||
                         OP == EwOp::kGeluQuake2Unfused)) {
    a = apply<OP, X86>(a, p);
    b = apply<OP, X86>(b, p);
  } else if constexpr (OP == EwOp::kGeluQuakeUnfused || OP == EwOp::kGeluQuake2Unfused) {
    // w = (fs*x) * (ik + x*x): x*x feeds an add (scalar add), fs*x and the
    // outer product feed no add, so all three products can be paired
    float s0, s1, f0, f1;
    unpack2(mul2_rn(pack2(a, b), pack2(a, b)), s0, s1);
    unpack2(mul2_rn(pack2(p.k1, p.k1), pack2(a, b)), f0, f1);
    float w0, w1;
    unpack2(mul2_rn(pack2(f0, f1), pack2(__fadd_rn(p.k0, s0), __fadd_rn(p.k0, s1))), w0, w1);
    w0 = saturate_fast(w0, p.lo, p.hi);
    w1 = saturate_fast(w1, p.lo, p.hi);
    float e0, e1;
    if constexpr (OP == EwOp::kGeluQuakeUnfused) {
      quake_body2(w0, w1, p.c0, p.c1, e0, e1);
    } else {
      quake2_body2<false>(w0, w1, p.c0, p.c1, 0.f, 0.f, 0.f, e0, e1);
    }
    const float y0 = __fdiv_rn(a, __fadd_rn(1.0f, e0));
    const float y1 = __fdiv_rn(b, __fadd_rn(1.0f, e1));
    a = y0 != y0 ? x86_quiet(a) : y0;
    b = y1 != y1 ? x86_quiet(b) : y1;
  } else if constexpr (OP == EwOp::kGeluQuake || OP == EwOp::kGeluQuake2) {
    // u = x * (x*x + 1/kappa): the first product is added (scalar add), the
    // second feeds the clamp, so both products can be paired
    float s0, s1;
    unpack2(mul2_rn(pack2(a, b), pack2(a, b)), s0, s1);
    float u0, u1;
    unpack2(mul2_rn(pack2(a, b), pack2(__fadd_rn(s0, p.k0), __fadd_rn(s1, p.k0))), u0, u1);
    u0 = saturate_fast(u0, p.lo, p.hi);
    u1 = saturate_fast(u1, p.lo, p.hi);
    float e0, e1;
    if constexpr (OP == EwOp::kGeluQuake) {
      quake_body2(u0, u1, p.c0, p.c1, e0, e1);
    } else {
      quake2_body2<false>(u0, u1, p.c0, p.c1, 0.f, 0.f, 0.f, e0, e1);
    }
    div2_ge1(a, b, __fadd_rn(1.0f, e0), __fadd_rn(1.0f, e1), g);
  } else {
    const float u0 = saturate_fast(a, p.lo, p.hi), u1 = saturate_fast(b, p.lo, p.hi);
    float e0, e1;
    if constexpr (OP == EwOp::kQuake || OP == EwOp::kLogisticQuake) {
      quake_body2(u0, u1, p.c0, p.c1, e0, e1);
    } else if constexpr (OP == EwOp::kQuake2General) {
      quake2_body2<true>(u0, u1, p.c0, p.c1, p.a0, p.a1, p.a2, e0, e1);
    } else {
      quake2_body2<false>(u0, u1, p.c0, p.c1, 0.f, 0.f, 0.f, e0, e1);
    }
    if constexpr (OP == EwOp::kLogisticQuake || OP == EwOp::kLogisticQuake2) {
      recip2_ge1(__fadd_rn(1.0f, e0), __fadd_rn(1.0f, e1), a, b, g);
    } else {
      a = e0;
      b = e1;
    }
  }
}

template <EwOp OP, bool X86>
__device__ __forceinline__ float4 apply4(float4 v, const EwParams& p, bool& ok) {
  DivGuard g;
  apply2<OP, X86>(v.x, v.y, p, g);
  apply2<OP, X86>(v.z, v.w, p, g);
  // one range test per float4 (paired fast divisions only)
  if constexpr (!X86 && (OP == EwOp::kGeluQuake || OP == EwOp::kGeluQuake2)) {
    ok = div_guard_ok(g);
  } else if constexpr (!X86 && (OP == EwOp::kLogisticQuake || OP == EwOp::kLogisticQuake2)) {
    ok = recip_guard_ok(g);
  }
  return v;
}

// The exact element-wise path (IEEE divisions), for float4s the fast path refused.
template <EwOp OP, bool X86>
__device__ __forceinline__ float4 apply4_exact(float4 v, const EwParams& p) {
  return make_float4(apply<OP, X86>(v.x, p), apply<OP, X86>(v.y, p), apply<OP, X86>(v.z, p),
                     apply<OP, X86>(v.w, p));
}

template <EwOp OP, bool X86>
__device__ __forceinline__ float4 apply4_checked(float4 v, const EwParams& p) {
  bool ok = true;
  const float4 y = apply4<OP, X86>(v, p, ok);
  return __builtin_expect(ok, 1) ? y : apply4_exact<OP, X86>(v, p);
}

// Vector path: in+head and out+head are both 16-byte aligned. Each CTA
// streams one contiguous tile of 256*U float4 (U loads in flight per thread,
// all issued before any compute); the grid covers the buffer in one wave of
// tiles. This non-persistent shape measured fastest on B200 for pure streams
// (scripts/stream_probe.cu: 6.6 TB/s at 1 GiB vs 5.8 for a persistent
// grid-stride loop and 6.2 for a persistent TMA bulk pipeline). The < 4
// leading elements (`head`) and the < 4 trailing ones go scalar in CTA 0.
template <EwOp OP, bool X86, int U>
__global__ void __launch_bounds__(kThreads, 4) ew_vec_kernel(const float* __restrict__ in,
                                                          float* __restrict__ out, size_t n,
                                                          size_t head, EwParams p) {
  pdl_entry();
  const size_t n4 = (n - head) >> 2;
  const float4* __restrict__ in4 = reinterpret_cast<const float4*>(in + head);
  float4* __restrict__ out4 = reinterpret_cast<float4*>(out + head);
  constexpr size_t kTile = static_cast<size_t>(kThreads) * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * kTile; base < n4;
       base += static_cast<size_t>(gridDim.x) * kTile) {
    float4 v[U];
    if (base + kTile <= n4) {
#pragma unroll
      for (int u = 0; u < U; ++u) v[u] = __ldcs(in4 + base + u * kThreads + threadIdx.x);
#pragma unroll
      for (int u = 0; u < U; ++u) {
        __stcs(out4 + base + u * kThreads + threadIdx.x, apply4_checked<OP, X86>(v[u], p));
      }
    } else {
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + u * kThreads + threadIdx.x;
        if (i < n4) v[u] = __ldcs(in4 + i);
      }
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const size_t i = base + u * kThreads + threadIdx.x;
        if (i < n4) __stcs(out4 + i, apply4_checked<OP, X86>(v[u], p));
      }
    }
  }
  if (blockIdx.x == 0) {
    const size_t tail0 = head + (n4 << 2);
    if (threadIdx.x < head) out[threadIdx.x] = apply<OP, X86>(in[threadIdx.x], p);
    if (threadIdx.x < n - tail0) out[tail0 + threadIdx.x] = apply<OP, X86>(in[tail0 + threadIdx.x], p);
  }
}

// Scalar path for buffers whose input and output are not co-aligned.
template <EwOp OP, bool X86, int U>
__global__ void __launch_bounds__(kThreads) ew_scalar_kernel(const float* __restrict__ in,
                                                             float* __restrict__ out, size_t n,
                                                             EwParams p) {
  pdl_entry();
  constexpr size_t kTile = static_cast<size_t>(kThreads) * U;
  for (size_t base = static_cast<size_t>(blockIdx.x) * kTile; base < n;
       base += static_cast<size_t>(gridDim.x) * kTile) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + u * kThreads + threadIdx.x;
      if (i < n) v[u] = __ldcs(in + i);
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const size_t i = base + u * kThreads + threadIdx.x;
      if (i < n) __stcs(out + i, apply<OP, X86>(v[u], p));
    }
  }
}

constexpr size_t kMaxGrid = 0x7FFFFFFFu;

template <EwOp OP, bool X86>
cudaError_t launch_op(const float* in, float* out, size_t n, const EwParams& p, int /*sm_count*/,
                      cudaStream_t stream) {
  const uintptr_t ai = reinterpret_cast<uintptr_t>(in) & 15u;
  const uintptr_t ao = reinterpret_cast<uintptr_t>(out) & 15u;
  const bool vec = ai == ao && (ai & 3u) == 0;
  if (vec) {
#ifndef QK_EW_U
#define QK_EW_U 4
#endif
    constexpr int U = QK_EW_U;
    const size_t head = ai == 0 ? 0 : (16u - ai) / 4u;
    const size_t h = head < n ? head : n;
    const size_t n4 = (n - h) / 4;
    size_t blocks = (n4 + static_cast<size_t>(kThreads) * U - 1) / (static_cast<size_t>(kThreads) * U);
    if (blocks > kMaxGrid) blocks = kMaxGrid;
    if (blocks == 0) blocks = 1;
    return launch_ex(ew_vec_kernel<OP, X86, U>, dim3(static_cast<unsigned>(blocks)), dim3(kThreads),
                     0, stream, 0, in, out, n, h, p);
  } else {
    constexpr int U = 8;
    size_t blocks = (n + static_cast<size_t>(kThreads) * U - 1) / (static_cast<size_t>(kThreads) * U);
    if (blocks > kMaxGrid) blocks = kMaxGrid;
    if (blocks == 0) blocks = 1;
    return launch_ex(ew_scalar_kernel<OP, X86, U>, dim3(static_cast<unsigned>(blocks)),
                     dim3(kThreads), 0, stream, 0, in, out, n, p);
  }
}

// Validation pass of the host-span softmax (nonlin.cpp:43-55 rejects any
// non-finite element): sets bit 0 of *flags when x[0..n) holds a NaN or an
// infinity. Reads only; used where `out` must stay untouched until every
// row has been checked (device `out` spans, inputs larger than the
// workspace). One flag write per CTA at most.
__global__ void __launch_bounds__(kThreads) check_finite_kernel(const float* __restrict__ x,
                                                                size_t n, size_t head,
                                                                uint32_t* __restrict__ flags) {
  pdl_entry();
  const size_t n4 = (n - head) >> 2;
  const float4* __restrict__ x4 = reinterpret_cast<const float4*>(x + head);
  bool bad = false;  // !(|v| <= FLT_MAX) holds exactly for NaN and +-Inf
  for (size_t i = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x; i < n4;
       i += static_cast<size_t>(gridDim.x) * kThreads) {
    const float4 v = __ldcs(x4 + i);
    const float a = fmaxf(fmaxf(fabsf(v.x), fabsf(v.y)), fmaxf(fabsf(v.z), fabsf(v.w)));
    // fmaxf drops a NaN operand: test NaN separately via self-comparison
    bad |= !(a <= 3.402823466e38f) || v.x != v.x || v.y != v.y || v.z != v.z || v.w != v.w;
  }
  if (blockIdx.x == 0) {
    const size_t tail0 = head + (n4 << 2);
    if (threadIdx.x < head) bad |= !(fabsf(x[threadIdx.x]) <= 3.402823466e38f);
    if (threadIdx.x < n - tail0) bad |= !(fabsf(x[tail0 + threadIdx.x]) <= 3.402823466e38f);
  }
  if (__syncthreads_or(bad) && threadIdx.x == 0) atomicOr(flags, 1u);
}

// One store to mapped pinned host memory (a plain launch: it starts after the
// preceding kernels of the stream have completed and their atomics landed).
__global__ void publish_flag_kernel(const uint32_t* __restrict__ flags, uint32_t* slot) {
  *reinterpret_cast<volatile uint32_t*>(slot) = *flags | kFlagPublished;
  __threadfence_system();
}

}  // namespace

cudaError_t launch_publish_flag(const uint32_t* flags, uint32_t* slot, cudaStream_t stream) {
  publish_flag_kernel<<<1, 1, 0, stream>>>(flags, slot);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const float* x, size_t n, uint32_t* flags, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  if (reinterpret_cast<uintptr_t>(x) & 3u) return cudaErrorMisalignedAddress;
  const uintptr_t a = reinterpret_cast<uintptr_t>(x) & 15u;
  const size_t head = std::min<size_t>(a == 0 ? 0 : (16u - a) / 4u, n);
  size_t blocks = ((n - head) / 4 + kThreads * 8 - 1) / (kThreads * 8);
  if (blocks == 0) blocks = 1;
  if (blocks > 148 * 8) blocks = 148 * 8;
  return launch_ex(check_finite_kernel, dim3(static_cast<unsigned>(blocks)), dim3(kThreads), 0,
                   stream, 0, x, n, head, flags);
}

cudaError_t launch_elementwise(EwOp op, const float* in, float* out, size_t n, const EwParams& p,
                               int sm_count, cudaStream_t stream) {
  if (n == 0) return cudaSuccess;
  const bool x86 = p.x86_overflow != 0;
  switch (op) {
    case EwOp::kQuake:
      return x86 ? launch_op<EwOp::kQuake, true>(in, out, n, p, sm_count, stream)
                 : launch_op<EwOp::kQuake, false>(in, out, n, p, sm_count, stream);
    case EwOp::kQuake2:
      return x86 ? launch_op<EwOp::kQuake2, true>(in, out, n, p, sm_count, stream)
                 : launch_op<EwOp::kQuake2, false>(in, out, n, p, sm_count, stream);
    case EwOp::kQuake2General:
      return x86 ? launch_op<EwOp::kQuake2General, true>(in, out, n, p, sm_count, stream)
                 : launch_op<EwOp::kQuake2General, false>(in, out, n, p, sm_count, stream);
    case EwOp::kExpExpf: return launch_op<EwOp::kExpExpf, false>(in, out, n, p, sm_count, stream);
    case EwOp::kExpFast: return launch_op<EwOp::kExpFast, false>(in, out, n, p, sm_count, stream);
    case EwOp::kLogisticQuake:
      return launch_op<EwOp::kLogisticQuake, false>(in, out, n, p, sm_count, stream);
    case EwOp::kLogisticQuake2:
      return launch_op<EwOp::kLogisticQuake2, false>(in, out, n, p, sm_count, stream);
    case EwOp::kLogisticExpf:
      return launch_op<EwOp::kLogisticExpf, false>(in, out, n, p, sm_count, stream);
    case EwOp::kLogisticFast:
      return launch_op<EwOp::kLogisticFast, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluQuake: return launch_op<EwOp::kGeluQuake, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluQuake2:
      return launch_op<EwOp::kGeluQuake2, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluTanh: return launch_op<EwOp::kGeluTanh, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluExpf: return launch_op<EwOp::kGeluExpf, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluFast: return launch_op<EwOp::kGeluFast, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluQuakeUnfused:
      return launch_op<EwOp::kGeluQuakeUnfused, false>(in, out, n, p, sm_count, stream);
    case EwOp::kGeluQuake2Unfused:
      return launch_op<EwOp::kGeluQuake2Unfused, false>(in, out, n, p, sm_count, stream);
  }
  return cudaErrorInvalidValue;
}

}  // namespace qk
