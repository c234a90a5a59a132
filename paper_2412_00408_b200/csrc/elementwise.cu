// Elementwise QuAKE kernels for sm_100a: exp (K1/K2), logistic (K3),
// GELU (K4) and the expf / __expf comparison kernels (K7/K8) of identical
// structure.
//
// Design (HBM-bound: 8 algorithmic bytes per element):
//  * persistent grid-stride CTAs sized from the SM count x occupancy,
//  * 128-bit coalesced ld.global.cs / st.global.cs (streaming: every byte is
//    touched exactly once, so keep it from displacing L2),
//  * U float4 loads in flight per thread before any compute (MLP),
//  * per-element arithmetic from numerics.cuh — bit-exact restatements of the
//    reference's no-FMA operation sequence.
// Reference paths cited relative to /root/reference/proj/.
#include <cuda_runtime.h>

#include <cmath>

#include "internal.h"
#include "numerics.cuh"

namespace qk {
namespace {

constexpr int kThreads = 256;

template <EwOp OP, bool X86>
__device__ __forceinline__ float apply(float x, const EwParams& p) {
  if constexpr (OP == EwOp::kQuake) {
    // kernels.cpp:103-104
    return quake_body<X86>(saturate(x, p.lo, p.hi), p.c0, p.c1);
  } else if constexpr (OP == EwOp::kQuake2) {
    // kernels.cpp:118-124
    return quake2_body<false, X86>(saturate(x, p.lo, p.hi), p.c0, p.c1, 0.f, 0.f, 0.f);
  } else if constexpr (OP == EwOp::kQuake2General) {
    // kernels.cpp:126-134
    return quake2_body<true, X86>(saturate(x, p.lo, p.hi), p.c0, p.c1, p.a0, p.a1, p.a2);
  } else if constexpr (OP == EwOp::kExpExpf) {
    return expf(x);
  } else if constexpr (OP == EwOp::kExpFast) {
    return __expf(x);
  } else if constexpr (OP == EwOp::kLogisticQuake) {
    // nonlin.cpp:229-231: 1 / (1 + e). __frcp_rn is the correctly rounded
    // reciprocal, i.e. exactly IEEE 1.0f / d.
    const float e = quake_body(saturate(x, p.lo, p.hi), p.c0, p.c1);
    return __frcp_rn(__fadd_rn(1.0f, e));
  } else if constexpr (OP == EwOp::kLogisticQuake2) {
    // nonlin.cpp:237-240
    const float e = quake2_body<false>(saturate(x, p.lo, p.hi), p.c0, p.c1, 0.f, 0.f, 0.f);
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
    const float s = saturate(u, p.lo, p.hi);
    const float e = OP == EwOp::kGeluQuake
                        ? quake_body(s, p.c0, p.c1)
                        : quake2_body<false>(s, p.c0, p.c1, 0.f, 0.f, 0.f);
    // 1 + e is finite and >= 1, so the quotient is NaN only for NaN x, where
    // SSE's divss returns x quieted (payload kept).
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

template <EwOp OP, bool X86>
__device__ __forceinline__ float4 apply4(float4 v, const EwParams& p) {
  v.x = apply<OP, X86>(v.x, p);
  v.y = apply<OP, X86>(v.y, p);
  v.z = apply<OP, X86>(v.z, p);
  v.w = apply<OP, X86>(v.w, p);
  return v;
}

// Vector path: in+head and out+head are both 16-byte aligned. The first
// `head` (< 4) elements and the < 4 trailing ones are done scalar by the
// first threads of the grid.
template <EwOp OP, bool X86, int U>
__global__ void __launch_bounds__(kThreads) ew_vec_kernel(const float* __restrict__ in,
                                                          float* __restrict__ out, size_t n,
                                                          size_t head, EwParams p) {
  const size_t n4 = (n - head) >> 2;
  const float4* __restrict__ in4 = reinterpret_cast<const float4*>(in + head);
  float4* __restrict__ out4 = reinterpret_cast<float4*>(out + head);
  const size_t tid = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * kThreads;
  size_t i = tid;
  for (; i + (U - 1) * stride < n4; i += U * stride) {
    float4 v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(in4 + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out4 + i + u * stride, apply4<OP, X86>(v[u], p));
  }
  for (; i < n4; i += stride) __stcs(out4 + i, apply4<OP, X86>(__ldcs(in4 + i), p));
  const size_t tail0 = head + (n4 << 2);
  if (tid < head) out[tid] = apply<OP, X86>(in[tid], p);
  if (tid < n - tail0) out[tail0 + tid] = apply<OP, X86>(in[tail0 + tid], p);
}

// Scalar path for buffers whose input and output are not co-aligned.
template <EwOp OP, bool X86, int U>
__global__ void __launch_bounds__(kThreads) ew_scalar_kernel(const float* __restrict__ in,
                                                             float* __restrict__ out, size_t n,
                                                             EwParams p) {
  const size_t tid = static_cast<size_t>(blockIdx.x) * kThreads + threadIdx.x;
  const size_t stride = static_cast<size_t>(gridDim.x) * kThreads;
  size_t i = tid;
  for (; i + (U - 1) * stride < n; i += U * stride) {
    float v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) v[u] = __ldcs(in + i + u * stride);
#pragma unroll
    for (int u = 0; u < U; ++u) __stcs(out + i + u * stride, apply<OP, X86>(v[u], p));
  }
  for (; i < n; i += stride) __stcs(out + i, apply<OP, X86>(__ldcs(in + i), p));
}

template <EwOp OP, bool X86>
cudaError_t launch_op(const float* in, float* out, size_t n, const EwParams& p, int sm_count,
                      cudaStream_t stream) {
  constexpr int U = 4;
  const uintptr_t ai = reinterpret_cast<uintptr_t>(in) & 15u;
  const uintptr_t ao = reinterpret_cast<uintptr_t>(out) & 15u;
  const bool vec = ai == ao && (ai & 3u) == 0;
  static int occ_vec = 0, occ_scalar = 0;  // resident CTAs per SM (per instantiation)
  if (vec) {
    if (occ_vec == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_vec, ew_vec_kernel<OP, X86, U>, kThreads,
                                                    0);
      if (occ_vec <= 0) occ_vec = 1;
    }
    const size_t head = ai == 0 ? 0 : (16u - ai) / 4u;
    const size_t h = head < n ? head : n;
    const size_t n4 = (n - h) / 4;
    size_t blocks = (n4 + static_cast<size_t>(kThreads) * U - 1) / (static_cast<size_t>(kThreads) * U);
    const size_t cap = static_cast<size_t>(sm_count) * occ_vec;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    ew_vec_kernel<OP, X86, U><<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(in, out, n, h,
                                                                                      p);
  } else {
    if (occ_scalar == 0) {
      cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ_scalar, ew_scalar_kernel<OP, X86, U>,
                                                    kThreads, 0);
      if (occ_scalar <= 0) occ_scalar = 1;
    }
    size_t blocks = (n + static_cast<size_t>(kThreads) * U - 1) / (static_cast<size_t>(kThreads) * U);
    const size_t cap = static_cast<size_t>(sm_count) * occ_scalar;
    if (blocks > cap) blocks = cap;
    if (blocks == 0) blocks = 1;
    ew_scalar_kernel<OP, X86, U><<<static_cast<unsigned>(blocks), kThreads, 0, stream>>>(in, out,
                                                                                         n, p);
  }
  return cudaGetLastError();
}

}  // namespace

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
  }
  return cudaErrorInvalidValue;
}

}  // namespace qk
