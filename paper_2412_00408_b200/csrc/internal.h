// Internal launch interface between the C++ host layer (host_api.cpp) and
// the sm_100a kernels (elementwise.cu, softmax.cu). Not part of the ABI.
#pragma once

#include <cuda_runtime.h>

#include <cstddef>
#include <cstdint>
#include <cstdlib>
#include <string>
#include <utility>

#include "quake_b200.h"

namespace qk {

// Elementwise operator families (one templated kernel per family).
enum class EwOp : int {
  kQuake = 0,         // kernels.cpp:95-107 quake_buffer
  kQuake2 = 1,        // kernels.cpp:109-136 quake2_buffer, continuity quad
  kQuake2General = 2, // quake2_buffer, any other quad (refine_general)
  kExpExpf = 3,       // comparison: expf(x), identical structure
  kExpFast = 4,       // comparison: __expf(x)
  kLogisticQuake = 5, // nonlin.cpp:225-233
  kLogisticQuake2 = 6,// nonlin.cpp:234-242
  kLogisticExpf = 7,  // nonlin.cpp:215-221 (Exact)
  kLogisticFast = 8,  // comparison: __expf
  kGeluQuake = 9,     // nonlin.cpp:310-319
  kGeluQuake2 = 10,   // nonlin.cpp:320-329
  kGeluTanh = 11,     // nonlin.cpp:298-306 (Exact, tanh form)
  kGeluExpf = 12,     // comparison: sigmoid form with expf
  kGeluFast = 13,     // comparison: sigmoid form with __expf
  kGeluQuakeUnfused = 14,  // ablation: bench.cpp:212-233, w = fs*x*(ik + x*x) into e^-w
  kGeluQuake2Unfused = 15,
};

struct EwParams {
  float c0, c1;          // fused affine coefficients
  float lo, hi;          // saturation range
  float a0, a1, a2;      // quad coefficients (kQuake2General)
  float k0, k1, k2;      // op constants (GELU: inverse_kappa / kappa / root2_over_pi)
  int x86_overflow;      // 1: emulate cvttss2si out-of-range semantics
};

// Launch the elementwise kernel for `op` over n floats. No allocation, no
// synchronisation. `sm_count` sizes the persistent grid.
cudaError_t launch_elementwise(EwOp op, const float* in, float* out, size_t n,
                               const EwParams& p, int sm_count, cudaStream_t stream);

// Validation pass: OR 1 into *flags (device) when x[0..n) holds a non-finite value.
cudaError_t launch_check_finite(const float* x, size_t n, uint32_t* flags, cudaStream_t stream);

// Publishes *flags (device) to *slot (mapped pinned host memory) as
// `*flags | kFlagPublished`, stream-ordered after the kernels that raise it:
// the host-span driver polls the slot instead of synchronising the stream.
constexpr uint32_t kFlagPublished = 0x80000000u;
cudaError_t launch_publish_flag(const uint32_t* flags, uint32_t* slot, cudaStream_t stream);

// ---- row softmax ----

enum class SmKernel : int { kExact = 0, kQuake = 1, kQuake2 = 2, kQuake2General = 3,
                            kExpf = 4, kFast = 5,
                            // ablation (bench.cpp:137-166): t*(x - m) computed
                            // explicitly, natural-exp QuAKE on the saturated value
                            kQuakeUnfused = 6, kQuake2Unfused = 7 };

// Reduction geometry of one launch (also reported through qk_softmax_plan so
// the tests can restate the exact summation order).
enum class SmVariant : int {
  // 0 (warp per row, float4 lanes), 1 (warp per row, scalar lanes), 5
  // (two-row lookahead pipeline), 8 (several short rows per warp) and 12
  // (TMA row tiles): retired, measured slower than the kernels below; the
  // numbers stay reserved
  kSmem = 2,        // CTA (or cluster of CTAs) per row, row staged in smem
  kGlobal3 = 3,     // CTA per row, three sweeps over global memory (huge rows)
  kPipe = 4,        // persistent cluster per row group, multi-stage TMA pipeline
  kPipeL2 = 6,      // long rows: one smem stage, prefix refilled under the exps
  kPipeS = 7,       // kPipe with one-float chunks: rows of cols % 4 != 0 (unaligned)
  kThreadRow = 9,   // one thread per row (<= 16 cols): the reference's sequential order
  kRowsSmem = 10,   // one thread per row, rows staged through smem (coalesced), <= 64 cols
  kSubWarp = 11,    // G lanes per aligned row, up to 8 float4 chunks each (lanes = G)
  kSpan = 13,       // row spans through smem at any address / length, float4 chunks, G lanes
  kWarpRing = 14,   // per-agent (1-8 warps) TMA ring of row spans, scalar lanes: rows of cols % 4 != 0
};

struct SmPlan {
  SmVariant variant;
  int width;        // elements per lane access (4 = float4, 1 = scalar)
  int lanes;        // threads contributing partial sums per CTA (tree size)
  int cluster;      // CTAs per row (1 = no cluster)
  long long slice;  // chunks (of `width` elements) per CTA slice; 0 = whole row
  int vpt;          // warp variants: chunks held per lane
  int threads;      // CTA size
  size_t smem;      // dynamic shared memory per CTA (bytes)
  int stages;       // kPipe: row slices in flight per CTA
  int balanced;     // kPipe: rank r owns q (+1 if r < nchunks % cluster) chunks
  int resident;     // kPipe: clusters resident at once (occupancy API; 0 = unknown)
  int rr;           // kWarpRing: rows per job
  int pf;           // kPipeL2: rows bulk-prefetched into L2 ahead (0 = off)
};

struct SmParams {
  float t;          // temperature (Exact paths)
  float c0;         // RN(2^23 * t * log2e)          nonlin.cpp:89
  double c1_base;   // 2^23 * (127 - beta)           nonlin.cpp:90-91
  double vmin_off;  // 126 * ln2 / t                 nonlin.cpp:92-93
  float a0, a1, a2; // quad (kQuake2General)
  int general_quad; // 1: y_m may leave [1, 2]; rows use SSE-exact semantics
  float nat_c0, nat_c1, nat_lo, nat_hi;  // unfused kinds: natural-exp coefficients / clamp
  int unfused;      // 1: kQuakeUnfused / kQuake2Unfused
  int pdl_late;     // persistent kernels: trigger the dependent launch after the last row
  // 16-byte phase of every row's input / output in floats (0..3). Nonzero only
  // for float4-chunk plans (cols % 4 == 0) on a base that is not 16-byte
  // aligned; the kernels then read straddling chunks and split the stores,
  // keeping the chunk order, so results do not depend on the address.
  int iph, oph;
};

// The plan depends on (device, cols, kind) and the planner options only —
// never on the row count or the data's address (see softmax.cu). Cached.
SmPlan plan_softmax(size_t cols, int device, SmKernel kind);
// Planner options (QK_SM_* measurement knobs): environment read once, then
// qk_set_plan_override. set_plan_opt(nullptr, ...) clears all; false = unknown name.
int plan_opt(const char* name, int dflt);
bool set_plan_opt(const char* name, int value, bool clear);

// Launch softmax over `rows` rows of `cols` columns. `flags` (device, may be
// null) receives bit 0 when a non-finite input was seen.
// Per-kind launchers (softmax_k_*.cu) and the planner's occupancy probe.
#define QK_SOFTMAX_LAUNCHER(name)                                                        \
  cudaError_t launch_softmax_##name(const SmPlan& plan, const float* in, float* out,      \
                                    size_t rows, size_t cols, const SmParams& p,         \
                                    uint32_t* flags, cudaStream_t stream);
QK_SOFTMAX_LAUNCHER(exact)
QK_SOFTMAX_LAUNCHER(fast)
QK_SOFTMAX_LAUNCHER(quake)
QK_SOFTMAX_LAUNCHER(quake2)
QK_SOFTMAX_LAUNCHER(quake2g)
QK_SOFTMAX_LAUNCHER(quake_unfused)
QK_SOFTMAX_LAUNCHER(quake2_unfused)
#undef QK_SOFTMAX_LAUNCHER
// Launch with programmatic stream serialization (PDL) unless QK_PDL=0, and
// optionally as clusters of `cluster` CTAs (x). The kernels call pdl_entry().
inline bool pdl_enabled() {
  static const bool on = [] {
    const char* v = std::getenv("QK_PDL");
    return !(v && v[0] == '0');
  }();
  return on;
}

// Persistent (one-wave) kernels: trigger the dependent launch after the last
// row instead of at entry, so the next grid's CTAs do not take the slots of
// this grid's early finishers (QK_PDL_LATE=0 restores the entry trigger).
inline int pdl_late_enabled() {
  static const int on = [] {
    const char* v = std::getenv("QK_PDL_LATE");
    return (v && v[0] == '0') ? 0 : 1;
  }();
  return on;
}

template <typename... KArgs, typename... Args>
cudaError_t launch_ex(void (*kern)(KArgs...), dim3 grid, dim3 block, size_t smem,
                      cudaStream_t stream, unsigned cluster, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = stream;
  cudaLaunchAttribute attr[2];
  unsigned na = 0;
  if (cluster > 0) {
    attr[na].id = cudaLaunchAttributeClusterDimension;
    attr[na].val.clusterDim.x = cluster;
    attr[na].val.clusterDim.y = 1;
    attr[na].val.clusterDim.z = 1;
    ++na;
  }
  if (pdl_enabled()) {
    attr[na].id = cudaLaunchAttributeProgrammaticStreamSerialization;
    attr[na].val.programmaticStreamSerializationAllowed = 1;
    ++na;
  }
  cfg.attrs = attr;
  cfg.numAttrs = na;
  return cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

// Record `msg` as this thread's qk_last_error() and return `s` (host_api.cpp).
qk_status set_error(qk_status s, const std::string& msg);

int pipe_resident_probe(int variant, int cluster, int threads, size_t smem);

cudaError_t launch_softmax(SmKernel k, const SmPlan& plan, const float* in, float* out,
                           size_t rows, size_t cols, const SmParams& p, uint32_t* flags,
                           cudaStream_t stream);
// launch_softmax with p.iph / p.oph already set
cudaError_t launch_softmax_phased(SmKernel k, const SmPlan& plan, const float* in, float* out,
                                  size_t rows, size_t cols, const SmParams& p, uint32_t* flags,
                                  cudaStream_t stream);

}  // namespace qk
