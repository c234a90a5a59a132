// C++ host layer of libquake_b200.so: implements include/quake_b200.h.
//
//  * coefficient derivation — bit-identical restatement of the reference's
//    fp64 derivations (kernels.cpp:25-87, nonlin.cpp:35-41, 85-93, 132-141,
//    248-264); compiled with -ffp-contract=off like the reference build;
//  * validation with the reference's preconditions, order and messages;
//  * dispatch to the sm_100a kernels (elementwise.cu, softmax.cu);
//  * the host-span path: per-shard cached workspace (rings of chunk buffers,
//    or the whole shard when it fits), chunked H2D / kernel / D2H pipelines
//    over three streams, and the multi-GPU driver that shards rows (softmax)
//    or 16-byte-aligned element ranges (elementwise) over the configured
//    devices with one host thread per shard and no collectives — the GPU
//    replacement of parallel_chunks (parallel.hpp:43-68).
// Reference paths cited relative to /root/reference/proj/.
#include <cuda_runtime.h>
#include <sched.h>

#include <algorithm>
#include <atomic>
#include <chrono>
#include <barrier>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "../../include/quake_b200.h"
#include "internal.h"

namespace {

// std::numbers::log2e / ln2 / pi as exact binary64 values.
constexpr double kLog2e = 0x1.71547652b82fep+0;
constexpr double kLn2 = 0x1.62e42fefa39efp-1;
constexpr double kPi = 0x1.921fb54442d18p+1;
constexpr double kCenteringBias = 0.0436;  // kernels.hpp:29
constexpr double kScale = 8388608.0;       // 2^23 = ldexp(1, mantissa_bits)
constexpr double kLowExponentEdge = 1.01;  // kernels.cpp:63
constexpr double kHighExponentEdge = 254.99;  // kernels.cpp:64

thread_local std::string g_error;

qk_status fail(qk_status s, const std::string& msg) {
  g_error = msg;
  return s;
}

qk_status cuda_fail(cudaError_t e, const char* where) {
  g_error = std::string(where) + ": " + cudaGetErrorString(e);
  return QK_ERR_CUDA;
}

#define QK_CUDA(call, where)                          \
  do {                                                \
    cudaError_t qk_e_ = (call);                       \
    if (qk_e_ != cudaSuccess) return cuda_fail(qk_e_, where); \
  } while (0)

// ---------------------------------------------------------------------------
// coefficient derivation

qk_affine_coeffs make_coeffs(float p, float q, bool bias, int mantissa_bits = 23,
                             int exp_bias = 127) {
  // kernels.cpp:30-39
  const double scale = std::ldexp(1.0, mantissa_bits);
  const double beta = bias ? kCenteringBias : 0.0;
  qk_affine_coeffs c;
  c.c0 = static_cast<float>(scale * static_cast<double>(p));
  c.c1 = static_cast<float>(scale * (static_cast<double>(exp_bias) + static_cast<double>(q) - beta));
  c.input_scale = p;
  c.input_shift = q;
  c.bias_applied = bias ? 1 : 0;
  return c;
}

qk_clamp_range solve_clamp(double c0, double c1, int mantissa_bits = 23) {
  // kernels.cpp:64-70
  const double scale = std::ldexp(1.0, mantissa_bits);
  double a = (kLowExponentEdge * scale - c1) / c0;
  double b = (kHighExponentEdge * scale - c1) / c0;
  if (a > b) std::swap(a, b);
  return {static_cast<float>(a), static_cast<float>(b)};
}

bool is_continuity(const qk_quad_coeffs& a) {
  // kernels.hpp:73-75
  return a.a0 == 1.0f / 3.0f && a.a1 == 0.0f && a.a2 == 2.0f / 3.0f;
}

bool resolve_bias(qk_kernel k, int32_t requested) {
  // nonlin.hpp:39-41 (the unfused ablation kernels resolve as their QuAKE body)
  return requested < 0 ? (k == QK_QUAKE || k == QK_QUAKE_UNFUSED) : (requested != 0);
}

qk_gelu_constants gelu_defaults() {
  // nonlin.cpp:132-141
  constexpr double kappa = 0.044715;
  const double root2_over_pi = std::sqrt(2.0 / kPi);
  qk_gelu_constants g;
  g.kappa = static_cast<float>(kappa);
  g.root2_over_pi = static_cast<float>(root2_over_pi);
  g.fused_scale = static_cast<float>(2.0 * kappa * root2_over_pi);
  g.inverse_kappa = static_cast<float>(1.0 / kappa);
  return g;
}

// fl(fl(c0*x) + c1) inside int32 range?
bool z_in_range(float c0, float x, float c1) {
  volatile float prod = c0 * x;
  volatile float z = prod + c1;
  return z >= -2147483648.0f && z < 2147483648.0f;
}

// Does saturate(x) in [lo, hi] keep c0*x+c1 inside int32 for every x
// (including NaN -> hi)? If not, the kernel emulates x86 cvttss2si.
bool needs_x86_overflow(const qk_affine_coeffs& c, const qk_clamp_range& r) {
  if (!std::isfinite(c.c0) || !std::isfinite(c.c1) || std::isnan(r.lo) || std::isnan(r.hi)) {
    return true;
  }
  return !(z_in_range(c.c0, r.lo, c.c1) && z_in_range(c.c0, r.hi, c.c1));
}

// ---------------------------------------------------------------------------
// devices and shards

std::mutex g_dev_mu;
std::vector<int> g_devices;  // one entry per shard; empty = current device

std::vector<int> active_devices() {
  std::lock_guard<std::mutex> lk(g_dev_mu);
  if (!g_devices.empty()) return g_devices;
  int d = 0;
  cudaGetDevice(&d);
  return {d};
}

int current_device() {
  int d = 0;
  cudaGetDevice(&d);
  return d;
}

constexpr int kMaxDevices = 64;
std::atomic<int> g_sm_count[kMaxDevices];

int sm_count_of(int dev) {
  int v = dev >= 0 && dev < kMaxDevices ? g_sm_count[dev].load(std::memory_order_acquire) : 0;
  if (v == 0) {
    if (cudaDeviceGetAttribute(&v, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || v <= 0) {
      cudaGetLastError();
      v = 148;
    }
    if (dev >= 0 && dev < kMaxDevices) g_sm_count[dev].store(v, std::memory_order_release);
  }
  return v;
}

// Device workspace of one shard of the host-span path: (device, slot), slot
// = how many earlier shards of the same call sit on that device. Buffers
// grow on demand and are kept (qk_release_workspace frees them).
struct Workspace {
  std::mutex mu;  // held by the calling thread for the whole call
  int dev = 0;
  int slot = 0;
  float* d_in = nullptr;
  size_t in_cap = 0;  // floats
  float* d_out = nullptr;
  size_t out_cap = 0;
  uint32_t* d_flags = nullptr;
  cudaStream_t streams[3] = {nullptr, nullptr, nullptr};
  // overlapped write-back (run_softmax_host): download stream, one event and
  // one mapped pinned flag slot per chunk
  cudaStream_t dl = nullptr;
  uint32_t* h_slots = nullptr;
  size_t slot_cap = 0;
  std::vector<cudaEvent_t> events;
};

std::mutex g_ws_mu;
std::vector<std::unique_ptr<Workspace>> g_ws;  // stable addresses, creation order
std::atomic<size_t> g_ws_limit{0};             // bytes per shard; 0 = automatic

Workspace* workspace_of(int dev, int slot) {
  std::lock_guard<std::mutex> lk(g_ws_mu);
  for (auto& w : g_ws) {
    if (w->dev == dev && w->slot == slot) return w.get();
  }
  g_ws.push_back(std::make_unique<Workspace>());
  g_ws.back()->dev = dev;
  g_ws.back()->slot = slot;
  return g_ws.back().get();
}

// The workspaces of one call's shards, locked in one global order (device,
// then slot) by the calling thread and released when it returns: concurrent
// multi-device calls cannot deadlock, and shard threads never lock.
class ShardLease {
 public:
  explicit ShardLease(const std::vector<int>& devs) {
    ws_.resize(devs.size());
    for (size_t i = 0; i < devs.size(); ++i) {
      int slot = 0;
      for (size_t j = 0; j < i; ++j) slot += devs[j] == devs[i] ? 1 : 0;
      ws_[i] = workspace_of(devs[i], slot);
    }
    std::vector<Workspace*> order = ws_;
    std::sort(order.begin(), order.end(), [](const Workspace* a, const Workspace* b) {
      return a->dev != b->dev ? a->dev < b->dev : a->slot < b->slot;
    });
    for (Workspace* w : order) locks_.emplace_back(w->mu);
  }
  Workspace& operator[](size_t i) { return *ws_[i]; }

 private:
  std::vector<Workspace*> ws_;
  std::vector<std::unique_lock<std::mutex>> locks_;
};

// Caller holds w.mu and has set w.dev current.
qk_status ensure_streams(Workspace& w) {
  if (w.streams[0] == nullptr) {
    for (auto& s : w.streams) QK_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking), "cudaStreamCreate");
    QK_CUDA(cudaMalloc(&w.d_flags, sizeof(uint32_t)), "cudaMalloc(flags)");
  }
  return QK_OK;
}

// Download stream, `n` chunk events and `n` mapped pinned flag slots.
qk_status ensure_chunk_state(Workspace& w, size_t n) {
  if (w.dl == nullptr) QK_CUDA(cudaStreamCreateWithFlags(&w.dl, cudaStreamNonBlocking), "cudaStreamCreate");
  if (n > w.slot_cap) {
    if (w.h_slots) cudaFreeHost(w.h_slots);
    w.h_slots = nullptr;
    w.slot_cap = 0;
    const size_t want = std::max<size_t>(n, 64);
    QK_CUDA(cudaHostAlloc(reinterpret_cast<void**>(&w.h_slots), want * sizeof(uint32_t),
                          cudaHostAllocPortable | cudaHostAllocMapped),
            "cudaHostAlloc(flag slots)");
    w.slot_cap = want;
  }
  while (w.events.size() < n) {
    cudaEvent_t e = nullptr;
    QK_CUDA(cudaEventCreateWithFlags(&e, cudaEventDisableTiming), "cudaEventCreate");
    w.events.push_back(e);
  }
  return QK_OK;
}

qk_status ensure_buf(float*& p, size_t& cap, size_t n, const char* what) {
  if (n <= cap) return QK_OK;
  if (p) cudaFree(p);
  p = nullptr;
  cap = 0;
  const size_t want = std::max<size_t>(n, 1 << 20);
  QK_CUDA(cudaMalloc(&p, want * sizeof(float)), what);
  cap = want;
  return QK_OK;
}

// Device bytes one shard may hold in workspace: the test hook's limit, or
// 90% of what is free plus what this workspace already holds.
size_t workspace_budget(const Workspace& w) {
  const size_t lim = g_ws_limit.load();
  if (lim != 0) return lim;
  size_t fr = 0, tot = 0;
  if (cudaMemGetInfo(&fr, &tot) != cudaSuccess) {
    cudaGetLastError();
    return 0;
  }
  return (fr + (w.in_cap + w.out_cap) * sizeof(float)) / 10 * 9;
}

bool device_pointer(const void* p, int* dev) {
  if (p == nullptr) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  if (a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged) {
    *dev = a.device;
    return true;
  }
  return false;
}

// ---------------------------------------------------------------------------
// elementwise resolution

enum class Family { kQuake, kQuake2, kLogistic, kGelu, kExp };

struct EwSpec {
  qk::EwOp op;
  qk::EwParams p;
};

qk_status resolve_ew(Family f, qk_kernel k, int32_t bias_req, const qk_affine_coeffs* c,
                     const qk_clamp_range* r, const qk_quad_coeffs* a, EwSpec* out) {
  qk::EwParams p{};
  switch (f) {
    case Family::kQuake:
    case Family::kQuake2: {
      p.c0 = c->c0;
      p.c1 = c->c1;
      p.lo = r->lo;
      p.hi = r->hi;
      p.x86_overflow = needs_x86_overflow(*c, *r) ? 1 : 0;
      if (f == Family::kQuake) {
        out->op = qk::EwOp::kQuake;
      } else if (is_continuity(*a)) {
        out->op = qk::EwOp::kQuake2;
      } else {
        out->op = qk::EwOp::kQuake2General;
        p.a0 = a->a0;
        p.a1 = a->a1;
        p.a2 = a->a2;
      }
      break;
    }
    case Family::kExp: {
      if (k == QK_EXACT || k == QK_EXPF) {
        out->op = qk::EwOp::kExpExpf;
      } else if (k == QK_FAST_EXP) {
        out->op = qk::EwOp::kExpFast;
      } else if (k == QK_QUAKE || k == QK_QUAKE2) {
        // quake_cli.cpp:277-289: natural-exp coefficients, per-kernel bias.
        const qk_affine_coeffs ce = make_coeffs(static_cast<float>(kLog2e), 0.0f,
                                                resolve_bias(k, bias_req));
        const qk_clamp_range rc = solve_clamp(ce.c0, ce.c1);
        p.c0 = ce.c0;
        p.c1 = ce.c1;
        p.lo = rc.lo;
        p.hi = rc.hi;
        out->op = k == QK_QUAKE ? qk::EwOp::kQuake : qk::EwOp::kQuake2;
      } else {
        return fail(QK_ERR_BAD_ARGUMENT, "exp_buffer: unknown kernel choice");
      }
      break;
    }
    case Family::kLogistic: {
      if (k == QK_EXACT || k == QK_EXPF) {
        out->op = qk::EwOp::kLogisticExpf;
      } else if (k == QK_FAST_EXP) {
        out->op = qk::EwOp::kLogisticFast;
      } else if (k == QK_QUAKE || k == QK_QUAKE2) {
        // nonlin.cpp:35-41 negated_exp_kernel
        const qk_affine_coeffs ce = make_coeffs(static_cast<float>(-kLog2e), 0.0f,
                                                resolve_bias(k, bias_req));
        const qk_clamp_range rc = solve_clamp(ce.c0, ce.c1);
        p.c0 = ce.c0;
        p.c1 = ce.c1;
        p.lo = rc.lo;
        p.hi = rc.hi;
        out->op = k == QK_QUAKE ? qk::EwOp::kLogisticQuake : qk::EwOp::kLogisticQuake2;
      } else {
        return fail(QK_ERR_BAD_ARGUMENT, "logistic_buffer: unknown kernel choice");
      }
      break;
    }
    case Family::kGelu: {
      const qk_gelu_constants g = gelu_defaults();
      p.k0 = g.inverse_kappa;
      p.k1 = g.kappa;
      p.k2 = g.root2_over_pi;
      if (k == QK_EXACT) {
        out->op = qk::EwOp::kGeluTanh;
      } else if (k == QK_EXPF || k == QK_FAST_EXP) {
        p.c0 = -g.fused_scale;
        out->op = k == QK_EXPF ? qk::EwOp::kGeluExpf : qk::EwOp::kGeluFast;
      } else if (k == QK_QUAKE || k == QK_QUAKE2) {
        // nonlin.cpp:248-264 gelu_exp_kernel
        const qk_affine_coeffs ce =
            make_coeffs(static_cast<float>(-kLog2e * static_cast<double>(g.fused_scale)), 0.0f,
                        resolve_bias(k, bias_req));
        const qk_clamp_range rc = solve_clamp(ce.c0, ce.c1);
        p.c0 = ce.c0;
        p.c1 = ce.c1;
        p.lo = rc.lo;
        p.hi = rc.hi;
        out->op = k == QK_QUAKE ? qk::EwOp::kGeluQuake : qk::EwOp::kGeluQuake2;
      } else if (k == QK_QUAKE_UNFUSED || k == QK_QUAKE2_UNFUSED) {
        // bench.cpp:212-233: explicit fused_scale*x*(ik + x*x) into e^-w
        const qk_affine_coeffs ce = make_coeffs(static_cast<float>(-kLog2e), 0.0f,
                                                resolve_bias(k, bias_req));
        const qk_clamp_range rc = solve_clamp(ce.c0, ce.c1);
        p.c0 = ce.c0;
        p.c1 = ce.c1;
        p.lo = rc.lo;
        p.hi = rc.hi;
        p.k1 = g.fused_scale;
        out->op = k == QK_QUAKE_UNFUSED ? qk::EwOp::kGeluQuakeUnfused
                                        : qk::EwOp::kGeluQuake2Unfused;
      } else {
        return fail(QK_ERR_BAD_ARGUMENT, "gelu_buffer: unknown kernel choice");
      }
      break;
    }
  }
  out->p = p;
  return QK_OK;
}

// ---------------------------------------------------------------------------
// softmax resolution (nonlin.cpp:71-116)

qk_status resolve_sm(const qk_softmax_params* prm, qk_kernel k, qk::SmKernel* sk,
                     qk::SmParams* sp) {
  const float t = prm->temperature;
  qk::SmParams p{};
  p.t = t;
  const double beta = resolve_bias(k, prm->centering_bias) ? kCenteringBias : 0.0;
  p.c0 = static_cast<float>(kScale * static_cast<double>(t) * kLog2e);  // nonlin.cpp:89
  p.c1_base = kScale * (static_cast<double>(127) - beta);               // nonlin.cpp:90-91
  p.vmin_off = 126.0 * kLn2 / static_cast<double>(t);                   // nonlin.cpp:92-93
  switch (k) {
    case QK_EXACT: *sk = qk::SmKernel::kExact; break;
    case QK_EXPF: *sk = qk::SmKernel::kExpf; break;
    case QK_FAST_EXP: *sk = qk::SmKernel::kFast; break;
    case QK_QUAKE: *sk = qk::SmKernel::kQuake; break;
    case QK_QUAKE_UNFUSED:
    case QK_QUAKE2_UNFUSED: {
      // bench.cpp:137-166: natural-exp coefficients and clamp, per-kernel bias
      const qk_affine_coeffs ce = make_coeffs(static_cast<float>(kLog2e), 0.0f,
                                              resolve_bias(k, prm->centering_bias));
      const qk_clamp_range rc = solve_clamp(ce.c0, ce.c1);
      p.nat_c0 = ce.c0;
      p.nat_c1 = ce.c1;
      p.nat_lo = rc.lo;
      p.nat_hi = rc.hi;
      p.unfused = 1;
      *sk = k == QK_QUAKE_UNFUSED ? qk::SmKernel::kQuakeUnfused : qk::SmKernel::kQuake2Unfused;
      break;
    }
    case QK_QUAKE2:
      if (is_continuity(prm->quad)) {
        *sk = qk::SmKernel::kQuake2;
      } else {
        *sk = qk::SmKernel::kQuake2General;
        p.general_quad = 1;
        p.a0 = prm->quad.a0;
        p.a1 = prm->quad.a1;
        p.a2 = prm->quad.a2;
      }
      break;
    default: return fail(QK_ERR_BAD_ARGUMENT, "softmax: unknown kernel choice");
  }
  *sp = p;
  return QK_OK;
}

// ---------------------------------------------------------------------------
// host-span drivers

// Run fn(shard, device, begin, end) for every shard, one host thread per
// shard beyond the first; returns the first failing status.
template <typename Fn>
qk_status for_each_shard(const std::vector<std::pair<size_t, size_t>>& shards,
                         const std::vector<int>& devs, Fn&& fn) {
  const size_t nd = devs.size();
  std::vector<qk_status> st(nd, QK_OK);
  std::vector<std::string> err(nd);
  auto run = [&](size_t i) {
    // fn always runs (dev = -1 when the device cannot be selected) so that
    // shard functions which rendezvous with their siblings never deadlock.
    const int dev = cudaSetDevice(devs[i]) == cudaSuccess ? devs[i] : -1;
    st[i] = fn(i, dev, shards[i].first, shards[i].second);
    err[i] = g_error;
  };
  int prev = current_device();
  std::vector<std::thread> pool;
  for (size_t i = 1; i < nd; ++i) pool.emplace_back(run, i);
  run(0);
  for (auto& t : pool) t.join();
  cudaSetDevice(prev);
  for (size_t i = 0; i < nd; ++i) {
    if (st[i] != QK_OK) {
      g_error = err[i];
      return st[i];
    }
  }
  return QK_OK;
}

// Contiguous shards of n units; boundaries multiples of `align` units.
std::vector<std::pair<size_t, size_t>> make_shards(size_t n, size_t parts, size_t align) {
  std::vector<std::pair<size_t, size_t>> s(parts);
  const size_t units = (n + align - 1) / align;
  size_t begin = 0;
  for (size_t i = 0; i < parts; ++i) {
    const size_t u = units / parts + (i < units % parts ? 1 : 0);
    const size_t end = std::min(n, begin + u * align);
    s[i] = {begin, end};
    begin = end;
  }
  return s;
}

constexpr size_t kChunkElems = size_t{16} << 20;  // 64 MiB per pipeline stage
constexpr int kRing = 3;                          // chunk buffers (= streams) per side

qk_status run_elementwise_host(const EwSpec& spec, const float* xs, float* out, size_t n) {
  if (n == 0) return QK_OK;
  int pdev = 0;
  const bool in_dev = device_pointer(xs, &pdev);
  int odev = 0;
  const bool out_dev = device_pointer(out, &odev);
  if (in_dev && out_dev) {
    // Device spans: one launch on the owning device, synchronous.
    int prev = current_device();
    cudaSetDevice(pdev);
    cudaError_t e = qk::launch_elementwise(spec.op, xs, out, n, spec.p, sm_count_of(pdev), nullptr);
    if (e == cudaSuccess) e = cudaDeviceSynchronize();
    cudaSetDevice(prev);
    if (e != cudaSuccess) return cuda_fail(e, "elementwise kernel");
    return QK_OK;
  }
  std::vector<int> devs = in_dev ? std::vector<int>{pdev} : (out_dev ? std::vector<int>{odev}
                                                                      : active_devices());
  const auto shards = make_shards(n, devs.size(), 4);
  ShardLease lease(devs);
  return for_each_shard(shards, devs, [&](size_t i, int dev, size_t b, size_t e) -> qk_status {
    const size_t len = e - b;
    if (dev < 0) return fail(QK_ERR_NO_DEVICE, "cudaSetDevice failed");
    if (len == 0) return QK_OK;
    Workspace& w = lease[i];
    if (qk_status s = ensure_streams(w)) return s;
    // a ring of kRing chunk buffers per host side: chunk ci uses buffer and
    // stream ci % kRing, so a buffer is reused only after its previous
    // chunk's kernel and copies have retired (stream order)
    const size_t cl_max = std::min(kChunkElems, len);
    const size_t nbuf = std::min<size_t>(kRing, (len + cl_max - 1) / cl_max);
    if (!in_dev) {
      if (qk_status s = ensure_buf(w.d_in, w.in_cap, cl_max * nbuf, "cudaMalloc(workspace in)")) return s;
    }
    if (!out_dev) {
      if (qk_status s = ensure_buf(w.d_out, w.out_cap, cl_max * nbuf, "cudaMalloc(workspace out)")) return s;
    }
    const int sms = sm_count_of(dev);
    size_t ci = 0;
    for (size_t off = 0; off < len; off += cl_max, ++ci) {
      const size_t cl = std::min(cl_max, len - off);
      const size_t slot = ci % nbuf;
      cudaStream_t str = w.streams[ci % kRing];
      const float* src = xs + b + off;
      const float* dsrc = src;
      if (!in_dev) {
        float* buf = w.d_in + slot * cl_max;
        QK_CUDA(cudaMemcpyAsync(buf, src, cl * sizeof(float), cudaMemcpyHostToDevice, str), "H2D");
        dsrc = buf;
      }
      float* ddst = out_dev ? out + b + off : w.d_out + slot * cl_max;
      QK_CUDA(qk::launch_elementwise(spec.op, dsrc, ddst, cl, spec.p, sms, str), "elementwise kernel");
      if (!out_dev) {
        QK_CUDA(cudaMemcpyAsync(out + b + off, ddst, cl * sizeof(float), cudaMemcpyDeviceToHost, str),
                "D2H");
      }
    }
    for (auto& str : w.streams) QK_CUDA(cudaStreamSynchronize(str), "stream sync");
    return QK_OK;
  });
}

qk_status validate_sm(const char* who, size_t n, size_t cols, const qk_softmax_params* prm,
                      size_t out_n, bool single_row) {
  if (single_row) {
    // nonlin.cpp:145-153
    if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, std::string(who) + ": output size mismatch");
    if (!(prm->temperature > 0.0f)) {
      return fail(QK_ERR_BAD_TEMPERATURE, std::string(who) + ": temperature must be positive");
    }
    if (n == 0) return fail(QK_ERR_EMPTY_ROW, "softmax: empty row");
    return QK_OK;
  }
  // nonlin.cpp:165-175
  if (cols == 0 || n % cols != 0) {
    return fail(QK_ERR_NOT_DIVISIBLE, std::string(who) + ": length not divisible by cols");
  }
  if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, std::string(who) + ": output size mismatch");
  if (!(prm->temperature > 0.0f)) {
    return fail(QK_ERR_BAD_TEMPERATURE, std::string(who) + ": temperature must be positive");
  }
  return QK_OK;
}

// ---- overlapped write-back: the host validates the tail of the shard ----
// The contract (every row validated before the first byte reaches `out`,
// nonlin.cpp:176-180) keeps the download behind the validation of the LAST
// row. With the device validating alone that is the end of the upload, and
// the two PCIe directions never overlap. Here host threads test the shard for
// non-finite values from its last element backwards while the device
// validates it from the front (the max pass of each uploaded chunk's softmax
// kernel); when the two fronts meet every row is validated, and the download
// of the computed chunks runs under the upload of the rest. The host threads
// only test exponent bits — every output value still comes from the kernels.
std::atomic<int> g_scan_threads{-1};                       // < 0: automatic; 0: off
std::atomic<size_t> g_scan_min_bytes{size_t{64} << 20};    // per shard

int scan_threads_auto() {
  static const int n = [] {
    const char* v = std::getenv("QK_HOST_SCAN");
    if (v != nullptr && *v != '\0') return std::max(0, std::atoi(v));
    cpu_set_t set;
    CPU_ZERO(&set);
    int c = sched_getaffinity(0, sizeof(set), &set) == 0 ? CPU_COUNT(&set) : 0;
    if (c <= 0) c = static_cast<int>(std::thread::hardware_concurrency());
    return std::clamp(c, 1, 16);
  }();
  return n;
}

bool has_non_finite(const uint32_t* w, size_t n) {
  // exponent all ones <=> (w & 0x7fffffff) >= 0x7f800000 <=> the sum carries into bit 31
  uint32_t acc = 0;
  for (size_t i = 0; i < n; ++i) acc |= (w[i] & 0x7fffffffu) + 0x00800000u;
  return (acc >> 31) != 0;
}

class TailScan {
 public:
  static constexpr size_t kBlock = size_t{256} << 10;  // elements per claim (1 MiB)

  TailScan(const float* x, size_t n, int threads)
      : w_(reinterpret_cast<const uint32_t*>(x)), n_(n), nblocks_((n + kBlock - 1) / kBlock),
        done_(new std::atomic<uint8_t>[nblocks_]) {
    for (size_t k = 0; k < nblocks_; ++k) done_[k].store(0, std::memory_order_relaxed);
    for (int t = 0; t < threads; ++t) pool_.emplace_back([this] { work(); });
  }
  ~TailScan() { finish(); }
  TailScan(const TailScan&) = delete;
  TailScan& operator=(const TailScan&) = delete;

  // Leading elements the device has validated so far (blocks below stop the scan).
  void device_front(size_t elems) { front_.store(elems, std::memory_order_release); }
  bool bad() const { return bad_.load(std::memory_order_acquire); }
  // First element of the suffix the host has finished scanning.
  size_t host_front() {
    while (contig_ < nblocks_ && done_[contig_].load(std::memory_order_acquire)) ++contig_;
    return contig_ * kBlock >= n_ ? 0 : n_ - contig_ * kBlock;
  }
  void finish() {
    stop_.store(true, std::memory_order_release);
    for (auto& t : pool_) t.join();
    pool_.clear();
  }

 private:
  void work() {
    while (!stop_.load(std::memory_order_acquire)) {
      const size_t k = next_.fetch_add(1, std::memory_order_relaxed);  // k-th block from the back
      if (k >= nblocks_) return;
      const size_t end = n_ - k * kBlock;
      const size_t begin = end > kBlock ? end - kBlock : 0;
      // blocks are claimed in descending order and the device front only
      // grows: once one is covered, every later claim is too
      if (end <= front_.load(std::memory_order_acquire)) return;
      if (has_non_finite(w_ + begin, end - begin)) {
        bad_.store(true, std::memory_order_release);
        return;
      }
      done_[k].store(1, std::memory_order_release);
    }
  }

  const uint32_t* w_;
  size_t n_, nblocks_;
  std::unique_ptr<std::atomic<uint8_t>[]> done_;
  std::atomic<size_t> next_{0}, front_{0};
  std::atomic<bool> stop_{false}, bad_{false};
  std::vector<std::thread> pool_;
  size_t contig_ = 0;  // polling thread only
};

bool pinned_host(const void* p) {
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeHost;
}

// softmax_rows over host or device spans (nonlin.cpp:162-189). The contract:
// every row is validated before anything reaches `out` (nonlin.cpp:176-180),
// across all shards. Per shard, one of two schedules:
//  * resident — the shard's host-side spans fit the workspace budget: phase 1
//    uploads the shard and runs the softmax into the device workspace (host
//    `out`; the kernel's max pass raises the non-finite flag) or a
//    validation pass (device `out`); after every shard reports clean, phase 2
//    downloads the workspace, or runs the softmax straight into device `out`;
//  * streamed — larger inputs: phase 1 streams the shard through a ring of
//    chunk buffers with the validation pass only; phase 2 streams it again
//    through H2D -> softmax -> D2H. Twice the upload, any size.
// Device input and device output need no workspace at all.
qk_status run_softmax_host(const float* m, size_t n, size_t cols, const qk_softmax_params* prm,
                           qk_kernel k, float* out) {
  qk::SmKernel sk;
  qk::SmParams sp;
  qk_status s = resolve_sm(prm, k, &sk, &sp);
  if (s != QK_OK) return s;
  const size_t rows = n / cols;
  if (rows == 0) return QK_OK;
  int pdev = 0, odev = 0;
  const bool in_dev = device_pointer(m, &pdev);
  const bool out_dev = device_pointer(out, &odev);
  std::vector<int> devs = in_dev ? std::vector<int>{pdev} : (out_dev ? std::vector<int>{odev}
                                                                      : active_devices());
  const auto shards = make_shards(rows, devs.size(), 1);
  std::atomic<bool> non_finite{false};
  std::atomic<bool> abort_all{false};
  std::barrier sync_point(static_cast<std::ptrdiff_t>(devs.size()));
  const size_t chunk_rows = std::max<size_t>(1, kChunkElems / cols);
  ShardLease lease(devs);

  s = for_each_shard(shards, devs, [&](size_t i, int dev, size_t rb, size_t re) -> qk_status {
    if (dev < 0) {
      abort_all.store(true);
      sync_point.arrive_and_wait();
      return fail(QK_ERR_NO_DEVICE, "cudaSetDevice failed");
    }
    Workspace& w = lease[i];
    const size_t nrows = re - rb;
    const qk::SmPlan plan = qk::plan_softmax(cols, dev, sk);
    const size_t shard_elems = nrows * cols;
    const size_t host_sides = (in_dev ? 0 : 1) + (out_dev ? 0 : 1);
    qk_status ss = ensure_streams(w);
    const bool resident =
        ss == QK_OK && host_sides * shard_elems * sizeof(float) <= workspace_budget(w);
    const size_t ring_rows = std::min(chunk_rows, std::max<size_t>(nrows, 1));
    const size_t nbuf = std::min<size_t>(kRing, (nrows + ring_rows - 1) / std::max<size_t>(ring_rows, 1));
    const size_t cap = resident ? shard_elems : ring_rows * cols * std::max<size_t>(nbuf, 1);
    if (ss == QK_OK && !in_dev) ss = ensure_buf(w.d_in, w.in_cap, cap, "cudaMalloc(workspace in)");
    if (ss == QK_OK && !out_dev && resident) ss = ensure_buf(w.d_out, w.out_cap, cap, "cudaMalloc(workspace out)");
    if (ss == QK_OK && !out_dev && !resident) ss = ensure_buf(w.d_out, w.out_cap, cap, "cudaMalloc(workspace out)");
    if (ss == QK_OK && cudaMemsetAsync(w.d_flags, 0, sizeof(uint32_t), w.streams[0]) != cudaSuccess) {
      ss = fail(QK_ERR_CUDA, "cudaMemset(flags)");
    }
    if (ss == QK_OK) cudaStreamSynchronize(w.streams[0]);
    // where chunk ci (rows r0..) of the input lives on the device, uploading
    // it first when the input is host memory
    auto stage_in = [&](size_t ci, size_t r0, size_t cr, cudaStream_t str, const float** dsrc) -> qk_status {
      if (in_dev) {
        *dsrc = m + (rb + r0) * cols;
        return QK_OK;
      }
      float* buf = resident ? w.d_in + r0 * cols : w.d_in + (ci % nbuf) * ring_rows * cols;
      if (cudaMemcpyAsync(buf, m + (rb + r0) * cols, cr * cols * sizeof(float),
                          cudaMemcpyHostToDevice, str) != cudaSuccess) {
        return fail(QK_ERR_CUDA, "H2D");
      }
      *dsrc = buf;
      return QK_OK;
    };
    // Phase 1: upload + (softmax into the workspace | validation pass).
    const bool compute_now = resident && !out_dev;
    const size_t nchunks = (nrows + chunk_rows - 1) / chunk_rows;
    // overlapped write-back (see TailScan): pinned host spans on both sides
    // (pageable copies are staged synchronously: nothing to overlap)
    int scan_threads = g_scan_threads.load();
    if (scan_threads < 0) scan_threads = scan_threads_auto();
    scan_threads = scan_threads > 0 ? std::max<int>(1, scan_threads / static_cast<int>(devs.size())) : 0;
    const bool overlap = ss == QK_OK && compute_now && scan_threads > 0 && nchunks >= 2 &&
                         shard_elems * sizeof(float) >= g_scan_min_bytes.load() && pinned_host(m) &&
                         pinned_host(out);
    if (overlap) ss = ensure_chunk_state(w, nchunks);
    std::unique_ptr<TailScan> scan;
    if (overlap && ss == QK_OK) {
      std::memset(w.h_slots, 0, nchunks * sizeof(uint32_t));
      scan = std::make_unique<TailScan>(m + rb * cols, shard_elems, scan_threads);
    }
    size_t ci = 0;
    for (size_t r0 = 0; ss == QK_OK && r0 < nrows; r0 += chunk_rows, ++ci) {
      const size_t cr = std::min(chunk_rows, nrows - r0);
      cudaStream_t str = w.streams[ci % kRing];
      const float* dsrc = nullptr;
      ss = stage_in(ci, r0, cr, str, &dsrc);
      if (ss != QK_OK) break;
      cudaError_t e = compute_now ? qk::launch_softmax(sk, plan, dsrc, w.d_out + r0 * cols, cr, cols,
                                                       sp, w.d_flags, str)
                                  : qk::launch_check_finite(dsrc, cr * cols, w.d_flags, str);
      if (e != cudaSuccess) ss = cuda_fail(e, compute_now ? "softmax kernel" : "validation kernel");
      if (scan && ss == QK_OK) {
        // the chunk's verdict goes to its host slot; its event gates its download
        e = qk::launch_publish_flag(w.d_flags, w.h_slots + ci, str);
        if (e == cudaSuccess) e = cudaEventRecord(w.events[ci], str);
        if (e != cudaSuccess) ss = cuda_fail(e, "publish flag");
      }
    }
    uint32_t flags = 0;
    if (scan && ss == QK_OK) {
      // wait until the device front (chunks validated, in order) reaches the
      // host front (suffix scanned), or either side finds a non-finite value
      volatile const uint32_t* slots = w.h_slots;
      size_t gchunks = 0;
      for (;;) {
        while (gchunks < nchunks && (slots[gchunks] & qk::kFlagPublished)) {
          flags |= slots[gchunks] & 1u;
          ++gchunks;
        }
        const size_t front = std::min(gchunks * chunk_rows, nrows) * cols;
        scan->device_front(front);
        if ((flags & 1u) || scan->bad() || front >= scan->host_front()) break;
        if (gchunks < nchunks) {
          const cudaError_t q = cudaEventQuery(w.events[gchunks]);
          if (q == cudaSuccess && !(slots[gchunks] & qk::kFlagPublished)) {
            // the chunk's stream has passed its event but the slot never arrived
            ss = fail(QK_ERR_CUDA, "softmax: flag slot not published");
            break;
          }
          if (q != cudaSuccess && q != cudaErrorNotReady) {
            ss = cuda_fail(q, "softmax chunk");
            break;
          }
          cudaGetLastError();  // cudaErrorNotReady from the query
        }
        std::this_thread::sleep_for(std::chrono::microseconds(20));
      }
      scan->finish();
      if (scan->bad()) flags |= 1u;
      if (flags & 1u) {
        // out stays untouched; let the queued uploads and kernels drain
        for (auto& str : w.streams) cudaStreamSynchronize(str);
      }
    } else {
      for (auto& str : w.streams) {
        if (str && cudaStreamSynchronize(str) != cudaSuccess && ss == QK_OK) ss = fail(QK_ERR_CUDA, "stream sync");
      }
      if (ss == QK_OK && cudaMemcpy(&flags, w.d_flags, sizeof(uint32_t), cudaMemcpyDeviceToHost) !=
                             cudaSuccess) {
        ss = fail(QK_ERR_CUDA, "D2H(flags)");
      }
    }
    if (flags & 1u) non_finite.store(true);
    if (ss != QK_OK) abort_all.store(true);  // no shard writes back
    // Every shard validated before anything reaches `out` (nonlin.cpp:176-180).
    sync_point.arrive_and_wait();
    if (ss != QK_OK) return ss;
    if (non_finite.load()) return fail(QK_ERR_NON_FINITE, "softmax: non-finite input");
    if (abort_all.load()) return fail(QK_ERR_CUDA, "softmax: aborted (another device failed)");
    // Phase 2: write back (download the workspace | softmax into out | stream).
    ci = 0;
    for (size_t r0 = 0; r0 < nrows; r0 += chunk_rows, ++ci) {
      const size_t cr = std::min(chunk_rows, nrows - r0);
      cudaStream_t str = w.streams[ci % kRing];
      float* hdst = out + (rb + r0) * cols;
      if (compute_now) {
        if (scan) {
          // on the download stream, behind the chunk's own kernel only: the
          // upload streams still carry the rest of the shard
          str = w.dl;
          QK_CUDA(cudaStreamWaitEvent(str, w.events[ci], 0), "cudaStreamWaitEvent");
        }
        QK_CUDA(cudaMemcpyAsync(hdst, w.d_out + r0 * cols, cr * cols * sizeof(float),
                                cudaMemcpyDeviceToHost, str),
                "D2H");
        continue;
      }
      const float* dsrc = nullptr;
      if (resident) {
        dsrc = in_dev ? m + (rb + r0) * cols : w.d_in + r0 * cols;  // uploaded in phase 1
      } else if (qk_status st2 = stage_in(ci, r0, cr, str, &dsrc)) {
        return st2;
      }
      float* ddst = out_dev ? hdst : w.d_out + (ci % nbuf) * ring_rows * cols;
      QK_CUDA(qk::launch_softmax(sk, plan, dsrc, ddst, cr, cols, sp, nullptr, str), "softmax kernel");
      if (!out_dev) {
        QK_CUDA(cudaMemcpyAsync(hdst, ddst, cr * cols * sizeof(float), cudaMemcpyDeviceToHost, str),
                "D2H");
      }
    }
    for (auto& str : w.streams) QK_CUDA(cudaStreamSynchronize(str), "stream sync");
    if (scan) QK_CUDA(cudaStreamSynchronize(w.dl), "stream sync");
    return QK_OK;
  });
  if (non_finite.load() && (s == QK_OK || s == QK_ERR_NON_FINITE)) {
    return fail(QK_ERR_NON_FINITE, "softmax: non-finite input");
  }
  return s;
}

}  // namespace

namespace qk {
qk_status set_error(qk_status s, const std::string& msg) { return fail(s, msg); }
}  // namespace qk

// ===========================================================================
extern "C" {

int qk_abi_version(void) { return QK_ABI_VERSION; }
const char* qk_last_error(void) { return g_error.c_str(); }
int qk_is_invalid_argument(qk_status s) { return s >= 1 && s < 100 ? 1 : 0; }

qk_status qk_device_count(int* count) {
  if (!count) return fail(QK_ERR_BAD_ARGUMENT, "device_count: null pointer");
  const cudaError_t e = cudaGetDeviceCount(count);
  if (e != cudaSuccess) {
    *count = 0;
    return cuda_fail(e, "cudaGetDeviceCount");
  }
  return QK_OK;
}

namespace {
qk_status set_device_list(const int* devices, int n, bool allow_repeat, const char* who) {
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess) count = 0;
  if (n > 0 && devices == nullptr) return fail(QK_ERR_BAD_ARGUMENT, std::string(who) + ": null pointer");
  std::vector<int> v;
  for (int i = 0; i < n; ++i) {
    if (devices[i] < 0 || devices[i] >= count || devices[i] >= kMaxDevices) {
      return fail(QK_ERR_NO_DEVICE, std::string(who) + ": no such device");
    }
    if (!allow_repeat && std::find(v.begin(), v.end(), devices[i]) != v.end()) {
      return fail(QK_ERR_BAD_ARGUMENT, std::string(who) + ": duplicate device");
    }
    v.push_back(devices[i]);
  }
  std::lock_guard<std::mutex> lk(g_dev_mu);
  g_devices = v;
  return QK_OK;
}
}  // namespace

qk_status qk_set_devices(const int* devices, int n) {
  return set_device_list(devices, n, false, "set_devices");
}

qk_status qk_set_device_shards(const int* devices, int n) {
  return set_device_list(devices, n, true, "set_device_shards");
}

int qk_get_devices(int* devices, int cap) {
  const std::vector<int> v = active_devices();
  for (int i = 0; i < cap && i < static_cast<int>(v.size()); ++i) devices[i] = v[i];
  return static_cast<int>(v.size());
}

void qk_set_workspace_limit(size_t bytes) { g_ws_limit.store(bytes); }

void qk_set_host_validation(int32_t threads, size_t min_bytes) {
  g_scan_threads.store(threads);
  g_scan_min_bytes.store(min_bytes);
}

qk_status qk_set_plan_override(const char* name, int32_t value, int32_t clear) {
  if (!qk::set_plan_opt(name, value, clear != 0)) {
    return fail(QK_ERR_BAD_ARGUMENT, std::string("set_plan_override: unknown option ") +
                                         (name ? name : "(null)"));
  }
  return QK_OK;
}

void qk_release_workspace(void) {
  int prev = current_device();
  std::lock_guard<std::mutex> g(g_ws_mu);
  for (auto& wp : g_ws) {
    Workspace& w = *wp;
    std::lock_guard<std::mutex> lk(w.mu);
    if (w.streams[0] == nullptr && w.d_in == nullptr && w.d_out == nullptr && w.dl == nullptr) continue;
    cudaSetDevice(w.dev);
    if (w.d_in) cudaFree(w.d_in);
    if (w.d_out) cudaFree(w.d_out);
    if (w.d_flags) cudaFree(w.d_flags);
    for (auto& st : w.streams) {
      if (st) cudaStreamDestroy(st);
      st = nullptr;
    }
    if (w.dl) cudaStreamDestroy(w.dl);
    if (w.h_slots) cudaFreeHost(w.h_slots);
    for (cudaEvent_t e : w.events) cudaEventDestroy(e);
    w.events.clear();
    w.dl = nullptr;
    w.h_slots = nullptr;
    w.slot_cap = 0;
    w.d_in = w.d_out = nullptr;
    w.d_flags = nullptr;
    w.in_cap = w.out_cap = 0;
  }
  cudaSetDevice(prev);
}

// ---- coefficients ----
qk_status qk_coeffs_for(float p, float q, int32_t bias, qk_affine_coeffs* out) {
  if (!out) return fail(QK_ERR_BAD_ARGUMENT, "coeffs_for: null pointer");
  if (p == 0.0f) return fail(QK_ERR_ZERO_SLOPE, "coeffs_for: input scale p must be non-zero");
  *out = make_coeffs(p, q, bias != 0);
  return QK_OK;
}
qk_affine_coeffs qk_natural_exp_coeffs(int32_t bias) {
  return make_coeffs(static_cast<float>(kLog2e), 0.0f, bias != 0);  // kernels.cpp:42-45
}
qk_affine_coeffs qk_base2_coeffs(int32_t bias) { return make_coeffs(1.0f, 0.0f, bias != 0); }
qk_affine_coeffs qk_negated_natural_exp_coeffs(int32_t bias) {
  return make_coeffs(static_cast<float>(-kLog2e), 0.0f, bias != 0);  // kernels.cpp:51-54
}
qk_status qk_default_clamp(float p, float q, qk_clamp_range* out) {
  if (!out) return fail(QK_ERR_BAD_ARGUMENT, "default_clamp: null pointer");
  if (p == 0.0f) return fail(QK_ERR_ZERO_SLOPE, "default_clamp: input scale p must be non-zero");
  // kernels.cpp:74-82
  *out = solve_clamp(kScale * static_cast<double>(p),
                     kScale * (static_cast<double>(127) + static_cast<double>(q)));
  return QK_OK;
}
qk_status qk_coeffs_for_format(float p, float q, const qk_fp_format* fmt, int32_t bias,
                               qk_affine_coeffs* out) {
  if (!out) return fail(QK_ERR_BAD_ARGUMENT, "coeffs_for: null pointer");
  if (p == 0.0f) return fail(QK_ERR_ZERO_SLOPE, "coeffs_for: input scale p must be non-zero");
  *out = fmt ? make_coeffs(p, q, bias != 0, fmt->mantissa_bits, fmt->bias)
             : make_coeffs(p, q, bias != 0);
  return QK_OK;
}
qk_status qk_default_clamp_format(float p, float q, const qk_fp_format* fmt, qk_clamp_range* out) {
  if (!out) return fail(QK_ERR_BAD_ARGUMENT, "default_clamp: null pointer");
  if (p == 0.0f) return fail(QK_ERR_ZERO_SLOPE, "default_clamp: input scale p must be non-zero");
  // kernels.cpp:74-82
  const int mb = fmt ? fmt->mantissa_bits : 23;
  const int eb = fmt ? fmt->bias : 127;
  const double scale = std::ldexp(1.0, mb);
  *out = solve_clamp(scale * static_cast<double>(p),
                     scale * (static_cast<double>(eb) + static_cast<double>(q)), mb);
  return QK_OK;
}
qk_clamp_range qk_clamp_for(const qk_affine_coeffs* c) {
  return solve_clamp(static_cast<double>(c->c0), static_cast<double>(c->c1));
}
qk_quad_coeffs qk_quad_continuity(void) { return {1.0f / 3.0f, 0.0f, 2.0f / 3.0f}; }
qk_quad_coeffs qk_quad_minimax(void) { return {0.33f, -0.017f, 0.68f}; }
int qk_quad_is_continuity_default(const qk_quad_coeffs* a) { return is_continuity(*a) ? 1 : 0; }
qk_gelu_constants qk_gelu_constants_defaults(void) { return gelu_defaults(); }
int32_t qk_resolve_centering_bias(qk_kernel k, int32_t requested) {
  return resolve_bias(k, requested) ? 1 : 0;
}
const char* qk_kernel_name(qk_kernel k) {
  switch (k) {  // nonlin.cpp:120-130
    case QK_EXACT: return "exact";
    case QK_QUAKE: return "quake";
    case QK_QUAKE2: return "quake2";
    case QK_EXPF: return "expf";
    case QK_FAST_EXP: return "fast_expf";
    case QK_QUAKE_UNFUSED: return "quake_unfused";
    case QK_QUAKE2_UNFUSED: return "quake2_unfused";
  }
  return "unknown";
}
qk_status qk_softmax_plan(size_t cols, int32_t /*aligned16: ignored since ABI 3*/, qk_kernel kernel,
                          qk_softmax_plan_info* out) {
  if (!out) return fail(QK_ERR_BAD_ARGUMENT, "softmax_plan: null pointer");
  qk::SmKernel sk;
  qk::SmParams sp;
  qk_softmax_params prm{1.0f, -1, {1.0f / 3.0f, 0.0f, 2.0f / 3.0f}};
  if (qk_status s = resolve_sm(&prm, kernel, &sk, &sp)) return s;
  const qk::SmPlan p = qk::plan_softmax(cols, current_device(), sk);
  out->variant = static_cast<int32_t>(p.variant);
  out->width = p.width;
  out->lanes = p.lanes;
  out->cluster = p.cluster;
  out->slice = p.slice;
  out->threads = p.threads;
  out->vpt = p.vpt;
  out->smem = static_cast<int64_t>(p.smem);
  out->stages = p.stages;
  out->balanced = p.balanced;
  out->resident = p.resident;
  return QK_OK;
}

// ---- host-span operators ----
qk_status qk_quake_buffer(const float* xs, size_t n, float* out, size_t out_n,
                          const qk_affine_coeffs* c, const qk_clamp_range* r) {
  if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, "quake_buffer: output size mismatch");
  if (!c || !r || (n && (!xs || !out))) return fail(QK_ERR_BAD_ARGUMENT, "quake_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kQuake, QK_QUAKE, -1, c, r, nullptr, &spec);
  return s != QK_OK ? s : run_elementwise_host(spec, xs, out, n);
}

qk_status qk_quake2_buffer(const float* xs, size_t n, float* out, size_t out_n,
                           const qk_affine_coeffs* c, const qk_quad_coeffs* a,
                           const qk_clamp_range* r) {
  if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, "quake2_buffer: output size mismatch");
  if (!c || !r || !a || (n && (!xs || !out))) {
    return fail(QK_ERR_BAD_ARGUMENT, "quake2_buffer: null pointer");
  }
  EwSpec spec;
  qk_status s = resolve_ew(Family::kQuake2, QK_QUAKE2, -1, c, r, a, &spec);
  return s != QK_OK ? s : run_elementwise_host(spec, xs, out, n);
}

qk_status qk_logistic_buffer(const float* xs, size_t n, float* out, size_t out_n, qk_kernel k,
                             int32_t bias) {
  if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, "logistic_buffer: output size mismatch");
  if (n && (!xs || !out)) return fail(QK_ERR_BAD_ARGUMENT, "logistic_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kLogistic, k, bias, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : run_elementwise_host(spec, xs, out, n);
}

qk_status qk_gelu_buffer(const float* xs, size_t n, float* out, size_t out_n, qk_kernel k,
                         int32_t bias) {
  if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, "gelu_buffer: output size mismatch");
  if (n && (!xs || !out)) return fail(QK_ERR_BAD_ARGUMENT, "gelu_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kGelu, k, bias, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : run_elementwise_host(spec, xs, out, n);
}

qk_status qk_exp_buffer(const float* xs, size_t n, float* out, size_t out_n, qk_kernel k) {
  if (out_n != n) return fail(QK_ERR_SIZE_MISMATCH, "exp_buffer: output size mismatch");
  if (n && (!xs || !out)) return fail(QK_ERR_BAD_ARGUMENT, "exp_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kExp, k, -1, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : run_elementwise_host(spec, xs, out, n);
}

qk_status qk_softmax_rows(const float* matrix, size_t n, size_t cols,
                          const qk_softmax_params* prm, qk_kernel k, float* out, size_t out_n) {
  if (!prm) return fail(QK_ERR_BAD_ARGUMENT, "softmax_rows: null params");
  qk_status s = validate_sm("softmax_rows", n, cols, prm, out_n, false);
  if (s != QK_OK) return s;
  if (n && (!matrix || !out)) return fail(QK_ERR_BAD_ARGUMENT, "softmax_rows: null pointer");
  return run_softmax_host(matrix, n, cols, prm, k, out);
}

qk_status qk_softmax_row(const float* v, size_t n, const qk_softmax_params* prm, qk_kernel k,
                         float* out, size_t out_n) {
  if (!prm) return fail(QK_ERR_BAD_ARGUMENT, "softmax_row: null params");
  qk_status s = validate_sm("softmax_row", n, n, prm, out_n, true);
  if (s != QK_OK) return s;
  if (!v || !out) return fail(QK_ERR_BAD_ARGUMENT, "softmax_row: null pointer");
  return run_softmax_host(v, n, n, prm, k, out);
}

// ---- scalar forms ----
namespace {
// Per-thread pinned mailbox {x, y} (mapped: the kernel reads x and writes y
// in host memory) and a stream, on the first configured device.
struct ScalarBox {
  int dev = -1;
  float* h = nullptr;
  cudaStream_t s = nullptr;
  ~ScalarBox() {
    if (h) cudaFreeHost(h);
    if (s) cudaStreamDestroy(s);
  }
};
thread_local ScalarBox t_box;

qk_status run_scalar(const EwSpec& spec, float x, float* y) {
  if (!y) return fail(QK_ERR_BAD_ARGUMENT, "scalar form: null output pointer");
  const int dev = active_devices()[0];
  const int prev = current_device();
  if (dev != prev) QK_CUDA(cudaSetDevice(dev), "cudaSetDevice");
  struct Restore {
    int prev, dev;
    ~Restore() {
      if (prev != dev) cudaSetDevice(prev);
    }
  } restore{prev, dev};
  if (t_box.dev != dev) {
    if (t_box.h) cudaFreeHost(t_box.h);
    if (t_box.s) cudaStreamDestroy(t_box.s);
    t_box.h = nullptr;
    t_box.s = nullptr;
    t_box.dev = -1;
    QK_CUDA(cudaHostAlloc(&t_box.h, 8 * sizeof(float), cudaHostAllocMapped | cudaHostAllocPortable),
            "cudaHostAlloc(scalar)");
    QK_CUDA(cudaStreamCreateWithFlags(&t_box.s, cudaStreamNonBlocking), "cudaStreamCreate");
    t_box.dev = dev;
  }
  float* d = nullptr;
  QK_CUDA(cudaHostGetDevicePointer(reinterpret_cast<void**>(&d), t_box.h, 0),
          "cudaHostGetDevicePointer");
  volatile float* h = t_box.h;
  h[0] = x;
  // x and y 16 bytes apart: both float4-aligned, one element each
  QK_CUDA(qk::launch_elementwise(spec.op, d, d + 4, 1, spec.p, sm_count_of(dev), t_box.s),
          "elementwise kernel");
  QK_CUDA(cudaStreamSynchronize(t_box.s), "stream sync");
  *y = h[4];
  return QK_OK;
}
}  // namespace

qk_status qk_quake(float x, const qk_affine_coeffs* c, const qk_clamp_range* r, float* y) {
  if (!c || !r) return fail(QK_ERR_BAD_ARGUMENT, "quake: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kQuake, QK_QUAKE, -1, c, r, nullptr, &spec);
  return s != QK_OK ? s : run_scalar(spec, x, y);
}
qk_status qk_quake2(float x, const qk_affine_coeffs* c, const qk_quad_coeffs* a,
                    const qk_clamp_range* r, float* y) {
  if (!c || !r || !a) return fail(QK_ERR_BAD_ARGUMENT, "quake2: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kQuake2, QK_QUAKE2, -1, c, r, a, &spec);
  return s != QK_OK ? s : run_scalar(spec, x, y);
}
qk_status qk_logistic(float x, qk_kernel k, int32_t bias, float* y) {
  EwSpec spec;
  qk_status s = resolve_ew(Family::kLogistic, k, bias, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : run_scalar(spec, x, y);
}
qk_status qk_gelu(float x, qk_kernel k, int32_t bias, float* y) {
  EwSpec spec;
  qk_status s = resolve_ew(Family::kGelu, k, bias, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : run_scalar(spec, x, y);
}

// ---- device operators ----
// The library links cudart statically, so its current device is not the
// caller's runtime's (e.g. torch's): launch on the device that owns the
// stream (the legacy stream: the device holding the data), restoring the
// previous device afterwards.
class LaunchDevice {
 public:
  LaunchDevice(qk_stream stream, const void* data) {
    cudaGetDevice(&prev_);
    int dev = prev_;
    if (stream != nullptr) {
      const cudaStream_t s = reinterpret_cast<cudaStream_t>(stream);
      cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
      if (cudaStreamIsCapturing(s, &cs) == cudaSuccess && cs != cudaStreamCaptureStatusNone) {
        // cudaStreamGetDevice invalidates a stream capture (CUDA graphs):
        // while capturing, take the device that holds the data
        if (!device_pointer(data, &dev)) dev = prev_;
      } else if (cudaStreamGetDevice(s, &dev) != cudaSuccess) {
        cudaGetLastError();
        dev = prev_;
      }
    } else if (!device_pointer(data, &dev)) {
      dev = prev_;
    }
    if (dev != prev_ && cudaSetDevice(dev) == cudaSuccess) switched_ = true;
  }
  ~LaunchDevice() {
    if (switched_) cudaSetDevice(prev_);
  }

 private:
  int prev_ = 0;
  bool switched_ = false;
};

static qk_status launch_ew_device(const EwSpec& spec, const float* xs, float* out, size_t n,
                                  qk_stream stream) {
  LaunchDevice on(stream, xs);
  const cudaError_t e = qk::launch_elementwise(spec.op, xs, out, n, spec.p,
                                               sm_count_of(current_device()),
                                               reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? QK_OK : cuda_fail(e, "elementwise kernel launch");
}

qk_status qk_quake_buffer_device(const float* xs, float* out, size_t n, const qk_affine_coeffs* c,
                                 const qk_clamp_range* r, qk_stream stream) {
  if (!c || !r || (n && (!xs || !out))) return fail(QK_ERR_BAD_ARGUMENT, "quake_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kQuake, QK_QUAKE, -1, c, r, nullptr, &spec);
  return s != QK_OK ? s : launch_ew_device(spec, xs, out, n, stream);
}

qk_status qk_quake2_buffer_device(const float* xs, float* out, size_t n, const qk_affine_coeffs* c,
                                  const qk_quad_coeffs* a, const qk_clamp_range* r,
                                  qk_stream stream) {
  if (!c || !r || !a || (n && (!xs || !out))) {
    return fail(QK_ERR_BAD_ARGUMENT, "quake2_buffer: null pointer");
  }
  EwSpec spec;
  qk_status s = resolve_ew(Family::kQuake2, QK_QUAKE2, -1, c, r, a, &spec);
  return s != QK_OK ? s : launch_ew_device(spec, xs, out, n, stream);
}

qk_status qk_logistic_buffer_device(const float* xs, float* out, size_t n, qk_kernel k,
                                    int32_t bias, qk_stream stream) {
  if (n && (!xs || !out)) return fail(QK_ERR_BAD_ARGUMENT, "logistic_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kLogistic, k, bias, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : launch_ew_device(spec, xs, out, n, stream);
}

qk_status qk_gelu_buffer_device(const float* xs, float* out, size_t n, qk_kernel k, int32_t bias,
                                qk_stream stream) {
  if (n && (!xs || !out)) return fail(QK_ERR_BAD_ARGUMENT, "gelu_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kGelu, k, bias, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : launch_ew_device(spec, xs, out, n, stream);
}

qk_status qk_exp_buffer_device(const float* xs, float* out, size_t n, qk_kernel k,
                               qk_stream stream) {
  if (n && (!xs || !out)) return fail(QK_ERR_BAD_ARGUMENT, "exp_buffer: null pointer");
  EwSpec spec;
  qk_status s = resolve_ew(Family::kExp, k, -1, nullptr, nullptr, nullptr, &spec);
  return s != QK_OK ? s : launch_ew_device(spec, xs, out, n, stream);
}

qk_status qk_softmax_rows_device(const float* matrix, size_t n, size_t cols,
                                 const qk_softmax_params* prm, qk_kernel k, float* out,
                                 uint32_t* d_flags, qk_stream stream) {
  if (!prm) return fail(QK_ERR_BAD_ARGUMENT, "softmax_rows: null params");
  qk_status s = validate_sm("softmax_rows", n, cols, prm, n, false);
  if (s != QK_OK) return s;
  if (n && (!matrix || !out)) return fail(QK_ERR_BAD_ARGUMENT, "softmax_rows: null pointer");
  qk::SmKernel sk;
  qk::SmParams sp;
  s = resolve_sm(prm, k, &sk, &sp);
  if (s != QK_OK) return s;
  const size_t rows = n / cols;
  LaunchDevice on(stream, matrix);
  if ((reinterpret_cast<uintptr_t>(matrix) | reinterpret_cast<uintptr_t>(out)) & 3u) {
    return fail(QK_ERR_BAD_ARGUMENT, "softmax_rows: pointer not aligned to a float");
  }
  const qk::SmPlan plan = qk::plan_softmax(cols, current_device(), sk);
  const cudaError_t e = qk::launch_softmax(sk, plan, matrix, out, rows, cols, sp, d_flags,
                                           reinterpret_cast<cudaStream_t>(stream));
  return e == cudaSuccess ? QK_OK : cuda_fail(e, "softmax kernel launch");
}

}  // extern "C"
