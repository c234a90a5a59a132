"""TEST INFRASTRUCTURE ONLY — numpy/ctypes front end of the CPU oracle.

Two back ends, same call surface:

* ``Restatement`` — ``oracle/liboracle.so``, the plain-C restatement
  (``quake_oracle.c``), built from this repo by ``oracle/Makefile``.
* ``Reference`` — ``oracle/_ref/libquake_ref.so``, the reference's own
  ``core/src/{kernels,nonlin,parallel,oracle}.cpp`` compiled in place from
  ``/root/reference`` (only where that tree exists; the built ``.so`` then
  travels to the GPU box with the repo snapshot).

Only tests/, ``__graft_entry__.smoke()`` and bench.py's CPU legs may import
this module. The product package never does.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import POINTER, c_double, c_float, c_int, c_size_t, c_uint, c_uint64, c_void_p

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
RESTATEMENT_SO = os.path.join(HERE, "liboracle.so")
REFERENCE_SO = os.path.join(HERE, "_ref", "libquake_ref.so")

EXACT, QUAKE, QUAKE2 = 0, 1, 2
# unfused ablation variants of the bench passes (bench.cpp:137-166, 212-233)
QUAKE_UNFUSED, QUAKE2_UNFUSED = 5, 6
CONTINUITY = (np.float32(1.0) / np.float32(3.0), np.float32(0.0), np.float32(2.0) / np.float32(3.0))
MINIMAX = (np.float32(0.33), np.float32(-0.017), np.float32(0.68))

_fp = POINTER(c_float)
_dp = POINTER(c_double)


def _f32(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32)


def _ptr(a: np.ndarray, t=_fp):
    return a.ctypes.data_as(t)


class OracleError(ValueError):
    """Raised for the reference's std::invalid_argument cases."""


class Restatement:
    """The plain-C restatement (quake_oracle.c)."""

    kind = "port"

    def __init__(self, path: str = RESTATEMENT_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: run `make -C oracle`")
        L = self.lib = ctypes.CDLL(path)
        L.or_coeffs_for.argtypes = [c_float, c_float, c_int, _fp, _fp]
        L.or_clamp_for.argtypes = [c_float, c_float, _fp, _fp]
        L.or_default_clamp.argtypes = [c_float, c_float, _fp, _fp]
        L.or_quake.argtypes = [c_float] * 5
        L.or_quake.restype = c_float
        L.or_quake2.argtypes = [c_float] * 8
        L.or_quake2.restype = c_float
        L.or_quake_buffer.argtypes = [_fp, _fp, c_size_t, c_float, c_float, c_float, c_float]
        L.or_quake2_buffer.argtypes = [_fp, _fp, c_size_t] + [c_float] * 7
        L.or_logistic_buffer.argtypes = [_fp, _fp, c_size_t, c_int, c_int]
        L.or_gelu_buffer.argtypes = [_fp, _fp, c_size_t, c_int, c_int]
        L.or_softmax_rows.argtypes = [_fp, c_size_t, c_size_t, c_float, c_int, c_float, c_float,
                                      c_float, c_int, c_int, _fp]
        L.or_softmax_rows_ordered.argtypes = [_fp, c_size_t, c_size_t, c_float, c_int, c_float,
                                              c_float, c_float, c_int, c_int, c_int, c_int,
                                              ctypes.c_longlong, c_int, _fp]
        L.or_softmax_row_scalars.argtypes = [c_float, c_float, c_int, _fp, _fp, _fp]
        L.or_gelu_constants.argtypes = [_fp] * 4
        for name in ("or_exact_exp", "or_exact_logistic", "or_exact_gelu_tanh",
                     "or_exact_gelu_sigmoid"):
            getattr(L, name).argtypes = [c_double]
            getattr(L, name).restype = c_double
        L.or_exact_softmax.argtypes = [_fp, c_size_t, c_double, _dp]
        L.or_check_div3_replacement.restype = c_uint64
        L.or_sweep_compare.argtypes = [c_int, c_int, c_int, c_uint64, c_uint64, c_void_p, c_int,
                                       POINTER(c_uint64)]
        L.or_sweep_compare.restype = c_uint64

    # --- coefficient derivation (kernels.cpp:25-87) ---
    def coeffs_for(self, p, q=0.0, centering_bias=False):
        c0, c1 = c_float(), c_float()
        if self.lib.or_coeffs_for(p, q, int(bool(centering_bias)), c0, c1) != 0:
            raise OracleError("coeffs_for: input scale p must be non-zero")
        return np.float32(c0.value), np.float32(c1.value)

    def clamp_for(self, c0, c1):
        lo, hi = c_float(), c_float()
        self.lib.or_clamp_for(c0, c1, lo, hi)
        return np.float32(lo.value), np.float32(hi.value)

    def default_clamp(self, p, q=0.0):
        lo, hi = c_float(), c_float()
        if self.lib.or_default_clamp(p, q, lo, hi) != 0:
            raise OracleError("default_clamp: input scale p must be non-zero")
        return np.float32(lo.value), np.float32(hi.value)

    def gelu_constants(self):
        v = [c_float() for _ in range(4)]
        self.lib.or_gelu_constants(*v)
        return tuple(np.float32(x.value) for x in v)

    def softmax_row_scalars(self, m, t, bias):
        v = [c_float() for _ in range(3)]
        self.lib.or_softmax_row_scalars(m, t, int(bias), *v)
        return tuple(np.float32(x.value) for x in v)

    # --- scalar kernels ---
    def quake(self, x, c0, c1, lo, hi):
        return np.float32(self.lib.or_quake(x, c0, c1, lo, hi))

    def quake2(self, x, c0, c1, quad, lo, hi):
        return np.float32(self.lib.or_quake2(x, c0, c1, *quad, lo, hi))

    # --- buffers ---
    def quake_buffer(self, xs, c0, c1, lo, hi):
        xs = _f32(xs)
        out = np.empty_like(xs)
        self.lib.or_quake_buffer(_ptr(xs), _ptr(out), xs.size, c0, c1, lo, hi)
        return out

    def quake2_buffer(self, xs, c0, c1, quad, lo, hi):
        xs = _f32(xs)
        out = np.empty_like(xs)
        self.lib.or_quake2_buffer(_ptr(xs), _ptr(out), xs.size, c0, c1, *quad, lo, hi)
        return out

    def logistic_buffer(self, xs, kernel, bias=-1):
        xs = _f32(xs)
        out = np.empty_like(xs)
        self.lib.or_logistic_buffer(_ptr(xs), _ptr(out), xs.size, kernel, bias)
        return out

    def gelu_buffer(self, xs, kernel, bias=-1):
        xs = _f32(xs)
        out = np.empty_like(xs)
        self.lib.or_gelu_buffer(_ptr(xs), _ptr(out), xs.size, kernel, bias)
        return out

    def softmax_rows(self, m, cols, temperature=1.0, kernel=QUAKE2, bias=-1,
                     quad=CONTINUITY, sum_mode=0):
        m = _f32(m)
        out = np.empty_like(m)
        st = self.lib.or_softmax_rows(_ptr(m), m.size, cols, temperature, bias, *quad, kernel,
                                      sum_mode, _ptr(out))
        if st != 0:
            raise OracleError(f"softmax_rows status {st}")
        return out

    def softmax_rows_ordered(self, m, cols, plan, temperature=1.0, kernel=QUAKE2, bias=-1,
                             quad=CONTINUITY):
        """Restatement summed in the GPU plan's declared order (see header)."""
        m = _f32(m)
        out = np.empty_like(m)
        st = self.lib.or_softmax_rows_ordered(_ptr(m), m.size, cols, temperature, bias, *quad,
                                              kernel, plan["width"], plan["lanes"],
                                              plan["cluster"], plan["slice"],
                                              int(plan.get("balanced", 0)), _ptr(out))
        if st != 0:
            raise OracleError(f"softmax_rows_ordered status {st}")
        return out

    # --- fp64 truth (oracle.cpp:30-61) ---
    def exact_exp(self, x):
        return self.lib.or_exact_exp(x)

    def exact_logistic(self, x):
        return self.lib.or_exact_logistic(x)

    def exact_gelu_tanh(self, x):
        return self.lib.or_exact_gelu_tanh(x)

    def exact_softmax(self, v, t):
        v = _f32(v)
        out = np.empty(v.size, dtype=np.float64)
        if self.lib.or_exact_softmax(_ptr(v), v.size, t, _ptr(out, _dp)) != 0:
            raise OracleError("exact_softmax: bad shapes")
        return out

    def sweep_compare(self, op, kernel, bias, start, got: np.ndarray, threads=None):
        """Mismatches of op over bit patterns start..start+len(got)-1 vs `got`."""
        threads = threads or max(1, os.cpu_count() or 1)
        fb = c_uint64()
        got = np.ascontiguousarray(got, dtype=np.float32)
        bad = self.lib.or_sweep_compare(op, kernel, bias, start, got.size, got.ctypes.data,
                                        threads, ctypes.byref(fb))
        return int(bad), int(fb.value)

    def check_div3_replacement(self) -> int:
        return int(self.lib.or_check_div3_replacement())


class Reference:
    """The reference library itself, compiled in place (oracle/_ref)."""

    kind = "reference"

    def __init__(self, path: str = REFERENCE_SO):
        if not os.path.exists(path):
            raise FileNotFoundError(f"{path} missing: build it with `make -C oracle` "
                                    "where /root/reference exists")
        L = self.lib = ctypes.CDLL(path)
        L.ref_last_error.restype = ctypes.c_char_p
        L.ref_effective_threads.restype = c_uint
        L.ref_coeffs_for.argtypes = [c_float, c_float, c_int, _fp, _fp]
        L.ref_default_clamp.argtypes = [c_float, c_float, _fp, _fp]
        L.ref_clamp_for.argtypes = [c_float, c_float, _fp, _fp]
        L.ref_named_coeffs.argtypes = [c_int, c_int, _fp, _fp]
        L.ref_quake.argtypes = [c_float] * 5
        L.ref_quake.restype = c_float
        L.ref_quake2.argtypes = [c_float] * 8
        L.ref_quake2.restype = c_float
        L.ref_quake_buffer.argtypes = [_fp, c_size_t, _fp] + [c_float] * 4
        L.ref_quake2_buffer.argtypes = [_fp, c_size_t, _fp] + [c_float] * 7
        L.ref_logistic_buffer.argtypes = [_fp, c_size_t, _fp, c_int, c_int]
        L.ref_gelu_buffer.argtypes = [_fp, c_size_t, _fp, c_int, c_int]
        L.ref_logistic.argtypes = [c_float, c_int, c_int]
        L.ref_logistic.restype = c_float
        L.ref_gelu.argtypes = [c_float, c_int, c_int]
        L.ref_gelu.restype = c_float
        L.ref_softmax_rows.argtypes = [_fp, c_size_t, c_size_t, c_float, c_int, c_float, c_float,
                                       c_float, c_int, _fp, c_size_t]
        L.ref_softmax_row.argtypes = [_fp, c_size_t, c_float, c_int, c_float, c_float, c_float,
                                      c_int, _fp, c_size_t]
        L.ref_gelu_constants.argtypes = [_fp] * 4
        for name in ("ref_exact_exp", "ref_exact_logistic", "ref_exact_gelu_tanh"):
            getattr(L, name).argtypes = [c_double]
            getattr(L, name).restype = c_double
        L.ref_exact_softmax.argtypes = [_fp, c_size_t, c_double, _dp]
        L.ref_bench_inputs.argtypes = [c_int, c_size_t, c_uint64, _fp]
        L.ref_bench_inputs.restype = None
        L.ref_fusion_ablation.argtypes = [c_int, c_int, c_size_t, c_size_t, c_size_t, c_float,
                                          c_uint64, _dp, _dp, _dp]
        _u64p = POINTER(c_uint64)
        L.ref_sweep_error.argtypes = [c_int, c_int, c_int, c_float, c_float, c_float, c_float,
                                      c_float, c_uint64, c_uint, _u64p, _dp, _dp, _fp]
        L.ref_quad_max_rel_err.argtypes = [c_double, c_double, c_double, c_size_t]
        L.ref_quad_max_rel_err.restype = c_double
        L.ref_grid_search_quad.argtypes = [_dp, _fp, _dp, _u64p]
        L.ref_continuity_probe.argtypes = [c_int, c_int, c_int, c_float, c_float, c_float, c_int,
                                           c_int, _dp, _fp]
        L.ref_bias_reoptimize.argtypes = [c_int, c_int, c_int, c_float, c_float, c_float,
                                          c_double, c_double, _fp, _dp, POINTER(c_int)]

    def _check(self, st):
        if st != 0:
            raise OracleError(self.lib.ref_last_error().decode())

    def effective_threads(self) -> int:
        return int(self.lib.ref_effective_threads())

    def coeffs_for(self, p, q=0.0, centering_bias=False):
        c0, c1 = c_float(), c_float()
        self._check(self.lib.ref_coeffs_for(p, q, int(bool(centering_bias)), c0, c1))
        return np.float32(c0.value), np.float32(c1.value)

    def named_coeffs(self, which: str, bias: bool):
        idx = {"natural": 0, "base2": 1, "negated": 2}[which]
        c0, c1 = c_float(), c_float()
        self.lib.ref_named_coeffs(idx, int(bias), c0, c1)
        return np.float32(c0.value), np.float32(c1.value)

    def clamp_for(self, c0, c1):
        lo, hi = c_float(), c_float()
        self.lib.ref_clamp_for(c0, c1, lo, hi)
        return np.float32(lo.value), np.float32(hi.value)

    def default_clamp(self, p, q=0.0):
        lo, hi = c_float(), c_float()
        self._check(self.lib.ref_default_clamp(p, q, lo, hi))
        return np.float32(lo.value), np.float32(hi.value)

    def gelu_constants(self):
        v = [c_float() for _ in range(4)]
        self.lib.ref_gelu_constants(*v)
        return tuple(np.float32(x.value) for x in v)

    def quake(self, x, c0, c1, lo, hi):
        return np.float32(self.lib.ref_quake(x, c0, c1, lo, hi))

    def quake2(self, x, c0, c1, quad, lo, hi):
        return np.float32(self.lib.ref_quake2(x, c0, c1, *quad, lo, hi))

    def logistic(self, x, kernel, bias=-1):
        return np.float32(self.lib.ref_logistic(x, kernel, bias))

    def gelu(self, x, kernel, bias=-1):
        return np.float32(self.lib.ref_gelu(x, kernel, bias))

    def quake_buffer(self, xs, c0, c1, lo, hi, out=None):
        xs = _f32(xs)
        out = np.empty_like(xs) if out is None else out
        self._check(self.lib.ref_quake_buffer(_ptr(xs), xs.size, _ptr(out), c0, c1, lo, hi))
        return out

    def quake2_buffer(self, xs, c0, c1, quad, lo, hi, out=None):
        xs = _f32(xs)
        out = np.empty_like(xs) if out is None else out
        self._check(self.lib.ref_quake2_buffer(_ptr(xs), xs.size, _ptr(out), c0, c1, *quad,
                                               lo, hi))
        return out

    def logistic_buffer(self, xs, kernel, bias=-1, out=None):
        xs = _f32(xs)
        out = np.empty_like(xs) if out is None else out
        self._check(self.lib.ref_logistic_buffer(_ptr(xs), xs.size, _ptr(out), kernel, bias))
        return out

    def gelu_buffer(self, xs, kernel, bias=-1, out=None):
        xs = _f32(xs)
        out = np.empty_like(xs) if out is None else out
        self._check(self.lib.ref_gelu_buffer(_ptr(xs), xs.size, _ptr(out), kernel, bias))
        return out

    def softmax_rows(self, m, cols, temperature=1.0, kernel=QUAKE2, bias=-1,
                     quad=CONTINUITY, out=None):
        m = _f32(m)
        out = np.empty_like(m) if out is None else out
        self._check(self.lib.ref_softmax_rows(_ptr(m), m.size, cols, temperature, bias, *quad,
                                              kernel, _ptr(out), out.size))
        return out

    def softmax_row(self, v, temperature=1.0, kernel=QUAKE2, bias=-1, quad=CONTINUITY):
        v = _f32(v)
        out = np.empty_like(v)
        self._check(self.lib.ref_softmax_row(_ptr(v), v.size, temperature, bias, *quad,
                                             kernel, _ptr(out), out.size))
        return out

    def exact_exp(self, x):
        return self.lib.ref_exact_exp(x)

    def exact_logistic(self, x):
        return self.lib.ref_exact_logistic(x)

    def exact_gelu_tanh(self, x):
        return self.lib.ref_exact_gelu_tanh(x)

    def exact_softmax(self, v, t):
        v = _f32(v)
        out = np.empty(v.size, dtype=np.float64)
        self._check(self.lib.ref_exact_softmax(_ptr(v), v.size, t, _ptr(out, _dp)))
        return out

    # --- bench.cpp: the fusion ablation's inputs and checksums ---
    WORKLOADS = {"softmax_matrix": 0, "gelu_vector": 1, "exp_vector": 2, "logistic_vector": 3}

    def bench_inputs(self, workload: str, count: int, seed: int = 42) -> np.ndarray:
        out = np.empty(count, dtype=np.float32)
        self.lib.ref_bench_inputs(self.WORKLOADS[workload], count, seed, _ptr(out))
        return out

    def fusion_ablation(self, workload: str, kernel: int, rows=0, cols=0, n=0,
                        temperature=1.0, seed=42):
        """(fused checksum, unfused checksum, max rel divergence), bench.cpp:425-513."""
        f, u, d = c_double(), c_double(), c_double()
        self._check(self.lib.ref_fusion_ablation(self.WORKLOADS[workload], kernel, rows, cols, n,
                                                 temperature, seed, f, u, d))
        return f.value, u.value, d.value

    # --- lab.cpp: the accuracy lab (pins the GPU lab) ---
    def sweep_error(self, kind, natural=True, bias=True, quad=CONTINUITY, lo=-80.0, hi=80.0,
                    uniform_samples=1 << 22, period_stride=1):
        """(samples, max_rel_err, mean_rel_err, argmax_input), lab.cpp:150-200."""
        n, mx, mean, arg = c_uint64(), c_double(), c_double(), c_float()
        self._check(self.lib.ref_sweep_error(kind, int(natural), int(bias), *quad, lo, hi,
                                             uniform_samples, period_stride, n, mx, mean, arg))
        return n.value, mx.value, mean.value, np.float32(arg.value)

    def quad_max_rel_err(self, a0, a1, a2, intervals=1 << 16):
        return self.lib.ref_quad_max_rel_err(a0, a1, a2, intervals)

    def grid_search_quad(self, axes=(0.30, 0.36, 0.001, -0.05, 0.02, 0.001, 0.64, 0.72, 0.001)):
        ax = np.asarray(axes, np.float64)
        best = np.zeros(3, np.float32)
        err, pts = c_double(), c_uint64()
        self._check(self.lib.ref_grid_search_quad(_ptr(ax, _dp), _ptr(best), err, pts))
        return tuple(best), err.value, pts.value

    def continuity_probe(self, kind, natural, bias, k_lo, k_hi, quad=CONTINUITY):
        w, at = c_double(), c_float()
        self._check(self.lib.ref_continuity_probe(kind, int(natural), int(bias), *quad, k_lo, k_hi,
                                                  w, at))
        return w.value, np.float32(at.value)

    def bias_reoptimize(self, kind, natural=True, bias=True, quad=CONTINUITY, lo=0.0, hi=0.1):
        b, err, near = c_float(), c_double(), c_int()
        self._check(self.lib.ref_bias_reoptimize(kind, int(natural), int(bias), *quad, lo, hi, b,
                                                 err, near))
        return np.float32(b.value), err.value, bool(near.value)


def restatement() -> Restatement:
    return Restatement()


def reference_or_none():
    try:
        return Reference()
    except (FileNotFoundError, OSError):
        return None


def best_cpu_baseline():
    """The reference's own CPU path where it was built, else the restatement."""
    ref = reference_or_none()
    return ref if ref is not None else restatement()
