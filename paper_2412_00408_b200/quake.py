"""Python mirror of the reference's operator interface for the QuAKE path.

Same names, argument meaning and error behaviour as the reference's
``quake::`` API (core/include/quake/kernels.hpp:39-171 and
core/include/quake/nonlin.hpp:32-97; paths relative to
/root/reference/proj/), implemented over the C-ABI of ``libquake_b200.so``:

* numpy arrays / CPU tensors go through the host-span entry points
  (``qk_<op>``): synchronous, reference validation, ``out`` untouched on error,
  sharded over :func:`set_devices`;
* CUDA tensors go through the device entry points (``qk_<op>_device``) on
  torch's current stream.

The reference's ``std::invalid_argument`` is :class:`QuakeInvalidArgument`
(a ``ValueError``) carrying the reference's message text.
"""
from __future__ import annotations

import ctypes
import enum
from dataclasses import dataclass, field
from typing import Optional

import numpy as np

from . import _lib
from ._lib import (AffineCoeffsC, ClampRangeC, GeluConstantsC, QuadCoeffsC, SoftmaxParamsC,
                   SoftmaxPlanC)


class QuakeInvalidArgument(ValueError):
    """The reference's std::invalid_argument (status 1..99)."""

    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


class QuakeCudaError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(msg)
        self.status = status


def _check(status: int) -> None:
    if status == 0:
        return
    msg = _lib.last_error()
    if 1 <= status < 100:
        raise QuakeInvalidArgument(status, msg)
    raise QuakeCudaError(status, msg or f"quake_b200 status {status}")


class KernelChoice(enum.IntEnum):
    """nonlin.hpp:32 KernelChoice, plus the GPU-only comparison kernels."""

    Exact = 0
    Quake = 1
    Quake2 = 2
    Expf = 3      # QuAKE structure with CUDA expf
    FastExp = 4   # QuAKE structure with __expf
    QuakeUnfused = 5   # fusion ablation (bench.cpp:137-166, 212-233): softmax / gelu only
    Quake2Unfused = 6


def kernel_name(k: KernelChoice) -> str:
    return _lib.lib().qk_kernel_name(int(k)).decode()


def resolve_centering_bias(k: KernelChoice, requested: Optional[bool]) -> bool:
    """nonlin.hpp:39-41."""
    req = -1 if requested is None else int(bool(requested))
    return bool(_lib.lib().qk_resolve_centering_bias(int(k), req))


F32 = np.float32


@dataclass(frozen=True)
class AffineCoeffs:
    """kernels.hpp:39-46."""

    c0: float
    c1: float
    input_scale: float = 0.0
    input_shift: float = 0.0
    bias_applied: bool = False

    def _c(self) -> AffineCoeffsC:
        return AffineCoeffsC(self.c0, self.c1, self.input_scale, self.input_shift,
                             int(self.bias_applied))

    @staticmethod
    def _from(c: AffineCoeffsC) -> "AffineCoeffs":
        return AffineCoeffs(F32(c.c0), F32(c.c1), F32(c.input_scale), F32(c.input_shift),
                            bool(c.bias_applied))


@dataclass(frozen=True)
class QuadCoeffs:
    """kernels.hpp:60-76."""

    a0: float
    a1: float
    a2: float

    @staticmethod
    def continuity() -> "QuadCoeffs":
        q = _lib.lib().qk_quad_continuity()
        return QuadCoeffs(F32(q.a0), F32(q.a1), F32(q.a2))

    @staticmethod
    def minimax() -> "QuadCoeffs":
        q = _lib.lib().qk_quad_minimax()
        return QuadCoeffs(F32(q.a0), F32(q.a1), F32(q.a2))

    def is_continuity_default(self) -> bool:
        return bool(_lib.lib().qk_quad_is_continuity_default(ctypes.byref(self._c())))

    def _c(self) -> QuadCoeffsC:
        return QuadCoeffsC(self.a0, self.a1, self.a2)


@dataclass(frozen=True)
class ClampRange:
    """kernels.hpp:81-84."""

    lo: float
    hi: float

    def _c(self) -> ClampRangeC:
        return ClampRangeC(self.lo, self.hi)


@dataclass(frozen=True)
class GeluConstants:
    """nonlin.hpp:55-62."""

    kappa: float
    root2_over_pi: float
    fused_scale: float
    inverse_kappa: float

    @staticmethod
    def defaults() -> "GeluConstants":
        g = _lib.lib().qk_gelu_constants_defaults()
        return GeluConstants(F32(g.kappa), F32(g.root2_over_pi), F32(g.fused_scale),
                             F32(g.inverse_kappa))


@dataclass
class SoftmaxParams:
    """nonlin.hpp:43-49."""

    temperature: float = 1.0
    centering_bias: Optional[bool] = None
    quad: QuadCoeffs = field(default_factory=lambda: QuadCoeffs.continuity())

    def _c(self) -> SoftmaxParamsC:
        cb = -1 if self.centering_bias is None else int(bool(self.centering_bias))
        return SoftmaxParamsC(self.temperature, cb, self.quad._c())


# ---- coefficient derivation (kernels.cpp:25-87) ----

@dataclass(frozen=True)
class FpFormat:
    """bitcore.hpp:32-53: exponent width, mantissa width, exponent bias."""
    exponent_bits: int = 8
    mantissa_bits: int = 23
    bias: int = 127

    @staticmethod
    def single() -> "FpFormat":
        return FpFormat(8, 23, 127)

    def _c(self):
        return _lib.FpFormatC(self.exponent_bits, self.mantissa_bits, self.bias)


kSingle = FpFormat.single()


def coeffs_for(p: float, q: float = 0.0, *args, centering_bias: bool = False,
               fmt: Optional[FpFormat] = None) -> AffineCoeffs:
    """kernels.cpp:25-40. Positional forms: (p, q, centering_bias) or the
    reference's (p, q, fmt, centering_bias)."""
    args = list(args)
    if args and isinstance(args[0], FpFormat):
        fmt = args.pop(0)
    if args:
        centering_bias = args.pop(0)
    out = AffineCoeffsC()
    f = (fmt or kSingle)._c()
    _check(_lib.lib().qk_coeffs_for_format(p, q, ctypes.byref(f), int(bool(centering_bias)),
                                           ctypes.byref(out)))
    return AffineCoeffs._from(out)


def natural_exp_coeffs(centering_bias: bool = True) -> AffineCoeffs:
    return AffineCoeffs._from(_lib.lib().qk_natural_exp_coeffs(int(bool(centering_bias))))


def base2_coeffs(centering_bias: bool = False) -> AffineCoeffs:
    return AffineCoeffs._from(_lib.lib().qk_base2_coeffs(int(bool(centering_bias))))


def negated_natural_exp_coeffs(centering_bias: bool = True) -> AffineCoeffs:
    return AffineCoeffs._from(
        _lib.lib().qk_negated_natural_exp_coeffs(int(bool(centering_bias))))


def default_clamp(p: float, q: float = 0.0, fmt: Optional[FpFormat] = None) -> ClampRange:
    """kernels.cpp:74-82."""
    out = ClampRangeC()
    f = (fmt or kSingle)._c()
    _check(_lib.lib().qk_default_clamp_format(p, q, ctypes.byref(f), ctypes.byref(out)))
    return ClampRange(F32(out.lo), F32(out.hi))


def clamp_for(c: AffineCoeffs) -> ClampRange:
    r = _lib.lib().qk_clamp_for(ctypes.byref(c._c()))
    return ClampRange(F32(r.lo), F32(r.hi))


def softmax_plan(cols: int, aligned16: bool = True,
                 kernel: "KernelChoice" = None) -> dict:
    """Launch geometry the library picks for rows of `cols` columns and the
    given kernel choice (default Quake2); it fixes the summation order. It
    depends on `cols`, the kernel and the device only, never on the data's
    address (`aligned16` is accepted for compatibility and ignored)."""
    p = SoftmaxPlanC()
    k = KernelChoice.Quake2 if kernel is None else kernel
    _check(_lib.lib().qk_softmax_plan(cols, int(aligned16), int(k), ctypes.byref(p)))
    return {k: getattr(p, k) for k, _ in SoftmaxPlanC._fields_}


# ---- devices ----

def device_count() -> int:
    n = ctypes.c_int(0)
    _lib.lib().qk_device_count(ctypes.byref(n))
    return n.value


def set_devices(devices) -> None:
    """Devices the host-buffer operators shard over (the QUAKE_THREADS analogue)."""
    devs = list(devices or [])
    arr = (ctypes.c_int * max(1, len(devs)))(*devs)
    _check(_lib.lib().qk_set_devices(arr, len(devs)))


def set_device_shards(devices) -> None:
    """Like set_devices, but a device may repeat: one shard (own workspace,
    own host thread) per entry — runs the multi-GPU split on one GPU."""
    devs = list(devices or [])
    arr = (ctypes.c_int * max(1, len(devs)))(*devs)
    _check(_lib.lib().qk_set_device_shards(arr, len(devs)))


def set_workspace_limit(nbytes: int) -> None:
    """Device workspace per host-span shard in bytes (0 = automatic). Larger
    host inputs stream through chunk rings (softmax: validation pass first)."""
    _lib.lib().qk_set_workspace_limit(int(nbytes))


def set_host_validation(threads: int = -1, min_bytes: int = 64 << 20) -> None:
    """Overlapped write-back of host-span softmax_rows (pinned spans): host
    threads validate the shard's tail while the device validates its front,
    so the download starts before the upload ends. threads < 0 automatic,
    0 off (the device validates alone)."""
    _lib.lib().qk_set_host_validation(int(threads), int(min_bytes))


def set_plan_override(name: Optional[str], value: int = 0, clear: bool = False) -> None:
    """Set (or with ``clear`` unset) a softmax planner knob (QK_SM_*); name
    None clears all. The environment is read once, at first use."""
    _check(_lib.lib().qk_set_plan_override(None if name is None else name.encode(),
                                           int(value), int(bool(clear))))


class plan_override:
    """Context manager: ``with plan_override(QK_SM_RING=0): ...``."""

    def __init__(self, **opts):
        self.opts = opts

    def __enter__(self):
        for k, v in self.opts.items():
            set_plan_override(k, v)
        return self

    def __exit__(self, *exc):
        for k in self.opts:
            set_plan_override(k, 0, clear=True)
        return False


def get_devices() -> list:
    arr = (ctypes.c_int * 64)()
    n = _lib.lib().qk_get_devices(arr, 64)
    return list(arr[:n])


def release_workspace() -> None:
    _lib.lib().qk_release_workspace()


# ---- buffer plumbing ----

def _is_cuda_tensor(x) -> bool:
    return getattr(x, "is_cuda", False) is True


def _stream_handle() -> int:
    import torch
    return torch.cuda.current_stream().cuda_stream


class _Host:
    """Host view of an array-like (numpy or CPU tensor) as contiguous float32."""

    def __init__(self, x, writable=False):
        if hasattr(x, "detach") and not _is_cuda_tensor(x):  # torch CPU tensor
            import torch
            if x.dtype != torch.float32 or not x.is_contiguous():
                if writable:
                    raise QuakeInvalidArgument(7, "output tensor must be contiguous float32")
                x = x.detach().to(torch.float32).contiguous()
            self.obj = x
            self.ptr = x.data_ptr()
            self.size = x.numel()
            return
        a = np.asarray(x)
        if writable:
            if a.dtype != np.float32 or not a.flags.c_contiguous or not a.flags.writeable:
                raise QuakeInvalidArgument(7, "output array must be writable C-contiguous float32")
        else:
            a = np.ascontiguousarray(a, dtype=np.float32)
        self.obj = a
        self.ptr = a.ctypes.data if a.size else 0
        self.size = a.size


def _new_like(x):
    if _is_cuda_tensor(x) or hasattr(x, "detach"):
        import torch
        return torch.empty(x.shape, dtype=torch.float32, device=x.device)
    return np.empty(np.shape(x), dtype=np.float32)


def _dev_tensor(x, writable=False):
    import torch
    if x.dtype != torch.float32 or not x.is_contiguous():
        if writable:
            raise QuakeInvalidArgument(7, "output tensor must be contiguous float32")
        x = x.to(torch.float32).contiguous()
    return x


def _mixed_spans(xs, out):
    """Pointers and sizes for a host-span call where at most one side may be a
    CUDA tensor. The converted tensors/arrays are returned in ``keep`` so they
    outlive the C call, and torch's current stream is synchronised AFTER the
    conversions: the library's host-span path runs on its own streams, so any
    pending producer (or the conversion itself) must have finished."""
    hx = _Host(xs) if not _is_cuda_tensor(xs) else None
    ho = _Host(out, writable=True) if not _is_cuda_tensor(out) else None
    dx = None if hx else _dev_tensor(xs)
    do = None if ho else _dev_tensor(out, True)
    xp, n = (hx.ptr, hx.size) if hx else (dx.data_ptr(), dx.numel())
    op, on = (ho.ptr, ho.size) if ho else (do.data_ptr(), do.numel())
    if dx is not None or do is not None:
        import torch
        dev = (dx if dx is not None else do).device
        torch.cuda.current_stream(dev).synchronize()
    return xp, n, op, on, (hx, ho, dx, do)


def _run_elementwise(xs, out, host_fn, dev_fn):
    """host_fn(xp, n, op, on) / dev_fn(xp, op, n, stream) -> status."""
    if out is None:
        out = _new_like(xs)
    if _is_cuda_tensor(xs) and _is_cuda_tensor(out):
        x = _dev_tensor(xs)
        o = _dev_tensor(out, writable=True)
        if o.numel() != x.numel():
            raise QuakeInvalidArgument(1, "output size mismatch")
        _check(dev_fn(x.data_ptr(), o.data_ptr(), x.numel(), _stream_handle()))
        return out
    xp, n, op, on, keep = _mixed_spans(xs, out)
    _check(host_fn(xp, n, op, on))
    del keep
    return out


def _split_out(args, n_rest):
    """Reference overloads: (xs, out, rest...) or (xs, rest...)."""
    if len(args) == n_rest + 1:
        return args[0], args[1:]
    return None, args


# ---- kernels.hpp:163-171 ----

def quake_buffer(xs, *args, out=None):
    """quake_buffer(xs, out, c, r) or quake_buffer(xs, c, r) -> out."""
    o, (c, r) = _split_out(args, 2)
    out = o if o is not None else out
    L = _lib.lib()
    cc, rr = c._c(), r._c()
    return _run_elementwise(
        xs, out,
        lambda xp, n, op, on: L.qk_quake_buffer(xp, n, op, on, ctypes.byref(cc), ctypes.byref(rr)),
        lambda xp, op, n, s: L.qk_quake_buffer_device(xp, op, n, ctypes.byref(cc),
                                                      ctypes.byref(rr), s))


def quake2_buffer(xs, *args, out=None):
    """quake2_buffer(xs, out, c, a, r) or quake2_buffer(xs, c, a, r) -> out."""
    o, (c, a, r) = _split_out(args, 3)
    out = o if o is not None else out
    L = _lib.lib()
    cc, aa, rr = c._c(), a._c(), r._c()
    return _run_elementwise(
        xs, out,
        lambda xp, n, op, on: L.qk_quake2_buffer(xp, n, op, on, ctypes.byref(cc),
                                                 ctypes.byref(aa), ctypes.byref(rr)),
        lambda xp, op, n, s: L.qk_quake2_buffer_device(xp, op, n, ctypes.byref(cc),
                                                       ctypes.byref(aa), ctypes.byref(rr), s))


def quake(x: float, c: AffineCoeffs, r: Optional[ClampRange] = None) -> np.float32:
    """kernels.hpp:141-143 / kernels.cpp:92 — evaluated on the GPU (qk_quake)."""
    r = clamp_for(c) if r is None else r
    y = ctypes.c_float()
    _check(_lib.lib().qk_quake(float(x), ctypes.byref(c._c()), ctypes.byref(r._c()),
                               ctypes.byref(y)))
    return np.float32(y.value)


def quake2(x: float, c: AffineCoeffs, a: Optional[QuadCoeffs] = None,
           r: Optional[ClampRange] = None) -> np.float32:
    """kernels.hpp:146-155 / kernels.cpp:94-96 — evaluated on the GPU (qk_quake2)."""
    a = QuadCoeffs.continuity() if a is None else a
    r = clamp_for(c) if r is None else r
    y = ctypes.c_float()
    _check(_lib.lib().qk_quake2(float(x), ctypes.byref(c._c()), ctypes.byref(a._c()),
                                ctypes.byref(r._c()), ctypes.byref(y)))
    return np.float32(y.value)


# ---- nonlin.hpp:83-97 ----

def _bias_arg(b: Optional[bool]) -> int:
    return -1 if b is None else int(bool(b))


def _split_kernel_args(args, out, centering_bias):
    """(out, kernel[, bias]) or (kernel[, bias]) -> (out, kernel, bias)."""
    args = list(args)
    if args and not isinstance(args[0], (int, np.integer)):
        out = args.pop(0)
    kernel = KernelChoice(args[0])
    if len(args) > 1:
        centering_bias = args[1]
    return out, kernel, centering_bias


def logistic_buffer(xs, *args, centering_bias: Optional[bool] = None, out=None):
    """logistic_buffer(xs, out, kernel[, bias]) or logistic_buffer(xs, kernel[, bias])."""
    out, kernel, centering_bias = _split_kernel_args(args, out, centering_bias)
    L = _lib.lib()
    b = _bias_arg(centering_bias)
    return _run_elementwise(
        xs, out,
        lambda xp, n, op, on: L.qk_logistic_buffer(xp, n, op, on, int(kernel), b),
        lambda xp, op, n, s: L.qk_logistic_buffer_device(xp, op, n, int(kernel), b, s))


def gelu_buffer(xs, *args, centering_bias: Optional[bool] = None, out=None):
    """gelu_buffer(xs, out, kernel[, bias]) or gelu_buffer(xs, kernel[, bias])."""
    out, kernel, centering_bias = _split_kernel_args(args, out, centering_bias)
    L = _lib.lib()
    b = _bias_arg(centering_bias)
    return _run_elementwise(
        xs, out,
        lambda xp, n, op, on: L.qk_gelu_buffer(xp, n, op, on, int(kernel), b),
        lambda xp, op, n, s: L.qk_gelu_buffer_device(xp, op, n, int(kernel), b, s))


def exp_buffer(xs, kernel: KernelChoice, out=None):
    """GPU exp comparison op (QuAKE natural exp / expf / __expf)."""
    L = _lib.lib()
    k = int(kernel)
    return _run_elementwise(
        xs, out,
        lambda xp, n, op, on: L.qk_exp_buffer(xp, n, op, on, k),
        lambda xp, op, n, s: L.qk_exp_buffer_device(xp, op, n, k, s))


def logistic(x: float, kernel: KernelChoice, centering_bias: Optional[bool] = None) -> np.float32:
    """nonlin.cpp:198-208 — evaluated on the GPU (qk_logistic)."""
    y = ctypes.c_float()
    _check(_lib.lib().qk_logistic(float(x), int(KernelChoice(kernel)), _bias_arg(centering_bias),
                                  ctypes.byref(y)))
    return np.float32(y.value)


def gelu(x: float, kernel: KernelChoice, centering_bias: Optional[bool] = None) -> np.float32:
    """nonlin.cpp:277-290 — evaluated on the GPU (qk_gelu)."""
    y = ctypes.c_float()
    _check(_lib.lib().qk_gelu(float(x), int(KernelChoice(kernel)), _bias_arg(centering_bias),
                              ctypes.byref(y)))
    return np.float32(y.value)


# ---- nonlin.hpp:70-81 ----

def softmax_rows(matrix, cols: int, params: Optional[SoftmaxParams] = None,
                 kernel: KernelChoice = KernelChoice.Quake2, out=None, check: bool = True):
    """softmax_rows(matrix, cols, params, kernel[, out]) -> out.

    CUDA tensors run on torch's current stream; with ``check`` the call
    synchronises and raises on non-finite input like the reference
    (nonlin.cpp:43-55). Host arrays follow the reference exactly: every row
    is validated before ``out`` is written.
    """
    params = SoftmaxParams() if params is None else params
    L = _lib.lib()
    pc = params._c()
    if out is None:
        out = _new_like(matrix)
    if _is_cuda_tensor(matrix) and _is_cuda_tensor(out):
        import torch
        x = _dev_tensor(matrix)
        o = _dev_tensor(out, writable=True)
        if o.numel() != x.numel():
            raise QuakeInvalidArgument(1, "softmax_rows: output size mismatch")
        flags = torch.zeros(1, dtype=torch.int32, device=x.device) if check else None
        _check(L.qk_softmax_rows_device(x.data_ptr(), x.numel(), cols, ctypes.byref(pc),
                                        int(kernel), o.data_ptr(),
                                        flags.data_ptr() if check else None, _stream_handle()))
        if check and int(flags.item()) & 1:
            raise QuakeInvalidArgument(5, "softmax: non-finite input")
        return out
    xp, n, op, on, keep = _mixed_spans(matrix, out)
    _check(L.qk_softmax_rows(xp, n, cols, ctypes.byref(pc), int(kernel), op, on))
    del keep
    return out


def softmax_row(v, params: Optional[SoftmaxParams] = None,
                kernel: KernelChoice = KernelChoice.Quake2, out=None):
    """softmax_row(v, params, kernel[, out]) -> out (nonlin.cpp:143-160)."""
    params = SoftmaxParams() if params is None else params
    L = _lib.lib()
    pc = params._c()
    if out is None:
        out = _new_like(v)
    xp, n, op, on, keep = _mixed_spans(v, out)
    _check(L.qk_softmax_row(xp, n, ctypes.byref(pc), int(kernel), op, on))
    del keep
    return out
