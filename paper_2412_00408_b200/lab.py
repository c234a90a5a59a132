"""GPU accuracy lab: the reference's ``quake::lab``
(core/include/quake/lab.hpp:30-125) over the C-ABI of include/quake_b200_lab.h.

Same configuration objects, defaults, error messages and result fields as the
reference; every approximation is evaluated by the product's sm_100a device
functions. ``sweep_exhaustive`` additionally walks every binary32 input of a
range (full fp32 resolution) for the error band, monotonicity across
consecutive floats and positivity (acceptance criteria c1, c2, c6).
"""
from __future__ import annotations

import ctypes
from dataclasses import dataclass, field
from typing import Optional

from . import _lib
from .quake import KernelChoice, QuadCoeffs
from .quake import _check as _call


@dataclass(frozen=True)
class ExpConfig:
    """lab.hpp:30-44."""

    kind: KernelChoice = KernelChoice.Quake
    natural_base: bool = True
    centering_bias: bool = True
    quad: QuadCoeffs = field(default_factory=QuadCoeffs.continuity)

    def _c(self) -> _lib.ExpConfigC:
        return _lib.ExpConfigC(int(self.kind), int(self.natural_base), int(self.centering_bias),
                               self.quad._c())

    def coeffs_and_clamp(self):
        """(AffineCoeffs, ClampRange) of ExpConfig::coeffs / clamp (lab.cpp:121-129)."""
        from .quake import AffineCoeffs, ClampRange
        c, r = _lib.AffineCoeffsC(), _lib.ClampRangeC()
        _call(_lib.lib().qk_lab_coeffs(ctypes.byref(self._c()), ctypes.byref(c), ctypes.byref(r)))
        return AffineCoeffs._from(c), ClampRange(r.lo, r.hi)

    def label(self) -> str:
        """lab.cpp:137-148 ExpConfig::label."""
        from .quake import kernel_name
        s = kernel_name(self.kind) + (":e" if self.natural_base else ":2")
        if self.kind != KernelChoice.Exact:
            s += ":bias" if self.centering_bias else ":nobias"
            if self.kind == KernelChoice.Quake2 and not self.quad.is_continuity_default():
                s += ":custom-quad"
        return s


@dataclass(frozen=True)
class SweepSpec:
    """lab.hpp:46-55."""

    lo: float = -80.0
    hi: float = 80.0
    uniform_samples: int = 1 << 22
    period_stride: int = 1


@dataclass(frozen=True)
class ErrorReport:
    """lab.hpp:57-66."""

    kernel: str
    lo: float
    hi: float
    samples: int
    max_rel_err: float
    mean_rel_err: float
    argmax_input: float


@dataclass(frozen=True)
class ExhaustiveReport:
    kernel: str
    lo: float
    hi: float
    samples: int
    max_rel_err: float
    mean_rel_err: float
    argmax_input: float
    monotonic_violations: int
    first_violation: float
    non_positive: int
    first_non_positive: float


@dataclass(frozen=True)
class GridAxis:
    """lab.hpp:72-78."""

    lo: float = 0.0
    hi: float = 0.0
    step: float = 0.0


@dataclass(frozen=True)
class GridSpec:
    """lab.hpp:80-84 (defaults: the published neighbourhood at step 0.001)."""

    a0: GridAxis = GridAxis(0.30, 0.36, 0.001)
    a1: GridAxis = GridAxis(-0.05, 0.02, 0.001)
    a2: GridAxis = GridAxis(0.64, 0.72, 0.001)

    def _c(self) -> _lib.GridSpecC:
        ax = lambda a: _lib.GridAxisC(a.lo, a.hi, a.step)  # noqa: E731
        return _lib.GridSpecC(ax(self.a0), ax(self.a1), ax(self.a2))


@dataclass(frozen=True)
class GridSearchResult:
    """lab.hpp:86-93."""

    best: QuadCoeffs
    best_max_rel_err: float
    step_a0: float
    step_a1: float
    step_a2: float
    points_searched: int


@dataclass(frozen=True)
class ContinuityReport:
    """lab.hpp:105-108."""

    worst_jump: float = 0.0
    at: float = 0.0


@dataclass(frozen=True)
class BiasSearchResult:
    """lab.hpp:115-121."""

    beta: float
    max_rel_err: float
    near_reference_bias: bool


def sweep_error(cfg: ExpConfig, spec: Optional[SweepSpec] = None) -> ErrorReport:
    """lab.cpp:150-200: uniform grid plus one exhaustive mantissa period."""
    spec = spec or SweepSpec()
    out = _lib.ErrorReportC()
    _call(_lib.lib().qk_sweep_error(ctypes.byref(cfg._c()), ctypes.byref(
        _lib.SweepSpecC(spec.lo, spec.hi, spec.uniform_samples, spec.period_stride)),
        ctypes.byref(out)))
    from .quake import kernel_name
    return ErrorReport(kernel_name(cfg.kind), out.lo, out.hi, out.samples, out.max_rel_err,
                       out.mean_rel_err, out.argmax_input)


def sweep_exhaustive(cfg: ExpConfig, lo: float = -80.0, hi: float = 80.0) -> ExhaustiveReport:
    """Every binary32 in [lo, hi]: error band, monotonicity, positivity."""
    out = _lib.ExhaustiveReportC()
    _call(_lib.lib().qk_sweep_exhaustive(ctypes.byref(cfg._c()), lo, hi, ctypes.byref(out)))
    from .quake import kernel_name
    return ExhaustiveReport(kernel_name(cfg.kind), out.lo, out.hi, out.samples, out.max_rel_err,
                            out.mean_rel_err, out.argmax_input, out.monotonic_violations,
                            out.first_violation, out.non_positive, out.first_non_positive)


def quad_max_rel_err(a0: float, a1: float, a2: float, intervals: int = 1 << 16) -> float:
    """lab.cpp:209-219."""
    out = ctypes.c_double()
    _call(_lib.lib().qk_quad_max_rel_err(a0, a1, a2, intervals, ctypes.byref(out)))
    return out.value


def grid_search_quad(spec: Optional[GridSpec] = None) -> GridSearchResult:
    """lab.cpp:221-279."""
    spec = spec or GridSpec()
    out = _lib.GridResultC()
    _call(_lib.lib().qk_grid_search_quad(ctypes.byref(spec._c()), ctypes.byref(out)))
    return GridSearchResult(QuadCoeffs(out.best.a0, out.best.a1, out.best.a2),
                            out.best_max_rel_err, out.step_a0, out.step_a1, out.step_a2,
                            out.points_searched)


def continuity_probe(cfg: ExpConfig, k_lo: int, k_hi: int) -> ContinuityReport:
    """lab.cpp:281-328."""
    out = _lib.ContinuityReportC()
    _call(_lib.lib().qk_continuity_probe(ctypes.byref(cfg._c()), k_lo, k_hi, ctypes.byref(out)))
    return ContinuityReport(out.worst_jump, out.at)


def bias_reoptimize(cfg: ExpConfig, beta_lo: float = 0.0, beta_hi: float = 0.1) -> BiasSearchResult:
    """lab.cpp:330-410."""
    out = _lib.BiasResultC()
    _call(_lib.lib().qk_bias_reoptimize(ctypes.byref(cfg._c()), beta_lo, beta_hi,
                                        ctypes.byref(out)))
    return BiasSearchResult(out.beta, out.max_rel_err, bool(out.near_reference_bias))


def report(out=None):
    """The GPU lab report (profiles/): acceptance criteria 1-6 of the reference
    (tests/acceptance.cpp:65-172) plus exhaustive every-binary32 sweeps, timed."""
    import json
    import time

    def emit(d):
        line = json.dumps(d)
        print(line, flush=True)
        if out:
            out.write(line + "\n")

    def timed(fn):
        t = time.perf_counter()
        r = fn()
        return r, time.perf_counter() - t

    acc = SweepSpec(-80.0, 80.0, 1 << 22, 1)
    r, dt = timed(lambda: sweep_error(ExpConfig(KernelChoice.Quake, True, True), acc))
    emit({"criterion": 1, "max_rel_err": r.max_rel_err, "band": [0.042, 0.044],
          "reference_recorded": 0.029883, "samples": r.samples, "seconds": dt})
    r, dt = timed(lambda: sweep_error(ExpConfig(KernelChoice.Quake2, True, False), acc))
    emit({"criterion": 2, "max_rel_err": r.max_rel_err, "band": [0.0030, 0.0035],
          "pass": 0.0030 <= r.max_rel_err <= 0.0035, "seconds": dt})
    g, dt = timed(grid_search_quad)
    emit({"criterion": 3, "best": [float(g.best.a0), float(g.best.a1), float(g.best.a2)],
          "best_max_rel_err": g.best_max_rel_err, "band": [0.0015, 0.0019],
          "reference_recorded": {"best": [0.336, -0.012, 0.677], "err": 0.001966},
          "points": g.points_searched, "seconds": dt})
    b, dt = timed(lambda: bias_reoptimize(ExpConfig(KernelChoice.Quake, True, True)))
    r = sweep_error(ExpConfig(KernelChoice.Quake, True, False), acc)
    emit({"criterion": 4, "beta": b.beta, "unbiased_max_rel_err": r.max_rel_err,
          "pass": 0.040 <= b.beta <= 0.047 and 0.058 <= r.max_rel_err <= 0.064, "seconds": dt})
    j = [continuity_probe(ExpConfig(k, False, False), -100, 100).worst_jump
         for k in (KernelChoice.Quake, KernelChoice.Quake2)]
    emit({"criterion": 5, "worst_jump": j, "limit": 1e-5, "pass": max(j) <= 1e-5})
    for kind, nat, bias, quad in ((KernelChoice.Quake, True, True, None),
                                  (KernelChoice.Quake, True, False, None),
                                  (KernelChoice.Quake2, True, False, None),
                                  (KernelChoice.Quake2, True, True, None),
                                  (KernelChoice.Quake, False, False, None),
                                  (KernelChoice.Quake2, False, False, None),
                                  (KernelChoice.Quake2, True, False, "minimax")):
        q = QuadCoeffs.minimax() if quad else QuadCoeffs.continuity()
        cfg = ExpConfig(kind, nat, bias, q)
        _, rng = cfg.coeffs_and_clamp()
        ex, dt = timed(lambda: sweep_exhaustive(cfg, rng.lo, rng.hi))
        emit({"exhaustive": cfg.label(), "lo": rng.lo, "hi": rng.hi, "samples": ex.samples,
              "max_rel_err": ex.max_rel_err, "mean_rel_err": ex.mean_rel_err,
              "argmax_input": ex.argmax_input, "monotonic_violations": ex.monotonic_violations,
              "first_violation": ex.first_violation, "non_positive": ex.non_positive,
              "seconds": dt, "inputs_per_second": ex.samples / dt,
              "criterion_6": ex.monotonic_violations == 0 if not quad else None})


if __name__ == "__main__":
    import sys
    with open(sys.argv[1], "w") if len(sys.argv) > 1 else open("/dev/null", "w") as fh:
        report(fh)
