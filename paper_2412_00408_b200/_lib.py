"""ctypes binding of ``libquake_b200.so`` (the C-ABI in include/quake_b200.h and
include/quake_b200_lab.h).

Loading fails loudly: there is no CPU fallback anywhere in this package.
"""
from __future__ import annotations

import ctypes
import os
from ctypes import (POINTER, Structure, c_char_p, c_double, c_float, c_int, c_int32, c_int64,
                    c_size_t, c_uint32, c_uint64, c_void_p)

PKG_DIR = os.path.dirname(os.path.abspath(__file__))
# QK_LIB_PATH: an alternative build of the same library (A/B measurements)
LIB_PATH = os.environ.get("QK_LIB_PATH") or os.path.join(PKG_DIR, "libquake_b200.so")
ABI_VERSION = 3

# qk_status
QK_OK = 0
QK_ERR_SIZE_MISMATCH = 1
QK_ERR_NOT_DIVISIBLE = 2
QK_ERR_BAD_TEMPERATURE = 3
QK_ERR_EMPTY_ROW = 4
QK_ERR_NON_FINITE = 5
QK_ERR_ZERO_SLOPE = 6
QK_ERR_BAD_ARGUMENT = 7
QK_ERR_CUDA = 100
QK_ERR_NO_DEVICE = 101


class AffineCoeffsC(Structure):
    _fields_ = [("c0", c_float), ("c1", c_float), ("input_scale", c_float),
                ("input_shift", c_float), ("bias_applied", c_int32)]


class QuadCoeffsC(Structure):
    _fields_ = [("a0", c_float), ("a1", c_float), ("a2", c_float)]


class ClampRangeC(Structure):
    _fields_ = [("lo", c_float), ("hi", c_float)]


class SoftmaxParamsC(Structure):
    _fields_ = [("temperature", c_float), ("centering_bias", c_int32), ("quad", QuadCoeffsC)]


class FpFormatC(Structure):
    _fields_ = [("exponent_bits", c_int32), ("mantissa_bits", c_int32), ("bias", c_int32)]


class GeluConstantsC(Structure):
    _fields_ = [("kappa", c_float), ("root2_over_pi", c_float), ("fused_scale", c_float),
                ("inverse_kappa", c_float)]


class SoftmaxPlanC(Structure):
    _fields_ = [("variant", c_int32), ("width", c_int32), ("lanes", c_int32),
                ("cluster", c_int32), ("slice", c_int64), ("threads", c_int32),
                ("vpt", c_int32), ("smem", c_int64), ("stages", c_int32),
                ("balanced", c_int32), ("resident", c_int32)]


# ---- include/quake_b200_lab.h ----
class ExpConfigC(Structure):
    _fields_ = [("kind", c_int), ("natural_base", c_int32), ("centering_bias", c_int32),
                ("quad", QuadCoeffsC)]


class SweepSpecC(Structure):
    _fields_ = [("lo", c_float), ("hi", c_float), ("uniform_samples", c_uint64),
                ("period_stride", c_uint32)]


class ErrorReportC(Structure):
    _fields_ = [("lo", c_float), ("hi", c_float), ("samples", c_uint64),
                ("max_rel_err", c_double), ("mean_rel_err", c_double),
                ("argmax_input", c_float)]


class ExhaustiveReportC(Structure):
    _fields_ = [("lo", c_float), ("hi", c_float), ("samples", c_uint64),
                ("max_rel_err", c_double), ("mean_rel_err", c_double),
                ("argmax_input", c_float), ("monotonic_violations", c_uint64),
                ("first_violation", c_float), ("non_positive", c_uint64),
                ("first_non_positive", c_float)]


class ContinuityReportC(Structure):
    _fields_ = [("worst_jump", c_double), ("at", c_float)]


class GridAxisC(Structure):
    _fields_ = [("lo", c_double), ("hi", c_double), ("step", c_double)]


class GridSpecC(Structure):
    _fields_ = [("a0", GridAxisC), ("a1", GridAxisC), ("a2", GridAxisC)]


class GridResultC(Structure):
    _fields_ = [("best", QuadCoeffsC), ("best_max_rel_err", c_double), ("step_a0", c_double),
                ("step_a1", c_double), ("step_a2", c_double), ("points_searched", c_uint64)]


class BiasResultC(Structure):
    _fields_ = [("beta", c_float), ("max_rel_err", c_double), ("near_reference_bias", c_int32)]


_fp = POINTER(c_float)
_P = c_void_p  # raw pointers (host or device) are passed as integers

# name -> (restype, argtypes); mirrors include/quake_b200.h
SIGNATURES = {
    "qk_abi_version": (c_int, []),
    "qk_last_error": (c_char_p, []),
    "qk_is_invalid_argument": (c_int, [c_int]),
    "qk_device_count": (c_int, [POINTER(c_int)]),
    "qk_set_devices": (c_int, [POINTER(c_int), c_int]),
    "qk_set_device_shards": (c_int, [POINTER(c_int), c_int]),
    "qk_set_workspace_limit": (None, [c_size_t]),
    "qk_set_host_validation": (None, [c_int32, c_size_t]),
    "qk_set_plan_override": (c_int, [c_char_p, c_int32, c_int32]),
    "qk_get_devices": (c_int, [POINTER(c_int), c_int]),
    "qk_release_workspace": (None, []),
    "qk_coeffs_for": (c_int, [c_float, c_float, c_int32, POINTER(AffineCoeffsC)]),
    "qk_natural_exp_coeffs": (AffineCoeffsC, [c_int32]),
    "qk_base2_coeffs": (AffineCoeffsC, [c_int32]),
    "qk_negated_natural_exp_coeffs": (AffineCoeffsC, [c_int32]),
    "qk_default_clamp": (c_int, [c_float, c_float, POINTER(ClampRangeC)]),
    "qk_coeffs_for_format": (c_int, [c_float, c_float, POINTER(FpFormatC), c_int32,
                                     POINTER(AffineCoeffsC)]),
    "qk_default_clamp_format": (c_int, [c_float, c_float, POINTER(FpFormatC),
                                        POINTER(ClampRangeC)]),
    "qk_quake": (c_int, [c_float, POINTER(AffineCoeffsC), POINTER(ClampRangeC), _fp]),
    "qk_quake2": (c_int, [c_float, POINTER(AffineCoeffsC), POINTER(QuadCoeffsC),
                          POINTER(ClampRangeC), _fp]),
    "qk_logistic": (c_int, [c_float, c_int, c_int32, _fp]),
    "qk_gelu": (c_int, [c_float, c_int, c_int32, _fp]),
    "qk_clamp_for": (ClampRangeC, [POINTER(AffineCoeffsC)]),
    "qk_quad_continuity": (QuadCoeffsC, []),
    "qk_quad_minimax": (QuadCoeffsC, []),
    "qk_quad_is_continuity_default": (c_int, [POINTER(QuadCoeffsC)]),
    "qk_gelu_constants_defaults": (GeluConstantsC, []),
    "qk_resolve_centering_bias": (c_int32, [c_int, c_int32]),
    "qk_kernel_name": (c_char_p, [c_int]),
    "qk_softmax_plan": (c_int, [c_size_t, c_int32, c_int, POINTER(SoftmaxPlanC)]),
    "qk_quake_buffer": (c_int, [_P, c_size_t, _P, c_size_t, POINTER(AffineCoeffsC),
                                POINTER(ClampRangeC)]),
    "qk_quake2_buffer": (c_int, [_P, c_size_t, _P, c_size_t, POINTER(AffineCoeffsC),
                                 POINTER(QuadCoeffsC), POINTER(ClampRangeC)]),
    "qk_logistic_buffer": (c_int, [_P, c_size_t, _P, c_size_t, c_int, c_int32]),
    "qk_gelu_buffer": (c_int, [_P, c_size_t, _P, c_size_t, c_int, c_int32]),
    "qk_softmax_rows": (c_int, [_P, c_size_t, c_size_t, POINTER(SoftmaxParamsC), c_int, _P,
                                c_size_t]),
    "qk_softmax_row": (c_int, [_P, c_size_t, POINTER(SoftmaxParamsC), c_int, _P, c_size_t]),
    "qk_exp_buffer": (c_int, [_P, c_size_t, _P, c_size_t, c_int]),
    "qk_quake_buffer_device": (c_int, [_P, _P, c_size_t, POINTER(AffineCoeffsC),
                                       POINTER(ClampRangeC), _P]),
    "qk_quake2_buffer_device": (c_int, [_P, _P, c_size_t, POINTER(AffineCoeffsC),
                                        POINTER(QuadCoeffsC), POINTER(ClampRangeC), _P]),
    "qk_logistic_buffer_device": (c_int, [_P, _P, c_size_t, c_int, c_int32, _P]),
    "qk_gelu_buffer_device": (c_int, [_P, _P, c_size_t, c_int, c_int32, _P]),
    "qk_exp_buffer_device": (c_int, [_P, _P, c_size_t, c_int, _P]),
    "qk_softmax_rows_device": (c_int, [_P, c_size_t, c_size_t, POINTER(SoftmaxParamsC), c_int,
                                       _P, _P, _P]),
}

# mirrors include/quake_b200_lab.h
LAB_SIGNATURES = {
    "qk_sweep_spec_defaults": (SweepSpecC, []),
    "qk_grid_spec_defaults": (GridSpecC, []),
    "qk_lab_coeffs": (c_int, [POINTER(ExpConfigC), POINTER(AffineCoeffsC), POINTER(ClampRangeC)]),
    "qk_sweep_error": (c_int, [POINTER(ExpConfigC), POINTER(SweepSpecC), POINTER(ErrorReportC)]),
    "qk_sweep_exhaustive": (c_int, [POINTER(ExpConfigC), c_float, c_float,
                                    POINTER(ExhaustiveReportC)]),
    "qk_continuity_probe": (c_int, [POINTER(ExpConfigC), c_int32, c_int32,
                                    POINTER(ContinuityReportC)]),
    "qk_quad_max_rel_err": (c_int, [c_double, c_double, c_double, c_uint64, POINTER(c_double)]),
    "qk_grid_search_quad": (c_int, [POINTER(GridSpecC), POINTER(GridResultC)]),
    "qk_bias_reoptimize": (c_int, [POINTER(ExpConfigC), c_double, c_double,
                                   POINTER(BiasResultC)]),
}


class QuakeLibraryMissing(ImportError):
    pass


_LIB = None


def lib() -> ctypes.CDLL:
    """The loaded library; raises QuakeLibraryMissing if it was never built."""
    global _LIB
    if _LIB is None:
        if not os.path.exists(LIB_PATH):
            raise QuakeLibraryMissing(
                f"{LIB_PATH} is missing: build it with `python -c 'import __graft_entry__ as g; "
                "g.build()'` (or `make -C paper_2412_00408_b200/csrc`). There is no CPU fallback.")
        L = ctypes.CDLL(LIB_PATH)
        for name, (res, args) in {**SIGNATURES, **LAB_SIGNATURES}.items():
            fn = getattr(L, name)
            fn.restype = res
            fn.argtypes = args
        if L.qk_abi_version() != ABI_VERSION:
            raise QuakeLibraryMissing(f"{LIB_PATH}: ABI {L.qk_abi_version()} != {ABI_VERSION}")
        _LIB = L
    return _LIB


def last_error() -> str:
    msg = lib().qk_last_error()
    return msg.decode() if msg else ""
