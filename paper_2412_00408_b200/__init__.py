"""B200-native (sm_100a) QuAKE hot path: exp / logistic / GELU / row softmax.

The compute lives in ``libquake_b200.so`` (hand-written CUDA kernels + a C++
host layer behind the C-ABI in ``include/quake_b200.h``). This package is the
Python face of that ABI, mirroring the reference's ``quake::`` operator API
(see :mod:`.quake`). There is no CPU fallback: every operator fails loudly if
the library is missing.
"""
from .quake import (AffineCoeffs, ClampRange, FpFormat, GeluConstants, KernelChoice, QuadCoeffs,
                    QuakeCudaError, QuakeInvalidArgument, SoftmaxParams, base2_coeffs, clamp_for,
                    coeffs_for, default_clamp, kSingle, device_count, exp_buffer, gelu, gelu_buffer,
                    get_devices, kernel_name, logistic, logistic_buffer, natural_exp_coeffs,
                    negated_natural_exp_coeffs, quake, quake2, quake2_buffer, quake_buffer,
                    plan_override, release_workspace, resolve_centering_bias, set_device_shards,
                    set_devices, set_host_validation, set_plan_override, set_workspace_limit, softmax_plan,
                    softmax_row, softmax_rows)
from ._lib import LIB_PATH, lib

__all__ = [n for n in dir() if not n.startswith("_")]
