"""CPU: the C-ABI library loads, exports every declared symbol, and its host
logic (coefficient derivation, validation order and messages, launch
planning) matches the reference — no GPU needed for any of this."""
import os
import re
import subprocess

import numpy as np
import pytest

import paper_2412_00408_b200 as qk
from paper_2412_00408_b200 import _lib
from oracle.oracle import CONTINUITY
from tests.helpers import bits, restatement

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "quake_b200.h")
LOG2E = np.float32(1.4426950408889634)


def declared_functions():
    src = open(HEADER).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(qk_[a-z0-9_]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    decl = declared_functions()
    assert len(decl) >= 33
    missing = [d for d in decl if d not in exported]
    assert not missing, missing
    # the ctypes binding covers the whole header
    assert set(decl) == set(_lib.SIGNATURES), set(decl) ^ set(_lib.SIGNATURES)


def test_abi_version_and_loud_failure(tmp_path, monkeypatch):
    assert qk.lib().qk_abi_version() == _lib.ABI_VERSION
    monkeypatch.setattr(_lib, "LIB_PATH", str(tmp_path / "missing.so"))
    monkeypatch.setattr(_lib, "_LIB", None)
    with pytest.raises(_lib.QuakeLibraryMissing):
        _lib.lib()


def test_no_oracle_in_product_package():
    pkg = os.path.join(ROOT, "paper_2412_00408_b200")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cpp", ".h", ".cuh")):
                text = open(os.path.join(dirpath, f), errors="ignore").read()
                assert "oracle.oracle" not in text and "liboracle" not in text, f
                assert "libquake_ref" not in text, f


@pytest.mark.parametrize("p,q", [(LOG2E, 0.0), (-LOG2E, 0.0), (1.0, 0.0), (0.7, 0.37),
                                 (np.float32(-0.10309318), 0.0), (3.0, -2.5)])
@pytest.mark.parametrize("bias", [False, True])
def test_coefficients_match_oracle(p, q, bias):
    R = restatement()
    c = qk.coeffs_for(p, q, bias)
    assert (c.c0, c.c1) == R.coeffs_for(p, q, bias)
    r = qk.clamp_for(c)
    assert (r.lo, r.hi) == R.clamp_for(c.c0, c.c1)
    d = qk.default_clamp(p, q)
    assert (d.lo, d.hi) == R.default_clamp(p, q)


def test_named_coefficients_and_constants():
    R = restatement()
    assert (qk.natural_exp_coeffs(True).c0, qk.natural_exp_coeffs(True).c1) == R.coeffs_for(LOG2E, 0, 1)
    assert (qk.negated_natural_exp_coeffs(False).c0,
            qk.negated_natural_exp_coeffs(False).c1) == R.coeffs_for(-LOG2E, 0, 0)
    assert (qk.base2_coeffs().c0, qk.base2_coeffs().c1) == (8388608.0, 1065353216.0)
    g = qk.GeluConstants.defaults()
    assert (g.kappa, g.root2_over_pi, g.fused_scale, g.inverse_kappa) == R.gelu_constants()
    cq = qk.QuadCoeffs.continuity()
    assert (cq.a0, cq.a1, cq.a2) == CONTINUITY and cq.is_continuity_default()
    assert not qk.QuadCoeffs.minimax().is_continuity_default()
    assert qk.QuadCoeffs(np.float32(1 / 3), np.float32(-0.0), np.float32(2 / 3)).is_continuity_default()
    assert qk.resolve_centering_bias(qk.KernelChoice.Quake, None)
    assert not qk.resolve_centering_bias(qk.KernelChoice.Quake2, None)
    assert qk.resolve_centering_bias(qk.KernelChoice.Quake2, True)
    assert [qk.kernel_name(k) for k in (0, 1, 2)] == ["exact", "quake", "quake2"]


def test_validation_errors_match_reference_messages():
    """Precondition order and messages of kernels.cpp / nonlin.cpp (no GPU reached)."""
    K = qk.KernelChoice
    x = np.zeros(8, np.float32)
    c = qk.natural_exp_coeffs(True)
    r = qk.clamp_for(c)
    cases = [
        (lambda: qk.quake_buffer(x, np.zeros(7, np.float32), c, r), "quake_buffer: output size mismatch"),
        (lambda: qk.quake2_buffer(x, np.zeros(9, np.float32), c, qk.QuadCoeffs.continuity(), r),
         "quake2_buffer: output size mismatch"),
        (lambda: qk.logistic_buffer(x, np.zeros(1, np.float32), K.Quake),
         "logistic_buffer: output size mismatch"),
        (lambda: qk.gelu_buffer(x, np.zeros(1, np.float32), K.Quake2), "gelu_buffer: output size mismatch"),
        (lambda: qk.softmax_rows(np.zeros(5, np.float32), 2, qk.SoftmaxParams(), K.Quake),
         "softmax_rows: length not divisible by cols"),
        (lambda: qk.softmax_rows(x, 0, qk.SoftmaxParams(), K.Quake),
         "softmax_rows: length not divisible by cols"),
        (lambda: qk.softmax_rows(x, 4, qk.SoftmaxParams(), K.Quake, out=np.zeros(4, np.float32)),
         "softmax_rows: output size mismatch"),
        (lambda: qk.softmax_rows(x, 4, qk.SoftmaxParams(temperature=0.0), K.Quake),
         "softmax_rows: temperature must be positive"),
        (lambda: qk.softmax_rows(x, 4, qk.SoftmaxParams(temperature=float("nan")), K.Quake),
         "softmax_rows: temperature must be positive"),
        (lambda: qk.softmax_row(np.zeros(0, np.float32), qk.SoftmaxParams(), K.Exact),
         "softmax: empty row"),
        (lambda: qk.softmax_row(x, qk.SoftmaxParams(temperature=-1.0), K.Exact),
         "softmax_row: temperature must be positive"),
        (lambda: qk.softmax_row(x, qk.SoftmaxParams(), K.Exact, out=np.zeros(3, np.float32)),
         "softmax_row: output size mismatch"),
        (lambda: qk.coeffs_for(0.0, 1.0), "coeffs_for: input scale p must be non-zero"),
        # the fusion-ablation kernels exist for softmax and gelu only
        (lambda: qk.logistic_buffer(x, K.QuakeUnfused), "logistic_buffer: unknown kernel choice"),
        (lambda: qk.default_clamp(0.0, 0.0), "default_clamp: input scale p must be non-zero"),
    ]
    for fn, msg in cases:
        with pytest.raises(qk.QuakeInvalidArgument) as ei:
            fn()
        assert str(ei.value) == msg
        assert isinstance(ei.value, ValueError)


def test_empty_inputs_are_noops():
    """Empty buffers and an empty matrix are valid (kernels.cpp:95-107, nonlin.cpp:162-189)."""
    K = qk.KernelChoice
    e = np.zeros(0, np.float32)
    c = qk.natural_exp_coeffs(True)
    assert qk.quake_buffer(e, c, qk.clamp_for(c)).size == 0
    assert qk.logistic_buffer(e, K.Quake).size == 0
    assert qk.softmax_rows(e, 4, qk.SoftmaxParams(), K.Quake2).size == 0


def test_softmax_plan_geometry():
    p = qk.softmax_plan(512)  # cfg4: 16 lanes per row, 8 float4 chunks each
    assert (p["variant"], p["width"], p["lanes"], p["vpt"]) == (11, 4, 16, 8)
    for cols in (20, 32, 64, 128, 1000, 1024):  # sub-warp rows cover every chunk
        p = qk.softmax_plan(cols)
        assert p["variant"] == 11 and p["lanes"] * p["vpt"] * 4 >= cols, (cols, p)
        assert p["lanes"] & (p["lanes"] - 1) == 0 and 2 <= p["lanes"] <= 32
    for cols, aligned in ((4, True), (16, True), (7, False), (10, False)):
        p = qk.softmax_plan(cols, aligned)  # one thread per row: the sequential order
        assert (p["variant"], p["lanes"]) == (9, 1), (cols, p)
    for cols in (17, 21, 31):  # unaligned 17-32: row spans, float4 chunks
        p = qk.softmax_plan(cols, False)
        assert (p["variant"], p["width"]) == (13, 4), (cols, p)
        assert p["lanes"] * p["vpt"] * 4 >= cols and p["lanes"] & (p["lanes"] - 1) == 0
    p = qk.softmax_plan(13, False)  # unaligned 11-16: one thread per row via smem
    assert (p["variant"], p["lanes"], p["width"]) == (10, 1, 1)
    p = qk.softmax_plan(1100)  # aligned 1025-1536: a full warp per row
    assert (p["variant"], p["lanes"], p["vpt"]) == (11, 32, 12)
    # unaligned 33-28000: per-agent TMA rings, width-1 order; the register form
    # (G lanes per row, vpt elements per lane, a multiple of four, the first
    # vpt-4 full for every lane) up to 1024 columns, above it three sweeps by
    # an agent of lanes/32 warps
    prev = 0
    for cols, g in ((33, 4), (77, 4), (127, 4), (129, 8), (193, 8), (229, 8), (257, 16), (513, 32),
                    (1001, 32), (1025, 0), (2049, 0),
                    (4097, 0), (8191, 0)):
        p = qk.softmax_plan(cols, False)
        assert (p["variant"], p["width"], p["cluster"]) == (14, 1, 1), (cols, p)
        assert p["stages"] in (2, 3), (cols, p)
        if cols <= 1024:
            assert p["lanes"] == g, (cols, p)
            assert p["vpt"] % 4 == 0 and g * (p["vpt"] - 4) < cols <= g * p["vpt"], (cols, p)
        else:  # agents of lanes/32 warps, never smaller for longer rows
            assert p["vpt"] == 0 and p["lanes"] in (32, 64, 128, 256), (cols, p)
            assert p["threads"] % p["lanes"] == 0 and p["lanes"] >= prev, (cols, p)
            prev = p["lanes"]
        assert p["threads"] % 32 == 0 and p["smem"] <= 225 * 1024
    p = qk.softmax_plan(1 << 23)
    assert p["variant"] == 3
    for cols in (2048, 4096, 16384, 50000, 65536, 128256, 300000):
        p = qk.softmax_plan(cols)
        assert p["variant"] == 4 and p["balanced"] == 1, (cols, p)
        chunks = cols // 4
        q, rem = divmod(chunks, p["cluster"])
        assert p["slice"] == q + (1 if rem else 0)
        # every thread owns KC-1 unconditional chunks, the last predicated
        assert p["threads"] % 32 == 0 and p["threads"] <= 512
        assert p["threads"] * (p["vpt"] - 1) <= q <= p["threads"] * p["vpt"]
        assert p["stages"] >= 2 and p["smem"] <= 227 * 1024
    # the plan follows the kernel's weight: at one CTA per row the light kinds
    # take the fewest, fullest warps, the heavier ones the most warps
    K = qk.KernelChoice
    light = qk.softmax_plan(16384, True, K.Quake)
    heavy = qk.softmax_plan(16384, True, K.Quake2)
    assert (light["cluster"], light["threads"], light["vpt"]) == (1, 256, 16)
    assert (heavy["cluster"], heavy["threads"], heavy["vpt"]) == (1, 512, 8)
    assert qk.softmax_plan(16384, True, K.FastExp)["threads"] == 256
    assert qk.softmax_plan(16384, True, K.Quake2Unfused)["threads"] == 512
    assert qk.softmax_plan(16384, True, K.QuakeUnfused)["threads"] == 256
    for cols in (1025, 600000):
        p = qk.softmax_plan(cols)
        if p["variant"] == 2:
            assert p["slice"] * p["cluster"] * p["width"] >= cols
            assert p["smem"] <= 227 * 1024


def test_warp_ring_plans_cover_every_unaligned_length():
    """Every row length of cols % 4 != 0 in 33..28000 gets a warp-ring plan the
    launcher accepts: an instantiated (lanes, vpt) pair whose unpredicated slots
    exist and which covers the row, or a three-sweep agent of 1-8 warps; rings
    of 2-3 buffers of whole jobs that fit a CTA's shared memory."""
    regs = {(4, v) for v in (12, 16, 20, 24, 28, 32)} | {(g, v) for g in (8, 16, 32)
                                                         for v in (20, 24, 28, 32)}
    K = qk.KernelChoice
    lengths = [c for c in list(range(33, 1100)) + list(range(1100, 28001, 37)) + [27999, 28000]
               if c % 4]
    for cols in lengths:
        for kern in (K.Quake, K.Quake2):
            p = qk.softmax_plan(cols, False, kern)
            assert (p["variant"], p["width"], p["cluster"]) == (14, 1, 1), (cols, p)
            if p["vpt"]:
                assert cols <= 1024 and (p["lanes"], p["vpt"]) in regs, (cols, p)
                assert p["lanes"] * (p["vpt"] - 4) < cols <= p["lanes"] * p["vpt"], (cols, p)
            else:
                assert cols > 1024 and p["lanes"] in (32, 64, 128, 256), (cols, p)
                assert p["threads"] % p["lanes"] == 0, (cols, p)
            assert p["stages"] in (2, 3) and 32 <= p["threads"] <= 256 and p["threads"] % 32 == 0
            # agents * buffers * (rows per job * cols + 8 floats, rounded to 32 floats)
            agents = p["threads"] // (p["lanes"] if not p["vpt"] else 32)
            per_buf = p["smem"] // (agents * p["stages"])
            assert per_buf * agents * p["stages"] == p["smem"] and per_buf % 128 == 0
            assert per_buf >= (cols + 8) * 4 and p["smem"] <= 225 * 1024, (cols, p)
    assert qk.softmax_plan(28001, False)["variant"] != 14
    assert qk.softmax_plan(29, False)["variant"] == 13


def test_cuda_calls_fail_loudly_without_gpu():
    import torch
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    K = qk.KernelChoice
    with pytest.raises(qk.QuakeCudaError):
        qk.logistic_buffer(np.ones(16, np.float32), K.Quake)


def test_kernel_names_and_unfused_bias_resolution():
    K = qk.KernelChoice
    names = {K.Exact: "exact", K.Quake: "quake", K.Quake2: "quake2", K.Expf: "expf",
             K.FastExp: "fast_expf", K.QuakeUnfused: "quake_unfused",
             K.Quake2Unfused: "quake2_unfused"}
    for k, name in names.items():
        assert qk.kernel_name(k) == name
    # the unfused ablation kernels resolve the centering bias as their QuAKE body
    assert qk.resolve_centering_bias(K.QuakeUnfused, None) is True
    assert qk.resolve_centering_bias(K.Quake2Unfused, None) is False
    assert qk.resolve_centering_bias(K.Quake2Unfused, True) is True


def test_coeffs_for_takes_the_reference_format_argument():
    """kernels.hpp:50-51, 89: coeffs_for(p, q, fmt = kSingle, bias) and
    default_clamp(p, q, fmt = kSingle); the derivation follows fmt's mantissa
    width and exponent bias (kernels.cpp:30-39, 74-82), computed in binary64."""
    import math
    import struct

    def f32(v):
        return struct.unpack("<f", struct.pack("<f", v))[0]

    p = f32(math.log2(math.e))
    a = qk.coeffs_for(p, 0.0, qk.kSingle, True)
    b = qk.coeffs_for(p, 0.0, True)
    assert (a.c0, a.c1) == (b.c0, b.c1) == (f32(2.0**23 * p), f32(2.0**23 * (127 - 0.0436)))
    half = qk.FpFormat(5, 10, 15)
    h = qk.coeffs_for(0.7, 0.25, half, False)
    assert h.c0 == f32(1024.0 * f32(0.7)) and h.c1 == f32(1024.0 * (15 + 0.25))
    r = qk.default_clamp(1.0, 0.0, half)
    lo = (1.01 * 1024 - 1024 * 15) / 1024.0
    hi = (254.99 * 1024 - 1024 * 15) / 1024.0
    assert (r.lo, r.hi) == (f32(lo), f32(hi))
    assert qk.default_clamp(1.0, 0.0) == qk.default_clamp(1.0, 0.0, qk.kSingle)
    with pytest.raises(ValueError, match="input scale p must be non-zero"):
        qk.coeffs_for(0.0, 1.0, half)
    with pytest.raises(ValueError, match="input scale p must be non-zero"):
        qk.default_clamp(0.0, 0.0, half)
