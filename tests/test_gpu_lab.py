"""§8(f3) GPU accuracy lab (include/quake_b200_lab.h) against the reference lab.

Parity: every report of the reference's own lab (core/src/lab.cpp, values in
tests/golden/reference_lab.json from make_lab_golden.py) is reproduced — the
approximations are bit-identical, only the binary64 ground truth comes from
the device libm (<= 1 ulp of binary64), so maxima agree to ~1e-15 relative.
Then the reference's unit-test bands (tests/test_lab.cpp) and acceptance
criteria 1-6 (tests/acceptance.cpp:65-172) on the GPU — c1 and c3 reproduce
the reference's recorded values, which miss its own bands the same way
(proj/test_output.txt:8-13) — and the exhaustive every-binary32 sweeps.
"""
import json
import os

import numpy as np
import pytest

import paper_2412_00408_b200 as qk
from paper_2412_00408_b200 import KernelChoice as K
from paper_2412_00408_b200 import lab

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLD = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_lab.json")))
KINDS = {0: K.Exact, 1: K.Quake, 2: K.Quake2}
ULP_REL = 1e-12  # device vs host binary64 exp: relative agreement of the error figures


def cfg_of(v):
    return lab.ExpConfig(KINDS[v["kind"]], v["natural"], v["bias"], lab.QuadCoeffs(*v["quad"]))


@pytest.mark.parametrize("name", sorted(GOLD["sweeps"]))
def test_sweep_error_matches_reference(name):
    v = GOLD["sweeps"][name]
    r = lab.sweep_error(cfg_of(v), lab.SweepSpec(**v["spec"]))
    assert r.samples == v["samples"]
    assert abs(r.max_rel_err - v["max_rel_err"]) <= ULP_REL * v["max_rel_err"]
    assert np.float32(r.argmax_input) == np.float32(v["argmax_input"])
    assert abs(r.mean_rel_err - v["mean_rel_err"]) <= 1e-9 * v["mean_rel_err"]
    assert r.lo == v["spec"]["lo"] and r.hi == v["spec"]["hi"]


@pytest.mark.parametrize("name", sorted(GOLD["continuity"]))
def test_continuity_probe_matches_reference(name):
    v = GOLD["continuity"][name]
    r = lab.continuity_probe(cfg_of(v), v["k_lo"], v["k_hi"])
    assert r.worst_jump == v["worst_jump"]
    assert np.float32(r.at) == np.float32(v["at"])


def test_quad_and_grid_search_match_reference():
    for v in GOLD["quad"].values():
        got = lab.quad_max_rel_err(*v["a"], v["intervals"])
        assert abs(got - v["value"]) <= ULP_REL * v["value"]
    for name, v in GOLD["grid"].items():
        a = v["axes"]
        g = lab.grid_search_quad(lab.GridSpec(lab.GridAxis(*a[0:3]), lab.GridAxis(*a[3:6]),
                                              lab.GridAxis(*a[6:9])))
        assert [np.float32(g.best.a0), np.float32(g.best.a1), np.float32(g.best.a2)] == \
            [np.float32(b) for b in v["best"]], name
        assert abs(g.best_max_rel_err - v["best_max_rel_err"]) <= ULP_REL * v["best_max_rel_err"]
        assert g.points_searched == v["points"]


def test_bias_reoptimize_matches_reference():
    for v in GOLD["bias"].values():
        b = lab.bias_reoptimize(lab.ExpConfig(KINDS[v["kind"]], v["natural"], v["bias"]))
        assert abs(b.beta - v["beta"]) <= 2e-6
        assert abs(b.max_rel_err - v["max_rel_err"]) <= 1e-9
        assert b.near_reference_bias == v["near"]


def test_reference_unit_test_bands():
    """tests/test_lab.cpp:35-103 on the GPU lab."""
    unit = lab.SweepSpec(-80.0, 80.0, 1 << 20, 8)
    r = lab.sweep_error(lab.ExpConfig(K.Quake, True, True), unit)
    assert 0.0295 <= r.max_rel_err <= 0.0302 and 0 < r.mean_rel_err <= r.max_rel_err
    assert r.kernel == "quake" and r.lo <= r.argmax_input <= r.hi
    r = lab.sweep_error(lab.ExpConfig(K.Quake, True, False), unit)
    assert 0.0610 <= r.max_rel_err <= 0.0620
    r = lab.sweep_error(lab.ExpConfig(K.Quake2, True, False), unit)
    assert 0.0033 <= r.max_rel_err <= 0.0035
    r = lab.sweep_error(lab.ExpConfig(K.Exact, False), lab.SweepSpec(0.0, 1.0, 100_000, 0))
    assert r.max_rel_err == 0.0 and r.mean_rel_err == 0.0
    spec = lab.SweepSpec(-20.0, 20.0, 1 << 18, 16)
    a = lab.sweep_error(lab.ExpConfig(K.Quake2, True, False), spec)
    assert a == lab.sweep_error(lab.ExpConfig(K.Quake2, True, False), spec)  # reproducible
    r = lab.sweep_error(lab.ExpConfig(K.Quake2, False, False), lab.SweepSpec(0.0, 1.0, 1 << 20, 1))
    assert abs(r.max_rel_err - lab.quad_max_rel_err(1 / 3, 0.0, 2 / 3, 1 << 20)) <= 1e-5
    # continuity (test_lab.cpp:158-170): endpoint-exact kernels are continuous,
    # the grid-search optimum keeps a genuine ~1% step
    assert lab.continuity_probe(lab.ExpConfig(K.Quake, False, False), -50, 50).worst_jump <= 1e-5
    assert lab.continuity_probe(lab.ExpConfig(K.Quake2, False, False), -50, 50).worst_jump <= 1e-5
    j = lab.continuity_probe(lab.ExpConfig(K.Quake2, False, False, qk.QuadCoeffs.minimax()),
                             -50, 50).worst_jump
    assert 0.005 <= j <= 0.02


def test_acceptance_criteria_1_to_6():
    acc = lab.SweepSpec(-80.0, 80.0, 1 << 22, 1)
    # c1: the reference records 0.029883 (FAIL of its [0.042, 0.044] band); reproduced
    r1 = lab.sweep_error(lab.ExpConfig(K.Quake, True, True), acc)
    assert abs(r1.max_rel_err - 0.029883) < 5e-7 and r1.samples == 12582912
    # c2: [0.30%, 0.35%]
    r2 = lab.sweep_error(lab.ExpConfig(K.Quake2, True, False), acc)
    assert 0.0030 <= r2.max_rel_err <= 0.0035
    # c3: the reference records best=(0.336, -0.012, 0.677) err=0.001966 (FAIL of
    # [0.0015, 0.0019]); reproduced, coordinates within its 0.005 window except a1
    g = lab.grid_search_quad()
    assert (round(float(g.best.a0), 6), round(float(g.best.a1), 6),
            round(float(g.best.a2), 6)) == (0.336, -0.012, 0.677)
    assert abs(g.best_max_rel_err - 0.001966) < 5e-7
    # c4: beta in [0.040, 0.047]; the unbiased kernel's error in [5.8%, 6.4%]
    b = lab.bias_reoptimize(lab.ExpConfig(K.Quake, True, True))
    assert 0.040 <= b.beta <= 0.047 and b.near_reference_bias
    r4 = lab.sweep_error(lab.ExpConfig(K.Quake, True, False), acc)
    assert 0.058 <= r4.max_rel_err <= 0.064
    # c5: exact at integer powers of two (GPU quake/quake2 buffers) + continuity
    b2 = qk.base2_coeffs(False)
    rr = qk.clamp_for(b2)
    ks = np.arange(-100, 101, dtype=np.float32)
    want = np.ldexp(np.float32(1.0), np.arange(-100, 101)).astype(np.float32)
    assert np.array_equal(qk.quake_buffer(ks, b2, rr), want)
    assert np.array_equal(qk.quake2_buffer(ks, b2, qk.QuadCoeffs.continuity(), rr), want)
    for kind in (K.Quake, K.Quake2):
        assert lab.continuity_probe(lab.ExpConfig(kind, False, False), -100, 100).worst_jump <= 1e-5
    # c6: monotonicity — every consecutive pair of binary32 inputs across the whole
    # clamp range (the reference samples 10^6 random pairs)
    for kind in (K.Quake, K.Quake2):
        cfg = lab.ExpConfig(kind, True, True)
        _, r = cfg.coeffs_and_clamp()
        ex = lab.sweep_exhaustive(cfg, r.lo, r.hi)
        assert ex.monotonic_violations == 0 and ex.non_positive == 0


@pytest.mark.parametrize("kind,natural,bias,quad", [
    (K.Quake, True, True, None), (K.Quake, True, False, None), (K.Quake2, True, False, None),
    (K.Quake2, True, True, None), (K.Quake, False, False, None), (K.Quake2, False, False, None),
    (K.Quake2, True, False, "minimax")])
def test_exhaustive_every_binary32(kind, natural, bias, quad):
    """Full fp32 resolution over [-80, 80] (inside every clamp range): the band the
    sampled sweep reports is the true maximum up to sampling; monotone and positive."""
    q = qk.QuadCoeffs.minimax() if quad else qk.QuadCoeffs.continuity()
    cfg = lab.ExpConfig(kind, natural, bias, q)
    lo, hi = (-80.0, 80.0) if natural else (-120.0, 120.0)
    ex = lab.sweep_exhaustive(cfg, lo, hi)
    n_floats = int(np.float32(hi).view(np.uint32)) + int(np.float32(-lo).view(np.uint32)) + 2
    assert ex.samples == n_floats
    assert ex.monotonic_violations == 0 and ex.non_positive == 0
    sampled = lab.sweep_error(cfg, lab.SweepSpec(lo, hi, 1 << 20, 8))
    assert sampled.max_rel_err <= ex.max_rel_err <= sampled.max_rel_err * 1.001
    assert lo <= ex.argmax_input <= hi
