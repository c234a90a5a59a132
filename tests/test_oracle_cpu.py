"""CPU: pin the oracle (C restatement) before trusting it.

* against the reference's golden vectors (tests/golden/reference_vectors.npz,
  produced by the reference's own entry points, see make_golden.py);
* against the reference's in-test known answers (test_kernels.cpp:35-131,
  test_nonlin.cpp:206-288) and SURVEY.md Appendix A.3 bit patterns;
* against the reference compiled in place (oracle/_ref), when present.
Paths relative to /root/reference/proj/.
"""
import os

import numpy as np
import pytest

from oracle.oracle import CONTINUITY, EXACT, MINIMAX, QUAKE, QUAKE2
from tests.helpers import assert_bitexact, bits, reference, restatement

GOLDEN = os.path.join(os.path.dirname(__file__), "golden", "reference_vectors.npz")
LOG2E = np.float32(1.4426950408889634)


@pytest.fixture(scope="module")
def golden():
    return np.load(GOLDEN)


def test_golden_elementwise(golden):
    R = restatement()
    x = golden["x"]
    for name in ("natural_bias", "natural_nobias", "base2", "negated_bias"):
        c0, c1, lo, hi = golden[f"coeffs_{name}"]
        assert_bitexact(R.quake_buffer(x, c0, c1, lo, hi), golden[f"quake_{name}"], name)
        assert_bitexact(R.quake2_buffer(x, c0, c1, CONTINUITY, lo, hi), golden[f"quake2_{name}"],
                        name)
        assert_bitexact(R.quake2_buffer(x, c0, c1, MINIMAX, lo, hi), golden[f"quake2mm_{name}"],
                        name)
    for k, kn in ((EXACT, "exact"), (QUAKE, "quake"), (QUAKE2, "quake2")):
        for b, bn in ((-1, "default"), (0, "off"), (1, "on")):
            if f"logistic_{kn}_{bn}" not in golden:
                continue
            assert_bitexact(R.logistic_buffer(x, k, b), golden[f"logistic_{kn}_{bn}"], kn + bn)
            assert_bitexact(R.gelu_buffer(x, k, b), golden[f"gelu_{kn}_{bn}"], kn + bn)
    assert_bitexact(np.array(R.gelu_constants(), np.float32), golden["gelu_constants"], "gelu")


def test_golden_softmax(golden):
    R = restatement()
    for key in [k[:-3] for k in golden.files if k.startswith("softmax_") and k.endswith("_in")]:
        m = golden[key + "_in"]
        rows, cols = (int(v) for v in key.split("_")[1].split("x"))
        t = float(key.split("_t")[1])
        for k, kn in ((EXACT, "exact"), (QUAKE, "quake"), (QUAKE2, "quake2")):
            assert_bitexact(R.softmax_rows(m, cols, t, k), golden[f"{key}_{kn}"], key + kn)


def test_appendix_a3_constants():
    """SURVEY.md A.3 bit patterns (extracted from the reference library)."""
    R = restatement()
    want = {  # (p, bias) -> c0, c1, lo, hi
        (LOG2E, 1): (0x4B38AA3B, 0x4E7DE9AD, 0xC2AE994A, 0x42B17E05),
        (LOG2E, 0): (0x4B38AA3B, 0x4E7E0000, 0xC2AEA8C3, 0x42B16E8C),
        (-LOG2E, 1): (0xCB38AA3B, 0x4E7DE9AD, 0xC2B17E05, 0x42AE994A),
        (-LOG2E, 0): (0xCB38AA3B, 0x4E7E0000, 0xC2B16E8C, 0x42AEA8C3),
    }
    for (p, bias), w in want.items():
        c0, c1 = R.coeffs_for(p, 0.0, bias)
        lo, hi = R.clamp_for(c0, c1)
        assert [int(v) for v in bits(np.array([c0, c1, lo, hi]))] == list(w)
    kappa, r2pi, fs, ik = R.gelu_constants()
    assert int(bits(np.array([fs]))[0]) == 0x3D922279
    assert int(bits(np.array([ik]))[0]) == 0x41B2E92F
    gp = np.float32(-1.4426950408889634 * float(fs))
    assert int(bits(np.array([gp]))[0]) == 0xBDD2D3E7
    for bias, w in ((1, (0xC952D3E7, 0x4E7DE9AD, 0xC49B775D, 0x4498EE8E)),
                    (0, (0xC952D3E7, 0x4E7E0000, 0xC49B69CF, 0x4498FC1C))):
        c0, c1 = R.coeffs_for(gp, 0.0, bias)
        lo, hi = R.clamp_for(c0, c1)
        assert [int(v) for v in bits(np.array([c0, c1, lo, hi]))] == list(w)
    # known answers
    cb = R.coeffs_for(LOG2E, 0.0, 1)
    rb = R.clamp_for(*cb)
    cn = R.coeffs_for(LOG2E, 0.0, 0)
    rn = R.clamp_for(*cn)
    kat = {-10: (0x3843C500, 0x383EE960), -1: (0x3EC1C100, 0x3EBCCEF3), 0: (0x3F7A6B40, 0x3F800000),
           0.5: (0x3FD6C040, 0x3FD3C178), 1: (0x40331580, 0x402E2335),
           3.3: (0x41DBD000, 0x41D9A1CC), 10: (0x46B11180, 0x46AC361C)}
    for x, (q1, q2) in kat.items():
        assert int(bits(np.array([R.quake(x, *cb, *rb)]))[0]) == q1
        assert int(bits(np.array([R.quake2(x, *cn, CONTINUITY, *rn)]))[0]) == q2
    xs = np.array([-3, 0, 0.7, 2], np.float32)
    assert list(bits(R.logistic_buffer(xs, QUAKE))) == [0x3D3E0DDA, 0x3F016920, 0x3F2C33AC, 0x3F61C637]
    assert list(bits(R.logistic_buffer(xs, QUAKE2))) == [0x3D425DDF, 0x3F000000, 0x3F2B0AA4, 0x3F6187FC]
    assert list(bits(R.gelu_buffer(xs, QUAKE))) == [0xBB6983A2, 0, 0x3F070096, 0x3FFA0764]
    assert list(bits(R.gelu_buffer(xs, QUAKE2))) == [0xBB6D95E6, 0, 0x3F07D5B6, 0x3FFA2C88]
    # softmax c0 / v_min offsets
    c0, _, vmin = R.softmax_row_scalars(np.float32(0.0), np.float32(0.125), 0)
    assert int(bits(np.array([c0]))[0]) == 0x49B8AA3B


def test_reference_test_kats():
    """test_kernels.cpp:35-92 and :106-131."""
    R = restatement()
    c0, c1 = R.coeffs_for(LOG2E, 0.0, 1)
    assert abs(float(c0) - 12102203.16) <= 12102203.16 * 1e-6
    assert abs(float(c1) - 1064987472.7) <= 1064987472.7 * 1e-7
    b2 = R.coeffs_for(1.0, 0.0, 0)
    assert b2 == (np.float32(8388608.0), np.float32(1065353216.0))
    rb = R.clamp_for(*b2)
    assert R.quake(0.5, *b2, *rb) == np.float32(1.5)
    assert R.quake(3.0, *b2, *rb) == np.float32(8.0)
    assert R.quake2(0.5, *b2, CONTINUITY, *rb) == (np.float32(1.5) ** 2 + np.float32(2)) / np.float32(3)
    for k in range(-100, 101):
        assert R.quake(k, *b2, *rb) == np.float32(2.0) ** k
        assert R.quake2(k, *b2, CONTINUITY, *rb) == np.float32(2.0) ** k
    with pytest.raises(ValueError):
        R.coeffs_for(0.0, 1.0)
    e = R.default_clamp(LOG2E)
    assert abs(float(e[0]) + 87.33) <= 87.33 * 2e-4 and e[1] > 88
    n = R.default_clamp(-LOG2E)
    assert n[0] == -e[1] and n[1] == -e[0]
    ne = R.coeffs_for(LOG2E, 0.0, 1)
    r = R.clamp_for(*ne)
    q = lambda v: R.quake(v, *ne, *r)
    assert q(r[0] - 50) == q(r[0]) and q(r[1] + 50) == q(r[1])
    assert q(-np.inf) == q(r[0]) and q(np.inf) == q(r[1]) and q(np.nan) == q(r[1])


def test_div3_replacement_exhaustive():
    """The device's (am^2+2)/3 = reciprocal multiply + FMA correction, proven equal to the
    IEEE quotient over every binary32 t in [3, 6] (numerics.cuh refine_default)."""
    assert restatement().check_div3_replacement() == 0


@pytest.mark.skipif(reference() is None, reason="reference not compiled here")
def test_restatement_matches_compiled_reference_random_bits():
    R, F = restatement(), reference()
    rng = np.random.default_rng(11)
    x = rng.integers(0, 2**32, size=1 << 20, dtype=np.uint64).astype(np.uint32).view(np.float32)
    for p, q in ((LOG2E, 0.0), (1.0, 0.0), (0.7, 0.37), (3.0, 0.0)):
        for bias in (0, 1):
            c = F.coeffs_for(p, q, bias)
            assert c == R.coeffs_for(p, q, bias)
            for r in (F.clamp_for(*c), (np.float32(-1e30), np.float32(1e30))):
                assert_bitexact(R.quake_buffer(x, *c, *r), F.quake_buffer(x, *c, *r))
                assert_bitexact(R.quake2_buffer(x, *c, CONTINUITY, *r),
                                F.quake2_buffer(x, *c, CONTINUITY, *r))
                assert_bitexact(R.quake2_buffer(x, *c, MINIMAX, *r),
                                F.quake2_buffer(x, *c, MINIMAX, *r))
    for k in (EXACT, QUAKE, QUAKE2):
        for b in (-1, 0, 1):
            assert_bitexact(R.logistic_buffer(x, k, b), F.logistic_buffer(x, k, b))
            assert_bitexact(R.gelu_buffer(x, k, b), F.gelu_buffer(x, k, b))


@pytest.mark.slow
@pytest.mark.skipif(reference() is None, reason="reference not compiled here")
def test_restatement_matches_compiled_reference_strided_exhaustive():
    """Every 64th binary32 bit pattern (2^26 inputs, all exponents, signs, NaN
    and infinity classes) for the six exhaustively GPU-swept variants:
    restatement == compiled reference. (The GPU sweep itself compares every
    one of the 2^32 patterns against the reference directly.)"""
    R, F = restatement(), reference()
    x = (np.arange(0, 1 << 26, dtype=np.uint64) * 64 + 37).astype(np.uint32).view(np.float32)
    for bias, quad_kernel in ((1, QUAKE), (0, QUAKE2)):
        c0, c1 = F.named_coeffs("natural", bias == 1)
        lo, hi = F.clamp_for(c0, c1)
        if quad_kernel == QUAKE:
            assert_bitexact(R.quake_buffer(x, c0, c1, lo, hi), F.quake_buffer(x, c0, c1, lo, hi))
        else:
            assert_bitexact(R.quake2_buffer(x, c0, c1, CONTINUITY, lo, hi),
                            F.quake2_buffer(x, c0, c1, CONTINUITY, lo, hi))
    for k in (QUAKE, QUAKE2):
        assert_bitexact(R.logistic_buffer(x, k), F.logistic_buffer(x, k))
        assert_bitexact(R.gelu_buffer(x, k), F.gelu_buffer(x, k))


@pytest.mark.skipif(reference() is None, reason="reference not compiled here")
def test_restatement_matches_compiled_reference_softmax():
    R, F = restatement(), reference()
    rng = np.random.default_rng(12)
    for cols, rows in ((512, 64), (3, 100), (1, 7), (4099, 3), (128256, 2)):
        m = (rng.standard_normal(rows * cols) * 4).astype(np.float32)
        for k in (EXACT, QUAKE, QUAKE2):
            for t in (0.125, 1.0, 4.0):
                for quad in (CONTINUITY, MINIMAX):
                    assert_bitexact(R.softmax_rows(m, cols, t, k, quad=quad),
                                    F.softmax_rows(m, cols, t, k, quad=quad), f"{cols} {k} {t}")
    # error behaviour: non-finite, bad temperature, non-divisible
    for bad, msg in (([1.0, np.nan], "non-finite"),):
        with pytest.raises(ValueError, match=msg):
            F.softmax_rows(np.array(bad, np.float32), 2)
        with pytest.raises(ValueError):
            R.softmax_rows(np.array(bad, np.float32), 2)


def test_ordered_restatement_is_a_reordering_only():
    """or_softmax_rows_ordered differs from the sequential sum only by summation order:
    with an integer-valued exact case (all-equal rows) both agree bit-for-bit, and on random
    rows they agree within the 2e-6 softmax tolerance."""
    R = restatement()
    plan = {"width": 4, "lanes": 32, "cluster": 1, "slice": 0}
    m = np.zeros(8 * 512, np.float32)
    assert_bitexact(R.softmax_rows_ordered(m, 512, plan, 1.0, QUAKE2),
                    R.softmax_rows(m, 512, 1.0, QUAKE2), "constant rows")
    m = (np.random.default_rng(1).standard_normal(64 * 512) * 2).astype(np.float32)
    a = R.softmax_rows_ordered(m, 512, plan, 0.125, QUAKE)
    b = R.softmax_rows(m, 512, 0.125, QUAKE)
    assert np.max(np.abs(a.astype(np.float64) - b) / b) <= 2e-6
    cplan = {"width": 4, "lanes": 512, "cluster": 8, "slice": 4008}
    m = (np.random.default_rng(2).standard_normal(2 * 128256) * 4).astype(np.float32)
    a = R.softmax_rows_ordered(m, 128256, cplan, 1.0, QUAKE2)
    b = R.softmax_rows(m, 128256, 1.0, QUAKE2, sum_mode=1)
    assert np.max(np.abs(a.astype(np.float64) - b) / b) <= 2e-6


@pytest.mark.skipif(reference() is None, reason="reference not compiled here")
def test_unfused_restatement_pinned_to_reference_fusion_ablation():
    """The ablation's unfused passes (bench.cpp:137-166, 212-233), restated as kernel ids
    QUAKE_UNFUSED / QUAKE2_UNFUSED, reproduce the reference's own fusion_ablation
    checksums exactly (sum of outputs in fp64, bench.cpp:309-313) — and so do the fused
    passes through the regular softmax / gelu restatement — on the reference's inputs."""
    from oracle.oracle import QUAKE2_UNFUSED, QUAKE_UNFUSED
    R, F = restatement(), reference()

    def checksum(y):
        s = 0.0
        for v in np.asarray(y, np.float64):
            s += v
        return s

    for kern, unf in ((QUAKE, QUAKE_UNFUSED), (QUAKE2, QUAKE2_UNFUSED)):
        for rows, cols, t, seed in ((37, 1000, 0.7, 42), (5, 4096, 1.0, 7), (64, 33, 0.125, 3)):
            x = F.bench_inputs("softmax_matrix", rows * cols, seed)
            fc, uc, div = F.fusion_ablation("softmax_matrix", kern, rows, cols, 0, t, seed)
            yf = R.softmax_rows(x, cols, t, kern, sum_mode=0)
            yu = R.softmax_rows(x, cols, t, unf, sum_mode=0)
            assert checksum(yf) == fc and checksum(yu) == uc, (kern, rows, cols, t)
            rel = np.abs(yf.astype(np.float64) - yu) / np.maximum(np.abs(yf), np.abs(yu))
            assert rel.max() == div
        for n, seed in ((100003, 42), (4099, 9)):
            x = F.bench_inputs("gelu_vector", n, seed)
            fc, uc, div = F.fusion_ablation("gelu_vector", kern, 0, 0, n, 1.0, seed)
            yf, yu = R.gelu_buffer(x, kern), R.gelu_buffer(x, unf)
            assert checksum(yf) == fc and checksum(yu) == uc, (kern, n)
            a, b = yf.astype(np.float64), yu.astype(np.float64)
            den = np.maximum(np.abs(a), np.abs(b))
            rel = np.where(den > 0, np.abs(a - b) / np.where(den > 0, den, 1), 0)
            assert rel.max() == div
