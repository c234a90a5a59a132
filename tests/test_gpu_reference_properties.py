"""The reference's property tests (tests/test_nonlin.cpp), run on the GPU path.

Same distributions, sizes and bounds as the reference cases (numpy's PCG64 in
place of std::mt19937, so the sampled values differ); exact references are
binary64 numpy or the GPU's own Exact kernel where the reference compares
against its Exact kernel.
"""
import numpy as np
import pytest
import torch

import paper_2412_00408_b200 as qk

pytestmark = pytest.mark.gpu
K = qk.KernelChoice
EPS = np.float32(1.1920928955078125e-07)


def softmax64(m):
    m = np.asarray(m, np.float64)
    e = np.exp(m - m.max(axis=-1, keepdims=True))
    return e / e.sum(axis=-1, keepdims=True)


def gpu_rows(x, cols, kernel, t=1.0):
    xd = torch.from_numpy(np.ascontiguousarray(x, np.float32).ravel()).cuda()
    return qk.softmax_rows(xd, cols, qk.SoftmaxParams(temperature=t), kernel).cpu().numpy()


def test_softmax_of_0_ln2_exact():
    """test_nonlin.cpp: softmax of [0, ln2] with the exact kernel."""
    y = qk.softmax_row(np.array([0.0, np.log(2.0)], np.float32), qk.SoftmaxParams(), K.Exact)
    assert abs(y[0] - 1 / 3) <= 1e-6 * (1 / 3) and abs(y[1] - 2 / 3) <= 1e-6 * (2 / 3)


def test_first_order_softmax_within_secant_envelope():
    """test_nonlin.cpp: |y - exact| <= 0.0634 * max(exact) + 1e-7 per element."""
    rng = np.random.default_rng(41)
    v = rng.uniform(-6, 6, (64, 256)).astype(np.float32)
    y = gpu_rows(v, 256, K.Quake).reshape(64, 256)
    ex = softmax64(v)
    assert np.all(np.abs(y - ex) <= 0.0634 * ex.max(axis=1, keepdims=True) + 1e-7)


def test_softmax_shift_behavior():
    """test_nonlin.cpp: sixteenths shifted by quarters (exact inputs): Exact within
    2 ulp, QuAKE within 1e-5."""
    rng = np.random.default_rng(47)
    by_n = {}
    for _ in range(500):
        n = int(2 + rng.integers(0, 48))
        v = rng.integers(-64, 65, n).astype(np.float32) / 16
        shift = np.float32(rng.integers(-64, 65) / 4)
        by_n.setdefault(n, []).append((v, v + shift))
    for n, pairs in by_n.items():
        a_in = np.stack([p[0] for p in pairs])
        b_in = np.stack([p[1] for p in pairs])
        a = gpu_rows(a_in, n, K.Exact).reshape(-1, n)
        b = gpu_rows(b_in, n, K.Exact).reshape(-1, n)
        assert np.all(np.abs(a - b) <= 2 * np.spacing(a)), n
        a = gpu_rows(a_in, n, K.Quake).reshape(-1, n)
        b = gpu_rows(b_in, n, K.Quake).reshape(-1, n)
        assert np.all(np.abs(a - b) <= 1e-5), n


def test_gelu_sign_structure():
    """test_nonlin.cpp: sign and lower bound of GELU for all three kernels."""
    x = np.random.default_rng(61).uniform(-10, 10, 100_000).astype(np.float32)
    pos, neg = x >= 0, x < 0
    for k, slack in ((K.Exact, 0.0), (K.Quake, 1e-4), (K.Quake2, 1e-4)):
        y = qk.gelu_buffer(x, k)
        assert np.all(y[pos] >= 0)
        assert np.all(y[neg] <= 0)
        assert np.all(y[neg] >= 0.5 * x[neg] - np.float32(slack))


def test_second_order_beats_first_order():
    """test_nonlin.cpp: QuAKE2's max deviation from Exact is below QuAKE's for GELU,
    logistic and softmax."""
    rng = np.random.default_rng(71)
    x = rng.uniform(-8, 8, 100_000).astype(np.float32)
    for op in (qk.gelu_buffer, qk.logistic_buffer):
        ex = op(x, K.Exact).astype(np.float64)
        d1 = np.max(np.abs(op(x, K.Quake) - ex))
        d2 = np.max(np.abs(op(x, K.Quake2) - ex))
        assert d2 < d1, op.__name__
    v = rng.uniform(-6, 6, (1600, 64)).astype(np.float32)
    ex = softmax64(v)
    d1 = np.max(np.abs(gpu_rows(v, 64, K.Quake).reshape(1600, 64) - ex))
    d2 = np.max(np.abs(gpu_rows(v, 64, K.Quake2).reshape(1600, 64) - ex))
    assert d2 < d1


def test_softmax_rows_normalize_within_4n_ulps():
    """test_nonlin.cpp: every kernel, n up to 65536, t in {0.25, 1, 4}: outputs
    non-negative, sum within 4 n eps of 1 (fp32 sequential sum)."""
    rng = np.random.default_rng(53)
    for trial in range(60):
        n = int(1 + rng.integers(0, 65536))
        v = rng.uniform(-50, 50, n).astype(np.float32)
        t = (0.25, 1.0, 4.0)[trial % 3]
        for k in (K.Exact, K.Quake, K.Quake2):
            y = qk.softmax_row(v, qk.SoftmaxParams(temperature=t), k)
            assert np.all(y >= 0)
            s = np.cumsum(y, dtype=np.float32)[-1]  # sequential fp32 sum, as the reference
            assert abs(float(s) - 1.0) <= 4.0 * n * float(EPS), (trial, n, t, k)
