"""§8(f2) GPU fusion ablation: the unfused kernels (bench.cpp:137-166 softmax,
212-233 GELU) bit-exact against the restatement — itself pinned to the
reference's own fusion_ablation checksums (test_oracle_cpu) — and the
harness (paper_2412_00408_b200/ablation.py, mirroring bench.cpp:286-513)."""
import numpy as np
import pytest
import torch

import paper_2412_00408_b200 as qk
from oracle.oracle import QUAKE, QUAKE2, QUAKE2_UNFUSED, QUAKE_UNFUSED
from paper_2412_00408_b200 import ablation as ab
from tests.helpers import assert_bitexact, restatement

pytestmark = pytest.mark.gpu
K = qk.KernelChoice


@pytest.mark.parametrize("cols", [33, 197, 512, 700, 1537, 4096, 4099, 16384, 128256, 262144])
@pytest.mark.parametrize("kern", [QUAKE_UNFUSED, QUAKE2_UNFUSED])
def test_unfused_softmax_bitexact(cols, kern):
    R = restatement()
    rows = max(2, min(48, (1 << 21) // cols))
    rng = np.random.default_rng(cols + kern)
    x = rng.uniform(-8, 8, rows * cols).astype(np.float32)  # bench.cpp:48-60 range
    x[: cols // 2] *= 20  # one row reaching the lower clamp of t*(x - m)
    xd = torch.from_numpy(x).cuda()
    plan = qk.softmax_plan(cols, True, K(kern))
    for t in (0.125, 0.7, 1.0, 4.0):
        y = qk.softmax_rows(xd, cols, qk.SoftmaxParams(temperature=t), K(kern)).cpu().numpy()
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, t, kern), f"{cols} {kern} {t}")
    for bias in (True, False):
        p = qk.SoftmaxParams(temperature=0.5, centering_bias=bias)
        y = qk.softmax_rows(xd, cols, p, K(kern)).cpu().numpy()
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 0.5, kern, bias=int(bias)),
                        f"bias {bias}")


@pytest.mark.parametrize("kern", [QUAKE_UNFUSED, QUAKE2_UNFUSED])
def test_unfused_gelu_bitexact(kern):
    R = restatement()
    rng = np.random.default_rng(kern)
    x = np.concatenate([rng.uniform(-6, 6, 200003), rng.uniform(-2000, 2000, 5000),
                        np.array([0.0, -0.0, np.inf, -np.inf, np.nan, 1e30, -1e30, 1e-40,
                                  -1e-40], np.float64)]).astype(np.float32)
    for bias, b in ((None, -1), (True, 1), (False, 0)):
        y = qk.gelu_buffer(torch.from_numpy(x).cuda(), K(kern), centering_bias=bias)
        assert_bitexact(y.cpu().numpy(), R.gelu_buffer(x, kern, b), f"gelu {kern} {bias}")
        # host-span path (pageable memory) too
        assert_bitexact(qk.gelu_buffer(x, K(kern), centering_bias=bias),
                        R.gelu_buffer(x, kern, b), "host")


def test_unfused_rejected_outside_softmax_and_gelu():
    x = torch.zeros(64, device="cuda")
    for k in (K.QuakeUnfused, K.Quake2Unfused):
        with pytest.raises(ValueError, match="unknown kernel choice"):
            qk.logistic_buffer(x, k)


def _rel(a, b):
    a, b = np.asarray(a, np.float64), np.asarray(b, np.float64)
    den = np.maximum(np.abs(a), np.abs(b))
    return float(np.max(np.where(den > 0, np.abs(a - b) / np.where(den > 0, den, 1), 0)))


def test_fusion_ablation_gelu_divergence_is_the_references():
    """GELU is elementwise and bit-exact, so the harness's divergence is exactly the one
    the restatement (and hence the reference, test_oracle_cpu) computes on the same inputs."""
    R = restatement()
    for kern, kid, uid in ((K.Quake, QUAKE, QUAKE_UNFUSED), (K.Quake2, QUAKE2, QUAKE2_UNFUSED)):
        cfg = ab.BenchConfig(workload="gelu_vector", n=300_000, kernel=kern)
        r = ab.fusion_ablation(cfg)
        x = ab.fill_inputs(cfg).cpu().numpy()
        assert r.max_rel_divergence == _rel(R.gelu_buffer(x, kid), R.gelu_buffer(x, uid))
        assert r.fused.fused and not r.unfused.fused
        assert r.fused.elements == 300_000 and r.fusion_speedup > 0
        assert r.fused.measured_iters == 10 and r.fused.speedup_vs_exact > 0


def test_fusion_ablation_softmax_and_validation():
    R = restatement()
    cfg = ab.BenchConfig(workload="softmax_matrix", rows=256, cols=4096, kernel=K.Quake2,
                         temperature=0.7)
    r = ab.fusion_ablation(cfg)
    x = ab.fill_inputs(cfg).cpu().numpy()
    fused_plan = qk.softmax_plan(4096, True, K.Quake2)
    unfused_plan = qk.softmax_plan(4096, True, K.Quake2Unfused)
    want = _rel(R.softmax_rows_ordered(x, 4096, fused_plan, 0.7, QUAKE2),
                R.softmax_rows_ordered(x, 4096, unfused_plan, 0.7, QUAKE2_UNFUSED))
    assert r.max_rel_divergence == want
    assert 0 < r.max_rel_divergence < 1e-4
    with pytest.raises(ValueError, match="two warm-up"):
        ab.fusion_ablation(ab.BenchConfig(workload="gelu_vector", warmup_iters=1))
    with pytest.raises(ValueError, match="ten measured"):
        ab.run_bench(ab.BenchConfig(measured_iters=9))
    with pytest.raises(ValueError, match="softmax_matrix or gelu_vector"):
        ab.fusion_ablation(ab.BenchConfig(workload="exp_vector"))
    with pytest.raises(ValueError, match="empty workload"):
        ab.run_bench(ab.BenchConfig(n=0))


def test_run_bench_and_kernel_matrix():
    reps = ab.kernel_matrix([ab.BenchConfig(workload=w, n=1 << 20, rows=64, cols=4096)
                             for w in ab.WORKLOADS])
    assert len(reps) == 4 * 5
    for r in reps:
        assert r.mean_seconds > 0 and r.min_seconds <= r.mean_seconds
        assert np.isfinite(r.checksum) and r.throughput_eps > 0
    # Exact against itself through the same scaffolding: ~1 (bench.hpp:67-72)
    ex = [r for r in reps if r.kernel == "exact"]
    assert all(0.5 < r.speedup_vs_exact < 2.0 for r in ex)


# ---- the reference's bench cases (tests/test_bench.cpp), GPU-adapted bounds ----

def test_reference_bench_cases():
    # run_bench produces a coherent report (test_bench.cpp:25-42); on a bandwidth-bound
    # chip QuAKE does not beat exp by > 1x, so only positivity of the ratio is required
    r = ab.run_bench(ab.BenchConfig(workload="exp_vector", n=1 << 18, kernel=K.Quake))
    assert (r.workload, r.kernel, r.elements) == ("exp_vector", "quake", 1 << 18)
    assert 0 < r.min_seconds <= r.mean_seconds and r.throughput_eps > 0
    assert np.isfinite(r.checksum) and r.speedup_vs_exact > 0
    # self-comparison lands near unity (:44-55)
    r = ab.run_bench(ab.BenchConfig(workload="exp_vector", n=1 << 24, kernel=K.Exact,
                                    measured_iters=12))
    assert 0.85 < r.speedup_vs_exact < 1.18
    # identical fused and unfused kernels time the same (:94-105)
    a = ab.fusion_ablation(ab.BenchConfig(workload="softmax_matrix", rows=8192, cols=1024,
                                          kernel=K.Exact, measured_iters=12))
    assert 0.85 < a.fusion_speedup < 1.18 and a.max_rel_divergence == 0.0
    # fusion keeps values put (:75-92): within 2e-5
    a = ab.fusion_ablation(ab.BenchConfig(workload="softmax_matrix", rows=256, cols=512,
                                          kernel=K.Quake))
    assert a.fused.fused and not a.unfused.fused and a.max_rel_divergence <= 2e-5
    a = ab.fusion_ablation(ab.BenchConfig(workload="gelu_vector", n=100_000, kernel=K.Quake2))
    assert a.max_rel_divergence <= 2e-5
    # mean time scales with the workload (:107-120), at bandwidth-bound sizes
    small = ab.run_bench(ab.BenchConfig(workload="exp_vector", n=1 << 25, kernel=K.Quake2,
                                        measured_iters=12))
    big = ab.run_bench(ab.BenchConfig(workload="exp_vector", n=1 << 26, kernel=K.Quake2,
                                      measured_iters=12))
    assert 1.6 <= big.mean_seconds / small.mean_seconds <= 2.6
    # workload names round-trip (:122-129)
    for w in ab.WORKLOADS:
        assert ab.workload_from_name(ab.workload_name(w)) == w
    assert ab.workload_from_name("matmul") is None
