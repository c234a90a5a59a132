"""GPU fusion ablation and kernel matrix.

Mirrors the reference's benchmark harness (core/include/quake/bench.hpp:28-84,
core/src/bench.cpp:286-513) on the sm_100a kernels:

* ``run_bench(cfg)`` — one workload / kernel, seeded uniform inputs in the
  reference's per-workload range (bench.cpp:48-60), >= 2 warm-ups and >= 10
  measured iterations (bench.cpp:361-372), outputs checksummed every
  iteration (drift raises, bench.cpp:315-339), and the Exact kernel timed
  through the same scaffolding for ``speedup_vs_exact``.
* ``fusion_ablation(cfg)`` — softmax_matrix / gelu_vector only: the fused
  kernel (affine transform folded into c0/c1) against the unfused one
  (``KernelChoice.QuakeUnfused`` / ``Quake2Unfused``: t*(x - m), resp.
  fused_scale*x*(1/kappa + x*x), computed explicitly and fed to the plain
  natural / negated-natural exponential, bench.cpp:137-166, 212-233), paired
  and interleaved with alternating order; ``fusion_speedup`` is the ratio of
  the minima, ``max_rel_divergence`` the elementwise drift (bench.cpp:425-513).
* ``kernel_matrix(...)`` — every workload x {Exact, Expf, FastExp, Quake,
  Quake2}: the paper's Table III "speedup w/o op fusion" column on the GPU.

Timing is per iteration with CUDA events on the launching stream (device
time; the reference times wall clock on one CPU thread). Inputs are
generated on the device (torch Philox, same range and distribution as the
reference's mt19937_64 stream, not the same values).
"""
from __future__ import annotations

import argparse
import ctypes
import json
from dataclasses import asdict, dataclass, field
from typing import Callable, List, Optional

import torch

from . import _lib
from .quake import KernelChoice, SoftmaxParams, kernel_name

WORKLOADS = ("softmax_matrix", "gelu_vector", "exp_vector", "logistic_vector")
# bench.cpp:48-60 input_range
INPUT_RANGE = {"softmax_matrix": (-8.0, 8.0), "gelu_vector": (-6.0, 6.0),
               "exp_vector": (-20.0, 20.0), "logistic_vector": (-12.0, 12.0)}
UNFUSED = {KernelChoice.Quake: KernelChoice.QuakeUnfused,
           KernelChoice.Quake2: KernelChoice.Quake2Unfused}


@dataclass
class BenchConfig:
    """bench.hpp:33-46 BenchConfig (same defaults)."""

    workload: str = "exp_vector"
    rows: int = 4096
    cols: int = 4096
    n: int = 260_000
    kernel: KernelChoice = KernelChoice.Quake
    warmup_iters: int = 2
    measured_iters: int = 10
    fused: bool = True
    temperature: float = 1.0
    centering_bias: Optional[bool] = None
    seed: int = 42


@dataclass
class BenchReport:
    """bench.hpp:48-65 BenchReport; the environment fingerprint is the GPU."""

    workload: str
    kernel: str
    fused: bool
    elements: int
    warmup_iters: int
    measured_iters: int
    mean_seconds: float
    min_seconds: float
    throughput_eps: float
    speedup_vs_exact: float
    checksum: float
    device: str = ""
    timing: str = "cuda events per iteration (device time)"
    seed: int = 0


@dataclass
class AblationReport:
    """bench.hpp:74-79 AblationReport."""

    fused: BenchReport
    unfused: BenchReport
    fusion_speedup: float
    max_rel_divergence: float
    divergence_note: str = field(default="max |a-b|/max(|a|,|b|) over elements, fp64")


def workload_name(w: str) -> str:
    """bench.cpp:385-397 (workloads are their names here)."""
    if w not in WORKLOADS:
        return "unknown"
    return w


def workload_from_name(name: str) -> Optional[str]:
    """bench.cpp:399-405."""
    return name if name in WORKLOADS else None


def element_count(cfg: BenchConfig) -> int:
    return cfg.rows * cfg.cols if cfg.workload == "softmax_matrix" else cfg.n


def validate(cfg: BenchConfig) -> None:
    """bench.cpp:350-363 validate (same messages)."""
    if cfg.workload not in WORKLOADS:
        raise ValueError(f"bench: unknown workload {cfg.workload}")
    if cfg.warmup_iters < 2:
        raise ValueError("bench: at least two warm-up iterations required")
    if cfg.measured_iters < 10:
        raise ValueError("bench: at least ten measured iterations required")
    if element_count(cfg) == 0:
        raise ValueError("bench: empty workload")


def fill_inputs(cfg: BenchConfig, device="cuda") -> torch.Tensor:
    """Seeded uniform inputs in the workload's range (bench.cpp:341-348)."""
    lo, hi = INPUT_RANGE[cfg.workload]
    g = torch.Generator(device=device)
    g.manual_seed(cfg.seed)
    x = torch.rand(element_count(cfg), generator=g, device=device, dtype=torch.float32)
    return x.mul_(hi - lo).add_(lo)


def make_pass(cfg: BenchConfig, kernel: KernelChoice, x: torch.Tensor,
              y: torch.Tensor) -> Callable[[], None]:
    """One launch of the workload's device operator on the current stream."""
    L = _lib.lib()
    n = x.numel()
    bias = -1 if cfg.centering_bias is None else int(bool(cfg.centering_bias))
    k = int(kernel)
    xp, yp = x.data_ptr(), y.data_ptr()

    def check(st):
        if st != 0:
            raise RuntimeError(f"{cfg.workload}/{kernel_name(kernel)}: {_lib.last_error()}")

    if cfg.workload == "softmax_matrix":
        prm = SoftmaxParams(temperature=cfg.temperature, centering_bias=cfg.centering_bias)._c()
        cols = cfg.cols
        return lambda: check(L.qk_softmax_rows_device(
            xp, n, cols, ctypes.byref(prm), k, yp, None, torch.cuda.current_stream().cuda_stream))
    if cfg.workload == "gelu_vector":
        return lambda: check(L.qk_gelu_buffer_device(
            xp, yp, n, k, bias, torch.cuda.current_stream().cuda_stream))
    if cfg.workload == "logistic_vector":
        return lambda: check(L.qk_logistic_buffer_device(
            xp, yp, n, k, bias, torch.cuda.current_stream().cuda_stream))
    return lambda: check(L.qk_exp_buffer_device(
        xp, yp, n, k, torch.cuda.current_stream().cuda_stream))


def checksum_of(y: torch.Tensor) -> float:
    """Sum of the outputs in fp64 (bench.cpp:309-313; device reduction order)."""
    return float(y.double().sum().item())


def _timed(fn: Callable[[], None]) -> float:
    a = torch.cuda.Event(enable_timing=True)
    b = torch.cuda.Event(enable_timing=True)
    a.record()
    fn()
    b.record()
    b.synchronize()
    dt = a.elapsed_time(b) * 1e-3
    return dt if dt > 0 else 1e-9  # zero-duration guard (bench.cpp:333)


def measure(fn, y, warmup: int, measured: int):
    """bench.cpp:315-339: warm-ups, then per-iteration timing + drift guard."""
    for _ in range(warmup):
        fn()
    torch.cuda.synchronize()
    ref = checksum_of(y)
    times = []
    for _ in range(measured):
        times.append(_timed(fn))
        if checksum_of(y) != ref:
            raise RuntimeError("bench: checksum drift across iterations")
    return sum(times) / len(times), min(times), ref


def _report(cfg, kernel, fused, mean, mn, chk, exact_mean) -> BenchReport:
    n = element_count(cfg)
    return BenchReport(workload=cfg.workload, kernel=kernel_name(kernel), fused=fused,
                       elements=n, warmup_iters=cfg.warmup_iters,
                       measured_iters=cfg.measured_iters, mean_seconds=mean, min_seconds=mn,
                       throughput_eps=n / mean, speedup_vs_exact=exact_mean / mean,
                       checksum=chk, device=torch.cuda.get_device_name(), seed=cfg.seed)


def run_bench(cfg: BenchConfig) -> BenchReport:
    """bench.cpp:407-423 run_bench."""
    validate(cfg)
    x = fill_inputs(cfg)
    y = torch.empty_like(x)
    k = cfg.kernel if cfg.fused or cfg.kernel not in UNFUSED else UNFUSED[cfg.kernel]
    mean, mn, chk = measure(make_pass(cfg, k, x, y), y, cfg.warmup_iters, cfg.measured_iters)
    # Exact through the same scaffolding, re-measured even for Exact itself
    ex_mean, _, _ = measure(make_pass(cfg, KernelChoice.Exact, x, y), y, cfg.warmup_iters,
                            cfg.measured_iters)
    return _report(cfg, cfg.kernel, cfg.fused, mean, mn, chk, ex_mean)


def fusion_ablation(cfg: BenchConfig) -> AblationReport:
    """bench.cpp:425-513 fusion_ablation."""
    if cfg.workload not in ("softmax_matrix", "gelu_vector"):
        raise ValueError("fusion_ablation: workload must be softmax_matrix or gelu_vector")
    validate(cfg)
    x = fill_inputs(cfg)
    y_f = torch.empty_like(x)
    y_u = torch.empty_like(x)
    fused = make_pass(cfg, cfg.kernel, x, y_f)
    # kernels without an affine fold (Exact, expf, __expf) run the same pass twice
    # (bench.cpp:95-100: "the exact path ignores fusion")
    unfused = make_pass(cfg, UNFUSED.get(cfg.kernel, cfg.kernel), x, y_u)
    for _ in range(cfg.warmup_iters):
        fused()
        unfused()
    torch.cuda.synchronize()
    chk_f, chk_u = checksum_of(y_f), checksum_of(y_u)
    tf, tu = [], []
    # paired, interleaved, alternating which variant goes first
    for i in range(cfg.measured_iters):
        if i % 2 == 0:
            tf.append(_timed(fused))
            tu.append(_timed(unfused))
        else:
            tu.append(_timed(unfused))
            tf.append(_timed(fused))
        if checksum_of(y_f) != chk_f or checksum_of(y_u) != chk_u:
            raise RuntimeError("bench: checksum drift across iterations")
    y_e = torch.empty_like(x)
    ex_mean, _, _ = measure(make_pass(cfg, KernelChoice.Exact, x, y_e), y_e, cfg.warmup_iters,
                            cfg.measured_iters)
    a, b = y_f.double(), y_u.double()
    den = torch.maximum(a.abs(), b.abs())
    rel = torch.where(den > 0, (a - b).abs() / torch.where(den > 0, den, 1.0), 0.0)
    div = float(rel.max().item())
    mf, mu = sum(tf) / len(tf), sum(tu) / len(tu)
    return AblationReport(
        fused=_report(cfg, cfg.kernel, True, mf, min(tf), chk_f, ex_mean),
        unfused=_report(cfg, cfg.kernel, False, mu, min(tu), chk_u, ex_mean),
        fusion_speedup=min(tu) / min(tf), max_rel_divergence=div)


def kernel_matrix(cfgs: List[BenchConfig],
                  kernels=(KernelChoice.Exact, KernelChoice.Expf, KernelChoice.FastExp,
                           KernelChoice.Quake, KernelChoice.Quake2)) -> List[BenchReport]:
    """Every workload x kernel through run_bench (the exact/__expf matrix)."""
    out = []
    for c in cfgs:
        for k in kernels:
            cc = BenchConfig(**{**asdict(c), "kernel": k})
            out.append(run_bench(cc))
    return out


def table3(softmax_rows=16384, softmax_cols=16384, gelu_n=260_000, measured=20):
    """The paper's Table III rows on this GPU (§V-A2 sizes):
    speedup w/o op fusion (Exact mean / kernel mean, unfused kernel) and the
    additional speedup due to op fusion (unfused min / fused min)."""
    rows = []
    for wl, shape in (("softmax_matrix", dict(rows=softmax_rows, cols=softmax_cols)),
                      ("gelu_vector", dict(n=gelu_n))):
        for k in (KernelChoice.Quake, KernelChoice.Quake2):
            r = fusion_ablation(BenchConfig(workload=wl, kernel=k, measured_iters=measured,
                                            **shape))
            rows.append({"op": wl, "kernel": kernel_name(k),
                         "elements": r.fused.elements,
                         "speedup_wo_fusion": r.unfused.speedup_vs_exact,
                         "additional_speedup_fusion": r.fusion_speedup,
                         "fused_min_us": r.fused.min_seconds * 1e6,
                         "unfused_min_us": r.unfused.min_seconds * 1e6,
                         "exact_mean_us": r.fused.mean_seconds * r.fused.speedup_vs_exact * 1e6,
                         "fused_gbps": 8 * r.fused.elements / r.fused.min_seconds / 1e9,
                         "max_rel_divergence": r.max_rel_divergence})
    return rows


def main(argv=None):
    ap = argparse.ArgumentParser(description=__doc__.split("\n")[0])
    ap.add_argument("--mode", choices=("table3", "matrix", "ablation"), default="table3")
    ap.add_argument("--workload", default="softmax_matrix")
    ap.add_argument("--kernel", default="quake")
    ap.add_argument("--rows", type=int, default=16384)
    ap.add_argument("--cols", type=int, default=16384)
    ap.add_argument("--n", type=int, default=260_000)
    ap.add_argument("--iters", type=int, default=20)
    a = ap.parse_args(argv)
    if a.mode == "table3":
        for r in table3(a.rows, a.cols, a.n, a.iters):
            print(json.dumps(r), flush=True)
        return
    if a.mode == "ablation":
        k = {"quake": KernelChoice.Quake, "quake2": KernelChoice.Quake2}[a.kernel]
        r = fusion_ablation(BenchConfig(workload=a.workload, kernel=k, rows=a.rows, cols=a.cols,
                                        n=a.n, measured_iters=a.iters))
        print(json.dumps(asdict(r)), flush=True)
        return
    cfgs = [BenchConfig(workload="softmax_matrix", rows=a.rows, cols=a.cols,
                        measured_iters=a.iters),
            BenchConfig(workload="gelu_vector", n=a.n, measured_iters=a.iters),
            BenchConfig(workload="exp_vector", n=a.n, measured_iters=a.iters),
            BenchConfig(workload="logistic_vector", n=a.n, measured_iters=a.iters)]
    for r in kernel_matrix(cfgs):
        d = asdict(r)
        d["gbps_min"] = 8 * r.elements / r.min_seconds / 1e9
        print(json.dumps(d), flush=True)


if __name__ == "__main__":
    main()
