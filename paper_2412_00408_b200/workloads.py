"""The five BASELINE.json configurations as seeded synthetic workloads.

No dataset is involved: BASELINE.json's configs name shapes and value
distributions only. Seeds are fixed per config (cfg k -> seed k). Two
generators produce the bytes:

* ``host(cfg)`` — numpy PCG64 (``default_rng(seed)``), float32 draws;
* ``device(cfg)`` — torch's CUDA Philox generator seeded the same way, for
  full-size runs (2 GB for cfg5) without a host round trip. Parity tests that
  use device inputs copy those exact bytes back for the oracle.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class Workload:
    name: str
    op: str            # exp | logistic | gelu | softmax
    shape: tuple
    dist: str          # uniform | normal
    a: float           # uniform lo / normal mean
    b: float           # uniform hi / normal std
    seed: int
    temperature: float = 1.0
    kernels: tuple = ("quake", "quake2")
    description: str = ""

    @property
    def n(self) -> int:
        n = 1
        for s in self.shape:
            n *= s
        return n

    @property
    def cols(self) -> int:
        return self.shape[-1]

    @property
    def rows(self) -> int:
        return self.n // self.cols

    def host(self, n: int | None = None) -> np.ndarray:
        rng = np.random.default_rng(self.seed)
        size = self.n if n is None else n
        if self.dist == "uniform":
            x = rng.uniform(self.a, self.b, size).astype(np.float32)
        else:
            x = (rng.standard_normal(size, dtype=np.float32) * np.float32(self.b)
                 + np.float32(self.a))
        return x

    def device(self, rows: tuple[int, int] | None = None, device="cuda"):
        """Full workload on the GPU (torch), optionally only rows [r0, r1)."""
        import torch
        g = torch.Generator(device=device)
        g.manual_seed(self.seed)
        if rows is None:
            shape = (self.n,)
        else:
            shape = ((rows[1] - rows[0]) * self.cols,)
            # Every rank draws its own rows from an independent stream.
            g.manual_seed(self.seed * 1000003 + rows[0])
        if self.dist == "uniform":
            x = torch.rand(shape, generator=g, device=device, dtype=torch.float32)
            x.mul_(self.b - self.a).add_(self.a)
        else:
            x = torch.randn(shape, generator=g, device=device, dtype=torch.float32)
            x.mul_(self.b).add_(self.a)
        return x


CFG1 = Workload("cfg1_exp", "exp", (1 << 24,), "uniform", -10.0, 10.0, 1,
                description="QuAKE exp, 2^24 fp32 U[-10,10]; first and second order")
CFG2 = Workload("cfg2_logistic", "logistic", (4096, 4096), "normal", 0.0, 3.0, 2,
                description="logistic, 4096x4096 fp32 N(0,3)")
CFG3 = Workload("cfg3_gelu", "gelu", (16384, 3072), "normal", 0.0, 1.0, 3,
                description="GELU, FFN activation 16384x3072 fp32 N(0,1)")
CFG4 = Workload("cfg4_softmax_attn", "softmax", (8, 12, 512, 512), "normal", 0.0, 2.0, 4,
                temperature=0.125,
                description="row softmax over attention scores 8x12x512x512, t=1/sqrt(64)")
CFG5 = Workload("cfg5_softmax_vocab", "softmax", (4096, 128256), "normal", 0.0, 4.0, 5,
                temperature=1.0, kernels=("quake2",),
                description="row softmax over LM vocab logits 4096x128256, QuAKE2")

# Not a bench line: the paper's Table III softmax size (§V-A2,
# 16384x16384, bench.cpp:48-60 input range), used for plan tuning / ablation.
PAPER_SOFTMAX = Workload("paper_softmax_16k", "softmax", (16384, 16384), "uniform", -8.0, 8.0,
                         42, temperature=1.0, kernels=("quake", "quake2"),
                         description="Table III softmax matrix 16384x16384, U(-8, 8)")

CONFIGS = {w.name: w for w in (CFG1, CFG2, CFG3, CFG4, CFG5)}
TUNING = {PAPER_SOFTMAX.name: PAPER_SOFTMAX}
