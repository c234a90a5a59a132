"""The five BASELINE.json configurations as seeded synthetic workloads.

No dataset is involved: BASELINE.json's configs name shapes and value
distributions only. Seeds are fixed per config (cfg k -> seed k).

Generator (counter-based, stated so any shard can be regenerated alone):
element i of a workload with seed s is a pure function of (s, i):

    h  = lowbias32(i)                      (Wellons' 32-bit integer hash)
    a  = lowbias32(h ^ k1),  b = lowbias32(h ^ k2),  k1/k2 = lowbias32(s*0x9E3779B9 + 1/2)
    uniform:  x = f32(lo + (hi - lo) * (a >> 8) * 2^-24)
    normal:   x = f32(mean + std * sqrt(-2 ln u1) * cos(2 pi u2)),
              u1 = ((a >> 8) + 0.5) * 2^-24, u2 = (b >> 8) * 2^-24  (binary64)

so a shard [r0, r1) of rows (or any element span) is bit-identical to the
same slice of the full draw, whichever process or GPU count produces it.
``device(span)`` evaluates it with torch on the GPU (no host round trip for
cfg5's 2 GB), ``host(span)`` with numpy; the two agree bit for bit except
where the two binary64 libms differ in a last place that moves the float32
rounding (none seen; see tests). Indices must stay below 2^32.
"""
from __future__ import annotations

from dataclasses import dataclass

import numpy as np

_M1, _M2 = 0x7FEB352D, 0x846CA68B
_MASK32 = 0xFFFFFFFF


def _lowbias32_int(x: int) -> int:
    x &= _MASK32
    x ^= x >> 16
    x = (x * _M1) & _MASK32
    x ^= x >> 15
    x = (x * _M2) & _MASK32
    x ^= x >> 16
    return x


def _keys(seed: int) -> tuple[int, int]:
    base = (seed * 0x9E3779B9) & _MASK32
    return _lowbias32_int(base + 1), _lowbias32_int(base + 2)


def _hash_np(x: np.ndarray) -> np.ndarray:
    """lowbias32 on uint32 arrays (numpy wraps uint32 products mod 2^32)."""
    x = x ^ (x >> np.uint32(16))
    x = x * np.uint32(_M1)
    x = x ^ (x >> np.uint32(15))
    x = x * np.uint32(_M2)
    return x ^ (x >> np.uint32(16))


def _mul32_t(x, c: int):
    """(x * c) mod 2^32 for int64 tensors holding uint32 values, without int64
    overflow: split c into 16-bit halves."""
    lo, hi = c & 0xFFFF, c >> 16
    return (x * lo + (((x * hi) & 0xFFFF) << 16)) & _MASK32


def _hash_t(x):
    x = x ^ (x >> 16)
    x = _mul32_t(x, _M1)
    x = x ^ (x >> 15)
    x = _mul32_t(x, _M2)
    return x ^ (x >> 16)


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

    def _span(self, span, rows) -> tuple[int, int]:
        if rows is not None:
            return rows[0] * self.cols, rows[1] * self.cols
        if span is None:
            return 0, self.n
        if isinstance(span, int):
            return 0, span
        return span

    def host(self, span=None, rows: tuple[int, int] | None = None) -> np.ndarray:
        """Elements [e0, e1) (span = (e0, e1), or n for [0, n); default all),
        or rows [r0, r1), as a float32 numpy array."""
        e0, e1 = self._span(span, rows)
        if e1 >= 1 << 32:
            raise ValueError("the counter-based generator indexes below 2^32")
        k1, k2 = _keys(self.seed)
        out = np.empty(e1 - e0, np.float32)
        step = 1 << 22

        def fill(c0):
            c1 = min(e1, c0 + step)
            h = _hash_np(np.arange(c0, c1, dtype=np.uint32))
            a = _hash_np(h ^ np.uint32(k1))
            if self.dist == "uniform":
                u = (a >> np.uint32(8)).astype(np.float64) * 2.0**-24
                out[c0 - e0:c1 - e0] = self.a + (self.b - self.a) * u
            else:
                b = _hash_np(h ^ np.uint32(k2))
                u1 = ((a >> np.uint32(8)).astype(np.float64) + 0.5) * 2.0**-24
                u2 = (b >> np.uint32(8)).astype(np.float64) * 2.0**-24
                z = np.sqrt(-2.0 * np.log(u1)) * np.cos(2.0 * np.pi * u2)
                out[c0 - e0:c1 - e0] = self.a + self.b * z

        starts = range(e0, e1, step)
        if e1 - e0 <= 2 * step:
            for c0 in starts:
                fill(c0)
        else:  # numpy releases the GIL inside the ufuncs
            import os
            from concurrent.futures import ThreadPoolExecutor
            with ThreadPoolExecutor(min(32, os.cpu_count() or 1)) as ex:
                list(ex.map(fill, starts))
        return out

    def device(self, span=None, rows: tuple[int, int] | None = None, device="cuda"):
        """The same elements as host(span, rows), generated on the GPU (torch)."""
        import torch
        e0, e1 = self._span(span, rows)
        if e1 >= 1 << 32:
            raise ValueError("the counter-based generator indexes below 2^32")
        k1, k2 = _keys(self.seed)
        out = torch.empty(e1 - e0, dtype=torch.float32, device=device)
        step = 1 << 26
        for c0 in range(e0, e1, step):
            c1 = min(e1, c0 + step)
            h = _hash_t(torch.arange(c0, c1, dtype=torch.int64, device=device))
            a = _hash_t(h ^ k1)
            if self.dist == "uniform":
                u = (a >> 8).to(torch.float64) * 2.0**-24
                out[c0 - e0:c1 - e0] = (self.a + (self.b - self.a) * u).to(torch.float32)
            else:
                b = _hash_t(h ^ k2)
                u1 = ((a >> 8).to(torch.float64) + 0.5) * 2.0**-24
                del a
                u2 = (b >> 8).to(torch.float64) * 2.0**-24
                del b, h
                z = torch.sqrt(-2.0 * torch.log(u1)) * torch.cos(2.0 * np.pi * u2)
                out[c0 - e0:c1 - e0] = (self.a + self.b * z).to(torch.float32)
        return out


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
