"""Shared test helpers (bit comparison, ulp distance, oracle access)."""
from __future__ import annotations

import numpy as np

from oracle.oracle import Restatement, reference_or_none

_R = None


def restatement() -> Restatement:
    global _R
    if _R is None:
        _R = Restatement()
    return _R


def reference():
    return reference_or_none()


def bits(a) -> np.ndarray:
    return np.ascontiguousarray(a, dtype=np.float32).view(np.uint32)


def assert_bitexact(got, want, what=""):
    g, w = bits(got).ravel(), bits(want).ravel()
    assert g.shape == w.shape, (what, g.shape, w.shape)
    bad = np.nonzero(g != w)[0]
    if bad.size:
        i = bad[0]
        gf = np.asarray(got, dtype=np.float32).ravel()
        wf = np.asarray(want, dtype=np.float32).ravel()
        raise AssertionError(f"{what}: {bad.size} of {g.size} differ; first at {i}: "
                             f"got {gf[i]!r} (0x{g[i]:08x}) want {wf[i]!r} (0x{w[i]:08x})")


def ordered_ulp(a) -> np.ndarray:
    """Map float32 bit patterns to a monotone integer line (for ulp distances)."""
    u = bits(a).astype(np.int64)
    return np.where(u & 0x80000000, 0x80000000 - u, u)


def max_ulp(got, want) -> int:
    g, w = np.asarray(got, np.float32).ravel(), np.asarray(want, np.float32).ravel()
    both_nan = np.isnan(g) & np.isnan(w)
    d = np.abs(ordered_ulp(g) - ordered_ulp(w))
    d[both_nan] = 0
    return int(d.max()) if d.size else 0


def max_rel(got, want) -> float:
    g = np.asarray(got, np.float64).ravel()
    w = np.asarray(want, np.float64).ravel()
    return float(np.max(np.abs(g - w) / np.abs(w))) if g.size else 0.0
