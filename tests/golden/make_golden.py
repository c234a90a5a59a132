"""Generate tests/golden/*.npz from the reference library compiled in place.

Run where /root/reference exists (this container), after `make -C oracle`:

    python tests/golden/make_golden.py

Every output array here is produced by the reference's own public entry
points (oracle/_ref/libquake_ref.so = /root/reference/proj/core/src/
{kernels,nonlin,parallel,oracle}.cpp built with the reference's Release
flags), on seeded inputs. The fixtures then pin both the C restatement
(CPU tests) and the CUDA path (GPU tests) without needing /root/reference.
"""
from __future__ import annotations

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle.oracle import CONTINUITY, EXACT, MINIMAX, QUAKE, QUAKE2, Reference  # noqa: E402


def elementwise_inputs() -> np.ndarray:
    rng = np.random.default_rng(20241200408)
    patterns = rng.integers(0, 2**32, size=16384, dtype=np.uint64).astype(np.uint32)
    specials = np.array([0x00000000, 0x80000000, 0x7F800000, 0xFF800000, 0x7FC00000, 0xFFC00000,
                         0x7F800001, 0x00000001, 0x80000001, 0x00800000, 0x80800000, 0x7F7FFFFF,
                         0xFF7FFFFF, 0x3F800000, 0xBF800000], dtype=np.uint32)
    ints = np.arange(-100, 101, dtype=np.float32)
    below = np.nextafter(ints, np.float32(-np.inf)).astype(np.float32)
    uniform = rng.uniform(-120, 120, 8192).astype(np.float32)
    gelu_range = rng.uniform(-12, 12, 4096).astype(np.float32)
    return np.concatenate([patterns.view(np.float32), specials.view(np.float32), ints, below,
                           uniform, gelu_range])


def main() -> None:
    ref = Reference()
    x = elementwise_inputs()
    out = {"x": x}
    for name, which, bias in (("natural_bias", "natural", 1), ("natural_nobias", "natural", 0),
                              ("base2", "base2", 0), ("negated_bias", "negated", 1)):
        c0, c1 = ref.named_coeffs(which, bias)
        lo, hi = ref.clamp_for(c0, c1)
        out[f"coeffs_{name}"] = np.array([c0, c1, lo, hi], dtype=np.float32)
        out[f"quake_{name}"] = ref.quake_buffer(x, c0, c1, lo, hi)
        out[f"quake2_{name}"] = ref.quake2_buffer(x, c0, c1, CONTINUITY, lo, hi)
        out[f"quake2mm_{name}"] = ref.quake2_buffer(x, c0, c1, MINIMAX, lo, hi)
    for k, kn in ((EXACT, "exact"), (QUAKE, "quake"), (QUAKE2, "quake2")):
        for b, bn in ((-1, "default"), (0, "off"), (1, "on")):
            if k == EXACT and b != -1:
                continue
            out[f"logistic_{kn}_{bn}"] = ref.logistic_buffer(x, k, b)
            out[f"gelu_{kn}_{bn}"] = ref.gelu_buffer(x, k, b)
    out["gelu_constants"] = np.array(ref.gelu_constants(), dtype=np.float32)
    # softmax: small matrices, the reference's own sequential-sum outputs
    rng = np.random.default_rng(4)
    for cols, rows, t, sd in ((512, 16, 0.125, 2.0), (1000, 6, 1.0, 3.0), (33, 40, 4.0, 5.0),
                              (4099, 2, 0.5, 4.0)):
        m = (rng.standard_normal(rows * cols) * sd).astype(np.float32)
        key = f"softmax_{rows}x{cols}_t{t}"
        out[f"{key}_in"] = m
        for k, kn in ((EXACT, "exact"), (QUAKE, "quake"), (QUAKE2, "quake2")):
            out[f"{key}_{kn}"] = ref.softmax_rows(m, cols, t, k)
    path = os.path.join(HERE, "reference_vectors.npz")
    np.savez_compressed(path, **out)
    print(f"wrote {path}: {len(out)} arrays, {os.path.getsize(path)} bytes")


if __name__ == "__main__":
    main()
