"""Generate tests/golden/reference_lab.json from the reference's own lab.

Run where /root/reference exists (this container), after `make -C oracle`:

    python tests/golden/make_lab_golden.py

Every number comes from the reference's public lab entry points
(core/src/lab.cpp compiled in place into oracle/_ref/libquake_ref.so):
sweep_error, continuity_probe, quad_max_rel_err, grid_search_quad and
bias_reoptimize, on the configurations of tests/test_lab.cpp and
tests/acceptance.cpp. The GPU lab (include/quake_b200_lab.h) is pinned to
these without needing /root/reference.
"""
from __future__ import annotations

import json
import os
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(os.path.dirname(HERE)))

from oracle.oracle import CONTINUITY, MINIMAX, QUAKE, QUAKE2, Reference  # noqa: E402

UNIT = dict(lo=-80.0, hi=80.0, uniform_samples=1 << 20, period_stride=8)        # test_lab.cpp:33
ACCEPT = dict(lo=-80.0, hi=80.0, uniform_samples=1 << 22, period_stride=1)      # acceptance.cpp:65
SWEEPS = [  # (name, kind, natural, bias, quad, spec)
    ("quake_e_bias_unit", QUAKE, True, True, CONTINUITY, UNIT),
    ("quake_e_nobias_unit", QUAKE, True, False, CONTINUITY, UNIT),
    ("quake2_e_nobias_unit", QUAKE2, True, False, CONTINUITY, UNIT),
    ("quake2_e_minimax_unit", QUAKE2, True, False, MINIMAX, UNIT),
    ("quake_2_nobias_unit", QUAKE, False, False, CONTINUITY, UNIT),
    ("quake2_2_bias_unit", QUAKE2, False, True, CONTINUITY, UNIT),
    ("quake2_2_poly_0_1", QUAKE2, False, False, CONTINUITY,
     dict(lo=0.0, hi=1.0, uniform_samples=1 << 20, period_stride=1)),           # test_lab.cpp:91-103
    ("quake2_e_repro", QUAKE2, True, False, CONTINUITY,
     dict(lo=-20.0, hi=20.0, uniform_samples=1 << 18, period_stride=16)),       # test_lab.cpp:81-89
    ("c1_quake_e_bias", QUAKE, True, True, CONTINUITY, ACCEPT),                 # acceptance.cpp:69-80
    ("c2_quake2_e_nobias", QUAKE2, True, False, CONTINUITY, ACCEPT),            # :84-93
    ("c4_quake_e_nobias", QUAKE, True, False, CONTINUITY, ACCEPT),              # :113-127
]
CONTINUITY_CASES = [  # (name, kind, natural, bias, quad, k_lo, k_hi)
    ("quake_2_nobias", QUAKE, False, False, CONTINUITY, -100, 100),
    ("quake2_2_nobias", QUAKE2, False, False, CONTINUITY, -100, 100),
    ("quake2_2_minimax", QUAKE2, False, False, MINIMAX, -50, 50),
    ("quake_e_bias", QUAKE, True, True, CONTINUITY, -125, 127),
]


def main():
    F = Reference()
    out = {"generator": "tests/golden/make_lab_golden.py (reference core/src/lab.cpp)",
           "sweeps": {}, "continuity": {}, "quad": {}, "grid": {}, "bias": {}}
    for name, kind, nat, bias, quad, spec in SWEEPS:
        n, mx, mean, arg = F.sweep_error(kind, nat, bias, quad, **spec)
        out["sweeps"][name] = dict(kind=kind, natural=nat, bias=bias, quad=[float(q) for q in quad],
                                   spec=spec, samples=n, max_rel_err=mx, mean_rel_err=mean,
                                   argmax_input=float(arg))
    for name, kind, nat, bias, quad, klo, khi in CONTINUITY_CASES:
        w, at = F.continuity_probe(kind, nat, bias, klo, khi, quad)
        out["continuity"][name] = dict(kind=kind, natural=nat, bias=bias,
                                       quad=[float(q) for q in quad], k_lo=klo, k_hi=khi,
                                       worst_jump=w, at=float(at))
    for name, (a0, a1, a2, iv) in {"continuity_2p20": (1 / 3, 0.0, 2 / 3, 1 << 20),
                                   "minimax_2p16": (0.33, -0.017, 0.68, 1 << 16),
                                   "grid_best_2p16_7": (0.336, -0.012, 0.677, (1 << 16) + 7)}.items():
        out["quad"][name] = dict(a=[a0, a1, a2], intervals=iv,
                                 value=F.quad_max_rel_err(a0, a1, a2, iv))
    for name, axes in {"default": (0.30, 0.36, 0.001, -0.05, 0.02, 0.001, 0.64, 0.72, 0.001),
                       "endpoint": (1 / 3, 1 / 3, 1.0, 0.0, 0.0, 1.0, 2 / 3, 2 / 3, 1.0),
                       "constant": (0.0, 0.0, 1.0, 0.0, 0.0, 1.0, 1.0, 1.0, 1.0)}.items():
        best, err, pts = F.grid_search_quad(axes)
        out["grid"][name] = dict(axes=list(axes), best=[float(b) for b in best],
                                 best_max_rel_err=err, points=pts)
    for name, kind in (("quake_e_bias", QUAKE), ("quake2_e_nobias", QUAKE2)):
        beta, err, near = F.bias_reoptimize(kind, True, kind == QUAKE, CONTINUITY)
        out["bias"][name] = dict(kind=kind, natural=True, bias=kind == QUAKE, beta=float(beta),
                                 max_rel_err=err, near=near)
    path = os.path.join(HERE, "reference_lab.json")
    with open(path, "w") as f:
        json.dump(out, f, indent=1)
    print("wrote", path)


if __name__ == "__main__":
    main()
