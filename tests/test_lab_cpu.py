"""CPU: the GPU lab's C-ABI (include/quake_b200_lab.h) is exported and bound,
and its argument validation follows the reference lab (lab.cpp:150-163,
221-237, 281-293, 330-338) — no GPU reached by any of these calls."""
import json
import os
import re
import subprocess

import pytest

from paper_2412_00408_b200 import KernelChoice as K
from paper_2412_00408_b200 import _lib
from paper_2412_00408_b200 import lab

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "quake_b200_lab.h")


def test_lab_header_exported_and_bound():
    src = re.sub(r"/\*.*?\*/", "", open(HEADER).read(), flags=re.S)
    decl = set(re.findall(r"\b(qk_[a-z0-9_]+)\s*\(", src))
    out = subprocess.run(["nm", "-D", "--defined-only", _lib.LIB_PATH], capture_output=True,
                         text=True, check=True).stdout
    exported = set(line.split()[-1] for line in out.splitlines() if line.strip())
    assert decl and decl <= exported, decl - exported
    assert decl == set(_lib.LAB_SIGNATURES), decl ^ set(_lib.LAB_SIGNATURES)


def test_lab_defaults_and_coefficients():
    L = _lib.lib()
    s = L.qk_sweep_spec_defaults()
    assert (s.lo, s.hi, s.uniform_samples, s.period_stride) == (-80.0, 80.0, 1 << 22, 1)
    g = L.qk_grid_spec_defaults()
    assert (g.a0.lo, g.a0.hi, g.a0.step, g.a1.lo, g.a2.hi) == (0.30, 0.36, 0.001, -0.05, 0.72)
    c, r = lab.ExpConfig(K.Quake, True, True).coeffs_and_clamp()
    # Appendix A.3: natural exp, bias on
    import numpy as np
    assert np.float32(c.c0).view(np.uint32) == 0x4B38AA3B
    assert np.float32(c.c1).view(np.uint32) == 0x4E7DE9AD
    assert np.float32(r.lo).view(np.uint32) == 0xC2AE994A
    c2, _ = lab.ExpConfig(K.Quake, False, False).coeffs_and_clamp()
    assert (c2.c0, c2.c1) == (8388608.0, 1065353216.0)
    assert lab.ExpConfig(K.Quake2, True, False, lab.QuadCoeffs.minimax()).label() == \
        "quake2:e:nobias:custom-quad"
    assert lab.ExpConfig(K.Exact, False).label() == "exact:2"


def test_lab_validation_matches_reference_messages():
    q = lab.ExpConfig(K.Quake, True, True)
    cases = [
        (lambda: lab.sweep_error(q, lab.SweepSpec(5.0, 5.0, 1 << 20, 1)), "sweep_error: range is empty"),
        (lambda: lab.sweep_error(q, lab.SweepSpec(0.0, 1.0, 100, 1)),
         "sweep_error: need at least 10^4 samples"),
        (lambda: lab.sweep_error(q, lab.SweepSpec(-200.0, 200.0, 1 << 20, 1)),
         "sweep_error: range exceeds clamp bounds"),
        (lambda: lab.grid_search_quad(lab.GridSpec(a0=lab.GridAxis(0.4, 0.3, 0.001))),
         "grid_search_quad: empty grid"),
        (lambda: lab.continuity_probe(q, 5, 4), "continuity_probe: empty range"),
        (lambda: lab.continuity_probe(q, -126, 0), "continuity_probe: range exceeds the normal band"),
        (lambda: lab.continuity_probe(q, 0, 128), "continuity_probe: range exceeds the normal band"),
        (lambda: lab.bias_reoptimize(lab.ExpConfig(K.Exact)),
         "bias_reoptimize: nothing to optimize for exact"),
        (lambda: lab.bias_reoptimize(q, 0.1, 0.1), "bias_reoptimize: empty search interval"),
        (lambda: lab.sweep_exhaustive(q, -200.0, 0.0), "sweep_exhaustive: range exceeds clamp bounds"),
        (lambda: lab.sweep_exhaustive(lab.ExpConfig(K.Expf)), "lab: unknown kernel choice"),
    ]
    for fn, msg in cases:
        with pytest.raises(ValueError) as ei:
            fn()
        assert str(ei.value) == msg
    # lab.cpp:282: the exact kernel has no wraparound to probe
    assert lab.continuity_probe(lab.ExpConfig(K.Exact), -100, 100) == lab.ContinuityReport(0.0, 0.0)


def test_reference_lab_fixture_is_current():
    """The committed fixture was produced by the compiled reference lab."""
    from tests.helpers import reference
    F = reference()
    d = json.load(open(os.path.join(ROOT, "tests", "golden", "reference_lab.json")))
    if F is None:
        pytest.skip("reference not compiled here")
    v = d["sweeps"]["quake_e_bias_unit"]
    n, mx, mean, arg = F.sweep_error(v["kind"], v["natural"], v["bias"], tuple(v["quad"]),
                                     **v["spec"])
    assert (n, mx, mean, float(arg)) == (v["samples"], v["max_rel_err"], v["mean_rel_err"],
                                         v["argmax_input"])
