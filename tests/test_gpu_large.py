"""Maximum sizes: buffers beyond 2^32 elements (B200 holds 180 GB), so every
index, row offset and grid computation must be 64-bit. Checked bit-exact
against the restatement on slices at the start, around 2^31 and 2^32 and at
the end."""
import numpy as np
import pytest
import torch

import paper_2412_00408_b200 as qk
from oracle.oracle import QUAKE, QUAKE2
from tests.helpers import assert_bitexact, restatement

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
K = qk.KernelChoice


@pytest.fixture(autouse=True)
def _room():
    free, _ = torch.cuda.mem_get_info()
    if free < 40e9:
        pytest.skip("needs ~40 GB of free device memory")
    yield
    torch.cuda.empty_cache()


def _filled(n, lo, hi, seed):
    g = torch.Generator(device="cuda")
    g.manual_seed(seed)
    return torch.empty(n, device="cuda").uniform_(lo, hi, generator=g)


def test_elementwise_beyond_2p32():
    R = restatement()
    n = (1 << 32) + 4099
    x = _filled(n, -90.0, 90.0, 1)
    c = qk.natural_exp_coeffs(False)
    r = qk.clamp_for(c)
    y = qk.quake2_buffer(x, c, qk.QuadCoeffs.continuity(), r)
    from oracle.oracle import CONTINUITY
    for b in (0, (1 << 31) - 2048, (1 << 32) - 2048, n - 4096):
        xs = x[b:b + 4096].cpu().numpy()
        assert_bitexact(y[b:b + 4096].cpu().numpy(),
                        R.quake2_buffer(xs, c.c0, c.c1, CONTINUITY, r.lo, r.hi), f"at {b}")
    del y
    z = qk.gelu_buffer(x, K.Quake)
    xs = x[-4096:].cpu().numpy()
    assert_bitexact(z[-4096:].cpu().numpy(), R.gelu_buffer(xs, QUAKE), "gelu tail")


# 512: sub-warp rows; 128256: cluster pipeline; 513 / 4099: warp rings (register form,
# three sweeps by two-warp agents) — 64-bit job cursors and row offsets
@pytest.mark.parametrize("cols", [512, 128256, 513, 4099])
def test_softmax_rows_beyond_2p32(cols):
    R = restatement()
    rows = (1 << 32) // cols + 3
    x = _filled(rows * cols, -12.0, 12.0, cols)
    y = qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2)
    plan = qk.softmax_plan(cols, True, K.Quake2)
    for r0 in (0, (1 << 31) // cols - 1, rows - 4):
        xs = x[r0 * cols:(r0 + 4) * cols].cpu().numpy()
        want = R.softmax_rows_ordered(xs, cols, plan, 1.0, QUAKE2)
        assert_bitexact(y[r0 * cols:(r0 + 4) * cols].cpu().numpy(), want, f"rows {r0}..")
