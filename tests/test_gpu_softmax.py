"""GPU parity of row softmax (K5/K6) through the C-ABI.

Two bars per case:
  * bit-exact against the restatement summed in the kernel's declared order
    (or_softmax_rows_ordered) — proves the per-element exps, the fp64 per-row
    c1 / v_min derivation and the division are the reference's;
  * within 2e-6 relative of the reference's own sequential-sum output
    (cfg4, short rows) or of the fp64-sum restatement (cfg5 vocab rows,
    SURVEY.md F5/H3); the deviation from the reference's fp32 sequential sum
    at vocab length is reported, not bounded (it is the reference's own
    rounding, ~3e-4).
Reference tests mirrored: tests/test_nonlin.cpp:42-204, acceptance.cpp:178-254.
"""
import os

import numpy as np
import pytest
import torch

import paper_2412_00408_b200 as qk
from oracle.oracle import CONTINUITY, MINIMAX, QUAKE, QUAKE2
from paper_2412_00408_b200.workloads import CFG4, CFG5
from tests.helpers import assert_bitexact, max_rel, reference, restatement

pytestmark = pytest.mark.gpu
K = qk.KernelChoice
TOL = 2e-6  # north star: Softmax within 2e-6 relative per element


def _gpu_softmax(x, cols, t, kernel, bias=None, quad=None):
    xd = torch.from_numpy(np.ascontiguousarray(x, dtype=np.float32)).cuda()
    p = qk.SoftmaxParams(temperature=t, centering_bias=bias,
                         quad=qk.QuadCoeffs(*(quad or CONTINUITY)))
    y = qk.softmax_rows(xd, cols, p, K(kernel))
    torch.cuda.synchronize()
    return y.cpu().numpy()


@pytest.mark.parametrize("cols", [1, 2, 3, 5, 31, 32, 33, 100, 127, 128, 129, 511, 512, 513, 1028, 1100, 1536,
                                  1000, 1024, 1025, 2048, 3001, 4096, 16384, 16387, 50000,
                                  128256, 131072, 300000])
@pytest.mark.parametrize("kernel", [QUAKE, QUAKE2])
def test_shapes_bitexact_vs_ordered_restatement(cols, kernel):
    R = restatement()
    rows = max(2, min(64, (1 << 22) // cols))
    x = (np.random.default_rng(cols).standard_normal(rows * cols) * 3).astype(np.float32)
    for t in (0.125, 1.0):
        y = _gpu_softmax(x, cols, t, kernel)
        plan = qk.softmax_plan(cols, True, K(kernel))
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, t, kernel),
                        f"cols={cols} k={kernel} t={t} plan={plan}")
        ref = R.softmax_rows(x, cols, t, kernel, sum_mode=1)  # fp64 row sum
        assert max_rel(y, ref) <= TOL


def test_cfg4_full_size():
    """cfg4 [8,12,512,512] N(0,2), t=1/8, both orders: ≤2e-6 vs the reference's output."""
    R = restatement()
    xd = CFG4.device()
    x = xd.cpu().numpy()
    ref_lib = reference()
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(512, True, K(kern))
        p = qk.SoftmaxParams(temperature=CFG4.temperature)
        y = qk.softmax_rows(xd, 512, p, K(kern)).cpu().numpy()
        assert_bitexact(y, R.softmax_rows_ordered(x, 512, plan, CFG4.temperature, kern), "cfg4")
        want = (ref_lib.softmax_rows(x, 512, CFG4.temperature, kern) if ref_lib
                else R.softmax_rows(x, 512, CFG4.temperature, kern))
        assert max_rel(y, want) <= TOL, max_rel(y, want)


@pytest.mark.slow
def test_cfg5_rows_and_full_properties():
    """cfg5 [4096,128256] N(0,4) QuAKE2, every row: bit-exact against the
    restatement in the plan's declared order and within 2e-6 of the fp64-sum
    restatement (row blocks checked on all host cores); the full matrix also
    through size-independent properties (normalisation, row independence)."""
    R = restatement()
    cols = CFG5.cols
    xd = CFG5.device()
    p = qk.SoftmaxParams(temperature=1.0)
    y = qk.softmax_rows(xd, cols, p, K.Quake2)
    torch.cuda.synchronize()
    plan = qk.softmax_plan(cols, True, K.Quake2)
    xs_all = xd.cpu().numpy()
    ys_all = y.cpu().numpy()

    def check(r0, r1):
        sub = slice(r0 * cols, r1 * cols)
        xs, ys = xs_all[sub], ys_all[sub]
        assert_bitexact(ys, R.softmax_rows_ordered(xs, cols, plan, 1.0, QUAKE2),
                        f"cfg5 rows {r0}..{r1 - 1}")
        return max_rel(ys, R.softmax_rows(xs, cols, 1.0, QUAKE2, sum_mode=1))

    from concurrent.futures import ThreadPoolExecutor
    blocks = [(r0, min(CFG5.rows, r0 + 64)) for r0 in range(0, CFG5.rows, 64)]
    with ThreadPoolExecutor(os.cpu_count() or 1) as ex:
        rels = list(ex.map(lambda b: check(*b), blocks))
    assert max(rels) <= TOL, max(rels)
    # reported, not bounded: the reference's own fp32 sequential-sum rounding
    xs, ys = xs_all[: 64 * cols], ys_all[: 64 * cols]
    dev_ref = max_rel(ys, R.softmax_rows(xs, cols, 1.0, QUAKE2, sum_mode=0))
    print(f"cfg5: all {CFG5.rows} rows bit-exact (ordered), max rel vs fp64 sum {max(rels):.3e}; "
          f"deviation from the reference's sequential fp32 sum: {dev_ref:.3e}")
    del xs_all, ys_all
    # full matrix: rows sum to 1 within 4N ulp (acceptance.cpp:225-254), all positive
    ym = y.view(CFG5.rows, cols).double()
    sums = ym.sum(dim=1)
    assert torch.all(y > 0)
    assert torch.max(torch.abs(sums - 1.0)).item() <= 4 * cols * 1.1920928955078125e-07
    # row independence: the last 64 rows computed alone are bit-identical
    tail = xd[-64 * cols:].clone()
    y_tail = qk.softmax_rows(tail, cols, p, K.Quake2)
    assert torch.equal(y_tail, y[-64 * cols:])


def test_general_quad_and_bias_overrides():
    R = restatement()
    cols = 700
    x = (np.random.default_rng(5).standard_normal(40 * cols) * 2).astype(np.float32)
    plan = qk.softmax_plan(cols, True, K.Quake2)
    y = _gpu_softmax(x, cols, 0.5, QUAKE2, quad=MINIMAX)
    assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 0.5, QUAKE2, quad=MINIMAX), "minimax")
    for bias in (True, False):
        for kern in (QUAKE, QUAKE2):
            plan = qk.softmax_plan(cols, True, K(kern))
            y = _gpu_softmax(x, cols, 2.0, kern, bias=bias)
            assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 2.0, kern, bias=int(bias)),
                            f"bias={bias} k={kern}")


@pytest.mark.parametrize("cols", [4, 6, 8, 12, 16, 20, 64, 512, 517, 1024, 1028, 1152, 4096, 5000,
                                  16384, 128256, 262144, 1 << 20])
def test_results_do_not_depend_on_the_address(cols):
    """The reference's output does not depend on where the buffers sit; neither
    does ours: the plan depends on cols only, and rows whose base is not 16-byte
    aligned (every row shares the phase when cols % 4 == 0) run the same chunk
    order with straddling loads and split stores. Input and output offsets of
    0-3 floats, independently: bit-identical to the aligned run and to the
    ordered restatement. Covers every float4 family: thread per row, sub-warp,
    staged smem (1028), two-stage and long-row pipelines, global sweeps (2^20)."""
    R = restatement()
    rows = max(2, min(40, (1 << 22) // cols))
    n = rows * cols
    rng = np.random.default_rng(cols + 5)
    base = (rng.standard_normal(n + 4) * 3).astype(np.float32)
    if n >= 8 * cols:
        base[1 + 3 * cols: 1 + 4 * cols] = rng.uniform(-1e30, 1e30, cols)  # x86 row (offset 1)
    xd_all = torch.from_numpy(base).cuda()
    out_all = torch.empty(n + 4, device="cuda")
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, True, K(kern))
        assert plan["width"] == (4 if cols % 4 == 0 or plan["variant"] == 13 else 1), plan
        ref = None
        for io, oo in ((0, 0), (1, 1), (2, 3), (3, 0), (0, 2), (1, 0)):
            xd = xd_all[io: io + n]
            out = out_all[oo: oo + n]
            out.fill_(7.0)
            qk.softmax_rows(xd, cols, qk.SoftmaxParams(temperature=0.5), K(kern), out=out)
            y = out.cpu().numpy().copy()
            if ref is None or io != 0:
                want = R.softmax_rows_ordered(base[io: io + n], cols, plan, 0.5, kern)
                assert_bitexact(y, want, f"cols={cols} k={kern} in+{io} out+{oo} plan={plan}")
            if io == 0:
                ref = y if ref is None else ref
                assert_bitexact(y, ref, f"cols={cols} k={kern} out offset {oo}")
        # neighbours of the written span are untouched
        out_all.fill_(7.0)
        qk.softmax_rows(xd_all[1: 1 + n], cols, qk.SoftmaxParams(), K(kern), out=out_all[1: 1 + n])
        assert out_all[0].item() == 7.0 and out_all[n + 1].item() == 7.0


@pytest.mark.parametrize("cols", [64, 63, 1001, 50257])
def test_extreme_rows_match_reference_conversion(cols):
    """Huge-magnitude rows: the reference's cvttss2si out-of-range behaviour is emulated
    (float4 and scalar-lane kernels: cols % 4 != 0 rows are not 16-byte aligned)."""
    R = restatement()
    x = np.concatenate([np.random.default_rng(1).uniform(-1e30, 1e30, cols),
                        np.random.default_rng(2).uniform(1e9, 2e9, cols),
                        np.random.default_rng(3).uniform(-5, 5, cols)]).astype(np.float32)
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, True, K(kern))
        y = _gpu_softmax(x, cols, 1.0, kern)
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 1.0, kern), "extreme rows")


@pytest.mark.parametrize("cols", [7, 63, 257, 1001, 4097, 50257])
def test_unaligned_rows_clamp_and_division_paths(cols):
    """Rows of cols % 4 != 0 (scalar lanes): narrow rows (no element reaches v_min:
    clamp-free exps, proven fast division), wide rows (clamped tails, quotients near
    the subnormal range: checked division), both kinds and temperatures."""
    R = restatement()
    rng = np.random.default_rng(cols)
    rows = max(4, min(48, (1 << 21) // cols))
    narrow = rng.standard_normal(rows * cols)
    wide = rng.uniform(-300, 40, rows * cols)
    for x in (narrow, wide):
        x = x.astype(np.float32)
        for kern in (QUAKE, QUAKE2):
            plan = qk.softmax_plan(cols, cols % 4 == 0, K(kern))
            for t in (0.125, 1.0):
                y = _gpu_softmax(x, cols, t, kern)
                assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, t, kern),
                                f"cols={cols} k={kern} t={t}")


def test_reference_properties():
    """tests/test_nonlin.cpp:42-62 (uniform rows), :191-204 (clamped elements)."""
    for kern in (K.Exact, K.Quake, K.Quake2):
        for c in (0.0, 5.25, -3.0):
            for n in (1, 2, 4, 7, 16, 4096):
                y = qk.softmax_row(np.full(n, c, np.float32), qk.SoftmaxParams(), kern)
                assert np.all(y == y[0])
                if n <= 16:
                    assert abs(y[0] - 1.0 / n) <= 2 * np.spacing(np.float32(1.0 / n))
    v = np.array([0.0, -500.0, 3.0, -1000.0], np.float32)
    for kern in (K.Quake, K.Quake2):
        y = qk.softmax_row(v, qk.SoftmaxParams(temperature=4.0), kern)
        assert np.all(np.isfinite(y)) and np.all(y >= 0)
        assert y[1] <= 2.0**-120 and y[3] <= 2.0**-120


def test_non_finite_rejected_and_out_untouched():
    """nonlin.cpp:43-55 + :176-180: every row validated before anything is written."""
    x = np.random.default_rng(0).standard_normal(64 * 512).astype(np.float32)
    for bad in (np.nan, np.inf, -np.inf):
        xb = x.copy()
        xb[40 * 512 + 7] = bad
        out = np.full_like(xb, 123.0)
        with pytest.raises(ValueError, match="softmax: non-finite input"):
            qk.softmax_rows(xb, 512, qk.SoftmaxParams(), K.Quake2, out=out)
        assert np.all(out == 123.0)
    with pytest.raises(ValueError, match="softmax: non-finite input"):
        qk.softmax_row(np.array([1.0, np.nan], np.float32), qk.SoftmaxParams(), K.Quake)
    xd = torch.from_numpy(xb).cuda()
    with pytest.raises(ValueError, match="non-finite"):
        qk.softmax_rows(xd, 512, qk.SoftmaxParams(), K.Quake2)


@pytest.mark.parametrize("cols", [512, 128256, 262144])
def test_exact_kernel_close_to_reference(cols):
    """Exact (expf) softmax through every pipeline (warp, two-stage, long-row)."""
    R = restatement()
    rows = max(4, min(64, (1 << 21) // cols))
    x = (np.random.default_rng(9).standard_normal(rows * cols) * 2).astype(np.float32)
    from oracle.oracle import EXACT
    y = _gpu_softmax(x, cols, 0.125, EXACT)
    assert max_rel(y, R.softmax_rows(x, cols, 0.125, EXACT, sum_mode=1)) <= 1e-5


def test_interleaved_shapes_keep_launching():
    """Planning one row length must not invalidate another's launch configuration
    (regression: occupancy queries used to lower the smem attribute)."""
    R = restatement()
    shapes = (128256, 16384, 4096, 300000, 50000, 128256, 2048, 128256)
    for cols in shapes:
        rows = 2 if cols > 100000 else 8
        x = (np.random.default_rng(cols).standard_normal(rows * cols) * 4).astype(np.float32)
        y = _gpu_softmax(x, cols, 1.0, QUAKE2)
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, qk.softmax_plan(cols, True, K.Quake2),
                                                  1.0, QUAKE2), f"cols={cols}")


def test_large_host_path_validates_every_row_before_writeback():
    """Host span > one pipeline chunk: every chunk is validated by the device max
    pass before any result is copied back (host_api.cpp). A bad value anywhere —
    first, middle or last chunk — must leave `out` untouched, and clean results
    equal the device path bit for bit (nonlin.cpp:176-180)."""
    cols = 65536
    rows = 600  # 39.3M elements: three 16M-element chunks
    x = (np.random.default_rng(17).standard_normal(rows * cols) * 4).astype(np.float32)
    y = qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2)
    yd = qk.softmax_rows(torch.from_numpy(x).cuda(), cols, qk.SoftmaxParams(), K.Quake2)
    assert_bitexact(y, yd.cpu().numpy(), "host overlap path vs device path")
    for pos in (5, rows * cols // 2 + 1, rows * cols - 3):
        for bad in (np.nan, np.inf, -np.inf):
            xb = x.copy()
            xb[pos] = bad
            out = np.full_like(xb, 123.0)
            with pytest.raises(ValueError, match="softmax: non-finite input"):
                qk.softmax_rows(xb, cols, qk.SoftmaxParams(), K.Quake2, out=out)
            assert np.all(out == 123.0), (pos, bad)
    # the library stays usable after a rejected call
    y2 = qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2)
    assert_bitexact(y2, y, "after a rejected call")


@pytest.mark.parametrize("cols", [202048, 262144, 300000])
def test_long_row_pipeline_is_default_and_bitexact(cols):
    """Long vocab rows take the one-stage long-row pipeline (kPipeL2) and keep the
    declared order: bit-exact against the ordered restatement of its plan, with
    more rows than resident clusters so every cluster runs several rows (stage
    refills, both exchange parities)."""
    R = restatement()
    plan = qk.softmax_plan(cols, True, K.Quake2)
    assert plan["variant"] == 6 and plan["stages"] == 1, plan
    rows = 2 * plan["resident"] + 3
    x = (np.random.default_rng(cols + 11).standard_normal(rows * cols) * 4).astype(np.float32)
    y = _gpu_softmax(x, cols, 1.0, QUAKE2)
    assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 1.0, QUAKE2), f"L2 cols={cols}")
    assert max_rel(y, R.softmax_rows(x, cols, 1.0, QUAKE2, sum_mode=1)) <= TOL


@pytest.mark.parametrize("cols,pf", [(16384, "0"), (128256, "0"), (128256, "2"), (50000, "1")])
def test_long_row_pipeline_forced_keeps_the_order(cols, pf, plan_opts):
    """kPipeL2 forced (QK_SM_L2=1) on shorter rows, with and without L2 bulk
    prefetch: both kernel kinds, both temperatures, bit-exact."""
    plan_opts(QK_SM_L2=1, QK_SM_PF=int(pf))
    R = restatement()
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, True, K(kern))
        assert plan["variant"] == 6, plan
        rows = min(3 * plan["resident"] + 1, (1 << 24) // cols)
        x = (np.random.default_rng(cols + 3).standard_normal(rows * cols) * 3).astype(np.float32)
        for t in (0.125, 1.0):
            y = _gpu_softmax(x, cols, t, kern)
            assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, t, kern),
                            f"forced L2 cols={cols} k={kern} t={t} pf={pf}")


def test_long_row_pipeline_extreme_and_non_finite_rows():
    """kPipeL2 rows on the x86-emulation path (huge magnitudes) and the clamp path
    stay bit-exact; a non-finite value in any row raises the flag."""
    R = restatement()
    cols = 262144
    rng = np.random.default_rng(4)
    rows = [rng.uniform(-1e30, 1e30, cols), rng.uniform(1e9, 2e9, cols),
            rng.standard_normal(cols) * 40, rng.standard_normal(cols)]
    x = np.concatenate(rows).astype(np.float32)
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, True, K(kern))
        assert plan["variant"] == 6
        y = _gpu_softmax(x, cols, 1.0, kern)
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 1.0, kern), f"extreme L2 k={kern}")
    for bad in (np.nan, np.inf):
        xb = x.copy()
        xb[3 * cols + 77] = bad
        xd = torch.from_numpy(xb).cuda()
        with pytest.raises(ValueError, match="non-finite"):
            qk.softmax_rows(xd, cols, qk.SoftmaxParams(), K.Quake2)


@pytest.mark.parametrize("cols", [1, 2, 3, 4, 5, 7, 8, 12, 15, 16, 17, 24, 31, 32, 33, 48, 63, 64,
                                  65])
def test_short_rows_mixed_paths(cols):
    """Short rows (one thread per row, smem-staged rows, sub-warp lanes, row spans):
    bit-exact against the ordered restatement, with a row count that leaves dead
    lanes in the last warp, and x86-emulated (huge-magnitude), clamped and
    ordinary rows interleaved so neighbouring rows in one warp take different paths."""
    R = restatement()
    rng = np.random.default_rng(cols + 100)
    rows = 1003
    x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
    x[1::7] = rng.uniform(-1e30, 1e30, (len(x[1::7]), cols))  # x86 conversion rows
    x[2::7] = rng.uniform(1e9, 2e9, (len(x[2::7]), cols))
    x[3::7] = rng.uniform(-300, 40, (len(x[3::7]), cols))      # clamped tails
    x = x.ravel()
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, cols % 4 == 0, K(kern))
        for t in (0.125, 1.0):
            y = _gpu_softmax(x, cols, t, kern)
            assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, t, kern),
                            f"cols={cols} k={kern} t={t} plan={plan}")
            if plan["variant"] == 9:  # one thread per row: the reference's own order
                assert plan["lanes"] == 1
                assert_bitexact(y, R.softmax_rows(x, cols, t, kern, sum_mode=0),
                                f"thread-per-row vs the reference's sequential sum, cols={cols}")
    from oracle.oracle import EXACT
    y = _gpu_softmax(x[: 40 * cols] / 1e20 if cols > 0 else x, cols, 1.0, EXACT)
    assert np.all(np.isfinite(y))
    # a non-finite value in one row of a packed warp raises the flag
    xb = x.copy()
    xb[5 * cols] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        qk.softmax_rows(torch.from_numpy(xb).cuda(), cols, qk.SoftmaxParams(), K.Quake2)


@pytest.mark.parametrize("cols", [1, 3, 8, 17, 31, 32, 33, 48, 63, 64])
def test_rows_staged_in_smem_sequential_order(cols, plan_opts):
    """kRowsSmem (one thread per row, rows staged through shared memory) keeps the
    reference's sequential order: bit-exact against the reference-order restatement
    for a row count that ends in a partial CTA, with x86 and clamped rows mixed in."""
    plan_opts(QK_SM_ROWSMEM=1)
    R = restatement()
    rng = np.random.default_rng(cols + 7)
    rows = 700
    x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
    x[1::9] = rng.uniform(-1e30, 1e30, (len(x[1::9]), cols))
    x[4::9] = rng.uniform(-300, 40, (len(x[4::9]), cols))
    x = x.ravel()
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, cols % 4 == 0, K(kern))
        assert plan["variant"] == 10 and plan["lanes"] == 1
        for t in (0.125, 1.0):
            y = _gpu_softmax(x, cols, t, kern)
            assert_bitexact(y, R.softmax_rows(x, cols, t, kern, sum_mode=0),
                            f"rows-smem vs the reference's sequential sum, cols={cols} t={t}")


@pytest.mark.parametrize("cols", [20, 32, 64, 100, 128, 256, 512, 1000, 1024])
def test_subwarp_rows_keep_the_declared_order(cols, plan_opts):
    """kSubWarp (G lanes per aligned row, chunks l, l+G, ... per lane; QK_SM_SUBWARP=1):
    bit-exact against the ordered restatement of its plan, x86 and clamped rows
    interleaved, a partial last warp."""
    plan_opts(QK_SM_SUBWARP=1)
    R = restatement()
    rng = np.random.default_rng(cols + 31)
    rows = 509
    x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
    x[1::9] = rng.uniform(-1e30, 1e30, (len(x[1::9]), cols))
    x[4::9] = rng.uniform(-300, 40, (len(x[4::9]), cols))
    x = x.ravel()
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, True, K(kern))
        assert plan["variant"] == 11, plan
        for t in (0.125, 1.0):
            y = _gpu_softmax(x, cols, t, kern)
            assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, t, kern),
                            f"subwarp cols={cols} k={kern} t={t} plan={plan}")


@pytest.mark.parametrize("cols", [7, 16, 31, 77, 127, 128, 257, 512, 1001, 4097, 16384, 50257,
                                  128256, 262144])
def test_in_place_matches_out_of_place(cols):
    """out aliasing the input (as the reference's span API permits): every kernel
    family reads a row (or tile) completely before writing it, so in-place results
    equal out-of-place ones bit for bit."""
    rows = max(3, min(200, (1 << 22) // cols))
    x = torch.randn(rows * cols, device="cuda", generator=torch.Generator("cuda").manual_seed(cols)) * 3
    p = qk.SoftmaxParams(temperature=0.5)
    y = qk.softmax_rows(x, cols, p, K.Quake2)
    xi = x.clone()
    qk.softmax_rows(xi, cols, p, K.Quake2, out=xi)
    torch.cuda.synchronize()
    assert torch.equal(y.view(torch.int32), xi.view(torch.int32)), cols


@pytest.mark.parametrize("cols", [17, 21, 31, 33, 63, 66, 97, 130, 161, 197, 257, 513, 1001, 1535])
@pytest.mark.parametrize("rows", [1, 37, 300])
def test_row_spans_keep_the_declared_order(cols, rows, plan_opts):
    """kSpan (row spans through smem, row-relative float4 chunks with a partial
    last chunk; default for unaligned 17-192 columns, QK_SM_SPAN=2 up to 1536):
    bit-exact against the ordered restatement with partial last spans, x86 and
    clamped rows interleaved, and at input/output offsets of 0-3 floats."""
    plan_opts(QK_SM_SPAN=2)
    R = restatement()
    rng = np.random.default_rng(cols * 13 + rows)
    x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
    x[1::9] = rng.uniform(-1e30, 1e30, (len(x[1::9]), cols))
    x[4::9] = rng.uniform(-300, 40, (len(x[4::9]), cols))
    x = x.ravel()
    n = x.size
    for kern in (QUAKE, QUAKE2):
        plan = qk.softmax_plan(cols, True, K(kern))
        if cols % 4:
            assert plan["variant"] == 13 and plan["width"] == 4, plan
        want = R.softmax_rows_ordered(x, cols, plan, 0.5, kern)
        for io, oo in ((0, 0), (1, 3), (2, 2), (3, 1)):
            xb = torch.zeros(n + 4, device="cuda")
            xb[io:io + n] = torch.from_numpy(x).cuda()
            ob = torch.full((n + 4,), 5.0, device="cuda")
            qk.softmax_rows(xb[io:io + n], cols, qk.SoftmaxParams(temperature=0.5), K(kern),
                            out=ob[oo:oo + n])
            assert_bitexact(ob[oo:oo + n].cpu().numpy(), want,
                            f"span cols={cols} rows={rows} k={kern} in+{io} out+{oo}")
            assert ob[:oo].eq(5.0).all() and ob[oo + n:].eq(5.0).all()
    xb = x.copy()
    xb[-1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        qk.softmax_rows(torch.from_numpy(xb).cuda(), cols, qk.SoftmaxParams(), K.Quake2)


@pytest.mark.parametrize("cols", [33, 47, 64, 65, 97, 127, 128, 129, 161, 193, 197, 256, 257, 321, 385,
                                  512, 513, 640, 769, 1001, 1024, 1027, 2047, 2305, 4099, 8191,
                                  16387, 27999])
@pytest.mark.parametrize("rows", [1, 37, 300])
def test_warp_rings_keep_the_declared_order(cols, rows, plan_opts):
    """kWarpRing (per-agent TMA rings of row spans; the register-resident form
    with G lanes per row up to 1024 columns, three smem sweeps per row above,
    by agents of 1-8 warps): bit-exact against the ordered restatement (width
    1, `lanes` lanes) with partial last jobs, x86 and clamped rows interleaved,
    at input/output offsets of 0-3 floats (equal and different phases), with
    2- and 3-buffer rings and every agent size."""
    R = restatement()
    rng = np.random.default_rng(cols * 17 + rows)
    x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
    x[1::9] = rng.uniform(-1e30, 1e30, (len(x[1::9]), cols))
    x[4::9] = rng.uniform(-300, 40, (len(x[4::9]), cols))
    x = x.ravel()
    n = x.size
    sets = [dict(), dict(QK_SM_RING_NB=3, QK_SM_RING_REGS=0, QK_SM_RING_AW=1), dict(QK_SM_RING_NB=2)]
    if cols > 1024:
        sets += [dict(QK_SM_RING_AW=aw) for aw in (2, 4, 8)]
    for opts in sets:
        plan_opts(QK_SM_RING=1, **opts)
        for kern in (QUAKE, QUAKE2):
            plan = qk.softmax_plan(cols, True, K(kern))
            if opts and plan["variant"] != 14:
                continue  # the forced ring depth / agent size does not fit rows this long
            assert plan["variant"] == 14 and plan["width"] == 1, plan
            if plan["vpt"] > 0:  # register form: G lanes per row, vpt elements per lane
                assert cols <= 1024 and "QK_SM_RING_REGS" not in opts, plan
                assert plan["lanes"] * (plan["vpt"] - 4) < cols <= plan["lanes"] * plan["vpt"], plan
                assert plan["lanes"] == (4 if cols <= 128 else 8 if cols <= 256 else 16 if cols <= 512 else 32)
            else:                # three sweeps by an agent of lanes/32 warps
                assert plan["lanes"] == 32 * opts.get("QK_SM_RING_AW", plan["lanes"] // 32), plan
            want = R.softmax_rows_ordered(x, cols, plan, 0.5, kern)
            for io, oo in ((0, 0), (1, 3), (2, 2), (3, 1), (1, 1)):
                xb = torch.zeros(n + 4, device="cuda")
                xb[io:io + n] = torch.from_numpy(x).cuda()
                ob = torch.full((n + 4,), 5.0, device="cuda")
                qk.softmax_rows(xb[io:io + n], cols, qk.SoftmaxParams(temperature=0.5), K(kern),
                                out=ob[oo:oo + n])
                assert_bitexact(ob[oo:oo + n].cpu().numpy(), want,
                                f"ring cols={cols} rows={rows} k={kern} {opts} {plan} in+{io} out+{oo}")
                assert ob[:oo].eq(5.0).all() and ob[oo + n:].eq(5.0).all()
        for k in opts:
            qk.set_plan_override(k, 0, clear=True)
    xb = x.copy()
    xb[-1] = np.nan
    with pytest.raises(ValueError, match="non-finite"):
        qk.softmax_rows(torch.from_numpy(xb).cuda(), cols, qk.SoftmaxParams(), K.Quake2)


def test_every_unaligned_row_length_up_to_1100_bitexact():
    """Every row length of cols % 4 != 0 from 17 to 1100 columns with the default
    planner (row spans, then every register shape of the warp rings and its
    boundaries, then the first three-sweep lengths): bit-exact against the
    ordered restatement, a partial last job included."""
    R = restatement()
    rng = np.random.default_rng(11)
    rows = 45
    for cols in range(17, 1101):
        if cols % 4 == 0:
            continue
        x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32)
        x[3] = rng.uniform(-300, 40, cols)
        x = x.ravel()
        plan = qk.softmax_plan(cols, False, K.Quake2)
        assert plan["variant"] == (13 if cols <= 32 else 14), (cols, plan)
        y = _gpu_softmax(x, cols, 1.0, QUAKE2)
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 1.0, QUAKE2), f"cols={cols} {plan}")


def test_unaligned_row_lengths_up_to_28000_bitexact():
    """Row lengths of cols % 4 != 0 sampled from 1101 to 28000 columns (every
    agent size of the three-sweep warp rings, the 2- and 3-buffer shapes and the
    last length before the cluster pipeline): bit-exact against the ordered
    restatement with the default planner."""
    R = restatement()
    rng = np.random.default_rng(12)
    rows = 7
    lengths = [c for c in list(range(1101, 28001, 61)) + [27998, 27999] if c % 4]
    seen = set()
    for cols in lengths:
        x = (rng.standard_normal((rows, cols)) * 3).astype(np.float32).ravel()
        plan = qk.softmax_plan(cols, False, K.Quake2)
        assert plan["variant"] == 14 and plan["vpt"] == 0, (cols, plan)
        seen.add((plan["lanes"], plan["stages"]))
        y = _gpu_softmax(x, cols, 1.0, QUAKE2)
        assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 1.0, QUAKE2), f"cols={cols} {plan}")
    assert {l for l, _ in seen} == {32, 64, 128, 256}, seen


@pytest.mark.parametrize("cols", [77, 197, 513, 1537, 4099, 12001])
def test_every_kernel_kind_on_the_warp_rings(cols):
    """Every kernel kind on rows of cols % 4 != 0 (the warp rings' register and
    three-sweep forms, every agent size): Exact / expf / __expf within their
    tolerances of the fp64-sum restatement, the general (minimax) quad bit-exact
    against the ordered restatement, input/output at different phases."""
    R = restatement()
    rows = max(5, min(64, (1 << 20) // cols))
    x = (np.random.default_rng(cols).standard_normal(rows * cols) * 2).astype(np.float32)
    from oracle.oracle import EXACT
    want = R.softmax_rows(x, cols, 0.125, EXACT, sum_mode=1)
    for kern, tol in ((K.Exact, 1e-5), (K.Expf, 1e-5), (K.FastExp, 5e-5)):
        assert qk.softmax_plan(cols, False, kern)["variant"] == 14
        xd = torch.zeros(x.size + 4, device="cuda")
        xd[1:1 + x.size] = torch.from_numpy(x).cuda()
        y = qk.softmax_rows(xd[1:1 + x.size], cols, qk.SoftmaxParams(temperature=0.125), kern)
        assert max_rel(y.cpu().numpy(), want) <= tol, (cols, kern)
    plan = qk.softmax_plan(cols, False, K.Quake2)
    y = _gpu_softmax(x, cols, 0.5, QUAKE2, quad=MINIMAX)
    assert_bitexact(y, R.softmax_rows_ordered(x, cols, plan, 0.5, QUAKE2, quad=MINIMAX), "minimax")
