"""GPU: the multi-GPU split and the host-span driver.

The reference's results do not depend on how the work is partitioned
(parallel.hpp:39-42; tests/test_cli.cpp:194-208 compares QUAKE_THREADS=1 with
the default). Here the split is over GPUs: rows (softmax) or
16-byte element ranges (elementwise), no collective. One GPU runs the 2-, 4-
and 8-way splits two ways:

  * in process: qk_set_device_shards([0]*k) gives the C++ driver k shards on
    device 0 — k host threads, k workspaces, the std::barrier that holds every
    write-back until all shards validated;
  * per rank: each rank's rows (shard.row_shard) launched on its own, from the
    counter-based generator's slice of the input (workloads.py).

Both must equal the unsharded output bit for bit. Also here: the streamed
host path (inputs larger than the workspace), `out` untouched on error for
device `out` spans, torch-stream safety of the Python wrapper and concurrent
multi-shard callers (no deadlock).
"""
import ctypes
import threading

import numpy as np
import pytest
import torch

import paper_2412_00408_b200 as qk
from paper_2412_00408_b200 import _lib
from paper_2412_00408_b200.shard import element_shard, row_shard
from paper_2412_00408_b200.workloads import CFG1, CFG4, CFG5
from tests.helpers import assert_bitexact

pytestmark = pytest.mark.gpu
K = qk.KernelChoice


@pytest.fixture(autouse=True)
def _reset_driver():
    yield
    qk.set_devices([])
    qk.set_workspace_limit(0)
    qk.set_host_validation(-1, 64 << 20)


def _same(a, b, what):
    a = a if isinstance(a, np.ndarray) else a.cpu().numpy()
    b = b if isinstance(b, np.ndarray) else b.cpu().numpy()
    assert_bitexact(a, b, what)


@pytest.mark.parametrize("w", [CFG4, CFG5], ids=["cfg4", "cfg5"])
def test_row_split_is_bit_identical(w):
    """cfg4 (49152 x 512) and cfg5 (4096 x 128256) at full size, 1/2/4/8-way."""
    p = qk.SoftmaxParams(temperature=w.temperature)
    kern = K.Quake2
    xd = w.device()
    y1 = qk.softmax_rows(xd, w.cols, p, kern)
    torch.cuda.synchronize()
    x_host = xd.cpu().numpy()
    want = y1.cpu().numpy()
    del y1
    # the generator's shards are the slices of the full draw
    for k in (2, 8):
        r0, r1 = row_shard(w.rows, k - 1, k)
        assert torch.equal(w.device(rows=(r0, r1)).view(torch.int32),
                           xd[r0 * w.cols:r1 * w.cols].view(torch.int32)), k
    for k in (2, 4, 8):
        # per rank: every rank's rows launched alone
        out = torch.empty_like(xd)
        for r in range(k):
            r0, r1 = row_shard(w.rows, r, k)
            sl = slice(r0 * w.cols, r1 * w.cols)
            qk.softmax_rows(w.device(rows=(r0, r1)), w.cols, p, kern, out=out[sl])
        _same(out, want, f"{w.name}: {k} per-rank launches")
        del out
        # in process: k shards of the C++ driver (host spans)
        qk.set_device_shards([0] * k)
        assert qk.get_devices() == [0] * k
        y = qk.softmax_rows(x_host, w.cols, p, kern)
        _same(y, want, f"{w.name}: {k} in-process shards")
        del y
        qk.set_devices([])
    qk.release_workspace()


def test_element_split_is_bit_identical():
    x = CFG1.device()
    x_host = x.cpu().numpy()
    c = qk.natural_exp_coeffs(False)
    r = qk.clamp_for(c)
    want = qk.quake2_buffer(x, c, qk.QuadCoeffs.continuity(), r).cpu().numpy()
    want_g = qk.gelu_buffer(x, K.Quake).cpu().numpy()
    for k in (2, 4, 8):
        spans = [element_shard(CFG1.n, i, k) for i in range(k)]
        assert all(a % 4 == 0 for a, _ in spans)
        for a, b in spans:
            assert torch.equal(CFG1.device((a, b)).view(torch.int32), x[a:b].view(torch.int32))
        qk.set_device_shards([0] * k)
        _same(qk.quake2_buffer(x_host, c, qk.QuadCoeffs.continuity(), r), want, f"quake2 {k}")
        _same(qk.gelu_buffer(x_host, K.Quake), want_g, f"gelu {k}")
        qk.set_devices([])


def test_in_process_shards_validate_before_any_write_back():
    """A non-finite value in the LAST shard: no shard writes back (barrier)."""
    cols = 4096
    x = CFG5.host(rows=(0, 64))[: 64 * cols].copy()
    for k in (2, 4, 8):
        qk.set_device_shards([0] * k)
        for pos in (7, x.size - 5):
            xb = x.copy()
            xb[pos] = np.nan
            out = np.full_like(xb, 123.0)
            with pytest.raises(ValueError, match="non-finite"):
                qk.softmax_rows(xb, cols, qk.SoftmaxParams(), K.Quake2, out=out)
            assert np.all(out == 123.0), (k, pos)
        y = qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2)
        assert np.all(np.isfinite(y))


def test_streamed_host_path_matches_resident():
    """Inputs larger than the workspace stream through chunk rings (softmax:
    validation pass, then H2D -> softmax -> D2H): same bits, same contract."""
    cols = 65536
    rows = 600  # 157 MB: several 64 MiB chunks
    x = CFG5.host((0, rows * cols))
    want = qk.softmax_rows(torch.from_numpy(x).cuda(), cols, qk.SoftmaxParams(),
                           K.Quake2).cpu().numpy()
    for k in (1, 3):
        qk.set_device_shards([0] * k)
        qk.set_workspace_limit(32 << 20)
        qk.release_workspace()
        y = qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2)
        _same(y, want, f"streamed softmax, {k} shards")
        for pos in (3, rows * cols // 2, rows * cols - 1):
            xb = x.copy()
            xb[pos] = np.inf
            out = np.full_like(xb, 123.0)
            with pytest.raises(ValueError, match="non-finite"):
                qk.softmax_rows(xb, cols, qk.SoftmaxParams(), K.Quake2, out=out)
            assert np.all(out == 123.0), pos
        # device output, host input, streamed: validated before the first write
        od = torch.full((rows * cols,), 123.0, device="cuda")
        xb = x.copy()
        xb[-2] = np.nan
        with pytest.raises(ValueError, match="non-finite"):
            qk.softmax_rows(xb, cols, qk.SoftmaxParams(), K.Quake2, out=od)
        assert bool(torch.all(od == 123.0))
        qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2, out=od)
        _same(od, want, "streamed, device out")
        # elementwise through the ring
        xe = CFG1.host((0, 40 << 20))
        ye = qk.logistic_buffer(xe, K.Quake2)
        _same(ye, qk.logistic_buffer(torch.from_numpy(xe).cuda(), K.Quake2), "ring logistic")
        qk.set_workspace_limit(0)
        qk.set_devices([])
    qk.release_workspace()


def test_overlapped_write_back_keeps_bits_and_contract():
    """Pinned host spans on both sides: host threads validate the shard from
    its last element backwards while the device validates the uploaded chunks
    from the front, and the download starts when the fronts meet
    (qk_set_host_validation). Same bits as the device path; a non-finite value
    anywhere (device side, host side, the meeting region) is reported before
    anything reaches `out` (nonlin.cpp:176-180)."""
    L = _lib.lib()
    cols, rows = 4096, 10000  # 164 MB: three 64 MiB chunks
    n = rows * cols
    xd = CFG5.device((0, n))
    want = qk.softmax_rows(xd, cols, qk.SoftmaxParams(), K.Quake2)
    hx = xd.cpu().pin_memory()
    hy = torch.empty_like(hx).pin_memory()
    prm = qk.SoftmaxParams()._c()
    torch.cuda.synchronize()

    def call(src, dst):
        return L.qk_softmax_rows(src.data_ptr(), n, cols, ctypes.byref(prm), int(K.Quake2),
                                 dst.data_ptr(), n)

    for threads, shards in ((4, 1), (2, 2), (0, 1), (-1, 1)):
        qk.set_device_shards([0] * shards)
        qk.set_host_validation(threads, 1 << 20)
        for rep in range(3):
            hy.fill_(-7.0)
            assert call(hx, hy) == 0, _lib.last_error()
            assert torch.equal(hy.cuda(), want), (threads, shards, rep)
        for pos in (5, n // 3, n // 2 + 17, n - 3 * cols, n - 1):
            hb = hx.clone().pin_memory()
            hb[pos] = float("nan") if pos % 2 else float("-inf")
            hy.fill_(123.0)
            assert call(hb, hy) == 5, (threads, shards, pos, _lib.last_error())
            assert bool(torch.all(hy == 123.0)), (threads, shards, pos)
        # and the next clean call is unaffected
        assert call(hx, hy) == 0
        assert torch.equal(hy.cuda(), want)
    qk.release_workspace()


def test_host_span_device_pointers_leave_out_untouched_on_error():
    """qk_softmax_rows (the host-span C-ABI) with a device `out`: validated
    before anything is written, for host and device inputs."""
    L = _lib.lib()
    cols, rows = 512, 64
    x = CFG4.host((0, rows * cols))
    x[40 * cols + 3] = np.nan
    prm = qk.SoftmaxParams()._c()
    for in_dev in (False, True):
        xd = torch.from_numpy(x).cuda() if in_dev else None
        od = torch.full((rows * cols,), 123.0, device="cuda")
        xp = xd.data_ptr() if in_dev else x.ctypes.data
        torch.cuda.synchronize()
        st = L.qk_softmax_rows(xp, x.size, cols, ctypes.byref(prm), int(K.Quake2),
                               od.data_ptr(), x.size)
        assert st == 5, (st, _lib.last_error())
        assert bool(torch.all(od == 123.0)), in_dev
    # and a clean call through the same path writes the device out
    xc = CFG4.host((0, rows * cols))
    xd = torch.from_numpy(xc).cuda()
    od = torch.empty_like(xd)
    torch.cuda.synchronize()
    assert L.qk_softmax_rows(xd.data_ptr(), xc.size, cols, ctypes.byref(prm), int(K.Quake2),
                             od.data_ptr(), xc.size) == 0
    _same(od, qk.softmax_rows(xd, cols, qk.SoftmaxParams(), K.Quake2), "host-span, device spans")


def test_wrapper_waits_for_pending_producer():
    """softmax_rows / softmax_row / elementwise with a CUDA input and a host
    `out` run on the library's streams: the wrapper must wait for work still
    queued on torch's stream (here: a sleep, then the copy that fills x)."""
    cols, rows = 4096, 256
    src = CFG5.device((0, rows * cols))
    want = qk.softmax_rows(src, cols, qk.SoftmaxParams(), K.Quake2).cpu().numpy()
    want_e = qk.logistic_buffer(src, K.Quake).cpu().numpy()
    for _ in range(3):
        x = torch.zeros_like(src)
        torch.cuda._sleep(50_000_000)  # ~25 ms of GPU time on the current stream
        x.copy_(src)
        out = np.empty(rows * cols, np.float32)
        qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2, out=out)
        _same(out, want, "softmax after a pending producer")
        x2 = torch.zeros_like(src)
        torch.cuda._sleep(50_000_000)
        x2.copy_(src)
        oe = np.empty(rows * cols, np.float32)
        qk.logistic_buffer(x2, K.Quake, out=oe)
        _same(oe, want_e, "logistic after a pending producer")
        # a non-float32 input converted on the fly: the converted copy must
        # outlive the call and be complete before the library reads it
        x3 = torch.zeros(rows * cols, dtype=torch.float64, device="cuda")
        torch.cuda._sleep(50_000_000)
        x3.copy_(src.double())
        o3 = np.empty(rows * cols, np.float32)
        qk.softmax_rows(x3, cols, qk.SoftmaxParams(), K.Quake2, out=o3)
        _same(o3, want, "converted input after a pending producer")


def test_concurrent_multi_shard_callers_do_not_deadlock():
    """Two threads, each a multi-shard host-span call over the same devices
    (workspaces are locked in one global order by the calling thread)."""
    cols = 8192
    x = CFG5.host((0, 128 * cols))
    want = qk.softmax_rows(torch.from_numpy(x).cuda(), cols, qk.SoftmaxParams(),
                           K.Quake2).cpu().numpy()
    qk.set_device_shards([0, 0, 0])
    errs, outs = [], []

    def worker():
        try:
            for _ in range(6):
                outs.append(qk.softmax_rows(x, cols, qk.SoftmaxParams(), K.Quake2))
        except Exception as e:  # pragma: no cover
            errs.append(e)

    ts = [threading.Thread(target=worker) for _ in range(3)]
    for t in ts:
        t.start()
    for t in ts:
        t.join(timeout=120)
    assert not any(t.is_alive() for t in ts), "deadlock"
    assert not errs, errs
    for y in outs:
        _same(y, want, "concurrent")
