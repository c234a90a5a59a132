"""The stream-ordered device operators (qk_*_device) inside CUDA graphs.

A serving loop captures its per-step kernels once and replays the graph; the
C-ABI device operators must be capturable (no capture-invalidating call such
as cudaStreamGetDevice on the capturing stream) and a replay must read the
buffers' current contents. Every kernel family is captured — elementwise, G
lanes per row, one thread per row (direct and smem-tiled), row spans, the
warp rings (register form, three sweeps, agents of several warps), the
two-stage pipeline (C = 1 and clusters), the scalar-lane pipeline and the
long-row pipeline — and replays are compared bit for bit with eager launches.
"""
import ctypes

import pytest
import torch

import paper_2412_00408_b200 as qk
from paper_2412_00408_b200 import _lib

pytestmark = pytest.mark.gpu
K = qk.KernelChoice


def _ops(L, sh):
    prm1 = qk.SoftmaxParams(temperature=1.0)._c()
    prm8 = qk.SoftmaxParams(temperature=0.125)._c()

    def ew(fn, kern, extra=()):
        return lambda x, y: fn(x.data_ptr(), y.data_ptr(), x.numel(), int(kern), *extra, sh)

    def sm(cols, prm, kern):
        return lambda x, y: L.qk_softmax_rows_device(x.data_ptr(), x.numel(), cols,
                                                     ctypes.byref(prm), int(kern), y.data_ptr(),
                                                     None, sh)

    return [
        ("exp quake", 1 << 20, ew(L.qk_exp_buffer_device, K.Quake)),
        ("logistic quake2", 1 << 20, ew(L.qk_logistic_buffer_device, K.Quake2, (-1,))),
        ("gelu quake", (1 << 20) + 3, ew(L.qk_gelu_buffer_device, K.Quake, (-1,))),
        ("softmax 512", 512 * 300, sm(512, prm8, K.Quake)),
        ("softmax 16384", 16384 * 40, sm(16384, prm1, K.Quake2)),
        ("softmax 128256", 128256 * 40, sm(128256, prm1, K.Quake2)),
        ("softmax 262144", 262144 * 40, sm(262144, prm1, K.Quake2)),
        ("softmax 50257 (scalar lanes)", 50257 * 40, sm(50257, prm1, K.Quake2)),
        ("softmax 1001 (warp ring, 32 lanes per row)", 1001 * 300, sm(1001, prm1, K.Quake2)),
        ("softmax 48 (sub-warp)", 48 * 3000, sm(48, prm8, K.Quake)),
        ("softmax 197 (warp ring, 8 lanes per row)", 197 * 3001, sm(197, prm1, K.Quake2)),
        ("softmax 513 (warp ring, partial last job)", 513 * 301, sm(513, prm1, K.Quake2)),
        ("softmax 1537 (warp ring, three sweeps)", 1537 * 201, sm(1537, prm1, K.Quake)),
        ("softmax 4099 (warp ring, 4-warp agents)", 4099 * 77, sm(4099, prm1, K.Quake2)),
        ("softmax 77 (row spans)", 77 * 3001, sm(77, prm1, K.Quake2)),
        ("softmax 16 (thread per row)", 16 * 3000, sm(16, prm8, K.Quake2)),
        ("softmax 31 (smem tile)", 31 * 3000, sm(31, prm1, K.Quake2)),
    ]


def test_device_ops_capture_and_replay_bitexact():
    L = _lib.lib()
    stream = torch.cuda.Stream()
    sh = stream.cuda_stream
    ops = _ops(L, sh)
    gen = torch.Generator(device="cuda").manual_seed(3)
    xs = [torch.randn(n, device="cuda", generator=gen) * 3 for _, n, _ in ops]
    ys_eager = [torch.empty_like(x) for x in xs]
    ys_graph = [torch.full_like(x, -1.0) for x in xs]
    with torch.cuda.stream(stream):
        for (name, _, f), x, y in zip(ops, xs, ys_eager):
            assert f(x, y) == 0, (name, _lib.last_error())  # warm: plans and attributes cached
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=stream):
        for (name, _, f), x, y in zip(ops, xs, ys_graph):
            assert f(x, y) == 0, (name, _lib.last_error())
    for round_ in range(2):
        g.replay()
        torch.cuda.synchronize()
        for (name, _, f), y_e, y_g in zip(ops, ys_eager, ys_graph):
            assert torch.equal(y_e.view(torch.int32), y_g.view(torch.int32)), (name, round_)
        # new inputs in place: the replay must read them, and match a fresh eager pass
        for x in xs:
            x.mul_(0.5).add_(0.25)
        with torch.cuda.stream(stream):
            for (name, _, f), x, y in zip(ops, xs, ys_eager):
                assert f(x, y) == 0, (name, _lib.last_error())
        torch.cuda.synchronize()
