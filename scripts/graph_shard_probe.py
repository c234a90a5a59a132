"""Probe (not product): per-GPU work of every BASELINE config at 1/2/4/8-way sharding,
device time and CUDA-Graph wall clock.

Under torchrun each rank runs its shard on its own GPU with no collective. This
box has one GPU, so rank 0's shard (the largest) is timed here:
  kernel_us — back-to-back launches between one CUDA event pair, / launches;
  graph_wall_us — host wall clock around replays of a CUDA graph holding R
              launches (one per rotating buffer pair), then a synchronize,
              / launches: what a host driving the shard sees, launch overheads
              amortised by the graph;
  eager_wall_us — the same launches issued one by one from Python through the
              C-ABI (ctypes), host wall clock.
Inputs rotate through buffer pairs >= 4x L2 (as bench.per_config), so no
launch reads input left in L2 by an earlier one.
"""
import ctypes
import json
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.shard import element_shard, row_shard  # noqa: E402
from paper_2412_00408_b200.workloads import CONFIGS  # noqa: E402

L = _lib.lib()
K = qk.KernelChoice
l2 = 126 << 20
stream = torch.cuda.Stream()
sh = stream.cuda_stream
peak = json.load(open(os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))),
                                   "MEASURED_PEAKS.json")))["hbm_gbs"]


def launcher(w, x, y, n, kern, prm):
    xp, yp = x.data_ptr(), y.data_ptr()
    if w.op == "exp":
        return lambda: L.qk_exp_buffer_device(xp, yp, n, kern, sh)
    if w.op == "logistic":
        return lambda: L.qk_logistic_buffer_device(xp, yp, n, kern, -1, sh)
    if w.op == "gelu":
        return lambda: L.qk_gelu_buffer_device(xp, yp, n, kern, -1, sh)
    return lambda: L.qk_softmax_rows_device(xp, n, w.cols, ctypes.byref(prm), kern, yp, None, sh)


only = os.environ.get("CONFIGS")
for name, w in CONFIGS.items():
    if only and name not in only.split(","):
        continue
    kern = int(K.Quake2 if name == "cfg5_softmax_vocab" else K.Quake)
    prm = qk.SoftmaxParams(temperature=w.temperature)._c()
    for world in (1, 2, 4, 8):
        if w.op == "softmax":
            r0, r1 = row_shard(w.rows, 0, world)
            n = (r1 - r0) * w.cols
        else:
            e0, e1 = element_shard(w.n, 0, world)
            n = e1 - e0
        pairs = max(2, -(-4 * l2 // (8 * n)))
        xs = [torch.randn(n, device="cuda") * 3 for _ in range(pairs)]
        ys = [torch.empty_like(xs[0]) for _ in range(pairs)]
        fns = [launcher(w, x, y, n, kern, prm) for x, y in zip(xs, ys)]
        reps = max(4, 64 // pairs)
        with torch.cuda.stream(stream):
            for f in fns:  # warm: plans, smem attributes and occupancy queries cached
                assert f() == 0, _lib.last_error()
        torch.cuda.synchronize()
        # device time, back to back
        with torch.cuda.stream(stream):
            a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            a.record(stream)
            for _ in range(reps):
                for f in fns:
                    f()
            b.record(stream)
        torch.cuda.synchronize()
        kern_us = a.elapsed_time(b) * 1e3 / (reps * pairs)
        # eager host wall clock
        t0 = time.perf_counter()
        for _ in range(reps):
            for f in fns:
                f()
        stream.synchronize()
        eager_us = (time.perf_counter() - t0) * 1e6 / (reps * pairs)
        # CUDA graph of one pass over the buffer pairs
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=stream,
                              capture_error_mode=os.environ.get("GRAPH_MODE", "global")):
            for f in fns:
                assert f() == 0, _lib.last_error()
        g.replay()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for _ in range(reps):
            g.replay()
        torch.cuda.synchronize()
        graph_us = (time.perf_counter() - t0) * 1e6 / (reps * pairs)
        gbs = 8 * n / kern_us / 1e3
        print(json.dumps({"config": name, "gpus": world, "elements_per_rank": n,
                          "kernel": "quake2" if kern == int(K.Quake2) else "quake",
                          "kernel_us": round(kern_us, 2), "kernel_gbps": round(gbs, 1),
                          "kernel_frac": round(gbs / peak, 4),
                          "graph_wall_us": round(graph_us, 2), "eager_wall_us": round(eager_us, 2),
                          "implied_job_elements_per_s": w.n / (graph_us * 1e-6),
                          "rotation_buffers": pairs}), flush=True)
        del g, xs, ys, fns
        torch.cuda.empty_cache()
