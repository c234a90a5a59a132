"""e2e of qk_softmax_rows (cfg5, pinned host spans) with and without the
overlapped write-back (qk_set_host_validation): wall clock per call."""
import ctypes
import json
import sys
import time

import torch

import paper_2412_00408_b200 as qk
from paper_2412_00408_b200 import _lib
from paper_2412_00408_b200.workloads import CONFIGS

L = _lib.lib()
w = CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "cfg5_softmax_vocab"]
x = w.device()
n = x.numel()
hx = x.cpu().pin_memory()
hy = torch.empty_like(hx).pin_memory()
prm = qk.SoftmaxParams(temperature=w.temperature)._c()
kern = int(qk.KernelChoice.Quake2)
want = qk.softmax_rows(x, w.cols, qk.SoftmaxParams(temperature=w.temperature), qk.KernelChoice.Quake2)
torch.cuda.synchronize()


def call():
    st = L.qk_softmax_rows(hx.data_ptr(), n, w.cols, ctypes.byref(prm), kern, hy.data_ptr(), n)
    assert st == 0, _lib.last_error()


for threads in (0, 4, 8, 12, 16, -1, 0, -1):
    qk.set_host_validation(threads, 64 << 20)
    call()
    ts = []
    for _ in range(5):
        t0 = time.perf_counter()
        call()
        ts.append(time.perf_counter() - t0)
    assert torch.equal(hy.cuda(), want)
    print(json.dumps({"workload": w.name, "scan_threads": threads, "min_ms": min(ts) * 1e3,
                      "mean_ms": sum(ts) / len(ts) * 1e3, "gelem_s": n / min(ts) / 1e9}), flush=True)
