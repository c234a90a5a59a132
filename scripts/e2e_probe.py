"""Probe (not product): wall time of host-span cfg5 softmax calls (pinned buffers).

The log in profiles/r01_e2e_host_scan_probe.log was taken with a since-removed
host-scan variant whose QK_HOST_SCAN_DEBUG=1 output shows when the scan and
the device check decided."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import paper_2412_00408_b200 as qk  # noqa: E402
from paper_2412_00408_b200 import _lib  # noqa: E402
from paper_2412_00408_b200.workloads import CFG5  # noqa: E402

L = _lib.lib()
x = CFG5.device()
hx = x.cpu().pin_memory()
hy = torch.empty_like(hx).pin_memory()
prm = qk.SoftmaxParams()._c()
for i in range(4):
    t0 = time.perf_counter()
    st = L.qk_softmax_rows(hx.data_ptr(), hx.numel(), CFG5.cols, ctypes.byref(prm), 2,
                           hy.data_ptr(), hy.numel())
    dt = time.perf_counter() - t0
    print(f"call {i}: status {st} {dt * 1e3:.1f} ms -> {hx.numel() / dt / 1e9:.2f} Gelem/s",
          file=sys.stderr, flush=True)
