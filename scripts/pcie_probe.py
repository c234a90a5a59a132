"""Probe (not product): PCIe H2D / D2H alone and concurrent, pinned 2 GiB; host scan speed."""
import os
import threading
import time

import numpy as np
import torch

n = 1 << 29  # 2 GiB of fp32
h_in = torch.empty(n, dtype=torch.float32).pin_memory()
h_out = torch.empty(n, dtype=torch.float32).pin_memory()
d_a = torch.empty(n, dtype=torch.float32, device="cuda")
d_b = torch.empty(n, dtype=torch.float32, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        t = time.perf_counter()
        fn()
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    return best


gb = n * 4 / 1e9
t_h2d = timed(lambda: d_a.copy_(h_in, non_blocking=True))
t_d2h = timed(lambda: h_out.copy_(d_b, non_blocking=True))


def both():
    with torch.cuda.stream(s1):
        d_a.copy_(h_in, non_blocking=True)
    with torch.cuda.stream(s2):
        h_out.copy_(d_b, non_blocking=True)


t_both = timed(both)
print(f"H2D {gb / t_h2d:.1f} GB/s  D2H {gb / t_d2h:.1f} GB/s  concurrent {2 * gb / t_both:.1f} GB/s "
      f"({t_both * 1e3:.1f} ms for {gb:.2f}+{gb:.2f} GB)")
a = h_in.numpy().view(np.uint32)
print("cpus", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
for nt in (1, 4, 8, 16, 32):
    per = (n + nt - 1) // nt

    def scan(i):
        blk = a[i * per:(i + 1) * per]
        ((blk & 0x7F800000) == 0x7F800000).any()

    t = time.perf_counter()
    th = [threading.Thread(target=scan, args=(i,)) for i in range(nt)]
    [x.start() for x in th]
    [x.join() for x in th]
    dt = time.perf_counter() - t
    print(f"numpy scan {nt:2d} threads: {gb / dt:.1f} GB/s")
