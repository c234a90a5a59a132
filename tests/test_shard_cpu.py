"""CPU: the N>1 path. Rows (softmax) or 16-byte element ranges (elementwise)
are sharded contiguously over ranks with no data-path collective; results must
be identical to the unsharded run (the reference's partition independence,
parallel.hpp:39-42, tests/test_cli.cpp:194-208). Exercised with two gloo
ranks; each rank computes its shard with the CPU oracle (no GPU here) and the
shards are gathered only to check the result."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2412_00408_b200.shard import element_shard, row_shard, shard_range


@pytest.mark.parametrize("n", [0, 1, 5, 7, 64, 1000, 4096, 4097])
@pytest.mark.parametrize("world", [1, 2, 3, 4, 8])
def test_shard_ranges_partition(n, world):
    for align in (1, 4):
        spans = [shard_range(n, r, world, align) for r in range(world)]
        assert spans[0][0] == 0 and spans[-1][1] == n
        for (a, b), (c, d) in zip(spans, spans[1:]):
            assert b == c and a <= b
        for a, b in spans:  # boundaries aligned, except the buffer end itself
            assert a % align == 0 or a == n
            assert b % align == 0 or b == n
        sizes = [b - a for a, b in spans]
        assert max(sizes) - min(sizes) < 2 * align


def test_cfg5_rows_per_gpu():
    # BASELINE cfg5: 4096 rows over 1/2/4/8 GPUs -> 4096/k rows each
    for k in (1, 2, 4, 8):
        assert {b - a for a, b in (row_shard(4096, r, k) for r in range(k))} == {4096 // k}
    assert element_shard(1 << 24, 3, 8) == (3 << 21, 4 << 21)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from oracle.oracle import QUAKE2, Restatement
    R = Restatement()
    rows, cols = 24, 257
    x = (np.random.default_rng(7).standard_normal(rows * cols) * 4).astype(np.float32)
    r0, r1 = row_shard(rows, rank, world)
    mine = R.softmax_rows(x[r0 * cols:r1 * cols], cols, 1.0, QUAKE2)
    # elementwise shard
    n = 1003
    e0, e1 = element_shard(n, rank, world)
    ex = x[:n]
    mine_e = R.gelu_buffer(ex[e0:e1], QUAKE2)
    # gather (test-only) and compare with the unsharded result on rank 0
    sizes = [torch.zeros(1, dtype=torch.int64) for _ in range(world)]
    dist.all_gather(sizes, torch.tensor([mine.size]))
    maxn = int(max(s.item() for s in sizes))
    buf = torch.zeros(maxn)
    buf[:mine.size] = torch.from_numpy(mine)
    parts = [torch.zeros(maxn) for _ in range(world)]
    dist.all_gather(parts, buf)
    parts_e = [None] * world
    dist.all_gather_object(parts_e, mine_e)
    if rank == 0:
        whole = np.concatenate([p[:int(s.item())].numpy() for p, s in zip(parts, sizes)])
        ok = np.array_equal(whole.view(np.uint32),
                            R.softmax_rows(x, cols, 1.0, QUAKE2).view(np.uint32))
        ok_e = np.array_equal(np.concatenate(parts_e).view(np.uint32),
                              R.gelu_buffer(ex, QUAKE2).view(np.uint32))
        q.put((ok, ok_e))
    dist.barrier()
    dist.destroy_process_group()


def test_two_rank_gloo_sharding_is_partition_independent():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    for p in procs:
        p.join(timeout=240)
        assert p.exitcode == 0
    ok, ok_e = q.get(timeout=10)
    assert ok and ok_e
