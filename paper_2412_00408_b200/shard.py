"""Row / element sharding for one-process-per-GPU runs (torchrun).

The reference's only parallelism is parallel_chunks (core/include/quake/
parallel.hpp:43-68): fixed chunks whose results never depend on the
partition. The GPU build shards whole rows (softmax) or 16-byte-aligned
element ranges (elementwise) across ranks; rows and elements are
independent, so there is no data-path collective. The same
partition rule is used in-process by the C++ multi-GPU driver
(host_api.cpp make_shards).
"""
from __future__ import annotations


def shard_range(n_units: int, rank: int, world: int, align: int = 1) -> tuple[int, int]:
    """[begin, end) of `rank`'s contiguous shard of n_units units.

    Boundaries are multiples of `align` units (the last shard takes the
    remainder); the first (units % world) ranks get one extra aligned block.
    """
    if world <= 0 or not 0 <= rank < world:
        raise ValueError("bad rank/world")
    blocks = (n_units + align - 1) // align
    begin = 0
    for r in range(world):
        b = blocks // world + (1 if r < blocks % world else 0)
        end = min(n_units, begin + b * align)
        if r == rank:
            return begin, end
        begin = end
    raise AssertionError("unreachable")


def row_shard(rows: int, rank: int, world: int) -> tuple[int, int]:
    """Softmax: whole rows, never split across GPUs."""
    return shard_range(rows, rank, world, 1)


def element_shard(n: int, rank: int, world: int) -> tuple[int, int]:
    """Elementwise ops: 4-element (16-byte) aligned ranges."""
    return shard_range(n, rank, world, 4)
