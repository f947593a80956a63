"""Batch sharding for multi-GPU runs.

Every operator on the fused path is per-sample (conv2d / dense / bias_add /
relu / add / the quantize chains / sum over (2, 3): kernels.cpp:640-716,
609-638, reduce_plan axes), so a batch splits into contiguous slices, one
per GPU, with weights replicated and NO collective on the data path.  The
executor of each rank is specialised at its slice size; the concatenation of
the per-rank outputs equals the unsharded result bit for bit.
"""
from __future__ import annotations

from typing import List, Tuple


def shard_range(total: int, rank: int, world: int) -> Tuple[int, int]:
    """Contiguous slice [start, stop) of `total` samples owned by `rank`;
    sizes differ by at most one (the first total % world ranks get one more)."""
    if world < 1 or not (0 <= rank < world):
        raise ValueError("bad rank %d / world %d" % (rank, world))
    if total < 0:
        raise ValueError("negative batch")
    base, extra = divmod(total, world)
    start = rank * base + min(rank, extra)
    return start, start + base + (1 if rank < extra else 0)


def shard_sizes(total: int, world: int) -> List[int]:
    return [b - a for a, b in (shard_range(total, r, world) for r in range(world))]
