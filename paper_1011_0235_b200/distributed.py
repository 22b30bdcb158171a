"""Multi-GPU: contiguous byte-range sharding + one allreduce of the 256 counts.

The histogram merge is a commutative monoid (core.py:142-149), and the reference
already partitions contiguously and merges partials (group_ranges kernels.py:311-316,
merge_all core.py:152-156). Across GPUs the same rule applies at word granularity:
rank r of P owns words [r*floor(W/P), (r+1)*floor(W/P)), the last rank the remainder.
Each rank counts its shard with one launch into a device uint64[256]; one
``all_reduce(SUM)`` of 2 KiB over NCCL (NVLink/NVSwitch) joins them. The collective is
latency-bound (tens of microseconds) next to a multi-millisecond per-GPU scan, so
there is no compute/collective fusion to do here: the path shards with no data
exchange and a single tiny reduction at the end.
"""
from __future__ import annotations

import numpy as np

from .kernels import group_ranges


def shard_range(n_bytes: int, rank: int, world: int) -> tuple[int, int]:
    """Byte range [lo, hi) of rank ``rank`` for a stream of n_bytes (word multiple)."""
    if n_bytes % 4:
        raise ValueError("stream length must be a multiple of 4 bytes")
    lo, hi = group_ranges(n_bytes // 4, world)[rank]
    return 4 * lo, 4 * hi


def allreduce_counts(counts, group=None):
    """Sum a device (or CPU, for gloo) int64[256] count tensor across ranks in place.

    Counts are exact integers below 2^63, so the int64 sum is the uint64 merge."""
    import torch.distributed as dist

    if dist.is_available() and dist.is_initialized() and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def as_uint64(counts) -> np.ndarray:
    return counts.detach().cpu().numpy().view(np.uint64).copy()
