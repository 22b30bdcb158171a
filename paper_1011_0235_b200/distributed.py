"""Multi-GPU: contiguous byte-range shards, one merged count per rank, one allreduce.

The histogram merge is a commutative monoid (core.py:142-149), and the reference
already partitions contiguously and merges partials (group_ranges kernels.py:311-316,
merge_all core.py:152-156). Across GPUs the same rule applies at word granularity:
rank r of P owns words [r*floor(W/P), (r+1)*floor(W/P)), the last rank the remainder.

Per rank, ONE library call counts the shard (any number of segments, run as chained
<= 1 GiB launches) with HS_KIND_FLAG_MERGE: the segments fold into a single uint64[256]
inside the kernel's ticketed epilogue, so there is no per-segment output and no eager
reduction on the way to the collective. One ``all_reduce(SUM)`` of those 2 KiB over
NCCL (NVLink/NVSwitch) joins the ranks. North star: "the 256-count partial histograms
are combined with a single NCCL allreduce over NVLink". The collective is
latency-bound (tens of microseconds) next to a multi-millisecond scan per rank, so the
path shards with no data exchange and a single tiny reduction at the end.

    sh = ShardedHistogram()                 # after torch.distributed.init_process_group
    lo, hi = sh.shard(n_bytes)              # this rank's byte range of the stream
    ... place bytes [lo, hi) of the stream in a CUDA tensor `mine` ...
    total = sh(mine)                        # device int64[256]: the whole stream's counts
    hist = sh.result()                      # Histogram256 (host)
"""
from __future__ import annotations

import logging
import os
import time
from typing import Callable, Sequence

import numpy as np

from .core import BINS, Histogram256
from .kernels import group_ranges

log = logging.getLogger(__name__)


def shard_range(n_bytes: int, rank: int, world: int) -> tuple[int, int]:
    """Byte range [lo, hi) of rank ``rank`` for a stream of n_bytes (word multiple)."""
    if n_bytes % 4:
        raise ValueError("stream length must be a multiple of 4 bytes")
    if not 0 <= rank < world:
        raise ValueError(f"rank {rank} outside world of {world}")
    lo, hi = group_ranges(n_bytes // 4, world)[rank]
    return 4 * lo, 4 * hi


def _dist():
    import torch.distributed as dist

    return dist if dist.is_available() and dist.is_initialized() else None


def allreduce_counts(counts, group=None):
    """Sum an int64[256] count tensor across ranks in place (NCCL on CUDA tensors, gloo
    on CPU ones). Counts are exact integers below 2^63, so the int64 sum is the uint64
    merge of core.py:142-149."""
    dist = _dist()
    if dist is not None and dist.get_world_size(group) > 1:
        dist.all_reduce(counts, op=dist.ReduceOp.SUM, group=group)
    return counts


def as_uint64(counts) -> np.ndarray:
    return counts.detach().cpu().numpy().view(np.uint64).copy()


class _StdoutToStderr:
    """fd-level redirect of stdout into stderr: NCCL/c10d print their banner ("NCCL
    version ...") from C at communicator creation, and the bench's stdout must carry
    exactly one JSON line."""

    def __enter__(self):
        import sys

        sys.stdout.flush()
        self._saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        import sys

        sys.stdout.flush()
        os.dup2(self._saved, 1)
        os.close(self._saved)


def init_process_group(backend: str | None = None, device=None):
    """One process per GPU (torchrun environment): initialise torch.distributed, bind the
    rank's device, create the communicator eagerly with a 2 KiB warm-up allreduce, and
    log rank, world size, backend and communicator set-up time (so a run's log shows how
    many ranks took part). Returns (rank, world, local_rank)."""
    import torch
    import torch.distributed as dist

    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if backend is None:
        backend = "nccl" if torch.cuda.is_available() else "gloo"
    t0 = time.perf_counter()
    with _StdoutToStderr():
        if not dist.is_initialized():
            if backend == "nccl":
                torch.cuda.set_device(local if device is None else device)
                dist.init_process_group("nccl", device_id=torch.device("cuda", local if device is None else device))
            else:
                dist.init_process_group(backend)
        dev = torch.device("cuda", torch.cuda.current_device()) if backend == "nccl" else torch.device("cpu")
        warm = torch.zeros(BINS, dtype=torch.int64, device=dev)
        dist.all_reduce(warm)
        if dev.type == "cuda":
            torch.cuda.synchronize(dev)
    msg = (f"[hs.distributed] rank {dist.get_rank()}/{dist.get_world_size()} backend={dist.get_backend()} "
           f"device={dev} communicator ready in {(time.perf_counter() - t0) * 1e3:.1f} ms")
    log.info(msg)
    if os.environ.get("HS_DIST_VERBOSE", "1") != "0":
        print(msg, flush=True, file=__import__("sys").stderr)
    return dist.get_rank(), dist.get_world_size(), local


class ShardedHistogram:
    """The multi-GPU product path: each rank counts its contiguous shard of a stream in
    one merged library call, and one allreduce of 256 counts joins the ranks.

    ``count_fn`` is a test-only hook (CPU gloo tests): a callable (shard) -> int64[256]
    tensor that replaces the device count, so sharding and the collective can be
    exercised without a GPU. The product path (count_fn None) always runs libhist256
    and raises without CUDA."""

    def __init__(self, group=None, device=None, count_fn: Callable | None = None):
        self.group = group
        self._count_fn = count_fn
        dist = _dist()
        self.rank = dist.get_rank(group) if dist is not None else 0
        self.world = dist.get_world_size(group) if dist is not None else 1
        self._counts = None
        self._dev = None
        if count_fn is None:
            from . import device as D

            t = D.require_cuda()
            self._dev = t.device("cuda", t.cuda.current_device() if device is None else t.device(device).index)
            self._staging = D.Staging(self._dev)
            self._counts = t.zeros(BINS, dtype=t.int64, device=self._dev)

    def shard(self, n_bytes: int) -> tuple[int, int]:
        """This rank's byte range [lo, hi) of an n_bytes stream (group_ranges rule)."""
        return shard_range(n_bytes, self.rank, self.world)

    def count(self, shard, kind: int | None = None, pattern=None, stream=None, segments: Sequence[tuple[int, int]] |
              None = None, chained: bool = False):
        """This rank's partial: one library call over ``shard`` (a uint8 CUDA tensor)
        merged into the device int64[256] in the kernel epilogue. ``segments`` optionally
        lists word-aligned byte ranges of the shard (default: the whole shard).
        ``chained``: the stream's previous kernel is a libhist256 launch over input that
        was already complete (HS_KIND_FLAG_CHAINED). Asynchronous."""
        if self._count_fn is not None:
            self._counts = self._count_fn(shard)
            return self._counts
        from . import _native as N
        from . import device as D

        t = D.torch()
        if not (isinstance(shard, t.Tensor) and shard.is_cuda and shard.dtype == t.uint8 and shard.is_contiguous()):
            raise TypeError("shard must be a contiguous uint8 CUDA tensor")
        if shard.device != self._dev:
            raise ValueError(f"shard on {shard.device}, ShardedHistogram on {self._dev}")
        n = shard.numel()
        if n % 4 or shard.data_ptr() % 4:
            raise ValueError("shard must be word aligned (length and start multiples of 4)")
        stream = stream or t.cuda.current_stream(self._dev)
        if segments is None:
            begin = np.zeros(1, np.uint64)
            end = np.full(1, n, np.uint64)
        else:
            begin = np.array([a for a, _ in segments], dtype=np.uint64)
            end = np.array([b for _, b in segments], dtype=np.uint64)
            if begin.size and (int(end.max()) > n):
                raise ValueError("segment outside the shard")
        if kind is None:
            kind = N.HS_KIND_NAIVE
        kind = D._with_hints(int(kind), pattern) | N.HS_KIND_FLAG_MERGE | (N.HS_KIND_FLAG_CHAINED if chained else 0)
        off_p, cnt_p, S, cap, keep = D._pattern_args(pattern)
        ws = self._staging.workspace(stream)
        N.check(N.lib().hs_histogram_batched(shard.data_ptr() if n else None, N.u64p(begin), N.u64p(end),
                                             int(begin.size), kind, N.HS_IMPL_AUTO, off_p, cnt_p, S, cap,
                                             self._counts.data_ptr(), ws.data_ptr(), ws.numel(), stream.cuda_stream),
                "hs_histogram_batched(merge)")
        return self._counts

    def allreduce(self, stream=None):
        """One all_reduce(SUM) of the rank's 256 counts (NCCL over NVLink on GPUs).
        Issued on ``stream`` (default: the current stream)."""
        if self._count_fn is not None or stream is None:
            return allreduce_counts(self._counts, self.group)
        import torch

        with torch.cuda.stream(stream):
            return allreduce_counts(self._counts, self.group)

    def __call__(self, shard, kind: int | None = None, pattern=None, stream=None, segments=None, chained=False):
        """count() then allreduce(): the device int64[256] of the whole stream."""
        self.count(shard, kind, pattern, stream, segments, chained)
        return self.allreduce(stream)

    def result(self) -> Histogram256:
        """The last call's counts as a host Histogram256 (synchronises)."""
        return Histogram256(as_uint64(self._counts))


def sharded_histogram(shard, kind: int | None = None, pattern=None, group=None) -> Histogram256:
    """One-shot form: this rank's shard counted, all ranks' counts summed; every rank
    gets the whole stream's Histogram256."""
    sh = ShardedHistogram(group)
    sh(shard, kind, pattern)
    return sh.result()
