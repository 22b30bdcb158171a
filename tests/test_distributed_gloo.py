"""The N>1 path on CPU: world_size-2 gloo processes shard a stream by contiguous
byte range (distributed.shard_range, the group_ranges rule) and join 256-count
partials with one all_reduce; the result equals the whole-stream histogram.
Per-shard counts come from the oracle here (no GPU); the device path swaps in
libhist256 and NCCL with the same host logic (bench.py)."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_1011_0235_b200.distributed import allreduce_counts, as_uint64, shard_range


def _free_port() -> int:
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def _worker(rank, world, port, n_bytes, kind, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from oracle import oracle as O

        px = O.generate(kind, n_bytes, seed=99, mean=128.0, sigma=32.0, value=3)
        lo, hi = shard_range(n_bytes, rank, world)
        counts = torch.from_numpy(O.histogram(px[lo:hi]).view(np.int64).copy())
        allreduce_counts(counts)
        if rank == 0:
            q.put((as_uint64(counts), O.histogram(px)))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world,n_bytes,kind", [(2, 1 << 16, "uniform"), (2, (1 << 16) + 12, "normal"), (3, 4096 + 8, "constant")])
def test_sharded_allreduce_equals_whole(world, n_bytes, kind):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, n_bytes, kind, q)) for r in range(world)]
    for p in procs:
        p.start()
    got, want = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert np.array_equal(got, want)


def test_shard_ranges_cover_stream():
    for n in (0, 4, 4096, (1 << 20) + 12):
        for world in (1, 2, 3, 8):
            parts = [shard_range(n, r, world) for r in range(world)]
            assert parts[0][0] == 0 and parts[-1][1] == n
            assert all(a[1] == b[0] for a, b in zip(parts, parts[1:]))
            assert all(lo % 4 == 0 and hi % 4 == 0 for lo, hi in parts)


def _max_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        import bench

        got = bench.max_over_ranks(1.5 + rank, world)  # bench's timing rule: max over ranks
        if rank == 0:
            q.put(got)
    finally:
        dist.destroy_process_group()


def test_bench_time_is_max_over_ranks():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_max_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    got = q.get(timeout=120)
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert got == 2.5
