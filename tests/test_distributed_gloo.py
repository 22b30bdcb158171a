"""The N>1 path on CPU: world_size-2/3 gloo processes go through the product API
(distributed.init_process_group + ShardedHistogram): each rank takes its contiguous
byte range (the group_ranges rule), counts it, and one all_reduce of the 256-count
partials joins them; the result equals the whole-stream histogram. The per-shard count
comes from the oracle through ShardedHistogram's test-only count_fn hook (no GPU); on
the B200 the same object runs one merged libhist256 call per rank and NCCL."""
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
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port), RANK=str(rank), WORLD_SIZE=str(world),
                      LOCAL_RANK=str(rank), HS_DIST_VERBOSE="0")
    from paper_1011_0235_b200.distributed import ShardedHistogram, init_process_group

    r, w, _ = init_process_group("gloo")
    assert (r, w) == (rank, world)
    try:
        import sys
        from pathlib import Path

        sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
        from oracle import oracle as O

        px = O.generate(kind, n_bytes, seed=99, mean=128.0, sigma=32.0, value=3)
        seen = []

        def count_fn(shard):  # test-only hook: the oracle instead of the device kernel
            seen.append(shard.size)
            return torch.from_numpy(O.histogram(shard).view(np.int64).copy())

        sh = ShardedHistogram(count_fn=count_fn)
        lo, hi = sh.shard(n_bytes)
        assert (lo, hi) == shard_range(n_bytes, rank, world)
        sh(px[lo:hi])
        hist = sh.result()
        assert seen == [hi - lo]
        q.put((rank, hist.counts, O.histogram(px)))
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
    res = [q.get(timeout=120) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    assert sorted(r for r, _, _ in res) == list(range(world))
    for _, got, want in res:  # every rank holds the whole stream's histogram
        assert np.array_equal(got, want)


def test_allreduce_counts_gloo_direct():
    """allreduce_counts is a no-op outside a process group."""
    c = torch.arange(256, dtype=torch.int64)
    assert allreduce_counts(c) is c and int(c.sum()) == 255 * 128
    assert np.array_equal(as_uint64(c), np.arange(256, dtype=np.uint64))


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
