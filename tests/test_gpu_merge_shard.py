"""GPU parity of the round-2 launch options and the multi-GPU product path:

- HS_KIND_FLAG_MERGE: all segments of a call fold into one uint64[256] in the kernel
  epilogue (merge_all of the per-slice histograms, core.py:152-156) -- random segment
  layouts, empty segments, calls over 1 GiB (chained launches) and > 256 segments,
  with and without a workspace, every impl;
- HS_KIND_FLAG_CHAINED and the default first-launch wait: a producer kernel writes the
  input right before the call on the same stream;
- distributed.ShardedHistogram on one GPU (world 1, no process group and an NCCL group
  of one): the rank's merged partial and the allreduce;
- the ADVICE fixes: strided device tensors, the device check, one workspace per stream,
  patterns with more than 65535 slots on the lane kernels, generate_device checks."""
import os
import socket

import numpy as np
import pytest
from conftest import ws_clean

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N
from paper_1011_0235_b200 import device as D
from paper_1011_0235_b200.distributed import ShardedHistogram, shard_range

pytestmark = pytest.mark.gpu


def _call(L, torch, buf, b0, b1, kind, impl=N.HS_IMPL_AUTO, ws=None, pat=None, out=None):
    out = out if out is not None else torch.full((max(len(b0), 1), 256), -1, dtype=torch.int64, device="cuda")
    off = N.i64p(pat.offset) if pat is not None else None
    cnt = N.i64p(pat.count) if pat is not None else None
    S, cap = (int(pat.total_slots), int(pat.cap)) if pat is not None else (0, 0)
    N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(np.asarray(b0, np.uint64)), N.u64p(np.asarray(b1, np.uint64)),
                                   len(b0), kind, impl, off, cnt, S, cap, out.data_ptr(),
                                   ws.data_ptr() if ws is not None else None, ws.numel() if ws is not None else 0,
                                   torch.cuda.current_stream().cuda_stream), "merge")
    return out


@pytest.mark.parametrize("seed", range(3))
def test_merge_random_layouts(cuda, oracle, seed):
    torch = cuda
    rng = np.random.default_rng(77 + seed)
    n = 40 << 20
    host = rng.integers(0, 256, n, dtype=np.uint8)
    host[: n // 4] = 17
    buf = torch.from_numpy(host).cuda()
    L = N.lib()
    pat = hs.compute_binning_pattern(hs.Histogram256(np.bincount(host[:1 << 20], minlength=256).astype(np.uint64)))
    for trial in range(10):
        nseg = int(rng.choice([1, 3, 64, 255, 256, 257, 300]))
        sizes = rng.choice([0, 4, 4096, 1 << 16, 1 << 20], size=nseg) + 4 * rng.integers(0, 64, nseg)
        sizes[rng.random(nseg) < 0.15] = 0
        starts = 4 * rng.integers(0, (n - int(sizes.max()) - 4) // 4, nseg)
        b0, b1 = starts.astype(np.uint64), (starts + sizes).astype(np.uint64)
        want = np.zeros(256, np.uint64)
        for a, b in zip(b0, b1):
            want += oracle.histogram(host[a:b])
        impl = int(rng.choice([N.HS_IMPL_AUTO, N.HS_IMPL_LANE, N.HS_IMPL_WARP, N.HS_IMPL_SUBBIN]))
        kind = int(rng.choice([N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE]))
        use_ws = bool(rng.integers(0, 2))
        ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda") if use_ws else None
        out = _call(L, torch, buf, b0, b1, kind | N.HS_KIND_FLAG_MERGE, impl, ws, pat)
        got = out[0].cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), (seed, trial, nseg, impl, kind, use_ws)
        if nseg > 1:  # only row 0 is written
            assert (out[1:] == -1).all().item()
        if use_ws:
            assert ws_clean(ws), "workspace left non-zero"


def test_merge_over_one_gib_and_all_empty(cuda, oracle):
    """A merged call over 2.25 GiB in 9 segments runs as chained <= 1 GiB launches; only
    the last finalizes. An all-empty merged call writes zeros."""
    torch = cuda
    L = N.lib()
    seg = (1 << 28)  # 256 MiB
    n = 9 * seg
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("sequential", n, 0), buf)  # closed form: n / 256 per bin
    b0 = np.arange(9, dtype=np.uint64) * seg
    b1 = b0 + seg
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    for chained in (0, N.HS_KIND_FLAG_CHAINED):
        out = _call(L, torch, buf, b0, b1, N.HS_KIND_NAIVE | N.HS_KIND_FLAG_MERGE | chained, ws=ws)
        assert (out[0] == n // 256).all().item()
        assert ws_clean(ws)
    out = _call(L, torch, buf, b0, b0, N.HS_KIND_NAIVE | N.HS_KIND_FLAG_MERGE, ws=ws)
    assert (out[0] == 0).all().item()


def test_first_launch_waits_for_producer(cuda):
    """A producer kernel writes the input immediately before the call on the same
    stream (torch fill_ and a device generator, both plain launches), many times in a
    row, alternating values: the call's first launch must see the new bytes."""
    torch = cuda
    L = N.lib()
    n = 256 << 20
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    b0, b1 = np.zeros(1, np.uint64), np.full(1, n, np.uint64)
    outs = []
    for k in range(12):
        buf.fill_(k)
        outs.append(_call(L, torch, buf, b0, b1, N.HS_KIND_NAIVE, ws=ws))
    for k, o in enumerate(outs):
        row = o[0].cpu()
        assert row[k].item() == n and row.sum().item() == n, k


def test_sharded_histogram_single_gpu(cuda, oracle):
    """The product multi-GPU object at world 1 without a process group: the merged
    partial of a shard given as segments equals the oracle."""
    torch = cuda
    n = (96 << 20) + 12
    host = oracle.generate("normal", n, 9, mean=128.0, sigma=32.0)
    dev = torch.from_numpy(host.copy()).cuda()
    sh = ShardedHistogram()
    assert (sh.rank, sh.world) == (0, 1) and sh.shard(n) == (0, n)
    got = sh(dev)
    assert np.array_equal(got.cpu().numpy().view(np.uint64), oracle.histogram(host))
    segs = [(0, 4096), (4096, 4096), (8192, 40 << 20), (40 << 20, n)]
    sh.count(dev, segments=segs)
    assert np.array_equal(sh.result().counts, oracle.histogram(host[:4096]) + oracle.histogram(host[8192:]))
    with pytest.raises(TypeError):
        sh(dev.to(torch.int32))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_histogram_nccl_world1(cuda, oracle):
    """The NCCL path (init_process_group + one allreduce) in a group of one: the code
    the bench runs under torchrun."""
    torch = cuda
    import torch.distributed as dist

    from paper_1011_0235_b200.distributed import init_process_group

    env = dict(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(_free_port()), RANK="0", WORLD_SIZE="1", LOCAL_RANK="0")
    old = {k: os.environ.get(k) for k in env}
    os.environ.update(env)
    try:
        rank, world, local = init_process_group("nccl")
        assert (rank, world) == (0, 1) and dist.get_backend() == "nccl"
        n = 64 << 20
        buf = torch.empty(n, dtype=torch.uint8, device="cuda")
        hs.generate_device(hs.SourceSpec("uniform", n, 3), buf)
        lo, hi = shard_range(n, rank, world)
        sh = ShardedHistogram()
        sh(buf[lo:hi])
        want = oracle.histogram(buf.cpu().numpy())
        assert np.array_equal(sh.result().counts, want)
    finally:
        if dist.is_initialized():
            dist.destroy_process_group()
        for k, v in old.items():
            if v is None:
                os.environ.pop(k, None)
            else:
                os.environ[k] = v


def test_strided_and_foreign_device_chunks(cuda, oracle):
    """ADVICE: a strided CUDA view is packed into stream order, not read as contiguous
    bytes from its data_ptr."""
    torch = cuda
    host = oracle.generate("uniform", 1 << 20, 21)
    t = torch.from_numpy(host.copy()).cuda()
    strided = t[::2]
    assert not strided.is_contiguous()
    c = hs.DeviceChunk(strided)
    want = oracle.histogram(host[::2].copy())
    assert np.array_equal(hs.naive_histogram(c, hs.WorkerGroupConfig()).counts, want)
    img = t.view(1024, 1024)[:, :512]
    got = hs.batch_histograms([hs.DeviceChunk(img), hs.DeviceChunk(t[:4096])], hs.KernelKind.NAIVE, None,
                              hs.WorkerGroupConfig())
    assert np.array_equal(got[0].counts, oracle.histogram(host.reshape(1024, 1024)[:, :512].copy().reshape(-1)))
    assert np.array_equal(got[1].counts, oracle.histogram(host[:4096]))


def test_workspace_per_stream(cuda, oracle):
    """ADVICE: launches on two unsynchronized streams never share accumulator rows."""
    torch = cuda
    st = D.default_staging()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    assert st.workspace(s1).data_ptr() != st.workspace(s2).data_ptr()
    assert st.workspace(s1).data_ptr() == st.workspace(s1.cuda_stream).data_ptr()
    n = 64 << 20
    hosts = [oracle.generate("normal", n, 50 + j, mean=60.0 + 80 * j, sigma=9.0) for j in range(2)]
    bufs = [torch.from_numpy(h.copy()).cuda() for h in hosts]
    torch.cuda.synchronize()
    outs = [[], []]
    for _ in range(6):
        for j, s in enumerate((s1, s2)):
            outs[j].append(D.histogram_tensor(bufs[j], stream=s))
    torch.cuda.synchronize()
    for j in range(2):
        want = oracle.histogram(hosts[j])
        for o in outs[j]:
            assert np.array_equal(o.cpu().numpy().view(np.uint64), want)
        assert ws_clean(st.workspace((s1, s2)[j]))


def test_lane_accepts_large_slot_totals(cuda, oracle):
    """ADVICE: a legal pattern with more than 65535 slots (cap 300) runs on the lane
    kernels, which use only its hot bin; the sub-bin kernel still rejects it."""
    torch = cuda
    host = oracle.generate("mixture", 1 << 20, 4, value=9, degeneracy=0.8)
    prior = hs.Histogram256(oracle.histogram(host))
    pat = hs.compute_binning_pattern(prior, 70000, 300)
    assert pat.total_slots == 70000
    chunk = hs.PackedChunk(oracle.pack(host))
    assert np.array_equal(hs.adaptive_histogram(chunk, pat, hs.WorkerGroupConfig()).counts, oracle.histogram(host))
    buf = torch.from_numpy(host.copy()).cuda()
    with pytest.raises(N.NativeCallError):
        _call(N.lib(), torch, buf, [0], [host.size], N.HS_KIND_ADAPTIVE, N.HS_IMPL_SUBBIN, pat=pat)


def test_generate_device_rejects_bad_tensors(cuda):
    torch = cuda
    spec = hs.SourceSpec("uniform", 1024, 1)
    with pytest.raises(TypeError):
        hs.generate_device(spec, torch.empty(256, dtype=torch.int32, device="cuda"))
    with pytest.raises(TypeError):
        hs.generate_device(spec, torch.empty(2048, dtype=torch.uint8, device="cuda")[::2])
    with pytest.raises(TypeError):
        hs.generate_device(spec, torch.empty(1024, dtype=torch.uint8))


def test_capture_workspace_never_leaks_into_eager_use(cuda, oracle):
    """A launch captured into a CUDA graph on a stream that had no workspace yet gets a
    graph-private one (zeroed by the graph); eager launches on that stream afterwards,
    and after the graph is gone, use a normally zeroed workspace (the CLI's graph-timed
    sweep followed by eager calls)."""
    torch = cuda
    host = oracle.generate("uniform", 8 << 20, 31)
    buf = torch.from_numpy(host.copy()).cuda()
    want = oracle.histogram(host)
    for rep in range(3):
        side = torch.cuda.Stream()
        out = torch.empty((1, 256), dtype=torch.int64, device="cuda")
        g = torch.cuda.CUDAGraph()
        with torch.cuda.graph(g, stream=side):
            for _ in range(4):
                D.histogram_tensor(buf, out=out)
        g.replay()
        torch.cuda.synchronize()
        assert np.array_equal(out[0].cpu().numpy().view(np.uint64), want)
        del g
        with torch.cuda.stream(side):
            got = D.histogram_tensor(buf)
        torch.cuda.synchronize()
        assert np.array_equal(got.cpu().numpy().view(np.uint64), want), rep
        assert np.array_equal(hs.naive_histogram(hs.PackedChunk(oracle.pack(host)), hs.WorkerGroupConfig()).counts,
                              want)
