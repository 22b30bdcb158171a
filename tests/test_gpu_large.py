"""GPU parity at BASELINE.json sizes: full 1 GiB streams against the oracle; the
64 GiB C5 stream (configs[4]) by closed forms (sequential, constant), by sampled 1 GiB
shards against the oracle bin for bin and by its 8-rank sharding; the 16 GiB C4
host-streamed run (configs[3]) bin for bin against a multithreaded oracle count of the
pinned bytes; sharded sums == whole stream; on-device generators == host generators;
and the 64 x 16 MiB batch of the C2 configuration chunk by chunk. Merge semantics
exercised at scale: core.py:142-156."""
import numpy as np
import pytest
from conftest import ws_clean

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N
from paper_1011_0235_b200 import device as D
from paper_1011_0235_b200.distributed import shard_range

pytestmark = pytest.mark.gpu
GiB = 1 << 30
CHUNK = 16 << 20


def dev_stream(cuda, spec):
    buf = cuda.empty(spec.pixels, dtype=cuda.uint8, device="cuda")
    hs.generate_device(spec, buf)
    return buf


@pytest.mark.parametrize("spec", [hs.SourceSpec("uniform", GiB, 5), hs.SourceSpec("normal", GiB, 6, mean=128.0, sigma=8.0)])
def test_full_gib_against_oracle(cuda, oracle, spec):
    buf = dev_stream(cuda, spec)
    want = oracle.histogram(buf.cpu().numpy())
    assert int(want.sum()) == GiB
    pat = hs.compute_binning_pattern(hs.Histogram256(want))
    for kind in (N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE):
        for impl in (N.HS_IMPL_LANE, N.HS_IMPL_WARP):
            got = D.histograms([hs.DeviceChunk(buf)], kind, pat, impl)[0]
            assert np.array_equal(got, want), (kind, impl)
    del buf


@pytest.mark.parametrize("gib", [1, 8])
def test_closed_form_constant_and_sequential(cuda, gib):
    n = gib * GiB
    buf = cuda.empty(n, dtype=cuda.uint8, device="cuda")
    for value in (0, 127, 255):
        buf.fill_(value)
        h = hs.naive_histogram(hs.DeviceChunk(buf), hs.WorkerGroupConfig())
        assert h.counts[value] == n and h.total() == n
        p = np.zeros(256, np.uint64)
        p[value] = 1
        a = hs.adaptive_histogram(hs.DeviceChunk(buf), hs.compute_binning_pattern(hs.Histogram256(p)), hs.WorkerGroupConfig())
        assert a == h
    hs.generate_device(hs.SourceSpec("sequential", n), buf)
    h = hs.naive_histogram(hs.DeviceChunk(buf), hs.WorkerGroupConfig())
    assert (h.counts == n // 256).all()
    del buf


def test_shards_sum_to_whole(cuda, oracle):
    spec = hs.SourceSpec("normal", GiB + 4096 + 12, 9, mean=100.0, sigma=50.0)
    buf = dev_stream(cuda, spec)
    whole = hs.naive_histogram(hs.DeviceChunk(buf), hs.WorkerGroupConfig())
    for world in (2, 4, 8):
        parts = []
        for r in range(world):
            lo, hi = shard_range(spec.pixels, r, world)
            parts.append(hs.naive_histogram(hs.DeviceChunk(buf[lo:hi]), hs.WorkerGroupConfig()))
        assert hs.merge_all(parts) == whole
    # each shard generated in place from its first pixel index equals the slice
    lo, hi = shard_range(spec.pixels, 3, 8)
    shard = cuda.empty(hi - lo, dtype=cuda.uint8, device="cuda")
    hs.generate_device(spec, shard, lo)
    assert bool((shard == buf[lo:hi]).all())
    del buf


def test_device_generator_matches_host_at_scale(cuda):
    for spec in (hs.SourceSpec("normal", 64 << 20, 1011, mean=128.0, sigma=32.0),
                 hs.SourceSpec("uniform", 256 << 20, 0xDEADBEEF)):
        host = hs.generate(spec).pixels()
        dev = dev_stream(cuda, spec)
        assert np.array_equal(dev.cpu().numpy(), host), spec.kind


def test_bench_configuration_per_chunk(cuda, oracle):
    """64 x 16 MiB chunks of a sigma-32 stream in one ADAPTIVE launch (bench.py)."""
    buf = cuda.empty(GiB, dtype=cuda.uint8, device="cuda")
    for c in range(64):
        hs.generate_device(hs.SourceSpec("normal", CHUNK, 0x10110235 ^ c, mean=128.0, sigma=32.0),
                           buf[c * CHUNK:(c + 1) * CHUNK])
    chunks = [hs.DeviceChunk(buf[c * CHUNK:(c + 1) * CHUNK]) for c in range(64)]
    host = buf.cpu().numpy()
    want = np.stack([oracle.histogram(host[c * CHUNK:(c + 1) * CHUNK]) for c in range(64)])
    pat = hs.compute_binning_pattern(hs.Histogram256(want.sum(axis=0)))
    got = hs.batch_histograms(chunks, hs.KernelKind.ADAPTIVE, pat, hs.WorkerGroupConfig())
    assert np.array_equal(np.stack([g.counts for g in got]), want)
    del buf


def test_large_launch_across_segments(cuda, oracle):
    """A 3 GiB call is cut into <= 1 GiB launches; segments of irregular sizes -- tiny,
    empty, and larger than a launch -- cross launch boundaries and accumulate across
    them. Every segment's counts equal the host's, ticketed and memset+RED alike."""
    torch = cuda
    n = 3 * GiB + 64
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("normal", n, 21, mean=128.0, sigma=40.0), buf)
    host = buf.cpu().numpy()
    cuts = [0, 700 << 20, (700 << 20) + 12, (700 << 20) + 12, (2300 << 20) + 4, n - 8, n]
    begin = np.array(cuts[:-1], np.uint64)
    end = np.array(cuts[1:], np.uint64)
    want = [oracle.histogram(host[a:b]) for a, b in zip(cuts[:-1], cuts[1:])]
    L = N.lib()
    out = torch.empty((len(want), 256), dtype=torch.int64, device="cuda")
    ws = D.default_staging().workspace()
    for use_ws in (True, False):
        out.fill_(-1)
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(begin), N.u64p(end), len(want), N.HS_KIND_NAIVE,
                                       N.HS_IMPL_LANE, None, None, 0, 0, out.data_ptr(),
                                       ws.data_ptr() if use_ws else None, ws.numel() if use_ws else 0,
                                       torch.cuda.current_stream().cuda_stream), "rounds")
        got = out.cpu().numpy().view(np.uint64)
        for s, w in enumerate(want):
            assert got[s].tolist() == w.tolist(), (use_ws, s)
    assert ws_clean(ws)  # tickets and accumulator rows are zero again


def test_split_launches_over_groups(cuda, oracle):
    """70 segments (two groups of <= 64) where a 1.25 GiB segment and a 0.5 GiB one are
    cut by launch boundaries between tiny and empty neighbours; batch_histograms
    agrees with the host per segment."""
    torch = cuda
    sizes = [4, 0, 1280 << 20, 8, 0, 512 << 20, 12] + [(k % 5) * 4096 + 4 * k for k in range(63)]
    n = sum(sizes)
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("uniform", n, 77), buf)
    host = buf.cpu().numpy()
    offs = np.cumsum([0] + sizes)
    chunks = [hs.DeviceChunk(buf[offs[i]:offs[i + 1]]) for i in range(len(sizes))]
    got = hs.batch_histograms(chunks, hs.KernelKind.NAIVE, None, hs.WorkerGroupConfig())
    for i, h in enumerate(got):
        assert h.counts.tolist() == oracle.histogram(host[offs[i]:offs[i + 1]]).tolist(), i


@pytest.mark.parametrize("seed", range(3))
def test_weighted_split_random_layouts(cuda, oracle, seed):
    """Full-grid launches with <= 148 segments take the cost-weighted CTA split (a CTA
    that crosses a segment boundary gets fewer units). Random word-multiple segment
    sizes over 1.5 GiB (some empty, one crossing the 1 GiB launch cut) at a base 0, 4
    or 8 bytes past a 16-B boundary, NAIVE and the register (HOT) form, against the
    oracle per segment; the workspace must be zero again afterwards."""
    torch = cuda
    rng = np.random.default_rng(77 + seed)
    n = 3 * GiB // 2
    off = 4 * seed
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("normal", n, seed, mean=60.0, sigma=5.0), buf)
    span = n - 16
    nseg = int(rng.integers(2, 140))
    cuts = np.sort(4 * rng.integers(0, span // 4, nseg - 1))
    cuts[: max(1, nseg // 10)] = cuts[0]  # a run of empty segments
    b0 = np.concatenate([[0], cuts]).astype(np.uint64)
    b1 = np.concatenate([cuts, [span]]).astype(np.uint64)
    host = buf.cpu().numpy()
    want = np.stack([oracle.histogram(host[off + int(a):off + int(b)]) for a, b in zip(b0, b1)])
    L = N.lib()
    ws = torch.zeros(int(L.hs_workspace_bytes(256)), dtype=torch.uint8, device="cuda")
    deg = np.zeros(256, np.uint64)
    deg[60] = 1
    hot = hs.compute_binning_pattern(hs.Histogram256(deg))
    for kind, p in ((N.HS_KIND_NAIVE, None), (N.HS_KIND_ADAPTIVE, hot)):
        out = torch.full((nseg, 256), -1, dtype=torch.int64, device="cuda")
        N.check(L.hs_histogram_batched(buf.data_ptr() + off, N.u64p(b0), N.u64p(b1), nseg, kind, N.HS_IMPL_AUTO,
                                       N.i64p(p.offset) if p else None, N.i64p(p.count) if p else None,
                                       960 if p else 0, 8 if p else 0, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                       torch.cuda.current_stream().cuda_stream), "weighted")
        assert np.array_equal(out.cpu().numpy().view(np.uint64), want.astype(np.uint64)), (seed, kind, nseg)
        assert ws_clean(ws)
    del buf


C5 = 64 * GiB
C5_SEED = 0x1011_0235 ^ 0xC5


def _merged(torch, buf, b0, b1, ws):
    L = N.lib()
    out = torch.full((len(b0), 256), -1, dtype=torch.int64, device="cuda")
    N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(np.asarray(b0, np.uint64)), N.u64p(np.asarray(b1, np.uint64)),
                                   len(b0), N.HS_KIND_NAIVE | N.HS_KIND_FLAG_MERGE, N.HS_IMPL_AUTO, None, None, 0, 0,
                                   out.data_ptr(), ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream),
            "merged")
    return out[0].cpu().numpy().view(np.uint64).copy()


def test_c5_64gib_closed_forms(cuda):
    """64 GiB in one call (64 chained 1 GiB launches): sequential bytes give exactly
    2^28 per bin, constant bytes 2^36 in one bin -- merged and per 1 GiB segment."""
    torch = cuda
    buf = torch.empty(C5, dtype=torch.uint8, device="cuda")
    ws = torch.zeros(int(N.lib().hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    b0 = np.arange(64, dtype=np.uint64) * GiB
    b1 = b0 + GiB
    try:
        hs.generate_device(hs.SourceSpec("sequential", C5), buf)
        assert (_merged(torch, buf, [0], [C5], ws) == C5 // 256).all()
        per = hs.batch_histograms([hs.DeviceChunk(buf[int(a):int(b)]) for a, b in zip(b0, b1)], hs.KernelKind.NAIVE,
                                  None, hs.WorkerGroupConfig())
        assert all((h.counts == GiB // 256).all() for h in per)
        for value in (0, 127):
            buf.fill_(value)
            got = _merged(torch, buf, b0, b1, ws)
            assert got[value] == C5 and got.sum() == C5
        assert ws_clean(ws)
    finally:
        del buf
        torch.cuda.empty_cache()


def test_c5_64gib_uniform_sampled_shards(cuda, oracle):
    """The bench's C5 stream itself (64 GiB uniform splitmix64, generated in place): the
    merged total is 64 GiB and equals the sum of the 64 per-segment rows; three sampled
    1 GiB segments equal the oracle's host count bin for bin; the 8-rank sharding
    (each shard generated from its own first pixel and counted by ShardedHistogram)
    sums to the whole."""
    torch = cuda
    from paper_1011_0235_b200.distributed import ShardedHistogram

    buf = torch.empty(C5, dtype=torch.uint8, device="cuda")
    ws = torch.zeros(int(N.lib().hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    try:
        hs.generate_device(hs.SourceSpec("uniform", C5, C5_SEED), buf)
        b0 = np.arange(64, dtype=np.uint64) * GiB
        b1 = b0 + GiB
        whole = _merged(torch, buf, [0], [C5], ws)
        assert int(whole.sum()) == C5
        rows = np.stack([h.counts for h in hs.batch_histograms(
            [hs.DeviceChunk(buf[int(a):int(b)]) for a, b in zip(b0, b1)], hs.KernelKind.NAIVE, None,
            hs.WorkerGroupConfig())])
        assert np.array_equal(rows.sum(axis=0, dtype=np.uint64), whole)
        for seg in (0, 41, 63):
            want = oracle.histogram_mt(buf[seg * GiB:(seg + 1) * GiB].cpu().numpy())
            assert np.array_equal(rows[seg], want), seg
        sh = ShardedHistogram()
        total = np.zeros(256, np.uint64)
        for r in range(8):
            lo, hi = shard_range(C5, r, 8)
            sh.count(buf[lo:hi])
            total += sh.result().counts
        assert np.array_equal(total, whole)
        del buf
        torch.cuda.empty_cache()
        lo, hi = shard_range(C5, 5, 8)  # a shard generated in place from its first pixel
        shard = torch.empty(hi - lo, dtype=torch.uint8, device="cuda")
        hs.generate_device(hs.SourceSpec("uniform", C5, C5_SEED), shard, first_pixel=lo)
        sh.count(shard)
        assert np.array_equal(sh.result().counts, rows[40:48].sum(axis=0, dtype=np.uint64))
        del shard
    finally:
        torch.cuda.empty_cache()


C4_SEGMENTS = (("uniform", {}), ("normal", {"mean": 128.0, "sigma": 32.0}), ("constant", {"value": 127}),
               ("normal", {"mean": 128.0, "sigma": 8.0}))


def test_c4_16gib_host_streamed_per_bin(cuda, oracle):
    """configs[3]: 16 GiB mixed stream (1024 x 16 MiB chunks) in pinned host memory
    through run_pipeline with the reference switch policy: the accumulator equals a
    multithreaded oracle count of the pinned bytes bin for bin, sampled per-slice
    histograms equal the oracle's, and the switch fires at the constant segment."""
    torch = cuda
    nchunks = 1024
    pinned = D.pinned_bytes(nchunks * CHUNK)
    stage = torch.empty(CHUNK, dtype=torch.uint8, device="cuda")
    for i in range(nchunks):
        kind, kw = C4_SEGMENTS[i // (nchunks // 4)]
        hs.generate_device(hs.SourceSpec(kind, CHUNK, (0x10110235 ^ 0xC4) ^ i, **kw), stage)
        torch.from_numpy(pinned[i * CHUNK:(i + 1) * CHUNK]).copy_(stage)
    words = pinned.view(np.uint32)
    chunks = [hs.PackedChunk(words[c * (CHUNK // 4):(c + 1) * (CHUNK // 4)]) for c in range(nchunks)]
    batch = 16
    cfg = hs.PipelineConfig(num_iterations=nchunks // batch, chunk_pixels=CHUNK, batch_size=batch, window_size=8)
    acc, _, rep, log = hs.run_pipeline((chunks[i * batch:(i + 1) * batch] for i in range(nchunks // batch)), cfg,
                                       hs.SwitchPolicy())
    assert np.array_equal(acc.running.counts, oracle.histogram_mt(pinned))
    for it, j in ((0, 0), (20, 7), (40, 15), (63, 3)):
        c = it * batch + j
        assert np.array_equal(rep.per_slice_histograms[it][j].counts,
                              oracle.histogram(pinned[c * CHUNK:(c + 1) * CHUNK])), (it, j)
    kinds = [k.value for k in log]
    assert kinds[:16] == ["naive"] * 16 and "adaptive" in kinds[32:49]
