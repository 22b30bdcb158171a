"""GPU parity at BASELINE.json sizes through size-independent properties: full
1 GiB streams against the oracle, closed-form counts for constant and sequential
streams up to 8 GiB, sharded sums == whole stream, on-device generators == host
generators, and the 64 x 16 MiB batch of the bench configuration chunk by chunk."""
import numpy as np
import pytest

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
    assert not ws.any().item()  # tickets and accumulator rows are zero again


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
def test_weighted_split_random_layouts(cuda, seed):
    """Full-grid launches with <= 148 segments take the cost-weighted CTA split (a CTA
    that crosses a segment boundary gets fewer units). Random word-multiple segment
    sizes over 1.5 GiB (some empty, one crossing the 1 GiB launch cut) at a base 0, 4
    or 8 bytes past a 16-B boundary, NAIVE and the register (HOT) form, against
    torch.bincount per segment; the workspace must be zero again afterwards."""
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
    want = np.stack([torch.bincount(buf[off + int(a):off + int(b)], minlength=256).cpu().numpy()
                     for a, b in zip(b0, b1)])
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
        assert not ws.any().item()
    del buf
