"""GPU parity of the histogram kernels through the drop-in API (and the C ABI under
it) against the oracle and reference-generated vectors. Bit-exact integer results.

Mirrors the reference's kernel tests (test_kernels.py) and acceptance c01
(test_acceptance.py:56-91), plus every device strategy (HS_IMPL_*), unaligned and
ragged device segments, and the slot-level compat outputs."""
import zlib

import numpy as np
import pytest
from conftest import ws_clean

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N
from paper_1011_0235_b200 import device as D

pytestmark = pytest.mark.gpu

IMPLS = [N.HS_IMPL_AUTO, N.HS_IMPL_LANE, N.HS_IMPL_WARP, N.HS_IMPL_SUBBIN]


def chunk_of(oracle, kind, pixels, seed=0, **kw):
    return hs.PackedChunk(oracle.pack(oracle.generate(kind, pixels, seed, **kw)))


def deg_pattern(value=127, slots=960, cap=8):
    c = np.zeros(256, np.uint64)
    c[value] = 1_000_000
    return hs.compute_binning_pattern(hs.Histogram256(c), slots, cap)


def test_hand_count_and_empty(cuda):
    cfg = hs.WorkerGroupConfig(8, 3)
    h = hs.naive_histogram(hs.pack_pixels([1, 1, 2, 0]), cfg)
    assert h.counts[0] == 1 and h.counts[1] == 2 and h.counts[2] == 1 and h.total() == 4
    assert hs.naive_histogram(hs.pack_pixels([]), cfg).total() == 0
    assert hs.adaptive_histogram(hs.pack_pixels([]), hs.uniform_pattern(960), cfg).total() == 0


@pytest.mark.parametrize("seed", range(40))
def test_randomized_triples(cuda, oracle, seed):
    # test_kernels.py:97-115
    rng = np.random.default_rng(900 + seed)
    pixels = int(rng.integers(1, 1 << 12)) * 4
    kind = str(rng.choice(["uniform", "mixture", "constant", "sequential", "normal"]))
    px = oracle.generate(kind, pixels, int(rng.integers(0, 2**32)), value=int(rng.integers(0, 256)),
                         degeneracy=float(rng.uniform(0, 1)), mean=float(rng.uniform(0, 255)),
                         sigma=float(rng.uniform(1, 80)))
    chunk = hs.PackedChunk(oracle.pack(px))
    cfg = hs.WorkerGroupConfig(int(rng.integers(1, 9)), int(rng.integers(1, 5)))
    cap = int(rng.integers(1, 9))
    slots = int(rng.integers(256, 256 * cap + 1))
    pattern = hs.compute_binning_pattern(hs.Histogram256(rng.integers(0, 1 << 16, 256).astype(np.uint64)), slots, cap)
    want = oracle.histogram(px)
    assert np.array_equal(hs.naive_histogram(chunk, cfg).counts, want)
    assert np.array_equal(hs.adaptive_histogram(chunk, pattern, cfg).counts, want)
    for impl in IMPLS:
        kindid = N.HS_KIND_ADAPTIVE if impl != N.HS_IMPL_WARP else N.HS_KIND_NAIVE
        assert np.array_equal(D.histograms([chunk], kindid, pattern, impl)[0], want), impl


@pytest.mark.parametrize("kind", ["uniform", "normal", "constant", "sequential", "mixture"])
@pytest.mark.parametrize("impl", IMPLS)
def test_sizes_and_impls(cuda, oracle, kind, impl):
    rng = np.random.default_rng(zlib.crc32(f"{kind}/{impl}".encode()))
    for pixels in (4, 60, 4096, (1 << 20) + 20, (9 << 20) + 4):  # below/above the AUTO switch at 8 MiB
        px = oracle.generate(kind, pixels, int(rng.integers(0, 2**40)), value=200, mean=128.0, sigma=8.0,
                             degeneracy=0.7)
        pat = hs.compute_binning_pattern(hs.Histogram256(oracle.histogram(px)))
        for k in (N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE):
            got = D.histograms([hs.PackedChunk(oracle.pack(px))], k, pat, impl)[0]
            assert np.array_equal(got, oracle.histogram(px)), (kind, impl, pixels, k)


def test_device_chunks_unaligned_and_ragged(cuda, oracle):
    torch = cuda
    px = oracle.generate("normal", (3 << 20) + 64, 5, mean=100.0, sigma=40.0)
    dev = torch.from_numpy(px).cuda()
    rng = np.random.default_rng(3)
    for _ in range(20):
        a = int(rng.integers(0, px.size // 4)) * 4
        b = int(rng.integers(a // 4, px.size // 4 + 1)) * 4
        for impl in IMPLS:
            pat = hs.uniform_pattern(960)
            got = D.histograms([hs.DeviceChunk(dev[a:b])], N.HS_KIND_ADAPTIVE, pat, impl)[0]
            assert np.array_equal(got, oracle.histogram(px[a:b])), (a, b, impl)


def test_batched_segments_mixed_host_device(cuda, oracle):
    torch = cuda
    rng = np.random.default_rng(7)
    base = oracle.generate("mixture", 1 << 20, 11, value=77, degeneracy=0.4)
    dev = torch.from_numpy(base).cuda()
    cuts = sorted(int(x) * 4 for x in rng.integers(0, base.size // 4 + 1, 140))  # > kMaxSeg -> several launches
    bounds = [0, *cuts, base.size]
    slices = []
    for i, (a, b) in enumerate(zip(bounds, bounds[1:])):
        slices.append(hs.DeviceChunk(dev[a:b]) if i % 3 == 0 else hs.PackedChunk(oracle.pack(base[a:b])))
    for kind, pattern in ((hs.KernelKind.NAIVE, None), (hs.KernelKind.ADAPTIVE, hs.uniform_pattern(960))):
        got = hs.batch_histograms(slices, kind, pattern, hs.WorkerGroupConfig(4, 2))
        assert [g.counts.tolist() for g in got] == [oracle.histogram(base[a:b]).tolist() for a, b in zip(bounds, bounds[1:])]
        assert hs.merge_all(got).counts.tolist() == oracle.histogram(base).tolist()


def test_batch_matches_reference_vectors(cuda, golden):
    for i, m in enumerate(golden.meta["batches"]):
        px = golden[f"batch_{i}_pixels"]
        words = px.view(np.uint32)
        b = m["bounds"]
        slices = [hs.PackedChunk(words[x:y]) for x, y in zip(b, b[1:])]
        got = hs.batch_histograms(slices, hs.KernelKind(m["kind"]), hs.uniform_pattern(960), hs.WorkerGroupConfig(4, 2))
        assert np.array_equal(np.stack([g.counts for g in got]), golden[f"batch_{i}_hists"])


def test_batch_errors(cuda):
    chunk = hs.generate(hs.SourceSpec("uniform", 64, 0))
    cfg = hs.WorkerGroupConfig(8, 2)
    with pytest.raises(ValueError):
        hs.batch_histograms([], hs.KernelKind.NAIVE, None, cfg)
    with pytest.raises(ValueError):
        hs.batch_histograms([chunk], hs.KernelKind.ADAPTIVE, None, cfg)
    with pytest.raises(ValueError):
        hs.batch_histograms([chunk], hs.KernelKind.COPY_ONLY, None, cfg)


def test_constant_maximal_contention(cuda, oracle):
    # test_kernels.py:75-81 at GPU scale: every lane of every warp on one bin
    for value in (127, 0, 255):
        chunk = hs.PackedChunk(oracle.pack(np.full(64 << 20, value, np.uint8)))
        cfg = hs.WorkerGroupConfig(32, 2)
        h = hs.naive_histogram(chunk, cfg)
        assert h.counts[value] == 64 << 20 and h.total() == 64 << 20
        assert hs.adaptive_histogram(chunk, deg_pattern(value), cfg) == h
        # hot bin differing from the data's value exercises the non-hot path
        assert hs.adaptive_histogram(chunk, deg_pattern((value + 1) % 256), cfg) == h


def test_slots_match_reference(cuda, golden, oracle):
    for i, m in enumerate(golden.meta["slots"]):
        px = golden[f"slots_{i}_pixels"]
        chunk = hs.PackedChunk(px.view(np.uint32))
        pattern = hs.BinningPattern(golden[f"slots_{i}_offset"], golden[f"slots_{i}_count"], m["total_slots"], m["cap"])
        cfg = hs.WorkerGroupConfig(m["group_size"], m["group_count"])
        hist, slots = hs.adaptive_histogram(chunk, pattern, cfg, return_slots=True)
        assert np.array_equal(np.stack(slots), golden[f"slots_{i}_slots"])
        assert np.array_equal(hist.counts, golden[f"slots_{i}_hist"])


def test_lane_touches_match_reference(cuda, golden):
    m = golden.meta["touch"]
    chunk = hs.PackedChunk(golden["touch_pixels"].view(np.uint32))
    c = golden["touch_count"]
    pattern = hs.BinningPattern(golden["touch_offset"], c, int(c.sum()), 8)
    result, touches = hs.adaptive_lane_touches(chunk, pattern, hs.WorkerGroupConfig(m["group_size"], m["group_count"]))
    assert np.array_equal(np.stack(touches), golden["touch_out"])
    assert result == hs.reference_histogram(chunk)


def test_eight_subbin_spread_and_remainder(cuda):
    # test_kernels.py:140-165
    chunk = hs.generate(hs.SourceSpec("constant", 1 << 16, 0, value=127))
    pattern = deg_pattern(127)
    result, gs = hs.adaptive_histogram(chunk, pattern, hs.WorkerGroupConfig(32, 2), return_slots=True)
    comb = np.sum(gs, axis=0)
    span = slice(int(pattern.offset[127]), int(pattern.offset[127]) + 8)
    assert (comb[span] == (1 << 16) // 8).all() and comb.sum() == 1 << 16
    pixels = (1 << 16) + 12
    chunk = hs.generate(hs.SourceSpec("constant", pixels, 0, value=127))
    _, gs = hs.adaptive_histogram(chunk, pattern, hs.WorkerGroupConfig(32, 2), return_slots=True)
    hot = np.sum(gs, axis=0)
    hot = hot[hot > 0]
    assert len(hot) == 8 and (np.abs(hot.astype(np.int64) - pixels / 8) <= 4 * 32 * 2).all()


def test_narrow_counters(cuda, golden):
    chunk = hs.PackedChunk(golden["narrow_pixels"].view(np.uint32))
    got, slots = hs.adaptive_histogram(chunk, hs.uniform_pattern(960), hs.WorkerGroupConfig(8, 2),
                                       narrow_counters=True, return_slots=True)
    assert np.array_equal(np.stack(slots), golden["narrow_slots"])
    assert got == hs.reference_histogram(chunk)
    big = hs.generate(hs.SourceSpec("constant", 1 << 20, 0, value=127))
    with pytest.raises(hs.SubCounterOverflow):
        hs.adaptive_histogram(big, deg_pattern(127), hs.WorkerGroupConfig(32, 1), narrow_counters=True)


def test_slot_simulation_random(cuda, oracle):
    # test_kernels.py:167-182 with the numpy simulation as oracle
    rng = np.random.default_rng(31)
    for _ in range(8):
        px = oracle.generate("mixture", int(rng.integers(1, 2000)) * 4, int(rng.integers(0, 1 << 32)),
                             value=int(rng.integers(0, 256)), degeneracy=float(rng.uniform(0, 1)))
        words = oracle.pack(px)
        cfg = hs.WorkerGroupConfig(int(rng.integers(1, 12)), int(rng.integers(1, 4)))
        pattern = hs.compute_binning_pattern(hs.Histogram256(rng.integers(0, 1000, 256).astype(np.uint64)))
        _, slots = hs.adaptive_histogram(hs.PackedChunk(words), pattern, cfg, return_slots=True)
        want = oracle.simulate_slots(words, pattern.offset, pattern.count, 960, cfg.group_size, cfg.group_count)
        for g, w in zip(slots, want):
            assert np.array_equal(g, w)


def test_dispatch_and_pattern_errors(cuda):
    chunk = hs.generate(hs.SourceSpec("uniform", 256, seed=1))
    cfg = hs.WorkerGroupConfig(4, 1)
    want = hs.reference_histogram(chunk)
    assert hs.compute_histogram(chunk, hs.KernelKind.NAIVE, None, cfg) == want
    assert hs.compute_histogram(chunk, hs.KernelKind.ADAPTIVE, hs.uniform_pattern(960), cfg) == want
    with pytest.raises(ValueError):
        hs.compute_histogram(chunk, hs.KernelKind.ADAPTIVE, None, cfg)
    with pytest.raises(ValueError):
        hs.compute_histogram(chunk, hs.KernelKind.COPY_ONLY, None, cfg)
    base = hs.uniform_pattern(960)
    counts = base.count.copy()
    counts[0] = 0
    with pytest.raises(hs.InvalidPattern):
        hs.adaptive_histogram(chunk, hs.BinningPattern(base.offset, counts, 960, 8), cfg)


def test_reduce_subbins(cuda):
    p = hs.uniform_pattern(960)
    slots = np.zeros(960, np.uint64)
    slots[int(p.offset[5]):int(p.offset[5]) + 3] = [2, 3, 4]
    assert hs.reduce_subbins(slots, p).counts[5] == 9
    with pytest.raises(ValueError):
        hs.reduce_subbins(np.zeros(959, np.uint64), p)


def test_ablation_stages(cuda, golden, oracle):
    """Genealogy stages on the device give the reference's own checksums (reference-
    generated run_ablation outputs, tests/golden) and, at 4 Mi pixels, the oracle's."""
    for i, case in enumerate(golden.meta["ablation"]):
        px = golden[f"ablation_{i}_pixels"]
        chunk = hs.PackedChunk(oracle.pack(px))
        pattern = hs.compute_binning_pattern(hs.reference_histogram(chunk))
        cfg = hs.WorkerGroupConfig(case["group_size"], case["group_count"])
        for stage in hs.ABLATION_STAGES:
            got = hs.run_ablation(chunk, stage, pattern, cfg)
            assert got.checksum == case["checksums"][stage.value], (i, stage)
    chunk = hs.generate(hs.SourceSpec("uniform", 1 << 22, seed=13))
    pattern = hs.compute_binning_pattern(hs.reference_histogram(chunk))
    cfg = hs.WorkerGroupConfig(32, 2)
    full = hs.run_ablation(chunk, hs.KernelKind.FULL, pattern, cfg)
    assert full.histogram == hs.reference_histogram(chunk) and full.throughput_bps > 0
    want = oracle.ablation_checksums(chunk.pixels(), pattern.offset, pattern.count, 2)
    for stage in hs.ABLATION_STAGES:
        a = hs.run_ablation(chunk, stage, pattern, cfg)
        b = hs.run_ablation(chunk, stage, pattern, cfg)
        assert a.checksum == b.checksum == want[stage.value], stage
    with pytest.raises(ValueError):
        hs.run_ablation(chunk, hs.KernelKind.NAIVE, pattern, cfg)


def test_scheduling_independent(cuda):
    chunk = hs.generate(hs.SourceSpec("mixture", 1 << 14, seed=6, value=127, degeneracy=0.7))
    cfg = hs.WorkerGroupConfig(32, 4)
    runs = [hs.naive_histogram(chunk, cfg) for _ in range(5)] + [hs.adaptive_histogram(chunk, deg_pattern(), cfg) for _ in range(5)]
    assert all(r == runs[0] for r in runs)
    s1 = hs.adaptive_histogram(chunk, deg_pattern(), cfg, return_slots=True)[1]
    s2 = hs.adaptive_histogram(chunk, deg_pattern(), cfg, return_slots=True)[1]
    assert all((a == b).all() for a, b in zip(s1, s2))


def test_device_generators_match_host(cuda, oracle):
    torch = cuda
    for spec in (hs.SourceSpec("uniform", 1 << 20, 0xABC), hs.SourceSpec("normal", (1 << 18) + 4, 5, mean=128.0, sigma=8.0),
                 hs.SourceSpec("sequential", 1000), hs.SourceSpec("constant", 4096, value=9)):
        want = hs.unpack_chunk(hs.generate(spec))
        for first in (0, 12, 4100):
            n = spec.pixels - first if first < spec.pixels else 0
            buf = torch.empty(n, dtype=torch.uint8, device="cuda")
            hs.generate_device(spec, buf, first)
            assert np.array_equal(buf.cpu().numpy(), want[first:]), (spec.kind, first)


def test_concurrent_threads(cuda, oracle):
    import threading

    px = oracle.generate("uniform", 1 << 20, 42)
    chunk = hs.PackedChunk(oracle.pack(px))
    want = oracle.histogram(px)
    errors = []

    def work():
        try:
            for _ in range(5):
                assert np.array_equal(hs.naive_histogram(chunk, hs.WorkerGroupConfig()).counts, want)
        except BaseException as e:  # pragma: no cover
            errors.append(e)

    th = [threading.Thread(target=work) for _ in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    assert not errors


def test_ticketed_output_matches_atomic_output(cuda, oracle):
    """Single-launch path (workspace tickets, no memset) vs the memset + RED path of
    the same ABI call, over ragged layouts: empty segments, tiny segments sharing a
    CTA, segments spanning many CTAs, > 64 segments (several launches)."""
    torch = cuda
    L = N.lib()
    rng = np.random.default_rng(77)
    px = oracle.generate("normal", 64 << 20, 3, mean=128.0, sigma=20.0)
    dev = torch.from_numpy(px).cuda()
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    stream = torch.cuda.current_stream().cuda_stream
    pat = hs.uniform_pattern(960)
    for trial in range(12):
        nseg = int(rng.integers(1, 150))
        lens = rng.integers(0, (px.size // nseg) // 4 + 1, nseg) * 4
        lens[rng.integers(0, nseg, max(1, nseg // 5))] = 0  # some empty segments
        if trial % 3 == 0:
            lens[:] = 4 * rng.integers(0, 64, nseg)  # tiny segments: many per CTA
        begin = np.concatenate([[0], np.cumsum(lens)[:-1]]).astype(np.uint64)
        end = begin + lens.astype(np.uint64)
        want = np.stack([oracle.histogram(px[int(a):int(b)]) for a, b in zip(begin, end)])
        for kind in (N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE):
            for use_ws in (True, False):
                out = torch.full((nseg, 256), -1, dtype=torch.int64, device="cuda")
                st = L.hs_histogram_batched(dev.data_ptr(), N.u64p(begin), N.u64p(end), nseg, kind, 0,
                                            N.i64p(pat.offset), N.i64p(pat.count), 960, 8, out.data_ptr(),
                                            ws.data_ptr() if use_ws else None, ws.numel() if use_ws else 0, stream)
                N.check(st, "hs_histogram_batched")
                assert np.array_equal(out.cpu().numpy().view(np.uint64), want), (trial, kind, use_ws)
    # every launch leaves the workspace (tickets and accumulator rows) zero again
    assert ws_clean(ws)


@pytest.mark.parametrize("p", [0.5, 0.99, 0.9995])
def test_register_path_on_partially_hot_data(cuda, oracle, p):
    """The ADAPTIVE register path (hot bin counted per all-hot 16-byte vector) forced on
    mixtures where only some vectors are all hot, at sizes with head/tail words and a
    remainder; and the API's choice (spread hint below dominance 0.999) on the same
    data. Both exact."""
    torch = cuda
    n = (1 << 22) + 4 * 37
    host = oracle.generate("mixture", n, 11, value=200, degeneracy=p)
    want = oracle.histogram(host)
    buf = torch.from_numpy(host.copy()).cuda()
    pat = deg_pattern(200)  # unique widest run at 200: hot_unique, dominance 1.0
    L = N.lib()
    for off in (0, 4, 12):
        seg = buf[off:n - 8]
        exp = oracle.histogram(host[off:n - 8])
        b0 = np.zeros(1, np.uint64)
        b1 = np.full(1, seg.numel(), np.uint64)
        out = torch.empty((1, 256), dtype=torch.int64, device="cuda")
        ws = D.default_staging().workspace()
        for kind in (N.HS_KIND_ADAPTIVE, N.HS_KIND_ADAPTIVE | N.HS_KIND_FLAG_SPREAD):
            N.check(L.hs_histogram_batched(seg.data_ptr(), N.u64p(b0), N.u64p(b1), 1, kind, N.HS_IMPL_LANE,
                                           N.i64p(pat.offset), N.i64p(pat.count), 960, 8, out.data_ptr(),
                                           ws.data_ptr(), ws.numel(), torch.cuda.current_stream().cuda_stream), "h")
            assert out.cpu().numpy().view(np.uint64)[0].tolist() == exp.tolist(), (p, off, kind)
    prior = hs.compute_binning_pattern(hs.Histogram256(want))
    assert (prior.dominance >= D.SPREAD_BELOW) == (p >= 0.999)
    got = hs.adaptive_histogram(hs.DeviceChunk(buf), prior, hs.WorkerGroupConfig())
    assert got.counts.tolist() == want.tolist()


def test_graph_replay_ticketed(cuda, oracle):
    """Ticketed launches captured into a CUDA graph (programmatic edges between them)
    give the same counts on every replay: each launch leaves its workspace zeroed."""
    torch = cuda
    n = (48 << 20) + 12
    host = oracle.generate("normal", n, 5, mean=100.0, sigma=20.0)
    buf = torch.from_numpy(host.copy()).cuda()
    want = oracle.histogram(host)
    L = N.lib()
    b0 = np.array([0, 4096, 12 << 20], np.uint64)
    b1 = np.array([4096, 12 << 20, n], np.uint64)
    parts = [oracle.histogram(host[int(a):int(b)]) for a, b in zip(b0, b1)]
    assert (sum(parts) == want).all()
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    outs = [torch.empty((3, 256), dtype=torch.int64, device="cuda") for _ in range(3)]
    side = torch.cuda.Stream()

    def enqueue():
        s = torch.cuda.current_stream().cuda_stream
        for o in outs:
            N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), 3, N.HS_KIND_NAIVE,
                                           N.HS_IMPL_LANE, None, None, 0, 0, o.data_ptr(), ws.data_ptr(),
                                           ws.numel(), s), "graph")

    with torch.cuda.stream(side):
        enqueue()
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=side):
        enqueue()
    for _ in range(3):
        for o in outs:
            o.fill_(-1)
        g.replay()
        torch.cuda.synchronize()
        for o in outs:
            got = o.cpu().numpy().view(np.uint64)
            for k in range(3):
                assert got[k].tolist() == parts[k].tolist()
    assert ws_clean(ws)


@pytest.mark.parametrize("seed", range(4))
def test_fuzz_segment_layouts(cuda, oracle, seed):
    """Random batches through the C ABI: 1-300 segments of random word-multiple sizes
    (empty ones included) at random word offsets of one buffer, every impl and kind,
    with a workspace sized for 64 or 256 segments or none. Counts equal the oracle's."""
    torch = cuda
    rng = np.random.default_rng(1000 + seed)
    n = 48 << 20
    host = rng.integers(0, 256, n, dtype=np.uint8)
    host[: n // 3] = rng.integers(120, 136, n // 3, dtype=np.uint8)  # a concentrated stretch
    buf = torch.from_numpy(host).cuda()
    L = N.lib()
    st = torch.cuda.current_stream().cuda_stream
    pat = hs.compute_binning_pattern(hs.Histogram256(np.bincount(host[:1 << 20], minlength=256).astype(np.uint64)))
    for trial in range(12):
        nseg = int(rng.choice([1, 2, 7, 64, 65, 200, 256, 300]))
        sizes = rng.choice([0, 4, 64, 4096, 1 << 16, 1 << 20, 3 << 20], size=nseg) + 4 * rng.integers(0, 64, nseg)
        sizes[rng.random(nseg) < 0.1] = 0
        starts = 4 * rng.integers(0, (n - int(sizes.max()) - 4) // 4, nseg)
        b0 = starts.astype(np.uint64)
        b1 = (starts + sizes).astype(np.uint64)
        want = np.stack([oracle.histogram(host[a:b]) for a, b in zip(b0, b1)])
        impl = int(rng.choice([N.HS_IMPL_AUTO, N.HS_IMPL_LANE, N.HS_IMPL_WARP]))
        kind = int(rng.choice([N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE]))
        ws_seg = int(rng.choice([0, 64, 256]))
        ws = torch.zeros(int(L.hs_workspace_bytes(ws_seg)) if ws_seg else 1, dtype=torch.uint8, device="cuda")
        out = torch.full((nseg, 256), -1, dtype=torch.int64, device="cuda")
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, kind, impl,
                                       N.i64p(pat.offset), N.i64p(pat.count), 960, 8, out.data_ptr(),
                                       ws.data_ptr() if ws_seg else None, ws.numel() if ws_seg else 0, st), "fuzz")
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), (seed, trial, nseg, impl, kind, ws_seg)
        if ws_seg:
            assert ws_clean(ws)


def test_concurrent_streams_separate_workspaces(cuda, oracle):
    """The bench's arrangement: three CUDA streams, each with its own workspace, each
    issuing chained (PDL) 64-segment launches while the others run; every output exact."""
    torch = cuda
    L = N.lib()
    seg = 1 << 20
    bufs, wants = [], []
    for j in range(3):
        host = oracle.generate("normal", 64 * seg, 40 + j, mean=128.0, sigma=8.0 * (j + 1))
        bufs.append(torch.from_numpy(host).cuda())
        wants.append(np.stack([oracle.histogram(host[c * seg:(c + 1) * seg]) for c in range(64)]))
    b0 = np.arange(64, dtype=np.uint64) * seg
    b1 = b0 + seg
    streams = [torch.cuda.Stream() for _ in range(3)]
    wss = [torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda") for _ in range(3)]
    outs = [[torch.full((64, 256), -1, dtype=torch.int64, device="cuda") for _ in range(5)] for _ in range(3)]
    torch.cuda.synchronize()
    for k in range(5):
        for j in range(3):
            N.check(L.hs_histogram_batched(bufs[j].data_ptr(), N.u64p(b0), N.u64p(b1), 64, N.HS_KIND_NAIVE,
                                           N.HS_IMPL_LANE, None, None, 0, 0, outs[j][k].data_ptr(),
                                           wss[j].data_ptr(), wss[j].numel(), streams[j].cuda_stream), "concurrent")
    torch.cuda.synchronize()
    for j in range(3):
        for k in range(5):
            assert np.array_equal(outs[j][k].cpu().numpy().view(np.uint64), wants[j]), (j, k)
        assert ws_clean(wss[j])


def _sync_call(lib, d, begin, end, h_out, d_out, ws, impl=N.HS_IMPL_AUTO):
    import torch

    b = np.ascontiguousarray(begin, np.uint64)
    e = np.ascontiguousarray(end, np.uint64)
    import ctypes

    h_p = N.u64p(h_out) if isinstance(h_out, np.ndarray) else ctypes.cast(h_out.data_ptr(), N._U64P)
    st = lib.hs_histogram_sync(d.data_ptr(), N.u64p(b), N.u64p(e), len(b), N.HS_KIND_NAIVE, impl, None, None, 0, 0,
                               d_out.data_ptr(), h_p, ws.data_ptr() if ws is not None else None,
                               ws.numel() if ws is not None else 0, torch.cuda.current_stream().cuda_stream)
    N.check(st, "hs_histogram_sync")


def test_blocking_entries_host_out_forms(cuda, oracle):
    """hs_histogram_sync / hs_histogram_host with a page-locked h_out (written by the
    kernel directly on the ticketed path), a pageable h_out (D2H copy), a non-ticketed
    impl and no workspace with a page-locked h_out (copy path), including empty and
    all-empty segment lists; the counts must be the same in every form."""
    import ctypes
    import torch

    lib = N.lib()
    rng = np.random.default_rng(11)
    px = rng.integers(0, 256, (3 << 20) + 40, dtype=np.uint8)
    d = torch.from_numpy(px).cuda()
    cuts = [0, 4, 4, 1 << 20, (1 << 20) + 4, (3 << 20) + 40]
    begin, end = cuts[:-1], cuts[1:]
    want = np.stack([oracle.histogram(px[a:b]) for a, b in zip(begin, end)])
    ws = torch.zeros(int(lib.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    n = len(begin)
    for h_kind in ("pinned", "pageable"):
        for impl, use_ws in ((N.HS_IMPL_AUTO, True), (N.HS_IMPL_LANE, True), (N.HS_IMPL_WARP, True),
                             (N.HS_IMPL_AUTO, False)):
            d_out = torch.full((n, 256), 7, dtype=torch.int64, device="cuda")
            if h_kind == "pinned":
                h = torch.full((n * 256,), 9, dtype=torch.int64).pin_memory()
                _sync_call(lib, d, begin, end, h, d_out, ws if use_ws else None, impl)
                got = h.numpy().view(np.uint64).reshape(n, 256)
            else:
                got = np.full((n, 256), 9, np.uint64)
                _sync_call(lib, d, begin, end, got, d_out, ws if use_ws else None, impl)
            assert np.array_equal(got, want), (h_kind, impl, use_ws)
    # all-empty list and an empty device chunk through the pinned direct form
    h = torch.full((2 * 256,), 9, dtype=torch.int64).pin_memory()
    _sync_call(lib, d, [0, 8], [0, 8], h, torch.empty((2, 256), dtype=torch.int64, device="cuda"), ws)
    assert not h.numpy().any()
    # hs_histogram_host: pinned and pageable h_out, pageable sources
    chunks = [px[:1 << 20], px[(1 << 20) + 4:(2 << 20)], px[:0]]
    ptrs = (ctypes.c_void_p * 3)(*[c.ctypes.data if c.size else None for c in chunks])
    sizes = np.array([c.size for c in chunks], np.uint64)
    stage = torch.empty(4 << 20, dtype=torch.uint8, device="cuda")
    d_out = torch.empty((3, 256), dtype=torch.int64, device="cuda")
    want_h = np.stack([oracle.histogram(c) for c in chunks])
    for pinned in (True, False):
        h = torch.full((3 * 256,), 9, dtype=torch.int64)
        if pinned:
            h = h.pin_memory()
        st = lib.hs_histogram_host(ptrs, N.u64p(sizes), 3, N.HS_KIND_NAIVE, N.HS_IMPL_AUTO, None, None, 0, 0,
                                   stage.data_ptr(), stage.numel(), d_out.data_ptr(),
                                   ctypes.cast(h.data_ptr(), N._U64P), ws.data_ptr(), ws.numel(),
                                   torch.cuda.current_stream().cuda_stream)
        N.check(st, "hs_histogram_host")
        assert np.array_equal(h.numpy().view(np.uint64).reshape(3, 256), want_h), pinned


def test_single_chunk_fast_path_buffers_regrow(cuda, oracle):
    """The one-chunk API path caches its ctypes arguments per staging; a larger batch in
    between replaces the staging buffers, and the next single call must use the new
    ones (and a new pattern object its own pointers)."""
    import torch

    cfg = hs.WorkerGroupConfig()
    px = oracle.generate("normal", (1 << 20) + 4, 5, mean=100.0, sigma=9.0)
    host = hs.PackedChunk(oracle.pack(px))
    dev = hs.DeviceChunk(torch.from_numpy(px).cuda())
    want = oracle.histogram(px)
    p1 = hs.compute_binning_pattern(hs.Histogram256(want))
    for _ in range(2):
        assert np.array_equal(hs.naive_histogram(host, cfg).counts, want)
        assert np.array_equal(hs.adaptive_histogram(dev, p1, cfg).counts, want)
        big = [hs.PackedChunk(oracle.pack(oracle.generate("uniform", 1 << 16, s))) for s in range(300)]
        outs = hs.batch_histograms(big, hs.KernelKind.NAIVE, None, cfg)
        assert all(o.total() == 1 << 16 for o in outs)
        long_px = oracle.generate("uniform", 24 << 20, 3)
        assert np.array_equal(hs.naive_histogram(hs.PackedChunk(oracle.pack(long_px)), cfg).counts,
                              oracle.histogram(long_px))
        p2 = hs.uniform_pattern(960)
        assert np.array_equal(hs.adaptive_histogram(host, p2, cfg).counts, want)
        assert np.array_equal(hs.adaptive_histogram(dev, p1, cfg).counts, want)
        assert hs.naive_histogram(hs.PackedChunk(np.zeros(0, np.uint32)), cfg).total() == 0
        assert hs.naive_histogram(hs.DeviceChunk(torch.empty(0, dtype=torch.uint8, device="cuda")), cfg).total() == 0
