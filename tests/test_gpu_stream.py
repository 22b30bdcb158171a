"""GPU streaming engine: run_pipeline == run_sequential, both == the reference's own
run_sequential output (golden streams), double-buffer protocol order, switching
latency and pipeline timing arithmetic. Mirrors test_stream.py and acceptance
c06/c07/c09/c10 (test_acceptance.py:201-314)."""
import io

import numpy as np
import pytest

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200.datagen import batch_stream, schedule_stream

pytestmark = pytest.mark.gpu

SMALL = hs.WorkerGroupConfig(group_size=8, group_count=2)
POLICY = hs.SwitchPolicy()


def small_cfg(**kw):
    base = dict(num_iterations=8, chunk_pixels=512, window_size=4, worker=SMALL)
    base.update(kw)
    return hs.PipelineConfig(**base)


def uniform_source(cfg, seed=0):
    return batch_stream(hs.SourceSpec("uniform", cfg.chunk_pixels, seed), cfg.num_iterations, cfg.batch_size)


def states_equal(a, b):
    return (a[0] == b[0] and a[1] == b[1] and a[3] == b[3]
            and a[2].per_slice_histograms == b[2].per_slice_histograms
            and a[2].degeneracy_log == b[2].degeneracy_log and a[2].divergence_log == b[2].divergence_log)


def _segments(meta):
    return [(hs.SourceSpec(s["kind"], s["pixels"], s["seed"], s["value"], s["mean"], s["sigma"], s["degeneracy"]), n)
            for s, n in meta["segments"]]


def test_streams_match_reference(cuda, golden):
    for i, m in enumerate(golden.meta["streams"]):
        cfg = hs.PipelineConfig(num_iterations=m["num_iterations"], chunk_pixels=m["chunk_pixels"],
                                batch_size=m["batch_size"], recompute_pattern_every=m["recompute_pattern_every"],
                                window_size=m["window_size"], worker=hs.WorkerGroupConfig(4, 2))
        for runner in (hs.run_sequential, hs.run_pipeline):
            acc, win, rep, log = runner(schedule_stream(_segments(m), m["batch_size"]), cfg, POLICY)
            assert [k.value for k in log] == m["kernel_log"], (i, runner.__name__)
            per = np.stack([np.stack([h.counts for h in it]) for it in rep.per_slice_histograms])
            assert np.array_equal(per, golden[f"stream_{i}_per_slice"])
            assert np.array_equal(acc.running.counts, golden[f"stream_{i}_acc"]) and acc.chunks_seen == m["chunks_seen"]
            assert np.array_equal(win.windowed.counts, golden[f"stream_{i}_window"])
            assert np.array_equal(np.stack([h.counts for h in win.ring]), golden[f"stream_{i}_ring"])
            assert rep.degeneracy_log == golden[f"stream_{i}_deg"].tolist()
            assert rep.divergence_log == golden[f"stream_{i}_div"].tolist()


def test_pipeline_equals_sequential_batched(cuda):
    cfg = small_cfg(batch_size=3, num_iterations=5)
    seq = hs.run_sequential(uniform_source(cfg, 8), cfg, POLICY)
    pipe = hs.run_pipeline(uniform_source(cfg, 8), cfg, POLICY)
    assert states_equal(seq, pipe) and seq[0].chunks_seen == 15


def test_degeneracy_flip(cuda):
    cfg = small_cfg(num_iterations=12, window_size=2)
    segs = [(hs.SourceSpec("uniform", cfg.chunk_pixels, 1), 6), (hs.SourceSpec("constant", cfg.chunk_pixels, 1, value=127), 6)]
    seq = hs.run_sequential(schedule_stream(segs), cfg, POLICY)
    pipe = hs.run_pipeline(schedule_stream(segs), cfg, POLICY)
    assert states_equal(seq, pipe) and hs.KernelKind.ADAPTIVE in pipe[3]


@pytest.mark.parametrize("every", [1, 3])
def test_switch_latency(cuda, every):
    # c10 (test_acceptance.py:292-314)
    pixels, change = 2048, 100
    segs = [(hs.SourceSpec("uniform", pixels, seed=10), change), (hs.SourceSpec("constant", pixels, seed=10, value=127), change)]
    cfg = hs.PipelineConfig(num_iterations=2 * change, chunk_pixels=pixels, window_size=2,
                            recompute_pattern_every=every, worker=hs.WorkerGroupConfig(4, 2))
    _, _, _, log = hs.run_pipeline(schedule_stream(segs), cfg, hs.SwitchPolicy(0.45))
    assert all(k is hs.KernelKind.NAIVE for k in log[:change + 1])
    flip = next(i for i, k in enumerate(log) if k is hs.KernelKind.ADAPTIVE)
    assert flip <= change + every + 1
    assert all(k is hs.KernelKind.ADAPTIVE for k in log[flip:])


def test_source_exhausted_and_errors(cuda):
    cfg = small_cfg(num_iterations=10)
    for runner in (hs.run_sequential, hs.run_pipeline):
        with pytest.raises(hs.SourceExhausted):
            runner(uniform_source(small_cfg(num_iterations=3), 1), cfg, POLICY)

    def broken():
        yield [hs.generate(hs.SourceSpec("uniform", 512, 0))]
        raise RuntimeError("source failure")

    with pytest.raises(RuntimeError, match="source failure"):
        hs.run_pipeline(broken(), small_cfg(num_iterations=3), POLICY)


def test_buffer_protocol_order(cuda):
    cfg = small_cfg(num_iterations=9)
    events = []
    hs.run_pipeline(uniform_source(cfg, 9), cfg, POLICY, instrument=events)
    for b in (0, 1):
        mine = [(ev, it) for buf, ev, it in events if buf == b]
        want = []
        for it in range(b, 9, 2):
            want += [("acquire_write", it), ("publish", it), ("take", it), ("release", it)]
        assert mine == want
    pos = {e: i for i, e in enumerate(events)}
    for b, ev, it in events:
        if ev == "acquire_write" and it >= 2:
            assert pos[(b, "release", it - 2)] < pos[(b, ev, it)]


def test_timing_structure(cuda):
    cfg = small_cfg()
    _, _, report, _ = hs.run_sequential(uniform_source(cfg, 2), cfg, POLICY)
    assert report.total_sequential_ns == report.total_pipelined_ns and report.pipelined_ratio == 1.0
    profile = hs.StageProfile(cpu_pre_us=1000, transfer_in_us=800, compute_us=3000, transfer_out_us=10)
    ratios = {}
    for n in (1, 8):
        cfg = small_cfg(num_iterations=n, stage_profile=profile)
        _, _, rep, _ = hs.run_pipeline(uniform_source(cfg, 4), cfg, POLICY)
        assert rep.total_pipelined_ns <= rep.total_sequential_ns
        ratios[n] = rep.pipelined_ratio
    assert ratios[8] < ratios[1]


def test_table3_pipeline_arithmetic(cuda):
    # c06 (test_acceptance.py:201-210): Table 3 stage shares, 256 iterations
    prof = hs.StageProfile(cpu_pre_us=2028.0, transfer_in_us=1768.0, compute_us=6201.0, transfer_out_us=2.0)
    cfg = hs.PipelineConfig(num_iterations=256, chunk_pixels=1024, window_size=8, worker=hs.WorkerGroupConfig(4, 2),
                            stage_profile=prof)
    _, _, rep, _ = hs.run_pipeline(batch_stream(hs.SourceSpec("uniform", 1024, 606), 256), cfg, POLICY)
    assert 0.60 <= rep.pipelined_ratio <= 0.68


def test_csv_schema(cuda):
    cfg = small_cfg(num_iterations=3)
    _, _, report, _ = hs.run_sequential(uniform_source(cfg, 11), cfg, POLICY)
    buf = io.StringIO()
    report.to_csv(buf)
    lines = buf.getvalue().strip().splitlines()
    assert lines[0] == "iteration,cpu_pre_us,transfer_in_us,compute_us,transfer_out_us,cpu_post_us,kernel_kind"
    assert len(lines) == 5 and lines[1].startswith("0,") and lines[1].endswith(",naive")
    assert abs(float(lines[-1].split(",")[3]) - 100.0) < 1.0


def test_device_resident_stream(cuda, oracle):
    torch = cuda
    # chunks already in HBM (the C2 configuration's device-resident form)
    n_chunks, px = 8, 1 << 20
    dev = torch.empty(n_chunks * px, dtype=torch.uint8, device="cuda")
    spec = hs.SourceSpec("normal", px, 77, mean=128.0, sigma=32.0)
    for i in range(n_chunks):
        hs.generate_device(hs.SourceSpec("normal", px, 77 ^ i, mean=128.0, sigma=32.0), dev[i * px:(i + 1) * px])

    def src():
        for i in range(n_chunks):
            yield [hs.DeviceChunk(dev[i * px:(i + 1) * px])]

    cfg = hs.PipelineConfig(num_iterations=n_chunks, chunk_pixels=px, window_size=4)
    acc, _, rep, log = hs.run_pipeline(src(), cfg, POLICY)
    want = [oracle.histogram(oracle.generate("normal", px, 77 ^ i, mean=128.0, sigma=32.0)) for i in range(n_chunks)]
    assert [h[0].counts.tolist() for h in rep.per_slice_histograms] == [w.tolist() for w in want]
    assert acc.running.counts.tolist() == np.sum(want, axis=0).tolist()


def _device_batches(torch, segments, batch_size):
    for batch in schedule_stream(segments, batch_size):
        yield [hs.DeviceChunk(torch.from_numpy(c.pixels().copy()).cuda()) for c in batch]


def test_device_stream_matches_reference(cuda, golden):
    """hs_stream_step (fold + policy on the device) reproduces the reference's own
    run_sequential: kernel log, per-slice histograms, accumulator, window ring and the
    float degeneracy/divergence logs, bit for bit."""
    for i, m in enumerate(golden.meta["streams"]):
        cfg = hs.PipelineConfig(num_iterations=m["num_iterations"], chunk_pixels=m["chunk_pixels"],
                                batch_size=m["batch_size"], recompute_pattern_every=m["recompute_pattern_every"],
                                window_size=m["window_size"], worker=hs.WorkerGroupConfig(4, 2))
        acc, win, rep, log = hs.run_device_stream(_device_batches(cuda, _segments(m), m["batch_size"]), cfg, POLICY)
        assert [k.value for k in log] == m["kernel_log"], i
        per = np.stack([np.stack([h.counts for h in it]) for it in rep.per_slice_histograms])
        assert np.array_equal(per, golden[f"stream_{i}_per_slice"])
        assert np.array_equal(acc.running.counts, golden[f"stream_{i}_acc"]) and acc.chunks_seen == m["chunks_seen"]
        assert np.array_equal(win.windowed.counts, golden[f"stream_{i}_window"])
        assert np.array_equal(np.stack([h.counts for h in win.ring]), golden[f"stream_{i}_ring"])
        assert rep.degeneracy_log == golden[f"stream_{i}_deg"].tolist(), i
        assert rep.divergence_log == golden[f"stream_{i}_div"].tolist(), i


def test_device_stream_equals_host_engine_at_scale(cuda):
    """16 MiB chunks (the C2/C3 configuration): normal sigma 8 -> mixture -> constant, so
    the on-device switch flips NAIVE -> ADAPTIVE mid-stream; equal to run_sequential."""
    px = 1 << 24
    segs = [(hs.SourceSpec("normal", px, 3, mean=128.0, sigma=8.0), 4),
            (hs.SourceSpec("mixture", px, 3, value=200, degeneracy=0.9), 3),
            (hs.SourceSpec("constant", px, 3, value=127), 3)]
    cfg = hs.PipelineConfig(num_iterations=10, chunk_pixels=px, window_size=2)
    seq = hs.run_sequential(schedule_stream(segs), cfg, POLICY)
    dev = hs.run_device_stream(_device_batches(cuda, segs, 1), cfg, POLICY)
    assert states_equal(seq, dev)
    assert hs.KernelKind.ADAPTIVE in dev[3] and dev[3][0] is hs.KernelKind.NAIVE


def test_device_stream_rejects_foreign_chunks(cuda):
    cfg = small_cfg(num_iterations=2)
    with pytest.raises(TypeError):
        hs.run_device_stream(iter([[np.zeros(16, np.uint8)], [np.zeros(16, np.uint8)]]), cfg, POLICY)


@pytest.mark.parametrize("kind", ["pageable", "pinned", "mixed"])
def test_device_stream_from_host_chunks(cuda, golden, kind):
    """Host PackedChunks through the device engine (staged a block at a time on a copy
    stream one block ahead): the reference's own run_sequential results bit for bit --
    pageable chunks (bounce buffer), page-locked ones (direct DMA) and blocks mixing host
    and device chunks; small blocks force many staging-slot reuses."""
    torch = cuda
    from paper_1011_0235_b200 import device as D

    def host_batches(m):
        for j, batch in enumerate(schedule_stream(_segments(m), m["batch_size"])):
            out = []
            for k, c in enumerate(batch):
                if kind == "pinned" or (kind == "mixed" and (j + k) % 3 == 1):
                    w = D.pinned_words(c.words.size)
                    w[:] = c.words
                    out.append(hs.PackedChunk(w))
                elif kind == "mixed" and (j + k) % 3 == 2:
                    out.append(hs.DeviceChunk(torch.from_numpy(c.pixels().copy()).cuda()))
                else:
                    out.append(c)
            yield out

    for i, m in enumerate(golden.meta["streams"]):
        cfg = hs.PipelineConfig(num_iterations=m["num_iterations"], chunk_pixels=m["chunk_pixels"],
                                batch_size=m["batch_size"], recompute_pattern_every=m["recompute_pattern_every"],
                                window_size=m["window_size"], worker=hs.WorkerGroupConfig(4, 2))
        block = 3 * m["chunk_pixels"] * m["batch_size"]  # a few iterations per block
        acc, win, rep, log = hs.run_device_stream(host_batches(m), cfg, POLICY, block_bytes=block)
        assert [k.value for k in log] == m["kernel_log"], (kind, i)
        per = np.stack([np.stack([h.counts for h in it]) for it in rep.per_slice_histograms])
        assert np.array_equal(per, golden[f"stream_{i}_per_slice"]), (kind, i)
        assert np.array_equal(acc.running.counts, golden[f"stream_{i}_acc"]) and acc.chunks_seen == m["chunks_seen"]
        assert np.array_equal(win.windowed.counts, golden[f"stream_{i}_window"])
        assert rep.degeneracy_log == golden[f"stream_{i}_deg"].tolist(), (kind, i)
        assert rep.divergence_log == golden[f"stream_{i}_div"].tolist(), (kind, i)


def test_device_stream_host_chunks_at_scale(cuda):
    """1 MiB pageable chunks, batch 1 (the reference's default pipeline shape), 600
    iterations in 64 MiB blocks: equal to run_sequential on the same source."""
    px = 1 << 20
    segs = [(hs.SourceSpec("uniform", px, 31), 250), (hs.SourceSpec("constant", px, 31, value=77), 150),
            (hs.SourceSpec("normal", px, 31, mean=100.0, sigma=16.0), 200)]
    cfg = hs.PipelineConfig(num_iterations=600, chunk_pixels=px, window_size=32)
    seq = hs.run_sequential(schedule_stream(segs), cfg, POLICY)
    dev = hs.run_device_stream(schedule_stream(segs), cfg, POLICY, block_bytes=64 << 20)
    assert states_equal(seq, dev)
    assert [k.value for k in seq[3]] == [k.value for k in dev[3]]


@pytest.mark.parametrize("window,batch", [(1, 37), (4, 64), (15, 20), (16, 5), (16, 37), (23, 16), (32, 40), (33, 64), (64, 64)])
def test_device_stream_batched_fold(cuda, window, batch):
    """Every fold path: windows < 16 keep the ring in shared memory, 16..31 read evicted
    slots one push at a time, >= 32 load the chunk histograms and the ring slots they
    evict 32 at a time before applying the pushes; batches of 5..64 chunks wrap the
    ring inside one iteration. Equal to the host engine."""
    px = 4096
    segs = [(hs.SourceSpec("uniform", px, 21), 4), (hs.SourceSpec("constant", px, 21, value=9), 3),
            (hs.SourceSpec("normal", px, 21, mean=128.0, sigma=4.0), 4)]
    cfg = hs.PipelineConfig(num_iterations=11, chunk_pixels=px, batch_size=batch, window_size=window)
    seq = hs.run_sequential(schedule_stream(segs, batch), cfg, POLICY)
    dev = hs.run_device_stream(_device_batches(cuda, segs, batch), cfg, POLICY)
    assert states_equal(seq, dev)
    assert [k.value for k in seq[3]] == [k.value for k in dev[3]]
    assert np.array_equal(np.stack([h.counts for h in seq[1].ring]), np.stack([h.counts for h in dev[1].ring]))


def test_pinned_chunks_dma_directly_pageable_through_bounce(cuda, oracle):
    """Staging keeps page-locked chunks on the direct DMA path for as long as any view of
    them lives (the registry follows the memory, not the tensor that allocated it), and
    copies pageable chunks through the staging's pinned bounce buffer; counts exact."""
    import gc

    torch = cuda
    from paper_1011_0235_b200 import device as D

    arr = D.pinned_bytes(1 << 20)
    arr[:] = oracle.generate("normal", 1 << 20, 5, mean=90.0, sigma=20.0)
    words = arr.view(np.uint32)[16:]
    want = oracle.histogram(arr[64:64 + 4096])
    del arr
    gc.collect()
    assert D.is_pinned(words)
    st = D.Staging()
    stream = torch.cuda.current_stream()
    staged = D.stage([hs.PackedChunk(words[:1024])], st, stream)
    assert st._bounce is None  # direct DMA
    out = D.launch(staged, 0, None, stream, staging=st)  # HS_KIND_NAIVE
    assert np.array_equal(out.cpu().numpy().view(np.uint64)[0], want)
    page = np.ascontiguousarray(words[:1024]).copy()
    assert not D.is_pinned(page)
    staged = D.stage([hs.PackedChunk(page)], st, stream)
    assert st._bounce is not None
    out = D.launch(staged, 0, None, stream, staging=st)
    assert np.array_equal(out.cpu().numpy().view(np.uint64)[0], want)


def test_pageable_batches_back_to_back_on_one_staging(cuda, oracle):
    """Two pageable batches staged on one Staging with no synchronisation in between: the
    second waits for the first's DMA out of the bounce buffer before refilling it."""
    torch = cuda
    from paper_1011_0235_b200 import device as D

    st = D.Staging()
    stream = torch.cuda.current_stream()
    a = oracle.generate("normal", 8 << 20, 11, mean=60.0, sigma=10.0)
    b = oracle.generate("normal", 8 << 20, 12, mean=190.0, sigma=10.0)
    s1 = D.stage([hs.PackedChunk(a.view(np.uint32))], st, stream)
    out1 = D.launch(s1, 0, None, stream, staging=st).clone()
    st2 = D.Staging()  # a second device buffer, the same bounce-buffer discipline
    s2 = D.stage([hs.PackedChunk(b.view(np.uint32))], st2, stream)
    out2 = D.launch(s2, 0, None, stream, staging=st2)
    s3 = D.stage([hs.PackedChunk(b.view(np.uint32))], st, stream)  # refills st's bounce buffer
    out3 = D.launch(s3, 0, None, stream, staging=st)
    assert np.array_equal(out1.cpu().numpy().view(np.uint64)[0], oracle.histogram(a))
    assert np.array_equal(out2.cpu().numpy().view(np.uint64)[0], oracle.histogram(b))
    assert np.array_equal(out3.cpu().numpy().view(np.uint64)[0], oracle.histogram(b))


def test_device_stream_host_chunks_source_errors(cuda):
    """A source that ends early or raises mid-run with host blocks staged: the
    reference's exceptions propagate (SourceExhausted, the source's own error)."""
    px = 1 << 16
    cfg = hs.PipelineConfig(num_iterations=40, chunk_pixels=px, window_size=4)

    def short():
        for j in range(25):
            yield [hs.generate(hs.SourceSpec("uniform", px, j))]

    with pytest.raises(hs.SourceExhausted):
        hs.run_device_stream(short(), cfg, POLICY, block_bytes=4 * px)

    def broken():
        for j in range(30):
            if j == 17:
                raise RuntimeError("source broke")
            yield [hs.generate(hs.SourceSpec("uniform", px, j))]

    with pytest.raises(RuntimeError, match="source broke"):
        hs.run_device_stream(broken(), cfg, POLICY, block_bytes=4 * px)


def test_pipeline_resources_reused_after_errors(cuda):
    # run_pipeline keeps its streams and readback staging per thread: a run that failed
    # (source error, exhausted source) must leave them usable, and every later run exact
    cfg = small_cfg(batch_size=3, num_iterations=6)
    want = hs.run_sequential(uniform_source(cfg, 21), cfg, POLICY)

    def broken():
        yield [hs.generate(hs.SourceSpec("uniform", cfg.chunk_pixels, 5)) for _ in range(3)]
        raise RuntimeError("source failure")

    for _ in range(3):
        with pytest.raises(RuntimeError, match="source failure"):
            hs.run_pipeline(broken(), cfg, POLICY)
        with pytest.raises(hs.SourceExhausted):
            hs.run_pipeline(uniform_source(small_cfg(batch_size=3, num_iterations=2), 1), cfg, POLICY)
        assert states_equal(hs.run_pipeline(uniform_source(cfg, 21), cfg, POLICY), want)


def test_pipeline_concurrent_threads(cuda):
    # each thread has its own streams and workspace: concurrent runs never share rows
    import threading

    cfgs = [small_cfg(batch_size=b, num_iterations=12, chunk_pixels=4096) for b in (1, 2, 3, 4)]
    want = [hs.run_sequential(uniform_source(c, 30 + k), c, POLICY) for k, c in enumerate(cfgs)]
    got, errors = [None] * len(cfgs), []

    def worker(k):
        try:
            for _ in range(3):
                got[k] = hs.run_pipeline(uniform_source(cfgs[k], 30 + k), cfgs[k], POLICY)
                assert states_equal(got[k], want[k])
        except BaseException as exc:  # reported by the main thread
            errors.append(exc)

    threads = [threading.Thread(target=worker, args=(k,)) for k in range(len(cfgs))]
    for th in threads:
        th.start()
    for th in threads:
        th.join()
    assert not errors, errors
    from paper_1011_0235_b200 import stream as S

    mine = S._pipeline_resources(__import__("torch"), 0)
    assert mine is S._pipeline_resources(__import__("torch"), 0)  # made once per thread


@pytest.mark.parametrize("sizes,pinned_mask", [
    ([3 << 20], [False]),                                  # one run, pieces shared by the pool, one DMA
    ([(1 << 20) + 4, 4, (5 << 20) - 12, 0, 12], [False] * 5),  # ragged runs, an empty chunk
    ([20 << 20, (9 << 20) + 4096 + 8], [False, False]),    # > 16 MiB: 4 MiB pieces, DMA per piece
    ([6 << 20, 6 << 20, 6 << 20], [False, True, False]),   # pinned run between pageable ones
])
def test_pageable_batches_through_copy_pool(cuda, oracle, sizes, pinned_mask):
    """Pageable host chunks of >= 2 MiB per batch are copied into the bounce buffer by the
    host copy pool (pieces DMA'd as they land); counts exact per chunk, through stage()
    and through the synchronous API (naive_histogram / batch_histograms)."""
    torch = cuda
    from paper_1011_0235_b200 import device as D

    rng = np.random.default_rng(sum(sizes))
    chunks, want = [], []
    for k, (n, pin) in enumerate(zip(sizes, pinned_mask)):
        b = oracle.generate("normal", n, 40 + k, mean=float(rng.uniform(20, 230)), sigma=9.0) if n else \
            np.zeros(0, np.uint8)
        if pin:
            p = D.pinned_bytes(n)
            p[:] = b
            b = p
        chunks.append(hs.PackedChunk(b.view(np.uint32)))
        want.append(oracle.histogram(b))
    st = D.Staging()
    stream = torch.cuda.current_stream()
    staged = D.stage(chunks, st, stream)
    out = D.launch(staged, 0, None, stream, staging=st)
    got = out.cpu().numpy().view(np.uint64)
    for k in range(len(chunks)):
        assert np.array_equal(got[k], want[k]), k
    got = hs.batch_histograms(chunks, hs.KernelKind.NAIVE, None, SMALL)
    assert [h.counts.tolist() for h in got] == [w.tolist() for w in want]
    big = max(range(len(chunks)), key=lambda k: sizes[k])
    assert np.array_equal(hs.naive_histogram(chunks[big], SMALL).counts, want[big])


def test_pageable_pipeline_through_copy_pool(cuda, oracle):
    """run_pipeline on pageable 4 MiB chunks, batches of 8 (32 MiB per batch through the
    pool): accumulator exact and equal to run_sequential."""
    px, batch, iters = 4 << 20, 8, 6
    data = oracle.generate("uniform", px * batch * iters, 77)
    words = data.view(np.uint32)
    chunks = [hs.PackedChunk(words[i * (px // 4):(i + 1) * (px // 4)].copy()) for i in range(batch * iters)]
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=px, batch_size=batch, window_size=3)

    def src():
        for i in range(iters):
            yield chunks[i * batch:(i + 1) * batch]

    pipe = hs.run_pipeline(src(), cfg, POLICY)
    assert np.array_equal(pipe[0].running.counts, oracle.histogram(data))
    assert states_equal(pipe, hs.run_sequential(src(), cfg, POLICY))
