"""Extra legs of bench.py (rank 0, N=1 layout): the other BASELINE configs, reported
beside the C5 headline.

  C1  configs[0]: one 1024x1024 uniform image -- latency through the public API
      (pageable, pinned, device), 256 images per call, graph-replayed single launches
  C2  configs[1]: X-ray-like normal streams (mean 128, sigma 8/32/64), 1 GiB each in
      16 MiB chunks, AHist (ADAPTIVE) with the lag-1 CPU-computed binning pattern
  C3  configs[2]: uniform -> bimodal 40/200 -> constant 127 through the device-resident
      stream engine (window, accumulator, lag-1 NVHist/AHist switch on the GPU)
  C4  configs[3]: a 16 GiB host-streamed mixed stream through run_pipeline
Each leg checks its counts against the oracle (or a closed form) before reporting.
"""
from __future__ import annotations

import time

import numpy as np

GiB = 1 << 30
CHUNK = 16 << 20
BASE_SEED = 0x1011_0235
MEAN = 128.0
SIGMAS = (8.0, 32.0, 64.0)


def host_cores() -> int:
    import os

    return len(os.sched_getaffinity(0))


C1_IMAGES = 256


def c1_image(hs, N, torch, dev):
    """BASELINE configs[0]: one 1024x1024 uniform image (seed 0). L2-resident and
    launch-bound, so reported beside the headline: latency through the public API
    (pageable, pinned and device-resident chunk),
    256 images per call (one launch of 256 segments), and single-image launches
    replayed from a CUDA graph."""
    from oracle import oracle as O
    from paper_1011_0235_b200 import device as D

    L = N.lib()

    n = 1 << 20
    spec = hs.SourceSpec("uniform", n, 0)
    chunk = hs.generate(spec)
    want = O.histogram(chunk.pixels())
    cfg = hs.WorkerGroupConfig()
    for _ in range(5):
        h = hs.naive_histogram(chunk, cfg)
    assert np.array_equal(h.counts, want)
    def per_call_us(c, reps=200):
        for _ in range(5):
            hs.naive_histogram(c, cfg)
        t0 = time.perf_counter()
        for _ in range(reps):
            hs.naive_histogram(c, cfg)
        return (time.perf_counter() - t0) / reps * 1e6

    api_us = per_call_us(chunk)  # pageable numpy words, as the reference's callers hold them
    pin = D.pinned_words(chunk.words.size)
    pin[:] = chunk.words
    pinned_us = per_call_us(hs.PackedChunk(pin))
    dev_chunk = hs.DeviceChunk(torch.from_numpy(chunk.pixels().copy()).to(dev))
    device_us = per_call_us(dev_chunk)
    assert np.array_equal(hs.naive_histogram(dev_chunk, cfg).counts, want)
    # C1_IMAGES images, one call
    imgs = torch.empty(C1_IMAGES * n, dtype=torch.uint8, device=dev)
    for i in range(C1_IMAGES):
        hs.generate_device(hs.SourceSpec("uniform", n, i), imgs[i * n:(i + 1) * n])
    b0 = (np.arange(C1_IMAGES, dtype=np.uint64) * n)
    b1 = b0 + n
    out = torch.empty((C1_IMAGES, 256), dtype=torch.int64, device=dev)
    ws = torch.zeros(int(L.hs_workspace_bytes(C1_IMAGES)), dtype=torch.uint8, device=dev)
    s = torch.cuda.current_stream()

    def batched():
        N.check(L.hs_histogram_batched(imgs.data_ptr(), N.u64p(b0), N.u64p(b1), C1_IMAGES,
                                       N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, 0, None,
                                       None, 0, 0, out.data_ptr(), ws.data_ptr(), ws.numel(), s.cuda_stream), "batched")

    for _ in range(3):
        batched()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda._sleep(20_000_000)
    a.record()
    for _ in range(20):
        batched()
    b.record()
    b.synchronize()
    batch_us = a.elapsed_time(b) / 20 * 1e3
    assert np.array_equal(out[C1_IMAGES - 1].cpu().numpy().view(np.uint64),
                          O.histogram(imgs[(C1_IMAGES - 1) * n:].cpu().numpy()))
    # single-image launches captured in a CUDA graph
    one0, one1 = np.zeros(1, np.uint64), np.full(1, n, np.uint64)
    out1 = torch.empty((1, 256), dtype=torch.int64, device=dev)
    g = torch.cuda.CUDAGraph()
    cs = torch.cuda.Stream()
    cs.wait_stream(s)
    with torch.cuda.stream(cs):
        N.check(L.hs_histogram_batched(imgs.data_ptr(), N.u64p(one0), N.u64p(one1), 1, N.HS_KIND_NAIVE, 0, None, None,
                                       0, 0, out1.data_ptr(), ws.data_ptr(), ws.numel(), cs.cuda_stream), "warm")
    s.wait_stream(cs)
    with torch.cuda.graph(g):
        gs = torch.cuda.current_stream()
        for _ in range(100):
            N.check(L.hs_histogram_batched(imgs.data_ptr(), N.u64p(one0), N.u64p(one1), 1,
                                           N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, 0, None,
                                           None, 0, 0, out1.data_ptr(), ws.data_ptr(), ws.numel(), gs.cuda_stream),
                    "capture")
    g.replay()
    torch.cuda.synchronize()
    a.record()
    g.replay()
    b.record()
    b.synchronize()
    graph_us = a.elapsed_time(b) / 100 * 1e3
    assert np.array_equal(out1[0].cpu().numpy().view(np.uint64), O.histogram(imgs[:n].cpu().numpy()))
    t0 = time.perf_counter()
    for _ in range(5):
        O.naive_histogram(chunk.words, 32, host_cores())
    cpu_us = (time.perf_counter() - t0) / 5 * 1e6
    return {"bytes": n, "public_api_us_per_image": round(api_us, 2),
            "public_api_pinned_us": round(pinned_us, 2), "public_api_device_chunk_us": round(device_us, 2),
            "batched_images": C1_IMAGES, "batched_us_per_image": round(batch_us / C1_IMAGES, 3),
            "batched_gbs": round(C1_IMAGES * n / (batch_us * 1e3), 1),
            "graph_single_image_us": round(graph_us, 3), "cpu_reference_port_us": round(cpu_us, 1)}


def c3_switch(hs, torch, dev, **engine_kw):
    """BASELINE configs[2]: a stream that turns degenerate -- 1 GiB uniform, then 1 GiB of
    a bimodal peak (50/50 of bytes 40 and 200; not a reference generator: uniform bytes
    < 128 map to 40, the rest to 200), then 2 GiB constant 127 -- in 16 MiB chunks,
    iterations of 16 chunks (256 MiB), through the device-resident engine
    (run_device_stream: window, accumulator and the lag-1 NVHist/AHist switch on the
    GPU, one block of iterations per histogram call). Once the device has decided
    ADAPTIVE on the constant window, the engine runs the register path for bin 127.
    Per-segment device rates from the commit kernels' device clock; the accumulator is
    checked bin for bin (closed form for the bimodal/constant parts, oracle for the
    uniform part)."""
    from oracle import oracle as O

    px, per_iter = CHUNK, 16
    plan = (("uniform", 4), ("bimodal", 4), ("constant", 8))  # iterations per segment
    iters = sum(n for _, n in plan)
    total = iters * per_iter
    buf = torch.empty(total * px, dtype=torch.uint8, device=dev)
    k = 0
    seg_of = []
    for kind, n in plan:
        for _ in range(n * per_iter):
            sl = buf[k * px:(k + 1) * px]
            if kind == "constant":
                hs.generate_device(hs.SourceSpec("constant", px, k, value=127), sl)
            else:
                hs.generate_device(hs.SourceSpec("uniform", px, (BASE_SEED ^ 0xC3) ^ k), sl)
                if kind == "bimodal":
                    sl.copy_((sl >= 128).to(torch.uint8) * 160 + 40)
            k += 1
        seg_of += [kind] * n
    torch.cuda.synchronize()
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=px, batch_size=per_iter, window_size=per_iter)
    batches = [[hs.DeviceChunk(buf[(i * per_iter + j) * px:(i * per_iter + j + 1) * px]) for j in range(per_iter)]
               for i in range(iters)]  # views built once, outside the timed call

    hs.run_device_stream(iter(batches), cfg, hs.SwitchPolicy(), **engine_kw)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    acc, _, rep, log = hs.run_device_stream(iter(batches), cfg, hs.SwitchPolicy(), **engine_kw)
    wall = time.perf_counter() - t0
    uni = O.histogram_mt(buf[:4 * per_iter * px].cpu().numpy())
    bim = buf[4 * per_iter * px:8 * per_iter * px]
    n40 = int((bim == 40).sum().item())
    want = uni.copy()
    want[40] += n40
    want[200] += 4 * per_iter * px - n40
    want[127] += 8 * per_iter * px
    assert np.array_equal(acc.running.counts, want), "C3 accumulator"
    it_bytes = per_iter * px
    rates = {}
    for kind, _ in plan:  # iteration 0 also holds the host's first staging: excluded
        idx = [i for i in range(1, iters) if seg_of[i] == kind]
        ns = sum(rep.stages[i].compute_ns for i in idx)
        rates[kind] = round(len(idx) * it_bytes / ns, 1) if ns else None
    hot = [i for i, e in enumerate(rep.executed_log) if "HOT" in e]
    hot_ns = sum(rep.stages[i].compute_ns for i in hot)
    del buf
    torch.cuda.empty_cache()
    return {"bytes": total * px, "chunks": total, "iterations": iters, "iteration_bytes": it_bytes,
            "device_gbs_by_segment": rates,
            "device_gbs_register_path_iterations": round(len(hot) * it_bytes / hot_ns, 1) if hot_ns else None,
            "device_gbs_method": "commit kernels' device clock (block time split over its iterations), iterations 1..n-1",
            "wall_gbs": round(total * px / wall / 1e9, 1), "blocks": rep.block_sizes,
            "host_issue_us_per_block": round(rep.host_issue_ns / 1e3 / len(rep.block_sizes), 1),
            "kernel_log": [k.value for k in log], "executed_log": rep.executed_log,
            "degeneracy_log": [round(d, 4) for d in rep.degeneracy_log],
            "parity": "accumulator == oracle (uniform part) + closed forms (bimodal, constant), bin for bin"}


def c2_normal_streams(hs, N, torch, dev, steps: int = 20):
    """BASELINE configs[1]: three X-ray-like normal streams (mean 128, sigma 8/32/64),
    1 GiB each as 64 chunks of 16 MiB (chunk seed = base ^ index, datagen.py:196-198),
    counted per chunk by ADAPTIVE with the binning pattern the host computes from that
    stream's previous step (lag 1, latency-hidden behind the other streams' kernels).
    One step = 3 GiB in three batched calls on three CUDA streams. The label names the
    kernel that runs: the normal priors have max-bin share < 0.999, so the ADAPTIVE
    launch carries the spread hint and the plain lane core runs."""
    from oracle import oracle as O
    from paper_1011_0235_b200 import device as D

    L = N.lib()
    streams = []
    for sigma in SIGMAS:
        buf = torch.empty(GiB, dtype=torch.uint8, device=dev)
        for c in range(64):
            spec = hs.SourceSpec("normal", CHUNK, (BASE_SEED + int(sigma)) ^ c, mean=MEAN, sigma=sigma)
            hs.generate_device(spec, buf[c * CHUNK:(c + 1) * CHUNK])
        streams.append(buf)
    begin = np.arange(64, dtype=np.uint64) * CHUNK
    end = begin + CHUNK
    side = [torch.cuda.Stream(device=dev) for _ in SIGMAS]
    wss = [torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device=dev) for _ in SIGMAS]
    outs = [[torch.empty((64, 256), dtype=torch.int64, device=dev) for _ in range(2)] for _ in SIGMAS]
    host = [[torch.empty((64, 256), dtype=torch.int64, pin_memory=True) for _ in range(2)] for _ in SIGMAS]
    evs = [[torch.cuda.Event() for _ in range(2)] for _ in SIGMAS]
    patterns = [hs.uniform_pattern(960) for _ in SIGMAS]
    pending = {}
    kinds = set()
    b_p, e_p = N.u64p(begin), N.u64p(end)
    torch.cuda.synchronize()  # inputs generated and workspaces zeroed (current stream) before the side streams

    def launch(j, k):
        if j in pending:
            ev, kk = pending.pop(j)
            ev.synchronize()
            prior = host[j][kk].numpy().view(np.uint64).sum(axis=0, dtype=np.uint64)
            patterns[j] = hs.compute_binning_pattern(hs.Histogram256(prior))
        p = patterns[j]
        kind = D._with_hints(N.HS_KIND_ADAPTIVE, p) | N.HS_KIND_FLAG_CHAINED
        kinds.add(D.kernel_form(kind, p))
        N.check(L.hs_histogram_batched(streams[j].data_ptr(), b_p, e_p, 64, kind, N.HS_IMPL_AUTO, N.i64p(p.offset),
                                       N.i64p(p.count), 960, 8, outs[j][k].data_ptr(), wss[j].data_ptr(),
                                       wss[j].numel(), side[j].cuda_stream), "c2")
        with torch.cuda.stream(side[j]):
            host[j][k].copy_(outs[j][k], non_blocking=True)
        evs[j][k].record(side[j])
        pending[j] = (evs[j][k], k)

    for w in range(3):
        for j in range(3):
            launch(j, w & 1)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    cur = torch.cuda.current_stream()
    a.record(cur)
    for s in side:
        s.wait_stream(cur)
    for st in range(steps):
        for j in range(3):
            launch(j, st & 1)
    for s in side:
        cur.wait_stream(s)
    b.record(cur)
    b.synchronize()
    ms = a.elapsed_time(b)
    k = (steps - 1) & 1
    for j in range(3):  # parity: every chunk's total, three chunks per stream bin for bin
        got = outs[j][k].cpu().numpy().view(np.uint64)
        assert (got.sum(axis=1) == CHUNK).all()
        for c in (0, 37, 63):
            assert np.array_equal(got[c], O.histogram(streams[j][c * CHUNK:(c + 1) * CHUNK].cpu().numpy())), (j, c)
    del streams
    torch.cuda.empty_cache()
    return {"bytes_per_step": 3 * GiB, "steps": steps, "ms_per_step": round(ms / steps, 4),
            "gbs": round(3 * GiB * steps / (ms / 1e3) / 1e9, 1), "kind": "ADAPTIVE + lag-1 CPU pattern per stream",
            "kernel_ran": sorted(kinds), "streams": "one CUDA stream per sigma stream",
            "parity": "chunk totals + 3 chunks per stream bin for bin vs the oracle"}


C4_SEGMENTS = (("uniform", {}), ("normal", {"mean": MEAN, "sigma": 32.0}), ("constant", {"value": 127}),
               ("normal", {"mean": MEAN, "sigma": 8.0}))


def c4_mixed(hs, torch, dev, pinned, steps: int = 2):
    """BASELINE configs[3]: a 16 GiB mixed-distribution stream (uniform -> normal sigma 32
    -> constant 127 -> normal sigma 8; 16 MiB chunks, seeds base ^ index) in pinned host
    memory (the first 16 GiB of the e2e leg's buffer, regenerated), through run_pipeline
    with the reference switch policy (threshold 0.45, window 8), batches of 16 chunks.
    The accumulator is checked bin for bin against the oracle's multithreaded count of
    the same pinned bytes."""
    from oracle import oracle as O

    nchunks = 1024
    if pinned.size < nchunks * CHUNK:
        nchunks = pinned.size // CHUNK // 64 * 64
    per_seg = nchunks // len(C4_SEGMENTS)
    stage = torch.empty(CHUNK, dtype=torch.uint8, device=dev)
    for i in range(nchunks):
        kind, kw = C4_SEGMENTS[i // per_seg]
        hs.generate_device(hs.SourceSpec(kind, CHUNK, (BASE_SEED ^ 0xC4) ^ i, **kw), stage)
        torch.from_numpy(pinned[i * CHUNK:(i + 1) * CHUNK]).copy_(stage)
    words = pinned.view(np.uint32)
    cw = CHUNK // 4
    chunks = [hs.PackedChunk(words[c * cw:(c + 1) * cw]) for c in range(nchunks)]
    batch = 16
    iters = nchunks // batch
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=CHUNK, batch_size=batch, window_size=8)

    def src():
        for i in range(iters):
            yield chunks[i * batch:(i + 1) * batch]

    hs.run_pipeline(src(), cfg, hs.SwitchPolicy())
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        acc, _, rep, log = hs.run_pipeline(src(), cfg, hs.SwitchPolicy())
        times.append(time.perf_counter() - t0)
    want = O.histogram_mt(pinned[:nchunks * CHUNK])
    assert np.array_equal(acc.running.counts, want), "C4 accumulator != oracle"
    kinds = [k.value for k in log]
    dt = float(np.median(times))
    return {"bytes": nchunks * CHUNK, "gbs": round(nchunks * CHUNK / dt / 1e9, 3),
            "api": "run_pipeline (pinned host chunks, 16 MiB, batch 16)",
            "kernel_switches": sum(1 for a, b in zip(kinds, kinds[1:]) if a != b),
            "adaptive_iterations": kinds.count("adaptive"), "iterations": len(kinds),
            "parity": "accumulator == oracle multithreaded count of the 16 GiB, bin for bin"}


def host_small_chunks(hs, torch, dev, pinned, n: int = 2048):
    """The reference's default pipeline shape (1 MiB chunks, batch 1, window 128) streamed
    from pinned host memory (the first 2 GiB of the e2e leg's buffer): run_pipeline (the
    reference's per-iteration host fold) vs run_device_stream (the same fold on the device,
    host chunks staged a block at a time on a copy stream). Both results must agree."""
    px = 1 << 20
    n = min(n, pinned.size // px)
    words = pinned.view(np.uint32)
    chunks = [hs.PackedChunk(words[i * (px // 4):(i + 1) * (px // 4)]) for i in range(n)]
    cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=px, window_size=128)

    def src():
        for c in chunks:
            yield [c]

    out, res = {}, {}
    for name, fn in (("run_pipeline", hs.run_pipeline), ("run_device_stream", hs.run_device_stream)):
        fn(src(), cfg, hs.SwitchPolicy())  # warm-up pass
        t0 = time.perf_counter()
        res[name] = fn(src(), cfg, hs.SwitchPolicy())
        out[name + "_gbs"] = round(n * px / (time.perf_counter() - t0) / 1e9, 3)
    a, b = res["run_pipeline"], res["run_device_stream"]
    assert a[0] == b[0] and a[1] == b[1] and a[3] == b[3], "device engine != host engine"
    out.update({"bytes": n * px, "iterations": n, "chunk": "1 MiB pinned, batch 1, window 128",
                "parity": "accumulator, window and kernel log equal between the two engines"})
    return out
