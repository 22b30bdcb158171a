"""Bench-step structure A/B: 3 x 1 GiB (64 x 16 MiB) ADAPTIVE launches per step with a
lag-1 host pattern per sigma stream, under different stream arrangements:
  three  -- one CUDA stream per sigma, D2H readback on the same stream (bench.py r1)
  one    -- one compute stream (PDL chains all launches), readback on a copy stream
            that waits on a per-launch event; outputs double-buffered
  bare   -- one compute stream, no readback, fixed patterns (upper bound)
GPU time per step = CUDA events around 100 steps."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

L = N.lib()
GiB, CHUNK = 1 << 30, 16 << 20
SIG = (8.0, 32.0, 64.0)
streams = []
for sg in SIG:
    b = torch.empty(GiB, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("normal", GiB, 7 + int(sg), mean=128.0, sigma=sg), b)
    streams.append(b)
begin = np.arange(64, dtype=np.uint64) * CHUNK
end = begin + CHUNK
outs = [[torch.empty((64, 256), dtype=torch.int64, device="cuda") for _ in range(2)] for _ in SIG]
host = [[torch.empty((64, 256), dtype=torch.int64, pin_memory=True) for _ in range(2)] for _ in SIG]
wss = [torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda") for _ in SIG]
main = torch.cuda.current_stream()


def run(mode, steps=100, warm=5):
    side = [torch.cuda.Stream() for _ in SIG] if mode == "three" else [main] * 3
    copy = torch.cuda.Stream()
    pats = [hs.uniform_pattern(960) for _ in SIG]
    pending = {}
    flip = [0, 0, 0]

    def launch(j):
        if mode != "bare" and j in pending:
            ev, hb = pending.pop(j)
            ev.synchronize()
            pats[j] = hs.compute_binning_pattern(hs.Histogram256(hb.numpy().view(np.uint64).sum(axis=0, dtype=np.uint64)))
        p = pats[j]
        o = outs[j][flip[j]]
        N.check(L.hs_histogram_batched(streams[j].data_ptr(), N.u64p(begin), N.u64p(end), 64, N.HS_KIND_ADAPTIVE,
                                       N.HS_IMPL_AUTO, N.i64p(p.offset), N.i64p(p.count), 960, 8, o.data_ptr(),
                                       wss[j if mode == "three" else 0].data_ptr(), wss[0].numel(),
                                       side[j].cuda_stream), "h")
        if mode == "bare":
            return
        hb = host[j][flip[j]]
        if mode == "three":
            with torch.cuda.stream(side[j]):
                hb.copy_(o, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(side[j])
        else:
            k = torch.cuda.Event()
            k.record(main)
            copy.wait_event(k)
            with torch.cuda.stream(copy):
                hb.copy_(o, non_blocking=True)
            ev = torch.cuda.Event()
            ev.record(copy)
        pending[j] = (ev, hb)
        flip[j] ^= 1

    for _ in range(warm):
        for j in range(3):
            launch(j)
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(main)
    for s in side:
        s.wait_stream(main)
    for _ in range(steps):
        for j in range(3):
            launch(j)
    for s in side:
        main.wait_stream(s)
    b.record(main)
    b.synchronize()
    ms = a.elapsed_time(b) / steps
    return ms, 3 * GiB / ms / 1e6


if __name__ == "__main__" and len(sys.argv) > 1:  # ab_step.py MODE STEPS [sampler]: one measurement in a fresh process
    import threading
    import time

    stop = threading.Event()
    if len(sys.argv) > 3:
        import pynvml

        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(0)
        clk = []

        def poll():
            while not stop.is_set():
                clk.append(pynvml.nvmlDeviceGetClockInfo(h, 1))
                pynvml.nvmlDeviceGetPowerUsage(h)
                time.sleep(0.005)

        threading.Thread(target=poll, daemon=True).start()
    ms, gbs = run(sys.argv[1], steps=int(sys.argv[2]))
    stop.set()
    print(f"{sys.argv[1]:6s} steps={sys.argv[2]} sampler={len(sys.argv) > 3} {ms:.4f} ms/step  {gbs:7.1f} GB/s", flush=True)
    sys.exit(0)
for r in range(2 if __name__ == "__main__" else 0):
    for mode in ("three", "one", "bare"):
        ms, gbs = run(mode)
        print(f"round {r} {mode:6s} {ms:.4f} ms/step  {gbs:7.1f} GB/s", flush=True)
