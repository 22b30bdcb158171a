"""The device stream engine (run_device_stream, block engine) on C3 and on 1 MiB batch-1
iterations, live (the host issues as the GPU runs) and fed (a
device-side delay first, so every block is queued before the GPU starts: the engine's
own device rate; blocks_ahead=None, since a bounded queue would wait out the delay). Device rates from the commit kernels' device clock."""
import json
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402

for _ in range(2):
    r = X.c3_switch(hs, torch, torch.device("cuda", 0))
    r.pop("kernel_log"); r.pop("degeneracy_log")
    print("C3", json.dumps(r), flush=True)

px, n = 1 << 20, 4096
buf = torch.empty(n * px, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", n * px, 3), buf)
batches = [[hs.DeviceChunk(buf[i * px:(i + 1) * px])] for i in range(n)]
torch.cuda.synchronize()
cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=px, window_size=128)
for bb in (64 << 20, 256 << 20):
    for fed, ahead in ((False, 2), (False, None), (True, None)):
        for rep in range(2):
            torch.cuda.synchronize()
            if fed:
                torch.cuda._sleep(100_000_000)  # ~50 ms: the host queues every block meanwhile
            t0 = time.perf_counter()
            acc, _, rr, _ = hs.run_device_stream(iter(batches), cfg, hs.SwitchPolicy(), block_bytes=bb,
                                                 blocks_ahead=ahead)
            wall = time.perf_counter() - t0
        dev_ns = sum(s.compute_ns for s in rr.stages)
        assert acc.running.total() == n * px
        print(f"1 MiB batch-1 {'fed ' if fed else 'live'} (blocks_ahead {ahead}): block {bb >> 20} MiB ({len(rr.block_sizes)} blocks): "
              f"device {n * px / dev_ns:.0f} GB/s, wall {n * px / wall / 1e9:.0f} GB/s, host issue "
              f"{rr.host_issue_ns / 1e3 / len(rr.block_sizes):.0f} us/block", flush=True)
