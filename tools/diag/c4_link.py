"""Is C4's spread (45-55 GB/s between runs) the pipeline or the host link? Per repetition:
bench_extras.c4_mixed (regenerates the 16 GiB pinned region, one warm-up run_pipeline
pass, then C4_STEPS timed passes), followed by copy-only passes over the same 16 GiB
(256 MiB H2D copies back to back on one stream, CUDA events). Prints both rates."""
import os
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

GiB = 1 << 30
n = 16 * GiB
pinned = D.pinned_bytes(n)
host = torch.from_numpy(pinned)
dst = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()


def link_pass():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with torch.cuda.stream(s):
        a.record()
        for off in range(0, n, 256 << 20):
            dst.copy_(host[off:off + (256 << 20)], non_blocking=True)
        b.record()
    b.synchronize()
    return n / (a.elapsed_time(b) / 1e3) / 1e9


steps = int(os.environ.get("C4_STEPS", "2"))
for rep in range(int(os.environ.get("C4_REPS", "5"))):
    t0 = time.perf_counter()
    r = X.c4_mixed(hs, torch, torch.device("cuda", 0), pinned, steps=steps)
    el = time.perf_counter() - t0
    links = [round(link_pass(), 2) for _ in range(2)]
    print(f"rep {rep}: C4 {r['gbs']} GB/s (call {el:.1f} s), copy-only passes {links} GB/s", flush=True)
