"""Does the bench's CPU-baseline leg (numba reference threads, the oracle's C port) slow the
C4 leg that follows it? C4 (bench_extras.c4_mixed) and a copy-only pass over the same
pinned 16 GiB, before and after bench.cpu_reference_run / cpu_port_run, in one process."""
import sys
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench  # noqa: E402
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

GiB = 1 << 30
n = 16 * GiB
pinned = D.pinned_bytes(n)
host = torch.from_numpy(pinned)
dst = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")


def link_pass():
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for off in range(0, n, 256 << 20):
        dst.copy_(host[off:off + (256 << 20)], non_blocking=True)
    b.record()
    b.synchronize()
    return round(n / (a.elapsed_time(b) / 1e3) / 1e9, 2)


def c4(tag):
    t0 = time.perf_counter()
    r = X.c4_mixed(hs, torch, torch.device("cuda", 0), pinned)
    print(f"{tag}: C4 {r['gbs']} GB/s ({time.perf_counter() - t0:.1f} s), copy-only {link_pass()} GB/s", flush=True)


c4("fresh")
c4("fresh again")
print("cpu_reference_run:", (bench.cpu_reference_run(20.0) or {}).get("value"), flush=True)
c4("after reference run")
c4("after reference run, again")
print("cpu_port_run:", bench.cpu_port_run(20.0).get("value"), flush=True)
print("cpu_reference_paths:", list((bench.cpu_reference_paths(6.0) or {}).keys()), flush=True)
c4("after port + paths")
time.sleep(10)
c4("after 10 s idle")
