"""Where does a 1-64 MiB pageable synchronous call spend its time? The threaded streaming
copy by thread count, then the phases of the bounce path (stage: copies + DMA issue; the
blocking call) against the driver's pageable path (hs_histogram_host)."""
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

page = np.random.default_rng(1).integers(0, 256, 64 << 20, dtype=np.uint8)
dst = D.pinned_bytes(64 << 20)
for size in (1 << 20, 2 << 20, 4 << 20, 16 << 20):
    row = []
    for th in (1, 2, 4, 8):
        ts = []
        for _ in range(20):
            t0 = time.perf_counter()
            D._copy_into(dst[:size], page[:size], th)
            ts.append(time.perf_counter() - t0)
        row.append(f"{th} thr {np.median(ts) * 1e6:.0f} us")
    print(f"streaming copy {size >> 20} MiB: " + ", ".join(row), flush=True)

st = D.default_staging()
stream = torch.cuda.current_stream()
for size in (1 << 20, 2 << 20, 4 << 20, 16 << 20, 64 << 20):
    ch = hs.PackedChunk(page[:size].view(np.uint32))
    res = {}
    for name in ("bounce", "driver"):
        ph = {"stage": [], "sync": [], "total": []}
        for r in range(12):
            t0 = time.perf_counter()
            if name == "bounce":
                staged = D.stage([ch], st, stream)
                t1 = time.perf_counter()
                D._sync_histograms(staged, 0, None, 0, st, stream)
            else:
                t1 = t0
                D._host_histograms([ch], 0, None, 0, st, stream)
            t2 = time.perf_counter()
            if r >= 2:
                ph["stage"].append(t1 - t0)
                ph["sync"].append(t2 - t1)
                ph["total"].append(t2 - t0)
        res[name] = {k: round(float(np.median(v)) * 1e6) for k, v in ph.items()}
    print(f"{size >> 20} MiB: bounce {res['bounce']} us, driver {res['driver']} us", flush=True)
