"""Per-step host cost of staging one pageable chunk through the bounce buffer (device.stage's
steps replayed one by one, medians over 30 calls)."""
import sys
import time
import warnings
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

page = np.random.default_rng(1).integers(0, 256, 16 << 20, dtype=np.uint8)
st = D.Staging()
stream = torch.cuda.current_stream()
for size in (1 << 20, 16 << 20):
    ch = hs.PackedChunk(page[:size].view(np.uint32))
    steps = {}

    def tick(name, t0):
        t1 = time.perf_counter()
        steps.setdefault(name, []).append(t1 - t0)
        return t1

    for _ in range(30):
        torch.cuda.synchronize()
        t = time.perf_counter()
        dev = st.device_bytes(size)
        t = tick("device_bytes", t)
        bounce = st.host_bounce(size)
        t = tick("host_bounce", t)
        pin = D._pinned.contains(ch.words.ctypes.data, size)
        t = tick("pinned.contains", t)
        D._copy_into(bounce[:size], ch.words.view(np.uint8), D.copy_threads() if size >= 2 << 20 else 1)
        t = tick("copy", t)
        with warnings.catch_warnings():
            warnings.simplefilter("ignore", UserWarning)
            t = tick("catch_warnings", t)
            src = torch.from_numpy(bounce[:size])
            t = tick("from_numpy", t)
            view = dev[0:size]
            t = tick("slice", t)
            view.copy_(src, non_blocking=True)
            t = tick("copy_ (issue)", t)
        ev = torch.cuda.Event()
        ev.record(stream)
        t = tick("event", t)
        staged = D.stage([ch], st, stream)
        t = tick("whole stage()", t)
        torch.cuda.synchronize()
    print(f"{size >> 20} MiB: " + ", ".join(f"{k} {np.median(v) * 1e6:.1f}" for k, v in steps.items()) + " us",
          flush=True)
