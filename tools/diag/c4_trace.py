"""C4 (bench_extras.c4_mixed) with every run_pipeline step timed (both threads); prints the
run rate and the steps that took > 3 ms beyond their own synthetic delay."""
import gc
import sys
import threading
import time
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402
from paper_1011_0235_b200 import stream as S  # noqa: E402

log = []


def wrap(owner, name):
    f = getattr(owner, name)

    def g(*a, **k):
        t0 = time.perf_counter_ns()
        try:
            return f(*a, **k)
        finally:
            d = (time.perf_counter_ns() - t0) / 1e6
            if d > 3.0:
                log.append((threading.current_thread().name[:10], name, round(d, 1)))
    setattr(owner, name, g)


for o, n in ((S, "_draw"), (D, "stage"), (S._Slot, "take"), (S._Slot, "acquire"), (S._Counter, "issue"),
             (S._Counter, "wait_kernel"), (S._Counter, "collect"), (S._Fold, "decide"), (S._Fold, "absorb")):
    wrap(o, n)
t_gc = {}
gc.callbacks.append(lambda ph, info: log.append(("gc", info["generation"], 0)) if ph == "start" else None)
pinned = D.pinned_bytes(16 << 30)
for rep in range(4):
    log.clear()
    r = X.c4_mixed(hs, torch, torch.device("cuda", 0), pinned, steps=1)
    print("C4", r["gbs"], "GB/s", "slow steps:", [x for x in log if x[0] != "gc"][:12], flush=True)
