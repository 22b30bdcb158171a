"""BASELINE configs[3] alone (bench_extras.c4_mixed): 16 GiB mixed stream from pinned host
memory through run_pipeline; prints GB/s and the kernel log summary."""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

pinned = D.pinned_bytes(16 << 30)
for rep in range(int(__import__("os").environ.get("REPS", "2"))):
    r = X.c4_mixed(hs, torch, torch.device("cuda", 0), pinned)
    print("C4", r["gbs"], "GB/s", r["kernel_switches"], "switches", r["adaptive_iterations"], "adaptive", flush=True)
