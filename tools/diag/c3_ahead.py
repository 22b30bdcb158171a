"""C3 (bench_extras.c3_switch) through run_device_stream with different host queue bounds
(blocks_ahead): per-segment device rates, register-path iterations and their rate."""
import os
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402

for rep in range(int(os.environ.get("C3_REPS", "2"))):
    for ahead in (1, 2, 3, 4, 6, None):
        r = X.c3_switch(hs, torch, torch.device("cuda", 0), blocks_ahead=ahead)
        hot = sum("HOT" in e for e in r["executed_log"])
        print(f"blocks_ahead {ahead}: by segment {r['device_gbs_by_segment']}, HOT iterations {hot} at "
              f"{r['device_gbs_register_path_iterations']} GB/s, wall {r['wall_gbs']} GB/s, host issue "
              f"{r['host_issue_us_per_block']} us/block", flush=True)
