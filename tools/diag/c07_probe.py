"""Reference criterion c07 (pipelined/sequential ratio must not rise with the iteration
count): distribution of the Table-3 profile's ratio at 4 and 16 iterations, and which
stage carries the outliers."""
import sys
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200.datagen import batch_stream  # noqa: E402

P = hs.StageProfile(cpu_pre_us=2028.0, transfer_in_us=1768.0, compute_us=6201.0, transfer_out_us=2.0, cpu_post_us=0.0)
for n in (4, 16):
    rows = []
    for rep in range(int(sys.argv[1]) if len(sys.argv) > 1 else 20):
        cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=1024, window_size=8,
                                worker=hs.WorkerGroupConfig(4, 2), stage_profile=P)
        _, _, r, _ = hs.run_pipeline(batch_stream(hs.SourceSpec("uniform", 1024, 700 + rep), n), cfg,
                                     hs.SwitchPolicy())
        tot = r.stage_totals_ns()
        rows.append((r.pipelined_ratio, r.total_pipelined_ns / 1e6, {k: round(v / 1e6 / n, 2) for k, v in tot.items()}))
    ratios = np.array([x[0] for x in rows])
    print(f"n={n} ratio median {np.median(ratios):.4f} min {ratios.min():.4f} max {ratios.max():.4f}", flush=True)
    for x in rows:
        if abs(x[0] - np.median(ratios)) > 0.03:
            print("   outlier", round(x[0], 4), "wall ms", round(x[1], 1), "per-iter stage ms", x[2], flush=True)
