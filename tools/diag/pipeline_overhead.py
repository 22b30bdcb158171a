"""Per-iteration host overhead of run_pipeline's consumer and feeder with no synthetic
delays (1 KiB chunks, batch 1): the stage totals per iteration, median of 5 runs."""
import statistics
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200.datagen import batch_stream  # noqa: E402

n = 256
rows = []
for rep in range(6):
    cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=1024, window_size=8, worker=hs.WorkerGroupConfig(4, 2))
    _, _, r, _ = hs.run_pipeline(batch_stream(hs.SourceSpec("uniform", 1024, 7 + rep), n), cfg, hs.SwitchPolicy())
    if rep:
        rows.append({k: v / n / 1e3 for k, v in r.stage_totals_ns().items()} | {"wall": r.total_pipelined_ns / n / 1e3})
for k in rows[0]:
    vals = [x[k] for x in rows]
    print(f"{k:16s} median {statistics.median(vals):8.1f} us  min {min(vals):8.1f}  max {max(vals):8.1f}")
