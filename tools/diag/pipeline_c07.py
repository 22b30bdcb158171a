"""Diagnostic for the reference acceptance criterion c07 (test_acceptance.py:200-212) and
test_stream.py's window-size structure test: per-stage times of run_pipeline under the
Table-3 stage profile, and the compute-stage spread by window size."""
import sys
import time
from pathlib import Path

import numpy as np

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200.datagen import batch_stream  # noqa: E402

P = hs.StageProfile(cpu_pre_us=2028.0, transfer_in_us=1768.0, compute_us=6201.0, transfer_out_us=2.0, cpu_post_us=0.0)


def run(n, seed):
    cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=1024, window_size=8, worker=hs.WorkerGroupConfig(4, 2),
                            stage_profile=P)
    t0 = time.perf_counter()
    _, _, rep, _ = hs.run_pipeline(batch_stream(hs.SourceSpec("uniform", 1024, seed), n), cfg, hs.SwitchPolicy())
    w = time.perf_counter() - t0
    tot = rep.stage_totals_ns()
    return rep.pipelined_ratio, w, {k: round(v / 1e6, 2) for k, v in tot.items()}, rep.total_pipelined_ns / 1e6, \
        [round(s.transfer_in_ns / 1e6, 2) for s in rep.stages[:4]], [round(s.cpu_pre_ns / 1e6, 2) for s in rep.stages[:4]]


for n in (1, 4, 16, 64, 256):
    for rep in range(3):
        r = run(n, 700 + rep)
        print(n, rep, "ratio %.4f wall %.1f ms" % (r[0], r[1] * 1e3), r[2], "pipelined %.1f" % r[3], "tin0..3", r[4],
              "pre0..3", r[5], flush=True)

W = hs.WorkerGroupConfig(8, 2)
for rep in range(2):
    for w in (32, 128, 256):
        cfg = hs.PipelineConfig(num_iterations=110, chunk_pixels=1 << 18, window_size=w, worker=W)
        _, _, r, _ = hs.run_sequential(batch_stream(hs.SourceSpec("uniform", cfg.chunk_pixels, 99), 110, 1), cfg,
                                       hs.SwitchPolicy())
        c = np.array([s.compute_ns for s in r.stages]) / 1e3
        ti = np.array([s.transfer_in_ns for s in r.stages]) / 1e3
        po = np.array([s.cpu_post_ns for s in r.stages]) / 1e3
        print("window", w, "compute us med %.1f p10 %.1f p90 %.1f | tin med %.1f | post med %.1f" % (
            np.median(c), np.percentile(c, 10), np.percentile(c, 90), np.median(ti), np.median(po)), flush=True)
