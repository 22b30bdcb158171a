"""Reference criterion c07 exactly as test_acceptance.py:221-230 computes it (median of 3
runs per iteration count), repeated, to see how often and how it fails."""
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200.datagen import batch_stream  # noqa: E402

P = hs.StageProfile(cpu_pre_us=2028.0, transfer_in_us=1768.0, compute_us=6201.0, transfer_out_us=2.0, cpu_post_us=0.0)


def run(n, seed):
    cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=1024, window_size=8, worker=hs.WorkerGroupConfig(4, 2),
                            stage_profile=P)
    _, _, r, _ = hs.run_pipeline(batch_stream(hs.SourceSpec("uniform", cfg.chunk_pixels, seed), n), cfg,
                                 hs.SwitchPolicy())
    return r.pipelined_ratio


fails = 0
for rep in range(int(sys.argv[1])):
    ratios = []
    for n in (1, 4, 16, 64, 256):
        ratios.append(sorted(run(n, 700 + k) for k in range(3))[1])
    ok = all(b <= a for a, b in zip(ratios, ratios[1:])) and 0.95 <= ratios[0] <= 1.0 and 0.60 <= ratios[-1] <= 0.68
    fails += not ok
    print("PASS" if ok else "FAIL", " ".join(f"{r:.4f}" for r in ratios), flush=True)
print("fails", fails)
