"""Are the 19-83 ms transfer_in spikes of run_pipeline (reference criterion c07) Python
gen-2 garbage collections? Records every collection's duration (gc.callbacks) next to
the per-iteration transfer_in of 16-iteration Table-3 runs."""
import gc
import sys
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200.datagen import batch_stream  # noqa: E402

P = hs.StageProfile(cpu_pre_us=2028.0, transfer_in_us=1768.0, compute_us=6201.0, transfer_out_us=2.0, cpu_post_us=0.0)
events = []
t_start = {}


def cb(phase, info):
    if phase == "start":
        t_start[info["generation"]] = time.perf_counter()
    else:
        g = info["generation"]
        events.append((g, (time.perf_counter() - t_start.get(g, time.perf_counter())) * 1e3))


gc.callbacks.append(cb)
mode = sys.argv[1] if len(sys.argv) > 1 else "gc-on"
for n in (16,) * 12 + (64,) * 3:
    events.clear()
    cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=1024, window_size=8, worker=hs.WorkerGroupConfig(4, 2),
                            stage_profile=P)
    _, _, rep, _ = hs.run_pipeline(batch_stream(hs.SourceSpec("uniform", 1024, 7), n), cfg, hs.SwitchPolicy())
    tins = [round(s.transfer_in_ns / 1e6, 1) for s in rep.stages]
    g2 = [round(d, 1) for g, d in events if g == 2]
    print(mode, n, "ratio %.4f" % rep.pipelined_ratio, "max tin %.1f ms" % max(tins), "gen2 ms", g2,
          "n_gc", len(events), flush=True)
