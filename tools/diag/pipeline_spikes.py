"""Where do run_pipeline's 20-110 ms transfer_in spikes come from (reference c07)?
Wraps the producer's and consumer's steps with timers (thread, step, start, duration)
and prints every step slower than 5 ms of 16-iteration Table-3 runs."""
import sys
import threading
import time
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import stream as S  # noqa: E402
from paper_1011_0235_b200.datagen import batch_stream  # noqa: E402

P = hs.StageProfile(cpu_pre_us=2028.0, transfer_in_us=1768.0, compute_us=6201.0, transfer_out_us=2.0, cpu_post_us=0.0)
log = []
T0 = [0.0]


def wrap(mod, name, expect_us=None):
    f = getattr(mod, name)

    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            d = (time.perf_counter() - t) * 1e3
            extra = d - (a[0] / 1e3 if expect_us and a and isinstance(a[0], (int, float)) else 0)  # _nap(us)
            log.append((threading.current_thread().name, name, round((t - T0[0]) * 1e3, 2), round(d, 2),
                        round(extra, 2)))
    setattr(mod, name, g)


wrap(S.D, "stage")
wrap(S._Counter, "wait_kernel")
wrap(S._Counter, "collect")
wrap(S, "_nap", expect_us=True)


class Src:
    def __init__(self, it):
        self.it = it

    def __iter__(self):
        return self

    def __next__(self):
        t = time.perf_counter()
        try:
            return next(self.it)
        finally:
            log.append((threading.current_thread().name, "next", round((t - T0[0]) * 1e3, 2),
                        round((time.perf_counter() - t) * 1e3, 2), 0))


for rep in range(12):
    log.clear()
    T0[0] = time.perf_counter()
    n = 16
    cfg = hs.PipelineConfig(num_iterations=n, chunk_pixels=1024, window_size=8, worker=hs.WorkerGroupConfig(4, 2),
                            stage_profile=P)
    _, _, r, _ = hs.run_pipeline(Src(batch_stream(hs.SourceSpec("uniform", 1024, 7), n)), cfg, hs.SwitchPolicy())
    tins = [round(s.transfer_in_ns / 1e6, 1) for s in r.stages]
    print(rep, "ratio %.4f" % r.pipelined_ratio, "tin", tins, flush=True)
    for row in log:
        if row[4] > 3.0 or (row[1] != "_nap" and row[3] > 3.0):
            print("   slow:", row, flush=True)
