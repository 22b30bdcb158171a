"""Where does a slow C4 pass lose time? bench_extras.c4_mixed once (generates the 16 GiB
mixed stream in pinned memory), then run_pipeline passes over the same chunks with the
stream timeline on: per pass the rate, the H2D busy fraction, the summed idle time of the
copy stream between copies and the largest gaps (iteration, us)."""
import os
import sys
import time
from pathlib import Path

import numpy as np
import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[2]))
import bench_extras as X  # noqa: E402
import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402

GiB = 1 << 30
pinned = D.pinned_bytes(int(os.environ.get("C4_PIN_GIB", "16")) * GiB)
print("c4_mixed:", X.c4_mixed(hs, torch, torch.device("cuda", 0), pinned)["gbs"], flush=True)
CHUNK, batch, nchunks = X.CHUNK, 16, 1024
words = pinned.view(np.uint32)
cw = CHUNK // 4
chunks = [hs.PackedChunk(words[c * cw:(c + 1) * cw]) for c in range(nchunks)]
iters = nchunks // batch
cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=CHUNK, batch_size=batch, window_size=8)


def src():
    for i in range(iters):
        yield chunks[i * batch:(i + 1) * batch]


import collections  # noqa: E402
import gc  # noqa: E402
import threading  # noqa: E402
import traceback  # noqa: E402

gc_ms = []
_gc_t = [0]


def _gc_cb(phase, info):
    if phase == "start":
        _gc_t[0] = time.perf_counter()
    else:
        gc_ms.append((info["generation"], round((time.perf_counter() - _gc_t[0]) * 1e3, 1)))


gc.callbacks.append(_gc_cb)
from paper_1011_0235_b200 import stream as S  # noqa: E402

stamps = {}


def _stamp(owner, name):
    f = getattr(owner, name)

    def g(*a, **k):
        t = time.perf_counter()
        stamps.setdefault(name + "_first_in", t)
        try:
            return f(*a, **k)
        finally:
            stamps[name + "_last_out"] = time.perf_counter()
    setattr(owner, name, g)


for o, nm in ((S, "_draw"), (S._Counter, "collect"), (S._Fold, "result"), (S, "_timeline_rows")):
    _stamp(o, nm)
from paper_1011_0235_b200 import device as D2  # noqa: E402

setup = collections.defaultdict(float)


def _acc(owner, name, label):
    f = getattr(owner, name)

    def g(*a, **k):
        t = time.perf_counter()
        try:
            return f(*a, **k)
        finally:
            setup[label] += time.perf_counter() - t
    setattr(owner, name, g)


for o, nm in ((D2.Staging, "device_bytes"), (D2.Staging, "host_out"), (D2.Staging, "workspace"),
              (D2.Staging, "__init__"), (S._Fold, "__init__"), (S._Counter, "__init__"), (S._Slot, "__init__"),
              (threading.Thread, "start"), (torch.cuda.Stream, "synchronize")):
    _acc(o, nm, f"{o.__name__}.{nm}")
_new = torch.cuda.Stream.__new__


def _stream_new(cls, *a, **k):
    t = time.perf_counter()
    try:
        return _new(cls, *a, **k)
    finally:
        setup["Stream()"] += time.perf_counter() - t


torch.cuda.Stream.__new__ = _stream_new
main_id = threading.get_ident()


def sampler(stop, samples):
    """The main thread's innermost frames every 5 ms (a poor man's profiler)."""
    while not stop.is_set():
        f = sys._current_frames().get(main_id)
        if f is not None:
            samples.append(" <- ".join(f"{Path(x.filename).name}:{x.lineno}:{x.name}"
                                       for x in traceback.extract_stack(f)[-4:][::-1]))
        time.sleep(0.005)


for rep in range(int(os.environ.get("C4_REPS", "6"))):
    tl = []
    gc_ms.clear()
    stop, samples = threading.Event(), []
    stamps.clear()
    setup.clear()
    th = threading.Thread(target=sampler, args=(stop, samples), daemon=True)
    if os.environ.get("C4_SAMPLE"):
        th.start()
    t0 = time.perf_counter()
    hs.run_pipeline(src(), cfg, hs.SwitchPolicy(), timeline=tl)
    dt = time.perf_counter() - t0
    t1 = time.perf_counter()
    stop.set()
    if th.is_alive():
        th.join()
    phases = {"to_first_draw": stamps["_draw_first_in"] - t0,
              "last_collect_to_result": stamps["result_first_in"] - stamps["collect_last_out"],
              "result": stamps["result_last_out"] - stamps["result_first_in"],
              "timeline_rows": stamps["_timeline_rows_last_out"] - stamps["_timeline_rows_first_in"],
              "after_result": t1 - stamps["result_last_out"]}
    phases = {k: round(v * 1e3, 1) for k, v in phases.items()}
    phases.update({k: round(v * 1e3, 2) for k, v in setup.items() if v > 1e-4})
    h2d = sorted((a, b, it) for it, st, a, b in tl if st == "h2d")
    ker = sorted((a, b, it) for it, st, a, b in tl if st == "kernel")
    span = max(b for _, _, _, b in tl) - min(a for _, _, a, _ in tl)
    gaps = [(round(h2d[k + 1][0] - h2d[k][1], 1), h2d[k + 1][2]) for k in range(len(h2d) - 1)]
    idle = sum(max(0.0, g) for g, _ in gaps)
    busy = sum(b - a for a, b, _ in h2d)
    rates = [round((CHUNK * batch) / ((b - a) * 1e-6) / 1e9, 1) for a, b, _ in h2d]
    print(f"pass {rep}: {nchunks * CHUNK / dt / 1e9:.2f} GB/s wall, span {span / 1e3:.1f} ms, h2d busy {busy / span:.3f}, "
          f"copy idle {idle / 1e3:.2f} ms, top gaps {sorted(gaps, reverse=True)[:5]}, "
          f"per-batch h2d GB/s min/med/max {min(rates)}/{sorted(rates)[len(rates) // 2]}/{max(rates)}, "
          f"first kernel at {ker[0][0] - h2d[0][0]:.0f} us, wall-span {dt * 1e3 - span / 1e3:.1f} ms, gc {gc_ms}, phases ms {phases}", flush=True)
    if dt * 1e3 - span / 1e3 > 20:
        for frame, k in collections.Counter(samples).most_common(6):
            print(f"    {k * 5:5d} ms  {frame}", flush=True)
