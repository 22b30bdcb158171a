"""Randomized parity of the stream engines against the host engine (run_sequential, itself
pinned to the reference's run_sequential by tests/test_gpu_stream.py): random segment
schedules (uniform / normal / constant / mixture / sequential), chunk sizes, batch sizes,
windows, recompute periods and switch thresholds; run_device_stream with random block
sizes, host queue bounds (blocks_ahead), register path on/off and device, pinned or
pageable chunks (mixed within a batch), and run_pipeline on the host chunks. Every run
must equal run_sequential: accumulator, window ring, kernel log, per-slice histograms,
degeneracy and divergence logs. Runs for SECONDS.
usage: python tools/fuzz_engine.py [SECONDS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import device as D  # noqa: E402
from paper_1011_0235_b200.datagen import schedule_stream  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 120.0
seed = int(os.environ.get("FUZZ_SEED", int(time.time())))
rng = np.random.default_rng(seed)
print(f"seed {seed}", flush=True)


def random_spec(px: int, k: int) -> hs.SourceSpec:
    kind = rng.choice(["uniform", "normal", "constant", "mixture", "sequential"])
    if kind == "normal":
        return hs.SourceSpec("normal", px, k, mean=float(rng.uniform(0, 255)), sigma=float(rng.choice([1, 4, 32])))
    if kind == "constant":
        return hs.SourceSpec("constant", px, k, value=int(rng.integers(0, 256)))
    if kind == "mixture":
        return hs.SourceSpec("mixture", px, k, value=int(rng.integers(0, 256)), degeneracy=float(rng.uniform(0.3, 1)))
    return hs.SourceSpec(str(kind), px, k)


def same(a, b) -> str | None:
    if a[0] != b[0]:
        return "accumulator"
    if a[1].windowed != b[1].windowed or [h.counts.tolist() for h in a[1].ring] != [h.counts.tolist() for h in b[1].ring]:
        return "window"
    if [k.value for k in a[3]] != [k.value for k in b[3]]:
        return "kernel log"
    if a[2].per_slice_histograms != b[2].per_slice_histograms:
        return "per-slice"
    if a[2].degeneracy_log != b[2].degeneracy_log or a[2].divergence_log != b[2].divergence_log:
        return "deg/div logs"
    return None


def place(batches, how: str):
    out = []
    for b in batches:
        row = []
        for c in b:
            mode = how if how != "mixed" else rng.choice(["device", "pinned", "pageable"])
            if mode == "device":
                row.append(hs.DeviceChunk(torch.from_numpy(c.pixels().copy()).cuda()))
            elif mode == "pinned":
                w = D.pinned_words(c.words.size)
                w[:] = c.words
                row.append(hs.PackedChunk(w))
            else:
                row.append(c)
        out.append(row)
    torch.cuda.synchronize()
    return out


trials = fails = 0
t_end = time.time() + secs
while time.time() < t_end:
    px = int(4 * rng.choice([1, 16, 1000, 4096, 65536, 262144]))
    batch = int(rng.choice([1, 1, 2, 5, 16]))
    n_seg = int(rng.integers(1, 4))
    segs = [(random_spec(px, int(rng.integers(0, 1 << 30))), int(rng.integers(1, 40))) for _ in range(n_seg)]
    iters = sum(n for _, n in segs)
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=px, batch_size=batch,
                            window_size=int(rng.choice([1, 2, 3, 8, 33])),
                            recompute_pattern_every=int(rng.choice([1, 1, 2, 5])))
    policy = hs.SwitchPolicy(float(rng.choice([0.45, 0.2, 0.9])))
    want = hs.run_sequential(schedule_stream(segs, batch), cfg, policy)
    batches = list(schedule_stream(segs, batch))
    how = str(rng.choice(["device", "pinned", "pageable", "mixed"]))
    placed = place(batches, how)
    kw = dict(block_bytes=int(rng.choice([4, 4096, 1 << 20, 16 << 20, 256 << 20])),
              blocks_ahead=[1, 2, 4, None][int(rng.integers(0, 4))], register_path=bool(rng.random() < 0.8))
    got = hs.run_device_stream(iter(placed), cfg, policy, **kw)
    bad = same(want, got)
    tag = f"device_stream {how} {kw}"
    if bad is None and how != "device":
        got = hs.run_pipeline(iter(placed), cfg, policy)
        bad = same(want, got)
        tag = f"run_pipeline {how}"
    trials += 1
    if bad is not None:
        fails += 1
        print(f"MISMATCH ({bad}) in {tag}: px {px} batch {batch} cfg {cfg} threshold {policy.threshold} segs {segs}",
              flush=True)
    if trials % 25 == 0:
        print(f"{trials} trials, {fails} mismatches", flush=True)
print(f"done: {trials} trials, {fails} mismatches, seed {seed}", flush=True)
sys.exit(1 if fails else 0)
