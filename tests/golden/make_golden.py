"""Generate golden vectors by importing the reference package itself.

Run in the build container (the GPU box has no /root/reference):

    PYTHONPATH=/root/reference/pkg/src NUMBA_CACHE_DIR=/tmp/numba_cache \
        python tests/golden/make_golden.py

Writes tests/golden/reference_vectors.npz and tests/golden/reference_vectors.json.
Every vector here is the output of the reference's own public API on a seeded input;
tests/test_oracle.py pins the oracle to them and the GPU parity tests reuse them.
"""
from __future__ import annotations

import hashlib
import json
import sys
from pathlib import Path

import numpy as np

import histostream as ref  # noqa: E402  (reference package, from PYTHONPATH)
from histostream.core import unpack_chunk
from histostream.datagen import SourceSpec, batch_stream, generate, schedule_stream
from histostream.kernels import adaptive_lane_touches, group_ranges

OUT = Path(__file__).resolve().parent
arrays: dict[str, np.ndarray] = {}
meta: dict = {"reference": str(Path(ref.__file__).resolve().parent), "version": ref.__version__}


def spec_dict(s: SourceSpec) -> dict:
    return {"kind": s.kind, "pixels": s.pixels, "seed": s.seed, "value": s.value, "mean": s.mean,
            "sigma": s.sigma, "degeneracy": s.degeneracy}


# 1. generators: small chunks byte-for-byte, larger ones by sha256 + histogram
gens = [
    SourceSpec("uniform", 4096, 0), SourceSpec("uniform", 64, 0xDEADBEEF), SourceSpec("uniform", 64, (1 << 64) - 1),
    SourceSpec("normal", 4096, 13, mean=127.0, sigma=24.0), SourceSpec("normal", 4096, 5, mean=128.0, sigma=8.0),
    SourceSpec("normal", 1024, 3, mean=0.0, sigma=500.0), SourceSpec("normal", 1024, 21, mean=128.0, sigma=64.0),
    SourceSpec("mixture", 4096, 77, value=200, degeneracy=0.5), SourceSpec("mixture", 4096, 9, value=127, degeneracy=0.6),
    SourceSpec("mixture", 2048, 5, value=31, degeneracy=1.0), SourceSpec("mixture", 2048, 6, degeneracy=0.0),
    SourceSpec("constant", 1024, 0, value=127), SourceSpec("sequential", 1000, 0),
]
meta["gen_small"] = []
for i, s in enumerate(gens):
    px = unpack_chunk(generate(s))
    arrays[f"gen_small_{i}"] = px
    arrays[f"gen_small_{i}_hist"] = ref.reference_histogram(generate(s)).counts
    meta["gen_small"].append(spec_dict(s))
big = [
    SourceSpec("uniform", 1 << 20, 0), SourceSpec("uniform", 65536, 222),
    SourceSpec("normal", 1 << 20, 5, mean=127.0, sigma=24.0), SourceSpec("normal", 1 << 20, 7, mean=128.0, sigma=32.0),
    SourceSpec("mixture", 1_000_000, 111, value=127, degeneracy=0.5),
]
meta["gen_big"] = []
for i, s in enumerate(big):
    c = generate(s)
    arrays[f"gen_big_{i}_hist"] = ref.reference_histogram(c).counts
    meta["gen_big"].append({**spec_dict(s), "sha256": hashlib.sha256(c.words.tobytes()).hexdigest()})

# 2. binning patterns
rng = np.random.default_rng(20241018)
priors = []
pat_cases = []
zero = np.zeros(256, np.uint64)
deg = np.zeros(256, np.uint64); deg[127] = 1_000_000
deg40 = np.zeros(256, np.uint64); deg40[40] = 1_000_000
pat_cases += [(zero, 960, 8), (deg, 960, 8), (deg40, 960, 8), (zero, 256, 1), (zero, 2048, 8), (deg, 2048, 8),
              (zero, 512, 4), (deg, 8192, 32), (zero, 300, 2)]
for k in range(40):
    shape = k % 4
    if shape == 0:
        c = rng.integers(0, 1 << 20, 256).astype(np.uint64)
    elif shape == 1:
        c = np.zeros(256, np.uint64); c[rng.integers(0, 256)] = rng.integers(1, 1 << 40)
    elif shape == 2:
        c = rng.zipf(1.7, 256).astype(np.uint64)
    else:
        c = ref.reference_histogram(generate(SourceSpec("normal", 1 << 14, int(rng.integers(0, 1 << 31)),
                                                        mean=float(rng.uniform(0, 255)), sigma=float(rng.uniform(1, 80))))).counts
    cap = int(rng.integers(1, 9))
    S = int(rng.integers(256, 256 * cap + 1))
    pat_cases.append((c, S, cap))
# near-tie priors exercise the (-frac, bin) ordering
for k in range(6):
    c = np.full(256, 1000 + k, np.uint64); c[::7] += 1
    pat_cases.append((c, 960, 8))
meta["patterns"] = []
for i, (c, S, cap) in enumerate(pat_cases):
    p = ref.compute_binning_pattern(ref.Histogram256(c), S, cap)
    arrays[f"pat_{i}_prior"] = np.asarray(c, np.uint64)
    arrays[f"pat_{i}_offset"] = p.offset.astype(np.int64)
    arrays[f"pat_{i}_count"] = p.count.astype(np.int64)
    meta["patterns"].append({"total_slots": S, "cap": cap})
meta["pattern_text_uniform960"] = ref.pattern_to_text(ref.uniform_pattern(960))

# 3. policy values
meta["policy"] = []
for i in range(12):
    a = rng.integers(0, 1000, 256).astype(np.uint64)
    b = rng.integers(0, 1000, 256).astype(np.uint64)
    if i == 0:
        a = np.zeros(256, np.uint64); a[127] = 4242
    if i == 1:
        a = np.full(256, 10, np.uint64)
    ha, hb = ref.Histogram256(a), ref.Histogram256(b)
    d = ref.degeneracy(ha)
    arrays[f"pol_{i}_a"] = a
    arrays[f"pol_{i}_b"] = b
    meta["policy"].append({"frac": d.max_bin_fraction, "argmax": d.argmax_bin, "total": d.total,
                           "divergence": ref.divergence(ha, hb) if ha.total() and hb.total() else None,
                           "kind": ref.select_kernel(d, ref.SwitchPolicy()).value})

# 4. slot-level vectors with the reference group/lane mapping
meta["slots"] = []
for i in range(8):
    pixels = int(rng.integers(1, 2000)) * 4
    s = SourceSpec("mixture", pixels, int(rng.integers(0, 1 << 32)), value=int(rng.integers(0, 256)),
                   degeneracy=float(rng.uniform(0, 1)))
    chunk = generate(s)
    cfg = ref.WorkerGroupConfig(int(rng.integers(1, 12)), int(rng.integers(1, 4)))
    pattern = ref.compute_binning_pattern(ref.Histogram256(rng.integers(0, 1000, 256).astype(np.uint64)))
    hist, slots = ref.adaptive_histogram(chunk, pattern, cfg, return_slots=True)
    arrays[f"slots_{i}_pixels"] = unpack_chunk(chunk)
    arrays[f"slots_{i}_offset"] = pattern.offset
    arrays[f"slots_{i}_count"] = pattern.count
    arrays[f"slots_{i}_slots"] = np.stack(slots)
    arrays[f"slots_{i}_hist"] = hist.counts
    meta["slots"].append({"group_size": cfg.group_size, "group_count": cfg.group_count,
                          "total_slots": pattern.total_slots, "cap": pattern.cap})
# lane touches
chunk = generate(SourceSpec("uniform", 4096, seed=8))
cfg = ref.WorkerGroupConfig(13, 2)
pattern = ref.compute_binning_pattern(ref.reference_histogram(chunk))
_, touches = adaptive_lane_touches(chunk, pattern, cfg)
arrays["touch_pixels"] = unpack_chunk(chunk)
arrays["touch_offset"] = pattern.offset
arrays["touch_count"] = pattern.count
arrays["touch_out"] = np.stack(touches)
meta["touch"] = {"group_size": 13, "group_count": 2}
# narrow 16-bit: small exact case slot arrays
chunk = generate(SourceSpec("uniform", 4096, seed=10))
_, slots16 = ref.adaptive_histogram(chunk, ref.uniform_pattern(960), ref.WorkerGroupConfig(8, 2),
                                    narrow_counters=True, return_slots=True)
arrays["narrow_pixels"] = unpack_chunk(chunk)
arrays["narrow_slots"] = np.stack(slots16).astype(np.uint16)

# 5. group_ranges
meta["group_ranges"] = [[n, g, group_ranges(n, g)] for n, g in [(10, 3), (2, 4), (0, 2), (1000, 7), (4096, 3), (5, 5)]]

# 6. batch_histograms on word-aligned cuts
meta["batches"] = []
for i in range(4):
    base = generate(SourceSpec("mixture", 4096 * (i + 1), 1000 + i, value=17 * i, degeneracy=0.3 * i))
    cuts = sorted(rng.integers(0, len(base.words) + 1, 3).tolist())
    bounds = [0, *cuts, len(base.words)]
    slices = [ref.PackedChunk(base.words[a:b]) for a, b in zip(bounds, bounds[1:])]
    kind = ref.KernelKind.ADAPTIVE if i % 2 else ref.KernelKind.NAIVE
    got = ref.batch_histograms(slices, kind, ref.uniform_pattern(960), ref.WorkerGroupConfig(4, 2))
    arrays[f"batch_{i}_pixels"] = unpack_chunk(base)
    arrays[f"batch_{i}_hists"] = np.stack([h.counts for h in got])
    meta["batches"].append({"bounds": bounds, "kind": kind.value})

# 7. streaming runs (run_sequential; run_pipeline is bit-identical, stream.py:503-510)
meta["streams"] = []
scen = []
for index in range(6):
    r = np.random.default_rng(900 + index)
    window = int(r.choice([1, 2, 8, 32]))
    batch = int(r.integers(1, 4))
    every = int(r.choice([1, 2, 5]))
    pixels = 4096
    style = index % 3
    u = SourceSpec("uniform", pixels, seed=index)
    c = SourceSpec("constant", pixels, seed=index, value=127)
    m = SourceSpec("mixture", pixels, seed=index, value=200, degeneracy=0.9)
    segs = [(u, 24)] if style == 0 else ([(u, 12), (c, 12)] if style == 1 else [(u, 8), (m, 8), (c, 8)])
    scen.append((segs, 24, pixels, batch, every, window))
scen.append(([(SourceSpec("uniform", 2048, seed=10), 20), (SourceSpec("constant", 2048, seed=10, value=127), 20)],
             40, 2048, 1, 3, 2))
scen.append(([(SourceSpec("normal", 8192, seed=4, mean=128.0, sigma=8.0), 10),
              (SourceSpec("mixture", 8192, seed=4, value=40, degeneracy=0.5), 10)], 20, 8192, 2, 1, 4))
for i, (segs, iters, pixels, batch, every, window) in enumerate(scen):
    cfg = ref.PipelineConfig(num_iterations=iters, chunk_pixels=pixels, batch_size=batch,
                             recompute_pattern_every=every, window_size=window,
                             worker=ref.WorkerGroupConfig(4, 2))
    acc, win, rep, log = ref.run_sequential(schedule_stream(segs, batch), cfg, ref.SwitchPolicy())
    arrays[f"stream_{i}_per_slice"] = np.stack([np.stack([h.counts for h in it]) for it in rep.per_slice_histograms])
    arrays[f"stream_{i}_acc"] = acc.running.counts
    arrays[f"stream_{i}_window"] = win.windowed.counts
    arrays[f"stream_{i}_ring"] = np.stack([h.counts for h in win.ring])
    arrays[f"stream_{i}_deg"] = np.asarray(rep.degeneracy_log, np.float64)
    arrays[f"stream_{i}_div"] = np.asarray(rep.divergence_log, np.float64)
    meta["streams"].append({
        "segments": [[spec_dict(s), n] for s, n in segs], "num_iterations": iters, "chunk_pixels": pixels,
        "batch_size": batch, "recompute_pattern_every": every, "window_size": window,
        "kernel_log": [k.value for k in log], "chunks_seen": acc.chunks_seen,
    })

# 8. genealogy stage checksums (run_ablation, kernels.py:421-496): seeded chunk, pattern
# from the data, several group counts (SUBHIST and FULL checksums depend on them)
meta["ablation"] = []
for i, (kind, px, seed, gc) in enumerate([("uniform", 1 << 14, 11, 2), ("normal", 1 << 14, 3, 3),
                                          ("mixture", 4096 + 12, 5, 1), ("uniform", 1 << 16, 12, 4),
                                          ("sequential", 1 << 12, 0, 5)]):
    spec = SourceSpec(kind, px, seed, mean=128.0, sigma=20.0, value=200, degeneracy=0.6)
    chunk = generate(spec)
    pattern = ref.compute_binning_pattern(ref.reference_histogram(chunk))
    cfg = ref.WorkerGroupConfig(8, gc)
    sums = {st.value: int(ref.run_ablation(chunk, st, pattern, cfg).checksum) for st in ref.ABLATION_STAGES}
    arrays[f"ablation_{i}_pixels"] = unpack_chunk(chunk)
    meta["ablation"].append({"spec": spec_dict(spec), "group_size": 8, "group_count": gc, "checksums": sums})

np.savez_compressed(OUT / "reference_vectors.npz", **arrays)
(OUT / "reference_vectors.json").write_text(json.dumps(meta, indent=1))
print(f"wrote {len(arrays)} arrays, {len(meta['streams'])} streams", file=sys.stderr)
