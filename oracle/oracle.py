"""ORACLE — test infrastructure only, never imported by the product package.

CPU restatement of the reference `histostream` (/root/reference/pkg/src/histostream)
for the 256-bin histogram path. Only tests/, __graft_entry__.smoke() and bench.py's
cpu_baseline / ``--impl reference`` legs may import this module.

Parity is pinned two ways (tests/test_oracle.py):
  * golden vectors produced by importing the reference itself in the build container
    (tests/golden/make_golden.py -> tests/golden/reference_vectors.npz, committed);
  * the known answers hard-coded in the reference's own tests (splitmix64 GOLDEN,
    the 960-slot split, the degenerate 8/187/68 pattern, the hand histogram, ...).

Byte/integer work runs in C (oracle/hist_oracle.c via ctypes, built by
oracle/Makefile); the float64 apportionment and policy are restated in plain Python,
operation for operation, citing the reference lines they follow.
"""
from __future__ import annotations

import ctypes
import math
import subprocess
from collections import deque
from pathlib import Path

import numpy as np

BINS = 256
HERE = Path(__file__).resolve().parent
LIB = HERE / "_build" / "liboracle.so"

_MASK = (1 << 64) - 1
_GOLDEN = 0x9E3779B97F4A7C15
_MIX1 = 0xBF58476D1CE4E5B9
_MIX2 = 0x94D049BB133111EB

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not LIB.exists():
            subprocess.run(["make", "-C", str(HERE)], check=True, capture_output=True)
        _lib = ctypes.CDLL(str(LIB))
        P = ctypes.c_void_p
        I = ctypes.c_int64
        U = ctypes.c_uint64
        _lib.or_histogram.argtypes = [P, U, P]
        _lib.or_group_ranges.argtypes = [I, I, P, P]
        _lib.or_naive_worker.argtypes = [P, I, I, I, P]
        _lib.or_adaptive_worker.argtypes = [P, I, I, I, P, P, I, P, P, ctypes.c_int]
        _lib.or_naive_histogram.argtypes = [P, I, I, I, P, P]
        _lib.or_naive_histogram.restype = ctypes.c_int
        _lib.or_adaptive_histogram.argtypes = [P, I, I, I, P, P, I, ctypes.c_int, P, P, P]
        _lib.or_fill_uniform.argtypes = [P, U, U]
        _lib.or_fill_normal.argtypes = [P, U, U, ctypes.c_double, ctypes.c_double]
        _lib.or_fill_mixture.argtypes = [P, U, U, ctypes.c_double, ctypes.c_int]
    return _lib


def _ptr(a: np.ndarray):
    return a.ctypes.data_as(ctypes.c_void_p)


# ----------------------------------------------------------------- histograms
def histogram(pixels: np.ndarray) -> np.ndarray:
    """reference_histogram (kernels.py:330-333) over a uint8 pixel stream."""
    p = np.ascontiguousarray(pixels, dtype=np.uint8)
    out = np.zeros(BINS, np.uint64)
    lib().or_histogram(_ptr(p), p.size, _ptr(out))
    return out


def histogram_mt(pixels: np.ndarray, threads: int | None = None, piece: int = 64 << 20) -> np.ndarray:
    """reference_histogram over a large pixel stream with host threads: the C count of
    each piece (ctypes releases the GIL) and the componentwise sum of the partials
    (merge_all, core.py:152-156). For multi-GiB parity checks."""
    import os
    from concurrent.futures import ThreadPoolExecutor

    p = np.ascontiguousarray(pixels, dtype=np.uint8).reshape(-1)
    threads = threads or len(os.sched_getaffinity(0))
    cuts = list(range(0, p.size, piece)) + [p.size]
    with ThreadPoolExecutor(max(1, threads)) as ex:
        parts = list(ex.map(lambda ab: histogram(p[ab[0]:ab[1]]), zip(cuts, cuts[1:])))
    out = np.zeros(BINS, np.uint64)
    for h in parts:
        out += h
    return out


def ablation_checksums(pixels: np.ndarray, offset, count, group_count: int) -> dict:
    """The genealogy stages' checksums (run_ablation, kernels.py:421-496, workers
    :212-264): copy_only / copy_init XOR every 32-bit word (copy_init adds slot 0 of a
    zeroed array); pattern_load XORs offset[b] + count[b] over every pixel;
    subhist_noreduce XORs each group's slot sum (its pixel count); full XORs counts[0]
    once per group. XOR is order independent, so lanes and groups drop out except where
    the per-group sums enter."""
    p = np.ascontiguousarray(pixels, dtype=np.uint8)
    words = p.view("<u4")
    x = int(np.bitwise_xor.reduce(words.astype(np.uint64))) if words.size else 0
    table = (np.asarray(offset, np.int64) + np.asarray(count, np.int64)).astype(np.uint64)
    pl = int(np.bitwise_xor.reduce(table[p])) if p.size else 0
    sub = 0
    full = 0
    c0 = int(histogram(p)[0])
    for start, stop in group_ranges(words.size, group_count):
        sub ^= 4 * (stop - start)
        full ^= c0
    return {"copy_only": x, "copy_init": x, "pattern_load": pl, "subhist_noreduce": sub, "full": full}


def group_ranges(word_count: int, group_count: int) -> list[tuple[int, int]]:
    """kernels.py:311-316 (the C restatement, returned as Python tuples)."""
    st = np.zeros(group_count, np.int64)
    sp = np.zeros(group_count, np.int64)
    lib().or_group_ranges(word_count, group_count, _ptr(st), _ptr(sp))
    return [(int(a), int(b)) for a, b in zip(st, sp)]


def naive_histogram(words: np.ndarray, group_size: int, group_count: int):
    """naive_histogram (kernels.py:336-346): (u64[256], per-group u64[G,256])."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    out = np.zeros(BINS, np.uint64)
    per = np.zeros((group_count, BINS), np.uint64)
    ovf = lib().or_naive_histogram(_ptr(w), w.size, group_size, group_count, _ptr(out), _ptr(per))
    if ovf:
        raise OverflowError("histogram bin count exceeded 64-bit range")
    return out, per


def adaptive_histogram(words, offset, count, total_slots, group_size, group_count,
                       narrow=False, touches=False):
    """adaptive_histogram (kernels.py:349-384) / adaptive_lane_touches (:387-407).

    Returns (u64[256] from the (possibly wrapped) slot arrays, slots u64[G,S],
    touches u64[G,gs,S] or None)."""
    w = np.ascontiguousarray(words, dtype=np.uint32)
    off = np.ascontiguousarray(offset, dtype=np.int64)
    cnt = np.ascontiguousarray(count, dtype=np.int64)
    out = np.zeros(BINS, np.uint64)
    slots = np.zeros((group_count, total_slots), np.uint64)
    tch = np.zeros((group_count, group_size, total_slots), np.uint64) if touches else None
    lib().or_adaptive_histogram(_ptr(w), w.size, group_size, group_count, _ptr(off), _ptr(cnt),
                                total_slots, int(bool(narrow)), _ptr(out), _ptr(slots),
                                _ptr(tch) if touches else None)
    return out, slots, tch


def simulate_slots(words, offset, count, total_slots, group_size, group_count):
    """Independent numpy prediction of slot totals (the reference test's
    simulate_adaptive_slots, test_kernels.py:28-44)."""
    words = np.asarray(words, dtype=np.uint32)
    offset = np.asarray(offset, dtype=np.int64)
    count = np.asarray(count, dtype=np.int64)
    per_group = []
    for start, stop in group_ranges(len(words), group_count):
        totals = np.zeros(total_slots, np.int64)
        if stop > start:
            w = words[start:stop]
            lanes = np.arange(stop - start) % group_size
            for k in range(4):
                vals = ((w >> (8 * k)) & 0xFF).astype(np.int64)
                np.add.at(totals, offset[vals] + lanes % count[vals], 1)
        per_group.append(totals.astype(np.uint64))
    return per_group


# ----------------------------------------------------------------- pattern (pattern.py)
def check_slot_range(total_slots: int, cap: int) -> str | None:
    """pattern.py:70-76; returns the error message or None."""
    if cap < 1:
        return f"cap must be at least 1, got {cap}"
    if not (BINS <= total_slots <= BINS * cap):
        return f"total_slots {total_slots} outside [{BINS}, {BINS * cap}] for cap {cap}"
    return None


def offsets_from_counts(counts):
    """pattern.py:79-82."""
    out = [0] * BINS
    for b in range(1, BINS):
        out[b] = out[b - 1] + counts[b - 1]
    return out


def uniform_pattern(total_slots: int = 960, cap: int = 8):
    """pattern.py:85-91: (offset, count) as Python lists."""
    err = check_slot_range(total_slots, cap)
    if err:
        raise ValueError(err)
    base, rem = divmod(total_slots, BINS)
    counts = [base + (1 if b < rem else 0) for b in range(BINS)]
    return offsets_from_counts(counts), counts


def binning_pattern(prior, total_slots: int = 960, cap: int = 8):
    """compute_binning_pattern (pattern.py:94-133) restated with Python floats.

    Every float op is the same IEEE double op numpy performs: counts -> float64 by
    round-to-nearest, ``extras / total`` as Python's correctly rounded int division."""
    err = check_slot_range(total_slots, cap)
    if err:
        raise ValueError(err)
    prior = [int(c) for c in prior]
    extras = total_slots - BINS
    total = sum(prior) & _MASK  # Histogram256.total(): uint64 sum
    if total == 0:
        ideal = [extras / BINS] * BINS
    else:
        r = extras / total
        ideal = [float(c) * r for c in prior]
    floors = [math.floor(x) for x in ideal]
    granted = [min(f, cap - 1) for f in floors]
    counts = [1 + g for g in granted]
    remaining = extras - sum(granted)
    if remaining > 0:
        frac = [ideal[b] - floors[b] for b in range(BINS)]
        order = sorted(range(BINS), key=lambda b: (-frac[b], b))
        pool = [b for b in order if counts[b] < cap]
        while remaining > 0:
            progressed = False
            for b in pool:
                if counts[b] < cap:
                    counts[b] += 1
                    remaining -= 1
                    progressed = True
                    if remaining == 0:
                        break
            if not progressed:
                raise ValueError("ran out of uncapped bins")
            pool = [b for b in pool if counts[b] < cap]
    return offsets_from_counts(counts), counts


def validate_pattern(offset, count, total_slots, cap) -> str | None:
    """validate_pattern (pattern.py:136-149): first violated invariant's message or None."""
    if len(count) != BINS or len(offset) != BINS:
        return "pattern arrays must have 256 entries"
    if any(c < 1 for c in count):
        return "count below 1"
    if any(c > cap for c in count):
        return "count above cap"
    if sum(count) != total_slots:
        return "slot total mismatch"
    if offset[0] != 0 or any(offset[b] != offset[b - 1] + count[b - 1] for b in range(1, BINS)):
        return "offsets not contiguous"
    return None


def pattern_text(offset, count) -> str:
    """pattern_to_text (pattern.py:152-158)."""
    return "".join(f"{b} {int(offset[b])} {int(count[b])}\n" for b in range(BINS))


def floor_shares(prior, total_slots=960):
    """pattern.py:176-183."""
    extras = total_slots - BINS
    total = sum(int(c) for c in prior) & _MASK
    if total == 0:
        return [math.floor(extras / BINS)] * BINS
    r = extras / total
    return [math.floor(float(int(c)) * r) for c in prior]


# ----------------------------------------------------------------- policy (policy.py)
def degeneracy(counts):
    """policy.py:39-46: (max_bin_fraction, argmax_bin, total)."""
    counts = [int(c) for c in counts]
    total = sum(counts) & _MASK
    if total == 0:
        return 0.0, 0, 0
    am = max(range(BINS), key=lambda b: (counts[b], -b))
    return counts[am] / total, am, total


def select_kernel(fraction: float, threshold: float = 0.45) -> str:
    """policy.py:49-53 (inclusive threshold)."""
    return "adaptive" if fraction >= threshold else "naive"


def divergence(a, b) -> float:
    """policy.py:56-64 — total variation; the same numpy expression (pairwise sum)."""
    a = np.asarray(a, dtype=np.uint64)
    b = np.asarray(b, dtype=np.uint64)
    ta, tb = int(a.sum(dtype=np.uint64)), int(b.sum(dtype=np.uint64))
    if ta == 0 or tb == 0:
        raise ValueError("divergence needs two non-empty histograms")
    pa = a.astype(np.float64) / ta
    pb = b.astype(np.float64) / tb
    return 0.5 * float(np.abs(pa - pb).sum())


# ----------------------------------------------------------------- generators (datagen.py)
def splitmix64(seed: int):
    """datagen.py:6-13 — the pure-Python mirror of the reference test (test_datagen.py:34-43)."""
    state = seed & _MASK
    while True:
        state = (state + _GOLDEN) & _MASK
        z = state
        z = ((z ^ (z >> 30)) * _MIX1) & _MASK
        z = ((z ^ (z >> 27)) * _MIX2) & _MASK
        yield z ^ (z >> 31)


def generate(kind: str, pixels: int, seed: int = 0, value: int = 127, mean: float = 127.0,
             sigma: float = 24.0, degeneracy: float = 0.0) -> np.ndarray:
    """generate (datagen.py:158-178) as a uint8 pixel array (C fills for speed)."""
    seed &= _MASK
    if kind == "constant" or (kind == "mixture" and degeneracy == 1.0):
        return np.full(pixels, value, np.uint8)
    if kind == "sequential":
        return (np.arange(pixels, dtype=np.uint64) & 0xFF).astype(np.uint8)
    out = np.empty(pixels, np.uint8)
    if kind == "uniform":
        lib().or_fill_uniform(_ptr(out), pixels, seed)
    elif kind == "normal":
        lib().or_fill_normal(_ptr(out), pixels, seed, float(mean), float(sigma))
    elif kind == "mixture":
        lib().or_fill_mixture(_ptr(out), pixels, seed, float(degeneracy), int(value))
    else:
        raise ValueError(kind)
    return out


def pack(pixels: np.ndarray) -> np.ndarray:
    """pack_pixels (core.py:101-122): little-endian words."""
    p = np.ascontiguousarray(pixels, dtype=np.uint8)
    return p.view(np.uint32).copy() if p.size else np.empty(0, np.uint32)


# ----------------------------------------------------------------- stream fold (stream.py)
def run_sequential(batches, num_iterations, window_size=128, recompute_every=1, total_slots=960,
                   cap=8, threshold=0.45):
    """The state fold of run_sequential (stream.py:445-500) with oracle histograms.

    batches: iterable of lists of uint8 pixel arrays. Returns a dict with the kernel
    log, per-slice histograms, accumulator/window state and the policy logs."""
    acc = np.zeros(BINS, np.uint64)
    chunks = 0
    ring: deque = deque()
    win = np.zeros(BINS, np.uint64)
    pattern = binning_pattern([0] * BINS, total_slots, cap)
    kind = "naive"
    kernel_log, per_slice, deg_log, div_log, pattern_log = [], [], [], [], []
    it = iter(batches)
    for i in range(num_iterations):
        if i % recompute_every == 0:  # stream.py:407-414 (lag 1: window as of i-1)
            pattern = binning_pattern(win, total_slots, cap)
            kind = select_kernel(degeneracy(win)[0], threshold)
        batch = next(it)
        hists = [histogram(p) for p in batch]
        per_slice.append(hists)
        for h in hists:  # stream.py:419-425
            acc = acc + h
            chunks += 1
            ring.append(h)
            win = win + h
            if len(ring) > window_size:
                ev = ring.popleft()
                if np.any(win < ev):
                    raise ArithmeticError("window sum fell behind its ring contents")
                win = win - ev
        kernel_log.append(kind)
        pattern_log.append(pattern)
        deg_log.append(degeneracy(win)[0])
        div_log.append(divergence(acc, win))
    return {
        "kernel_log": kernel_log, "per_slice": per_slice, "acc": acc, "chunks_seen": chunks,
        "window": win, "ring": list(ring), "degeneracy_log": deg_log, "divergence_log": div_log,
        "pattern_log": pattern_log,
    }
