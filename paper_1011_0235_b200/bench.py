"""Timing helpers with the reference's names and semantics (histostream/bench.py), for
scripts that import them: medians, interleaved wall-time sampling, the interquartile
spread and the guarded ordering verdict the CLI applies.

These time host calls with the wall clock, as the reference does; device-side kernel
timing (CUDA events, graph replays) lives in the CLI and in the repository's bench.py.
"""
from __future__ import annotations

import enum
import random
import time
from typing import Callable

NOISE_GUARD = 0.10      # two medians are "ordered" only beyond this relative margin
NOISE_FLOOR_S = 0.005   # below this median duration an ordering is reported, not enforced


class Verdict(enum.Enum):
    CONFIRMED = "confirmed"
    INCONCLUSIVE = "inconclusive"
    INVERTED = "inverted"


def median(values: list[float]) -> float:
    """Middle value (mean of the two middle values for an even count)."""
    s = sorted(values)
    m = len(s) // 2
    return s[m] if len(s) % 2 else 0.5 * (s[m - 1] + s[m])


def median_duration_s(fn: Callable[[], object], repetitions: int) -> float:
    """Median wall time of ``repetitions`` calls after one untimed warm call."""
    fn()
    out = []
    for _ in range(repetitions):
        t0 = time.perf_counter()
        fn()
        out.append(time.perf_counter() - t0)
    return median(out)


def interleaved_samples(fns: dict[str, Callable[[], object]], repetitions: int,
                        shuffle_seed: int | None = None) -> dict[str, list[float]]:
    """Wall-time samples per candidate, the candidates interleaved within each
    repetition (order shuffled per repetition when a seed is given), after one warm
    call each."""
    for fn in fns.values():
        fn()
    rng = random.Random(shuffle_seed) if shuffle_seed is not None else None
    order = list(fns)
    out: dict[str, list[float]] = {k: [] for k in fns}
    for _ in range(repetitions):
        if rng is not None:
            rng.shuffle(order)
        for k in order:
            t0 = time.perf_counter()
            fns[k]()
            out[k].append(time.perf_counter() - t0)
    return out


def interleaved_median_durations(fns: dict[str, Callable[[], object]], repetitions: int,
                                 shuffle_seed: int | None = None) -> dict[str, float]:
    return {k: median(v) for k, v in interleaved_samples(fns, repetitions, shuffle_seed).items()}


def relative_spread(samples: list[float]) -> float:
    """Interquartile range over the median (0 for fewer than two samples). Quartiles are
    order statistics at indices (n-1)//4 and ceil(3(n-1)/4)."""
    s = sorted(samples)
    n = len(s)
    if n < 2:
        return 0.0
    lo = s[max(0, (n - 1) // 4)]
    hi = s[min(n - 1, -(-3 * (n - 1) // 4))]
    m = median(samples)
    return (hi - lo) / m if m > 0 else 0.0


def ordering(expected_faster: float, expected_slower: float, guard: float = NOISE_GUARD) -> Verdict:
    """CONFIRMED when the expected-faster throughput leads by more than ``guard``,
    INVERTED when it trails by more than ``guard``, INCONCLUSIVE otherwise."""
    if expected_faster > expected_slower * (1.0 + guard):
        return Verdict.CONFIRMED
    if expected_slower > expected_faster * (1.0 + guard):
        return Verdict.INVERTED
    return Verdict.INCONCLUSIVE
