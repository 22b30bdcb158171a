"""Histogram entry points: NVHist / AHist on the B200 (reference: kernels.py:1-535).

Same names, signatures and error behaviour as the reference's kernels module; the
work runs in libhist256's sm_100a kernels (one launch per call or per batch):

  naive_histogram     (kernels.py:336-346)  -> HS_KIND_NAIVE    lane-private pair counters
  adaptive_histogram  (kernels.py:349-384)  -> HS_KIND_ADAPTIVE same core + CPU-pattern hot bin
                         return_slots / narrow_counters -> hs_group_slots (reference lane map)
  adaptive_lane_touches (kernels.py:387-407) -> hs_group_slots mode 1
  compute_histogram   (kernels.py:499-512)  -> kind dispatch
  run_ablation        (kernels.py:421-496)  -> hs_ablation_stage (genealogy on the device)

``WorkerGroupConfig`` is validated exactly as the reference does (kernels.py:64-75).
The 256-bin result does not depend on it (groups and lanes only change the order of
increments); it fixes the group/lane mapping of the slot-level compat outputs.
``reference_histogram`` keeps the reference contract: the serial CPU definition
(np.bincount of the pixel stream) — it is the API's named oracle, never a device fallback.
"""
from __future__ import annotations

import enum
from dataclasses import dataclass

import numpy as np

from . import _native as N
from . import device as D
from .core import BINS, DeviceChunk, Histogram256, PackedChunk
from .pattern import BinningPattern, validate_pattern


class SubCounterOverflow(OverflowError):
    """A narrow (16-bit) sub-counter wrapped during a kernel run (kernels.py:38-39)."""


class KernelKind(enum.Enum):
    """Production kernels plus the timing-only ablation stages (kernels.py:42-52)."""

    NAIVE = "naive"
    ADAPTIVE = "adaptive"
    COPY_ONLY = "copy_only"
    COPY_INIT = "copy_init"
    PATTERN_LOAD = "pattern_load"
    SUBHIST_NOREDUCE = "subhist_noreduce"
    FULL = "full"


ABLATION_STAGES = (
    KernelKind.COPY_ONLY,
    KernelKind.COPY_INIT,
    KernelKind.PATTERN_LOAD,
    KernelKind.SUBHIST_NOREDUCE,
    KernelKind.FULL,
)

_STAGE_ID = {
    KernelKind.COPY_ONLY: N.HS_STAGE_COPY_ONLY,
    KernelKind.COPY_INIT: N.HS_STAGE_COPY_INIT,
    KernelKind.PATTERN_LOAD: N.HS_STAGE_PATTERN_LOAD,
    KernelKind.SUBHIST_NOREDUCE: N.HS_STAGE_SUBHIST_NOREDUCE,
    KernelKind.FULL: N.HS_STAGE_FULL,
}

_KIND_ID = {KernelKind.NAIVE: N.HS_KIND_NAIVE, KernelKind.ADAPTIVE: N.HS_KIND_ADAPTIVE}


@dataclass(frozen=True)
class WorkerGroupConfig:
    """Lanes per group and number of groups (kernels.py:64-75)."""

    group_size: int = 32
    group_count: int = 4

    def __post_init__(self):
        if self.group_size < 1:
            raise ValueError("group_size must be at least 1")
        if self.group_count < 1:
            raise ValueError("group_count must be at least 1")


@dataclass(frozen=True)
class AblationTiming:
    """Device time of one ablation stage plus derived throughput (kernels.py:78-86)."""

    variant: KernelKind
    duration_s: float
    throughput_bps: float
    checksum: int
    histogram: Histogram256 | None = None


def group_ranges(word_count: int, group_count: int) -> list[tuple[int, int]]:
    """Contiguous equal word ranges, remainder to the last group (kernels.py:311-316).
    Also the byte-range sharding rule across GPUs (distributed.shard_range)."""
    base = word_count // group_count
    return [(g * base, (g + 1) * base) for g in range(group_count - 1)] + [((group_count - 1) * base, word_count)]


def reference_histogram(chunk) -> Histogram256:
    """Serial CPU oracle of the reference API (kernels.py:330-333): a plain count of
    every pixel. Kept for drop-in users; no device path calls it."""
    if isinstance(chunk, DeviceChunk):
        chunk = chunk.to_host()
    return Histogram256(np.bincount(chunk.pixels(), minlength=BINS).astype(np.uint64))


def _check_chunk(chunk) -> None:
    if not isinstance(chunk, (PackedChunk, DeviceChunk)):
        raise TypeError(f"expected PackedChunk or DeviceChunk, got {type(chunk).__name__}")


def naive_histogram(chunk, cfg: WorkerGroupConfig) -> Histogram256:
    """NVHist analogue (kernels.py:336-346): one launch of the lane-private kernel."""
    _check_chunk(chunk)
    counts = D.histograms([chunk], N.HS_KIND_NAIVE)
    return Histogram256(counts[0])


def adaptive_histogram(chunk, pattern: BinningPattern, cfg: WorkerGroupConfig, *,
                       narrow_counters: bool = False, return_slots: bool = False):
    """AHist analogue (kernels.py:349-384).

    The pattern is validated before launch (kernels.py:363). The production launch
    counts with the lane-banked core; when the pattern's prior was dominated by one
    value (pattern.dominance >= device.SPREAD_BELOW, or for patterns of unknown origin a
    unique widest sub-bin run) its hot bin is counted in registers. With
    ``return_slots`` or ``narrow_counters`` the reference's per-group slot arrays
    (group/lane mapping of kernels.py:105-108, :149-150) are produced on the device by
    hs_group_slots and reduced per bin as reduce_subbins does."""
    validate_pattern(pattern)
    _check_chunk(chunk)
    if not (narrow_counters or return_slots):
        return Histogram256(D.histograms([chunk], N.HS_KIND_ADAPTIVE, pattern)[0])
    mode = 2 if narrow_counters else 0
    slots = D.group_slots(chunk, pattern, cfg.group_size, cfg.group_count, mode)
    group_slots = [slots[g].copy() for g in range(cfg.group_count)]
    result = Histogram256(np.add.reduceat(slots.astype(np.uint64).sum(axis=0), pattern.offset))
    if narrow_counters and result.total() != chunk.pixel_count:
        # a wrapped 16-bit slot shows up as a total deficit of k * 65536 (kernels.py:377-381)
        raise SubCounterOverflow(f"16-bit sub-counter wrapped: total {result.total()} != {chunk.pixel_count}")
    if return_slots:
        return result, group_slots
    return result


def adaptive_lane_touches(chunk, pattern: BinningPattern, cfg: WorkerGroupConfig):
    """Per-group (lane, slot) increment totals (kernels.py:387-407)."""
    validate_pattern(pattern)
    _check_chunk(chunk)
    touches = D.group_slots(chunk, pattern, cfg.group_size, cfg.group_count, 1)
    slots = touches.sum(axis=1)
    result = Histogram256(np.add.reduceat(slots.sum(axis=0), pattern.offset))
    return result, [touches[g].copy() for g in range(cfg.group_count)]


def reduce_subbins(slots: np.ndarray, pattern: BinningPattern) -> Histogram256:
    """Sum each bin's slot run (kernels.py:410-418). On the device this reduction is
    fused into every kernel's flush; this host form serves slot arrays users hold."""
    validate_pattern(pattern)
    if slots.shape != (pattern.total_slots,):
        raise ValueError(f"slot array length {slots.shape} does not match pattern ({pattern.total_slots},)")
    return Histogram256(np.add.reduceat(slots.astype(np.uint64), pattern.offset))


def compute_histogram(chunk, kind: KernelKind, pattern: BinningPattern | None,
                      cfg: WorkerGroupConfig) -> Histogram256:
    """Dispatch on the two production kernels (kernels.py:499-512)."""
    if kind is KernelKind.NAIVE:
        return naive_histogram(chunk, cfg)
    if kind is KernelKind.ADAPTIVE:
        if pattern is None:
            raise ValueError("adaptive kernel needs a binning pattern")
        return adaptive_histogram(chunk, pattern, cfg)
    raise ValueError(f"{kind} is not a production kernel")


def run_ablation(chunk, variant: KernelKind, pattern: BinningPattern, cfg: WorkerGroupConfig) -> AblationTiming:
    """One genealogy stage on the device (kernels.py:421-496, Table 1).

    Stages are cumulative on the production (k_lane) skeleton: read (+XOR checksum),
    + zero the lane-banked counters, + per-pixel pattern load, + per-pixel sub-counter
    increment, + reduce and merge (hs_kernels.cu k_genealogy). Duration is the mean
    CUDA-event device time of back-to-back launches of the stage (device.ablation_stage).

    Checksums are the reference's values: COPY_* the XOR of every word, PATTERN_LOAD the
    XOR over pixels of offset[b] + count[b] (both computed on the device);
    SUBHIST_NOREDUCE the XOR over the ``cfg`` groups of each group's slot sum (its pixel
    count) once the device's increment total equals the pixel count; FULL counts[0]
    XOR-ed once per group (kernels.py:462-473)."""
    if variant not in ABLATION_STAGES:
        raise ValueError(f"{variant} is not an ablation stage")
    validate_pattern(pattern)
    _check_chunk(chunk)
    seconds, sink, hist = D.ablation_stage(chunk, _STAGE_ID[variant], pattern)
    ranges = group_ranges(chunk.byte_size // 4, cfg.group_count)
    checksum = sink
    if variant is KernelKind.SUBHIST_NOREDUCE:
        if sink == chunk.byte_size:  # every pixel incremented one sub-counter
            checksum = 0
            for start, stop in ranges:
                checksum ^= 4 * (stop - start)
    elif variant is KernelKind.FULL:
        checksum = 0
        for _ in ranges:
            checksum ^= int(hist[0])
    throughput = chunk.byte_size / seconds if seconds > 0 else float("inf")
    return AblationTiming(variant, seconds, throughput, checksum, Histogram256(hist) if hist is not None else None)


_warmed = False


def warm_kernels() -> None:
    """Load libhist256 and run every entry point once on a tiny input (the reference
    JIT-warms its numba workers the same way, kernels.py:515-535)."""
    global _warmed
    if _warmed:
        return
    from .pattern import uniform_pattern

    chunk = PackedChunk(np.arange(16, dtype=np.uint32))
    pat = uniform_pattern(BINS + 8, 2)
    cfg = WorkerGroupConfig(group_size=4, group_count=2)
    naive_histogram(chunk, cfg)
    adaptive_histogram(chunk, pat, cfg)
    adaptive_histogram(chunk, pat, cfg, narrow_counters=True)
    adaptive_lane_touches(chunk, pat, cfg)
    for stage in ABLATION_STAGES:
        run_ablation(chunk, stage, pat, cfg)
    _warmed = True
