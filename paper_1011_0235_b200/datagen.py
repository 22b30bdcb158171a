"""Seeded input streams (reference: datagen.py:1-237).

Byte-exact with the reference generators: splitmix64 outputs consumed 8 bytes at a
time LSB first; unit doubles (z >> 11) * 2^-53; normal = Irwin-Hall of 12 units,
floor(mean + sigma*z + 0.5) clamped; mixture draws its Bernoulli first; chunk seed =
base seed XOR chunk index (datagen.py:6-29, :196-198).

Host generation is native (``hs_generate_host``, multi-threaded for the counter-based
kinds). ``generate_device`` fills HBM directly (``hs_generate_device``) — counter-based
kinds only — so >= 16 GiB benchmark streams never cross PCIe; shards of one logical
stream are generated in place from their first pixel index.
"""
from __future__ import annotations

import logging
import os
from dataclasses import dataclass, replace
from pathlib import Path
from typing import Iterator

import numpy as np

from . import _native as N
from .core import PackedChunk, pack_pixels

log = logging.getLogger(__name__)

UNIFORM = "uniform"
SEQUENTIAL = "sequential"
CONSTANT = "constant"
NORMAL = "normal"
MIXTURE = "mixture"
FILE = "file"
_KINDS = (UNIFORM, SEQUENTIAL, CONSTANT, NORMAL, MIXTURE, FILE)
_GEN_ID = {UNIFORM: N.HS_GEN_UNIFORM, SEQUENTIAL: N.HS_GEN_SEQUENTIAL, CONSTANT: N.HS_GEN_CONSTANT,
           NORMAL: N.HS_GEN_NORMAL, MIXTURE: N.HS_GEN_MIXTURE}
_MASK64 = (1 << 64) - 1


class SpecInvalid(ValueError):
    """A SourceSpec field violated its range (datagen.py:55-56)."""


class FileUnreadable(OSError):
    """The file behind a file-kind spec could not be read (datagen.py:59-60)."""


@dataclass(frozen=True)
class SourceSpec:
    """Distribution kind, size, seed and shape parameters (datagen.py:63-89)."""

    kind: str
    pixels: int
    seed: int = 0
    value: int = 127
    mean: float = 127.0
    sigma: float = 24.0
    degeneracy: float = 0.0
    path: str | None = None

    def validate(self) -> None:
        if self.kind not in _KINDS:
            raise SpecInvalid(f"unknown source kind {self.kind!r}")
        if self.kind != FILE and (self.pixels < 0 or self.pixels % 4):
            raise SpecInvalid("pixels must be a non-negative multiple of 4")
        if not (0 <= self.value <= 255):
            raise SpecInvalid("value must be in 0..=255")
        if self.kind == NORMAL and self.sigma <= 0:
            raise SpecInvalid("sigma must be positive")
        if self.kind == MIXTURE and not (0.0 <= self.degeneracy <= 1.0):
            raise SpecInvalid("degeneracy must be in [0, 1]")
        if self.kind == FILE and not self.path:
            raise SpecInvalid("file kind needs a path")


def _host_threads() -> int:
    try:
        return max(1, len(os.sched_getaffinity(0)))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def fill_pixels(spec: SourceSpec, out: np.ndarray) -> np.ndarray:
    """Write the spec's pixel stream into the uint8 array ``out`` (e.g. pinned memory)."""
    spec.validate()
    n = out.size
    kind = CONSTANT if (spec.kind == MIXTURE and spec.degeneracy == 1.0) else spec.kind
    status = N.lib().hs_generate_host(_GEN_ID[kind], spec.seed & _MASK64, int(spec.value), float(spec.mean),
                                      float(spec.sigma), float(spec.degeneracy), out.ctypes.data, n,
                                      _host_threads())
    N.check(status, "hs_generate_host")
    return out


def generate(spec: SourceSpec, out: np.ndarray | None = None) -> PackedChunk:
    """Deterministically generate the chunk a spec describes (datagen.py:158-178).
    ``out`` (uint8, >= spec.pixels) lets callers generate straight into pinned memory."""
    spec.validate()
    if spec.kind == FILE:
        return load_raw_file(spec.path)
    buf = np.empty(spec.pixels, np.uint8) if out is None else out[: spec.pixels]
    fill_pixels(spec, buf)
    return PackedChunk(buf.view(np.uint32))


def generate_device(spec: SourceSpec, data, first_pixel: int = 0, stream=None):
    """Fill the uint8 CUDA tensor ``data`` with pixels [first_pixel, first_pixel + n)
    of the spec's stream, on the device (uniform, sequential, constant, normal)."""
    import torch

    spec.validate()
    if spec.kind not in (UNIFORM, SEQUENTIAL, CONSTANT, NORMAL):
        raise SpecInvalid(f"{spec.kind} has a data-dependent draw count: generate it on the host")
    if (not isinstance(data, torch.Tensor) or not data.is_cuda or data.dtype != torch.uint8
            or not data.is_contiguous()):
        raise TypeError("generate_device needs a contiguous uint8 CUDA tensor")
    st = stream or torch.cuda.current_stream(data.device)
    if st.device != data.device:
        raise ValueError(f"tensor on {data.device} but stream on {st.device}")
    s = st.cuda_stream
    N.check(N.lib().hs_generate_device(_GEN_ID[spec.kind], spec.seed & _MASK64, int(spec.value),
                                       float(spec.mean), float(spec.sigma), int(first_pixel),
                                       data.data_ptr(), data.numel(), s), "hs_generate_device")
    return data


def load_raw_file(path: str | Path) -> PackedChunk:
    """Headerless raw bytes; a trailing partial word is dropped with a warning (datagen.py:181-193)."""
    try:
        data = Path(path).read_bytes()
    except OSError as exc:
        raise FileUnreadable(f"cannot read {path}: {exc}") from exc
    usable = len(data) & ~3
    if usable != len(data):
        log.warning("truncating %s: dropped %d trailing bytes to reach a word boundary", path, len(data) - usable)
    return pack_pixels(np.frombuffer(data[:usable], dtype=np.uint8))


def derived_spec(spec: SourceSpec, chunk_index: int) -> SourceSpec:
    """Per-chunk spec: seed = base seed XOR chunk index (datagen.py:196-198)."""
    return replace(spec, seed=spec.seed ^ chunk_index)


def chunk_stream(spec: SourceSpec, count: int, start_index: int = 0) -> Iterator[PackedChunk]:
    """``count`` chunks with consecutive derived seeds (datagen.py:201-204)."""
    for i in range(start_index, start_index + count):
        yield generate(derived_spec(spec, i))


def batch_stream(spec: SourceSpec, num_iterations: int, batch_size: int = 1) -> Iterator[list[PackedChunk]]:
    """Iteration i carries chunk indices [i*batch_size, (i+1)*batch_size) (datagen.py:207-216)."""
    for i in range(num_iterations):
        yield [generate(derived_spec(spec, i * batch_size + j)) for j in range(batch_size)]


def schedule_stream(segments: list[tuple[SourceSpec, int]], batch_size: int = 1) -> Iterator[list[PackedChunk]]:
    """Concatenated (spec, iterations) segments; the chunk index keeps counting across
    segment boundaries (datagen.py:219-231)."""
    index = 0
    for spec, iterations in segments:
        for _ in range(iterations):
            batch = [generate(derived_spec(spec, index + j)) for j in range(batch_size)]
            index += batch_size
            yield batch


def warm_generators() -> None:
    """Load the native generators once (the reference JIT-warms here, datagen.py:234-237)."""
    for kind in (UNIFORM, NORMAL, MIXTURE):
        generate(SourceSpec(kind=kind, pixels=8, seed=1, degeneracy=0.5))
