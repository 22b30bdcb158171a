"""Device runtime around libhist256: staging, launches and readback.

PyTorch is used only as plumbing — the CUDA caching allocator for device buffers,
pinned host memory and streams/events. All counting happens in libhist256's sm_100a
kernels through the C ABI (include/hist256.h); if CUDA or the library is missing
every entry point raises (there is no CPU fallback).

Data flow for one batch (the reference's batch_histograms, stream.py:260-316):
  host PackedChunks --H2D (pinned: async; pageable: copied into a pinned bounce buffer with
  threaded streaming stores, large batches piecewise with each piece DMA'd as it lands)--> one device
  staging buffer -> hs_histogram_batched (one launch, one segment per chunk) ->
  uint64[n, 256] on device --D2H 2 KiB per chunk--> read-only Histogram256 values.
DeviceChunks skip the H2D: their tensors are segments of the same launch.
"""
from __future__ import annotations

import bisect
import ctypes
import os
import threading
import warnings
import weakref
from dataclasses import dataclass, field
from typing import Sequence

import numpy as np

from . import _native as N
from .core import BINS, DeviceChunk, PackedChunk

_torch = None


def torch():
    """Import torch lazily (host-only helpers must not pay for it)."""
    global _torch
    if _torch is None:
        import torch as t

        _torch = t
    return _torch


class DeviceUnavailable(RuntimeError):
    """No CUDA device: the histogram path runs only on the GPU (no CPU fallback)."""


_cuda_ok = False


def require_cuda():
    """torch, once a CUDA device and libhist256 are known to be there (checked on the
    first call; later calls are on the per-image latency path and skip the probe)."""
    global _cuda_ok
    t = torch()
    if not _cuda_ok:
        if not t.cuda.is_available():
            raise DeviceUnavailable("CUDA device required: libhist256 has no CPU fallback")
        N.lib()
        _cuda_ok = True
    return t


# ------------------------------------------------------------------ pinned host memory
class _PinnedRegistry:
    """Address ranges of pinned buffers handed out by pinned_words()/pinned_bytes()."""

    def __init__(self):
        self._lock = threading.Lock()
        self._starts: list[int] = []
        self._ends: list[int] = []

    def add(self, arr: np.ndarray) -> None:
        start = arr.ctypes.data
        end = start + arr.nbytes
        with self._lock:
            i = bisect.bisect_left(self._starts, start)
            self._starts.insert(i, start)
            self._ends.insert(i, end)
        # The range lives as long as the memory: tie it to the object at the end of the
        # array's base chain, which every numpy view of it keeps alive (not to the torch
        # tensor that allocated it: tensor.numpy() holds another alias of the storage,
        # and the original tensor object can die while the memory is still in use).
        owner = arr
        while isinstance(owner, np.ndarray) and owner.base is not None:
            owner = owner.base
        weakref.finalize(owner, self._drop, start)

    def _drop(self, start: int) -> None:
        with self._lock:
            i = bisect.bisect_left(self._starts, start)
            if i < len(self._starts) and self._starts[i] == start:
                del self._starts[i]
                del self._ends[i]

    def contains(self, ptr: int, nbytes: int) -> bool:
        with self._lock:
            i = bisect.bisect_right(self._starts, ptr) - 1
            return i >= 0 and ptr + nbytes <= self._ends[i]


_pinned = _PinnedRegistry()


def pinned_bytes(n: int) -> np.ndarray:
    """A uint8 numpy array backed by page-locked host memory (async H2D source)."""
    t = require_cuda().empty(max(int(n), 1), dtype=torch().uint8, pin_memory=True)
    full = t.numpy()
    _pinned.add(full)
    return full[: int(n)]


def pinned_words(n_words: int) -> np.ndarray:
    """A uint32 numpy array backed by page-locked host memory."""
    return pinned_bytes(4 * int(n_words)).view(np.uint32)


def is_pinned(arr: np.ndarray) -> bool:
    return _pinned.contains(arr.ctypes.data, arr.nbytes)


# ------------------------------------------------------------------ pageable copies
# Pageable chunks reach the device through a page-locked bounce buffer. Two things set
# the rate (tools/diag/pageable_rate.py, pageable_small.py): one host thread copies
# 15-26 GB/s, below the PCIe link (8 threads: 74-79 GB/s); and a DMA out of a bounce
# buffer the CPU has just written through its caches runs at 14-20 GB/s. So copies use
# streaming stores (hs_copy_streaming). Up to 16 MiB of pageable input per batch is
# copied in one call split over native threads; larger batches go in 4 MiB pieces to a
# pool of copy threads, each piece DMA'd as soon as it has landed while the pool copies
# on (pageable run_pipeline 14 -> 47 GB/s; native-thread pieces on the staging thread
# reached 38). The driver's own pageable copy runs ~11 GB/s.
_COPY_POOLED_ABOVE = 16 << 20
_COPY_PIECE = 4 << 20
_COPY_SYNC_MIN = 8 << 20  # synchronous calls with less pageable input use the driver's copy
_copy_pool = None
_copy_pool_lock = threading.Lock()


def copy_threads() -> int:
    """Host threads for pageable -> page-locked copies (HS_COPY_THREADS overrides)."""
    env = os.environ.get("HS_COPY_THREADS")
    if env:
        return max(1, int(env))
    return max(1, min(8, (os.cpu_count() or 2) // 2))


def _threads_for(n: int) -> int:
    # measured per copy: 1 MiB fastest on 1 thread (40 us; 4: 53), 2-4 MiB on 4, 16 MiB on 8
    return 1 if n < (2 << 20) else min(copy_threads(), 4 if n < (16 << 20) else 8)


def _copy_into(dst: np.ndarray, src: np.ndarray, threads: int = 1) -> None:
    """dst[:] = src with streaming stores over up to ``threads`` host threads
    (hs_copy_streaming; ctypes drops the GIL for the call)."""
    N.check(N.lib().hs_copy_streaming(dst.ctypes.data, src.ctypes.data, src.nbytes, int(threads)),
            "hs_copy_streaming")


def _pool():
    global _copy_pool
    if _copy_pool is None:
        with _copy_pool_lock:
            if _copy_pool is None:
                from concurrent.futures import ThreadPoolExecutor

                _copy_pool = ThreadPoolExecutor(max_workers=copy_threads(), thread_name_prefix="hs-h2d-copy")
    return _copy_pool


# ------------------------------------------------------------------ staging
class Staging:
    """A growable device buffer (+ pinned readback buffer) owned by one stream user.

    Reuse is safe once the work that read it has completed; the synchronous API
    waits for its readback, the pipeline releases a slot only after its batch is
    folded (stream.py:_Slot protocol)."""

    def __init__(self, device=None):
        t = require_cuda()
        self.device = t.device("cuda", t.cuda.current_device() if device is None else t.device(device).index)
        self._dev = None
        self._bounce = None
        self._bounce_done = None  # event after the last copies out of the bounce buffer
        self._out_host = None
        self._out_dev = None
        self._ws: dict[int, object] = {}  # stream handle -> workspace (insertion = LRU order)
        self._cap: dict[int, object] = {}  # the same during a CUDA-graph capture
        self._one = None  # _OneCall: prepared arguments of the one-chunk blocking calls

    def device_bytes(self, n: int):
        t = torch()
        if self._dev is None or self._dev.numel() < n:
            cap = max(n, 1 << 20)
            self._dev = t.empty(cap + 256, dtype=t.uint8, device=self.device)
        # 256-B aligned start (the allocator returns 512-B aligned blocks)
        return self._dev

    def host_bounce(self, n: int) -> np.ndarray:
        """Page-locked bounce buffer for pageable host chunks: they are copied here on
        the host and DMA'd from here, so the H2D stays asynchronous and never goes
        through the driver's pageable-copy path (which serialises with other threads'
        CUDA calls: 20-110 ms stalls in run_pipeline, tools/diag/c07_probe.py)."""
        if self._bounce is None or self._bounce.size < n:
            self._bounce = pinned_bytes(max(int(n), 1 << 20))
        return self._bounce

    _MAX_WS = 32

    def workspace(self, stream=None):
        """Device workspace of hs_histogram_batched (per-segment tickets + partials) for
        launches on ``stream`` (a torch stream, a raw handle, or None for the current
        stream), zeroed once; every call leaves its slots zero again. Launches that share a
        workspace must be stream-ordered, so there is one per CUDA stream: two calls on
        unsynchronized streams never share accumulator rows. Each is allocated and
        zeroed on its own stream, so the caching allocator only ever hands its memory
        back to work ordered after it."""
        t = torch()
        if stream is None:
            h = _raw_stream(self.device.index)
        else:
            h = int(stream) if isinstance(stream, int) else int(stream.cuda_stream)
        if t.cuda.is_current_stream_capturing():
            # Inside a CUDA-graph capture nothing executes: a workspace created here is
            # zeroed by a memset node of the graph (and lives in the graph's private
            # pool), so it serves only launches of this capture and never leaks into
            # eager use. One per stream per capture; dropped once capturing ends.
            ws = self._cap.get(h)
            if ws is None:
                n = int(N.lib().hs_workspace_bytes(256))
                with t.cuda.stream(t.cuda.ExternalStream(h, device=self.device)):
                    ws = t.zeros(max(n, 256), dtype=t.uint8, device=self.device)
                self._cap[h] = ws
            return ws
        if self._cap:
            self._cap.clear()
        ws = self._ws.get(h)
        if ws is None:
            n = int(N.lib().hs_workspace_bytes(256))  # launches of up to 256 segments
            if len(self._ws) >= self._MAX_WS:  # bounded: drop the least recently created
                self._ws.pop(next(iter(self._ws)))
            with t.cuda.stream(t.cuda.ExternalStream(h, device=self.device)):
                ws = t.zeros(max(n, 256), dtype=t.uint8, device=self.device)
            self._ws[h] = ws
        return ws

    def device_out(self, nseg: int):
        """Device int64 [nseg, 256] counts buffer for the synchronous host path."""
        t = torch()
        if self._out_dev is None or self._out_dev.shape[0] < nseg:
            self._out_dev = t.empty((max(nseg, 64), BINS), dtype=t.int64, device=self.device)
        return self._out_dev[:nseg]

    def host_out(self, nseg: int):
        t = torch()
        need = nseg * BINS
        if self._out_host is None or self._out_host.numel() < need:
            self._out_host = t.empty(max(need, 64 * BINS), dtype=t.int64, pin_memory=True)
        return self._out_host[:need]

    def one_call(self, stream: int, n_bytes: int = 0) -> "_OneCall":
        """Arguments of one-chunk blocking calls (the per-image path) on raw stream
        ``stream``, built once: the device, host and workspace buffers are only ever
        replaced by larger ones, so the cached pointers stay valid until a buffer grows
        or the stream changes."""
        one = self._one
        if (one is None or one.stream != stream or one.out_dev is not self._out_dev or one.h_out is not self._out_host
                or one.dev is not self._dev or (n_bytes and (self._dev is None or self._dev.numel() < n_bytes))):
            if n_bytes:
                self.device_bytes(n_bytes)
            one = self._one = _OneCall(self, self.device_out(1), self.host_out(1), self.workspace(stream), self._dev,
                                       stream)
        return one


class _OneCall:
    """ctypes arguments of hs_histogram_sync / hs_histogram_host for one chunk."""

    def __init__(self, staging: Staging, out_dev, h_out, ws, dev, stream: int):
        self.stream = stream
        self.out_dev = staging._out_dev  # the owning tensors (identity = validity)
        self.h_out = staging._out_host
        self.dev = staging._dev
        self.out_dev_ptr = out_dev.data_ptr()
        self.h_np = h_out.numpy().view(np.uint64)
        self.h_out_p = ctypes.cast(h_out.data_ptr(), N._U64P)
        self.ws_ptr, self.ws_n = ws.data_ptr(), ws.numel()
        self.dev_ptr, self.dev_n = (dev.data_ptr(), dev.numel()) if dev is not None else (None, 0)
        self.begin = (ctypes.c_uint64 * 1)(0)
        self.end = (ctypes.c_uint64 * 1)(0)
        self.ptrs = (ctypes.c_void_p * 1)()
        self.pattern = None
        self.pattern_args = (None, None, 0, 0)

    def pattern_ptrs(self, pattern):
        if pattern is None:
            return None, None, 0, 0
        if pattern is not self.pattern:  # patterns are immutable; keep it alive with its pointers
            self.pattern = pattern
            self.pattern_args = (N.i64p(pattern.offset), N.i64p(pattern.count), int(pattern.total_slots),
                                 int(pattern.cap))
        return self.pattern_args


@dataclass
class StagedBatch:
    """A batch whose bytes are on the device: segment s is [base+begin[s], base+end[s])."""

    base: int
    begin: np.ndarray
    end: np.ndarray
    keepalive: list = field(default_factory=list)
    ready: object = None  # torch.cuda.Event recorded after the H2D copies, or None

    @property
    def nseg(self) -> int:
        return int(self.begin.size)

    @property
    def nbytes(self) -> int:
        return int((self.end - self.begin).sum())


def stage(chunks: Sequence, staging: Staging | None, stream=None) -> StagedBatch:
    """Place a batch on the device. Host chunks are copied (async when their memory is
    pinned) into ``staging``'s buffer at word-aligned offsets on ``stream``; device
    chunks are referenced in place. Records ``ready`` after the copies."""
    t = require_cuda()
    dev_index = staging.device.index if staging is not None else t.cuda.current_device()
    for c in chunks:
        if type(c) is DeviceChunk and c._dev != dev_index:
            raise ValueError(f"DeviceChunk on cuda:{c._dev} staged for cuda:{dev_index}")
    if chunks and all(type(c) is DeviceChunk for c in chunks):
        # fast path (device-resident batches, e.g. the device stream engine): addresses
        # and sizes are cached on the chunks, so staging 64 chunks is a few microseconds
        ptrs = np.array([c._ptr for c in chunks], dtype=np.uint64)
        sizes = np.array([c._n for c in chunks], dtype=np.uint64)
        nz = sizes > 0
        base = int(ptrs[nz].min()) if nz.any() else 0
        begin = np.where(nz, ptrs - np.uint64(base), np.uint64(0)).astype(np.uint64)
        return StagedBatch(base, begin, begin + sizes, [c.data for c in chunks], None)
    stream = stream or t.cuda.current_stream()
    host = [(i, c) for i, c in enumerate(chunks) if isinstance(c, PackedChunk)]
    ptrs = [0] * len(chunks)
    sizes = [0] * len(chunks)
    keep: list = []
    ready = None
    if host:
        total = sum(c.byte_size for _, c in host)
        if staging is None:
            staging = Staging()
        dev = staging.device_bytes(total)
        keep.append(dev)
        base = dev.data_ptr()
        off = 0
        # chunks that sit back to back in host memory (slices of one pinned stream) go
        # in one copy: 16 MiB copies reach 54.5 GB/s, 128 MiB ones 55.2 GB/s
        runs: list[list] = []  # [host_ptr, dev_off, nbytes, first chunk array]
        bounce = None  # pageable chunks go through the staging's pinned bounce buffer
        for i, c in host:
            n = c.byte_size
            ptrs[i] = base + off
            sizes[i] = n
            if n:
                hp = c.words.ctypes.data
                if runs and runs[-1][0] + runs[-1][2] == hp and runs[-1][1] + runs[-1][2] == off:
                    runs[-1][2] += n
                else:
                    runs.append([hp, off, n, c.words])
                keep.append(c.words)
            off += n
        srcs = []  # (device offset, bytes, host array, page-locked?) per run
        for hp, doff, n, first in runs:
            if n == first.nbytes:
                arr = first.view(np.uint8)
            else:  # the run spans several chunks' memory (all kept alive above)
                arr = np.ctypeslib.as_array((ctypes.c_uint8 * n).from_address(hp))
            srcs.append((doff, n, arr, _pinned.contains(hp, n)))
        pageable = sum(n for _, n, _, pinned in srcs if not pinned)
        pool = _pool() if pageable > _COPY_POOLED_ABOVE else None
        if pageable:
            bounce = staging.host_bounce(total)
            if staging._bounce_done is not None:  # its previous DMA must have read it
                staging._bounce_done.synchronize()
        jobs: list = []  # (device offset, page-locked source, pool future or None), in DMA order
        try:
            for doff, n, arr, pinned in srcs:
                if pinned:
                    jobs.append((doff, arr, None))
                elif pool is not None:
                    for a in range(0, n, _COPY_PIECE):
                        dst = bounce[doff + a:doff + min(n, a + _COPY_PIECE)]
                        jobs.append((doff + a, dst, pool.submit(_copy_into, dst, arr[a:a + _COPY_PIECE])))
                else:
                    jobs.append((doff, bounce[doff:doff + n], (arr, _threads_for(n))))
            with t.cuda.stream(stream), warnings.catch_warnings():
                warnings.simplefilter("ignore", UserWarning)  # chunks are read-only; torch only reads them
                for doff, src_arr, job in jobs:
                    if isinstance(job, tuple):  # copied here, over native threads
                        _copy_into(src_arr, job[0], job[1])
                    elif job is not None:
                        job.result()  # this piece is in the bounce buffer: DMA it now
                    src = t.from_numpy(src_arr)
                    dev[doff:doff + src_arr.size].copy_(src, non_blocking=True)
                    keep.append(src)
        except BaseException:
            for _, _, job in jobs:  # no pool copy may still write the bounce buffer after this
                if job is not None and not isinstance(job, tuple):
                    job.cancel() or job.exception()
            raise
        with t.cuda.stream(stream):
            ready = t.cuda.Event()
            ready.record(stream)
            if bounce is not None:
                staging._bounce_done = ready
    for i, c in enumerate(chunks):
        if isinstance(c, DeviceChunk):
            ptrs[i] = c.data.data_ptr()
            sizes[i] = c.byte_size
            keep.append(c.data)
        elif not isinstance(c, PackedChunk):
            raise TypeError(f"expected PackedChunk or DeviceChunk, got {type(c).__name__}")
    nonempty = [p for p, s in zip(ptrs, sizes) if s]
    base = min(nonempty) if nonempty else 0
    begin = np.array([(p - base) if s else 0 for p, s in zip(ptrs, sizes)], dtype=np.uint64)
    end = begin + np.array(sizes, dtype=np.uint64)
    return StagedBatch(base, begin, end, keep, ready)


def _pattern_args(pattern):
    if pattern is None:
        return None, None, 0, 0, None
    off = np.ascontiguousarray(pattern.offset, dtype=np.int64)
    cnt = np.ascontiguousarray(pattern.count, dtype=np.int64)
    return N.i64p(off), N.i64p(cnt), int(pattern.total_slots), int(pattern.cap), (off, cnt)


# ADAPTIVE takes the register path for the hot bin only when the prior's max-bin share
# reaches this. The path skips a warp's atomics only when all 32 lanes hold an all-hot
# 16-byte vector, P = share^512 (0.60 at 0.999); below that the per-vector test and the
# 768-thread CTAs cost 3-4% (profiles/paper_tables_b200.md Fig. 5: no gain even at 0.99)
SPREAD_BELOW = 0.999


def _with_hints(kind: int, pattern) -> int:
    dom = getattr(pattern, "dominance", None)
    if kind == N.HS_KIND_ADAPTIVE and dom is not None and dom < SPREAD_BELOW:
        kind |= N.HS_KIND_FLAG_SPREAD
    return kind


def kernel_form(kind: int, pattern=None, impl: int = N.HS_IMPL_AUTO) -> str:
    """The device kernel a hs_histogram_batched call with these arguments runs (the
    library's own rule, hs_kernels.cu launch_batch): for labels that must name what ran."""
    if impl == N.HS_IMPL_WARP:
        return "k_warp"
    if impl == N.HS_IMPL_SUBBIN:
        return "k_subbin"
    base = kind & ~(N.HS_KIND_FLAG_SPREAD | N.HS_KIND_FLAG_CHAINED | N.HS_KIND_FLAG_MERGE)
    if base == N.HS_KIND_ADAPTIVE and pattern is not None and not kind & N.HS_KIND_FLAG_SPREAD:
        c = np.asarray(pattern.count)
        top = int(c.max())
        if top > 1 and int((c == top).sum()) == 1:
            return f"k_lane<HOT> (register path for bin {int(np.argmax(c))})"
    return "k_lane (lane-banked core)"


def launch(staged: StagedBatch, kind: int, pattern=None, stream=None, impl: int = N.HS_IMPL_AUTO, out=None,
           staging: Staging | None = None):
    """hs_histogram_batched on ``stream`` (waits for the staging copies first): one
    kernel launch per <= 256 segments and 1 GiB, output written in-kernel through ``staging``'s
    workspace. Returns the device int64 tensor [nseg, 256] (reinterpret as uint64)."""
    t = require_cuda()
    stream = stream or t.cuda.current_stream()
    ws = (staging or default_staging()).workspace(stream)
    if staged.ready is not None:
        stream.wait_event(staged.ready)
    nseg = staged.nseg
    if out is None:
        with t.cuda.stream(stream):
            out = t.empty((max(nseg, 1), BINS), dtype=t.int64, device=t.cuda.current_device())
    off_p, cnt_p, S, cap, keep = _pattern_args(pattern)
    kind = _with_hints(kind, pattern)
    begin = np.ascontiguousarray(staged.begin, dtype=np.uint64)
    end = np.ascontiguousarray(staged.end, dtype=np.uint64)
    status = N.lib().hs_histogram_batched(
        staged.base or None, N.u64p(begin), N.u64p(end), nseg, int(kind), int(impl),
        off_p, cnt_p, S, cap, out.data_ptr(), ws.data_ptr(), ws.numel(), stream.cuda_stream)
    N.check(status, "hs_histogram_batched")
    return out[:nseg] if nseg else out[:0]


def readback(out_dev, staging: Staging | None = None, stream=None, timed: bool = False):
    """D2H of [n, 256] counts (pinned, async) then wait; returns uint64 numpy (a copy).
    With ``timed`` also returns the timing-enabled completion event."""
    t = torch()
    stream = stream or t.cuda.current_stream()
    n = out_dev.shape[0]
    if n == 0:
        res = np.zeros((0, BINS), np.uint64)
        return (res, None) if timed else res
    host = staging.host_out(n) if staging is not None else t.empty(n * BINS, dtype=t.int64, pin_memory=True)
    with t.cuda.stream(stream):
        host.view(n, BINS).copy_(out_dev, non_blocking=True)
        ev = t.cuda.Event(enable_timing=timed)
        ev.record(stream)
    ev.synchronize()
    res = host.numpy().reshape(n, BINS).view(np.uint64).copy()
    return (res, ev) if timed else res


_local = threading.local()


def default_staging() -> Staging:
    """Per-thread staging for the synchronous API (the reference's workers are called
    from several Python threads concurrently, kernels.py:319-327)."""
    s = getattr(_local, "staging", None)
    t = require_cuda()
    if s is None or s.device.index != t.cuda.current_device():
        s = Staging()
        _local.staging = s
    return s


def histograms(chunks: Sequence, kind: int, pattern=None, impl: int = N.HS_IMPL_AUTO) -> np.ndarray:
    """Synchronous batched histograms of host/device chunks -> uint64 [n, 256]."""
    t = require_cuda()
    st = default_staging()
    all_host = bool(chunks) and all(type(c) is PackedChunk for c in chunks)
    if all_host and _pageable_bytes(chunks) >= _COPY_SYNC_MIN:
        # >= 8 MiB of pageable host memory: threaded streaming copies into the bounce
        # buffer and their DMAs beat the driver's pageable copy (16 MiB 0.66 vs 0.78 ms,
        # 64 MiB 1.9 vs 4.7 ms); below that the driver's copy is as fast
        stream = t.cuda.current_stream()
        return _sync_histograms(stage(chunks, st, stream), kind, pattern, impl, st, stream)
    if len(chunks) == 1 and type(chunks[0]) in (PackedChunk, DeviceChunk):
        return _one_histogram(chunks[0], kind, pattern, impl, st)[None, :]
    stream = t.cuda.current_stream()
    if all_host:
        return _host_histograms(chunks, kind, pattern, impl, st, stream)
    if chunks and all(type(c) is DeviceChunk for c in chunks):
        staged = stage(chunks, st, stream)
        return _sync_histograms(staged, kind, pattern, impl, st, stream)
    staged = stage(chunks, st, stream)
    out = launch(staged, kind, pattern, stream, impl, staging=st)
    return readback(out, st, stream)


def _pageable_bytes(chunks) -> int:
    return sum(c.byte_size for c in chunks if c.byte_size and not is_pinned(c.words))


def _raw_stream(index: int) -> int:
    """The current stream's handle on device ``index`` (torch's raw accessor skips the
    Stream object; public API otherwise)."""
    t = torch()
    raw = getattr(t._C, "_cuda_getCurrentRawStream", None)
    return raw(index) if raw is not None else t.cuda.current_stream(index).cuda_stream


def _one_histogram(chunk, kind, pattern, impl, st: "Staging") -> np.ndarray:
    """One chunk (the per-image path of naive_histogram / adaptive_histogram) through
    the blocking native entries with arguments prepared once per staging: on a
    1024x1024 image, marshalling the arguments anew each call cost as much as the
    launch, kernel, readback and wait together (tools/c1_breakdown.py)."""
    stream = _raw_stream(st.device.index)
    kind = int(_with_hints(kind, pattern))
    if type(chunk) is DeviceChunk:
        if chunk._dev != st.device.index:
            raise ValueError(f"DeviceChunk on cuda:{chunk._dev} used on cuda:{st.device.index}")
        one = st.one_call(stream)
        off_p, cnt_p, S, cap = one.pattern_ptrs(pattern)
        n = chunk._n
        one.end[0] = n
        status = N.lib().hs_histogram_sync(chunk._ptr if n else None, one.begin, one.end, 1, kind, int(impl),
                                           off_p, cnt_p, S, cap, one.out_dev_ptr, one.h_out_p, one.ws_ptr,
                                           one.ws_n, stream)
        N.check(status, "hs_histogram_sync")
    else:
        n = chunk.byte_size
        one = st.one_call(stream, max(n, 16))
        off_p, cnt_p, S, cap = one.pattern_ptrs(pattern)
        one.end[0] = n
        one.ptrs[0] = chunk.words.ctypes.data if n else None
        status = N.lib().hs_histogram_host(one.ptrs, one.end, 1, kind, int(impl), off_p, cnt_p, S, cap,
                                           one.dev_ptr, one.dev_n, one.out_dev_ptr, one.h_out_p, one.ws_ptr,
                                           one.ws_n, stream)
        N.check(status, "hs_histogram_host")
    return one.h_np[:BINS].copy()


def _host_histograms(chunks, kind, pattern, impl, st: "Staging", stream) -> np.ndarray:
    """All-host batches in one native call (hs_histogram_host): H2D of every chunk, one
    launch, D2H of the counts and the wait, without a Python round trip in between."""
    import ctypes

    n = len(chunks)
    ptrs = (ctypes.c_void_p * n)(*[c.words.ctypes.data if c.words.size else None for c in chunks])
    sizes = np.array([c.byte_size for c in chunks], dtype=np.uint64)
    need = int(((sizes + 15) // 16 * 16).sum())
    dev = st.device_bytes(max(need, 16))
    out_dev = st.device_out(n)
    h_out = st.host_out(n)  # pinned: the D2H stays a DMA
    ws = st.workspace(stream)
    off_p, cnt_p, S, cap, keep = _pattern_args(pattern)
    status = N.lib().hs_histogram_host(ptrs, N.u64p(sizes), n, int(_with_hints(kind, pattern)), int(impl),
                                       off_p, cnt_p, S, cap, dev.data_ptr(), dev.numel(), out_dev.data_ptr(),
                                       ctypes.cast(h_out.data_ptr(), N._U64P), ws.data_ptr(), ws.numel(),
                                       stream.cuda_stream)
    N.check(status, "hs_histogram_host")
    return h_out.numpy().reshape(n, BINS).view(np.uint64).copy()


def _sync_histograms(staged: StagedBatch, kind, pattern, impl, st: "Staging", stream) -> np.ndarray:
    """Device-resident batches in one native call (hs_histogram_sync)."""
    import ctypes

    n = staged.nseg
    out_dev = st.device_out(n)
    h_out = st.host_out(n)
    ws = st.workspace(stream)
    off_p, cnt_p, S, cap, keep = _pattern_args(pattern)
    begin = np.ascontiguousarray(staged.begin, dtype=np.uint64)
    end = np.ascontiguousarray(staged.end, dtype=np.uint64)
    status = N.lib().hs_histogram_sync(staged.base or None, N.u64p(begin), N.u64p(end), n,
                                       int(_with_hints(kind, pattern)), int(impl), off_p, cnt_p, S, cap,
                                       out_dev.data_ptr(), ctypes.cast(h_out.data_ptr(), N._U64P), ws.data_ptr(),
                                       ws.numel(), stream.cuda_stream)
    N.check(status, "hs_histogram_sync")
    return h_out.numpy().reshape(n, BINS).view(np.uint64).copy()


def histogram_tensor(data, kind: int = N.HS_KIND_NAIVE, pattern=None, impl: int = N.HS_IMPL_AUTO,
                     stream=None, out=None):
    """Histogram of a device-resident uint8 tensor; returns the device int64[256] without
    synchronising (for device pipelines, multi-GPU reduction and benchmarks)."""
    staged = stage([DeviceChunk(data)], None, stream)
    return launch(staged, kind, pattern, stream, impl, out=out)[0]


def group_slots(chunk, pattern, group_size: int, group_count: int, mode: int) -> np.ndarray:
    """Reference-mapping slot totals (hs_group_slots): mode 0 u64[G,S], 1 u64[G,gs,S],
    2 u16[G,S] wrapped."""
    t = require_cuda()
    stream = t.cuda.current_stream()
    staged = stage([chunk], default_staging(), stream)
    if staged.ready is not None:
        stream.wait_event(staged.ready)
    S = int(pattern.total_slots)
    shape = (group_count, group_size, S) if mode == 1 else (group_count, S)
    dtype = t.int16 if mode == 2 else t.int64
    out = t.empty(shape, dtype=dtype, device=t.cuda.current_device())
    off_p, cnt_p, S, cap, keep = _pattern_args(pattern)
    base = staged.base + int(staged.begin[0]) if staged.nbytes else 0
    ws_n = int(N.lib().hs_group_slots_ws_bytes(int(group_size), int(group_count), S, int(mode)))
    ws = t.empty(max(ws_n, 8), dtype=t.uint8, device=t.cuda.current_device())
    status = N.lib().hs_group_slots(base or None, staged.nbytes, int(group_size), int(group_count),
                                    off_p, cnt_p, S, cap, int(mode), out.data_ptr(), ws.data_ptr(), ws_n,
                                    stream.cuda_stream)
    N.check(status, "hs_group_slots")
    host = out.cpu().numpy()
    return host.view(np.uint16) if mode == 2 else host.view(np.uint64)


def ablation_stage(chunk, stage_id: int, pattern, repeats: int | None = None):
    """One genealogy stage (hs_ablation_stage): ``repeats`` back-to-back launches over
    the chunk between two CUDA events on the launch stream (default: enough to stream
    >= 1 GiB, 8..32 launches, all queued before the first runs), so a stage is timed as a
    streaming kernel rather than as one isolated launch's latency or the host's issue
    rate. Returns (seconds per launch, device sink of the last
    launch, histogram-or-None)."""
    t = require_cuda()
    stream = t.cuda.current_stream()
    staged = stage([chunk], default_staging(), stream)
    if staged.ready is not None:
        stream.wait_event(staged.ready)
    sink = t.empty(1, dtype=t.int64, device=t.cuda.current_device())
    out = t.empty(BINS, dtype=t.int64, device=t.cuda.current_device())
    off_p, cnt_p, S, cap, keep = _pattern_args(pattern)
    base = staged.base + int(staged.begin[0]) if staged.nbytes else 0
    n = staged.nbytes
    if repeats is None:  # >= 1 GiB streamed per sample, 8..32 launches
        repeats = int(min(32, max(8, -(-(1 << 30) // max(n, 1)))))
    L = N.lib()

    def once():
        N.check(L.hs_ablation_stage(base or None, n, int(stage_id), off_p, cnt_p, S, cap, sink.data_ptr(),
                                    out.data_ptr(), None, 0, stream.cuda_stream), "hs_ablation_stage")

    once()  # first-launch costs (module load, smem attribute) outside the timing
    a = t.cuda.Event(enable_timing=True)
    b = t.cuda.Event(enable_timing=True)
    # hold the stream (~2 ms) while the host queues every launch, so the events time the
    # launches back to back on the device, not the host's issue rate (a 64 MiB stage
    # launch is ~15 us of device time, about what one Python-issued call takes)
    with t.cuda.stream(stream):
        t.cuda._sleep(4_000_000)
    a.record(stream)
    for _ in range(repeats):
        once()
    b.record(stream)
    b.synchronize()
    seconds = a.elapsed_time(b) / 1e3 / repeats
    dev_sink = int(sink.cpu().numpy().view(np.uint64)[0])
    hist = out.cpu().numpy().view(np.uint64).copy() if stage_id == N.HS_STAGE_FULL else None
    return seconds, dev_sink, hist
