#!/usr/bin/env python
"""Benchmark of the 256-bin histogram hot path (BASELINE.json metric: input GB/s at
1/2/4/8 B200 vs the HBM roofline; CPU reference GB/s beside it).

Headline workload = BASELINE configs[4] (C5): a 64 GiB device-resident synthetic uint8
stream (uniform splitmix64 bytes, bit-exact with the reference generator), sharded by
contiguous byte range across the ranks (the group_ranges rule, kernels.py:311-316) --
strong scaling: 64 GiB in total at every N. One step = each rank counts its whole
shard in ONE library call (distributed.ShardedHistogram: chained <= 1 GiB k_lane
launches, segments merged into one uint64[256] in the ticketed epilogue) and the 256
counts are joined by one NCCL all_reduce (N > 1). Inputs are 64/N GiB per GPU, far
larger than the 126 MB L2, so no flush is needed between steps.

  value         64 GiB x steps / max-over-ranks device time (CUDA events)
  roofline      the k_lane launches of the timed region themselves: bytes per launch /
                (timed region / launches), against MEASURED_PEAKS hbm_gbs
  e2e           the same 64 GiB stream from pinned HOST memory through the public
                streaming API (run_pipeline, 16 MiB chunks, batches of 16, the reference
                switch policy): every H2D and every 2 KiB readback in the timed region
  cpu_baseline  the reference's own CPU path (numba naive_histogram from baseline/_ref,
                WorkerGroupConfig(32, host cores)) on a bounded sample of the stream,
                with the oracle's C port beside it
  extras        C1 (1024x1024 image), C2 (X-ray normal streams, AHist + CPU pattern),
                C3 (degenerate switch stream on the device engine), C4 (16 GiB
                host-streamed mixed stream), sustained rate under the power cap

Parity inside the run: the last step's 64 GiB counts equal an independent device count
(torch.bincount, summed over 1 GiB pieces) bin for bin, two sampled 1 GiB shards equal
the oracle's host count bin for bin, and the e2e run's accumulator equals the device
counts of the same bytes bin for bin.

``--impl reference`` times the reference CPU implementation only (rank 0) on the same
config and metric.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import sys
import threading
import time
from pathlib import Path

import numpy as np

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

GiB = 1 << 30
CHUNK = 16 << 20
READ_ONLY_CEILING_GBS = 6973.3  # profiles/r1_mapping.txt (grid-stride read, 64 GiB)
BASE_SEED = 0x1011_0235
C5_BYTES = 64 << 30
C5_SEED = BASE_SEED ^ 0xC5
METRIC = "256-bin histogram input GB/s at 1/2/4/8 B200 vs HBM roofline; CPU ref GB/s"
WORKLOAD = ("C5 (BASELINE configs[4]): 64 GiB device-resident synthetic uint8 stream (uniform splitmix64), "
            "sharded by contiguous byte range across the GPUs, NCCL all_reduce of the 256-count partials")
REF_SAMPLE_CHUNKS = 16  # reference arm: 16 x 16 MiB = 256 MiB of the stream per step
REF_POOL_CHUNKS = 64    # ... drawn in turn from the first 1 GiB of the stream (>> host caches)


def peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    try:
        d = json.loads(p.read_text())
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs)"
    except (OSError, ValueError, KeyError, TypeError):
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_cores() -> int:
    try:
        return len(os.sched_getaffinity(0))
    except AttributeError:  # pragma: no cover
        return os.cpu_count() or 1


def config_dict(world: int) -> dict:
    """The workload named identically by both arms."""
    return {"workload": WORKLOAD, "total_bytes": C5_BYTES, "bytes_per_gpu": C5_BYTES // max(world, 1),
            "distribution": "uniform", "seed": C5_SEED, "kernel": "naive (the reference switch policy's choice "
            "for uniform data: degeneracy 0.004 < 0.45)", "parallelism": f"shard{world}" + ("+nccl_allreduce" if
                                                                                           world > 1 else ""),
            "l2": "inputs 64/N GiB per GPU >> 126 MB L2 (no flush needed)"}


# ----------------------------------------------------------------------- clocks
class ClockSampler:
    """NVML SM clock, memory clock, power and clock-event reasons, sampled every ~5 ms by
    a thread started ahead of the timed region (its first NVML calls can be slow right
    after an idle period); the summary keeps the samples taken inside the window that
    mark_start()/mark_end() bracket."""

    NAMES = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
             0x10: "sync_boost", 0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown",
             0x80: "hw_power_brake_slowdown", 0x100: "display_clock_setting"}

    def __init__(self, index: int):
        self.rows: list[tuple] = []  # (t, sm_mhz, mem_mhz, power_w, reasons)
        self.max_mhz = None
        self.t0 = self.t1 = None
        self._stop = threading.Event()
        try:
            import pynvml

            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
        except Exception:  # pragma: no cover - NVML missing
            self.nv = None

    def _run(self):
        nv, h = self.nv, self.h
        while not self._stop.is_set():
            try:
                self.rows.append((time.perf_counter(), nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_SM),
                                  nv.nvmlDeviceGetClockInfo(h, nv.NVML_CLOCK_MEM), nv.nvmlDeviceGetPowerUsage(h) / 1000.0,
                                  nv.nvmlDeviceGetCurrentClocksEventReasons(h)))
            except Exception:
                pass
            time.sleep(0.005)

    def __enter__(self):
        if self.nv is not None:
            self._t = threading.Thread(target=self._run, daemon=True)
            self._t.start()
        return self

    def mark_start(self):
        self.t0 = time.perf_counter()

    def mark_end(self):
        self.t1 = time.perf_counter()

    def __exit__(self, *exc):
        self._stop.set()
        if self.nv is not None:
            self._t.join()

    def summary(self):
        if self.nv is None or not self.rows:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unavailable"]}
        t0 = self.t0 if self.t0 is not None else self.rows[0][0]
        t1 = self.t1 if self.t1 is not None else self.rows[-1][0]
        inside = [r for r in self.rows if t0 <= r[0] <= t1]
        if not inside:  # a sample could not be taken inside: the nearest one on each side
            before = [r for r in self.rows if r[0] < t0]
            after = [r for r in self.rows if r[0] > t1]
            inside = before[-1:] + after[:1]
        bits = 0
        for r in inside:
            bits |= r[4]
        reasons = [n for bit, n in self.NAMES.items() if bits & bit and bit != 0x1]
        return {"sm_mhz": float(statistics.median(r[1] for r in inside)), "sm_max_mhz": self.max_mhz,
                "reasons": reasons, "samples": len(inside),
                "mem_mhz": float(statistics.median(r[2] for r in inside)),
                "power_w_max": round(max(r[3] for r in inside), 1)}


# ----------------------------------------------------------------------- distributed
def relaunch_under_torchrun(n: int, argv) -> int:
    """`python bench.py --gpus N` without a launcher: re-run under torch.distributed.run
    with one process per GPU (rendezvous on 127.0.0.1), as the driver launches it."""
    import socket
    import subprocess

    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        port = s.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", "--master-port", str(port), str(Path(__file__).resolve()),
           *(sys.argv[1:] if argv is None else argv)]
    return subprocess.call(cmd)


def _dist_on() -> bool:
    import torch.distributed as dist

    return dist.is_available() and dist.is_initialized()


def barrier(world=None):
    if _dist_on():
        import torch.distributed as dist

        dist.barrier()


def max_over_ranks(x: float, world: int) -> float:
    if not _dist_on():
        return x
    import torch
    import torch.distributed as dist

    dev = "cuda" if dist.get_backend() == "nccl" else "cpu"  # gloo in the CPU tests
    t = torch.tensor([x], dtype=torch.float64, device=dev)
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


# ----------------------------------------------------------------------- CPU reference
def _ref_module():
    """The unmodified reference from baseline/_ref (pip-installed there), or None."""
    ref = ROOT / "baseline" / "_ref"
    if not (ref / "histostream" / "__init__.py").exists():
        return None
    os.environ.setdefault("NUMBA_CACHE_DIR", str(Path("/tmp") / "hs_numba_cache"))
    if str(ref) not in sys.path:
        sys.path.insert(0, str(ref))
    try:
        import histostream
        from histostream import kernels as K

        if Path(histostream.__file__).resolve().parent != (ref / "histostream").resolve():
            return None
        return K
    except Exception as exc:  # pragma: no cover
        print(f"[bench] reference import failed: {exc}", file=sys.stderr)
        return None


def c5_sample_words(nchunks: int, first_chunk: int = 0) -> list[np.ndarray]:
    """Chunks [first, first+n) of 16 MiB of the C5 stream as uint32 words, generated on
    the host with the oracle's splitmix64 restatement (the same bytes as the device
    generator and as the reference's generate())."""
    from oracle import oracle as O

    lib = O.lib()
    out = []
    for c in range(first_chunk, first_chunk + nchunks):
        # uniform pixel i = byte (i & 7) of splitmix output (i >> 3); a chunk starting at
        # pixel p = c * CHUNK is the tail of a longer generation, so generate from 0 of a
        # stream whose state is advanced: the C helper fills from pixel 0, hence a slice
        buf = np.empty(CHUNK, np.uint8)
        _fill_uniform_at(lib, buf, C5_SEED, c * CHUNK)
        out.append(buf.view(np.uint32))
    return out


def _fill_uniform_at(lib, buf: np.ndarray, seed: int, first: int) -> None:
    """Pixels [first, first + len) of the uniform stream of ``seed`` (datagen.py:98-112:
    pixel i is byte i & 7 of splitmix64 output i >> 3, state = seed + (k + 1) * golden)."""
    assert first % 8 == 0 and buf.size % 8 == 0
    k0 = first >> 3
    golden = 0x9E3779B97F4A7C15
    mask = (1 << 64) - 1
    # output k of the stream seeded s equals output k - k0 of the stream seeded
    # s + k0 * golden (the state is a counter)
    import ctypes

    lib.or_fill_uniform(buf.ctypes.data_as(ctypes.c_void_p), buf.size, (seed + k0 * golden) & mask)


def cpu_reference_run(seconds: float, chunks_per_step: int | None = None, steps: int | None = None,
                      warmup: int = 1):
    """The reference's CPU path (numba naive_histogram, WorkerGroupConfig(32, cores)) on
    16 MiB chunks of the C5 stream, each checked against the oracle. Either for about
    ``seconds`` of CPU work, or ``steps`` steps of ``chunks_per_step`` chunks. Returns a
    dict (value GB/s, per-step seconds, cores, kind, sample) or None without baseline/_ref."""
    K = _ref_module()
    if K is None:
        return None
    from histostream.core import PackedChunk as RefChunk
    from oracle import oracle as O

    cores = host_cores()
    cfg = K.WorkerGroupConfig(32, cores)
    pool = c5_sample_words(REF_POOL_CHUNKS)
    chunks = [RefChunk(w) for w in pool]
    for _ in range(warmup):  # numba JIT + first-touch outside the timing
        K.naive_histogram(chunks[0], cfg)
    times, done = [], 0
    nsteps = steps if steps is not None else 10 ** 9
    per = chunks_per_step or 1
    t_all = time.perf_counter()
    for s in range(nsteps):
        t0 = time.perf_counter()
        hs_ = [K.naive_histogram(chunks[(s * per + j) % len(chunks)], cfg) for j in range(per)]
        times.append(time.perf_counter() - t0)
        done += per
        if s == 0:
            for j, h in enumerate(hs_):  # the reference arm's own parity against the oracle
                w = pool[(s * per + j) % len(pool)]
                assert np.array_equal(np.asarray(h.counts), O.histogram(w.view(np.uint8))), "reference != oracle"
        if steps is None and time.perf_counter() - t_all >= seconds:
            break
    total = sum(times)
    return {"value": round(done * CHUNK / total / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "reference",
            "sample": f"{done} x 16 MiB chunks ({done * CHUNK / GiB:.2f} GiB) taken in turn from the first "
                      f"{len(pool) * CHUNK / GiB:.0f} GiB of the C5 stream, unmodified reference numba naive_histogram "
                      f"from baseline/_ref, "
                      f"WorkerGroupConfig(32, {cores})",
            "step_seconds": times}


def cpu_reference_paths(seconds: float):
    """The reference's other two CPU entry points on the same 16 MiB C5 chunks (SURVEY
    §8(d)): the serial oracle reference_histogram (kernels.py:330-333) and
    adaptive_histogram (kernels.py:349-384, pattern from the previous chunk's histogram,
    WorkerGroupConfig(32, cores)), each for about ``seconds`` and checked against the
    oracle. Returns {name: {value GB/s, chunks}} or None without baseline/_ref."""
    K = _ref_module()
    if K is None:
        return None
    from histostream.core import PackedChunk as RefChunk
    from histostream.pattern import compute_binning_pattern
    from oracle import oracle as O

    cores = host_cores()
    cfg = K.WorkerGroupConfig(32, cores)
    pool = c5_sample_words(4)
    chunks = [RefChunk(w) for w in pool]
    pattern = compute_binning_pattern(K.reference_histogram(chunks[-1]))
    runs = {"reference_histogram": lambda c: K.reference_histogram(c),
            "adaptive_histogram": lambda c: K.adaptive_histogram(c, pattern, cfg)}
    out = {}
    for name, fn in runs.items():
        fn(chunks[0])  # JIT / first touch
        done, t0 = 0, time.perf_counter()
        while True:
            h = fn(chunks[done % len(chunks)])
            if done < len(chunks):
                assert np.array_equal(np.asarray(h.counts), O.histogram(pool[done].view(np.uint8))), name
            done += 1
            if time.perf_counter() - t0 >= seconds:
                break
        dt = time.perf_counter() - t0
        out[name] = {"value": round(done * CHUNK / dt / 1e9, 4), "unit": "GB/s", "chunks": done,
                     "cores": 1 if name == "reference_histogram" else cores}
    return out


def cpu_port_run(seconds: float):
    """The oracle's C restatement of the reference's naive worker (kernels.py:97-130,
    arbitration loop), one group thread per host core, on the same sample."""
    from oracle import oracle as O

    cores = host_cores()
    pool = c5_sample_words(REF_POOL_CHUNKS)
    done, elapsed = 0, 0.0
    O.naive_histogram(pool[0], 32, cores)
    while elapsed < seconds:
        w = pool[done % len(pool)]
        t0 = time.perf_counter()
        O.naive_histogram(w, 32, cores)
        elapsed += time.perf_counter() - t0
        done += 1
    return {"value": round(done * CHUNK / elapsed / 1e9, 4), "unit": "GB/s", "cores": cores, "kind": "port",
            "sample": f"{done} x 16 MiB chunks taken in turn from the first {len(pool) * CHUNK / GiB:.0f} GiB of the "
                      f"C5 stream, oracle C naive worker (arbitration loop), "
                      f"WorkerGroupConfig(32, {cores})"}


def run_reference(args):
    """--impl reference: the reference's own CPU path on the box's host cores, rank 0
    only, same metric/config; each step one bounded sample (256 MiB) of the C5 stream."""
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    world = int(os.environ.get("WORLD_SIZE", str(args.gpus)))
    res = cpu_reference_run(0, chunks_per_step=REF_SAMPLE_CHUNKS, steps=args.steps, warmup=1)
    kind = "reference"
    if res is None:  # baseline/_ref missing: the oracle port
        kind = "port"
        res = cpu_port_run(10.0)
        res["step_seconds"] = [REF_SAMPLE_CHUNKS * CHUNK / (res["value"] * 1e9)] * args.steps
    value = res["value"]
    ms = statistics.mean(res["step_seconds"]) * 1e3
    line = {
        "impl": "reference", "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": round(ms, 3), "higher_is_better": True,
        "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
        "config": config_dict(world),
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": res["cores"], "kind": kind,
                         "sample": res["sample"] + f"; each step {REF_SAMPLE_CHUNKS} chunks (256 MiB)"},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ----------------------------------------------------------------------- device arm
def main(argv=None):
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=20)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--e2e-steps", type=int, default=2)
    ap.add_argument("--cpu-seconds", type=float, default=10.0)
    ap.add_argument("--sustain-seconds", type=float, default=2.0)
    ap.add_argument("--settle-seconds", type=float, default=1.0)
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-extras", action="store_true")
    args = ap.parse_args(argv)
    args.warmup = max(args.warmup, 3)
    if args.gpus > 1 and "RANK" not in os.environ:
        return relaunch_under_torchrun(args.gpus, argv)
    if args.impl == "reference":
        return run_reference(args)

    import torch

    import paper_1011_0235_b200 as hs
    from paper_1011_0235_b200 import _native as N
    from paper_1011_0235_b200 import distributed as dist_api

    if "RANK" in os.environ:
        rank, world, local = dist_api.init_process_group("nccl")  # logs the communicator (rank/world)
    else:
        rank, world, local = 0, 1, 0
    dev = torch.device("cuda", local)
    torch.cuda.set_device(dev)
    stream = torch.cuda.current_stream()
    N.lib()

    # ---- inputs: this rank's contiguous shard of the 64 GiB stream, generated in HBM
    lo, hi = dist_api.shard_range(C5_BYTES, rank, world)
    shard = torch.empty(hi - lo, dtype=torch.uint8, device=dev)
    hs.generate_device(hs.SourceSpec("uniform", C5_BYTES, C5_SEED), shard, first_pixel=lo)
    torch.cuda.synchronize()
    sh = dist_api.ShardedHistogram()
    launches_per_step = -(-(hi - lo) // GiB)  # the library cuts a call into <= 1 GiB k_lane launches
    dist_on = _dist_on()

    def step():
        # one merged library call over the shard (chained: the stream's previous kernel
        # is our own launch over bytes generated long before), then the 2 KiB allreduce
        sh.count(shard, chained=True)
        if dist_on:
            sh.allreduce()

    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    # The timed region starts from an idle GPU: this kernel draws the board's 1000 W limit
    # within ~50 ms, so whatever ran just before would decide how much of
    # the region runs power-capped.
    clocks = ClockSampler(local).__enter__()
    time.sleep(args.settle_seconds)
    barrier()
    torch.cuda.synchronize()
    t0 = torch.cuda.Event(enable_timing=True)
    t1 = torch.cuda.Event(enable_timing=True)
    try:
        clocks.mark_start()
        t0.record(stream)
        h0 = time.perf_counter()
        for _ in range(args.steps):
            step()
        host_issue_ms = (time.perf_counter() - h0) * 1e3 / args.steps
        t1.record(stream)
        torch.cuda.synchronize()
        clocks.mark_end()
    finally:
        clocks.__exit__(None, None, None)
    local_ms = t0.elapsed_time(t1)
    barrier()
    elapsed_ms = max_over_ranks(local_ms, world)
    value = C5_BYTES * args.steps / (elapsed_ms / 1e3) / 1e9

    # ---- parity of the last step, bin for bin
    counts = sh.result().counts
    assert int(counts.sum(dtype=np.uint64)) == C5_BYTES, "C5 total"
    independent = torch.zeros(256, dtype=torch.int64, device=dev)
    for a in range(0, hi - lo, GiB):  # torch's own bincount, an independent device count
        independent += torch.bincount(shard[a:min(a + GiB, hi - lo)], minlength=256)
    dist_api.allreduce_counts(independent)
    assert np.array_equal(counts, dist_api.as_uint64(independent)), "C5 counts != torch.bincount"
    parity = {"total_equals_stream_bytes": True, "bins_equal_torch_bincount_64GiB": True}
    if rank == 0:
        from oracle import oracle as O

        picks = sorted({0, (hi - lo) // GiB // 2 * GiB, (hi - lo) - GiB})
        for a in picks[:3]:  # sampled 1 GiB shards: our kernel vs the oracle's host count
            b0, b1 = np.array([a], np.uint64), np.array([a + GiB], np.uint64)
            out = torch.empty((1, 256), dtype=torch.int64, device=dev)
            N.check(N.lib().hs_histogram_batched(shard.data_ptr(), N.u64p(b0), N.u64p(b1), 1, N.HS_KIND_NAIVE,
                                                 N.HS_IMPL_AUTO, None, None, 0, 0, out.data_ptr(), None, 0,
                                                 stream.cuda_stream), "sample")
            want = O.histogram_mt(shard[a:a + GiB].cpu().numpy())
            assert np.array_equal(out[0].cpu().numpy().view(np.uint64), want), f"sampled shard at {a}"
        parity["sampled_1GiB_shards_equal_oracle"] = [int(lo + a) for a in picks[:3]]
        if lo == 0:  # the reference arm's sample is these same bytes
            assert np.array_equal(c5_sample_words(1)[0].view(np.uint8), shard[:CHUNK].cpu().numpy())
            parity["reference_arm_sample_equals_stream_head"] = True

    # ---- roofline: the timed k_lane launches themselves
    peak, peak_src = peaks()
    n_launch = args.steps * launches_per_step
    launch_ms = local_ms / n_launch
    per_launch_bytes = (hi - lo) / launches_per_step
    achieved = per_launch_bytes / (launch_ms / 1e3) / 1e9
    traffic = None
    tf = ROOT / "profiles" / "traffic.json"
    if tf.exists():
        try:
            traffic = json.loads(tf.read_text()).get("k_lane_bytes_per_launch")
        except Exception:
            traffic = None
    roofline = {"bound": "hbm", "achieved": round(achieved, 1), "peak": peak, "unit": "GB/s",
                "frac": round(achieved / peak, 4), "traffic": traffic, "peak_source": peak_src,
                "kernel": "k_lane<2,false> (NAIVE, merged output), 1 GiB per launch",
                "algorithmic_bytes_per_launch": int(per_launch_bytes),
                "achieved_method": (f"rank-0 timed region / {n_launch} launches ({launches_per_step} chained 1 GiB "
                                    "launches per step, back to back; k_lane is >99% of the step's GPU time, "
                                    "profiles/r2end_launches_summary.txt)"),
                "avg_launch_ms": round(launch_ms, 5),
                # a 1-byte-read kernel's ceiling: a read-only grid-stride stream reaches this
                "read_only_ceiling_gbs": READ_ONLY_CEILING_GBS,
                "frac_of_read_only_ceiling": round(achieved / READ_ONLY_CEILING_GBS, 4)}

    # ---- sustained: the same step for ~2 s (the power controller's settled clock)
    sustained = None
    if args.sustain_seconds > 0:
        n_sus = max(1, int(args.sustain_seconds * 1e3 / (elapsed_ms / args.steps)))
        barrier()
        torch.cuda.synchronize()
        s0e, s1e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with ClockSampler(local) as sus_clocks:
            sus_clocks.mark_start()
            s0e.record(stream)
            for _ in range(n_sus):
                step()
            s1e.record(stream)
            torch.cuda.synchronize()
            sus_clocks.mark_end()
        sus_ms = max_over_ranks(s0e.elapsed_time(s1e), world)
        sustained = {"steps": n_sus, "seconds": round(sus_ms / 1e3, 3),
                     "value": round(C5_BYTES * n_sus / (sus_ms / 1e3) / 1e9, 2), "unit": "GB/s",
                     "clocks": sus_clocks.summary()}

    # ---- e2e: the same stream from pinned host memory through run_pipeline
    e2e, pinned = None, None
    if not args.no_e2e:
        e2e, pinned = e2e_run(hs, torch, rank, world, lo, hi, shard, sh, args.e2e_steps)

    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu:  # the CPU baseline is an N=1 measurement
        ref = cpu_reference_run(args.cpu_seconds)
        port = cpu_port_run(args.cpu_seconds)
        if ref is not None:
            ref.pop("step_seconds", None)
            cpu = dict(ref, port=port)
            others = cpu_reference_paths(max(2.0, args.cpu_seconds / 3))
            if others:
                cpu["other_reference_paths"] = others
        else:
            cpu = port

    extra = {}
    del shard
    torch.cuda.empty_cache()
    if rank == 0 and not args.no_extras:
        import bench_extras as X

        extra["c2_xray_normal"] = X.c2_normal_streams(hs, N, torch, dev)
        extra["c1_image_1024x1024"] = X.c1_image(hs, N, torch, dev)
        extra["c3_switch_stream"] = X.c3_switch(hs, torch, dev)
        if pinned is not None:
            extra["c4_host_streamed_mixed"] = X.c4_mixed(hs, torch, dev, pinned)
            extra["host_small_chunks_reference_default"] = X.host_small_chunks(hs, torch, dev, pinned)
    del pinned

    if rank == 0:
        line = {
            "metric": METRIC, "value": round(value, 2), "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": round(elapsed_ms / args.steps, 4), "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "u8", "data": "synthetic",
            "config": config_dict(world),  # identical to the reference arm's
            "timed_region_start": f"idle GPU ({args.settle_seconds:g} s settle)",
            "roofline": roofline,
            "cpu_baseline": cpu,
            "e2e": e2e,
            "gpu_launches": n_launch,  # k_lane launches in the timed region (plus world>1: NCCL allreduces)
            "clocks": clocks.summary(),
            "parity": parity,
            "sustained": sustained,
            "host_issue_ms_per_step": round(host_issue_ms, 4),
            **extra,
        }
        print(json.dumps(line), flush=True)
    if _dist_on():
        torch.distributed.destroy_process_group()
    return 0


E2E_BATCH = 16  # chunks per run_pipeline iteration (256 MiB): 0.97-0.98 of the link in round 1


def e2e_run(hs, torch, rank, world, lo, hi, shard, sh, steps):
    """The C5 stream end to end through the public streaming API: this rank's shard in
    pinned host memory (setup, untimed: page-locking 64 GiB takes tens of seconds), then
    run_pipeline over 16 MiB chunks in batches of 16 with the reference switch policy --
    the producer H2D-copies batch i+1 on the copy stream while the consumer's launch for
    batch i runs, and every batch's counts come back (2 KiB per chunk). Wall time of
    whole run_pipeline calls, max over ranks. The accumulator must equal the device
    counts of the same bytes, bin for bin. Returns (e2e dict, pinned buffer)."""
    from paper_1011_0235_b200 import device as D

    n = hi - lo
    t_pin = time.perf_counter()
    pinned = D.pinned_bytes(n)
    pin_s = time.perf_counter() - t_pin
    host = torch.from_numpy(pinned)
    for a in range(0, n, GiB):  # the stream's bytes, device -> host once (setup)
        host[a:min(a + GiB, n)].copy_(shard[a:min(a + GiB, n)])
    torch.cuda.synchronize()
    words = pinned.view(np.uint32)
    cw = CHUNK // 4
    chunks = [hs.PackedChunk(words[c * cw:(c + 1) * cw]) for c in range(n // CHUNK)]
    iters = len(chunks) // E2E_BATCH
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=CHUNK, batch_size=E2E_BATCH, window_size=8)
    policy = hs.SwitchPolicy()

    def src():
        for i in range(iters):
            yield chunks[i * E2E_BATCH:(i + 1) * E2E_BATCH]

    hs.run_pipeline(src(), cfg, policy)  # warm-up pass
    torch.cuda.synchronize()
    barrier()
    times = []
    for _ in range(steps):
        t0 = time.perf_counter()
        acc, _, rep, log = hs.run_pipeline(src(), cfg, policy)
        times.append(time.perf_counter() - t0)
    dt = max_over_ranks(float(np.median(times)), world)
    sh.count(shard)  # this rank's device counts of the same bytes
    assert np.array_equal(acc.running.counts, sh.result().counts), "e2e accumulator != device counts"
    link = []
    dst = torch.empty(GiB, dtype=torch.uint8, device="cuda")
    for _ in range(3):  # copy-only link bandwidth of the same pinned buffer
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        dst.copy_(host[:GiB], non_blocking=True)
        b.record()
        b.synchronize()
        link.append(GiB / (a.elapsed_time(b) / 1e3) / 1e9)
    del dst
    value = C5_BYTES / dt / 1e9
    kinds = [k.value for k in log]
    return ({"value": round(value, 3), "unit": "GB/s", "h2d_bytes_per_step": n, "d2h_bytes_per_step":
             len(chunks) * 2048, "api": "paper_1011_0235_b200.run_pipeline (pinned host chunks, 16 MiB, batch 16)",
             "workload": "C5 from host memory: each rank streams its shard over its own PCIe link",
             "per_rank_gbs": round(n / dt / 1e9, 3), "h2d_link_gbs": round(max(link), 2),
             "frac_of_link": round(n / dt / 1e9 / max(link), 4), "iterations": len(kinds),
             "adaptive_iterations": kinds.count("adaptive"), "pin_setup_s": round(pin_s, 1),
             "parity": "accumulator == device counts of the shard, bin for bin"}, pinned)


if __name__ == "__main__":
    raise SystemExit(main())
