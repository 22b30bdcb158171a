"""Long randomized parity run of the C ABI against torch.bincount (per segment) on a
6 GiB device buffer: random segment counts (1-600), sizes (0 B - 2.5 GiB, word
multiples), overlapping offsets, every impl and kind, hot-bin hints, workspaces for
64/256/1000 segments or none, and the blocking entry with page-locked and pageable
result buffers; round 2: merged outputs (HS_KIND_FLAG_MERGE: one row = the sum of
the segments), chained calls (HS_KIND_FLAG_CHAINED) and bursts of 8-40 calls issued back
to back on one workspace with no synchronisation in between (the rotating call slots).
Runs for SECONDS; prints a progress line every 25 trials and a summary.
usage: python tools/fuzz_long.py [SECONDS]"""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N  # noqa: E402

secs = float(sys.argv[1]) if len(sys.argv) > 1 else 300.0
L = N.lib()
n = 6 << 30
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
# stretches of different distributions (uniform, concentrated, constant, normal)
hs.generate_device(hs.SourceSpec("uniform", 2 << 30, 1), buf[: 2 << 30])
hs.generate_device(hs.SourceSpec("normal", 2 << 30, 2, mean=128.0, sigma=4.0), buf[2 << 30: 4 << 30])
hs.generate_device(hs.SourceSpec("constant", 1 << 30, 3, value=200), buf[4 << 30: 5 << 30])
_r = torch.randint(0, 256, (1 << 30,), dtype=torch.uint8, device="cuda")  # 90% value 7, 10% uniform
_keep = torch.randint(0, 10, (1 << 30,), dtype=torch.uint8, device="cuda") == 0
buf[5 << 30:].copy_(torch.where(_keep, _r, torch.full_like(_r, 7)))
del _r, _keep
st = torch.cuda.current_stream().cuda_stream
rng = np.random.default_rng(int(time.time()))
pats = [hs.compute_binning_pattern(hs.Histogram256(torch.bincount(buf[a:a + (64 << 20)].to(torch.int64),
                                                                  minlength=256).cpu().numpy().astype(np.uint64)))
        for a in (0, 2 << 30, 4 << 30, 5 << 30)]
wss = {k: torch.zeros(int(L.hs_workspace_bytes(k)), dtype=torch.uint8, device="cuda") for k in (64, 256, 1000)}
pinned = torch.empty(600 * 256, dtype=torch.int64).pin_memory()
trials = bytes_total = 0
t_end = time.time() + secs
HEAD = 384  # include/hist256.h HS_WS_HEAD_BYTES: the slots after it are zero between calls


def slots_clean(ws) -> bool:
    return not ws[HEAD:].any().item()


def burst() -> int:
    """8-40 calls back to back on one workspace (small ones rotate through the call
    slots, large ones use the serial slot), then every output checked."""
    ws = wss[int(rng.choice([64, 256, 1000]))]
    calls = []
    for _ in range(int(rng.integers(8, 41))):
        nseg = int(rng.choice([1, 1, 1, 2, 7, 64]))
        sizes = (rng.choice([4, 4096, 1 << 20, 4 << 20, 16 << 20, 40 << 20], size=nseg)
                 + 4 * rng.integers(0, 1 << 12, nseg)).astype(np.int64)
        if rng.random() < 0.05:
            sizes[0] = 4 * rng.integers(1 << 28, 5 << 27)
        starts = 4 * rng.integers(0, (n - sizes) // 4)
        b0, b1 = starts.astype(np.uint64), (starts + sizes).astype(np.uint64)
        kind = int(rng.choice([N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE]))
        if rng.random() < 0.6:
            kind |= N.HS_KIND_FLAG_CHAINED
        merge = rng.random() < 0.3
        if merge:
            kind |= N.HS_KIND_FLAG_MERGE
        pat = pats[rng.integers(0, 4)]
        out = torch.full((nseg, 256), -1, dtype=torch.int64, device="cuda")
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, kind, N.HS_IMPL_AUTO,
                                       N.i64p(pat.offset), N.i64p(pat.count), 960, 8, out.data_ptr(),
                                       ws.data_ptr(), ws.numel(), st), "burst")
        calls.append((b0, b1, merge, out))
    total = 0
    for k, (b0, b1, merge, out) in enumerate(calls):
        want = np.stack([torch.bincount(buf[int(a):int(b)], minlength=256).cpu().numpy().astype(np.uint64)
                         for a, b in zip(b0, b1)])
        got = out.cpu().numpy().view(np.uint64)
        if merge:
            got, want = got[:1], want.sum(axis=0, dtype=np.uint64)[None, :]
        if not np.array_equal(got, want):
            print(f"MISMATCH burst call {k}: nseg {b0.size} merge {merge}", flush=True)
            raise SystemExit(1)
        total += int((b1 - b0).sum())
    if not slots_clean(ws):
        print("MISMATCH burst: workspace slots not left zero", flush=True)
        raise SystemExit(1)
    return total


while time.time() < t_end:
    if rng.random() < 0.3:
        bytes_total += burst()
        trials += 1
        continue
    nseg = int(rng.choice([1, 3, 64, 65, 255, 256, 257, 511, 600]))
    big = rng.random() < 0.15
    scale = [0, 4, 4096, 1 << 20, 16 << 20] + ([1 << 30, (5 << 29)] if big else [])
    sizes = (rng.choice(scale, size=nseg) + 4 * rng.integers(0, 1 << 12, nseg)).astype(np.int64)
    sizes[rng.random(nseg) < 0.1] = 0
    if big:
        sizes[rng.integers(0, nseg)] = 4 * rng.integers(1 << 28, (5 << 29) // 4)
    sizes = np.minimum(sizes, n - 4096)
    starts = 4 * rng.integers(0, (n - sizes) // 4)
    b0, b1 = starts.astype(np.uint64), (starts + sizes).astype(np.uint64)
    impl = int(rng.choice([N.HS_IMPL_AUTO, N.HS_IMPL_LANE, N.HS_IMPL_WARP]))
    kind = int(rng.choice([N.HS_KIND_NAIVE, N.HS_KIND_ADAPTIVE, N.HS_KIND_ADAPTIVE | N.HS_KIND_FLAG_SPREAD]))
    pat = pats[rng.integers(0, 4)]
    ws_key = rng.choice([0, 64, 256, 1000])
    ws = wss.get(int(ws_key))
    entry = rng.choice(["batched", "sync_pinned", "sync_pageable"])
    merge = rng.random() < 0.3
    if merge:
        kind |= N.HS_KIND_FLAG_MERGE
    if entry == "batched" and rng.random() < 0.5:
        kind |= N.HS_KIND_FLAG_CHAINED  # the previous kernel on the stream is ours (or the bincounts)
    out = torch.full((nseg, 256), -1, dtype=torch.int64, device="cuda")
    args = (buf.data_ptr(), N.u64p(b0), N.u64p(b1), nseg, kind, impl, N.i64p(pat.offset), N.i64p(pat.count),
            960, 8, out.data_ptr())
    wsargs = (ws.data_ptr(), ws.numel()) if ws is not None else (None, 0)
    if entry == "batched":
        N.check(L.hs_histogram_batched(*args, *wsargs, st), "batched")
        got = out.cpu().numpy().view(np.uint64)
    elif entry == "sync_pinned":
        h = pinned[: nseg * 256]
        h.fill_(-1)
        N.check(L.hs_histogram_sync(*args, N.ctypes.cast(h.data_ptr(), N._U64P), *wsargs, st), "sync")
        got = h.numpy().view(np.uint64).reshape(nseg, 256).copy()
    else:
        got = np.full((nseg, 256), 7, np.uint64)
        N.check(L.hs_histogram_sync(*args, N.u64p(got), *wsargs, st), "sync")
    want = np.zeros((nseg, 256), np.uint64)
    for s in range(nseg):
        if sizes[s]:
            want[s] = torch.bincount(buf[int(b0[s]):int(b1[s])], minlength=256).cpu().numpy().astype(np.uint64)
    if merge:  # one row: the sum of every segment
        got, want = got[:1], want.sum(axis=0, dtype=np.uint64)[None, :]
    ok = np.array_equal(got, want)
    if ws is not None:
        ok = ok and slots_clean(ws)
    trials += 1
    bytes_total += int(sizes.sum())
    if not ok:
        bad = [s for s in range(nseg) if not np.array_equal(got[s], want[s])]
        print(f"MISMATCH trial {trials}: nseg {nseg} impl {impl} kind {kind:#x} ws {ws_key} entry {entry} "
              f"bad segments {bad[:10]} sizes {[int(sizes[s]) for s in bad[:5]]}", flush=True)
        raise SystemExit(1)
    if trials % 25 == 0:
        print(f"{trials} trials ok, {bytes_total / (1 << 30):.1f} GiB counted", flush=True)
print(f"fuzz ok: {trials} trials, {bytes_total / (1 << 30):.1f} GiB counted, {secs:.0f} s", flush=True)
