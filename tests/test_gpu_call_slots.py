"""GPU parity of the workspace call slots (include/hist256.h HS_WS_SLOTS): consecutive
ticketed calls on one workspace count into rotating slots, so a call's CTAs flush while
its predecessor is still draining and only the CTAs that store the output wait for it.

Checked here, all against the oracle's counts and with the workspace clean afterwards:
- long unsynchronised sequences of random calls on one stream and one workspace --
  single and multi-segment, merged and per-segment, tiny (one CTA) to > 1 GiB
  (several chained launches per call), groups larger than the workspace's rows,
  ADAPTIVE register path, chained and waiting first launches;
- many calls writing the SAME output buffer: the last call's counts win;
- a torch kernel that reads a call's output right behind it on the stream;
- the call counter and drain counts of the header after N calls;
- waiting (unflagged) calls take the serial slot, interleaved with chained ones.
"""
import numpy as np
import pytest
from conftest import WS_DRAINED, WS_HEAD_BYTES, ws_clean

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N

pytestmark = pytest.mark.gpu

SLOTS = 4  # HS_WS_SLOTS


def _issue(L, torch, buf, b0, b1, kind, ws, out, pat=None):
    off = N.i64p(pat.offset) if pat is not None else None
    cnt = N.i64p(pat.count) if pat is not None else None
    S, cap = (int(pat.total_slots), int(pat.cap)) if pat is not None else (0, 0)
    N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(np.asarray(b0, np.uint64)),
                                   N.u64p(np.asarray(b1, np.uint64)), len(b0), kind, N.HS_IMPL_AUTO, off, cnt,
                                   S, cap, out.data_ptr(), ws.data_ptr(), ws.numel(),
                                   torch.cuda.current_stream().cuda_stream), "hs_histogram_batched")


@pytest.fixture(scope="module")
def stream_data(cuda):
    torch = cuda
    n = (1 << 30) + (96 << 20)
    buf = torch.empty(n, dtype=torch.uint8, device="cuda")
    hs.generate_device(hs.SourceSpec("normal", n, 41, mean=128.0, sigma=40.0), buf)
    buf[: 8 << 20] = 201  # a degenerate head for the ADAPTIVE register path
    return torch, buf, buf.cpu().numpy()


def _counts(host, a, b):
    from oracle import oracle as O

    return O.histogram_mt(host[a:b]) if b - a > (64 << 20) else O.histogram(host[a:b])


@pytest.mark.parametrize("seed", range(3))
def test_unsynchronised_call_sequences(stream_data, seed):
    torch, buf, host = stream_data
    L = N.lib()
    rng = np.random.default_rng(900 + seed)
    rows = 64 if seed == 0 else 256
    ws = torch.zeros(int(L.hs_workspace_bytes(rows)), dtype=torch.uint8, device="cuda")
    pat = hs.compute_binning_pattern(hs.Histogram256(_counts(host, 0, 1 << 20)))
    n = host.size
    calls = []
    for k in range(160):
        shape = rng.choice(["tiny", "small", "mid", "multi", "many", "huge"], p=[.25, .25, .2, .15, .1, .05])
        if shape == "tiny":
            sizes = 4 * rng.integers(1, 4096, 1)
        elif shape == "small":
            sizes = np.array([int(rng.choice([1, 4, 16])) << 20])
        elif shape == "mid":
            sizes = 4 * rng.integers(1 << 20, 24 << 20, 1)
        elif shape == "multi":
            sizes = 4 * rng.integers(0, 1 << 18, int(rng.integers(2, 40)))
        elif shape == "many":
            sizes = 4 * rng.integers(0, 1 << 14, int(rng.integers(65, 300)))
        else:
            sizes = np.array([(1 << 30) + (int(rng.integers(1, 64)) << 20)])
        starts = 4 * rng.integers(0, (n - int(sizes.max()) - 8) // 4, sizes.size)
        b0 = starts.astype(np.uint64)
        b1 = (starts + sizes).astype(np.uint64)
        merge = bool(rng.random() < 0.4) or shape == "huge"
        kind = N.HS_KIND_ADAPTIVE if rng.random() < 0.3 else N.HS_KIND_NAIVE
        if rng.random() < 0.5:
            kind |= N.HS_KIND_FLAG_CHAINED
        if merge:
            kind |= N.HS_KIND_FLAG_MERGE
        out = torch.full((1 if merge else sizes.size, 256), -1, dtype=torch.int64, device="cuda")
        _issue(L, torch, buf, b0, b1, kind, ws, out, pat if (kind & 0xff) == N.HS_KIND_ADAPTIVE else None)
        calls.append((b0, b1, merge, out))
    torch.cuda.synchronize()
    for k, (b0, b1, merge, out) in enumerate(calls):
        rows_ = [_counts(host, int(a), int(b)) for a, b in zip(b0, b1)]
        want = np.sum(rows_, axis=0).reshape(1, 256) if merge else np.stack(rows_)
        got = out.cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), (seed, k, b0.size, merge)
    assert ws_clean(ws)
    head = ws[:WS_HEAD_BYTES].cpu().numpy()
    calls_ctr = int(head[:8].view(np.uint64)[0])
    drained = head[WS_DRAINED].view(np.uint32)
    assert calls_ctr % 4096 == 0
    assert int(drained.sum()) == calls_ctr // 4096  # every call released its slot


def test_same_output_last_call_wins(stream_data):
    torch, buf, host = stream_data
    L = N.lib()
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    out = torch.full((1, 256), -1, dtype=torch.int64, device="cuda")
    rng = np.random.default_rng(5)
    for rep in range(20):
        last = None
        for k in range(int(rng.integers(2, 24))):
            size = 4 * int(rng.integers(1, 4 << 20))
            a = 4 * int(rng.integers(0, (host.size - size) // 4))
            _issue(L, torch, buf, [a], [a + size], N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, ws, out)
            last = (a, a + size)
        torch.cuda.synchronize()
        assert np.array_equal(out.cpu().numpy().view(np.uint64)[0], _counts(host, *last)), rep
    assert ws_clean(ws)


def test_reader_behind_call_sees_final_counts(stream_data):
    torch, buf, host = stream_data
    L = N.lib()
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    outs = torch.zeros((64, 256), dtype=torch.int64, device="cuda")
    sums = torch.zeros(64, dtype=torch.int64, device="cuda")
    sizes = [4 * (1 + 97 * k) for k in range(32)] + [(k + 1) << 18 for k in range(32)]
    for k, size in enumerate(sizes):
        _issue(L, torch, buf, [4096 * k], [4096 * k + size], N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, ws, outs[k:k + 1])
        sums[k] = outs[k].sum()  # a torch kernel right behind the call on the stream
    torch.cuda.synchronize()
    assert sums.cpu().tolist() == sizes
    assert ws_clean(ws)


def test_slot_rotation_counts(stream_data):
    """N calls advance the call counter by N marks and release each slot N/SLOTS times."""
    torch, buf, host = stream_data
    L = N.lib()
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    out = torch.zeros((1, 256), dtype=torch.int64, device="cuda")
    ncalls = 4 * SLOTS * 5 + 3
    for k in range(ncalls):
        _issue(L, torch, buf, [0], [1 << 16], N.HS_KIND_NAIVE | N.HS_KIND_FLAG_CHAINED, ws, out)
    torch.cuda.synchronize()
    head = ws[:WS_HEAD_BYTES].cpu().numpy()
    assert int(head[:8].view(np.uint64)[0]) == ncalls * 4096
    drained = head[WS_DRAINED].view(np.uint32).tolist()
    assert drained == [ncalls // SLOTS + (1 if j < ncalls % SLOTS else 0) for j in range(SLOTS)]
    assert ws_clean(ws)


def test_waiting_calls_take_the_serial_slot(stream_data):
    """Calls without HS_KIND_FLAG_CHAINED wait for their predecessor before loading, so
    they use the serial slot: the call counter does not move, no slot is released, and
    interleaving them with chained (rotating) calls keeps every count exact."""
    torch, buf, host = stream_data
    L = N.lib()
    ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
    sizes = [4096, 1 << 16, 1 << 20, 4 << 20, 16 << 20]
    outs = torch.zeros((2 * len(sizes), 256), dtype=torch.int64, device="cuda")
    for k, size in enumerate(sizes):
        _issue(L, torch, buf, [4096 * k], [4096 * k + size], N.HS_KIND_NAIVE, ws, outs[k:k + 1])
    torch.cuda.synchronize()
    head = ws[:WS_HEAD_BYTES].cpu().numpy()
    assert int(head[:8].view(np.uint64)[0]) == 0
    assert not head[WS_DRAINED].view(np.uint32).any()
    for k, size in enumerate(sizes):  # now alternate waiting and chained calls
        kind = N.HS_KIND_NAIVE | (N.HS_KIND_FLAG_CHAINED if k % 2 else 0)
        _issue(L, torch, buf, [8192 * k], [8192 * k + size], kind, ws, outs[len(sizes) + k:len(sizes) + k + 1])
    torch.cuda.synchronize()
    got = outs.cpu().numpy().view(np.uint64)
    for k, size in enumerate(sizes):
        assert np.array_equal(got[k], _counts(host, 4096 * k, 4096 * k + size))
        assert np.array_equal(got[len(sizes) + k], _counts(host, 8192 * k, 8192 * k + size))
    head = ws[:WS_HEAD_BYTES].cpu().numpy()
    assert int(head[:8].view(np.uint64)[0]) == 4096 * (len(sizes) // 2)  # the chained calls only
    assert ws_clean(ws)
