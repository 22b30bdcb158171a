"""GPU parity of the block engine behind run_device_stream (hs_stream_block): many
iterations per histogram call, the per-iteration fold reproduced from prefix sums over
(ring ++ block chunks). Everything is compared with the host engine (run_sequential,
itself pinned to the reference's run_sequential by tests/test_gpu_stream.py): kernel log,
per-slice histograms, accumulator, window ring and the float degeneracy/divergence logs,
bit for bit -- across window sizes, batch sizes, recompute periods and block sizes that
put block boundaries inside and across windows. Also: the lagged register path engages
on a dominated segment without changing a count, and the per-iteration C ABI
(hs_stream_step) and the block ABI give the same state."""
import numpy as np
import pytest

import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N
from paper_1011_0235_b200.datagen import schedule_stream

pytestmark = pytest.mark.gpu
POLICY = hs.SwitchPolicy()


def _device_batches(torch, segments, batch_size):
    # every chunk is placed on the device before the run (the engine's input contract)
    batches = [[hs.DeviceChunk(torch.from_numpy(c.pixels().copy()).cuda()) for c in b]
               for b in schedule_stream(segments, batch_size)]
    torch.cuda.synchronize()
    return iter(batches)


def _equal(seq, dev):
    assert dev[0] == seq[0], "accumulator"
    assert dev[1].windowed == seq[1].windowed, "window"
    assert [h.counts.tolist() for h in dev[1].ring] == [h.counts.tolist() for h in seq[1].ring], "ring"
    assert [k.value for k in dev[3]] == [k.value for k in seq[3]], "kernel log"
    assert dev[2].per_slice_histograms == seq[2].per_slice_histograms, "per-slice"
    assert dev[2].degeneracy_log == seq[2].degeneracy_log, "degeneracy log"
    assert dev[2].divergence_log == seq[2].divergence_log, "divergence log"


@pytest.mark.parametrize("window,batch,every,block", [
    (1, 1, 1, 1), (2, 1, 2, 3 << 12), (7, 3, 1, 1 << 14), (16, 5, 5, 1 << 16), (32, 1, 1, 1 << 30),
    (128, 2, 3, 1 << 15), (300, 4, 1, 1 << 13), (5, 64, 2, 1 << 20), (64, 17, 1, 1 << 30)])
def test_block_engine_equals_host_engine(cuda, window, batch, every, block):
    px = 4096
    segs = [(hs.SourceSpec("uniform", px, 31), 9), (hs.SourceSpec("mixture", px, 31, value=77, degeneracy=0.8), 7),
            (hs.SourceSpec("constant", px, 31, value=200), 8), (hs.SourceSpec("normal", px, 31, mean=90.0,
                                                                               sigma=3.0), 6)]
    iters = 30
    cfg = hs.PipelineConfig(num_iterations=iters, chunk_pixels=px, batch_size=batch, window_size=window,
                            recompute_pattern_every=every)
    seq = hs.run_sequential(schedule_stream(segs, batch), cfg, POLICY)
    dev = hs.run_device_stream(_device_batches(cuda, segs, batch), cfg, POLICY, block_bytes=block)
    _equal(seq, dev)
    assert sum(dev[2].block_sizes) == iters
    if block <= px:
        assert max(dev[2].block_sizes) == 1
    if block >= 1 << 30 and batch * iters <= 256:
        assert dev[2].block_sizes == [iters]


def test_block_engine_small_iterations_and_register_path(cuda, oracle):
    """1 MiB batch-1 iterations (the reference's default PipelineConfig chunk size):
    uniform then constant, 384 iterations in 256 MiB blocks. Logs and state equal the
    host engine; once the device has decided ADAPTIVE on the constant window the
    engine runs the register path for bin 200 (lagged), with identical counts."""
    torch = cuda
    px = 1 << 20
    segs = [(hs.SourceSpec("uniform", px, 5), 128), (hs.SourceSpec("constant", px, 5, value=200), 256)]
    cfg = hs.PipelineConfig(num_iterations=384, chunk_pixels=px, window_size=8)
    seq = hs.run_sequential(schedule_stream(segs), cfg, POLICY)
    dev = hs.run_device_stream(_device_batches(torch, segs, 1), cfg, POLICY)
    _equal(seq, dev)
    ex = dev[2].executed_log
    assert ex[0] == "k_lane" and ex[-1] == "k_lane<HOT bin 200>", (ex[:3], ex[-3:])
    assert all(e == "k_lane" for e in ex[:128])
    off = hs.run_device_stream(_device_batches(torch, segs, 1), cfg, POLICY, register_path=False)
    _equal(seq, off)
    assert set(off[2].executed_log) == {"k_lane"}


@pytest.mark.parametrize("ahead", [1, 2, None])
def test_blocks_ahead_bounds_register_path_lag(cuda, ahead):
    """Large iterations, one per block: with at most ``ahead`` blocks queued the host
    issues block k only after block k - ahead finished, so the register path engages
    within ``ahead`` blocks of the device's decision (with no bound a fast host may have
    issued every block first). Counts, state and logs equal the host engine either way."""
    torch = cuda
    px = 16 << 20
    segs = [(hs.SourceSpec("uniform", px, 9), 4), (hs.SourceSpec("constant", px, 9, value=77), 12)]
    cfg = hs.PipelineConfig(num_iterations=16, chunk_pixels=px, window_size=2)
    seq = hs.run_sequential(schedule_stream(segs), cfg, POLICY)
    dev = hs.run_device_stream(_device_batches(torch, segs, 1), cfg, POLICY, block_bytes=px, blocks_ahead=ahead)
    _equal(seq, dev)
    assert dev[2].block_sizes == [1] * 16
    ex = dev[2].executed_log
    assert all(e == "k_lane" for e in ex[:5]), ex
    if ahead is not None:
        # the window is all-77 after iteration 5 (window 2), the decision for iteration 6
        # is published by block 5's commit; block 5 + ahead is issued after it completed
        first = 6 + ahead - 1
        assert all(e == "k_lane<HOT bin 77>" for e in ex[first:]), ex
    with pytest.raises(ValueError):
        hs.run_device_stream(_device_batches(torch, segs[:1], 1), hs.PipelineConfig(num_iterations=4, chunk_pixels=px),
                             POLICY, blocks_ahead=0)


def test_step_abi_equals_block_abi(cuda):
    """hs_stream_step per iteration and one hs_stream_block over the same iterations
    leave identical state and logs."""
    torch = cuda
    L = N.lib()
    W, iters, per, px = 3, 6, 2, 1 << 16
    rng = np.random.default_rng(8)
    host = rng.integers(0, 256, iters * per * px, dtype=np.uint8)
    host[: per * px * 2] = 17
    buf = torch.from_numpy(host).cuda()
    s = torch.cuda.current_stream().cuda_stream
    res = []
    for mode in ("step", "block"):
        state = torch.empty(int(L.hs_stream_state_bytes(W)), dtype=torch.uint8, device="cuda")
        N.check(L.hs_stream_reset(state.data_ptr(), W, s), "reset")
        deg = torch.zeros(iters, dtype=torch.float64, device="cuda")
        div = torch.zeros(iters, dtype=torch.float64, device="cuda")
        kinds = torch.zeros(iters, dtype=torch.int32, device="cuda")
        out = torch.empty((iters * per, 256), dtype=torch.int64, device="cuda")
        if mode == "step":
            ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
            for i in range(iters):
                b0 = (np.arange(per, dtype=np.uint64) + i * per) * px
                b1 = b0 + px
                N.check(L.hs_stream_step(buf.data_ptr(), N.u64p(b0), N.u64p(b1), per, state.data_ptr(), W, 0.45, 1, i,
                                         out[i * per:(i + 1) * per].data_ptr(), deg.data_ptr(), div.data_ptr(),
                                         kinds.data_ptr(), None, ws.data_ptr(), ws.numel(), s), "step")
        else:
            n = int(L.hs_stream_block_ws_bytes(W, iters * per))
            ws = torch.zeros(n, dtype=torch.uint8, device="cuda")
            b0 = np.arange(iters * per, dtype=np.uint64) * px
            b1 = b0 + px
            import ctypes

            chunks = (ctypes.c_int32 * iters)(*([per] * iters))
            N.check(L.hs_stream_block(buf.data_ptr(), N.u64p(b0), N.u64p(b1), iters * per, chunks, iters,
                                      state.data_ptr(), W, 0.45, 1, 0, -1, out.data_ptr(), deg.data_ptr(),
                                      div.data_ptr(), kinds.data_ptr(), None, None, ws.data_ptr(), n, s), "block")
        torch.cuda.synchronize()
        st = state.cpu().numpy()
        res.append((st[:40].tobytes(), st[48:56].tobytes(), st[64:].tobytes(), deg.cpu().tolist(), div.cpu().tolist(),
                    kinds.cpu().tolist(), out.cpu().numpy().tobytes()))
    assert res[0] == res[1]


def test_block_abi_errors(cuda):
    torch = cuda
    L = N.lib()
    import ctypes

    st = torch.empty(int(L.hs_stream_state_bytes(2)), dtype=torch.uint8, device="cuda")
    out = torch.empty((2, 256), dtype=torch.int64, device="cuda")
    logs = torch.zeros(4, dtype=torch.float64, device="cuda")
    kinds = torch.zeros(4, dtype=torch.int32, device="cuda")
    b0, b1 = np.zeros(2, np.uint64), np.full(2, 16, np.uint64)
    ok_chunks = (ctypes.c_int32 * 2)(1, 1)
    bad_chunks = (ctypes.c_int32 * 2)(1, 2)
    n = int(L.hs_stream_block_ws_bytes(2, 2))
    ws = torch.zeros(n, dtype=torch.uint8, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    args = lambda ch, wsb, thr=0.45: (out.data_ptr(), N.u64p(b0), N.u64p(b1), 2, ch, 2, st.data_ptr(), 2, thr, 1, 0,
                                      -1, out.data_ptr(), logs.data_ptr(), logs.data_ptr(), kinds.data_ptr(), None,
                                      None, ws.data_ptr(), wsb, s)
    assert L.hs_stream_block(*args(bad_chunks, n)) == N.HS_ERR_INVALID_ARG  # chunk counts != nseg
    assert L.hs_stream_block(*args(ok_chunks, n - 1)) == N.HS_ERR_WORKSPACE
    assert L.hs_stream_block(*args(ok_chunks, n, 1.0)) == N.HS_ERR_INVALID_ARG
    assert L.hs_stream_block_ws_bytes(0, 2) == 0 and L.hs_stream_block_ws_bytes(2, 257) == 0
