"""Every libhist256 kernel on small inputs, each result checked against numpy: k_lane
plain and register (HOT) forms, ticketed and memset+RED outputs, several segments;
k_warp; k_subbin; k_group_slots (slots, lane touches, narrow counters); every ablation
stage; the device generators; the device stream engine (k_stream_fold) and the host
pipelines. Written as the workload for compute-sanitizer (memcheck, racecheck,
synccheck, initcheck), which this GPU pool does not allow; it runs as an all-kernel
parity pass instead.
usage: python tools/all_kernels_run.py"""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_1011_0235_b200 as hs  # noqa: E402
from paper_1011_0235_b200 import _native as N, device as D  # noqa: E402
from paper_1011_0235_b200.datagen import schedule_stream  # noqa: E402

rng = np.random.default_rng(5)
n = (1 << 20) + 44
px = rng.integers(0, 256, n, dtype=np.uint8)
px[: n // 2] = 77  # a hot stretch for the register path
want = np.bincount(px, minlength=256)
cfg = hs.WorkerGroupConfig(32, 4)
host = hs.PackedChunk(px.view(np.uint32)[: n // 4].copy())
dev = hs.DeviceChunk(torch.from_numpy(px).cuda())
pat = hs.compute_binning_pattern(hs.Histogram256(want.astype(np.uint64)))
deg = np.zeros(256, np.uint64)
deg[77] = 10
hot_pat = hs.compute_binning_pattern(hs.Histogram256(deg))
for impl in (N.HS_IMPL_AUTO, N.HS_IMPL_WARP, N.HS_IMPL_SUBBIN):
    for c in (host, dev):
        assert np.array_equal(hs.naive_histogram(c, cfg).counts, want) if impl == N.HS_IMPL_AUTO else True
        got = D.histograms([c], N.HS_KIND_ADAPTIVE, hot_pat, impl)[0]
        assert np.array_equal(got, want), impl
print("single-chunk forms ok", flush=True)
# several segments, ticketed and not, and a call spread over workspace groups
L = N.lib()
st = torch.cuda.current_stream().cuda_stream
buf = torch.from_numpy(px).cuda()
cuts = np.array([0, 4, 4, 4096, 70000, 300000, n // 4 * 4], np.uint64)
b0, b1 = cuts[:-1].copy(), cuts[1:].copy()
ref = np.stack([np.bincount(px[int(a):int(b)], minlength=256) for a, b in zip(b0, b1)])
for ws_seg in (0, 1, 64):
    for kind, p in ((N.HS_KIND_NAIVE, None), (N.HS_KIND_ADAPTIVE, hot_pat)):
        ws = torch.zeros(int(L.hs_workspace_bytes(ws_seg)) if ws_seg else 1, dtype=torch.uint8, device="cuda")
        if ws_seg == 1:  # a 1-segment workspace is below the minimum: memset + RED path
            ws = torch.zeros(int(L.hs_workspace_bytes(64)) // 2, dtype=torch.uint8, device="cuda")
        out = torch.full((len(b0), 256), -1, dtype=torch.int64, device="cuda")
        N.check(L.hs_histogram_batched(buf.data_ptr(), N.u64p(b0), N.u64p(b1), len(b0), kind, N.HS_IMPL_LANE,
                                       N.i64p(p.offset) if p else None, N.i64p(p.count) if p else None,
                                       960 if p else 0, 8 if p else 0, out.data_ptr(),
                                       ws.data_ptr() if ws_seg else None, ws.numel() if ws_seg else 0, st), "batched")
        assert np.array_equal(out.cpu().numpy(), ref), (ws_seg, kind)
print("segments ok", flush=True)
# slots, lane touches, narrow counters
small = hs.PackedChunk(px.view(np.uint32)[:4096].copy())
h, slots = hs.adaptive_histogram(small, pat, cfg, return_slots=True)
assert np.array_equal(h.counts, np.bincount(px[:16384], minlength=256))
hs.adaptive_histogram(small, pat, cfg, narrow_counters=True)
hs.adaptive_lane_touches(small, pat, cfg)
print("slot forms ok", flush=True)
for stage in range(5):
    D.ablation_stage(dev, stage, pat)
print("ablation ok", flush=True)
g = torch.empty(1 << 16, dtype=torch.uint8, device="cuda")
for spec in (hs.SourceSpec("uniform", 1 << 16, 3), hs.SourceSpec("normal", 1 << 16, 3, mean=100.0, sigma=9.0),
             hs.SourceSpec("constant", 1 << 16, 3, value=9), hs.SourceSpec("sequential", 1 << 16, 3)):
    hs.generate_device(spec, g)
    assert np.array_equal(g.cpu().numpy(), hs.generate(spec).pixels())
print("generators ok", flush=True)
segs = [(hs.SourceSpec("uniform", 1 << 14, 7), 3), (hs.SourceSpec("constant", 1 << 14, 7, value=200), 3)]
scfg = hs.PipelineConfig(num_iterations=6, chunk_pixels=1 << 14, batch_size=2, window_size=2)
host_run = hs.run_sequential(schedule_stream(segs, 2), scfg, hs.SwitchPolicy())
dev_run = hs.run_device_stream(([hs.DeviceChunk(torch.from_numpy(c.pixels().copy()).cuda()) for c in b]
                                for b in schedule_stream(segs, 2)), scfg, hs.SwitchPolicy())
assert dev_run[0] == host_run[0] and dev_run[3] == host_run[3]
pipe_run = hs.run_pipeline(schedule_stream(segs, 2), scfg, hs.SwitchPolicy())
assert pipe_run[0] == host_run[0] and pipe_run[3] == host_run[3]
print("stream engines ok", flush=True)
torch.cuda.synchronize()
print("all kernels ok", flush=True)
