"""Device stream engine: GPU span of 6 x 1 GiB hs_stream_step iterations with and without
an event pair per step (events between the chained launches break their overlap)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import paper_1011_0235_b200 as hs
from paper_1011_0235_b200 import _native as N
L = N.lib()
px, per_iter, iters = 16 << 20, 64, 6
buf = torch.empty(iters * per_iter * px, dtype=torch.uint8, device="cuda")
hs.generate_device(hs.SourceSpec("uniform", buf.numel(), 3), buf)
W = 1
state = torch.empty(int(L.hs_stream_state_bytes(W)), dtype=torch.uint8, device="cuda")
deg = torch.zeros(iters, dtype=torch.float64, device="cuda"); div = torch.zeros_like(deg); kinds = torch.zeros(iters, dtype=torch.int32, device="cuda")
ws = torch.zeros(int(L.hs_workspace_bytes(64)), dtype=torch.uint8, device="cuda")
outs = [torch.empty((per_iter, 256), dtype=torch.int64, device="cuda") for _ in range(iters)]
st = torch.cuda.current_stream()
begin = np.arange(per_iter, dtype=np.uint64) * px
end = begin + px
def run(events):
    N.check(L.hs_stream_reset(state.data_ptr(), W, st.cuda_stream), "r")
    evs = []
    a0 = torch.cuda.Event(enable_timing=True); a0.record()
    for i in range(iters):
        if events:
            e = torch.cuda.Event(enable_timing=True); e.record(); evs.append(e)
        base = buf.data_ptr() + i * per_iter * px
        N.check(L.hs_stream_step(base, N.u64p(begin), N.u64p(end), per_iter, state.data_ptr(), W, 0.45, 1, i,
                                 outs[i].data_ptr(), deg.data_ptr(), div.data_ptr(), kinds.data_ptr(), None, ws.data_ptr(), ws.numel(), st.cuda_stream), "s")
        if events:
            e = torch.cuda.Event(enable_timing=True); e.record(); evs.append(e)
    b0 = torch.cuda.Event(enable_timing=True); b0.record(); b0.synchronize()
    tot = a0.elapsed_time(b0) / 1e3
    per = sum(evs[2*k].elapsed_time(evs[2*k+1]) for k in range(iters)) / 1e3 if events else None
    return buf.numel() / tot / 1e9, (buf.numel() / per / 1e9 if per else None)
for _ in range(2): run(True); run(False)
for r in range(3):
    print("events  span %.1f GB/s  sum-of-iterations %.1f GB/s" % run(True))
    print("no-events span %.1f GB/s" % run(False)[0])
