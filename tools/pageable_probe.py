"""Host-side costs behind a pageable 1 MiB H2D (the per-image path from numpy):
driver pageable copy vs memcpy into page-locked memory + DMA, single and in pieces."""
import ctypes
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

n = 1 << 20
src = np.random.default_rng(0).integers(0, 256, n, dtype=np.uint8)
pin = torch.empty(n, dtype=torch.uint8).pin_memory()
pin_np = pin.numpy()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.current_stream()


def T(name, f, reps=500):
    for _ in range(20):
        f()
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(reps):
        f()
    torch.cuda.synchronize()
    print(f"{name:48s} {(time.perf_counter() - t0) / reps * 1e6:8.2f} us", flush=True)


src_t = torch.from_numpy(src)
T("pageable H2D (torch copy_, driver staging)", lambda: (dst.copy_(src_t), s.synchronize()))
T("memmove 1 MiB into page-locked", lambda: ctypes.memmove(pin_np.ctypes.data, src.ctypes.data, n))
T("np.copyto 1 MiB into page-locked", lambda: np.copyto(pin_np, src))
T("pinned H2D async + sync", lambda: (dst.copy_(pin, non_blocking=True), s.synchronize()))


def pieces(k):
    step = n // k
    for i in range(k):
        ctypes.memmove(pin_np.ctypes.data + i * step, src.ctypes.data + i * step, step)
        dst[i * step:(i + 1) * step].copy_(pin[i * step:(i + 1) * step], non_blocking=True)
    s.synchronize()


for k in (1, 2, 4, 8):
    T(f"memmove + DMA in {k} pieces (python)", lambda: pieces(k))
big = np.random.default_rng(1).integers(0, 256, 64 << 20, dtype=np.uint8)
pin_big = torch.empty(64 << 20, dtype=torch.uint8).pin_memory().numpy()
T("memmove 64 MiB (cold source) GB/s-> see us", lambda: ctypes.memmove(pin_big.ctypes.data, big.ctypes.data, 64 << 20), 20)
print("cpu count", os.cpu_count(), "affinity", len(os.sched_getaffinity(0)))
