"""The C-ABI library loads on a CPU box and exports every symbol include/hist256.h
declares; argument validation that happens before any device call returns the
documented status codes. No kernels are launched here."""
import ctypes
import re
from pathlib import Path

import numpy as np

from paper_1011_0235_b200 import _native as N

HEADER = Path(__file__).resolve().parents[1] / "include" / "hist256.h"


def declared_functions():
    text = re.sub(r"/\*.*?\*/", "", HEADER.read_text(), flags=re.S)
    return sorted(set(re.findall(r"\b(hs_[a-z0-9_]+)\s*\(", text)))


def test_header_and_binding_agree():
    assert declared_functions() == sorted(N.EXPORTED)


def test_library_exports_every_declared_symbol():
    lib = N.lib()
    raw = ctypes.CDLL(str(N.library_path()))
    for name in declared_functions():
        assert hasattr(raw, name), name
        assert getattr(lib, name) is not None


def test_library_is_sm100a_only():
    import subprocess

    out = subprocess.run(["cuobjdump", "--list-elf", str(N.library_path())], capture_output=True, text=True)
    if out.returncode == 0:
        archs = set(re.findall(r"sm_(\d+a?)", out.stdout))
        assert archs == {"100a"}, archs


def test_status_strings():
    lib = N.lib()
    assert lib.hs_abi_version() == 1
    assert lib.hs_strerror(N.HS_OK) == b"ok"
    assert lib.hs_strerror(N.HS_ERR_PATTERN_COUNT_LOW) == b"count below 1"
    assert lib.hs_strerror(N.HS_ERR_PATTERN_OFFSETS) == b"offsets not contiguous"


def test_argument_validation_before_device_work():
    lib = N.lib()
    b = np.zeros(1, np.uint64)
    e = np.full(1, 8, np.uint64)
    # bad kind / impl / missing pattern for ADAPTIVE are rejected up front
    assert lib.hs_histogram_batched(None, N.u64p(b), N.u64p(e), 1, 7, 0, None, None, 0, 0, None, None, 0, None) == N.HS_ERR_INVALID_ARG
    assert lib.hs_histogram_batched(None, N.u64p(b), N.u64p(e), 1, 0, 9, None, None, 0, 0, None, None, 0, None) == N.HS_ERR_INVALID_ARG
    out = ctypes.c_void_p(16)  # never dereferenced: validation fails first
    assert lib.hs_histogram_batched(None, N.u64p(b), N.u64p(e), 1, N.HS_KIND_ADAPTIVE, 0, None, None, 960, 8, out, None, 0, None) == N.HS_ERR_INVALID_ARG
    # misaligned segment bounds
    e3 = np.full(1, 6, np.uint64)
    assert lib.hs_histogram_batched(ctypes.c_void_p(256), N.u64p(b), N.u64p(e3), 1, 0, 0, None, None, 0, 0, out, None, 0, None) == N.HS_ERR_ALIGNMENT
    # a segment that ends before it begins
    assert lib.hs_histogram_batched(ctypes.c_void_p(256), N.u64p(e), N.u64p(b), 1, 0, 0, None, None, 0, 0, out, None, 0, None) == N.HS_ERR_INVALID_ARG
    # invalid patterns, in the reference's check order
    off = np.arange(256, dtype=np.int64) * 3
    cnt = np.full(256, 3, np.int64)
    assert lib.hs_validate_pattern(N.i64p(off), N.i64p(cnt), 768, 8) == N.HS_OK
    cnt[5] = 0
    assert lib.hs_validate_pattern(N.i64p(off), N.i64p(cnt), 768, 8) == N.HS_ERR_PATTERN_COUNT_LOW
    cnt[5] = 9
    assert lib.hs_validate_pattern(N.i64p(off), N.i64p(cnt), 768, 8) == N.HS_ERR_PATTERN_COUNT_HIGH
    cnt[5] = 3
    assert lib.hs_validate_pattern(N.i64p(off), N.i64p(cnt), 767, 8) == N.HS_ERR_PATTERN_TOTAL
    off[7] += 1
    assert lib.hs_validate_pattern(N.i64p(off), N.i64p(cnt), 768, 8) == N.HS_ERR_PATTERN_OFFSETS
    prior = np.zeros(256, np.uint64)
    o2, c2 = np.zeros(256, np.int64), np.zeros(256, np.int64)
    assert lib.hs_binning_pattern(N.u64p(prior), 255, 8, N.i64p(o2), N.i64p(c2)) == N.HS_ERR_SLOT_RANGE
    assert lib.hs_binning_pattern(N.u64p(prior), 960, 0, N.i64p(o2), N.i64p(c2)) == N.HS_ERR_SLOT_RANGE


def test_missing_library_fails_loudly(monkeypatch, tmp_path):
    import pytest

    monkeypatch.setattr(N, "_lib", None)
    monkeypatch.setenv("HS_LIBHIST256", str(tmp_path / "nope.so"))
    with pytest.raises(N.NativeLibraryError):
        N.lib()
    monkeypatch.setattr(N, "_lib", None)


def test_stream_engine_abi_validation():
    """hs_stream_* reject bad arguments before any device work."""
    lib = N.lib()
    assert lib.hs_stream_state_bytes(0) == 0
    assert lib.hs_stream_state_bytes(4) == 64 + (2 + 4) * 256 * 8
    assert lib.hs_stream_reset(None, 4, None) == N.HS_ERR_INVALID_ARG
    b = np.zeros(1, np.uint64)
    e = np.full(1, 8, np.uint64)
    p = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    step = lib.hs_stream_step
    ws_need = lib.hs_workspace_bytes(64)
    # nseg out of range, threshold outside (0, 1), missing workspace
    assert step(p, N.u64p(b), N.u64p(e), 0, p, 4, 0.45, 1, 0, p, p, p, p, None, p, ws_need, None) == N.HS_ERR_INVALID_ARG
    assert step(p, N.u64p(b), N.u64p(e), 65, p, 4, 0.45, 1, 0, p, p, p, p, None, p, ws_need, None) == N.HS_ERR_INVALID_ARG
    assert step(p, N.u64p(b), N.u64p(e), 1, p, 4, 1.0, 1, 0, p, p, p, p, None, p, ws_need, None) == N.HS_ERR_INVALID_ARG
    assert step(p, N.u64p(b), N.u64p(e), 1, p, 4, 0.45, 0, 0, p, p, p, p, None, p, ws_need, None) == N.HS_ERR_INVALID_ARG
    assert step(p, N.u64p(b), N.u64p(e), 1, p, 4, 0.45, 1, 0, p, p, p, p, None, None, 0, None) == N.HS_ERR_WORKSPACE
    e6 = np.full(1, 6, np.uint64)
    assert step(p, N.u64p(b), N.u64p(e6), 1, p, 4, 0.45, 1, 0, p, p, p, p, None, p, ws_need, None) == N.HS_ERR_ALIGNMENT
    q = ctypes.c_void_p(264)  # 8-aligned: the fold's 16-B moves need 16
    assert step(p, N.u64p(b), N.u64p(e), 1, p, 4, 0.45, 1, 0, q, p, p, p, None, p, ws_need, None) == N.HS_ERR_ALIGNMENT
    assert step(p, N.u64p(b), N.u64p(e), 1, q, 4, 0.45, 1, 0, p, p, p, p, None, p, ws_need, None) == N.HS_ERR_ALIGNMENT


def test_streaming_loop_sass_is_clean():
    """The k_lane streaming loops (the hot path) compile without local-memory traffic
    and without per-iteration R2UR moves: both cost measured throughput before
    (tools/loopcheck.py)."""
    import shutil
    import sys

    import pytest

    if shutil.which("cuobjdump") is None:
        pytest.skip("cuobjdump not available")
    sys.path.insert(0, str(HEADER.parents[1] / "tools"))
    import loopcheck

    loops = loopcheck.report(str(N.library_path()))
    kernels = {r["kernel"] for r in loops}
    assert len(kernels) == 2, kernels  # plain (1024 threads) and HOT (768 threads) k_lane
    main = [r for r in loops if r["atoms"] == 64]
    assert len(main) == 2 and all(r["ldg"] == 4 for r in main), loops
    for r in loops:
        assert r["local"] == 0 and r["r2ur"] == 0, r
    # per 16 B x 4 vectors x 4 bytes: PRMT + address + ATOMS, plus loads and loop control
    assert all(r["len"] <= 210 for r in main if "Lb0" in r["kernel"]), main


def test_sync_entry_points_validate_first():
    """hs_histogram_host / hs_histogram_sync reject bad arguments before any copy."""
    lib = N.lib()
    host = np.zeros(64, np.uint8)
    ptrs = (ctypes.c_void_p * 1)(host.ctypes.data)
    p = ctypes.c_void_p(256)  # never dereferenced: validation fails first
    h_out = np.zeros((1, 256), np.uint64)
    bad = np.array([6], np.uint64)  # not a word multiple
    assert lib.hs_histogram_host(ptrs, N.u64p(bad), 1, 0, 0, None, None, 0, 0, p, 1 << 20, p, N.u64p(h_out),
                                 None, 0, None) == N.HS_ERR_ALIGNMENT
    sizes = np.array([64], np.uint64)
    assert lib.hs_histogram_host(ptrs, N.u64p(sizes), 1, 0, 0, None, None, 0, 0, p, 32, p, N.u64p(h_out),
                                 None, 0, None) == N.HS_ERR_WORKSPACE
    assert lib.hs_histogram_host(ptrs, N.u64p(sizes), 1, 0, 0, None, None, 0, 0, p, 64, p, None,
                                 None, 0, None) == N.HS_ERR_INVALID_ARG
    assert lib.hs_histogram_host(ptrs, N.u64p(sizes), 0, 0, 0, None, None, 0, 0, None, 0, None, None,
                                 None, 0, None) == N.HS_OK
    b = np.zeros(1, np.uint64)
    e = np.full(1, 8, np.uint64)
    assert lib.hs_histogram_sync(p, N.u64p(b), N.u64p(e), 1, 0, 0, None, None, 0, 0, p, None, None, 0,
                                 None) == N.HS_ERR_INVALID_ARG
    assert lib.hs_histogram_sync(p, N.u64p(b), N.u64p(e), 1, 7, 0, None, None, 0, 0, p, N.u64p(h_out), None, 0,
                                 None) == N.HS_ERR_INVALID_ARG


def _build_c_demo(tmp_path):
    """Compile examples/c_api_demo.c (plain C against include/hist256.h, linked with
    libhist256.so and the CUDA runtime) into tmp_path."""
    import shutil
    import subprocess

    root = Path(__file__).resolve().parents[1]
    exe = tmp_path / "c_api_demo"
    cuda = Path("/usr/local/cuda")
    cmd = ["gcc", "-O2", "-std=c11", "-Wall", "-Wextra", "-Werror", "-I", str(root / "include"),
           "-I", str(cuda / "include"), str(root / "examples" / "c_api_demo.c"),
           "-L", str(N.library_path().parent), "-lhist256", "-L", str(cuda / "lib64"), "-lcudart",
           f"-Wl,-rpath,{N.library_path().parent}", f"-Wl,-rpath,{cuda / 'lib64'}", "-o", str(exe)]
    if shutil.which("gcc") is None:
        import pytest

        pytest.skip("gcc not available")
    r = subprocess.run(cmd, capture_output=True, text=True)
    assert r.returncode == 0, r.stderr
    return exe


def test_c_demo_compiles_against_the_header(tmp_path):
    """The ABI is usable from plain C: the demo builds with -Wall -Wextra -Werror."""
    assert _build_c_demo(tmp_path).exists()


def test_workspace_layout_matches_header():
    """hs_workspace_bytes(n) = HS_WS_HEAD_BYTES + (HS_WS_SLOTS + 1) call slots of 1 KiB of
    tickets + one 2 KiB accumulator row per segment (n clamped to [64, 256]); the stream
    block workspace embeds the 256-row form."""
    hdr = HEADER.read_text()
    head = int(re.search(r"#define HS_WS_HEAD_BYTES (\d+)", hdr).group(1))
    slots = int(re.search(r"#define HS_WS_SLOTS (\d+)", hdr).group(1))
    lib = N.lib()
    for n, rows in ((1, 64), (64, 64), (100, 100), (256, 256), (1000, 256)):
        assert lib.hs_workspace_bytes(n) == head + (slots + 1) * (1024 + rows * 2048), n
    assert lib.hs_workspace_bytes(-1) == 0
    assert head % 16 == 0 and head >= 8 + 2 * 4 * slots
    assert lib.hs_stream_block_ws_bytes(4, 8) > lib.hs_workspace_bytes(256)
