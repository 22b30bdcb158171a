"""ctypes binding of libhist256.so (include/hist256.h).

The shared library is built in-tree (``paper_1011_0235_b200/_lib/libhist256.so``,
see ``build.py``). There is deliberately no fallback: if the library is missing
or cannot be loaded, every entry point raises ``NativeLibraryError`` — the product
path never drops to a CPU implementation.

ctypes releases the GIL for the duration of each foreign call, which keeps the
reference's threading contract (its numba workers run ``nogil=True``,
kernels.py:97) for the pipeline's producer thread.
"""
from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

LIB_DIR = Path(__file__).resolve().parent / "_lib"
LIB_PATH = LIB_DIR / "libhist256.so"

HS_OK = 0
HS_ERR_INVALID_ARG = -1
HS_ERR_PATTERN_SHAPE = -2
HS_ERR_PATTERN_COUNT_LOW = -3
HS_ERR_PATTERN_COUNT_HIGH = -4
HS_ERR_PATTERN_TOTAL = -5
HS_ERR_PATTERN_OFFSETS = -6
HS_ERR_SLOT_RANGE = -7
HS_ERR_WORKSPACE = -8
HS_ERR_UNSUPPORTED = -9
HS_ERR_ALIGNMENT = -10
HS_ERR_NO_DEVICE = -11
HS_ERR_CUDA_BASE = -1000

HS_KIND_NAIVE = 0
HS_KIND_ADAPTIVE = 1
HS_KIND_FLAG_SPREAD = 0x100
HS_KIND_FLAG_CHAINED = 0x200
HS_KIND_FLAG_MERGE = 0x400

HS_IMPL_AUTO = 0
HS_IMPL_LANE = 1
HS_IMPL_WARP = 2
HS_IMPL_SUBBIN = 3

HS_STAGE_COPY_ONLY = 0
HS_STAGE_COPY_INIT = 1
HS_STAGE_PATTERN_LOAD = 2
HS_STAGE_SUBHIST_NOREDUCE = 3
HS_STAGE_FULL = 4

HS_GEN_UNIFORM = 0
HS_GEN_SEQUENTIAL = 1
HS_GEN_CONSTANT = 2
HS_GEN_NORMAL = 3
HS_GEN_MIXTURE = 4

# every symbol include/hist256.h declares (checked by tests/test_native_abi.py)
EXPORTED = (
    "hs_abi_version",
    "hs_strerror",
    "hs_device_query",
    "hs_validate_pattern",
    "hs_workspace_bytes",
    "hs_histogram_batched",
    "hs_histogram_host",
    "hs_histogram_sync",
    "hs_histogram",
    "hs_group_slots_ws_bytes",
    "hs_group_slots",
    "hs_ablation_stage",
    "hs_binning_pattern",
    "hs_degeneracy",
    "hs_divergence",
    "hs_copy_streaming",
    "hs_generate_host",
    "hs_generate_device",
    "hs_stream_state_bytes",
    "hs_stream_reset",
    "hs_stream_step",
    "hs_stream_block_ws_bytes",
    "hs_stream_block",
)

_c = ctypes
_P = _c.c_void_p
_U64 = _c.c_uint64
_I64 = _c.c_int64
_I64P = _c.POINTER(_c.c_int64)
_U64P = _c.POINTER(_c.c_uint64)

_SIGNATURES = {
    "hs_abi_version": (_c.c_int, []),
    "hs_strerror": (_c.c_char_p, [_c.c_int]),
    "hs_device_query": (_c.c_int, [_c.c_int, _c.POINTER(_c.c_int), _c.POINTER(_c.c_int), _c.POINTER(_c.c_int)]),
    "hs_validate_pattern": (_c.c_int, [_I64P, _I64P, _I64, _I64]),
    "hs_workspace_bytes": (_c.c_size_t, [_c.c_int]),
    "hs_histogram_batched": (
        _c.c_int,
        [_P, _U64P, _U64P, _c.c_int, _c.c_int, _c.c_int, _I64P, _I64P, _I64, _I64, _P, _P, _c.c_size_t, _P],
    ),
    "hs_histogram_sync": (
        _c.c_int,
        [_P, _U64P, _U64P, _c.c_int, _c.c_int, _c.c_int, _I64P, _I64P, _I64, _I64, _P, _U64P, _P, _c.c_size_t, _P],
    ),
    "hs_histogram_host": (
        _c.c_int,
        [_c.POINTER(_c.c_void_p), _U64P, _c.c_int, _c.c_int, _c.c_int, _I64P, _I64P, _I64, _I64, _P,
         _c.c_size_t, _P, _U64P, _P, _c.c_size_t, _P],
    ),
    "hs_histogram": (
        _c.c_int,
        [_P, _U64, _c.c_int, _c.c_int, _I64P, _I64P, _I64, _I64, _P, _P, _c.c_size_t, _P],
    ),
    "hs_group_slots_ws_bytes": (_c.c_size_t, [_c.c_int, _c.c_int, _I64, _c.c_int]),
    "hs_group_slots": (
        _c.c_int,
        [_P, _U64, _c.c_int, _c.c_int, _I64P, _I64P, _I64, _I64, _c.c_int, _P, _P, _c.c_size_t, _P],
    ),
    "hs_ablation_stage": (
        _c.c_int,
        [_P, _U64, _c.c_int, _I64P, _I64P, _I64, _I64, _P, _P, _P, _c.c_size_t, _P],
    ),
    "hs_binning_pattern": (_c.c_int, [_U64P, _I64, _I64, _I64P, _I64P]),
    "hs_degeneracy": (_c.c_int, [_U64P, _c.POINTER(_c.c_double), _c.POINTER(_c.c_int), _U64P]),
    "hs_divergence": (_c.c_int, [_U64P, _U64P, _c.POINTER(_c.c_double)]),
    "hs_copy_streaming": (_c.c_int, [_P, _P, _U64, _c.c_int]),
    "hs_generate_host": (
        _c.c_int,
        [_c.c_int, _U64, _c.c_int, _c.c_double, _c.c_double, _c.c_double, _P, _U64, _c.c_int],
    ),
    "hs_generate_device": (
        _c.c_int,
        [_c.c_int, _U64, _c.c_int, _c.c_double, _c.c_double, _U64, _P, _U64, _P],
    ),
    "hs_stream_state_bytes": (_c.c_size_t, [_c.c_int]),
    "hs_stream_reset": (_c.c_int, [_P, _c.c_int, _P]),
    "hs_stream_block_ws_bytes": (_c.c_size_t, [_c.c_int, _c.c_int]),
    "hs_stream_block": (
        _c.c_int,
        [_P, _U64P, _U64P, _c.c_int, _c.POINTER(_c.c_int32), _c.c_int, _P, _c.c_int, _c.c_double, _c.c_int,
         _c.c_int, _c.c_int, _P, _P, _P, _P, _P, _P, _P, _c.c_size_t, _P],
    ),
    "hs_stream_step": (
        _c.c_int,
        [_P, _U64P, _U64P, _c.c_int, _P, _c.c_int, _c.c_double, _c.c_int, _c.c_int, _P, _P, _P, _P, _P, _P,
         _c.c_size_t, _P],
    ),
}


class NativeLibraryError(RuntimeError):
    """libhist256.so is missing or failed to load; there is no fallback."""


class NativeCallError(RuntimeError):
    """A libhist256 call returned a non-zero status."""

    def __init__(self, status: int, where: str):
        self.status = status
        super().__init__(f"{where}: {strerror(status)} (status {status})")


_lock = threading.Lock()
_lib = None


def library_path() -> Path:
    override = os.environ.get("HS_LIBHIST256")
    return Path(override) if override else LIB_PATH


def lib():
    """The loaded library (loaded once; raises NativeLibraryError if absent)."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not path.exists():
            raise NativeLibraryError(
                f"{path} not found: build it with `python -m paper_1011_0235_b200.build` "
                "(there is no CPU fallback)"
            )
        try:
            handle = ctypes.CDLL(str(path))
        except OSError as exc:  # pragma: no cover - depends on the box
            raise NativeLibraryError(f"cannot load {path}: {exc}") from exc
        override = "HS_LIBHIST256" in os.environ  # A/B runs of older builds may lack newer symbols
        for name, (restype, argtypes) in _SIGNATURES.items():
            try:
                fn = getattr(handle, name)
            except AttributeError:
                if override:
                    continue
                raise
            fn.restype = restype
            fn.argtypes = argtypes
        _lib = handle
        return _lib


def strerror(status: int) -> str:
    try:
        return lib().hs_strerror(int(status)).decode()
    except NativeLibraryError:
        return f"status {status}"


def check(status: int, where: str) -> None:
    if status != HS_OK:
        raise NativeCallError(status, where)


def i64p(arr):
    """Pointer to a contiguous int64 numpy array."""
    return arr.ctypes.data_as(_I64P)


def u64p(arr):
    return arr.ctypes.data_as(_U64P)
