"""Build recipe for libhist256.so (sm_100a only, in-tree so it travels with the repo).

    python -m paper_1011_0235_b200.build [--force]

nvcc cross-compiles here without a GPU. Host code is compiled with
-ffp-contract=off so the float64 pattern/generator arithmetic matches numpy/numba
operation by operation.
"""
from __future__ import annotations

import argparse
import os
import shutil
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
CSRC = PKG / "csrc"
INCLUDE = PKG.parent / "include"
OUT = PKG / "_lib" / "libhist256.so"
SOURCES = [CSRC / "hs_kernels.cu", CSRC / "hs_host.cpp"]
HEADERS = [INCLUDE / "hist256.h"]
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and Path(cand).exists():
            return cand
    raise RuntimeError("nvcc not found")


def command(out: Path = OUT) -> list[str]:
    return [
        nvcc(), "-shared", "-Xcompiler", "-fPIC", "-O3", "-lineinfo", "-std=c++17",
        *ARCH, "-Xcompiler", "-ffp-contract=off", "-I", str(INCLUDE),
        *[str(s) for s in SOURCES], "-o", str(out),
    ]


def stale(out: Path = OUT) -> bool:
    if not out.exists():
        return True
    t = out.stat().st_mtime
    return any(p.stat().st_mtime > t for p in [*SOURCES, *HEADERS, Path(__file__)])


def build(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return OUT
    OUT.parent.mkdir(parents=True, exist_ok=True)
    tmp = OUT.with_suffix(".so.tmp")
    cmd = command(tmp)
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, OUT)
    return OUT


def main(argv=None) -> int:
    ap = argparse.ArgumentParser()
    ap.add_argument("--force", action="store_true")
    args = ap.parse_args(argv)
    print(build(force=args.force, verbose=True))
    return 0


if __name__ == "__main__":
    raise SystemExit(main())
