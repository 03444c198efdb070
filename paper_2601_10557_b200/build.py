"""Build libbse200.so in-tree with nvcc for sm_100a (no JIT cache: the .so
travels to the GPU box with the repo snapshot)."""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = PKG / "csrc" / "bse200.cu"
OUT = PKG / "libbse200.so"
DEPS = sorted((PKG / "csrc").glob("*.cu*")) + [ROOT / "include" / "bse200.h"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    raise RuntimeError("nvcc not found")


def stale() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build_library(force: bool = False, verbose: bool = False) -> Path:
    if not force and not stale():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT), str(SRC), "-lcublas", "-lcusolver"]  # driver API via cudaGetDriverEntryPoint
    proc = subprocess.run(cmd, capture_output=True, text=True)
    log = proc.stdout + proc.stderr
    (PKG / "build.log").write_text(log)
    if proc.returncode != 0:
        sys.stderr.write(log)
        raise RuntimeError(f"nvcc failed ({proc.returncode})")
    if verbose:
        print(log)
    return OUT


if __name__ == "__main__":
    print(build_library(force="--force" in sys.argv, verbose="-v" in sys.argv))
