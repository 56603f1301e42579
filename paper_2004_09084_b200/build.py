"""In-tree build of ``libqcldpc_b200.so`` for sm_100a (no GPU needed; nvcc cross-compiles).

The library is a single translation unit (``csrc/qcldpc.cu``) compiled with
``-gencode arch=compute_100a,code=sm_100a -lineinfo`` so ncu's source page maps to
the kernels.  Rebuilds only when a source is newer than the library.
"""

from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SOURCES = [PKG / "csrc" / "qcldpc.cu"]
DEPS = SOURCES + sorted((PKG / "csrc").glob("*.cuh")) + [ROOT / "include" / "qcldpc_b200.h"]
OUT = PKG / "libqcldpc_b200.so"

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-warn-spills",
    f"-I{ROOT / 'include'}",
]


def nvcc():
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (Path(cand).exists() or cand == "nvcc"):
            return cand
    return "nvcc"


def stale():
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    return any(p.stat().st_mtime > t for p in DEPS)


def build(force=False, verbose=False):
    if not force and not stale():
        return OUT
    cmd = [nvcc(), *NVCC_FLAGS, "-o", str(OUT) + ".tmp", *map(str, SOURCES)]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(str(OUT) + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose=True)
    print(OUT)
