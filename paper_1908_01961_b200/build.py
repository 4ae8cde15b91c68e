"""Build the sm_100a extension in-tree: paper_1908_01961_b200/liblumisplit_b200.so.

    python -m paper_1908_01961_b200.build          (or __graft_entry__.build())

Plain nvcc, no torch extension machinery: the product is a C-ABI shared
library (include/lumisplit_b200.h) that the Python host binds with ctypes.
"""
from __future__ import annotations

import os
import subprocess
import sys
from pathlib import Path

PKG = Path(__file__).resolve().parent
ROOT = PKG.parent
SRC = sorted((PKG / "csrc").glob("*.cu"))
OUT = PKG / "liblumisplit_b200.so"
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", *os.environ.get("LS_NVCC_DEFS", "").split(),
         "-Xcompiler", "-fvisibility=hidden", "-cudart", "static", "--expt-relaxed-constexpr"]


def needs_build() -> bool:
    if not OUT.exists():
        return True
    t = OUT.stat().st_mtime
    deps = SRC + list((PKG / "csrc").glob("*.h")) + list((PKG / "csrc").glob("*.cuh")) + \
        [ROOT / "include" / "lumisplit_b200.h", Path(__file__)]
    return any(p.stat().st_mtime > t for p in deps)


def build(force: bool = False, verbose: bool = True) -> Path:
    if not force and not needs_build():
        return OUT
    objs = []
    build_dir = PKG / "build"
    build_dir.mkdir(exist_ok=True)
    procs = []
    for src in SRC:
        obj = build_dir / (src.stem + ".o")
        cmd = [NVCC, *ARCH, *FLAGS, "-I", str(ROOT / "include"), "-c", str(src), "-o", str(obj)]
        if verbose:
            print(" ".join(cmd), flush=True)
        procs.append((subprocess.Popen(cmd), cmd))
        objs.append(str(obj))
    for p, cmd in procs:
        if p.wait() != 0:
            raise RuntimeError("nvcc failed: " + " ".join(cmd))
    link = [NVCC, *ARCH, "-shared", "-cudart", "static", "-Xcompiler", "-fPIC", *objs, "-o", str(OUT)]
    if verbose:
        print(" ".join(link), flush=True)
    subprocess.check_call(link)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv)
