"""In-tree build of libbl.so (sm_100a) -- `python -m paper_1701_05936_b200.build`."""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SRC = [os.path.join(PKG, "csrc", "bl.cu")]
DEPS = SRC + [os.path.join(PKG, "csrc", "bl_kernels.cuh"), os.path.join(PKG, "csrc", "bl_tc.cuh"), os.path.join(ROOT, "include", "bl.h")]
LIB = os.path.join(PKG, "libbl.so")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for c in ("/usr/local/cuda/bin/nvcc", "nvcc"):
        if os.path.exists(c) or c == "nvcc":
            return c
    raise RuntimeError("nvcc not found")


def nccl_dirs():
    """Use the NCCL that torch itself loads (one libnccl.so.2 per process)."""
    import importlib.util
    spec = importlib.util.find_spec("nvidia.nccl")
    if spec and spec.submodule_search_locations:
        base = list(spec.submodule_search_locations)[0]
        inc, lib = os.path.join(base, "include"), os.path.join(base, "lib")
        if os.path.exists(os.path.join(inc, "nccl.h")):
            return inc, lib
    return "/usr/include", "/usr/lib/x86_64-linux-gnu"


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIB):
        mt = os.path.getmtime(LIB)
        if all(os.path.getmtime(d) <= mt for d in DEPS):
            return LIB
    ninc, nlib = nccl_dirs()
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-I", ninc, "-o", LIB, *SRC,
           "-L", nlib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nlib]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError("nvcc failed building libbl.so")
    if verbose:
        sys.stderr.write(res.stderr)
    with open(os.path.join(PKG, "ptxas_info.txt"), "w") as f:
        f.write(res.stderr)
    return LIB


def build_variant(name: str, defines: list[str]) -> str:
    """An instrumented copy of the library (e.g. -DBL_G7_SUBPHASES=1) for micro-benchmarks:
    lib<name>.so next to libbl.so; scripts load it by setting bl.LIB_PATH before the first call."""
    out = os.path.join(PKG, f"lib{name}.so")
    ninc, nlib = nccl_dirs()
    cmd = [nvcc(), *NVCC_FLAGS, *defines, "-I", os.path.join(ROOT, "include"), "-I", ninc, "-o", out, *SRC,
           "-L", nlib, "-l:libnccl.so.2", "-Xlinker", "-rpath=" + nlib]
    res = subprocess.run(cmd, capture_output=True, text=True)
    if res.returncode != 0:
        sys.stderr.write(res.stdout + res.stderr)
        raise RuntimeError(f"nvcc failed building {out}")
    return out


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
