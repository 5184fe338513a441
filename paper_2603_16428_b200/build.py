"""Builds libslf_lce.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
SO = os.path.join(HERE, "libslf_lce.so")
SRC = os.path.join(HERE, "csrc", "slf_lce.cu")
SRC_HOST = os.path.join(HERE, "csrc", "layer_adam.cpp")  # Layer-Adam host optimizer (C++/OpenMP/AVX-512)
DEPS = [os.path.join(HERE, "csrc", f) for f in ("slf_lce.cu", "gemm.cuh", "aux_kernels.cuh", "s_kernels.cuh", "rmsnorm.cuh", "ptx.cuh", "comm.cuh", "layer_adam.cpp")] + [
    os.path.join(ROOT, "include", "slf_lce.h"), os.path.join(ROOT, "include", "slf_adam.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-std=c++17", "-lineinfo",
    "-Xcompiler", "-fPIC,-fopenmp,-ffp-contract=off", "-shared",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.sep not in c or os.path.exists(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(d) <= t for d in DEPS if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return SO
    tmp = SO + ".tmp"
    cmd = [nvcc(), *NVCC_FLAGS, "-o", tmp, SRC, SRC_HOST, "-ldl", "-lgomp"]
    if verbose:
        print(" ".join(cmd), file=sys.stderr)
    subprocess.run(cmd, check=True)
    os.replace(tmp, SO)
    return SO


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
