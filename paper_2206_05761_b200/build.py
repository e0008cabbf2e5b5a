"""In-tree build of the sm_100a library and the CPU oracle.

`python -m paper_2206_05761_b200.build` (or __graft_entry__.build()) runs
nvcc directly — the .so lands next to this file so it travels with the repo
snapshot to the GPU box.
"""
from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
LIB = os.path.join(HERE, "libswamp_gpu.so")
SOURCES = [os.path.join(HERE, "csrc", "swamp_gpu.cu"), os.path.join(HERE, "csrc", "swamp_io.cpp")]
DEPS = SOURCES + [
    os.path.join(HERE, "csrc", "hwfv1_kernels.cuh"),
    os.path.join(HERE, "csrc", "hwfv1_physics.cuh"),
    os.path.join(ROOT, "include", "swamp_gpu.h"),
    os.path.join(ROOT, "include", "swamp_io.h"),
    os.path.join(ROOT, "include", "swamp", "zorder.hpp"),
]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo",
    "--fmad=false",          # DESIGN.md D2: no contraction, bit parity with the oracle
    "-std=c++20",
    "-Xcompiler", "-fPIC", "-shared",
    "-Xptxas", "-v",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", shutil.which("nvcc")):
        if c and os.path.exists(c):
            return c
    raise RuntimeError("nvcc not found")


def _stale(target, deps) -> bool:
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build_gpu(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale(LIB, DEPS):
        return LIB
    cmd = [nvcc(), *NVCC_FLAGS, "-I", os.path.join(ROOT, "include"), "-o", LIB, *SOURCES]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed:\n{' '.join(cmd)}\n{r.stdout}\n{r.stderr}")
    with open(os.path.join(HERE, "ptxas_info.txt"), "w") as f:
        f.write(r.stderr)
    if verbose:
        print(r.stderr, file=sys.stderr)
    return LIB


def build_oracle(force: bool = False) -> None:
    d = os.path.join(ROOT, "oracle")
    args = ["make", "-C", d]
    if force:
        args.append("-B")
    r = subprocess.run(args, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"oracle build failed:\n{r.stdout}\n{r.stderr}")


def build_all(force: bool = False) -> None:
    build_gpu(force)
    build_oracle(force)


if __name__ == "__main__":
    build_all(force="--force" in sys.argv)
    print(LIB)
