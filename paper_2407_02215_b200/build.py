"""Builds libcbtm.so (the C-ABI CUDA library) in-tree with nvcc for sm_100a."""

from __future__ import annotations

import os
import shutil
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libcbtm.so")
SOURCES = ["cbtm.cu"]
HEADERS = ["cbtm_common.cuh", "cbtm_cbt.cuh", "cbtm_classify.cuh",
           "cbtm_frame.cuh", "cbtm_mesh.cuh", os.path.join("..", "..", "include", "cbtm.h")]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-fmad=false",          # fp64 classifier must round like the reference (no FMA)
    "--shared", "-Xcompiler", "-fPIC",
    "-Xptxas", "-v",
]


def nvcc_path() -> str:
    for cand in (shutil.which("nvcc"), "/usr/local/cuda/bin/nvcc"):
        if cand and os.path.exists(cand):
            return cand
    raise RuntimeError("nvcc not found: libcbtm.so cannot be built")


def is_stale() -> bool:
    if not os.path.exists(LIB):
        return True
    built = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, f) for f in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > built for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not is_stale():
        return LIB
    cmd = [nvcc_path(), *NVCC_FLAGS, "-o", LIB,
           *[os.path.join(CSRC, f) for f in SOURCES]]
    env = dict(os.environ)
    # some images export CC/CXX pointing at a wrapper nvcc cannot drive
    proc = subprocess.run(cmd + ["-ccbin", "/usr/bin/g++"], capture_output=True,
                          text=True, env=env)
    if proc.returncode != 0:
        sys.stderr.write(proc.stdout + proc.stderr)
        raise RuntimeError("nvcc failed building libcbtm.so")
    if verbose:
        sys.stderr.write(proc.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
