"""In-tree build of libgridse_b200.so (nvcc, sm_100a only)."""

from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgridse_b200.so")
SOURCES = ["symbolic.cpp", "partition.cpp", "kernels.cu", "front_kernels.cu", "solve_kernel.cu", "api.cu"]
HEADERS = ["plan.hpp", "kernels.cuh", "unit_bodies.cuh", "front_body.cuh", os.path.join("..", "..", "include", "gridse_b200.h")]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC", "-Xcompiler", "-O2", "-diag-suppress", "39,179",
]


def needs_build():
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, s) for s in SOURCES + HEADERS]
    return any(os.path.getmtime(d) > t for d in deps)


def build(force=False, verbose=False):
    """Compile the CUDA/C++ sources into the shared library; returns its path."""
    if not force and not needs_build():
        return LIB
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    extra = os.environ.get("GSE_NVCC_DEFINES", "").split()      # e.g. "-DGSE_XPOLL_NS=100" (development A/B builds)
    objs = []
    for src in SOURCES:
        obj = os.path.join(CSRC, os.path.splitext(src)[0] + ".o")
        cmd = [nvcc, *NVCC_FLAGS, *extra, "-c", os.path.join(CSRC, src), "-o", obj]
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        subprocess.run(cmd, check=True)
        objs.append(obj)
    subprocess.run([nvcc, "-shared", "-o", LIB, *objs, "-gencode", "arch=compute_100a,code=sm_100a",
                    "-lcudart", "-lpthread"], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
