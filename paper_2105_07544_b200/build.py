"""Build libmpkb200.so for sm_100a in-tree (``python -m paper_2105_07544_b200.build``).

nvcc flags: -gencode arch=compute_100a,code=sm_100a, -O3, -lineinfo, no
fast-math (IEEE division/sqrt, subnormals kept), host code without FP
contraction, static cudart (no clash with torch's bundled runtime).
"""

from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
SRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "_lib", "libmpkb200.so")
SOURCES = ["abi.cu", "host_rcm.cpp"]
DEPS = ["abi.cu", "host_rcm.cpp", "fused.cuh", "fused_reg.cuh", "fused_dcgs2.cuh", "kernels.cuh", "ops.cuh", "common.cuh", "comm.cuh", "../../include/mpk_b200.h"]


def nvcc() -> str:
    for cand in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if cand and (os.path.isabs(cand) and os.path.exists(cand) or not os.path.isabs(cand)):
            return cand
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(OUT):
        return False
    t = os.path.getmtime(OUT)
    return all(os.path.getmtime(os.path.join(SRC, d)) <= t for d in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and up_to_date():
        return OUT
    os.makedirs(os.path.dirname(OUT), exist_ok=True)
    cmd = [nvcc(), "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
           "-Xcompiler", "-fPIC,-ffp-contract=off", "-cudart", "static", "-shared",
           "-o", OUT + ".tmp"] + [os.path.join(SRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    if os.environ.get("MPK_SPLIT_COMPILE"):
        # development builds only: parallel cicc/ptxas changes code generation
        # (measured: different stack frames), so shipped builds never use it
        cmd.insert(1, "--split-compile=%s" % os.environ["MPK_SPLIT_COMPILE"])
    subprocess.run(cmd, check=True)
    os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
