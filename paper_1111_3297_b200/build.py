"""Compile the sm_100a extension in-tree (no JIT cache: the .so travels with the repo).

    python -m paper_1111_3297_b200.build
"""
from __future__ import annotations

import os
import subprocess
import sys

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
SO = os.path.join(PKG, "liberato_gpu.so")
CLI = os.path.join(PKG, "erato-gpu")
CLI_SRC = os.path.join(PKG, "csrc", "erato_cli.cpp")
SOURCES = [os.path.join(PKG, "csrc", "erato_gpu.cu")]
DEPS = SOURCES + [os.path.join(PKG, "csrc", "sieve_kernels.cuh"), os.path.join(ROOT, "include", "erato_gpu.h")]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC",
]


def nvcc() -> str:
    for c in (os.environ.get("NVCC"), "/usr/local/cuda/bin/nvcc", "nvcc"):
        if c and (os.path.isabs(c) and os.path.exists(c) or not os.path.isabs(c)):
            return c
    return "nvcc"


def up_to_date() -> bool:
    if not os.path.exists(SO):
        return False
    t = os.path.getmtime(SO)
    return all(os.path.getmtime(d) <= t for d in DEPS)


def build_cli(verbose: bool = False) -> str:
    """erato-gpu: the reference CLI contract (tools/erato.cpp) over liberato_gpu.so."""
    cmd = ["g++", "-O2", "-std=c++17", CLI_SRC, "-o", CLI, f"-L{PKG}", "-lerato_gpu", "-Wl,-rpath,$ORIGIN"]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    return CLI


def build(force: bool = False, verbose: bool = False, debug: bool = False) -> str:
    so = SO.replace(".so", "_debug.so") if debug else SO
    if not force and not debug and up_to_date() and os.path.exists(CLI) \
            and os.path.getmtime(CLI) >= os.path.getmtime(CLI_SRC):
        return SO
    cmd = [nvcc(), *NVCC_FLAGS, *(["-DEG_DEBUG"] if debug else []), "-o", so, *SOURCES]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.run(cmd, check=True)
    if not debug:
        build_cli(verbose)
    return so


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True, debug="--debug" in sys.argv))
