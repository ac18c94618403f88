"""Builds libhelios.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with gpurun)."""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
SO = os.path.join(HERE, "libhelios.so")
SO_TRACE = os.path.join(HERE, "libhelios_trace.so")  # -DHELIOS_TRACE: device pipeline timeline (tools)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources() -> list[str]:
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps() -> list[str]:
    return sources() + glob.glob(os.path.join(CSRC, "*.cuh")) + [os.path.join(HERE, "..", "include", "helios.h")]


def _build_one(so: str, defines: list[str], force: bool, verbose: bool) -> str:
    if not force and os.path.exists(so) and all(os.path.getmtime(so) >= os.path.getmtime(d) for d in deps()):
        return so
    cmd = [NVCC, "-O3", "-std=c++17", *ARCH, "-lineinfo", "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
           "-Xcompiler", "-pthread", "--expt-relaxed-constexpr", *defines, "-o", so, *sources()]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)
    return so


def build(force: bool = False, verbose: bool = False, trace: bool = True) -> str:
    """libhelios.so (the product) and, unless trace=False, libhelios_trace.so (same sources with the
    device pipeline tracer compiled in)."""
    _build_one(SO, [], force, verbose)
    if trace:
        _build_one(SO_TRACE, ["-DHELIOS_TRACE"], force, verbose)
    return SO


if __name__ == "__main__":
    build(force="-f" in sys.argv, verbose="-v" in sys.argv)
