"""Build libfg.so in-tree for sm_100a (nvcc -shared), so it travels to the GPU box."""
from __future__ import annotations

import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIBFG = os.path.join(HERE, "libfg.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) +
                              glob.glob(os.path.join(CSRC, "*.cuh")) +
                              [os.path.join(ROOT, "include", "fg.h")])


def build_libfg(force: bool = False, verbose: bool = False) -> str:
    if not force and os.path.exists(LIBFG):
        t = os.path.getmtime(LIBFG)
        if all(os.path.getmtime(d) <= t for d in deps()):
            return LIBFG
    cmd = ["nvcc", "-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2",
           "-shared", "-cudart", "static", "-I", os.path.join(ROOT, "include"),
           "-Xptxas", "-v" if verbose else "-O3", "-o", LIBFG, *sources()]
    subprocess.check_call(cmd)
    return LIBFG


if __name__ == "__main__":
    import sys
    print(build_libfg(force=True, verbose="-v" in sys.argv))
