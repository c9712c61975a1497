"""Build libfg.so in-tree for sm_100a (nvcc), so it travels to the GPU box.

Each csrc/*.cu is compiled to an object in parallel (the multi-row kernel's layouts
live in separate translation units), then linked with the static CUDA runtime.
"""
from __future__ import annotations

import concurrent.futures as cf
import glob
import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
OBJ = os.path.join(ROOT, "build", "libfg")
LIBFG = os.path.join(HERE, "libfg.so")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", *ARCH, "-lineinfo", "-Xcompiler", "-fPIC,-O2",
         "-I", os.path.join(ROOT, "include")]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def headers():
    return sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) +
                  [os.path.join(ROOT, "include", "fg.h")])


def _compile(src: str, verbose: bool) -> str:
    obj = os.path.join(OBJ, os.path.basename(src) + ".o")
    newest_dep = max(os.path.getmtime(p) for p in headers() + [src])
    if os.path.exists(obj) and os.path.getmtime(obj) >= newest_dep and not verbose:
        return obj
    cmd = ["nvcc", *FLAGS, "-c", src, "-o", obj] + (["-Xptxas", "-v"] if verbose else [])
    subprocess.check_call(cmd)
    return obj


def build_libfg(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(OBJ, exist_ok=True)
    srcs = sources()
    if not force and os.path.exists(LIBFG):
        t = os.path.getmtime(LIBFG)
        if all(os.path.getmtime(d) <= t for d in srcs + headers()):
            return LIBFG
    if force:
        for o in glob.glob(os.path.join(OBJ, "*.o")):
            os.unlink(o)
    with cf.ThreadPoolExecutor(max_workers=max(2, os.cpu_count() or 2)) as ex:
        objs = list(ex.map(lambda s: _compile(s, verbose), srcs))
    subprocess.check_call(["nvcc", *ARCH, "-shared", "-cudart", "static", "-o", LIBFG, *objs])
    return LIBFG


if __name__ == "__main__":
    import sys
    print(build_libfg(force=True, verbose="-v" in sys.argv))
