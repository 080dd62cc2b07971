"""Build libfdtdrom.so in-tree with nvcc for sm_100a (no JIT cache; the .so travels with the repo)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libfdtdrom.so")
SOURCES = ["fdtd_kernels.cu", "fdtd_api.cpp", "rom_build.cu"]
HEADERS = ["fdtd_kernels.cuh", "dense.hpp"]
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _inputs():
    return [os.path.join(CSRC, s) for s in SOURCES + HEADERS] + [os.path.join(ROOT, "include", "fdtdrom.h"), os.path.join(ROOT, "include", "fdtdrom_build.h"),
                                                              os.path.abspath(__file__)]


def up_to_date() -> bool:
    if not os.path.exists(LIB):
        return False
    t = os.path.getmtime(LIB)
    return all(os.path.getmtime(p) <= t for p in _inputs())


def build(force: bool = False, verbose: bool = False, out: str = LIB, defines=()) -> str:
    if out == LIB and not force and up_to_date():
        return LIB
    tmp = out + ".tmp%d" % os.getpid()
    cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O3", "-shared",
           "-Xptxas", "-v" if verbose else "-O3", "-I", os.path.join(ROOT, "include"), "-I", CSRC,
           *["-D" + d for d in defines], *[os.path.join(CSRC, s) for s in SOURCES], "-o", tmp, "-ldl"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError("nvcc failed building libfdtdrom.so")
    if verbose:
        sys.stderr.write(r.stderr)
    os.replace(tmp, out)
    return out


CHECK_LIB = os.path.join(HERE, "libfdtdrom_check.so")


def build_checked(force: bool = False) -> str:
    """The checked build (-DFDTD_CHECK=1: device-side bounds checks; tools/checked_run.py)."""
    if not force and os.path.exists(CHECK_LIB) and all(os.path.getmtime(p) <= os.path.getmtime(CHECK_LIB)
                                                       for p in _inputs()):
        return CHECK_LIB
    return build(force=True, out=CHECK_LIB, defines=("FDTD_CHECK=1",))


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
    if "--checked" in sys.argv:
        print(build_checked(force="--force" in sys.argv))
