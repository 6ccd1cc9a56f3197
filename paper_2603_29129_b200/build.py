"""Build libozfft.so (sm_100a) in-tree with nvcc + g++.

    python -m paper_2603_29129_b200.build [--force]

The library is the C-ABI boundary declared in include/ozfft.h; the Python binding
(paper_2603_29129_b200/__init__.py) loads it with ctypes.
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libozfft.so")
BUILD = os.path.join(HERE, "_build")
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA_HOME, "bin", "nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]

SOURCES_CU = ["kernels.cu"]
SOURCES_CPP = ["capi.cpp", "plan_host.cpp"]
HEADERS = ["internal.h"]


def _git_rev() -> str:
    try:
        return subprocess.check_output(["git", "-C", ROOT, "rev-parse", "--short", "HEAD"],
                                       stderr=subprocess.DEVNULL).decode().strip()
    except Exception:
        return "nogit"


def _stale(out: str, deps: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(d) > t for d in deps)


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(ROOT, "include", "ozfft.h")]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs + [__file__]):
            extra = os.environ.get("OZFFT_NVCC_EXTRA", "").split()
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "--fmad=false", *extra,
                   "-Xcompiler", "-fPIC", "-Xptxas", "-v" if verbose else "-O3",
                   "-c", s, "-o", o]
            subprocess.check_call(cmd)
        objs.append(o)
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _stale(o, [s] + hdrs + [__file__]):
            cmd = ["g++", "-O2", "-std=gnu++17", "-fPIC", "-ffp-contract=off", "-Wall",
                   f"-DOZFFT_GIT=\"{_git_rev()}\"", f"-I{CUDA_HOME}/include", "-c", s, "-o", o]
            subprocess.check_call(cmd)
        objs.append(o)
    if force or _stale(LIB, objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lquadmath", "-cudart", "static"]
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
