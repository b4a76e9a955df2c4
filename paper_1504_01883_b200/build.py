"""Builds the in-tree CUDA shared library liblbpfused.so for sm_100a with nvcc.

The library is the C ABI of include/lbpfused.h; the Python binding
(paper_1504_01883_b200/lbpfused.py) loads it with ctypes.  It is built in-tree
so that it travels to the GPU box with the repo snapshot.
"""
from __future__ import annotations

import fcntl
import glob
import os
import subprocess

PKG = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(PKG)
CSRC = os.path.join(PKG, "csrc")
INCLUDE = os.path.join(ROOT, "include")
LIB = os.path.join(PKG, "liblbpfused.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared", "-cudart", "static",
    "--expt-relaxed-constexpr",
    "-Xptxas", "-v",
]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [
        os.path.join(INCLUDE, "lbpfused.h"), __file__]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in deps())


def build(force: bool = False, verbose: bool = False) -> str:
    """Compile when the library is missing or older than a source.  Concurrent callers (one
    process per GPU) serialise on a lock file; the library is written to a temporary name and
    renamed into place, so a loader never sees a partial file."""
    if not force and not needs_build():
        return LIB
    with open(LIB + ".lock", "w") as lock:
        fcntl.flock(lock, fcntl.LOCK_EX)
        if not force and not needs_build():  # built by another process meanwhile
            return LIB
        extra = os.environ.get("LBP_NVCC_EXTRA", "").split()  # developer A/B builds only
        tmp = f"{LIB}.tmp{os.getpid()}"
        cmd = [NVCC, *NVCC_FLAGS, *extra, "-I", INCLUDE, "-I", CSRC, "-o", tmp, *sources()]
        res = subprocess.run(cmd, capture_output=True, text=True)
        log = os.path.join(PKG, "build.log")
        with open(log, "w") as f:
            f.write(" ".join(cmd) + "\n" + res.stdout + res.stderr)
        if res.returncode != 0:
            raise RuntimeError(f"nvcc failed (see {log}):\n{res.stderr[-4000:]}")
        os.replace(tmp, LIB)
    if verbose:
        print(res.stderr)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
