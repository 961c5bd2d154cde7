"""Build libisdc.so in-tree for sm_100a (nvcc cross-compiles without a GPU).

    python -m paper_1401_7824_b200.build [--force]
"""
from __future__ import annotations

import glob
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "build")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libisdc.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
# --fmad=false: no FMA contraction anywhere on the device path (bit-identical to the oracle,
# DESIGN.md §4); -ffp-contract=off for the host-side scalar coefficients.
NVFLAGS = ["-O3", "-lineinfo", "--fmad=false", "-std=c++17", "-Xcompiler", "-fPIC,-ffp-contract=off",
           "-Xptxas", "-v", "-I", INCLUDE]
CXXFLAGS = ["-O2", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-std=gnu++17", "-fext-numeric-literals", "-I", INCLUDE]


def _sources():
    return sorted(glob.glob(os.path.join(CSRC, "*"))) + [os.path.join(INCLUDE, "isdc.h")]


STAMP = LIB + ".sha256"


def source_hash() -> str:
    """SHA-256 over every source file (name + bytes), the compilers' flags and nvcc's version: the
    library is rebuilt whenever any of them differs from the stamp written by the last build (file
    modification times are not trusted: a checkout or a copy can make an old library look new)."""
    h = hashlib.sha256()
    for s in _sources():
        h.update(os.path.basename(s).encode())
        with open(s, "rb") as f:
            h.update(f.read())
    h.update(" ".join(ARCH + NVFLAGS + CXXFLAGS).encode())
    try:
        h.update(subprocess.run([NVCC, "--version"], capture_output=True, text=True).stdout.encode())
    except OSError:
        pass
    return h.hexdigest()


def _stale() -> bool:
    if not os.path.exists(LIB) or not os.path.exists(STAMP):
        return True
    with open(STAMP) as f:
        return f.read().strip() != source_hash()


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    os.makedirs(BUILD, exist_ok=True)
    os.makedirs(LIBDIR, exist_ok=True)
    objs = []
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cpp"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        subprocess.run(["g++", *CXXFLAGS, "-c", src, "-o", obj], check=True)
        objs.append(obj)
    for src in sorted(glob.glob(os.path.join(CSRC, "*.cu"))):
        obj = os.path.join(BUILD, os.path.basename(src) + ".o")
        r = subprocess.run([NVCC, *ARCH, *NVFLAGS, "-c", src, "-o", obj], capture_output=True, text=True)
        with open(os.path.join(BUILD, os.path.basename(src) + ".ptxas.txt"), "w") as f:
            f.write(r.stdout + r.stderr)
        if r.returncode != 0:
            sys.stderr.write(r.stdout + r.stderr)
            raise RuntimeError(f"nvcc failed on {src}")
        if verbose:
            sys.stderr.write(r.stderr)
        objs.append(obj)
    tmp = LIB + ".tmp"
    subprocess.run([NVCC, *ARCH, "-shared", "-o", tmp, *objs, "-lquadmath"], check=True)
    os.replace(tmp, LIB)
    with open(STAMP, "w") as f:
        f.write(source_hash() + "\n")
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose="-v" in sys.argv)
    print(LIB)
