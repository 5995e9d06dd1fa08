"""Build libpa.so (the C-ABI library of include/pa.h) for sm_100a, in-tree.

    python paper_1805_02372_b200/build.py [--force] [--verbose]

(run as a script or load it by path: importing the package itself loads
libpa.so, so the builder must not depend on the package being importable)

Compiles every .cu under csrc/ with nvcc
(-gencode arch=compute_100a,code=sm_100a -lineinfo -O3) and links one shared
library next to this file.  Rebuilds only when a source is newer than the .so.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
LIB = os.environ.get("PA_LIB_OUT", os.path.join(HERE, "libpa.so"))
# the developer build: honours the PA_* environment overrides of plan and kernel variants
# (tools/dev/, and the tests of the opt-in variants); the product libpa.so ignores them
DEV_LIB = os.path.join(HERE, "libpa_dev.so")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC,-O2",
         "-Xptxas", "-O3", "--expt-relaxed-constexpr"] + os.environ.get("PA_NVCC_EXTRA", "").split()


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh"))) \
        + [os.path.join(INCLUDE, "pa.h")]


def stale(lib: str) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(d) > t for d in deps())


def build(force: bool = False, verbose: bool = False, dev: bool | None = None) -> str:
    """Compile and link the product library (dev=False) or the PA_DEV developer build."""
    from concurrent.futures import ThreadPoolExecutor
    if dev is None:
        dev = os.environ.get("PA_DEV", "0") == "1"
    lib = os.environ.get("PA_LIB_OUT", DEV_LIB) if dev else LIB
    if not force and not stale(lib):
        return lib
    objdir = os.path.join(HERE, "build_dev" if dev else "build")
    os.makedirs(objdir, exist_ok=True)
    flags = FLAGS + (["-DPA_DEV"] if dev else [])

    def compile_one(src):
        obj = os.path.join(objdir, os.path.basename(src).replace(".cu", ".o"))
        cmd = [NVCC, *ARCH, *flags, "-I", INCLUDE, "-c", src, "-o", obj]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.check_call(cmd)
        return obj
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    tmp = lib + ".tmp%d" % os.getpid()
    subprocess.check_call([NVCC, *ARCH, "-shared", "-cudart", "shared", "-o", tmp, *objs])
    os.replace(tmp, lib)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, dev="--dev" in sys.argv or None))
