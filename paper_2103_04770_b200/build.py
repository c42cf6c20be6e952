"""Build libfgd.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2103_04770_b200.build [--verbose]

The shared library is written next to this file (git-ignored, but it travels to the GPU box
with the repo snapshot).  Rebuilds only when a source is newer than the library.
"""
from __future__ import annotations

import glob
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")


def _nccl_dir():
    import importlib.util
    spec = importlib.util.find_spec("nvidia")
    for base in (list(spec.submodule_search_locations) if spec else []):
        d = os.path.join(base, "nccl")
        if os.path.exists(os.path.join(d, "include", "nccl.h")):
            return d
    raise RuntimeError("NCCL headers not found (nvidia-nccl wheel)")


LIB = os.path.join(HERE, "libfgd.so")
LIB_JITTER = os.path.join(HERE, "libfgd_jitter.so")   # race-hunting build (-DFGD_JITTER, tests only)
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def sources():
    return sorted(glob.glob(os.path.join(CSRC, "*.cu")))


def deps():
    return sources() + sorted(glob.glob(os.path.join(CSRC, "*.cuh"))) + [os.path.join(INCLUDE, "fgd.h")]


def up_to_date(lib=LIB) -> bool:
    if not os.path.exists(lib):
        return False
    t = os.path.getmtime(lib)
    return all(os.path.getmtime(d) <= t for d in deps())


def build(force: bool = False, verbose: bool = False, jitter: bool = False) -> str:
    lib = LIB_JITTER if jitter else LIB
    if not force and up_to_date(lib):
        return lib
    def compile_one(src):
        obj = os.path.join(CSRC, os.path.basename(src)[:-3] + ("_jit.o" if jitter else ".o"))
        cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-I", INCLUDE,
               "-I", os.path.join(_nccl_dir(), "include"), "--expt-relaxed-constexpr", "-c", src, "-o", obj]
        if jitter:
            cmd.insert(1, "-DFGD_JITTER")
        if verbose:
            cmd.insert(1, "-Xptxas=-v")
        r = subprocess.run(cmd, capture_output=True, text=True)
        if r.returncode != 0:
            raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
        if verbose:
            sys.stderr.write(r.stderr)
        return obj

    from concurrent.futures import ThreadPoolExecutor
    with ThreadPoolExecutor(max_workers=min(8, os.cpu_count() or 1)) as ex:
        objs = list(ex.map(compile_one, sources()))
    nlib = os.path.join(_nccl_dir(), "lib")
    cmd = [NVCC, *ARCH, "-shared", "-cudart", "static", "-o", lib, *objs, "-L", nlib, "-l:libnccl.so.2",
           "-Xlinker", "-rpath", "-Xlinker", nlib]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    for o in objs:
        os.remove(o)
    return lib


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="--verbose" in sys.argv, jitter="--jitter" in sys.argv))
