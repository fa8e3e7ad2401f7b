"""Build the native libraries in-tree with nvcc for sm_100a (no JIT cache, no
torch extension machinery): the .so files travel with the repo snapshot to
the GPU box.

* libconv.so        -- the convolution library (include/conv.h): csrc/*
* libconv_probes.so -- the bench-only peak probes (include/conv_probes.h)

Each translation unit is compiled to an object in parallel, then linked."""
from __future__ import annotations

import glob
import os
import subprocess
from concurrent.futures import ThreadPoolExecutor

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
PROBES = os.path.join(HERE, "probes")
LIB = os.path.join(HERE, "libconv.so")
PROBES_LIB = os.path.join(HERE, "libconv_probes.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
OBJ = os.path.join(os.path.dirname(HERE), "build", "obj")

ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
CFLAGS = [*ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC", "-Xcompiler", "-fvisibility=hidden"]
LDFLAGS = [*ARCH, "-shared", "-cudart", "static"]
# kept for scripts that compile single files the same way
NVCC_FLAGS = [*CFLAGS, "-shared", "-cudart", "static"]


def sources(d: str = CSRC):
    return sorted(glob.glob(os.path.join(d, "*.cu")) + glob.glob(os.path.join(d, "*.cpp")))


def _headers():
    return glob.glob(os.path.join(CSRC, "*.h")) + glob.glob(os.path.join(CSRC, "*.cuh")) \
        + glob.glob(os.path.join(CSRC, "*.inc")) + glob.glob(os.path.join(INCLUDE, "*.h"))


def deps():
    return sources() + _headers()


def _stale(lib: str, files) -> bool:
    if not os.path.exists(lib):
        return True
    t = os.path.getmtime(lib)
    return any(os.path.getmtime(f) > t for f in files)


def needs_build() -> bool:
    return _stale(LIB, deps()) or _stale(PROBES_LIB, sources(PROBES) + _headers())


def _link(nvcc: str, lib: str, srcs, extra, verbose: bool, tag: str):
    os.makedirs(OBJ, exist_ok=True)

    def compile_one(src):
        obj = os.path.join(OBJ, f"{tag}_{os.path.basename(src)}.o")
        cmd = [nvcc, *CFLAGS, *extra, "-c", "-o", obj, src]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
        return obj

    with ThreadPoolExecutor(max_workers=max(1, min(len(srcs), os.cpu_count() or 1))) as ex:
        objs = list(ex.map(compile_one, srcs))
    cmd = [nvcc, *LDFLAGS, "-o", lib + ".tmp", *objs]
    if verbose:
        print(" ".join(cmd), flush=True)
    subprocess.check_call(cmd)
    os.replace(lib + ".tmp", lib)


def build(force: bool = False, verbose: bool = False) -> str:
    nvcc = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
    # CONV_BUILD_TRACE=1: a trace build (kernel timeline instrumentation,
    # env CONV_TRACE at run time; scripts/trace_tc.py) -- study only
    extra = ["-DCONV_ENABLE_TRACE=1"] if os.environ.get("CONV_BUILD_TRACE") == "1" else []
    if force or _stale(LIB, deps()):
        _link(nvcc, LIB, sources(), extra, verbose, "conv")
    if force or _stale(PROBES_LIB, sources(PROBES) + _headers()):
        _link(nvcc, PROBES_LIB, sources(PROBES), [], verbose, "probes")
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
