"""Build libgpulet.so in-tree with nvcc for sm_100a (B200).

    python -m paper_2109_01611_b200.build          # incremental
    python -m paper_2109_01611_b200.build --force

The library is the product: the executor kernel, the layer kernels, the
program builders, the runtime and the native scheduler.  cudart is linked
statically; driver entry points are resolved at run time through cudart, so the
.so loads on a machine without a GPU (for the export checks).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libgpulet.so")
BUILD = os.path.join(HERE, "_build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
COMMON = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-Wall"]

SOURCES = [
    ("executor.cu", []),
    ("detect.cu", []),
    ("probe.cu", []),
    ("runtime.cpp", []),
    ("models.cpp", []),
    ("frontend.cpp", []),
    ("sched.cpp", ["-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-fno-fast-math"]),
    ("workload.cpp", ["-Xcompiler", "-ffp-contract=off", "-Xcompiler", "-fno-fast-math"]),
]
HEADERS = ["program.h", "ptx.cuh", "runtime.h"]


def _mtime(p):
    return os.path.getmtime(p) if os.path.exists(p) else 0.0


def build(force=False, verbose=True):
    os.makedirs(BUILD, exist_ok=True)
    hdr_t = max([_mtime(os.path.join(CSRC, h)) for h in HEADERS] +
                [_mtime(os.path.join(HERE, "..", "include", "gpulet.h"))])
    objs = []
    for src, extra in SOURCES:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        objs.append(o)
        if force or _mtime(o) < max(_mtime(s), hdr_t):
            cmd = [NVCC, *ARCH, *COMMON, *extra, "-c", s, "-o", o]
            if verbose:
                print(" ".join(cmd), flush=True)
            subprocess.check_call(cmd)
    if force or _mtime(LIB) < max(_mtime(o) for o in objs):
        cmd = [NVCC, *ARCH, "-shared", "-o", LIB, *objs, "-lpthread", "-ldl", "-lrt"]
        if verbose:
            print(" ".join(cmd), flush=True)
        subprocess.check_call(cmd)
    return LIB


if __name__ == "__main__":
    build(force="--force" in sys.argv)
