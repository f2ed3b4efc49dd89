"""Build the in-tree C-ABI library `csrc/liblobe.so` for sm_100a.

nvcc -gencode arch=compute_100a,code=sm_100a -lineinfo -fmad=false for the
kernels (no fast math, no FTZ: the bit-exact contract of DESIGN.md), g++ with
-ffp-contract=off for the host runtime. The .so stays in-tree (it travels to
the GPU box with the repo snapshot).
"""
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(CSRC, "liblobe.so")
BUILD = os.path.join(CSRC, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
CUDA_INC = "/usr/local/cuda/include"
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
SOURCES_CU = ["lobe_kernels.cu"]
SOURCES_CPP = ["lobe_api.cpp", "lobe_bo.cpp", "lobe_comm.cpp"]
HEADERS = ["lobe_internal.h", "lobe_comm.h", os.path.join("..", "..", "include", "lobe.h")]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    print(" ".join(cmd), file=sys.stderr)
    subprocess.check_call(cmd)


def build(force=False, verbose_ptxas=False):
    os.makedirs(BUILD, exist_ok=True)
    deps_h = [os.path.join(CSRC, h) for h in HEADERS]
    objs = []
    for src in SOURCES_CU:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _newer(o, [s] + deps_h):
            cmd = [NVCC, *ARCH, "-O3", "-lineinfo", "-fmad=false", "-std=c++17", "-Xcompiler", "-fPIC",
                   "-Xcompiler", "-ffp-contract=off", "-c", s, "-o", o]
            if verbose_ptxas:
                cmd.insert(1, "-Xptxas=-v")
            _run(cmd)
        objs.append(o)
    for src in SOURCES_CPP:
        s = os.path.join(CSRC, src)
        o = os.path.join(BUILD, src + ".o")
        if force or _newer(o, [s] + deps_h):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-fno-fast-math", "-Wall",
                  "-Wno-unused-function", "-I", CUDA_INC, "-c", s, "-o", o])
        objs.append(o)
    if force or _newer(OUT, objs):
        _run([NVCC, *ARCH, "-shared", "-o", OUT + ".tmp", *objs, "-ldl"])
        os.replace(OUT + ".tmp", OUT)
    return OUT


if __name__ == "__main__":
    build(force="--force" in sys.argv, verbose_ptxas="-v" in sys.argv)
