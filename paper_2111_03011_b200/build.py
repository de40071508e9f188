"""Build libtnb200.so in-tree: host C++ (g++) + sm_100a CUDA (nvcc), linked against static cudart.

    python -m paper_2111_03011_b200.build [--force]
"""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
BUILD = os.path.join(HERE, "_build")
LIB = os.path.join(HERE, "libtnb200.so")
CUDA = os.environ.get("CUDA_HOME", "/usr/local/cuda")
NVCC = os.path.join(CUDA, "bin", "nvcc")

CXX_SRCS = ["network.cpp", "planner.cpp", "partition.cpp", "planfile.cpp", "lower.cpp", "api.cpp"]
CU_SRCS = ["executor.cu"]
HEADERS = ["tnb.h", "exec.h", "kernels.cuh", "gemm_tc.cuh", "gate_tc.cuh"]
GENCODE = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _newer(target, deps):
    if not os.path.exists(target):
        return True
    t = os.path.getmtime(target)
    return any(os.path.getmtime(d) > t for d in deps)


def _run(cmd):
    r = subprocess.run(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT, text=True)
    if r.returncode != 0:
        sys.stderr.write(" ".join(cmd) + "\n" + r.stdout)
        raise RuntimeError(f"build step failed: {cmd[0]} {cmd[-1]}")
    return r.stdout


def build(force: bool = False, verbose: bool = False) -> str:
    os.makedirs(BUILD, exist_ok=True)
    hdrs = [os.path.join(CSRC, h) for h in HEADERS] + [os.path.join(HERE, "..", "include", "tn.h"),
                                                     os.path.join(HERE, "..", "include", "tn_debug.h")]
    objs = []
    for s in CXX_SRCS:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        if force or _newer(obj, [src] + hdrs):
            _run(["g++", "-O2", "-std=c++17", "-fPIC", "-ffp-contract=off", "-Wall", "-Wno-unused-function",
                  f"-I{CUDA}/include", "-c", src, "-o", obj])
        objs.append(obj)
    extra = os.environ.get("TNB_NVCC_FLAGS", "").split()  # diagnostics builds, e.g. -DTNB_CHAIN_CLOCK
    for s in CU_SRCS:
        src = os.path.join(CSRC, s)
        obj = os.path.join(BUILD, s + ".o")
        # the flag string is stored next to the object: a change of TNB_NVCC_FLAGS forces a rebuild (a
        # diagnostics object is never reused silently)
        stamp = obj + ".flags"
        flags_changed = not os.path.exists(stamp) or open(stamp).read() != " ".join(extra)
        if force or flags_changed or _newer(obj, [src] + hdrs):
            out = _run([NVCC, *GENCODE, "-O3", "-lineinfo", "-std=c++17", "-Xcompiler", "-fPIC",
                        "-Xptxas", "-v", "--expt-relaxed-constexpr", *extra, "-c", src, "-o", obj])
            if verbose:
                print(out)
            with open(os.path.join(BUILD, s + ".ptxas.txt"), "w") as f:
                f.write(out)
            with open(stamp, "w") as f:
                f.write(" ".join(extra))
        objs.append(obj)
    if force or _newer(LIB, objs):
        _run(["g++", "-shared", "-o", LIB, *objs, f"-L{CUDA}/lib64", "-lcudart_static", "-ldl", "-lrt", "-lpthread"])
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
