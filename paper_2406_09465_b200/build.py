"""Build libkorch.so in-tree (host C++; kernels are generated and compiled for
sm_100a at run time with NVRTC, or ahead of time by `precompile`)."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libkorch.so")
SOURCES = ["ir.cpp", "enumerate.cpp", "expr.cpp", "codegen.cpp", "gemm_gen.cpp", "cuda_api.cpp", "korch_api.cpp"]
CUDA_HOME = os.environ.get("CUDA_HOME", "/usr/local/cuda")


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    for f in os.listdir(CSRC):
        if os.path.getmtime(os.path.join(CSRC, f)) > t:
            return True
    return os.path.getmtime(os.path.join(HERE, "..", "include", "korch.h")) > t


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    objs = []
    os.makedirs(os.path.join(HERE, "build"), exist_ok=True)
    procs = []
    for s in SOURCES:
        o = os.path.join(HERE, "build", s.replace(".cpp", ".o"))
        cmd = ["g++", "-std=c++17", "-O2", "-g", "-fPIC", "-Wall", "-Wno-unused-function",
               f"-I{CUDA_HOME}/include", "-c", os.path.join(CSRC, s), "-o", o]
        procs.append((cmd, subprocess.Popen(cmd, stdout=subprocess.PIPE, stderr=subprocess.STDOUT)))
        objs.append(o)
    for cmd, p in procs:
        out, _ = p.communicate()
        if p.returncode != 0:
            raise RuntimeError("compile failed: " + " ".join(cmd) + "\n" + out.decode())
        if verbose and out:
            print(out.decode(), file=sys.stderr)
    tmp = LIB + ".tmp"
    cmd = ["g++", "-shared", "-o", tmp] + objs + ["-ldl", "-lpthread"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError("link failed: " + r.stderr)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose=True))
