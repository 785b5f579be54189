"""Builds the in-tree CUDA/C++ shared library libtgnn_b200.so for sm_100a.

nvcc cross-compiles without a GPU; the .so lands next to this file so it
travels with the repository snapshot to the GPU box.
"""
from __future__ import annotations

import concurrent.futures as cf
import hashlib
import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
OUT = os.path.join(HERE, "libtgnn_b200.so")
OBJ = os.path.join(HERE, "build")
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]
FLAGS = ["-O3", "-std=c++17", "-lineinfo", "-Xcompiler", "-fPIC", "-Xcompiler", "-O2",
         "--expt-relaxed-constexpr", "-I", CSRC, "-I", os.path.join(HERE, "..", "include")]
SOURCES = ["plan.cu", "gemm_simt.cu", "gemm_tc.cu", "gemm_tma.cu", "gru_fused.cu", "step.cu", "graph.cu", "api.cu",
           "host/dataset.cpp"]
CXX = os.environ.get("TGNN_HOST_CXX", "g++")
CXXFLAGS = ["-O2", "-std=c++20", "-fPIC", "-pthread", "-g", "-I", CSRC, "-I", "/usr/local/cuda/include"]


def _deps_hash(src: str) -> str:
    h = hashlib.sha1()
    for root, _, files in os.walk(CSRC):
        for f in sorted(files):
            if f.endswith((".cuh", ".hpp", ".h")):
                h.update(open(os.path.join(root, f), "rb").read())
    h.update(open(os.path.join(HERE, "..", "include", "tgnn_b200.h"), "rb").read())
    h.update(open(os.path.join(CSRC, src), "rb").read())
    h.update(" ".join(ARCH + FLAGS + CXXFLAGS).encode())
    return h.hexdigest()[:16]


def _compile(src: str) -> str:
    os.makedirs(OBJ, exist_ok=True)
    obj = os.path.join(OBJ, f"{src.replace('/', '_')}.{_deps_hash(src)}.o")
    if os.path.exists(obj):
        return obj
    if src.endswith(".cpp"):
        cmd = [CXX, *CXXFLAGS, "-c", os.path.join(CSRC, src), "-o", obj + ".tmp"]
    else:
        cmd = [NVCC, *ARCH, *FLAGS, "-c", os.path.join(CSRC, src), "-o", obj + ".tmp"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"nvcc failed for {src}:\n{r.stdout}\n{r.stderr}")
    os.replace(obj + ".tmp", obj)
    return obj


def build(verbose: bool = False) -> str:
    with cf.ThreadPoolExecutor(max_workers=len(SOURCES)) as ex:
        objs = list(ex.map(_compile, SOURCES))
    stamp = hashlib.sha1("".join(objs).encode()).hexdigest()[:16]
    stamp_file = OUT + ".stamp"
    if os.path.exists(OUT) and os.path.exists(stamp_file) and open(stamp_file).read() == stamp:
        return OUT
    cmd = [NVCC, *ARCH, "-shared", "-o", OUT + ".tmp", *objs, "-ldl", "-lpthread", "-cudart", "static",
           "-Xlinker", "--no-undefined"]
    r = subprocess.run(cmd, capture_output=True, text=True)
    if r.returncode != 0:
        raise RuntimeError(f"link failed:\n{r.stdout}\n{r.stderr}")
    os.replace(OUT + ".tmp", OUT)
    open(stamp_file, "w").write(stamp)
    if verbose:
        print("built", OUT)
    return OUT


if __name__ == "__main__":
    print(build(verbose=True))
    sys.exit(0)
