"""Build libs3.so (CUDA kernels + C++ control plane) in-tree for sm_100a."""
from __future__ import annotations

import os
import subprocess
import sys

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIBDIR = os.path.join(HERE, "lib")
LIB = os.path.join(LIBDIR, "libs3.so")
INCLUDE = os.path.join(os.path.dirname(HERE), "include")
SOURCES = [os.path.join(CSRC, "s3_kernels.cu"), os.path.join(CSRC, "s3_attn_tc.cu"),
           os.path.join(CSRC, "s3_gemm.cu"), os.path.join(CSRC, "s3_host.cpp")]
DEPS = SOURCES + [os.path.join(CSRC, "s3_internal.h"), os.path.join(INCLUDE, "s3.h")]

NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-lineinfo", "-O3", "-std=c++17",
    "-Xcompiler", "-fPIC,-O3", "-shared",
    "-cudart", "static",
    "-I", INCLUDE,
    "-ldl",
]


def needs_build() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    return any(os.path.getmtime(p) > t for p in DEPS)


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not needs_build():
        return LIB
    os.makedirs(LIBDIR, exist_ok=True)
    tmp = LIB + f".tmp{os.getpid()}"
    cmd = [NVCC, *FLAGS, *(["-Xptxas", "-v"] if verbose else []), "-o", tmp, *SOURCES]
    subprocess.check_call(cmd)
    os.replace(tmp, LIB)
    return LIB


if __name__ == "__main__":
    print(build(force="--force" in sys.argv, verbose="-v" in sys.argv))
