"""Build recipe for liblmc_b200.so (sm_100a, cudart static, in-tree)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
SO = os.path.join(HERE, "liblmc_b200.so")
SRC_DIR = os.path.join(HERE, "csrc")
SOURCES = ["capi.cu", "compress.cu", "decompress.cu", "lmc_common.cuh"]
NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo", "-std=c++17",
    "-shared", "-Xcompiler", "-fPIC", "-cudart", "static",
]


def _stale() -> bool:
    if not os.path.exists(SO):
        return True
    t = os.path.getmtime(SO)
    deps = [os.path.join(SRC_DIR, s) for s in SOURCES]
    deps.append(os.path.join(os.path.dirname(HERE), "include", "lmc_b200.h"))
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if force or _stale():
        nvcc = os.environ.get("NVCC", "nvcc")
        cmd = [nvcc, *NVCC_FLAGS, "-o", SO, os.path.join(SRC_DIR, "capi.cu")]
        if verbose:
            cmd += ["-Xptxas", "-v"]
        subprocess.check_call(cmd)
    return SO


if __name__ == "__main__":
    build(force=True, verbose=True)
    print(SO)
