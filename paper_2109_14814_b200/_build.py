"""In-tree build of libmcx.so for sm_100a (nvcc; no JIT cache, so the .so travels
with the repo snapshot to the GPU box)."""
from __future__ import annotations

import os
import subprocess

HERE = os.path.dirname(os.path.abspath(__file__))
CSRC = os.path.join(HERE, "csrc")
LIB = os.path.join(HERE, "libmcx.so")
SOURCES = ["mcx_pack.cu", "mcx_search.cu", "mcx_records.cu", "mcx_runtime.cu"]
DEPS = SOURCES + ["mcx_common.cuh", "mcx_search.cuh", "mcx_prefilter.cuh", "mcx_records.cuh", "mcx_format.cuh",
                  "mcx_internal.cuh"]

NVCC_FLAGS = [
    "-gencode", "arch=compute_100a,code=sm_100a",
    "-O3", "-lineinfo",
    "--fmad=false",          # never contract the canonical solve into DFMA
    "-std=c++17",
    "-Xcompiler", "-fPIC", "-shared",
    "-cudart", "static",     # loadable without a GPU (CPU tests check the exports)
]


def _stale() -> bool:
    if not os.path.exists(LIB):
        return True
    t = os.path.getmtime(LIB)
    deps = [os.path.join(CSRC, d) for d in DEPS] + [os.path.join(HERE, "..", "include", "mcx.h")]
    return any(os.path.getmtime(d) > t for d in deps if os.path.exists(d))


def build(force: bool = False, verbose: bool = False) -> str:
    if not force and not _stale():
        return LIB
    nvcc = os.environ.get("NVCC", "nvcc")
    cmd = [nvcc, *NVCC_FLAGS, "-o", LIB] + [os.path.join(CSRC, s) for s in SOURCES]
    if verbose:
        cmd.insert(1, "-Xptxas=-v")
    subprocess.run(cmd, check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
