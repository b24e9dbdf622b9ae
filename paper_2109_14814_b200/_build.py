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
    """Compile the translation units in parallel (one nvcc each), then link libmcx.so."""
    if not force and not _stale():
        return LIB
    import tempfile
    from concurrent.futures import ThreadPoolExecutor
    nvcc = os.environ.get("NVCC", "nvcc")
    compile_flags = [f for f in NVCC_FLAGS if f != "-shared"]
    with tempfile.TemporaryDirectory() as tmp:
        objs = [os.path.join(tmp, os.path.splitext(src)[0] + ".o") for src in SOURCES]

        def cc(k):
            cmd = [nvcc, *compile_flags, "-c", os.path.join(CSRC, SOURCES[k]), "-o", objs[k]]
            if verbose:
                cmd.insert(1, "-Xptxas=-v")
            subprocess.run(cmd, check=True)

        with ThreadPoolExecutor(len(SOURCES)) as pool:
            list(pool.map(cc, range(len(SOURCES))))
        subprocess.run([nvcc, "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-cudart", "static",
                        "-o", LIB, *objs], check=True)
    return LIB


if __name__ == "__main__":
    print(build(force=True, verbose=True))
