"""Build libmcx.so with extra nvcc flags into another path, for A/B timing of a kernel
variant (loaded with MCX_LIB=<path>):
    python tools/microbench/build_variant.py OUT.so -DPACK_MIN_BLOCKS=2 ..."""
import os
import sys

sys.path.insert(0, os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", ".."))
from paper_2109_14814_b200 import _build  # noqa: E402

_build.LIB = os.path.abspath(sys.argv[1])
_build.NVCC_FLAGS = _build.NVCC_FLAGS + sys.argv[2:]
print(_build.build(force=True))
