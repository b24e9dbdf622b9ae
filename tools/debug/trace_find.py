"""MCX_TRACE=1 latency breakdown of one runtime find_intersections call (pinned host grids)."""
import os
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_14814_b200 import _lib, runtime  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C2"
A, sa, B, sb = config_pair(name)
pa = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
pb = torch.from_numpy(np.ascontiguousarray(B)).pin_memory()
ctx = runtime.context(0)
for k in range(4):
    t0 = time.perf_counter()
    ctx.find(pa, sa, pb, sb, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC, text=True)
    print(f"python wall {1e3 * (time.perf_counter() - t0):.3f} ms", file=sys.stderr, flush=True)
