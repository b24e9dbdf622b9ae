"""initcheck bisection: one mesh pack, then one search per mode, progress on stderr."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.mesh import manifold_like  # noqa: E402

A, sa = manifold_like(48, 21, 3)
B, sb = manifold_like(40, 19, 3)
Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B + 1e-3, 0)
print("packed", file=sys.stderr, flush=True)
for name in os.environ.get("MODES", "cull,brute,prefilter").split(","):
    r = D.search_device(Am, Bm, mode=_lib.MODE_NAMES[name])
    print(name, len(r.hits), file=sys.stderr, flush=True)
