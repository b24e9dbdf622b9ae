"""Worst-case probe for the exhaustive modes: a mesh searched against itself (every
triangle touches its neighbours) at growing sizes; prints
kernel time per mode and the prefilter's exact-test count."""
import json
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.mesh import manifold_like  # noqa: E402

for N, M in ((128, 129), (256, 257), (512, 257)):
    A, _ = manifold_like(N, M, 3)
    Am = D.DeviceMesh(A, 0)
    row = {"grid": f"{N}x{M}", "tri": Am.n_tri}
    for name in ("brute", "prefilter", "cull"):
        mode = _lib.MODE_NAMES[name]
        D.search_device(Am, Am, mode=mode)
        st = min((D.search_device(Am, Am, mode=mode, timing=True).stats for _ in range(3)), key=lambda s: s["kernel_ms"])
        row[name] = {"ms": round(st["kernel_ms"], 3), "exact_tests": st["n_exact_tests"], "hits": st["n_hits"],
                     "aabb_pass": st["n_aabb_pass"]}
    print(json.dumps(row), flush=True)
