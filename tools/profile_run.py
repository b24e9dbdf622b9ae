"""Small driver for ncu: build the named config's meshes on cuda:0 and run the
search `--iters` times (the first call is the warm-up)."""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="C2")
ap.add_argument("--mode", default="brute")
ap.add_argument("--iters", type=int, default=2)
a = ap.parse_args()
A, sa, B, sb = config_pair(a.config)
Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
m = _lib.MODE_NAMES[a.mode]
for _ in range(a.iters):
    r = D.search_device(Am, Bm, mode=m, timing=True)
print(r.stats)
