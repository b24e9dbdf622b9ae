"""Kernel time of MCX_VARIANT settings on one config and mode (env MCX_VARIANT is read per call)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402

cfg, mode = sys.argv[1], sys.argv[2]
variants = sys.argv[3].split(",")
A, _, B, _ = config_pair(cfg)
Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
for v in variants:
    os.environ["MCX_VARIANT"] = v
    D.search_device(Am, Bm, mode=_lib.MODE_NAMES[mode])
    ts = [D.search_device(Am, Bm, mode=_lib.MODE_NAMES[mode], timing=True).stats["kernel_ms"] for _ in range(5)]
    print(cfg, mode, "variant", v, "min %.3f ms  median %.3f ms" % (min(ts), sorted(ts)[2]), flush=True)
