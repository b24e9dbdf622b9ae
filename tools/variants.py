"""Time kernel variants (MCX_VARIANT) on a config, with a parity check on C4i."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
from paper_2109_14814_b200 import device as D, _lib
from paper_2109_14814_b200.mesh import config_pair
from oracle import c_oracle as C

cfgs = sys.argv[1].split(",") if len(sys.argv) > 1 else ["C3"]
variants = sys.argv[2].split(",") if len(sys.argv) > 2 else ["0", "1", "2", "3"]
mode = _lib.MODE_NAMES[sys.argv[3] if len(sys.argv) > 3 else "brute"]
A, _, B, _ = config_pair("C4i")
ref = C.search(A, B, sweep=True)
Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
for v in variants:
    os.environ["MCX_VARIANT"] = v
    r = D.search_device(Am, Bm, mode=mode)
    ok = np.array_equal(r.hits["ia"], ref["ia"]) and np.array_equal(r.hits["ib"], ref["ib"]) and \
        np.array_equal(r.hits["s"].view(np.uint64), ref["s"].view(np.uint64)) and r.stats["n_aabb_pass"] == ref["n_aabb_pass"]
    print("parity C4i variant", v, ok, flush=True)
for name in cfgs:
    A, _, B, _ = config_pair(name)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    for v in variants:
        os.environ["MCX_VARIANT"] = v
        D.search_device(Am, Bm, mode=mode)
        ts = [D.search_device(Am, Bm, mode=mode, timing=True).stats for _ in range(3)]
        st = min(ts, key=lambda s: s["kernel_ms"])
        ms = st["kernel_ms"]
        print(json.dumps({"cfg": name, "variant": v, "mode": sys.argv[3] if len(sys.argv) > 3 else "brute", "exact_tests": st["n_exact_tests"], "ms": ms,
                          "pairs_per_s": st["n_pairs"] / ms * 1e3, "tested": st["n_tested"],
                          # FP64-pipe lane-ops and fraction of the 18.6 T lane-op/s peak: meaningful for
                          # the FP64 kernels (brute, cull) only
                          "fp64_lane_ops_T": (8 * st["n_exact_tests"] + 100 * st["n_aabb_pass"]) / ms / 1e9,
                          "fp64_frac": (8 * st["n_exact_tests"] + 100 * st["n_aabb_pass"]) / ms / 1e9 / 18.61248,
                          "hits": int(st["n_hits"]), "pass": int(st["n_aabb_pass"])}), flush=True)
