"""Kernel time of every search mode on every BASELINE config (+ the C5hd and dense
self-search stress shapes): one JSON line per (config, mode), median of 5 timed calls
with inputs resident.  "prefilter" forces the quantised kernel at every size (kernel
comparison); "prefilter_default" is what MCX_MODE_PREFILTER does for a user (calls under
2^28 pairs run the FP64 sweep, same results).
`python tools/mode_table.py > profiles/r02_modes.jsonl`"""
import json
import os

os.environ.setdefault("MCX_PREFILTER_MIN_PAIRS", "0")
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair, manifold_like  # noqa: E402


def shapes():
    for name in ("C1", "C2", "C3", "C4i", "C4ii", "C4iii", "C5", "C5hd"):
        A, _, B, _ = config_pair(name)
        yield name, A, B
    A, _ = manifold_like(512, 257, 3)
    yield "dense-self-512x257", A, A
    A, _ = manifold_like(2048, 1025, 1)  # 4.2M x 4.2M triangles, 1.76e13 pairs (beyond configs)
    B, _ = manifold_like(2048, 1025, 2)
    yield "4Mx4M", A, B


for name, A, B in shapes():
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    hits = None
    for mode in (("prefilter", "cull") if name == "4Mx4M" else ("brute", "prefilter", "prefilter_default", "cull")):
        # prefilter: the quantised kernel forced at every size; prefilter_default: the
        # product rule (calls under 2^28 pairs run the FP64 sweep — identical results)
        os.environ["MCX_PREFILTER_MIN_PAIRS"] = "0" if mode == "prefilter" else str(1 << 28)
        m = _lib.MODE_NAMES["prefilter" if mode == "prefilter_default" else mode]
        D.search_device(Am, Bm, mode=m)
        runs = [D.search_device(Am, Bm, mode=m, timing=True) for _ in range(5)]
        st = runs[0].stats
        ms = statistics.median(r.stats["kernel_ms"] for r in runs)
        if hits is None:
            hits = st["n_hits"]
        assert st["n_hits"] == hits, (name, mode)
        print(json.dumps({"config": name, "mode": mode, "tri_a": Am.n_tri, "tri_b": Bm.n_tri, "pairs": st["n_pairs"],
                          "kernel_ms": round(ms, 4), "pair_tests_per_s": st["n_pairs"] / (ms * 1e-3),
                          "executed_box_tests": st["n_tested"], "exact_fp64_box_tests": st["n_exact_tests"],
                          "aabb_pass": st["n_aabb_pass"], "hits": st["n_hits"]}), flush=True)
