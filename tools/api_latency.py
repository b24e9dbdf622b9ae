"""Host-to-host latency of the user-facing calls on one config (default C3): numpy grids
in, results out, wall clock (median of 7 after 2 warm-ups).
    python tools/api_latency.py [config]"""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_14814_b200 import isect  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C3"
A, sA, B, sB = config_pair(name)


def wall(fn):
    for _ in range(2):
        fn()
    ts = []
    for _ in range(7):
        t0 = time.perf_counter()
        fn()
        ts.append(time.perf_counter() - t0)
    return statistics.median(ts) * 1e3


out = {"config": name}
for mode in ("cull", "prefilter"):
    out[f"search_hits[{mode}]_ms"] = wall(lambda: isect.search_hits(A, B, mode=mode))
out["find_intersections[cull]_ms"] = wall(lambda: isect.find_intersections(A, B))
out["pair_candidates[cull]_ms"] = wall(lambda: isect.pair_candidates(A, B))
print(json.dumps({k: (round(v, 3) if isinstance(v, float) else v) for k, v in out.items()}))
