"""End-to-end latency of the reference-facing calls on one GPU (host grids in, records out):

* H2D floor: the same bytes copied host→device alone (pinned, CUDA events), i.e. the
  PCIe time no implementation can avoid;
* find_intersections through the C-ABI runtime (mcx_find_intersections) from pinned and
  from pageable host grids, per mode / pipeline, wall clock around the call;
* the paper's 14-layer plan through layers.search_plan (records + text on the device).
Prints one JSON object per line."""
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2109_14814_b200 import _lib, layers, runtime  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair, layered_mesh  # noqa: E402


def h2d_floor(*arrays, reps=10):
    pins = [torch.from_numpy(np.ascontiguousarray(a)).pin_memory() for a in arrays]
    devs = [torch.empty_like(p, device="cuda") for p in pins]
    s = torch.cuda.current_stream()
    ts = []
    for _ in range(reps + 2):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        for p, d in zip(pins, devs):
            d.copy_(p, non_blocking=True)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    return min(ts[2:]), sum(p.numel() * 8 for p in pins)


def wall(fn, reps=10):
    fn()
    ts = []
    for _ in range(reps):
        t0 = time.perf_counter()
        fn()
        ts.append((time.perf_counter() - t0) * 1e3)
    return min(ts), statistics.median(ts)


def main(configs=("C3", "C2", "C5hd")):
    ctx = runtime.context(0)
    for name in configs:
        A, sa, B, sb = config_pair(name)
        floor_ms, nbytes = h2d_floor(A, B)
        pa = torch.from_numpy(np.ascontiguousarray(A)).pin_memory()
        pb = torch.from_numpy(np.ascontiguousarray(B)).pin_memory()
        row = {"config": name, "h2d_bytes": nbytes, "h2d_floor_ms": floor_ms}
        for label, mode, pipe in (("cull_spec", _lib.MODE_CULL, _lib.PIPE_SPEC),
                                  ("cull_triangle", _lib.MODE_CULL, _lib.PIPE_TRIANGLE),
                                  ("prefilter", _lib.MODE_PREFILTER, _lib.PIPE_TRIANGLE)):
            if name == "C5hd" and label == "prefilter":
                continue
            best, med = wall(lambda: ctx.find(pa, sa, pb, sb, mode=mode, pipeline=pipe, text=True),
                             reps=5 if label == "prefilter" else 10)
            recs, text, st = ctx.find(pa, sa, pb, sb, mode=mode, pipeline=pipe, text=True)
            row[label] = {"pinned_ms_min": best, "pinned_ms_median": med, "records": len(recs),
                          "text_bytes": len(text), "hits": st["n_hits"], "over_floor_ms": best - floor_ms}
            if label == "cull_spec":
                b2, m2 = wall(lambda: ctx.find(A, sa, B, sb, mode=mode, pipeline=pipe, text=True))
                row[label]["pageable_ms_min"] = b2
        print(json.dumps(row), flush=True)
    um = layered_mesh(1024, "unstable", 14, 1.6, 0.1, 1, K=17, per_layer=34)
    sm = layered_mesh(2048, "stable", 14, 1 / 1.6, 0.1, 2, K=17, per_layer=34)
    plan = layers.enumerate_layer_pairs(um, sm, 14)
    # the plugin call on HalfLayer views of the paper meshes (the plan's busiest task, U13+ x S13+):
    # read in place with the mesh's plane stride vs a contiguous host copy first
    from paper_2109_14814_b200 import isect
    from paper_2109_14814_b200.mesh import half_layer
    hu, hs = half_layer(um, 13, 1), half_layer(sm, 13, 1)
    t_view, _ = wall(lambda: isect.find_intersections(hu, hs), reps=10)
    t_copy, _ = wall(lambda: ctx.find(np.ascontiguousarray(hu.coords), hu.s_values, np.ascontiguousarray(hs.coords),
                                      hs.s_values, (13, "+", 13, "+")), reps=10)
    print(json.dumps({"plugin_halflayer": "isect.find_intersections(U13+, S13+) on HalfLayer views of the paper "
                      "meshes (pageable, read in place)", "grid_bytes": hu.coords.nbytes + hs.coords.nbytes,
                      "view_ms_min": t_view, "copy_then_find_ms_min": t_copy,
                      "records": len(isect.find_intersections(hu, hs))}), flush=True)
    for pipe in ("spec", "triangle"):
        best, med = wall(lambda: layers.search_plan(um, sm, plan, pipeline=pipe, text=True), reps=5)
        res = layers.search_plan(um, sm, plan, pipeline=pipe, text=True)
        print(json.dumps({"paper_plan": f"108 tasks, U 1024 x S 2048, pipeline {pipe}", "wall_ms_min": best,
                          "wall_ms_median": med, "records": len(res.records), "text_bytes": len(res.text)}),
              flush=True)


if __name__ == "__main__":
    main(tuple(sys.argv[1:]) or ("C3", "C2", "C5hd"))
