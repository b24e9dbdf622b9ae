import os, sys, time, json
sys.path.insert(0, '/root/repo')
import numpy as np, torch
from paper_2109_14814_b200 import layers
from paper_2109_14814_b200.mesh import layered_mesh
um = layered_mesh(1024, "unstable", 14, 1.6, 0.1, 1, K=17, per_layer=34)
sm = layered_mesh(2048, "stable", 14, 1 / 1.6, 0.1, 2, K=17, per_layer=34)
plan = layers.enumerate_layer_pairs(um, sm, 14)
print("shapes", um.coords.shape, sm.coords.shape, um.coords.nbytes + sm.coords.nbytes)
for _ in range(3): layers.search_plan(um, sm, plan, pipeline="spec", text=True)
ts = []
for _ in range(5):
    t = time.perf_counter(); layers.search_plan(um, sm, plan, pipeline="spec", text=True); ts.append(time.perf_counter() - t)
print("plan wall ms", sorted(ts))
# H2D floors
for pin in (False, True):
    a = torch.from_numpy(np.ascontiguousarray(um.coords)); b = torch.from_numpy(np.ascontiguousarray(sm.coords))
    if pin: a, b = a.pin_memory(), b.pin_memory()
    da = torch.empty_like(a, device="cuda"); db = torch.empty_like(b, device="cuda")
    for _ in range(3): da.copy_(a); db.copy_(b); torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(5): da.copy_(a); db.copy_(b); torch.cuda.synchronize()
    print("h2d pinned" if pin else "h2d pageable", (time.perf_counter() - t) / 5 * 1e3, "ms")
os.environ["MCX_TRACE"] = "1"
layers.search_plan(um, sm, plan, pipeline="spec", text=True)
