"""Where the time of layers.search_plan on the paper's 108-task plan goes (host profile)."""
import cProfile
import os
import pstats
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2109_14814_b200 import layers  # noqa: E402
from paper_2109_14814_b200.mesh import layered_mesh  # noqa: E402

um = layered_mesh(1024, "unstable", 14, 1.6, 0.1, 1, K=17, per_layer=34)
sm = layered_mesh(2048, "stable", 14, 1 / 1.6, 0.1, 2, K=17, per_layer=34)
plan = layers.enumerate_layer_pairs(um, sm, 14)
layers.search_plan(um, sm, plan, text=True)
t0 = time.perf_counter()
layers.search_plan(um, sm, plan, text=True)
print(f"wall {1e3 * (time.perf_counter() - t0):.2f} ms, U {um.coords.shape}, S {sm.coords.shape}")
pr = cProfile.Profile()
pr.enable()
layers.search_plan(um, sm, plan, text=True)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(18)
