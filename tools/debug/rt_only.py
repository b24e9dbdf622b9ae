"""Runtime-only probe for initcheck bisection: one small find (small path)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
from paper_2109_14814_b200 import _lib, runtime  # noqa: E402
from paper_2109_14814_b200.mesh import manifold_like  # noqa: E402

A, sa = manifold_like(48, 21, 3)
B, sb = manifold_like(40, 19, 3)
B = B + 1e-3
ctx = runtime.context(0)
step = os.environ.get("STEP", "find")
if step in ("ctx",):
    print("ctx ok")
    sys.exit(0)
m = ctx.mesh(A, sa)
print("mesh ok", flush=True)
if step == "mesh":
    sys.exit(0)
recs, text, st = ctx.find(A, sa, B, sb, pipeline=_lib.PIPE_TRIANGLE, text=True)
print("find ok", len(recs), flush=True)
