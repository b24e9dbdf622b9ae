"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of libmcx.so on small meshes — the fused pack, the three search
modes and the solve stage (single and batched, sharded, both orientations, the SPEC
pipeline), pair_candidates (grids and packed meshes), device-side records, and the host
runtime (mcx_find_intersections / mcx_intersect / mcx_finish_hits: the single-kernel and
the general records paths, dedup, text).  Exits non-zero on any result mismatch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_14814_b200 import _lib, device as D, isect, runtime  # noqa: E402
from paper_2109_14814_b200.mesh import manifold_like  # noqa: E402

A, sa = manifold_like(48, 21, 3)
B, sb = manifold_like(40, 19, 3)
B = B + 1e-3
Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
ref = D.search_device(Am, Bm, mode=_lib.MODE_BRUTE)
assert len(ref.hits) > 0
for mode in (_lib.MODE_PREFILTER, _lib.MODE_CULL):
    r = D.search_device(Am, Bm, mode=mode)
    assert np.array_equal(r.hits, ref.hits), mode
    parts = [D.search_device(Am, Bm, mode=mode, shard=(g, 3)) for g in range(3)]
    assert np.array_equal(D._merge(parts).hits, ref.hits), mode
    batch = D.search_batch([(Am, Bm), (Bm, Am), (Am, Am)], mode=mode)
    assert np.array_equal(batch[0].hits, ref.hits), mode
# small hit capacity: the grow-and-rerun path
r = D.search_device(Am, Bm, mode=_lib.MODE_PREFILTER, cap=1)
assert np.array_equal(r.hits, ref.hits)
g1 = D.pair_candidates_device(A, B, device=0)
g2, _ = D.pair_candidates_mesh(Am, Bm)
assert np.array_equal(g1, g2)
D.record_fields_device(A, sa, B, sb, ref.hits, device=0)
# orientation: B larger than A, sweep with exchanged roles
small, _ = manifold_like(16, 9, 3)
Sm = D.DeviceMesh(small + 1e-3, 0)
for mode in (_lib.MODE_BRUTE, _lib.MODE_PREFILTER, _lib.MODE_CULL):
    r0 = D.search_device(Sm, Am, mode=mode, orient=_lib.ORIENT_AS_GIVEN)
    r1 = D.search_device(Sm, Am, mode=mode, orient=_lib.ORIENT_LARGER_A)
    assert np.array_equal(r0.hits, r1.hits), mode
spec = D.search_device(Am, Bm, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC)
if os.environ.get("SANITIZE_PART") == "core":
    print(f"sanitize workload ok: {len(ref.hits)} hits (core part only)")
    sys.exit(0)
# host runtime: small path, general path (dedup on a mesh against itself), batch, finish
ctx = runtime.context(0)
recs, text, st = ctx.find(A, sa, B, sb, (1, "+", 2, "-"), pipeline=_lib.PIPE_TRIANGLE, text=True)
want = isect.hits_to_records(A, sa, B, sb, ref.hits, layer=(1, "+", 2, "-"))
assert text == "".join(w.to_line() + "\n" for w in want).encode()
C, sc = manifold_like(80, 30, 3)
hc = D.search(C, C, mode=_lib.MODE_CULL).hits
assert len(hc) > 1024  # the general (multi-kernel) records path
r2, t2, _ = ctx.find(C, sc, C, sc, pipeline=_lib.PIPE_TRIANGLE, text=True)
assert t2 == "".join(w.to_line() + "\n" for w in isect.hits_to_records(C, sc, C, sc, hc)).encode()
ma, mb = ctx.mesh(A, sa), ctx.mesh(B, sb)
r3, t3, _ = ctx.intersect([(ma, mb, (1, "+", 1, "+")), (mb, ma, (1, "-", 1, "-"))], text=True)
r4, t4 = ctx.finish_hits(ref.hits, ma, mb, text=True)
ma.free()
mb.free()
print(f"sanitize workload ok: {len(ref.hits)} hits, {len(g1)} quad candidates, {len(spec.hits)} spec hits, "
      f"{len(recs)} + {len(r2)} runtime records")
