"""Small end-to-end workload for compute-sanitizer (memcheck / racecheck / synccheck /
initcheck): every kernel of libmcx.so on small meshes — pack + levels, the three search
modes (single and batched, sharded), pair_candidates (grids and packed meshes) and
device-side records.  Exits non-zero on any result mismatch."""
import os
import sys

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2109_14814_b200 import _lib, device as D  # noqa: E402
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
print(f"sanitize workload ok: {len(ref.hits)} hits, {len(g1)} quad candidates")
