"""Debug probe: device records text vs host formatting on small cases."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))))
import numpy as np  # noqa: E402

from paper_2109_14814_b200 import _lib, device as D, isect, runtime  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402

ctx = runtime.context(0)
for name in ("C1", "C4ii"):
    A, sa, B, sb = config_pair(name)
    for dedup in (False, True):
        recs, text, st = ctx.find(A, sa, B, sb, (2, "+", 2, "-"), pipeline=_lib.PIPE_TRIANGLE, dedup=dedup, text=True)
        hits = D.search(A, B, mode=_lib.MODE_CULL).hits
        want = isect.hits_to_records(A, sa, B, sb, hits, layer=(2, "+", 2, "-"), dedup=dedup)
        wt = "".join(w.to_line() + "\n" for w in want).encode()
        print(name, dedup, len(recs), len(want), len(text), len(wt), text == wt)
        if text != wt:
            print("GOT ", text[:200])
            print("WANT", wt[:200])
