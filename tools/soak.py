"""Randomised parity soak: many random mesh pairs (shapes, surfaces, affine scalings,
translations, near-coincident and identical copies, dyadic lattices), each searched in
every mode — single call, 3-way cyclic shards, inside a batch, and with the roles
oriented (MCX_ORIENT_LARGER_A) — against the C oracle's exact sweep; the SPEC pipeline
against the C restatement of the serial backend (hits, candidate counts); and the host
runtime's records text (device sort / dedup / %.17g) against the host path built from the
oracle's hits.  Prints one summary line per 50 cases and a final JSON line.
    MCX_PREFILTER_MIN_PAIRS=0 python tools/soak.py [n_cases] [seed]"""
import json
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from oracle import c_oracle as C  # noqa: E402
os.environ.setdefault("MCX_PREFILTER_MIN_PAIRS", "0")  # the quantised kernel at every size
from paper_2109_14814_b200 import _lib, device as D, isect, runtime  # noqa: E402
from paper_2109_14814_b200.mesh import dyadic, manifold_like  # noqa: E402

n_cases = int(sys.argv[1]) if len(sys.argv) > 1 else 200
rng = np.random.default_rng(int(sys.argv[2]) if len(sys.argv) > 2 else 2026)
MODES = [_lib.MODE_BRUTE, _lib.MODE_PREFILTER, _lib.MODE_CULL]
bad, hits_total, pass_total, pairs_total = [], 0, 0, 0
t0 = time.time()


def same(ref, h):
    return (np.array_equal(ref["ia"], h["ia"]) and np.array_equal(ref["ib"], h["ib"]) and
            all(np.array_equal(np.asarray(ref[f]).view(np.uint64), np.asarray(h[f]).view(np.uint64)) for f in "stab"))


for case in range(n_cases):
    na, ma = int(rng.integers(1, 300)), int(rng.integers(2, 120))
    nb, mb = int(rng.integers(1, 300)), int(rng.integers(2, 120))
    kind = case % 5
    A, _ = manifold_like(na, ma, int(rng.integers(0, 1000)))
    if kind == 0:
        B, _ = manifold_like(nb, mb, int(rng.integers(0, 1000)))
    elif kind == 1:
        sd = int(rng.integers(0, 1000))
        A, _ = manifold_like(na, ma, sd)
        B, _ = manifold_like(nb, mb, sd)
        B = B + rng.normal(0, 10 ** rng.uniform(-9, -2), (4, 1, 1))
    elif kind == 2:
        B = A.copy()
    elif kind == 3:
        A = dyadic(A, 8)
        B = A + np.round(rng.normal(0, 4, (4, 1, 1))) / 2 ** 8
    else:
        B = A + rng.normal(0, 1e-2, (4, 1, 1))
    scale = 10.0 ** rng.uniform(-6, 6)
    shift = np.round(rng.normal(0, 10, (4, 1, 1)) * scale) if kind == 3 else rng.normal(0, 10, (4, 1, 1)) * scale
    if kind == 3:
        scale = 2.0 ** int(rng.integers(-10, 10))
    A, B = A * scale + shift + 0.0, B * scale + shift + 0.0
    ref = C.search(A, B, sweep=True, cap=1 << 22)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    ok = True
    for mode in MODES:
        r = D.search_device(Am, Bm, mode=mode)
        ok &= same(ref, r.hits) and r.stats["n_aabb_pass"] == ref["n_aabb_pass"]
        parts = D._merge([D.search_device(Am, Bm, mode=mode, shard=(g, 3)) for g in range(3)])
        ok &= same(ref, parts.hits)
        bt = D.search_batch([(Bm, Am), (Am, Bm)], mode=mode)[1]
        ok &= same(ref, bt.hits)
        for orient in (_lib.ORIENT_AS_GIVEN, _lib.ORIENT_LARGER_A):
            ok &= same(ref, D.search_device(Am, Bm, mode=mode, orient=orient).hits)
    spec = C.spec_search(A, B, cap=1 << 22)
    rs = D.search_device(Am, Bm, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC)
    ok &= same(spec, rs.hits) and rs.stats["n_candidates"] == spec["n_candidates"]
    sa, sb = np.linspace(-1, 1, A.shape[1]), np.linspace(-1, 1, B.shape[1])
    h = np.zeros(len(ref["ia"]), dtype=D.HIT_DTYPE)
    for f in ("ia", "ib", "s", "t", "a", "b"):
        h[f] = ref[f]
    want = "".join(w.to_line() + "\n" for w in isect.hits_to_records(A, sa, B, sb, h, layer=(2, "-", 1, "+")))
    _, text, _ = runtime.context(0).find(A, sa, B, sb, (2, "-", 1, "+"), pipeline=_lib.PIPE_TRIANGLE, text=True)
    ok &= text == want.encode()
    if not ok:
        bad.append(case)
    hits_total += len(ref["ia"])
    pass_total += int(ref["n_aabb_pass"])
    pairs_total += Am.n_tri * Bm.n_tri
    if (case + 1) % 50 == 0:
        print(f"{case + 1} cases, {len(bad)} mismatches, {hits_total} hits, {time.time() - t0:.0f} s", flush=True)
print(json.dumps({"cases": n_cases, "mismatches": bad, "hits": hits_total, "aabb_passes": pass_total,
                  "pairs": pairs_total, "checks_per_case": 5 * len(MODES) + 2, "seconds": round(time.time() - t0, 1)}))
