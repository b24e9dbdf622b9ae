"""Generate the committed golden fixtures under tests/golden/.

Run here (this container has /root/reference; the GPU box does not):
    python tests/golden/make_golden.py

What is pinned, and against what:
  * theta_grid.npz — θ_i from the REFERENCE's own ``maniconn.fourier.grid_points``
    (imported from /root/reference/pkg/src), for N in a few sizes; our mesh
    generator must reproduce them bit-for-bit (fourier.py:23-25).
  * kat_precise.npz — SPEC.md:466-468 known answers, solved exactly with
    ``fractions.Fraction`` (oracle/exact.py) on integer / dyadic inputs:
      shared vertex → (1, 0, 1, 0); parallel translate → singular;
      constructed crossing at (0.1, 0.1, 0.1, 0.1) → interior barycentrics.
  * pair_counts.json — PAPER.md / SPEC.md:493 pair-count arithmetic.
  * c1.npz, c4ii.npz — the meshes (so cross-machine libm differences in the
    generator cannot move the fixture) and the canonical hit lists
    (iA, iB and the IEEE bit patterns of s, t, a, b) from O1.  For the dyadic
    stress mesh C4(ii) every AABB-surviving pair's accept/reject decision is also
    decided EXACTLY by O4 (Fraction) and stored; the canonical arithmetic is
    exact on that lattice, so O1 must agree with the exact decisions pair for
    pair.
"""
from __future__ import annotations

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(os.path.dirname(HERE))
sys.path.insert(0, ROOT)

from oracle import canonical as O  # noqa: E402
from oracle import exact as X  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair  # noqa: E402


def theta_fixture():
    sys.path.insert(0, "/root/reference/pkg/src")
    from maniconn import fourier  # the reference's own implementation

    sizes = [4, 64, 256, 1024, 2048]
    np.savez(os.path.join(HERE, "theta_grid.npz"), **{f"n{n}": fourier.grid_points(n) for n in sizes})


def kat_fixture():
    rng = np.random.default_rng(20260917)
    rows = []  # (p, e1, e2, q, f1, f2) as 24 doubles, expected (s,t,a,b) or NaN, singular flag
    exp = []
    sing = []
    # shared vertex: A = (x2, x1, x3), B = (y2, y1, y3) with x1 == y1 → (a,b,c,d) = (1,0,1,0)
    # In the packed form p = x2, e1 = x1 - x2, e2 = x3 - x2 (SPEC eq. 26) → s=1, t=0, a=1, b=0.
    for _ in range(200):
        x1 = rng.integers(-50, 50, 4).astype(float)
        x2 = rng.integers(-50, 50, 4).astype(float)
        x3 = rng.integers(-50, 50, 4).astype(float)
        y2 = rng.integers(-50, 50, 4).astype(float)
        y3 = rng.integers(-50, 50, 4).astype(float)
        p, e1, e2 = x2, x1 - x2, x3 - x2
        q, f1, f2 = y2, x1 - y2, y3 - y2
        sol = X.solve_exact(p, e1, e2, q, f1, f2)
        if sol is None:
            continue
        rows.append(np.concatenate([p, e1, e2, q, f1, f2]))
        exp.append([float(v) for v in sol])
        sing.append(False)
    # parallel translate: t1 in plane {px = 0, py = 0}, t2 = t1 + (0, 0, 1, 1) → singular, none
    for _ in range(50):
        v = rng.integers(-20, 20, (3, 2)).astype(float)
        t1 = np.concatenate([v, np.zeros((3, 2))], axis=1)
        t2 = t1 + np.array([0.0, 0.0, 1.0, 1.0])
        rows.append(np.concatenate([t1[0], t1[1] - t1[0], t1[2] - t1[0], t2[0], t2[1] - t2[0], t2[2] - t2[0]]))
        exp.append([np.nan] * 4)
        sing.append(True)
    # constructed crossing: T1 spans (ê1, ê2), T2 spans (ê3, ê4), planes meet at (0.1, 0.1, 0.1, 0.1)
    for k in range(50):
        sc = 0.5 + k / 64.0
        c = np.full(4, 0.1)
        p = c - sc * 0.25 * np.array([1.0, 1.0, 0.0, 0.0])
        e1 = np.array([sc, 0.0, 0.0, 0.0])
        e2 = np.array([0.0, sc, 0.0, 0.0])
        q = c - sc * 0.25 * np.array([0.0, 0.0, 1.0, 1.0])
        f1 = np.array([0.0, 0.0, sc, 0.0])
        f2 = np.array([0.0, 0.0, 0.0, sc])
        sol = X.solve_exact(p, e1, e2, q, f1, f2)
        rows.append(np.concatenate([p, e1, e2, q, f1, f2]))
        exp.append([float(v) for v in sol])
        sing.append(False)
    np.savez(os.path.join(HERE, "kat_precise.npz"), rows=np.array(rows), expected=np.array(exp),
             singular=np.array(sing))


def pair_count_fixture():
    out = {"paper": {"N1": 1024, "N2": 2048, "M1": 35, "M2": 35, "quad_pairs": 2424307712,
                     "triangle_pairs": 9697230848}}
    with open(os.path.join(HERE, "pair_counts.json"), "w") as fh:
        json.dump(out, fh, indent=1)


def hits_record(r):
    return dict(ia=r["ia"], ib=r["ib"], s=r["s"].view(np.uint64), t=r["t"].view(np.uint64),
                a=r["a"].view(np.uint64), b=r["b"].view(np.uint64),
                n_aabb_pass=np.array(r["n_aabb_pass"]), n_singular=np.array(r["n_singular"]))


def mesh_fixtures():
    A, sa, B, sb = config_pair("C1")
    r = O.search(A, B)
    np.savez_compressed(os.path.join(HERE, "c1.npz"), A=A, B=B, sa=sa, sb=sb, **hits_record(r))
    A, sa, B, sb = config_pair("C4ii")
    r = O.search(A, B)
    # exact decisions for every AABB-surviving pair
    pA, pB = O.pack(A), O.pack(B)
    ia_l, ib_l = [], []
    for c0 in range(0, pA["lo"].shape[0], 256):
        c1 = min(c0 + 256, pA["lo"].shape[0])
        ov = O.aabb_overlap(pA["lo"][c0:c1, None], pA["hi"][c0:c1, None], pB["lo"][None], pB["hi"][None])
        ii, jj = np.nonzero(ov)
        ia_l.append(ii + c0)
        ib_l.append(jj)
    ia = np.concatenate(ia_l)
    ib = np.concatenate(ib_l)
    acc = np.zeros(ia.size, dtype=bool)
    sing = np.zeros(ia.size, dtype=bool)
    for n in range(ia.size):
        a, b = ia[n], ib[n]
        sol = X.solve_exact(pA["p"][a], pA["e1"][a], pA["e2"][a], pB["p"][b], pB["e1"][b], pB["e2"][b])
        sing[n] = sol is None
        acc[n] = X.accepted(sol)
    np.savez_compressed(os.path.join(HERE, "c4ii.npz"), A=A, B=B, sa=sa, sb=sb, surv_ia=ia.astype(np.uint32),
                        surv_ib=ib.astype(np.uint32), exact_accept=acc, exact_singular=sing, **hits_record(r))


if __name__ == "__main__":
    theta_fixture()
    kat_fixture()
    pair_count_fixture()
    mesh_fixtures()
    print("golden fixtures written to", HERE)
