"""O5 — the canonical precise test vs a SPEC-shaped LAPACK restatement.  TEST
INFRASTRUCTURE ONLY (see oracle/canonical.py header).

The reference's own code solves its linear systems with ``np.linalg.solve``
(maniconn/torus.py:236, 256); a restatement of SPEC.md:460-468 in that style solves
Eq. (26) as M·(s, t, a, b) = q − p with M = [e1, e2, −f1, −f2] and gates "condition
estimate > 1e12" with ``np.linalg.cond``.  That is numpy's bundled OpenBLAS
— the third-party arithmetic SURVEY.md §8(c) names.  ``compare`` runs both over EVERY
triangle-AABB survivor of a config (the C oracle's exact sweep): the hit-set difference,
each differing pair classified as boundary-gated (either solver puts s, t, a, b, s+t or
a+b within 1e-9 + 1e-14/hadamard of an acceptance boundary) or Hadamard-gated (the
canonical singular gate or cond > 1e12 fired), and the point agreement on the common hits
bucketed by the Hadamard ratio |D|/(‖e1‖‖e2‖‖f1‖‖f2‖).
"""
import numpy as np

from . import c_oracle, canonical as O


def compare(name):
    from paper_2109_14814_b200.mesh import config_pair
    A, _, B, _ = config_pair(name)
    ia, ib = c_oracle.survivors(A, B)
    pA, pB = O.take(O.pack(A), ia), O.take(O.pack(B), ib)
    s, t, a, b, sing, hit = O.solve_pairs(pA, pB)
    can = np.stack([s, t, a, b], 1)
    M = np.stack([pA["e1"], pA["e2"], -pB["e1"], -pB["e2"]], axis=2)  # columns: M @ (s,t,a,b) = q - p
    rhs = pB["p"] - pA["p"]
    with np.errstate(all="ignore"):
        cond = np.linalg.cond(M)
    lap = np.full((len(ia), 4), np.nan)
    ok = np.isfinite(cond) & (cond < 1e15)
    if ok.any():
        lap[ok] = np.linalg.solve(M[ok], rhs[ok][..., None])[..., 0]
    lap_sing = ~(cond <= 1e12)
    with np.errstate(invalid="ignore"):
        lap_hit = ~lap_sing & (lap >= 0).all(1) & (lap[:, 0] + lap[:, 1] <= 1) & (lap[:, 2] + lap[:, 3] <= 1)
    P, Q = pA["P"], pB["P"]
    D = P[:, 0] * Q[:, 5] - P[:, 1] * Q[:, 4] + P[:, 2] * Q[:, 3] + P[:, 3] * Q[:, 2] - P[:, 4] * Q[:, 1] + P[:, 5] * Q[:, 0]
    had = np.abs(D) / (pA["nrm"] * pB["nrm"])

    def margin(x):
        with np.errstate(invalid="ignore"):
            m = np.stack([x[:, 0], x[:, 1], x[:, 2], x[:, 3], 1 - x[:, 0] - x[:, 1], 1 - x[:, 2] - x[:, 3]], 1)
            return np.min(np.where(np.isnan(m), np.inf, np.abs(m)), axis=1)

    tol = 1e-9 + 1e-14 / np.maximum(had, 1e-300)
    boundary = (margin(can) <= tol) | (margin(lap) <= tol)
    hgate = sing | lap_sing
    differ = hit != lap_hit
    unexplained = differ & ~boundary & ~hgate
    both = hit & lap_hit
    pc = O.hit_points(A, ia[both], s[both], t[both])
    pl = (pA["p"][both] + lap[both, 0:1] * pA["e1"][both]) + lap[both, 1:2] * pA["e2"][both]
    rel = np.max(np.abs(pc - pl), axis=1) / np.maximum(np.max(np.abs(pc), axis=1), 1e-300)
    buckets = []
    hb = had[both]
    for lo in (1e-1, 1e-2, 1e-3, 1e-4, 1e-6, 1e-8, 1e-10, 1e-12, 0.0):
        hi = 10.0 if not buckets else buckets[-1]["hadamard_lo"]
        m = (hb >= lo) & (hb < hi)
        if m.any():
            buckets.append({"hadamard_lo": lo, "hadamard_hi": hi, "hits": int(m.sum()),
                            "median_rel_point_diff": float(np.median(rel[m])), "max_rel_point_diff": float(rel[m].max()),
                            "frac_above_1e-12": float(np.mean(rel[m] > 1e-12))})
        else:
            buckets.append({"hadamard_lo": lo, "hadamard_hi": hi, "hits": 0})
    return {"config": name, "aabb_survivors": int(len(ia)), "canonical_hits": int(hit.sum()),
            "lapack_hits": int(lap_hit.sum()), "common_hits": int(both.sum()),
            "canonical_only": int((hit & ~lap_hit).sum()), "lapack_only": int((lap_hit & ~hit).sum()),
            "differ_boundary_gated": int((differ & boundary).sum()),
            "differ_hadamard_gated": int((differ & hgate & ~boundary).sum()), "differ_unexplained": int(unexplained.sum()),
            "canonical_singular": int(sing.sum()), "lapack_cond_gt_1e12": int(lap_sing.sum()),
            "point_agreement_by_hadamard": [b for b in buckets if b["hits"]],
            "lapack": "numpy %s bundled OpenBLAS (np.linalg.solve / np.linalg.cond)" % np.__version__}


