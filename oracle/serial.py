"""O3 — SPEC-literal serial backend of the reference's ``isect`` module.

TEST INFRASTRUCTURE ONLY (see oracle/canonical.py header).

Restates the quad-level three-stage pipeline exactly as specified:

* ``gid_to_cartesian`` — PAPER.md kernel step 2 / SPEC.md:433-441:
  i = gid % N1; j = (gid % (N1·N2)) / N1; k1 = (gid % (N1·N2·(M1−1))) / (N1·N2);
  l1 = gid / (N1·N2·(M1−1)).
* ``aabb_reject(qa, qb)`` on quad boxes — SPEC.md:442-450 (strict ``<``).
* ``moller_reject(qa, qb)`` — SPEC.md:451-459, Eqs. (24)-(25): project to
  (x, y, px); reject iff all four qb vertices are strictly on one side of the
  plane of T¹(qa) AND strictly on one side of the plane of T²(qa), or the same
  with roles swapped; a degenerate normal (‖N‖ < 1e-14·‖U‖‖W‖) forces "not
  rejected" for that sub-test.
* ``pair_candidates`` — sorted surviving gids.
* ``find_intersections`` — the 4 triangle-pair precise tests per survivor
  (SPEC.md:478-486), with the canonical solve of O1.

Arithmetic: FMA-free, fixed order (planes: N = U × W componentwise
``N0 = U1·W2 − U2·W1``, ``N1 = U2·W0 − U0·W2``, ``N2 = U0·W1 − U1·W0``; plane
value ``(N0·(X0−O0) + N1·(X1−O1)) + N2·(X2−O2)``), so the GPU quad stage
(csrc/mcx_common.cuh: moller_reject) reproduces the survivor list bit-exactly.
"""
from __future__ import annotations

import numpy as np

from . import canonical

DEGEN_RTOL2 = 1e-28  # (1e-14)^2, compared on squared norms


def gid_to_cartesian(gid, N1, N2, M1):
    gid = np.asarray(gid, dtype=np.uint64)
    N1, N2, M1 = np.uint64(N1), np.uint64(N2), np.uint64(M1)
    i = gid % N1
    j = (gid % (N1 * N2)) // N1
    k1 = (gid % (N1 * N2 * (M1 - np.uint64(1)))) // (N1 * N2)
    l1 = gid // (N1 * N2 * (M1 - np.uint64(1)))
    return i, j, k1, l1


def cartesian_to_gid(i, j, k1, l1, N1, N2, M1):
    u = np.uint64
    n12 = u(N1) * u(N2)
    return (np.asarray(i, u) + u(N1) * np.asarray(j, u) + n12 * np.asarray(k1, u)
            + n12 * (u(M1) - u(1)) * np.asarray(l1, u))


def quad_vertices(coords):
    """(nq, 4 verts, 4 coords) in quad order q = i + N·k1; verts v00, v10, v01, v11."""
    c = np.asarray(coords, dtype=np.float64)
    _, M, N = c.shape
    W = np.transpose(c, (1, 2, 0))
    ip = (np.arange(N) + 1) % N
    V = np.stack([W[:-1, :, :], W[:-1, ip, :], W[1:, :, :], W[1:, ip, :]], axis=2)  # (M-1, N, 4, 4)
    return V.reshape(N * (M - 1), 4, 4)


def quad_boxes(V):
    lo = np.minimum(np.minimum(np.minimum(V[:, 0], V[:, 1]), V[:, 2]), V[:, 3])
    hi = np.maximum(np.maximum(np.maximum(V[:, 0], V[:, 1]), V[:, 2]), V[:, 3])
    return lo, hi


def _plane(O, U, W):
    N0 = U[..., 1] * W[..., 2] - U[..., 2] * W[..., 1]
    N1 = U[..., 2] * W[..., 0] - U[..., 0] * W[..., 2]
    N2 = U[..., 0] * W[..., 1] - U[..., 1] * W[..., 0]
    nn = (N0 * N0 + N1 * N1) + N2 * N2
    uu = (U[..., 0] * U[..., 0] + U[..., 1] * U[..., 1]) + U[..., 2] * U[..., 2]
    ww = (W[..., 0] * W[..., 0] + W[..., 1] * W[..., 1]) + W[..., 2] * W[..., 2]
    degen = nn < (uu * ww) * DEGEN_RTOL2
    return (N0, N1, N2), degen


def _side_reject(Vq, Vo):
    """For quads Vq (n,4,4) and other quads Vo (n,4,4): all Vo verts strictly on one side of
    T¹(Vq)'s plane AND of T²(Vq)'s plane (in x, y, px)."""
    out = np.ones(Vq.shape[0], dtype=bool)
    for (o, u, w) in ((0, 1, 2), (2, 1, 3)):  # T¹: O=v00 U=v10-v00 W=v01-v00; T²: O=v01 U=v10-v01 W=v11-v01
        O = Vq[:, o, :3]
        U = Vq[:, u, :3] - O
        W = Vq[:, w, :3] - O
        (N0, N1, N2), degen = _plane(O, U, W)
        f = [(N0 * (Vo[:, m, 0] - O[:, 0]) + N1 * (Vo[:, m, 1] - O[:, 1])) + N2 * (Vo[:, m, 2] - O[:, 2])
             for m in range(4)]
        pos = (f[0] > 0) & (f[1] > 0) & (f[2] > 0) & (f[3] > 0)
        neg = (f[0] < 0) & (f[1] < 0) & (f[2] < 0) & (f[3] < 0)
        out &= (~degen) & (pos | neg)
    return out


def moller_reject_quads(VA, VB):
    return _side_reject(VA, VB) | _side_reject(VB, VA)


def pair_candidates(coords_a, coords_b, chunk: int = 0):
    """Sorted u64 gids with ¬aabb_reject ∧ ¬moller_reject, plus the AABB-pass count."""
    ca, cb = np.asarray(coords_a), np.asarray(coords_b)
    if chunk <= 0:  # bound the (chunk, nB, 4) temporaries to ~2^24 elements
        chunk = max(1, (1 << 22) // max(1, cb.shape[2] * (cb.shape[1] - 1)))
    _, MA, NA = ca.shape
    _, MB, NB = cb.shape
    VA, VB = quad_vertices(ca), quad_vertices(cb)
    loA, hiA = quad_boxes(VA)
    loB, hiB = quad_boxes(VB)
    qa_l, qb_l = [], []
    n_pass = 0
    for c0 in range(0, VA.shape[0], chunk):
        c1 = min(c0 + chunk, VA.shape[0])
        ov = canonical.aabb_overlap(loA[c0:c1, None], hiA[c0:c1, None], loB[None], hiB[None])
        ii, jj = np.nonzero(ov)
        n_pass += ii.size
        ii = ii + c0
        keep = ~moller_reject_quads(VA[ii], VB[jj])
        qa_l.append(ii[keep])
        qb_l.append(jj[keep])
    qa = np.concatenate(qa_l) if qa_l else np.zeros(0, np.int64)
    qb = np.concatenate(qb_l) if qb_l else np.zeros(0, np.int64)
    gid = cartesian_to_gid(qa % NA, qb % NB, qa // NA, qb // NB, NA, NB, MA)
    return np.sort(gid), n_pass


def find_intersections(coords_a, coords_b):
    """SPEC-literal pipeline: quad survivors → 4 canonical precise tests each.

    Returns the same hit dict layout as canonical.search (triangle indices).
    """
    ca, cb = np.asarray(coords_a), np.asarray(coords_b)
    _, MA, NA = ca.shape
    _, MB, NB = cb.shape
    gids, _ = pair_candidates(ca, cb)
    i, j, k1, l1 = (x.astype(np.int64) for x in gid_to_cartesian(gids, NA, NB, MA))
    qa = i + NA * k1
    qb = j + NB * l1
    ia = np.concatenate([2 * qa + ta for ta in (0, 1) for tb in (0, 1)])
    ib = np.concatenate([2 * qb + tb for ta in (0, 1) for tb in (0, 1)])
    A, B = canonical.pack(ca), canonical.pack(cb)
    s, t, a, b, sing, hit = canonical.solve_pairs(canonical.take(A, ia), canonical.take(B, ib))
    order = np.lexsort((ib[hit], ia[hit]))
    return {"ia": ia[hit][order].astype(np.uint32), "ib": ib[hit][order].astype(np.uint32),
            "s": s[hit][order], "t": t[hit][order], "a": a[hit][order], "b": b[hit][order]}
