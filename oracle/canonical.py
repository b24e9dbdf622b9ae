"""O1 — canonical CPU oracle for the triangle-level mesh-intersection search.

TEST INFRASTRUCTURE ONLY.  Nothing in ``paper_2109_14814_b200/`` imports this
module; only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs do, and there only as the checker
or the timed CPU baseline.

What it restates
----------------
The reference ships no implementation of this path: the
``isect`` module is specified in SPEC.md:414-514 and described in PAPER.md
"GPU-Accelerated Manifold Mesh Intersection Search" / "Computational
Implementation" (PAPER.md:173-251 of the original; mesh §Discrete Mesh).  This is
a plain-NumPy restatement of that search at triangle granularity:

* triangle split of quad (i, k):  T¹ = {v00, v10, v01},  T² = {v10, v01, v11},
  θ index wrapping mod N  (PAPER.md T^{u1}/T^{u2} displays)
* bounding-box rejection with strict ``<`` in both directions over x, y, px, py
  (PAPER.md "Bounding Box Test")
* precise test: the 4×4 system of Eq. (26) with acceptance a, b, c, d ≥ 0,
  a+b ≤ 1, c+d ≤ 1 (PAPER.md "Precise Test"); near-singular
  systems are "no intersection" plus a diagnostics counter.

Parity contract
--------------------------------
Accept/reject at exact boundaries (shared vertices/edges) is decided by
rounding, so the CUDA kernel and this oracle run the *identical IEEE-754
operation sequence on identically packed triangles*: FMA-free, fixed
association order, no ``np.sum``/``np.dot``/``einsum``/BLAS (they reorder or
fuse).  Every expression below is a sequence of single rounded ufunc ops.

Pinning
-------
The reference has no golden vectors or fixtures for this path.
This oracle is pinned to (1) the SPEC's known-answer tests (SPEC.md:439-441,
448-450, 466-468, 493), (2) an exact ``fractions.Fraction`` solve (``exact.py``)
on dyadic inputs where the canonical arithmetic is provably exact, and (3) the
SPEC-literal quad pipeline (``serial.py``).  It is NOT pinned against a run of
a reference implementation, because none exists: "parity unpinned" in that
sense, see DESIGN.md §Oracle.
"""
from __future__ import annotations

import numpy as np

SINGULAR_RTOL = 1e-12  # condition-estimate gate ("condition estimate > 1e12")

# bivector index pairs (i, j), i < j, in the canonical order 01, 02, 03, 12, 13, 23
BIV = ((0, 1), (0, 2), (0, 3), (1, 2), (1, 3), (2, 3))


# ---------------------------------------------------------------- packing
def triangle_vertices(coords: np.ndarray):
    """Return (V0, V1, V2), each (n_tri, 4), in canonical triangle order.

    ``coords``: (4, M, N) half-layer grid.  Triangle index ``2·(i + N·k) + τ``
    (column-major quad index of PAPER.md kernel step 3, τ = 0 for T¹, 1 for T²).
    V0 is the packing origin: v00 for T¹, v01 for T².  Edges are V1−V0, V2−V0:
    T¹: (v10−v00, v01−v00);  T²: (v10−v01, v11−v01).
    """
    c = np.asarray(coords, dtype=np.float64)
    _, M, N = c.shape
    W = np.transpose(c, (1, 2, 0))  # (M, N, 4): W[k, i] = W(θ_i, s_k)
    ip = (np.arange(N) + 1) % N
    v00 = W[:-1, :, :]
    v10 = W[:-1, ip, :]
    v01 = W[1:, :, :]
    v11 = W[1:, ip, :]
    nq = N * (M - 1)
    V0 = np.empty((M - 1, N, 2, 4))
    V1 = np.empty_like(V0)
    V2 = np.empty_like(V0)
    V0[:, :, 0], V1[:, :, 0], V2[:, :, 0] = v00, v10, v01
    V0[:, :, 1], V1[:, :, 1], V2[:, :, 1] = v01, v10, v11
    return V0.reshape(2 * nq, 4), V1.reshape(2 * nq, 4), V2.reshape(2 * nq, 4)


def pack(coords: np.ndarray) -> dict:
    """Canonical SoA packing.

    Returns dict with ``lo``, ``hi`` (n,4) exact AABB; ``p``, ``e1``, ``e2`` (n,4);
    ``P`` (n,6) bivector e1∧e2 in BIV order; ``nrm`` (n,) = ‖e1‖·‖e2‖ with
    left-to-right sums of squares.
    """
    V0, V1, V2 = triangle_vertices(coords)
    V0 = V0 + 0.0  # canonicalise -0.0 (x + 0.0 == +0.0 for x = -0.0 under RN)
    V1 = V1 + 0.0
    V2 = V2 + 0.0
    lo = np.minimum(np.minimum(V0, V1), V2)
    hi = np.maximum(np.maximum(V0, V1), V2)
    e1 = V1 - V0
    e2 = V2 - V0
    P = np.empty((V0.shape[0], 6))
    for k, (i, j) in enumerate(BIV):
        P[:, k] = e1[:, i] * e2[:, j] - e1[:, j] * e2[:, i]
    n1 = ((e1[:, 0] * e1[:, 0] + e1[:, 1] * e1[:, 1]) + e1[:, 2] * e1[:, 2]) + e1[:, 3] * e1[:, 3]
    n2 = ((e2[:, 0] * e2[:, 0] + e2[:, 1] * e2[:, 1]) + e2[:, 2] * e2[:, 2]) + e2[:, 3] * e2[:, 3]
    nrm = np.sqrt(n1) * np.sqrt(n2)
    return {"lo": lo, "hi": hi, "p": V0, "e1": e1, "e2": e2, "P": P, "nrm": nrm}


def take(pk: dict, idx) -> dict:
    return {k: v[idx] for k, v in pk.items()}


# ---------------------------------------------------------------- predicate
def aabb_overlap(loA, hiA, loB, hiB):
    """Not rejected iff no coordinate is strictly separated.

    Shapes broadcast; last axis is the coordinate.  Exact, order-free.
    """
    sep = (hiA < loB) | (hiB < loA)
    return ~(sep[..., 0] | sep[..., 1] | sep[..., 2] | sep[..., 3])


def _contract(r, B):
    """g_j = Σ_i r_i K_ij for the antisymmetric K of bivector B.

    K01=+B23, K02=−B13, K03=+B12, K12=+B03, K13=−B02, K23=+B01; each component is
    summed left to right over ascending i ≠ j (negations are exact).
    B columns: 0:01 1:02 2:03 3:12 4:13 5:23.
    """
    r0, r1, r2, r3 = r[..., 0], r[..., 1], r[..., 2], r[..., 3]
    B01, B02, B03, B12, B13, B23 = (B[..., k] for k in range(6))
    c0 = (r2 * B13 - r1 * B23) - r3 * B12
    c1 = (r0 * B23 - r2 * B03) + r3 * B02
    c2 = (r1 * B03 - r0 * B13) - r3 * B01
    c3 = (r0 * B12 - r1 * B02) + r2 * B01
    return c0, c1, c2, c3


def _dot4(c, x):
    return ((c[0] * x[..., 0] + c[1] * x[..., 1]) + c[2] * x[..., 2]) + c[3] * x[..., 3]


def solve_pairs(A: dict, B: dict):
    """Canonical FMA-free bivector-Cramer solve for paired rows of A and B.

    Solves p + s·e1 + t·e2 = q + a·f1 + b·f2 (Eq. 26 with (s,t,a,b) =
    the SPEC's (a,b,c,d)).  Returns (s, t, a, b, singular, hit) arrays.
    """
    P, Q = A["P"], B["P"]
    r = B["p"] - A["p"]
    D = P[:, 0] * Q[:, 5] - P[:, 1] * Q[:, 4]
    D = D + P[:, 2] * Q[:, 3]
    D = D + P[:, 3] * Q[:, 2]
    D = D - P[:, 4] * Q[:, 1]
    D = D + P[:, 5] * Q[:, 0]
    thr = (A["nrm"] * B["nrm"]) * SINGULAR_RTOL
    singular = np.abs(D) <= thr
    g = _contract(r, Q)
    h = _contract(r, P)
    with np.errstate(divide="ignore", invalid="ignore"):
        s = _dot4(g, A["e2"]) / D
        t = -_dot4(g, A["e1"]) / D
        a = -_dot4(h, B["e2"]) / D
        b = _dot4(h, B["e1"]) / D
        hit = (~singular) & (s >= 0) & (t >= 0) & (a >= 0) & (b >= 0) & ((s + t) <= 1) & ((a + b) <= 1)
    return s, t, a, b, singular, hit


def search(coords_a, coords_b, chunk: int = 0, a_range=None, packed=None):
    """All-pairs triangle search, CPU, single process.

    Returns dict: ``ia``, ``ib`` (uint32, sorted by (ia, ib)), ``s``, ``t``, ``a``,
    ``b`` (float64), and counters ``n_pairs``, ``n_aabb_pass``, ``n_singular``.
    ``a_range`` restricts A triangles to [a0, a1) (for timed slices / sharding).
    """
    A = packed[0] if packed else pack(coords_a)
    B = packed[1] if packed else pack(coords_b)
    nA, nB = A["lo"].shape[0], B["lo"].shape[0]
    if chunk <= 0:  # bound the (chunk, nB, 4) temporaries to ~2^22 elements
        chunk = max(1, (1 << 22) // max(1, nB))
    a0, a1 = (0, nA) if a_range is None else a_range
    ia_l, ib_l = [], []
    for c0 in range(a0, a1, chunk):
        c1 = min(c0 + chunk, a1)
        ov = aabb_overlap(A["lo"][c0:c1, None, :], A["hi"][c0:c1, None, :],
                          B["lo"][None, :, :], B["hi"][None, :, :])
        ii, jj = np.nonzero(ov)
        ia_l.append(ii + c0)
        ib_l.append(jj)
    ia = np.concatenate(ia_l) if ia_l else np.zeros(0, np.int64)
    ib = np.concatenate(ib_l) if ib_l else np.zeros(0, np.int64)
    s, t, a, b, sing, hit = solve_pairs(take(A, ia), take(B, ib))
    order = np.lexsort((ib[hit], ia[hit]))
    return {
        "ia": ia[hit][order].astype(np.uint32), "ib": ib[hit][order].astype(np.uint32),
        "s": s[hit][order], "t": t[hit][order], "a": a[hit][order], "b": b[hit][order],
        "n_pairs": (a1 - a0) * nB, "n_aabb_pass": int(ia.size), "n_singular": int(sing.sum()),
    }


def hit_points(coords_a, ia, s, t):
    """Intersection points p + s·e1 + t·e2, FMA-free, fixed order."""
    A = take(pack(coords_a), np.asarray(ia, dtype=np.int64))
    return (A["p"] + s[:, None] * A["e1"]) + t[:, None] * A["e2"]
