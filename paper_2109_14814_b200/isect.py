"""Mesh-intersection search — the reference ``isect`` API with ``backend="cuda"``.

Mirrors the operations of the reference's ``isect`` module:
``QuadIndex``, ``IntersectionRecord``, ``gid_to_cartesian``, ``pair_candidates``,
``find_intersections`` and the records text format, with the same
names, argument meanings and error behaviour, so a caller switches by passing
``backend="cuda"``.  The reference's own CPU backends (``"serial"``,
``"parallel"``) are not part of this package: passing them raises
``ConfigError`` (their restatement lives in ``oracle/`` and is test-only).

Semantics:

* ``find_intersections`` — every pair (T_A, T_B) of triangles of the two
  half-layers whose bounding boxes overlap (strict-separation rejection,
  SPEC.md:442-450) gets the precise test of SPEC.md:460-468, evaluated with the
  canonical FMA-free FP64 sequence of SURVEY.md §7.3; accepted pairs become
  records with Eq. (28)-(29) parameter estimates, sorted by (gid, τ_A, τ_B) and
  deduplicated within 1e-9.  The Möller quick test is a pure
  filter in exact arithmetic; it is not applied here because its floating-point
  form can drop touching hits — ``pair_candidates`` exposes it.
* ``pair_candidates`` — the SPEC-literal quad-level survivor list:
  ¬aabb_reject ∧ ¬moller_reject over all N1·N2·(M1−1)·(M2−1) gids, sorted.

Everything heavy runs on the GPU through the C ABI (include/mcx.h); the host
only slices grids, sorts the small hit list and formats records.
"""
from __future__ import annotations

from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as _device
from .errors import ConfigError, FileFormatError
from .mesh import HalfLayer, grid_points

BACKENDS = ("cuda",)
DEDUP_TOL = 1e-9


# ---------------------------------------------------------------- types
@dataclass(frozen=True)
class QuadIndex:
    """gid ↔ (i, j, k, l) with the paper's k = k1 + 1 convention."""

    gid: int
    i: int
    j: int
    k: int
    l: int


@dataclass
class IntersectionRecord:
    """One mesh intersection.

    ``bary`` = (a, b, c, d) of Eq. (26) for the intersecting triangle pair,
    ``params`` = (θ_u, s_u, θ_s, s_s) estimates (Eqs. 28-29), ``tri`` = (τ_A, τ_B)
    (0 = T¹, 1 = T²), ``pair`` = the QuadIndex, ``layer`` = (n1, sign1, n2, sign2).
    """

    point: np.ndarray
    bary: tuple
    params: tuple
    pair: QuadIndex
    tri: tuple = (0, 0)
    layer: tuple = (0, "+", 0, "+")
    tof: float = float("nan")
    tri_index: tuple = field(default=(0, 0), repr=False)

    def to_line(self) -> str:
        n1, s1, n2, s2 = self.layer
        vals = [*self.point, *self.bary, *self.params]
        return f"{n1} {s1} {n2} {s2} {self.pair.gid} " + " ".join(f"{v:.17g}" for v in vals)


# ---------------------------------------------------------------- gid arithmetic
def gid_to_cartesian(gid, N1: int, N2: int, M1: int):
    """PAPER.md kernel step 2; returns (i, j, k1, l1). u64-safe."""
    if np.isscalar(gid):
        g = int(gid)
        if g < 0:
            raise ConfigError(f"gid {g} out of range")
        n12 = N1 * N2
        return g % N1, (g % n12) // N1, (g % (n12 * (M1 - 1))) // n12, g // (n12 * (M1 - 1))
    g = np.asarray(gid, dtype=np.uint64)
    u = np.uint64
    n12 = u(N1) * u(N2)
    return g % u(N1), (g % n12) // u(N1), (g % (n12 * u(M1 - 1))) // n12, g // (n12 * u(M1 - 1))


def cartesian_to_gid(i, j, k1, l1, N1: int, N2: int, M1: int):
    if np.isscalar(i):
        return int(i) + N1 * int(j) + N1 * N2 * int(k1) + N1 * N2 * (M1 - 1) * int(l1)
    u = np.uint64
    n12 = u(N1) * u(N2)
    return (np.asarray(i, u) + u(N1) * np.asarray(j, u) + n12 * np.asarray(k1, u)
            + n12 * u(M1 - 1) * np.asarray(l1, u))


def quad_index(gid: int, N1: int, N2: int, M1: int, M2: int) -> QuadIndex:
    total = N1 * N2 * (M1 - 1) * (M2 - 1)
    if not (0 <= int(gid) < total):
        raise ConfigError(f"gid {gid} out of range [0, {total})")
    i, j, k1, l1 = gid_to_cartesian(int(gid), N1, N2, M1)
    return QuadIndex(int(gid), i, j, k1 + 1, l1 + 1)


def pair_counts(N1: int, N2: int, M1: int, M2: int):
    """(quad pairs, triangle pairs) — PAPER.md: 2,424,307,712 / 9,697,230,848 at (1024, 2048, 35, 35)."""
    q = N1 * N2 * (M1 - 1) * (M2 - 1)
    return q, 4 * q


# ---------------------------------------------------------------- helpers
def _coords(h, copy: bool = True) -> np.ndarray:
    if isinstance(h, HalfLayer):
        return np.ascontiguousarray(h.coords) if copy else h.coords
    c = np.asarray(h, dtype=np.float64)
    if c.ndim != 3 or c.shape[0] != 4:
        raise ConfigError("expected a HalfLayer or a (4, M, N) grid")
    return np.ascontiguousarray(c)


def _svals(h, M: int) -> np.ndarray:
    if isinstance(h, HalfLayer):
        return np.asarray(h.s_values, dtype=np.float64)
    return np.linspace(-1.0, 1.0, M)


def _task(u_half, s_half):
    if isinstance(u_half, HalfLayer) and isinstance(s_half, HalfLayer):
        return (u_half.n, "+" if u_half.sign >= 0 else "-", s_half.n, "+" if s_half.sign >= 0 else "-")
    return None


def _check_backend(backend: str):
    if backend not in BACKENDS:
        raise ConfigError(
            f"backend {backend!r} is not provided by this package (available: {BACKENDS}); the reference's "
            "'serial'/'parallel' CPU backends are restated only as test oracles under oracle/")


# ---------------------------------------------------------------- search API
def _mode_pipeline(mode: str, pipeline: str):
    m = _lib.MODE_NAMES.get(mode)
    if m is None:
        raise ConfigError(f"mode must be one of {sorted(_lib.MODE_NAMES)}, got {mode!r}")
    p = _lib.PIPELINE_NAMES.get(pipeline)
    if p is None:
        raise ConfigError(f"pipeline must be one of {sorted(_lib.PIPELINE_NAMES)}, got {pipeline!r}")
    if p == _lib.PIPE_SPEC and m != _lib.MODE_CULL:
        raise ConfigError("pipeline='spec' runs on the culling kernels (mode='cull')")
    return m, p


def search_hits(u_half, s_half, backend: str = "cuda", *, devices=(0,), mode: str = "cull",
                pipeline: str = "triangle", timing: bool = False):
    """Triangle-level hits (iA, iB, s, t, a, b), sorted by (iA, iB), plus kernel stats."""
    _check_backend(backend)
    m, p = _mode_pipeline(mode, pipeline)
    return _device.search(_coords(u_half), _coords(s_half), devices=devices, mode=m, timing=timing,
                          task=_task(u_half, s_half), pipeline=p)


def pair_candidates(u_half, s_half, backend: str = "cuda", *, device: int = 0, mode: str = "cull") -> np.ndarray:
    """Sorted u64 gids with ¬aabb_reject ∧ ¬moller_reject.

    ``mode="cull"`` (default) runs the quad tests only inside overlapping union boxes
    of the packed meshes; ``"brute"`` tests every quad pair.  Same result.
    """
    _check_backend(backend)
    if mode == "brute":
        return _device.pair_candidates_device(_coords(u_half), _coords(s_half), device=device,
                                              task=_task(u_half, s_half))
    if mode != "cull":
        raise ConfigError(f"mode must be 'brute' or 'cull', got {mode!r}")
    A = _device.DeviceMesh(_coords(u_half), device)
    B = _device.DeviceMesh(_coords(s_half), device)
    gids, _ = _device.pair_candidates_mesh(A, B, task=_task(u_half, s_half))
    return gids


def record_fields(coords_a, s_a, coords_b, s_b, hits):
    """Host (NumPy) record fields for hits: (gid u64, point (n,4), params (n,4)).

    Same op sequence as the device version (csrc/mcx_records.cu), bit-identical.
    """
    _, MA, NA = coords_a.shape
    _, MB, NB = coords_b.shape
    ia = hits["ia"].astype(np.int64)
    ib = hits["ib"].astype(np.int64)
    tauA, qa = ia & 1, ia >> 1
    tauB, qb = ib & 1, ib >> 1
    i, k1 = qa % NA, qa // NA
    j, l1 = qb % NB, qb // NB
    gid = cartesian_to_gid(i, j, k1, l1, NA, NB, MA)
    s, t, a, b = (hits[f] for f in ("s", "t", "a", "b"))
    # points p + s·e1 + t·e2 from A's grid (FMA-free, fixed order — SURVEY.md §7.3 step 8)
    W = np.transpose(coords_a, (1, 2, 0))
    ip = (i + 1) % NA
    v00, v10, v01, v11 = W[k1, i], W[k1, ip], W[k1 + 1, i], W[k1 + 1, ip]
    T2 = (tauA == 1)[:, None]
    p = np.where(T2, v01, v00)
    e1 = v10 - p
    e2 = np.where(T2, v11, v01) - p
    pts = (p + s[:, None] * e1) + t[:, None] * e2
    thA_n = np.append(grid_points(NA), 2.0 * np.pi)  # θ_N = 2π at the wrap (eq. 28)
    thB_n = np.append(grid_points(NB), 2.0 * np.pi)

    def est(theta_n, sv, ii, kk, tau, x, y):
        th0, th1 = theta_n[ii], theta_n[ii + 1]
        s0, s1 = sv[kk], sv[kk + 1]
        # T¹ (origin v00, edges to v10, v01): Eqs. 28-29, θ = (1−x)θ_i + xθ_{i+1}, s = (1−y)s_k + y s_{k+1};
        # T² (origin v01, edges to v10, v11): the affine map of its vertex parameters,
        #     θ = (1−x−y)θ_i + (x+y)θ_{i+1},  s = (1−x)s_{k+1} + x s_k.
        th = np.where(tau == 0, (1 - x) * th0 + x * th1, (1 - (x + y)) * th0 + (x + y) * th1)
        ss = np.where(tau == 0, (1 - y) * s0 + y * s1, (1 - x) * s1 + x * s0)
        return th, ss

    thu, su = est(thA_n, np.asarray(s_a, dtype=np.float64), i, k1, tauA, s, t)
    ths, ss = est(thB_n, np.asarray(s_b, dtype=np.float64), j, l1, tauB, a, b)
    return gid.astype(np.uint64), pts, np.stack([thu, su, ths, ss], axis=1)


def assemble_records(coords_a, coords_b, hits, gid, pts, params, layer=(0, "+", 0, "+"), tof=float("nan"),
                     dedup: bool = True):
    """Sort by (gid, τ_A, τ_B), deduplicate within 1e-9 and build records."""
    _, MA, NA = coords_a.shape
    _, MB, NB = coords_b.shape
    ia = hits["ia"].astype(np.int64)
    ib = hits["ib"].astype(np.int64)
    order = np.lexsort((ib & 1, ia & 1, gid))
    ia, ib, gid, pts, params = ia[order], ib[order], gid[order], pts[order], params[order]
    bary = np.stack([hits[f][order] for f in ("s", "t", "a", "b")], axis=1)
    keep = _dedup_mask(pts, DEDUP_TOL) if (dedup and len(gid) > 1) else np.ones(len(gid), dtype=bool)
    recs = []
    for n in np.nonzero(keep)[0]:
        qa, qb = int(ia[n]) >> 1, int(ib[n]) >> 1
        recs.append(IntersectionRecord(
            point=pts[n].copy(), bary=tuple(float(v) for v in bary[n]), params=tuple(float(v) for v in params[n]),
            pair=QuadIndex(int(gid[n]), qa % NA, qb % NB, qa // NA + 1, qb // NB + 1),
            tri=(int(ia[n]) & 1, int(ib[n]) & 1), layer=layer, tof=tof, tri_index=(int(ia[n]), int(ib[n]))))
    return recs


def hits_to_records(coords_a, s_a, coords_b, s_b, hits, layer=(0, "+", 0, "+"), tof=float("nan"),
                    dedup: bool = True):
    """Build sorted, deduplicated IntersectionRecords from triangle hits (host path)."""
    gid, pts, params = record_fields(coords_a, s_a, coords_b, s_b, hits)
    return assemble_records(coords_a, coords_b, hits, gid, pts, params, layer=layer, tof=tof, dedup=dedup)


def _dedup_mask(pts: np.ndarray, tol: float) -> np.ndarray:
    """Greedy in record order: drop a record whose point is within tol of a KEPT
    earlier record in every coordinate (|fl(p_c − q_c)| ≤ tol; the device runtime
    implements the same rule, csrc/mcx_runtime.cu).  Candidate pairs come from an
    x-sorted sweep with a 2·tol window (a superset, filtered exactly below); only
    records that have an earlier candidate are resolved in a Python loop."""
    n = len(pts)
    keep = np.ones(n, dtype=bool)
    order = np.argsort(pts[:, 0], kind="stable")
    xs = pts[order, 0]
    hi = np.searchsorted(xs, xs + 2.0 * tol, side="right")
    cnt = hi - np.arange(n) - 1
    if cnt.sum() == 0:
        return keep
    src = np.repeat(np.arange(n), cnt)
    dst = np.arange(cnt.sum()) - np.repeat(np.cumsum(cnt) - cnt, cnt) + src + 1
    a, b = order[src], order[dst]
    close = np.max(np.abs(pts[a] - pts[b]), axis=1) <= tol
    a, b = a[close], b[close]
    lo_, hi_ = np.minimum(a, b), np.maximum(a, b)  # record order: lo_ earlier
    earlier = {}
    for x, y in zip(lo_.tolist(), hi_.tolist()):
        earlier.setdefault(y, []).append(x)
    for y in sorted(earlier):
        if any(keep[x] for x in earlier[y]):
            keep[y] = False
    return keep


def record_fields_device(coords_a, s_a, coords_b, s_b, hits, device: int = 0):
    """Device record fields (csrc/mcx_records.cu, §8(f) row 4) for host hit arrays."""
    return _device.record_fields_device(coords_a, s_a, coords_b, s_b, hits, device=device)


def records_to_objects(recs, NA: int, NB: int, layer=(0, "+", 0, "+"), tof: float = float("nan")):
    """IntersectionRecords from the runtime's record array (runtime.RECORD_DTYPE)."""
    out = []
    ia = recs["ia"].astype(np.int64)
    ib = recs["ib"].astype(np.int64)
    qa, qb = ia >> 1, ib >> 1
    for n in range(len(recs)):
        out.append(IntersectionRecord(
            point=recs["point"][n].copy(), bary=tuple(float(v) for v in recs["bary"][n]),
            params=tuple(float(v) for v in recs["params"][n]),
            pair=QuadIndex(int(recs["gid"][n]), int(qa[n] % NA), int(qb[n] % NB), int(qa[n] // NA) + 1,
                           int(qb[n] // NB) + 1),
            tri=(int(ia[n]) & 1, int(ib[n]) & 1), layer=layer, tof=tof, tri_index=(int(ia[n]), int(ib[n]))))
    return out


def find_intersections(u_half, s_half, backend: str = "cuda", *, devices=(0,), mode: str = "cull",
                       pipeline: str = "spec", dedup: bool = True, tof: float = float("nan")):
    """All mesh intersections of two half-layers as IntersectionRecords.

    ``pipeline="spec"`` (default) is the SPEC's literal pipeline — quad AABB + Möller
    survivors, then the 4 triangle-pair precise tests of each — so the records equal
    the reference's serial backend's record for record.
    ``pipeline="triangle"`` tests every triangle pair's boxes (no Möller), which also
    keeps the touching hits floating-point Möller can drop.

    One GPU: one ``mcx_find_intersections`` call — upload, pack, search, records,
    (gid, τ_A, τ_B) sort and dedup all on the device.  Several GPUs: A's blocks are
    sharded over ``devices``, the hit lists gathered, and the records stage runs on
    ``devices[0]`` (``mcx_finish_hits``).
    """
    from . import runtime
    _check_backend(backend)
    m, p = _mode_pipeline(mode, pipeline)
    # a HalfLayer is read in place from its mesh (column range: contiguous within each
    # plane, the planes at the mesh's plane stride) — no host copy
    ca, cb = _coords(u_half, copy=False), _coords(s_half, copy=False)
    layer = _task(u_half, s_half) or (0, "+", 0, "+")
    sa, sb = _svals(u_half, ca.shape[1]), _svals(s_half, cb.shape[1])
    devices = list(devices)
    if not devices:
        raise ConfigError("devices must be non-empty")
    ctx = runtime.context(devices[0])
    if len(devices) == 1:
        recs, _, _ = ctx.find(ca, sa, cb, sb, layer, mode=m, pipeline=p, dedup=dedup, task=_task(u_half, s_half))
    else:
        ca, cb = np.ascontiguousarray(ca), np.ascontiguousarray(cb)
        res = _device.search(ca, cb, devices=devices, mode=m, task=_task(u_half, s_half), pipeline=p)
        A, B = ctx.mesh(ca, sa), ctx.mesh(cb, sb)
        try:
            recs, _ = ctx.finish_hits(res.hits, A, B, layer, dedup=dedup)
        finally:
            A.free()
            B.free()
    return records_to_objects(recs, ca.shape[2], cb.shape[2], layer=layer, tof=tof)


# ---------------------------------------------------------------- records file
def write_records(path, records) -> None:
    """Records text: ``n1 sign1 n2 sign2 gid x y px py a b c d theta_u s_u theta_s s_s``."""
    with open(path, "w") as fh:
        for r in records:
            fh.write(r.to_line() + "\n")


def read_records(path):
    out = []
    with open(path) as fh:
        for ln, line in enumerate(fh, 1):
            f = line.split()
            if not f:
                continue
            if len(f) != 17:
                raise FileFormatError(f"{path}:{ln}: expected 17 fields, got {len(f)}")
            try:
                n1, s1, n2, s2, gid = int(f[0]), f[1], int(f[2]), f[3], int(f[4])
                v = [float(x) for x in f[5:]]
            except ValueError as exc:
                raise FileFormatError(f"{path}:{ln}: {exc}") from None
            out.append(IntersectionRecord(point=np.array(v[0:4]), bary=tuple(v[4:8]), params=tuple(v[8:12]),
                                          pair=QuadIndex(gid, -1, -1, -1, -1), layer=(n1, s1, n2, s2)))
    return out
