"""Mesh and half-layer views — the input side of the search.

Layout (PAPER.md "Discrete Mesh", paper's storage convention):
a manifold mesh is four N×M float64 planes (x, y, px, py) in **column-major**
order, entry (i, k) = coordinate of W(θ_i, s_k) at linear index ``i + N·k``
(θ fastest, θ periodic).  Here that is one C-contiguous array
``coords[c, k, i]`` of shape (4, M, N), i.e. plane-major, then column, then θ
— byte-identical to the paper's four column-major planes laid end to end, and
to the MNF1 file body.

A half-layer is a contiguous column range of a mesh; its
triangles are the ``2·N·(M_h−1)`` triangles of the quads between consecutive
columns of that range.

Also here: the frozen synthetic generators the benchmark and parity tests use
 and the MNF1 reader/writer (house style of the
reference's ICR1 I/O, torus.py:285-309).
"""
from __future__ import annotations

import struct
from dataclasses import dataclass, field

import numpy as np

from .errors import ConfigError, FileFormatError

MESH_MAGIC = b"MNF1"


def grid_points(n: int) -> np.ndarray:
    """θ_i = 2πi/N — same expression as the reference (fourier.py:23-25)."""
    return 2.0 * np.pi * np.arange(n) / n


@dataclass
class ManifoldMesh:
    """A globalized manifold mesh.

    ``coords``: float64 (4, M, N), C-contiguous, ``coords[c, k, i]`` = coordinate
    c of W(θ_i, s_k).  ``s_values``: sorted (M,).
    """

    coords: np.ndarray
    s_values: np.ndarray
    kind: str = "unstable"
    omega: float = float("nan")
    lam: float = float("nan")
    D: float = float("nan")
    n_max: int = 0
    boundary_cols: tuple = field(default_factory=tuple)

    def __post_init__(self):
        c = np.ascontiguousarray(np.asarray(self.coords, dtype=np.float64))
        if c.ndim != 3 or c.shape[0] != 4:
            raise ConfigError(f"mesh coords must have shape (4, M, N), got {c.shape}")
        self.coords = c
        self.s_values = np.ascontiguousarray(np.asarray(self.s_values, dtype=np.float64))
        if self.s_values.shape != (c.shape[1],):
            raise ConfigError(f"s_values must have shape ({c.shape[1]},), got {self.s_values.shape}")
        if self.kind not in ("unstable", "stable"):
            raise ConfigError(f"mesh kind must be 'unstable' or 'stable', got {self.kind!r}")

    @classmethod
    def from_planes(cls, x, y, px, py, s_values, **kw) -> "ManifoldMesh":
        """Build from the paper's four N×M arrays (row i = θ_i, column k = s_k)."""
        planes = [np.asarray(p, dtype=np.float64) for p in (x, y, px, py)]
        shape = planes[0].shape
        if any(p.shape != shape for p in planes) or len(shape) != 2:
            raise ConfigError("the four coordinate planes must be N×M arrays of one shape")
        coords = np.stack([p.T for p in planes])  # (4, M, N)
        return cls(coords=coords, s_values=s_values, **kw)

    @property
    def N(self) -> int:
        return self.coords.shape[2]

    @property
    def M(self) -> int:
        return self.coords.shape[1]

    def plane(self, c: int) -> np.ndarray:
        """Coordinate plane c as the paper's N×M array (a view)."""
        return self.coords[c].T


@dataclass
class HalfLayer:
    """Contiguous column range [first, last] of a parent mesh."""

    mesh: ManifoldMesh
    n: int = 0
    sign: int = 1
    col_range: tuple = (0, 0)

    def __post_init__(self):
        first, last = (int(v) for v in self.col_range)
        if not (0 <= first < last < self.mesh.M):
            raise ConfigError(
                f"half-layer column range {self.col_range} must satisfy 0 <= first < last < M={self.mesh.M}"
                " (pair_candidates needs >= 2 columns, SPEC.md:473)")
        self.col_range = (first, last)

    @classmethod
    def whole(cls, mesh: ManifoldMesh, n: int = 0, sign: int = 1) -> "HalfLayer":
        return cls(mesh=mesh, n=n, sign=sign, col_range=(0, mesh.M - 1))

    @property
    def N(self) -> int:
        return self.mesh.N

    @property
    def M(self) -> int:
        return self.col_range[1] - self.col_range[0] + 1

    @property
    def coords(self) -> np.ndarray:
        """(4, M_h, N) view of this half-layer's columns (C-contiguous per plane)."""
        a, b = self.col_range
        return self.mesh.coords[:, a:b + 1, :]

    @property
    def s_values(self) -> np.ndarray:
        a, b = self.col_range
        return self.mesh.s_values[a:b + 1]

    @property
    def n_quads(self) -> int:
        return self.N * (self.M - 1)

    @property
    def n_triangles(self) -> int:
        return 2 * self.n_quads

    @property
    def task(self):
        return (self.n, "+" if self.sign >= 0 else "-")


def half_layer(mesh: ManifoldMesh, n: int, sign: int) -> HalfLayer:
    """Columns spanning layer n on the given side (Eqs. 17-20).

    Unstable: s ∈ sign·[Dλ^(n−1), Dλ^n]; stable: s ∈ sign·[D/λ^(n−1), D/λ^n].
    Endpoints must be members of ``s_values`` within 1e-12 (layer boundaries are
    grid members by construction, PAPER.md "Discrete Mesh").  ``n = 0`` is the
    fundamental-domain core s ∈ [−D, D] (one half-layer, sign +), searched only
    with ``--include-core``.
    """
    if n == 0:
        if sign != 1:
            raise ConfigError("the core (n = 0) is one half-layer, sign '+'")
        lo, hi = -mesh.D, mesh.D
    else:
        if not (1 <= n <= mesh.n_max):
            raise ConfigError(f"layer index n={n} out of range 1..{mesh.n_max}")
        if sign not in (1, -1):
            raise ConfigError(f"sign must be +1 or -1, got {sign}")
        lam = mesh.lam if mesh.kind == "unstable" else 1.0 / mesh.lam
        e0 = sign * mesh.D * lam ** (n - 1)
        e1 = sign * mesh.D * lam ** n
        lo, hi = min(e0, e1), max(e0, e1)
    s = mesh.s_values
    tol = 1e-12 * max(1.0, abs(hi))
    k_lo = int(np.argmin(np.abs(s - lo)))
    k_hi = int(np.argmin(np.abs(s - hi)))
    if abs(s[k_lo] - lo) > tol or abs(s[k_hi] - hi) > tol:
        raise ConfigError(f"layer {n}{'+' if sign > 0 else '-'} boundaries {lo}, {hi} are not grid members")
    return HalfLayer(mesh=mesh, n=n, sign=sign, col_range=(k_lo, k_hi))


# --------------------------------------------------------------------------- MNF1
def write_mesh(path, mesh: ManifoldMesh) -> None:
    """MNF1 file: magic, u32 N, u32 M, u8 kind, f64 ω, λ, D, u32 n_max,
    4 column-major N×M planes, M s-values, u32 count + u32 boundary-column indices."""
    with open(path, "wb") as fh:
        fh.write(MESH_MAGIC)
        fh.write(struct.pack("<IIB", mesh.N, mesh.M, 0 if mesh.kind == "unstable" else 1))
        fh.write(struct.pack("<ddd", mesh.omega, mesh.lam, mesh.D))
        fh.write(struct.pack("<I", mesh.n_max))
        fh.write(np.ascontiguousarray(mesh.coords, dtype="<f8").tobytes())
        fh.write(np.ascontiguousarray(mesh.s_values, dtype="<f8").tobytes())
        fh.write(struct.pack("<I", len(mesh.boundary_cols)))
        fh.write(np.asarray(mesh.boundary_cols, dtype="<u4").tobytes())


def read_mesh(path) -> ManifoldMesh:
    with open(path, "rb") as fh:
        magic = fh.read(4)
        if magic != MESH_MAGIC:
            raise FileFormatError(f"{path}: bad magic {magic!r}, expected MNF1")
        try:
            n, m, kind = struct.unpack("<IIB", fh.read(9))
            omega, lam, D = struct.unpack("<ddd", fh.read(24))
            (n_max,) = struct.unpack("<I", fh.read(4))
            body = fh.read(8 * 4 * n * m)
            sv = fh.read(8 * m)
            if len(body) != 32 * n * m or len(sv) != 8 * m:
                raise FileFormatError(f"{path}: truncated mesh data")
            (nb,) = struct.unpack("<I", fh.read(4))
            bc = fh.read(4 * nb)
            if len(bc) != 4 * nb:
                raise FileFormatError(f"{path}: truncated boundary list")
        except struct.error as exc:
            raise FileFormatError(f"{path}: truncated header ({exc})") from None
        if fh.read(1):
            raise FileFormatError(f"{path}: trailing bytes after mesh data")
    coords = np.frombuffer(body, dtype="<f8").reshape(4, m, n).copy()
    return ManifoldMesh(coords=coords, s_values=np.frombuffer(sv, dtype="<f8").copy(),
                        kind="unstable" if kind == 0 else "stable", omega=omega, lam=lam, D=D,
                        n_max=n_max, boundary_cols=tuple(int(v) for v in np.frombuffer(bc, dtype="<u4")))


# ------------------------------------------------------------ synthetic generators
def manifold_like(N: int, M: int, seed: int, s_values=None):
    """Smooth annulus-like sheet in 4D, frozen per SURVEY.md §8(d).

    Returns ``(coords (4, M, N), s_values (M,))``.  Draws do not depend on (N, M),
    so one seed samples the same surface at any resolution.  ``s_values``
    (optional, length M) evaluates the surface at arbitrary s instead of
    ``linspace(-1, 1, M)``.
    """
    theta = grid_points(N)
    s = np.linspace(-1.0, 1.0, M) if s_values is None else np.asarray(s_values, dtype=np.float64)
    M = s.shape[0]
    rng = np.random.default_rng(seed)
    S = s[:, None]
    T = theta[None, :]
    out = np.empty((4, M, N))
    base = (np.cos(T), np.sin(T), np.zeros_like(T), np.zeros_like(T))
    for c in range(4):
        acc = np.broadcast_to(base[c], (M, N)).copy()
        for m in range(1, 4):
            a, b, e, f = rng.normal(0.0, 0.3 / m, 4)
            cm, sm = np.cos(m * T), np.sin(m * T)
            acc = acc + (a * cm + b * sm) + S * (e * cm + f * sm)
        acc = acc + S * rng.normal(0.0, 0.5) + 0.05 * S * S * rng.normal()
        out[c] = acc
    out += 0.0  # canonicalise -0.0 to +0.0
    return out, s


def layered_mesh(N: int, kind: str, n_max: int, lam: float, D: float, seed: int, K: int = 4,
                 per_layer: int = 4) -> ManifoldMesh:
    """Synthetic globalized mesh with layer bookkeeping.

    s grid: the fundamental grid kD/K (k = −K..K) plus ``per_layer`` points per
    layer on each side, with every layer boundary ±D·μ^n (μ = λ unstable, 1/λ
    stable) a grid member, as globalization guarantees (PAPER.md "Discrete Mesh").
    Coordinates: the frozen smooth surface of ``manifold_like`` at those s
    (scaled to [-1, 1]).
    """
    mu = lam if kind == "unstable" else 1.0 / lam
    if mu <= 1.0:
        raise ConfigError("layers need |multiplier| > 1 in the growing direction")
    sv = {k * D / K for k in range(-K, K + 1)}
    for n in range(1, n_max + 1):
        lo, hi = D * mu ** (n - 1), D * mu ** n
        for j in range(per_layer + 1):
            v = lo + (hi - lo) * j / per_layer
            sv.add(v)
            sv.add(-v)
    s = np.array(sorted(sv))
    coords, _ = manifold_like(N, len(s), seed, s_values=s / s.max())
    bcols = tuple(int(np.argmin(np.abs(s - sg * D * mu ** n))) for n in range(0, n_max + 1) for sg in (-1, 1))
    return ManifoldMesh(coords=coords, s_values=s, kind=kind, omega=1.0, lam=lam, D=D, n_max=n_max,
                        boundary_cols=tuple(sorted(set(bcols))))


def dyadic(coords: np.ndarray, bits: int = 8) -> np.ndarray:
    """Round to multiples of 2^-bits (exact-arithmetic stress grid)."""
    q = float(2 ** bits)
    return np.round(coords * q) / q + 0.0


def stress_pair(kind: str, N: int = 64, M: int = 64, seed: int = 3):
    """Near-degenerate stress pairs C4.

    ``"same"`` (i): B = A.  ``"dyadic"`` (ii): A on a 2^-8 lattice, B = A with
    alternate nodes displaced by multiples of 2^-8 along ê3/ê4.  ``"tangent"``
    (iii): B = A + 1e-9·(sin 5θ·ê3 + sin 3πs·ê4).  Returns (A, B, s_values).
    """
    A, s = manifold_like(N, M, seed)
    if kind == "same":
        return A, A.copy(), s
    if kind == "dyadic":
        A = dyadic(A, 8)
        B = A.copy()
        rng = np.random.default_rng(seed + 100)
        k_idx, i_idx = np.meshgrid(np.arange(M), np.arange(N), indexing="ij")
        alt = ((k_idx + i_idx) % 2) == 1
        d3 = rng.integers(-2, 3, size=(M, N)) / 256.0
        d4 = rng.integers(-2, 3, size=(M, N)) / 256.0
        B[2] = np.where(alt, B[2] + d3, B[2])
        B[3] = np.where(alt, B[3] + d4, B[3])
        return A, B + 0.0, s
    if kind == "tangent":
        theta = grid_points(N)
        B = A.copy()
        B[2] = B[2] + 1e-9 * np.sin(5 * theta)[None, :]
        B[3] = B[3] + 1e-9 * np.sin(3 * np.pi * s)[:, None]
        return A, B, s
    raise ConfigError(f"unknown stress kind {kind!r}")


def unbalanced_pair(scale: int = 1, dense: bool = False):
    """C5: A = manifold_like(2048/scale, 1024/scale+1, 1); B = the same
    surface at (256/scale, 128/scale+1) plus a small offset and a lift L(s) that
    raises B off A outside s ≤ −0.75, concentrating hits in A's first ~1/8 columns.

    ``dense=True`` is the high-hit-density variant the SURVEY asks for (configs[4]:
    "exercising hit compaction"): offset frequencies raised to sin(64θ) and sin(64πs)
    (B's 256 θ-samples resolve up to ~sin(64θ)) and the band widened to s ≤ −0.625.
    Frozen at full scale: 13,226 hits, all in A's first quarter of columns (65 % in the
    first eighth), 2.38M AABB passes (measured with the C oracle's exact sweep)."""
    NA, MA = 2048 // scale, 1024 // scale + 1
    NB, MB = 256 // scale, 128 // scale + 1
    A, sA = manifold_like(NA, MA, 1)
    B, sB = manifold_like(NB, MB, 1)
    theta = grid_points(NB)
    ds = sB[1] - sB[0]
    band, ft, fs = (-0.625, 64, 64) if dense else (-0.75, 16, 8)
    L = np.clip((sB - band) / ds, 0.0, 1.0) * 3.0
    B[2] = B[2] + 1e-3 * np.sin(ft * theta)[None, :] + L[:, None]
    B[3] = B[3] + 1e-3 * np.sin(fs * np.pi * sB)[:, None]
    return A, sA, B + 0.0, sB


def ruled_pair(NA: int = 128, MA: int = 33, NB: int = 96, MB: int = 9, a: float = 0.5):
    """Two ruled-surface meshes crossing along a known curve (SPEC.md:485's synthetic
    geometry oracle).  A(θ, s) = (cos θ, sin θ, s, 0): a cylinder in the hyperplane py = 0,
    ruled along px.  B(φ, t) = c(φ) + t·d(φ) with c(φ) = (cos φ, sin φ, h(φ), 0) on that
    cylinder, h(φ) = 0.3 sin 2φ + 0.1, and d(φ) = (a cos φ, a sin φ, 0, 1) leaving the
    hyperplane, so A ∩ B is exactly the curve c(φ) (B's py = t vanishes only at t = 0).
    B's t grid avoids 0 and its θ grid differs from A's, so the discrete surfaces cross
    transversally near the curve.  Returns (A, s_A, B, t_B); ``curve(φ)`` gives c."""
    th = grid_points(NA)
    s = np.linspace(-1.0, 1.0, MA)
    A = np.empty((4, MA, NA))
    A[0], A[1], A[2], A[3] = np.cos(th)[None, :], np.sin(th)[None, :], s[:, None], 0.0
    ph = grid_points(NB)
    t = np.linspace(-0.31, 0.29, MB)
    R = 1.0 + a * t[:, None]
    B = np.empty((4, MB, NB))
    B[0], B[1] = R * np.cos(ph)[None, :], R * np.sin(ph)[None, :]
    B[2] = (0.3 * np.sin(2.0 * ph) + 0.1)[None, :]
    B[3] = t[:, None]
    return A + 0.0, s, B + 0.0, t


def ruled_curve(phi):
    """The analytic intersection curve of ``ruled_pair``: (cos φ, sin φ, 0.3 sin 2φ + 0.1, 0)."""
    phi = np.asarray(phi, dtype=np.float64)
    return np.stack([np.cos(phi), np.sin(phi), 0.3 * np.sin(2.0 * phi) + 0.1, 0.0 * phi], axis=-1)


CONFIGS = {
    # name: (NA, MA, seedA, NB, MB, seedB)
    "C1": (64, 64, 1, 64, 64, 2),
    "C2": (256, 256, 1, 256, 256, 2),
    "C3": (1024, 512, 1, 1024, 512, 2),
}


def config_pair(name: str):
    """(A coords, A s, B coords, B s) for the named BASELINE config."""
    if name in CONFIGS:
        na, ma, sa, nb, mb, sb = CONFIGS[name]
        A, s_a = manifold_like(na, ma, sa)
        B, s_b = manifold_like(nb, mb, sb)
        return A, s_a, B, s_b
    if name.startswith("C4"):
        kind = {"C4i": "same", "C4ii": "dyadic", "C4iii": "tangent"}[name]
        A, B, s = stress_pair(kind)
        return A, s, B, s.copy()
    if name == "C5":
        return unbalanced_pair(1)
    if name == "C5hd":
        return unbalanced_pair(1, dense=True)
    if name.startswith("C5/"):
        return unbalanced_pair(int(name[3:]))
    raise ConfigError(f"unknown config {name!r}")
