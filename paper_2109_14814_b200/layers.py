"""Layer-pair plan (SPEC module ``layers``) — the task list the
reference's intersection stage dispatches to ``isect``.

Only the bookkeeping on the search path is here: ``enumerate_layer_pairs``
(SPEC.md:382-390), the plan text file ``n1 sign1 n2 sign2 tof``, and
``search_plan``, which runs every task of a plan as ONE batched device job
(``mcx_search_batch``: one launch per kernel for all tasks, §8(f) row 3), each
distinct half-layer uploaded and packed once.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as _device, isect
from .errors import ConfigError, FileFormatError
from .mesh import ManifoldMesh, half_layer


@dataclass
class LayerPairPlan:
    """Tasks (U_n1^sign1, S_n2^sign2) with time of flight 2π(n1+n2)/Ω_p."""

    tasks: list = field(default_factory=list)  # (n1, sign1, n2, sign2)
    tof: list = field(default_factory=list)

    def __len__(self):
        return len(self.tasks)


def enumerate_layer_pairs(u_mesh: ManifoldMesh, s_mesh: ManifoldMesh, n_max: int, omega_p: float = 1.0):
    """Pairs (U_n, S_n) and (U_n, S_{n−1}) for n = 1..n_max over all four sign
    combinations; (U_1, S_0) is skipped because layers start at 1 (SPEC.md:382-390,
    design decision).  Counts: n_max = 1 → 4, 2 → 12, 5 → 36, i.e. 4·(2·n_max − 1)."""
    if n_max < 1:
        raise ConfigError("n_max must be >= 1")
    if n_max > u_mesh.n_max or n_max > s_mesh.n_max:
        raise ConfigError(f"meshes are globalized to n_max = {u_mesh.n_max}/{s_mesh.n_max} < {n_max}")
    plan = LayerPairPlan()
    for n in range(1, n_max + 1):
        for n2 in (n, n - 1):
            if n2 < 1:
                continue
            for s1 in ("+", "-"):
                for s2 in ("+", "-"):
                    plan.tasks.append((n, s1, n2, s2))
                    plan.tof.append(2.0 * math.pi * (n + n2) / omega_p)
    return plan


def write_plan(path, plan: LayerPairPlan) -> None:
    with open(path, "w") as fh:
        for (n1, s1, n2, s2), tof in zip(plan.tasks, plan.tof):
            fh.write(f"{n1} {s1} {n2} {s2} {tof:.17g}\n")


def read_plan(path) -> LayerPairPlan:
    plan = LayerPairPlan()
    with open(path) as fh:
        for ln, line in enumerate(fh, 1):
            f = line.split()
            if not f:
                continue
            if len(f) != 5 or f[1] not in "+-" or f[3] not in "+-":
                raise FileFormatError(f"{path}:{ln}: expected 'n1 sign1 n2 sign2 tof'")
            try:
                plan.tasks.append((int(f[0]), f[1], int(f[2]), f[3]))
                plan.tof.append(float(f[4]))
            except ValueError as exc:
                raise FileFormatError(f"{path}:{ln}: {exc}") from None
    return plan


def _sign(s: str) -> int:
    return 1 if s == "+" else -1


def search_plan(u_mesh: ManifoldMesh, s_mesh: ManifoldMesh, plan: LayerPairPlan, backend: str = "cuda", *,
                mode: str = "cull", device: int = 0, dedup: bool = True):
    """Run every layer-pair task of ``plan`` as one batched device job.

    Returns ``(records, per_task_stats)``: records of all tasks in plan order (each
    task's records sorted by gid and deduplicated as ``find_intersections`` does),
    and the per-task counters (the RunManifest's survivor/hit counts).
    """
    isect._check_backend(backend)
    m = _lib.MODE_NAMES.get(mode)
    if m is None:
        raise ConfigError(f"mode must be one of {sorted(_lib.MODE_NAMES)}, got {mode!r}")
    halves = {}

    def get(mesh, key, n, s):
        if key not in halves:
            h = half_layer(mesh, n, _sign(s))
            halves[key] = (h, _device.DeviceMesh(np.ascontiguousarray(h.coords), device))
        return halves[key]

    pairs, meta = [], []
    for (n1, s1, n2, s2), tof in zip(plan.tasks, plan.tof):
        hu, du = get(u_mesh, ("u", n1, s1), n1, s1)
        hs, ds = get(s_mesh, ("s", n2, s2), n2, s2)
        pairs.append((du, ds))
        meta.append((hu, hs, (n1, s1, n2, s2), tof))
    results = _device.search_batch(pairs, mode=m, task_ids=None)
    records, stats = [], []
    for res, (hu, hs, layer, tof) in zip(results, meta):
        ca, cb = np.ascontiguousarray(hu.coords), np.ascontiguousarray(hs.coords)
        gid, pts, params = _device.record_fields_device(ca, hu.s_values, cb, hs.s_values, res.hits, device=device)
        records.extend(isect.assemble_records(ca, cb, res.hits, gid, pts, params, layer=layer, tof=tof,
                                              dedup=dedup))
        stats.append({"layer": layer, **res.stats})
    return records, stats
