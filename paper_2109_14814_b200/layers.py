"""Layer-pair plan (SPEC module ``layers``) — the task list the
reference's intersection stage dispatches to ``isect``.

Only the bookkeeping on the search path is here: ``enumerate_layer_pairs``
(with the ``--include-core`` extension of SPEC.md:398), the plan
text file ``n1 sign1 n2 sign2 tof``, and ``search_plan``, which runs
a plan as ONE batched device job per GPU (``mcx_intersect``: one launch per kernel
for all of the GPU's tasks, §8(f) row 3), each distinct half-layer uploaded and
packed once, records sorted / deduplicated / formatted on the device.  With several
GPUs the tasks are dealt out whole (they are independent) by a
deterministic longest-first assignment, one host thread per GPU.
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

from . import _lib, device as _device, isect, runtime
from .errors import ConfigError, FileFormatError
from .mesh import ManifoldMesh, half_layer


@dataclass
class LayerPairPlan:
    """Tasks (U_n1^sign1, S_n2^sign2) with time of flight 2π(n1+n2)/Ω_p."""

    tasks: list = field(default_factory=list)  # (n1, sign1, n2, sign2)
    tof: list = field(default_factory=list)

    def __len__(self):
        return len(self.tasks)


def enumerate_layer_pairs(u_mesh: ManifoldMesh, s_mesh: ManifoldMesh, n_max: int, omega_p: float = 1.0,
                          include_core: bool = False):
    """Pairs (U_n, S_n) and (U_n, S_{n−1}) for n = 1..n_max over all four sign
    combinations; (U_1, S_0) is skipped because layers start at 1 (SPEC.md:382-390,
    design decision).  Counts: n_max = 1 → 4, 2 → 12, 5 → 36, i.e. 4·(2·n_max − 1).

    ``include_core`` re-enables the fundamental-domain cores |s| < D as
    layer 0 (one half-layer per mesh, sign '+'): the same family extended to n = 0 adds
    (U_0, S_0) and (U_1^±, S_0), three tasks, listed first."""
    if n_max < 1:
        raise ConfigError("n_max must be >= 1")
    if n_max > u_mesh.n_max or n_max > s_mesh.n_max:
        raise ConfigError(f"meshes are globalized to n_max = {u_mesh.n_max}/{s_mesh.n_max} < {n_max}")
    plan = LayerPairPlan()
    if include_core:
        for task in ((0, "+", 0, "+"), (1, "+", 0, "+"), (1, "-", 0, "+")):
            plan.tasks.append(task)
            plan.tof.append(2.0 * math.pi * (task[0] + task[2]) / omega_p)
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


_SIGNS = ("+", "-")


def read_plan(path) -> LayerPairPlan:
    plan = LayerPairPlan()
    with open(path) as fh:
        for ln, line in enumerate(fh, 1):
            f = line.split()
            if not f:
                continue
            if len(f) != 5 or f[1] not in _SIGNS or f[3] not in _SIGNS:
                raise FileFormatError(f"{path}:{ln}: expected 'n1 sign1 n2 sign2 tof' with signs '+' / '-'")
            try:
                plan.tasks.append((int(f[0]), f[1], int(f[2]), f[3]))
                plan.tof.append(float(f[4]))
            except ValueError as exc:
                raise FileFormatError(f"{path}:{ln}: {exc}") from None
    return plan


def _sign(s: str) -> int:
    return 1 if s == "+" else -1


def assign_tasks(costs, n_devices: int):
    """Deterministic longest-processing-time-first assignment of whole tasks to GPUs
    (ties by task index).  Returns one sorted task-index list per device."""
    load = [0.0] * n_devices
    out = [[] for _ in range(n_devices)]
    for k in sorted(range(len(costs)), key=lambda k: (-costs[k], k)):
        d = min(range(n_devices), key=lambda d: (load[d], d))
        out[d].append(k)
        load[d] += costs[k]
    return [sorted(o) for o in out]


@dataclass
class PlanResult:
    records: list      # IntersectionRecords of all tasks, plan order
    stats: list        # per task: counters (+ "layer", "device")
    text: bytes = b""  # the records file body, when requested

    def __iter__(self):  # records, stats = search_plan(...)
        return iter((self.records, self.stats))


def _halves(u_mesh, s_mesh, plan):
    halves = {}
    for (n1, s1, n2, s2) in plan.tasks:
        for key, mesh, n, sg in ((("u", n1, s1), u_mesh, n1, s1), (("s", n2, s2), s_mesh, n2, s2)):
            if key not in halves:
                halves[key] = half_layer(mesh, n, _sign(sg))
    return halves


def plan_parts(u_mesh, s_mesh, plan, n_parts: int):
    """(half-layers by key, task-index lists): whole tasks dealt over n_parts GPUs/ranks by
    estimated cost (triangle pairs), deterministically."""
    halves = _halves(u_mesh, s_mesh, plan)
    costs = [halves[("u", n1, s1)].n_triangles * halves[("s", n2, s2)].n_triangles
             for (n1, s1, n2, s2) in plan.tasks]
    return halves, assign_tasks(costs, n_parts)


def run_part(halves, plan, mine, device: int, mode: int, pipeline: int, dedup: bool, text: bool):
    """One GPU's share: each mesh its tasks need uploaded once (mcx_grid_load), every
    half-layer a zero-copy column view of it packed in place, one mcx_intersect over the
    tasks.  Returns (records with task = index into ``mine``, text,
    per-task stats)."""
    if not mine:
        return np.zeros(0, runtime.RECORD_DTYPE), b"", []
    ctx = runtime.context(device)
    grids, meshes = {}, {}
    try:
        jobs = []
        for k in mine:
            n1, s1, n2, s2 = plan.tasks[k]
            for key in (("u", n1, s1), ("s", n2, s2)):
                if key not in meshes:
                    h = halves[key]
                    parent = id(h.mesh)
                    if parent not in grids:  # each mesh crosses PCIe once, in one copy
                        grids[parent] = ctx.grid(h.mesh.coords, h.mesh.s_values)
                    meshes[key] = ctx.view(grids[parent], *h.col_range)
            jobs.append((meshes[("u", n1, s1)], meshes[("s", n2, s2)], plan.tasks[k]))
        return ctx.intersect(jobs, mode=mode, pipeline=pipeline, dedup=dedup, text=text,
                             task_ids=[plan.tasks[k] for k in mine])
    finally:
        for mesh in meshes.values():
            mesh.free()
        for g in grids.values():
            g.free()


def merge_parts(plan, halves, parts, outs, devices, text: bool) -> PlanResult:
    """Plan-order records / stats / text from every part's (records, text, stats)."""
    per_task = [None] * len(plan)
    for rank, (recs, txt, stats) in enumerate(outs):
        mine = parts[rank]
        lines = txt.split(b"\n")[:-1] if txt else []
        cut = np.searchsorted(recs["task"], np.arange(len(mine) + 1)) if len(recs) else np.zeros(len(mine) + 1, int)
        for j, k in enumerate(mine):
            seg = recs[cut[j]:cut[j + 1]]
            body = b"".join(ln + b"\n" for ln in lines[cut[j]:cut[j + 1]]) if text else b""
            per_task[k] = (seg, body, {"layer": plan.tasks[k], "device": devices[rank], **stats[j]})
    records, stats, chunks = [], [], []
    for k, (seg, body, st) in enumerate(per_task):
        n1, s1, n2, s2 = plan.tasks[k]
        hu, hs = halves[("u", n1, s1)], halves[("s", n2, s2)]
        records.extend(isect.records_to_objects(seg, hu.N, hs.N, layer=plan.tasks[k], tof=plan.tof[k]))
        stats.append(st)
        chunks.append(body)
    return PlanResult(records=records, stats=stats, text=b"".join(chunks))


def search_plan(u_mesh: ManifoldMesh, s_mesh: ManifoldMesh, plan: LayerPairPlan, backend: str = "cuda", *,
                mode: str = "cull", pipeline: str = "spec", device: int = 0, devices=None, dedup: bool = True,
                text: bool = False) -> PlanResult:
    """Run every layer-pair task of ``plan``.

    Per GPU one ``mcx_intersect`` call over its tasks: the distinct half-layers it
    needs are uploaded and packed once, every task's search runs in one batched
    launch, and records come back sorted by (gid, τ_A, τ_B) and deduplicated per task
    exactly as ``isect.find_intersections`` returns them.  ``devices`` deals whole tasks
    over several GPUs (one host thread each); the result is in plan order either way.
    """
    isect._check_backend(backend)
    m, p = isect._mode_pipeline(mode, pipeline)
    devices = list(devices) if devices is not None else [device]
    if not devices:
        raise ConfigError("devices must be non-empty")
    halves, parts = plan_parts(u_mesh, s_mesh, plan, len(devices))
    outs = _device.run_on_devices(lambda r: run_part(halves, plan, parts[r], devices[r], m, p, dedup, text), devices)
    return merge_parts(plan, halves, parts, outs, devices, text)


def search_plan_distributed(u_mesh: ManifoldMesh, s_mesh: ManifoldMesh, plan: LayerPairPlan,
                            backend: str = "cuda", *, mode: str = "cull", pipeline: str = "spec", device: int = 0,
                            dedup: bool = True, text: bool = False, dst: int = 0, group=None):
    """``search_plan`` as one rank of a torch.distributed job (one process per GPU,
    torchrun): every rank runs its whole tasks on ``device`` and the (small) record
    lists are gathered to ``dst``, which returns the plan-order PlanResult (None on the
    other ranks).  Result collection only — no collective on the data path."""
    import torch.distributed as dist
    isect._check_backend(backend)
    m, p = isect._mode_pipeline(mode, pipeline)
    world, rank = dist.get_world_size(group), dist.get_rank(group)
    halves, parts = plan_parts(u_mesh, s_mesh, plan, world)
    out = run_part(halves, plan, parts[rank], device, m, p, dedup, text)
    gathered = [None] * world if rank == dst else None
    dist.gather_object((out[0].tobytes(), out[1], out[2], device), gathered, dst=dst, group=group)
    if rank != dst:
        return None
    outs = [(np.frombuffer(r, dtype=runtime.RECORD_DTYPE), t, st) for r, t, st, _ in gathered]
    return merge_parts(plan, halves, parts, outs, [g[3] for g in gathered], text)
