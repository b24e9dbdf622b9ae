"""Device-side orchestration: HBM buffers (torch as the allocator), packing,
search calls through the C ABI, capacity handling and multi-GPU sharding.

HBM layout per mesh (DESIGN.md §Data layout):
  coords  (4, M, N) f64  — the half-layer grid as uploaded (32·N·M bytes); the
                           precise test rebuilds survivor triangles from it
  box     (n, 8)    f64  — per-triangle AABB lo[4], hi[4] (64 B/tri), the only
                           array the hot loops stream
  perm    (n,)      u32  — storage position → original triangle index
  gbox/tbox/bbox         — union boxes per 32 / 512 / 1024 records (culling)
Hits come back as (iA, iB, s, t, a, b) records of 40 B.

Multi-GPU: A's triangle range is cut into blocks of
``mcx_a_block()`` triangles assigned cyclically (block b → GPU b mod G), B is
replicated, each GPU searches its blocks independently on its own host thread
and the host concatenates and sorts the small hit lists.  No collective.
"""
from __future__ import annotations

import threading
from concurrent.futures import ThreadPoolExecutor
from dataclasses import dataclass

import numpy as np

from . import _lib
from .errors import BackendError, CapacityError, ConfigError

HIT_DTYPE = np.dtype([("ia", "<u4"), ("ib", "<u4"), ("s", "<f8"), ("t", "<f8"), ("a", "<f8"), ("b", "<f8")])
assert HIT_DTYPE.itemsize == 40

_torch = None


def torch():
    global _torch
    if _torch is None:
        import torch as _t
        _torch = _t
    return _torch


def _require_cuda(device: int):
    t = torch()
    if not t.cuda.is_available():
        raise BackendError("backend='cuda' requires a CUDA device (none visible)")
    if device >= t.cuda.device_count():
        raise ConfigError(f"device {device} not present ({t.cuda.device_count()} visible)")


def _check_coords(coords) -> None:
    if coords.ndim != 3 or coords.shape[0] != 4:
        raise ConfigError(f"coords must have shape (4, M, N), got {tuple(coords.shape)}")
    if coords.shape[1] < 2 or coords.shape[2] < 1:
        raise ConfigError("a half-layer needs >= 2 columns (SPEC.md:473)")


class DeviceMesh:
    """A half-layer grid resident in HBM, packed into triangle boxes on the device.

    One ``mcx_pack`` call writes the boxes in the tiled order (``_lib.ORDER_TILED``)
    with ``perm`` mapping storage position → original triangle index, plus the
    culling hierarchy (group / tile / block union boxes).  All search modes use this
    layout; hits always carry original indices.
    """

    def __init__(self, coords, device: int = 0, stream=None, order: int = _lib.ORDER_TILED):
        t = torch()
        _require_cuda(device)
        dev = t.device("cuda", device)
        _check_coords(coords)
        if isinstance(coords, np.ndarray):
            coords = t.from_numpy(np.ascontiguousarray(coords, dtype=np.float64))
        self.device = device
        L = _lib.load()
        # NaN/Inf are detected on the device by mcx_pack (status flag) and reported
        # by the search; no host-side pass over the coordinates.
        with t.cuda.device(device):
            s = stream or t.cuda.current_stream(device)
            with t.cuda.stream(s):
                pinned = coords.device.type == "cpu" and coords.is_pinned()
                self.coords = coords.to(dev, dtype=t.float64, non_blocking=pinned).contiguous()
                _, self.M, self.N = (int(v) for v in self.coords.shape)
                self.n_tri = 2 * self.N * (self.M - 1)
                if self.n_tri >= 2 ** 31:
                    raise ConfigError("triangle count must be < 2^31")
                n = self.n_tri
                self.order = order
                self.box = t.empty((n, _lib.BOX_STRIDE), dtype=t.float64, device=dev)
                self.perm = t.empty(n, dtype=t.int32, device=dev) if order == _lib.ORDER_TILED else None
                self.gbox = t.empty((-(-n // _lib.GROUP), 8), dtype=t.float64, device=dev)
                self.tbox = t.empty((-(-n // _lib.TILE), 8), dtype=t.float64, device=dev)
                self.bbox = t.empty((-(-n // _lib.BLOCK), 8), dtype=t.float64, device=dev)
                self.status = t.empty(1, dtype=t.int32, device=dev)
            rc = L.mcx_pack(self.coords.data_ptr(), self.N, self.M, order, self.box.data_ptr(),
                            self.perm.data_ptr() if self.perm is not None else None, self.gbox.data_ptr(),
                            self.tbox.data_ptr(), self.bbox.data_ptr(), self.status.data_ptr(), device, s.cuda_stream)
        _lib.check(rc, "mcx_pack")

    def struct(self) -> _lib.MeshDev:
        """The mcx_mesh_dev view of this mesh (built once: the buffers never move)."""
        if getattr(self, "_struct", None) is None:
            self._struct = _lib.MeshDev(self.n_tri, self.coords.data_ptr(), self.N, self.M, self.box.data_ptr(),
                                        self.perm.data_ptr() if self.perm is not None else None,
                                        self.gbox.data_ptr(), self.tbox.data_ptr(), self.bbox.data_ptr(),
                                        self.status.data_ptr(), self.M, 0)
            self._struct_ptr = ctypes_pointer(self._struct)
        return self._struct

    def struct_ptr(self):
        self.struct()
        return self._struct_ptr


@dataclass
class SearchResult:
    hits: np.ndarray       # HIT_DTYPE, sorted by (ia, ib)
    stats: dict

    @property
    def ia(self):
        return self.hits["ia"]

    @property
    def ib(self):
        return self.hits["ib"]


class _Workspace:
    """Per-device scratch (counters) and a growable hit buffer, reused across calls."""

    _per_thread = threading.local()

    @classmethod
    def get(cls, device: int):
        cache = getattr(cls._per_thread, "cache", None)
        if cache is None:
            cache = cls._per_thread.cache = {}
        if device not in cache:
            cache[device] = cls(device)
        return cache[device]

    def __init__(self, device: int):
        t = torch()
        self.device = device
        self.ws = t.empty(1 << 16, dtype=t.uint8, device=t.device("cuda", device))
        self.hits = None
        self.cand_cap = _lib.DEFAULT_CAND_CAP

    def hit_buffer(self, cap: int):
        t = torch()
        if self.hits is None or self.hits.numel() < cap * 5:
            self.hits = t.empty(max(cap, 1) * 5, dtype=t.float64, device=t.device("cuda", self.device))
        return self.hits

    def workspace(self, nbytes: int):
        t = torch()
        if self.ws.numel() < nbytes:
            self.ws = t.empty(nbytes, dtype=t.uint8, device=t.device("cuda", self.device))
        return self.ws

    def task_buffer(self, cap: int):
        t = torch()
        if getattr(self, "tasks", None) is None or self.tasks.numel() < cap:
            self.tasks = t.empty(max(cap, 1), dtype=t.int32, device=t.device("cuda", self.device))
        return self.tasks


def _grow_for(rc, stats_list, cap, cand_cap):
    """After MCX_E_CAPACITY: the new (hit cap, candidate cap) from the exact counts."""
    hits = sum(int(st.n_hits) for st in stats_list)
    cands = sum(int(st.n_aabb_pass) for st in stats_list)
    if cands > cand_cap:
        cand_cap = cands + 1024
    if hits > cap:
        cap = hits + 1024
    return cap, cand_cap


def search_device(A: DeviceMesh, B: DeviceMesh, *, mode: int = _lib.MODE_BRUTE, a_range=None,
                  shard=(0, 1), cap: int = 1 << 16, timing: bool = False, stream=None, task=None,
                  sort: bool = True, pipeline: int = _lib.PIPE_TRIANGLE,
                  orient: int = _lib.ORIENT_LARGER_A) -> SearchResult:
    """Run one search call on A.device; grows the hit / candidate buffers and reruns on overflow.
    ``orient`` (default: the larger mesh is blocked / sharded) never changes the results."""
    t = torch()
    if A.device != B.device:
        raise ConfigError("A and B must live on the same device")
    L = _lib.load()
    W = _Workspace.get(A.device)
    a0, a1 = (0, 0) if a_range is None else (int(a_range[0]), int(a_range[1]))
    As, Bs = A.struct(), B.struct()
    st = _lib.Stats()
    cand_cap = W.cand_cap
    with t.cuda.device(A.device):
        s = stream or t.cuda.current_stream(A.device)
        for _attempt in range(4):
            opts = _lib.Opts(A.device, s.cuda_stream, a0, a1, int(shard[0]), int(shard[1]), int(mode), int(timing),
                             None, 0, int(pipeline), cand_cap, int(orient))
            ws = W.workspace(L.mcx_workspace_bytes(As, Bs, opts))
            opts.workspace, opts.workspace_bytes = ws.data_ptr(), ws.numel()
            buf = W.hit_buffer(cap)
            cap_eff = buf.numel() // 5
            rc = L.mcx_search(As, Bs, opts, buf.data_ptr(), cap_eff, st)
            if rc == _lib.MCX_E_CAPACITY:
                cap, cand_cap = _grow_for(rc, [st], cap_eff, cand_cap)
                W.cand_cap = max(W.cand_cap, cand_cap)
                continue
            _lib.check(rc, "mcx_search", task=task)
            break
        else:
            raise CapacityError("hit / candidate buffer overflow persisted after regrowing", required=int(st.n_hits),
                                task=task)
        n = int(st.n_hits)
        raw = buf[: n * 5].cpu().numpy() if n else np.zeros(0)
    hits = raw.view(HIT_DTYPE).copy() if n else np.zeros(0, HIT_DTYPE)
    if sort and n:
        hits = hits[np.lexsort((hits["ib"], hits["ia"]))]
    return SearchResult(hits=hits, stats=st.as_dict())


def search_batch(pairs, *, mode: int = _lib.MODE_BRUTE, shard=(0, 1), cap: int = 1 << 16, timing: bool = False,
                 stream=None, task_ids=None, pipeline: int = _lib.PIPE_TRIANGLE, orient: int = _lib.ORIENT_LARGER_A):
    """Many (A, B) DeviceMesh searches in one launch per kernel (mcx_search_batch).

    ``pairs``: list of (A, B) or (A, B, (a_begin, a_end)).  Returns one
    SearchResult per task, hits sorted by (ia, ib).  ``task_ids`` (optional, one per
    pair) tags errors with the failing layer pair.
    """
    t = torch()
    if not pairs:
        return []
    dev = pairs[0][0].device
    for p in pairs:
        if p[0].device != dev or p[1].device != dev:
            raise ConfigError("all meshes of a batch must live on one device")
    L = _lib.load()
    W = _Workspace.get(dev)
    n = len(pairs)
    tasks = (_lib.Task * n)()
    for k, p in enumerate(pairs):  # mesh structs are cached on the DeviceMesh (kept alive by it)
        t_k = tasks[k]
        t_k.A, t_k.B = p[0].struct_ptr(), p[1].struct_ptr()
        if len(p) > 2:
            t_k.a_begin, t_k.a_end = int(p[2][0]), int(p[2][1])
    stats = (_lib.Stats * n)()
    cand_cap = W.cand_cap
    with t.cuda.device(dev):
        s = stream or t.cuda.current_stream(dev)
        for _attempt in range(4):
            opts = _lib.Opts(dev, s.cuda_stream, 0, 0, int(shard[0]), int(shard[1]), int(mode), int(timing), None, 0,
                             int(pipeline), cand_cap, int(orient))
            ws = W.workspace(L.mcx_batch_workspace_bytes(tasks, n, opts))
            opts.workspace, opts.workspace_bytes = ws.data_ptr(), ws.numel()
            buf = W.hit_buffer(cap)
            cap_eff = buf.numel() // 5
            tb = W.task_buffer(cap_eff)
            rc = L.mcx_search_batch(tasks, n, opts, buf.data_ptr(), tb.data_ptr(), cap_eff, stats)
            if rc == _lib.MCX_E_CAPACITY:
                cap, cand_cap = _grow_for(rc, list(stats), cap_eff, cand_cap)
                W.cand_cap = max(W.cand_cap, cand_cap)
                continue
            if rc != _lib.MCX_OK:
                _raise_for_task(rc, "mcx_search_batch", pairs, stats, task_ids)
            break
        else:
            raise CapacityError("hit / candidate buffer overflow persisted after regrowing",
                                required=sum(int(x.n_hits) for x in stats), task=task_ids)
        total = sum(int(stats[k].n_hits) for k in range(n))
        hits = buf[: total * 5].cpu().numpy().view(HIT_DTYPE).copy() if total else np.zeros(0, HIT_DTYPE)
        owner = tb[:total].cpu().numpy() if total else np.zeros(0, np.int32)
    # one sort by (task, ia, ib), then split at the task boundaries (O(hits log hits), not O(tasks x hits))
    order = np.lexsort((hits["ib"], hits["ia"], owner))
    hits, owner = hits[order], owner[order]
    cuts = np.searchsorted(owner, np.arange(n + 1))
    return [SearchResult(hits=hits[cuts[k]:cuts[k + 1]].copy(), stats=stats[k].as_dict()) for k in range(n)]


def _raise_for_task(rc, what, pairs, stats, task_ids):
    """A failed batch names the layer pair it failed on when that is knowable: a
    non-finite mesh is found from the per-mesh status flags."""
    if rc == _lib.MCX_E_ARG and task_ids is not None:
        for k, p in enumerate(pairs):
            if int(p[0].status.item()) or int(p[1].status.item()):
                _lib.check(rc, what, task=task_ids[k])
    _lib.check(rc, what, task=task_ids)


def ctypes_pointer(x):
    import ctypes
    return ctypes.pointer(x)


def _merge(results) -> SearchResult:
    hits = np.concatenate([r.hits for r in results]) if results else np.zeros(0, HIT_DTYPE)
    hits = hits[np.lexsort((hits["ib"], hits["ia"]))]
    stats = {}
    for r in results:
        for k, v in r.stats.items():
            stats[k] = stats.get(k, 0) + v
    if results:
        stats["kernel_ms"] = max(r.stats["kernel_ms"] for r in results)
    return SearchResult(hits=hits, stats=stats)


_SIDE_STREAMS: dict = {}
_POOLS: dict = {}
_POOLS_LOCK = threading.Lock()


def _side_stream(device: int):
    """One persistent side stream per (thread, device): a fresh stream per call would
    defeat the caching allocator (its blocks are cached per stream).  Multi-GPU calls
    run on the per-device worker threads (_device_pool), so the set stays bounded."""
    key = (threading.get_ident(), device)
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = torch().cuda.Stream(device)
    return _SIDE_STREAMS[key]


def _device_pool(device: int) -> ThreadPoolExecutor:
    """One persistent worker thread per GPU: per-thread workspaces and side streams are
    created once per device instead of once per call."""
    with _POOLS_LOCK:
        if device not in _POOLS:
            _POOLS[device] = ThreadPoolExecutor(max_workers=1, thread_name_prefix=f"mcx-gpu{device}")
        return _POOLS[device]


def run_on_devices(fn, devices):
    """fn(rank) for every rank, each on its device's worker thread (ctypes releases the
    GIL, so the GPUs run concurrently); re-raises the first error."""
    if len(devices) == 1:
        return [fn(0)]
    futs = [_device_pool(d).submit(fn, r) for r, d in enumerate(devices)]
    return [f.result() for f in futs]


def search_one(coords_a, coords_b, *, device: int = 0, mode: int = _lib.MODE_BRUTE, shard=(0, 1),
               timing: bool = False, task=None, stream=None, pipeline: int = _lib.PIPE_TRIANGLE,
               orient: int = _lib.ORIENT_LARGER_A) -> SearchResult:
    """Host grids → hits on one device: B is uploaded and packed on a side stream so
    its H2D overlaps A's packing; then one search call.  Pinned CPU tensors give
    asynchronous copies."""
    t = torch()
    with t.cuda.device(device):
        main = stream or t.cuda.current_stream(device)
        side = _side_stream(device)
        side.wait_stream(main)
        Bm = DeviceMesh(coords_b, device, stream=side)
        ready = side.record_event()
        Am = DeviceMesh(coords_a, device, stream=main)
        main.wait_event(ready)
        return search_device(Am, Bm, mode=mode, shard=shard, timing=timing, stream=main, task=task,
                             pipeline=pipeline, orient=orient)


def search(coords_a, coords_b, *, devices=(0,), mode: int = _lib.MODE_BRUTE, timing: bool = False,
           task=None, pipeline: int = _lib.PIPE_TRIANGLE, orient: int = _lib.ORIENT_LARGER_A) -> SearchResult:
    """Host-to-host triangle search: upload, pack, search (sharded over ``devices``,
    one persistent host thread per GPU; the larger mesh is the sharded one), gather, sort."""
    devices = list(devices)
    if not devices:
        raise ConfigError("devices must be non-empty")
    for d in devices:
        _require_cuda(d)
    G = len(devices)
    results = run_on_devices(lambda r: search_one(coords_a, coords_b, device=devices[r], mode=mode, shard=(r, G),
                                                  timing=timing, task=task, pipeline=pipeline, orient=orient), devices)
    return _merge(results)


def pair_candidates_device(coords_a, coords_b, device: int = 0, cap: int = 1 << 16, task=None) -> np.ndarray:
    """Sorted u64 quad-pair gids surviving ¬aabb_reject ∧ ¬moller_reject, brute force."""
    t = torch()
    _require_cuda(device)
    L = _lib.load()
    dev = t.device("cuda", device)
    with t.cuda.device(device):
        ca = t.from_numpy(np.ascontiguousarray(coords_a, dtype=np.float64)).to(dev)
        cb = t.from_numpy(np.ascontiguousarray(coords_b, dtype=np.float64)).to(dev)
        _, MA, NA = ca.shape
        _, MB, NB = cb.shape
        nq = NA * (MA - 1) + NB * (MB - 1)
        s = t.cuda.current_stream(device)
        st = _lib.Stats()
        n_cand = 1 << 16
        for _ in range(4):
            # include/mcx.h: 1024 + 64·quads + 16 per quad-AABB survivor
            ws = t.empty(1024 + 64 * nq + 16 * n_cand, dtype=t.uint8, device=dev)
            gids = t.empty(max(cap, 1), dtype=t.int64, device=dev)
            rc = L.mcx_pair_candidates(ca.data_ptr(), NA, MA, cb.data_ptr(), NB, MB, device, s.cuda_stream,
                                       ws.data_ptr(), ws.numel(), gids.data_ptr(), cap, st)
            if rc == _lib.MCX_E_CAPACITY:
                n_cand = max(n_cand, int(st.n_aabb_pass) + 1024)
                cap = max(cap, int(st.n_hits) + 1024)
                continue
            _lib.check(rc, "mcx_pair_candidates", task=task)
            break
        else:
            raise CapacityError("candidate buffer overflow persisted after regrowing", required=int(st.n_hits),
                                task=task)
        n = int(st.n_hits)
        out = gids[:n].cpu().numpy().view(np.uint64)
    return np.sort(out)


def record_fields_device(coords_a, s_a, coords_b, s_b, hits: np.ndarray, device: int = 0):
    """gid / point / params of every hit computed on the device (mcx_records)."""
    t = torch()
    n = len(hits)
    if n == 0:
        return np.zeros(0, np.uint64), np.zeros((0, 4)), np.zeros((0, 4))
    _require_cuda(device)
    L = _lib.load()
    dev = t.device("cuda", device)
    with t.cuda.device(device):
        ca = t.as_tensor(np.ascontiguousarray(coords_a, dtype=np.float64)).to(dev)
        _, MA, NA = ca.shape
        _, MB, NB = np.asarray(coords_b).shape
        sa = t.as_tensor(np.ascontiguousarray(s_a, dtype=np.float64)).to(dev)
        sb = t.as_tensor(np.ascontiguousarray(s_b, dtype=np.float64)).to(dev)
        h = t.from_numpy(np.ascontiguousarray(hits).view(np.uint8)).to(dev)
        gid = t.empty(n, dtype=t.int64, device=dev)
        pts = t.empty((n, 4), dtype=t.float64, device=dev)
        par = t.empty((n, 4), dtype=t.float64, device=dev)
        s = t.cuda.current_stream(device)
        rc = L.mcx_records(h.data_ptr(), n, ca.data_ptr(), NA, MA, sa.data_ptr(), NB, MB, sb.data_ptr(),
                           gid.data_ptr(), pts.data_ptr(), par.data_ptr(), device, s.cuda_stream)
        _lib.check(rc, "mcx_records")
        return gid.cpu().numpy().view(np.uint64), pts.cpu().numpy(), par.cpu().numpy()


def pair_candidates_mesh(A: DeviceMesh, B: DeviceMesh, *, shard=(0, 1), cap: int = 1 << 16, stream=None,
                         task=None, timing: bool = False):
    """SPEC-literal quad-pair candidates from packed meshes with exact culling
    (mcx_pair_candidates_mesh).  Returns (sorted u64 gids, stats)."""
    t = torch()
    if A.device != B.device:
        raise ConfigError("A and B must live on the same device")
    L = _lib.load()
    W = _Workspace.get(A.device)
    As, Bs = A.struct(), B.struct()
    st = _lib.Stats()
    dev = t.device("cuda", A.device)
    cand_cap = W.cand_cap
    with t.cuda.device(A.device):
        s = stream or t.cuda.current_stream(A.device)
        for _ in range(4):
            opts = _lib.Opts(A.device, s.cuda_stream, 0, 0, int(shard[0]), int(shard[1]), _lib.MODE_CULL, int(timing),
                             None, 0, _lib.PIPE_TRIANGLE, cand_cap, _lib.ORIENT_AS_GIVEN)
            ws = W.workspace(L.mcx_pair_candidates_mesh_workspace_bytes(As, Bs, opts))
            opts.workspace, opts.workspace_bytes = ws.data_ptr(), ws.numel()
            gids = t.empty(max(cap, 1), dtype=t.int64, device=dev)
            rc = L.mcx_pair_candidates_mesh(As, Bs, opts, gids.data_ptr(), cap, st)
            if rc == _lib.MCX_E_CAPACITY:
                cap, cand_cap = _grow_for(rc, [st], cap, cand_cap)
                W.cand_cap = max(W.cand_cap, cand_cap)
                continue
            _lib.check(rc, "mcx_pair_candidates_mesh", task=task)
            break
        else:
            raise CapacityError("candidate buffer overflow persisted after regrowing", required=int(st.n_hits),
                                task=task)
        n = int(st.n_hits)
        return np.sort(gids[:n].cpu().numpy().view(np.uint64)), st.as_dict()


def ctypes_u64():
    import ctypes
    return ctypes.c_uint64(0)


# ------------------------------------------------------------ multi-process helpers
def shard_ranges(n_tri: int, rank: int, world: int, a_block: int | None = None):
    """A-triangle ranges owned by ``rank`` under the kernel's cyclic block sharding
    (block b of ``mcx_a_block()`` triangles → rank b mod world)."""
    if not (0 <= rank < world):
        raise ConfigError(f"rank {rank} outside world of {world}")
    if a_block is None:
        a_block = int(_lib.load().mcx_a_block())
    nblk = (n_tri + a_block - 1) // a_block
    return [(b * a_block, min((b + 1) * a_block, n_tri)) for b in range(rank, nblk, world)]


def gather_hits(hits: np.ndarray, dst: int = 0, group=None):
    """Gather every rank's (small) hit list to ``dst`` over torch.distributed and
    return the merged, (iA, iB)-sorted list there (None on other ranks).  This is
    result collection after the independent shard searches, not a data-path
    collective; it works over gloo (CPU tests) and nccl."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    objs = [None] * world if rank == dst else None
    dist.gather_object(np.ascontiguousarray(hits).tobytes(), objs, dst=dst, group=group)
    if rank != dst:
        return None
    merged = np.concatenate([np.frombuffer(b, dtype=HIT_DTYPE) for b in objs]) if objs else np.zeros(0, HIT_DTYPE)
    return merged[np.lexsort((merged["ib"], merged["ia"]))]
