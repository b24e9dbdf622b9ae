"""Host-to-host runtime: ctypes wrapper of the context API of include/mcx.h.

One ``Context`` per (host thread, GPU) owns the device's streams, a stream-ordered
memory pool and pinned result buffers (csrc/mcx_runtime.cu).  A call hands the
library HOST grids and gets back host records (and the records text): upload, pack,
search, record fields, the (gid, τ_A, τ_B) sort, the 1e-9 dedup and the "%.17g"
text all run on the device.

Records come back as a NumPy structured array with the layout of ``mcx_record``.
"""
from __future__ import annotations

import ctypes
import threading

import numpy as np

from . import _lib
from .errors import BackendError, ConfigError

RECORD_DTYPE = np.dtype([("gid", "<u8"), ("ia", "<u4"), ("ib", "<u4"), ("point", "<f8", (4,)), ("bary", "<f8", (4,)),
                         ("params", "<f8", (4,)), ("task", "<u4"), ("pad", "<u4", (3,))])
assert RECORD_DTYPE.itemsize == ctypes.sizeof(_lib.Record)


def _sign(s) -> int:
    if s in ("+", 1, "1", "+1"):
        return 1
    if s in ("-", -1, "-1"):
        return -1
    raise ConfigError(f"layer sign must be '+' or '-', got {s!r}")


def layer_struct(layer) -> _lib.Layer:
    n1, s1, n2, s2 = layer
    return _lib.Layer(int(n1), _sign(s1), int(n2), _sign(s2))


def _host_f64(a):
    """(pointer, keep-alive) of a C-contiguous float64 host array (NumPy or CPU torch tensor;
    a pinned torch tensor gives an asynchronous copy)."""
    if isinstance(a, np.ndarray):
        a = np.ascontiguousarray(a, dtype=np.float64)
        return a.ctypes.data, a
    import torch
    if isinstance(a, torch.Tensor):
        if a.device.type != "cpu" or a.dtype != torch.float64 or not a.is_contiguous():
            raise ConfigError("expected a contiguous float64 CPU tensor")
        return a.data_ptr(), a
    a = np.ascontiguousarray(np.asarray(a, dtype=np.float64))
    return a.ctypes.data, a


def _host_grid(a):
    """(pointer, keep-alive, plane stride in doubles) of a (4, M, N) float64 host grid.  A
    NumPy view whose rows are contiguous within each plane (a half-layer's column range of
    a larger mesh) is passed in place with its plane stride (0: dense)."""
    if (isinstance(a, np.ndarray) and a.dtype == np.float64 and a.ndim == 3 and a.shape[0] == 4
            and a.strides[2] == 8 and a.strides[1] == 8 * a.shape[2] and a.strides[0] % 8 == 0
            and a.strides[0] >= 8 * a.shape[1] * a.shape[2]):
        plane = a.strides[0] // 8
        return a.ctypes.data, a, (0 if plane == a.shape[1] * a.shape[2] else plane)
    p, keep = _host_f64(a)
    return p, keep, 0


def find_opts(mode: int, pipeline: int, dedup: bool, text: bool, shard=(0, 1),
              orient: int = _lib.ORIENT_LARGER_A) -> _lib.FindOpts:
    return _lib.FindOpts(int(mode), int(pipeline), int(bool(dedup)), int(bool(text)), int(shard[0]), int(shard[1]),
                         int(orient))


class Mesh:
    """A half-layer resident on a context's device (mcx_mesh_load), a whole mesh uploaded
    unpacked (``grid=True``, mcx_grid_load) as the source of half-layer views, or a view
    (``Context.view``: columns [c0, c1] of a resident grid, packed in place, no upload)."""

    @classmethod
    def _from_handle(cls, ctx, handle, N, M, parent=None):
        m = cls.__new__(cls)
        m.ctx, m.handle, m.N, m.M, m.parent = ctx, handle, N, M, parent
        return m

    def __init__(self, ctx: "Context", coords, s_values, grid: bool = False):
        self.parent = None
        c = np.asarray(coords) if isinstance(coords, np.ndarray) else coords
        if c.ndim != 3 or c.shape[0] != 4:
            raise ConfigError(f"coords must have shape (4, M, N), got {tuple(c.shape)}")
        _, M, N = (int(v) for v in c.shape)
        if M < 2:
            raise ConfigError("a half-layer needs >= 2 columns (SPEC.md:473)")
        sv = np.ascontiguousarray(s_values, dtype=np.float64)
        if sv.shape != (M,):
            raise ConfigError(f"s_values must have length M = {M}")
        p, keep = _host_f64(c)
        h = ctypes.c_void_p()
        fn = _lib.load().mcx_grid_load if grid else _lib.load().mcx_mesh_load
        _lib.check(fn(ctx.handle, p, N, M, sv.ctypes.data, ctypes.byref(h)), "mcx_grid_load" if grid else "mcx_mesh_load")
        self.ctx, self.handle, self.N, self.M = ctx, h, N, M
        del keep

    def free(self):
        if self.handle:
            _lib.load().mcx_mesh_free(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.free()
        except Exception:
            pass


class Context:
    """One device's runtime context (mcx_context_create)."""

    def __init__(self, device: int = 0):
        h = ctypes.c_void_p()
        _lib.check(_lib.load().mcx_context_create(int(device), ctypes.byref(h)), "mcx_context_create")
        self.device, self.handle = int(device), h

    def close(self):
        if self.handle:
            _lib.load().mcx_context_destroy(self.handle)
            self.handle = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def mesh(self, coords, s_values) -> Mesh:
        return Mesh(self, coords, s_values)

    def grid(self, coords, s_values) -> Mesh:
        """A whole mesh uploaded once, unpacked: the source of ``view`` half-layers."""
        return Mesh(self, coords, s_values, grid=True)

    def view(self, parent: Mesh, c0: int, c1: int) -> Mesh:
        """Columns [c0, c1] of a resident grid as a packed half-layer, without copying
        (a half-layer is a contiguous column range of its mesh)."""
        h = ctypes.c_void_p()
        _lib.check(_lib.load().mcx_mesh_view_columns(self.handle, parent.handle, int(c0), int(c1), ctypes.byref(h)),
                   "mcx_mesh_view_columns")
        return Mesh._from_handle(self, h, parent.N, int(c1) - int(c0) + 1, parent=parent)

    @staticmethod
    def _out(recp, n, textp, tlen):
        n = int(n.value)
        addr = ctypes.cast(recp, ctypes.c_void_p).value
        recs = np.zeros(0, RECORD_DTYPE) if n == 0 else \
            np.frombuffer(ctypes.string_at(addr, n * RECORD_DTYPE.itemsize), dtype=RECORD_DTYPE).copy()
        text = ctypes.string_at(textp.value, int(tlen.value)) if textp.value else b""
        return recs, text

    def find(self, coords_a, s_a, coords_b, s_b, layer=(0, "+", 0, "+"), *, mode=_lib.MODE_CULL,
             pipeline=_lib.PIPE_SPEC, dedup=True, text=False, task=None, shard=(0, 1),
             orient=_lib.ORIENT_LARGER_A):
        """mcx_find_intersections: host grids → (records, text bytes, stats dict).  ``shard``
        restricts the search to a cyclic share of the (larger) mesh's blocks, as one rank
        of a multi-GPU job (the records are then that shard's)."""
        pa, ka, plane_a = _host_grid(coords_a)
        pb, kb, plane_b = _host_grid(coords_b)
        sa = np.ascontiguousarray(s_a, dtype=np.float64)
        sb = np.ascontiguousarray(s_b, dtype=np.float64)
        _, MA, NA = (int(v) for v in ka.shape)
        _, MB, NB = (int(v) for v in kb.shape)
        if MA < 2 or MB < 2:
            raise ConfigError("a half-layer needs >= 2 columns (SPEC.md:473)")
        if sa.shape != (MA,) or sb.shape != (MB,):
            raise ConfigError("s_values must have one entry per column")
        fo = find_opts(mode, pipeline, dedup, text, shard, orient)
        recp, n, textp, tlen, st = ctypes.POINTER(_lib.Record)(), ctypes.c_uint64(), ctypes.c_void_p(), \
            ctypes.c_uint64(), _lib.Stats()
        rc = _lib.load().mcx_find_intersections_strided(self.handle, pa, NA, MA, plane_a, sa.ctypes.data, pb, NB, MB,
                                                        plane_b, sb.ctypes.data, layer_struct(layer),
                                                        ctypes.byref(fo), ctypes.byref(recp), ctypes.byref(n),
                                                        ctypes.byref(textp), ctypes.byref(tlen), ctypes.byref(st))
        _lib.check(rc, "mcx_find_intersections", task=task)
        recs, txt = self._out(recp, n, textp, tlen)
        return recs, txt, st.as_dict()

    def intersect(self, jobs, *, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC, dedup=True, text=False,
                  task_ids=None):
        """mcx_intersect over resident meshes: jobs = [(Mesh A, Mesh B, layer)] →
        (records of all jobs in (job, gid, τ_A, τ_B) order, text bytes, [stats dict])."""
        n = len(jobs)
        if n == 0:
            return np.zeros(0, RECORD_DTYPE), b"", []
        arr = (_lib.Job * n)()
        for k, (A, B, layer) in enumerate(jobs):
            if A.ctx is not self or B.ctx is not self:
                raise ConfigError("job meshes must be loaded on this context")
            arr[k].A, arr[k].B, arr[k].layer = A.handle, B.handle, layer_struct(layer)
        fo = find_opts(mode, pipeline, dedup, text)
        recp, cnt, textp, tlen = ctypes.POINTER(_lib.Record)(), ctypes.c_uint64(), ctypes.c_void_p(), ctypes.c_uint64()
        stats = (_lib.Stats * n)()
        rc = _lib.load().mcx_intersect(self.handle, arr, n, ctypes.byref(fo), ctypes.byref(recp), ctypes.byref(cnt),
                                       ctypes.byref(textp), ctypes.byref(tlen), stats)
        if rc != _lib.MCX_OK:
            import re
            m = re.match(r"job (\d+) ", _lib.last_error())
            task = task_ids[int(m.group(1))] if (m and task_ids is not None) else task_ids
            _lib.check(rc, "mcx_intersect", task=task)
        recs, txt = self._out(recp, cnt, textp, tlen)
        return recs, txt, [s.as_dict() for s in stats]

    def finish_hits(self, hits, A: Mesh, B: Mesh, layer=(0, "+", 0, "+"), *, dedup=True, text=False):
        """mcx_finish_hits: records for a host hit list (e.g. gathered from several GPUs)."""
        h = np.ascontiguousarray(hits)
        fo = find_opts(_lib.MODE_CULL, _lib.PIPE_TRIANGLE, dedup, text)
        recp, cnt, textp, tlen = ctypes.POINTER(_lib.Record)(), ctypes.c_uint64(), ctypes.c_void_p(), ctypes.c_uint64()
        rc = _lib.load().mcx_finish_hits(self.handle, h.ctypes.data if len(h) else None, len(h), A.handle, B.handle,
                                         layer_struct(layer), ctypes.byref(fo), ctypes.byref(recp), ctypes.byref(cnt),
                                         ctypes.byref(textp), ctypes.byref(tlen))
        _lib.check(rc, "mcx_finish_hits")
        return self._out(recp, cnt, textp, tlen)


_local = threading.local()


def context(device: int = 0) -> Context:
    """This thread's context for ``device`` (created on first use; contexts are not shared
    between threads)."""
    cache = getattr(_local, "ctx", None)
    if cache is None:
        cache = _local.ctx = {}
    if device not in cache:
        import torch
        if not torch.cuda.is_available():
            raise BackendError("backend='cuda' requires a CUDA device (none visible)")
        if device >= torch.cuda.device_count():
            raise ConfigError(f"device {device} not present ({torch.cuda.device_count()} visible)")
        cache[device] = Context(device)
    return cache[device]
