"""ctypes binding of the C ABI in include/mcx.h (libmcx.so, built in-tree).

There is no fallback: if the library is missing or fails to load, every entry
point raises ``BackendError`` ("the product path must fail loudly").  ctypes
releases the GIL during foreign calls, so one host thread per GPU runs its
search concurrently.
"""
from __future__ import annotations

import ctypes
import os
import threading

from .errors import BackendError, CapacityError

HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("MCX_LIB") or os.path.join(HERE, "libmcx.so")  # MCX_LIB: A/B builds (tools)

ABI_VERSION = 3  # include/mcx.h MCX_ABI_VERSION
MCX_OK, MCX_E_CAPACITY, MCX_E_CUDA, MCX_E_ARG = 0, 1, 2, 3
MODE_BRUTE, MODE_CULL, MODE_PREFILTER = 0, 1, 2
MODE_NAMES = {"brute": MODE_BRUTE, "cull": MODE_CULL, "prefilter": MODE_PREFILTER}
PIPE_TRIANGLE, PIPE_SPEC = 0, 1
PIPELINE_NAMES = {"triangle": PIPE_TRIANGLE, "spec": PIPE_SPEC}
ORDER_NATURAL, ORDER_TILED = 0, 1
BOX_STRIDE = 8
GROUP, TILE, BLOCK = 32, 512, 1024
DEFAULT_CAND_CAP = 1 << 20
ORIENT_AS_GIVEN, ORIENT_LARGER_A = 0, 1

EXPORTS = ("mcx_a_block", "mcx_workspace_bytes", "mcx_batch_workspace_bytes", "mcx_pack", "mcx_levels",
           "mcx_search", "mcx_search_batch", "mcx_pair_candidates", "mcx_pair_candidates_mesh",
           "mcx_pair_candidates_mesh_workspace_bytes", "mcx_records", "mcx_context_create",
           "mcx_context_destroy", "mcx_mesh_load", "mcx_mesh_free", "mcx_mesh_view", "mcx_grid_load",
           "mcx_mesh_view_columns", "mcx_intersect",
           "mcx_find_intersections", "mcx_find_intersections_strided", "mcx_finish_hits", "mcx_format_g17", "mcx_last_error", "mcx_version")


class MeshDev(ctypes.Structure):
    _fields_ = [("n_tri", ctypes.c_uint64), ("coords", ctypes.c_void_p), ("N", ctypes.c_uint32),
                ("M", ctypes.c_uint32), ("box", ctypes.c_void_p), ("perm", ctypes.c_void_p),
                ("gbox", ctypes.c_void_p), ("tbox", ctypes.c_void_p), ("bbox", ctypes.c_void_p),
                ("status", ctypes.c_void_p), ("plane_rows", ctypes.c_uint32), ("reserved", ctypes.c_uint32)]


class Task(ctypes.Structure):
    _fields_ = [("A", ctypes.POINTER(MeshDev)), ("B", ctypes.POINTER(MeshDev)), ("a_begin", ctypes.c_uint64),
                ("a_end", ctypes.c_uint64)]


class Hit(ctypes.Structure):
    _fields_ = [("ia", ctypes.c_uint32), ("ib", ctypes.c_uint32), ("s", ctypes.c_double),
                ("t", ctypes.c_double), ("a", ctypes.c_double), ("b", ctypes.c_double)]


class Stats(ctypes.Structure):
    _fields_ = [("n_pairs", ctypes.c_uint64), ("n_tested", ctypes.c_uint64), ("n_aabb_pass", ctypes.c_uint64),
                ("n_singular", ctypes.c_uint64), ("n_hits", ctypes.c_uint64), ("kernel_ms", ctypes.c_double),
                ("n_exact_tests", ctypes.c_uint64), ("n_candidates", ctypes.c_uint64)]

    def as_dict(self):
        return {k: getattr(self, k) for k, _ in self._fields_}


class Opts(ctypes.Structure):
    _fields_ = [("device", ctypes.c_int), ("stream", ctypes.c_void_p), ("a_begin", ctypes.c_uint64),
                ("a_end", ctypes.c_uint64), ("shard_index", ctypes.c_uint32), ("shard_count", ctypes.c_uint32),
                ("mode", ctypes.c_int), ("timing", ctypes.c_int), ("workspace", ctypes.c_void_p),
                ("workspace_bytes", ctypes.c_uint64), ("pipeline", ctypes.c_int), ("cand_cap", ctypes.c_uint64),
                ("orient", ctypes.c_int)]


class Record(ctypes.Structure):  # mcx_record, 128 bytes
    _fields_ = [("gid", ctypes.c_uint64), ("ia", ctypes.c_uint32), ("ib", ctypes.c_uint32),
                ("point", ctypes.c_double * 4), ("bary", ctypes.c_double * 4), ("params", ctypes.c_double * 4),
                ("task", ctypes.c_uint32), ("pad", ctypes.c_uint32 * 3)]


class Layer(ctypes.Structure):
    _fields_ = [("n1", ctypes.c_int32), ("sign1", ctypes.c_int32), ("n2", ctypes.c_int32), ("sign2", ctypes.c_int32)]


class Job(ctypes.Structure):
    _fields_ = [("A", ctypes.c_void_p), ("B", ctypes.c_void_p), ("layer", Layer)]


class FindOpts(ctypes.Structure):
    _fields_ = [("mode", ctypes.c_int), ("pipeline", ctypes.c_int), ("dedup", ctypes.c_int), ("text", ctypes.c_int),
                ("shard_index", ctypes.c_uint32), ("shard_count", ctypes.c_uint32), ("orient", ctypes.c_int)]


assert ctypes.sizeof(Hit) == 40
assert ctypes.sizeof(Record) == 128

_lib = None
_load_lock = threading.Lock()


def load():
    """Load libmcx.so (raises BackendError if absent — no CPU fallback).  Thread-safe:
    the per-GPU worker threads of device.search may race to the first call."""
    global _lib
    if _lib is not None:
        return _lib
    with _load_lock:
        if _lib is None:
            _lib = _load()
    return _lib


def _load():
    if not os.path.exists(LIB_PATH):
        raise BackendError(f"CUDA backend library not built: {LIB_PATH} (run __graft_entry__.build())")
    try:
        L = ctypes.CDLL(LIB_PATH)
    except OSError as exc:
        raise BackendError(f"cannot load {LIB_PATH}: {exc}") from None
    u32, u64, i32, vp = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int, ctypes.c_void_p
    P = ctypes.POINTER
    L.mcx_a_block.restype = u32
    L.mcx_a_block.argtypes = []
    L.mcx_workspace_bytes.restype = u64
    L.mcx_workspace_bytes.argtypes = [P(MeshDev), P(MeshDev), P(Opts)]
    L.mcx_batch_workspace_bytes.restype = u64
    L.mcx_batch_workspace_bytes.argtypes = [P(Task), u32, P(Opts)]
    L.mcx_search_batch.restype = i32
    L.mcx_search_batch.argtypes = [P(Task), u32, P(Opts), vp, vp, u64, P(Stats)]
    L.mcx_pack.restype = i32
    L.mcx_pack.argtypes = [vp, u32, u32, i32, vp, vp, vp, vp, vp, vp, i32, vp]
    L.mcx_levels.restype = i32
    L.mcx_levels.argtypes = [vp, u64, vp, vp, vp, i32, vp]
    L.mcx_search.restype = i32
    L.mcx_search.argtypes = [P(MeshDev), P(MeshDev), P(Opts), vp, u64, P(Stats)]
    L.mcx_pair_candidates.restype = i32
    L.mcx_pair_candidates.argtypes = [vp, u32, u32, vp, u32, u32, i32, vp, vp, u64, vp, u64, P(Stats)]
    L.mcx_pair_candidates_mesh.restype = i32
    L.mcx_pair_candidates_mesh.argtypes = [P(MeshDev), P(MeshDev), P(Opts), vp, u64, P(Stats)]
    L.mcx_pair_candidates_mesh_workspace_bytes.restype = u64
    L.mcx_pair_candidates_mesh_workspace_bytes.argtypes = [P(MeshDev), P(MeshDev), P(Opts)]
    L.mcx_records.restype = i32
    L.mcx_records.argtypes = [vp, u64, vp, u32, u32, vp, u32, u32, vp, vp, vp, vp, i32, vp]
    L.mcx_context_create.restype = i32
    L.mcx_context_create.argtypes = [i32, P(vp)]
    L.mcx_context_destroy.restype = i32
    L.mcx_context_destroy.argtypes = [vp]
    L.mcx_mesh_load.restype = i32
    L.mcx_mesh_load.argtypes = [vp, vp, u32, u32, vp, P(vp)]
    L.mcx_mesh_free.restype = i32
    L.mcx_mesh_free.argtypes = [vp]
    L.mcx_mesh_view.restype = P(MeshDev)
    L.mcx_mesh_view.argtypes = [vp]
    L.mcx_grid_load.restype = i32
    L.mcx_grid_load.argtypes = [vp, vp, u32, u32, vp, P(vp)]
    L.mcx_mesh_view_columns.restype = i32
    L.mcx_mesh_view_columns.argtypes = [vp, vp, u32, u32, P(vp)]
    cp = ctypes.c_char_p
    L.mcx_intersect.restype = i32
    L.mcx_intersect.argtypes = [vp, P(Job), u32, P(FindOpts), P(P(Record)), P(u64), P(vp), P(u64), P(Stats)]
    L.mcx_find_intersections.restype = i32
    L.mcx_find_intersections.argtypes = [vp, vp, u32, u32, vp, vp, u32, u32, vp, Layer, P(FindOpts), P(P(Record)),
                                         P(u64), P(vp), P(u64), P(Stats)]
    L.mcx_find_intersections_strided.restype = i32
    L.mcx_find_intersections_strided.argtypes = [vp, vp, u32, u32, u64, vp, vp, u32, u32, u64, vp, Layer, P(FindOpts),
                                                 P(P(Record)), P(u64), P(vp), P(u64), P(Stats)]
    L.mcx_finish_hits.restype = i32
    L.mcx_finish_hits.argtypes = [vp, vp, u64, vp, vp, Layer, P(FindOpts), P(P(Record)), P(u64), P(vp), P(u64)]
    L.mcx_format_g17.restype = i32
    L.mcx_format_g17.argtypes = [ctypes.c_double, cp]
    L.mcx_last_error.restype = ctypes.c_char_p
    L.mcx_last_error.argtypes = []
    L.mcx_version.restype = i32
    L.mcx_version.argtypes = []
    if L.mcx_version() != ABI_VERSION:
        raise BackendError(f"{LIB_PATH} has ABI version {L.mcx_version()}, expected {ABI_VERSION}: rebuild it")
    return L


def last_error() -> str:
    return load().mcx_last_error().decode(errors="replace")


def check(rc: int, what: str, task=None, required: int = 0):
    if rc == MCX_OK:
        return
    msg = f"{what}: {last_error()}"
    if rc == MCX_E_CAPACITY:
        raise CapacityError(msg, required=required, task=task)
    raise BackendError(msg, task=task, status=rc)
