"""ctypes binding of O2 (oracle/mcx_oracle.c).  TEST INFRASTRUCTURE ONLY.

See oracle/canonical.py for what the oracle restates and why its arithmetic is
canonical.  ``build()`` compiles the library with oracle/Makefile.
"""
from __future__ import annotations

import ctypes
import os
import subprocess

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "liboracle_mcx.so")
_lib = None


def build(force: bool = False) -> str:
    if force or not os.path.exists(LIB_PATH) or (
            os.path.getmtime(LIB_PATH) < os.path.getmtime(os.path.join(_HERE, "mcx_oracle.c"))):
        subprocess.run(["make", "-s", "-C", _HERE] + (["-B"] if force else []), check=True)
    return LIB_PATH


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(LIB_PATH):
            build()
        L = ctypes.CDLL(LIB_PATH)
        u32, u64, i32 = ctypes.c_uint32, ctypes.c_uint64, ctypes.c_int
        vp = ctypes.c_void_p
        L.mcxo_search.argtypes = [vp, u32, u32, vp, u32, u32, u64, u64, i32, i32, vp, vp, vp, u64, vp, vp]
        L.mcxo_search.restype = i32
        L.mcxo_pack.argtypes = [vp, u32, u32, vp, vp]
        L.mcxo_pack.restype = i32
        L.mcxo_max_threads.restype = i32
        L.mcxo_pack_new.argtypes = [vp, u32, u32]
        L.mcxo_pack_new.restype = vp
        L.mcxo_pack_free.argtypes = [vp]
        L.mcxo_pack_free.restype = None
        L.mcxo_search_packed.argtypes = [vp, vp, u64, u64, i32, i32, vp, vp, vp, u64, vp, vp]
        L.mcxo_search_packed.restype = i32
        _lib = L
    return _lib


def max_threads() -> int:
    return int(lib().mcxo_max_threads())


def pack(coords):
    c = np.ascontiguousarray(coords, dtype=np.float64)
    _, M, N = c.shape
    n = 2 * N * (M - 1)
    box = np.empty((n, 8))
    geo = np.empty((n, 19))
    lib().mcxo_pack(c.ctypes.data, N, M, box.ctypes.data, geo.ctypes.data)
    return box, geo


def search(coords_a, coords_b, a_range=None, sweep=True, threads=0, cap=1 << 20):
    """Same return dict as canonical.search (hits sorted by (ia, ib))."""
    A = np.ascontiguousarray(coords_a, dtype=np.float64)
    B = np.ascontiguousarray(coords_b, dtype=np.float64)
    _, MA, NA = A.shape
    _, MB, NB = B.shape
    nA = 2 * NA * (MA - 1)
    a0, a1 = (0, nA) if a_range is None else a_range
    while True:
        ia = np.empty(cap, np.uint32)
        ib = np.empty(cap, np.uint32)
        st = np.empty((cap, 4))
        nh = np.zeros(1, np.uint64)
        stats = np.zeros(3, np.uint64)
        rc = lib().mcxo_search(A.ctypes.data, NA, MA, B.ctypes.data, NB, MB, a0, a1, int(sweep), threads,
                               ia.ctypes.data, ib.ctypes.data, st.ctypes.data, cap,
                               nh.ctypes.data, stats.ctypes.data)
        n = int(nh[0])
        if rc == 0:
            break
        cap = n
    ia, ib, st = ia[:n], ib[:n], st[:n]
    order = np.lexsort((ib, ia))
    ia, ib, st = ia[order], ib[order], st[order]
    return {"ia": ia, "ib": ib, "s": st[:, 0].copy(), "t": st[:, 1].copy(), "a": st[:, 2].copy(),
            "b": st[:, 3].copy(), "n_pairs": int(stats[0]), "n_aabb_pass": int(stats[1]),
            "n_singular": int(stats[2])}


class Packed:
    """A mesh packed once by the C oracle (for timed searches that exclude packing)."""

    def __init__(self, coords):
        c = np.ascontiguousarray(coords, dtype=np.float64)
        _, M, N = c.shape
        self.n = 2 * N * (M - 1)
        self.handle = lib().mcxo_pack_new(c.ctypes.data, N, M)

    def __del__(self):
        if getattr(self, "handle", None):
            lib().mcxo_pack_free(self.handle)
            self.handle = None


def search_packed(PA: Packed, PB: Packed, a_range=None, sweep=False, threads=0, cap=1 << 20):
    """search() on pre-packed meshes; returns (hit count, n_pairs)."""
    a0, a1 = (0, PA.n) if a_range is None else a_range
    while True:
        ia = np.empty(cap, np.uint32)
        ib = np.empty(cap, np.uint32)
        st = np.empty((cap, 4))
        nh = np.zeros(1, np.uint64)
        stats = np.zeros(3, np.uint64)
        rc = lib().mcxo_search_packed(PA.handle, PB.handle, a0, a1, int(sweep), threads, ia.ctypes.data,
                                      ib.ctypes.data, st.ctypes.data, cap, nh.ctypes.data, stats.ctypes.data)
        if rc == 0:
            return int(nh[0]), int(stats[0])
        cap = int(nh[0])


def survivors(coords_a, coords_b, threads=0, cap=1 << 20):
    """Every AABB-pass pair (ia, ib) of A x B (exact x-sweep), sorted by (ia, ib)."""
    PA, PB = Packed(coords_a), Packed(coords_b)
    L = lib()
    L.mcxo_survivors.argtypes = [ctypes.c_void_p] * 2 + [ctypes.c_int] + [ctypes.c_void_p] * 3 + \
        [ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    L.mcxo_survivors.restype = ctypes.c_int
    while True:
        ia = np.empty(cap, np.uint32)
        ib = np.empty(cap, np.uint32)
        st = np.empty((cap, 4))
        n = np.zeros(1, np.uint64)
        stats = np.zeros(3, np.uint64)
        rc = L.mcxo_survivors(PA.handle, PB.handle, threads, ia.ctypes.data, ib.ctypes.data, st.ctypes.data, cap,
                              n.ctypes.data, stats.ctypes.data)
        if rc == 0:
            k = int(n[0])
            order = np.lexsort((ib[:k], ia[:k]))
            return ia[:k][order].astype(np.int64), ib[:k][order].astype(np.int64)
        cap = int(n[0])


def spec_search(coords_a, coords_b, threads=0, cap=1 << 20):
    """O3 (the SPEC-literal serial backend, oracle/serial.py) in C: quad AABB x-sweep,
    Moller, 4 canonical precise tests per candidate.  Same dict as search(), plus
    n_quad_pairs / n_quad_aabb_pass / n_candidates."""
    A = np.ascontiguousarray(coords_a, dtype=np.float64)
    B = np.ascontiguousarray(coords_b, dtype=np.float64)
    _, MA, NA = A.shape
    _, MB, NB = B.shape
    L = lib()
    L.mcxo_spec_search.argtypes = [ctypes.c_void_p, ctypes.c_uint32, ctypes.c_uint32, ctypes.c_void_p,
                                   ctypes.c_uint32, ctypes.c_uint32, ctypes.c_int, ctypes.c_void_p, ctypes.c_void_p,
                                   ctypes.c_void_p, ctypes.c_uint64, ctypes.c_void_p, ctypes.c_void_p]
    L.mcxo_spec_search.restype = ctypes.c_int
    while True:
        ia = np.empty(cap, np.uint32)
        ib = np.empty(cap, np.uint32)
        st = np.empty((cap, 4))
        nh = np.zeros(1, np.uint64)
        stats = np.zeros(4, np.uint64)
        rc = L.mcxo_spec_search(A.ctypes.data, NA, MA, B.ctypes.data, NB, MB, threads, ia.ctypes.data,
                                ib.ctypes.data, st.ctypes.data, cap, nh.ctypes.data, stats.ctypes.data)
        n = int(nh[0])
        if rc == 0:
            break
        cap = n
    ia, ib, st = ia[:n], ib[:n], st[:n]
    order = np.lexsort((ib, ia))
    ia, ib, st = ia[order], ib[order], st[order]
    return {"ia": ia, "ib": ib, "s": st[:, 0].copy(), "t": st[:, 1].copy(), "a": st[:, 2].copy(),
            "b": st[:, 3].copy(), "n_quad_pairs": int(stats[0]), "n_quad_aabb_pass": int(stats[1]),
            "n_candidates": int(stats[2]), "n_singular": int(stats[3])}
