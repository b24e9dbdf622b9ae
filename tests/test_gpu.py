"""GPU parity tests (B200): the CUDA path through the C ABI against the oracles.

Bar: the sorted (iA, iB) hit set is bit-exact, and so are
s, t, a, b (identical canonical IEEE op sequence), and the AABB-pass / singular
counters equal the oracle's.  At full sizes parity uses the C oracle's exact
sweep-and-prune (same predicate, only skips x-disjoint pairs) plus
size-independent properties: partition / shard / variant invariance.
"""
import os
import sys

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

from oracle import canonical as O  # noqa: E402
from oracle import serial as S  # noqa: E402
from paper_2109_14814_b200 import _lib, device as D, isect  # noqa: E402
from paper_2109_14814_b200.mesh import config_pair, manifold_like  # noqa: E402

GOLD = os.path.join(os.path.dirname(__file__), "golden")


def _bits(x):
    return np.asarray(x, dtype=np.float64).view(np.uint64)


def assert_same_hits(ref, hits, stats=None):
    assert np.array_equal(ref["ia"], hits["ia"]), "iA differ"
    assert np.array_equal(ref["ib"], hits["ib"]), "iB differ"
    for f in "stab":
        assert np.array_equal(_bits(ref[f]), _bits(hits[f])), f"{f} not bit-exact"
    if stats is not None:
        assert stats["n_aabb_pass"] == ref["n_aabb_pass"]
        assert stats["n_singular"] == ref["n_singular"]
        assert stats["n_hits"] == len(ref["ia"])


@pytest.fixture(scope="module")
def c1():
    z = np.load(os.path.join(GOLD, "c1.npz"))
    return z


@pytest.mark.parametrize("order", [_lib.ORDER_TILED, _lib.ORDER_NATURAL])
@pytest.mark.parametrize("shape", [(64, 64), (37, 23), (5, 2), (1024, 3), (33, 50), (48, 40), (96, 33), (256, 129), (66, 35)])
def test_device_pack_bit_exact(order, shape):
    """Every packed box equals the oracle's box of its original triangle (tiled order:
    via perm, which must be a bijection), and the level boxes written by the same
    pass are the exact unions of their records."""
    A, _ = manifold_like(shape[0], shape[1], 1)
    m = D.DeviceMesh(A, 0, order=order)
    pk = O.pack(A)
    box = m.box.cpu().numpy()
    if order == _lib.ORDER_TILED:
        perm = m.perm.cpu().numpy().astype(np.int64)
        assert np.array_equal(np.sort(perm), np.arange(m.n_tri))
    else:
        perm = np.arange(m.n_tri)
    pk = O.take(pk, perm)
    assert np.array_equal(_bits(box[:, :4]), _bits(pk["lo"])) and np.array_equal(_bits(box[:, 4:]), _bits(pk["hi"]))
    n = m.n_tri
    for lev, size in ((m.gbox, 32), (m.tbox, 512), (m.bbox, 1024)):
        lb = lev.cpu().numpy()
        assert len(lb) == -(-n // size)
        for g in range(len(lb)):
            seg = box[g * size:(g + 1) * size]
            assert np.array_equal(lb[g, :4], seg[:, :4].min(0)) and np.array_equal(lb[g, 4:], seg[:, 4:].max(0))


def test_tiled_pack_requires_perm():
    A, _ = manifold_like(16, 5, 1)
    t = D.torch()
    c = t.from_numpy(A).cuda()
    box = t.empty((2 * 16 * 4, 8), dtype=t.float64, device="cuda")
    rc = _lib.load().mcx_pack(c.data_ptr(), 16, 5, _lib.ORDER_TILED, box.data_ptr(), None, None, None, None, None, 0,
                              None)
    assert rc == _lib.MCX_E_ARG and "perm" in _lib.last_error()


def test_tiled_order_is_spatially_compact():
    A, _ = manifold_like(256, 129, 1)
    tiled, nat = D.DeviceMesh(A, 0), D.DeviceMesh(A, 0, order=_lib.ORDER_NATURAL)
    ext = lambda m: float(np.mean(np.max(m.gbox.cpu().numpy()[:, 4:] - m.gbox.cpu().numpy()[:, :4], axis=1)))
    assert ext(tiled) < 0.5 * ext(nat)


def test_golden_c1(c1):
    r = D.search(c1["A"], c1["B"])
    ref = {"ia": c1["ia"], "ib": c1["ib"], "n_aabb_pass": int(c1["n_aabb_pass"]),
           "n_singular": int(c1["n_singular"])}
    for f in "stab":
        ref[f] = c1[f].view(np.float64)
    assert_same_hits(ref, r.hits, r.stats)


def test_golden_c4ii_exact_lattice():
    z = np.load(os.path.join(GOLD, "c4ii.npz"))
    r = D.search(z["A"], z["B"])
    ref = {"ia": z["ia"], "ib": z["ib"], "n_aabb_pass": int(z["n_aabb_pass"]), "n_singular": int(z["n_singular"])}
    for f in "stab":
        ref[f] = z[f].view(np.float64)
    assert_same_hits(ref, r.hits, r.stats)


MODES = [_lib.MODE_BRUTE, _lib.MODE_CULL, _lib.MODE_PREFILTER]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", ["C1", "C4i", "C4ii", "C4iii"])
def test_parity_small(name, mode, oracle_lib):
    A, _, B, _ = config_pair(name)
    ref = oracle_lib.search(A, B, sweep=True)
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)
    if mode == _lib.MODE_CULL:
        assert r.stats["n_tested"] < r.stats["n_pairs"]
    else:
        assert r.stats["n_tested"] == r.stats["n_pairs"]
    assert r.stats["n_pairs"] == A.shape[2] * (A.shape[1] - 1) * 2 * B.shape[2] * (B.shape[1] - 1) * 2


@pytest.mark.parametrize("mode", [_lib.MODE_BRUTE, _lib.MODE_PREFILTER])
@pytest.mark.parametrize("variant", [str(v) for v in range(53)])
def test_kernel_variants_identical(variant, mode, monkeypatch, oracle_lib):
    monkeypatch.setenv("MCX_VARIANT", variant)
    A, _, B, _ = config_pair("C4i")
    ref = oracle_lib.search(A, B, sweep=True)
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)


@pytest.mark.parametrize("mode", MODES)
def test_parity_c2_full(mode, oracle_lib):
    """C2 (256×256 each, 1.7e10 pairs) against the C oracle's exact sweep-and-prune."""
    A, _, B, _ = config_pair("C2")
    ref = oracle_lib.search(A, B, sweep=True)
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("scale", [8, 4])
def test_parity_c5_reduced(scale, mode, oracle_lib):
    """C5 at 1/8 and 1/4 scale: unbalanced meshes, hits concentrated in A's first columns."""
    A, _, B, _ = config_pair(f"C5/{scale}")
    ref = oracle_lib.search(A, B, sweep=True)
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)
    assert len(ref["ia"]) > 50


@pytest.fixture(scope="module")
def c3_ref(oracle_lib):
    A, _, B, _ = config_pair("C3")
    return A, B, oracle_lib.search(A, B, sweep=True)


@pytest.mark.slow
@pytest.mark.parametrize("mode", MODES)
def test_parity_c3_vs_oracle(mode, c3_ref):
    """C3 (1M x 1M triangles, 1.095e12 pairs: the north-star size) in every mode against
    the C oracle's exact sweep-and-prune: hit set, solution bits and counters."""
    A, B, ref = c3_ref
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)
    assert r.stats["n_pairs"] == 1046528 * 1046528


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("G", [2, 3, 8])
def test_shard_invariance(G, mode, oracle_lib):
    """Cyclic A-block sharding (the multi-GPU partition) never changes the hit set."""
    A, _, B, _ = config_pair("C4i")
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    full = D.search_device(Am, Bm, mode=mode)
    parts = [D.search_device(Am, Bm, shard=(g, G), mode=mode) for g in range(G)]
    merged = D._merge(parts)
    assert np.array_equal(merged.hits, full.hits)
    assert sum(p.stats["n_pairs"] for p in parts) == full.stats["n_pairs"]
    assert merged.stats["n_aabb_pass"] == full.stats["n_aabb_pass"]


@pytest.mark.parametrize("mode", MODES)
def test_a_range_partition(mode):
    A, _, B, _ = config_pair("C4iii")
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    full = D.search_device(Am, Bm, mode=mode)
    cuts = [0, 1000, 4097, 4100, Am.n_tri]
    parts = [D.search_device(Am, Bm, a_range=(a, b), mode=mode) for a, b in zip(cuts[:-1], cuts[1:])]
    assert np.array_equal(D._merge(parts).hits, full.hits)
    assert sum(p.stats["n_pairs"] for p in parts) == full.stats["n_pairs"]


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("name", ["C4i", "C5/8"])
def test_natural_and_tiled_orders_agree(name, mode):
    A, _, B, _ = config_pair(name)
    r1 = D.search_device(D.DeviceMesh(A, 0, order=_lib.ORDER_NATURAL), D.DeviceMesh(B, 0, order=_lib.ORDER_NATURAL),
                         mode=mode)
    r2 = D.search_device(D.DeviceMesh(A, 0), D.DeviceMesh(B, 0), mode=_lib.MODE_BRUTE)
    assert np.array_equal(r1.hits, r2.hits)
    r3 = D.search_device(D.DeviceMesh(A, 0, order=_lib.ORDER_NATURAL), D.DeviceMesh(B, 0), mode=mode)  # mixed
    assert np.array_equal(r3.hits, r2.hits)


@pytest.mark.parametrize("mode", MODES)
def test_capacity_regrow(mode):
    A, _, B, _ = config_pair("C4ii")  # 54k hits
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    D._Workspace.get(0).hits = None
    r_small = D.search_device(Am, Bm, cap=7, mode=mode)
    D._Workspace.get(0).hits = None
    r_big = D.search_device(Am, Bm, cap=1 << 20, mode=mode)
    assert len(r_small.hits) == len(r_big.hits) == 54201
    assert np.array_equal(r_small.hits, r_big.hits)


def test_swap_roles_symmetry():
    """Searching B against A gives the transposed hit set (roles of s,t and a,b swap)."""
    A, _, B, _ = config_pair("C1")
    r1 = D.search(A, B)
    r2 = D.search(B, A)
    k1 = set(zip(r1.hits["ia"].tolist(), r1.hits["ib"].tolist()))
    k2 = set(zip(r2.hits["ib"].tolist(), r2.hits["ia"].tolist()))
    assert k1 == k2


@pytest.mark.parametrize("mode", MODES)
def test_disjoint_and_degenerate_inputs(mode):
    A, _ = manifold_like(32, 9, 1)
    far = A + 100.0
    r = D.search(A, far, mode=mode)
    assert len(r.hits) == 0 and r.stats["n_aabb_pass"] == 0
    if mode == _lib.MODE_CULL:
        assert r.stats["n_tested"] == 0
    # ragged sizes: A smaller than one block, B smaller than one tile, N odd
    for na, ma, nb, mb in ((5, 2, 7, 3), (37, 23, 19, 41), (1, 2, 3, 2)):
        A2, _ = manifold_like(na, ma, 3)
        B2, _ = manifold_like(nb, mb, 3)
        ref = O.search(A2, B2)
        assert_same_hits(ref, D.search(A2, B2, mode=mode).hits)
    # flat/degenerate triangles (all vertices identical) are singular, never hits
    Z = np.zeros((4, 3, 4))
    rz = D.search(Z, Z, mode=mode)
    assert len(rz.hits) == 0 and rz.stats["n_singular"] == rz.stats["n_aabb_pass"] == (2 * 4 * 2) ** 2


def test_multi_device_api_single_gpu():
    """The in-process multi-GPU path (one host thread per device) with the same device twice."""
    A, _, B, _ = config_pair("C4i")
    r1 = D.search(A, B, devices=(0,))
    r2 = D.search(A, B, devices=(0, 0))
    assert np.array_equal(r1.hits, r2.hits)


def test_find_intersections_records(oracle_lib):
    A, sa, B, sb = config_pair("C1")
    recs = isect.find_intersections(A, B, pipeline="triangle")
    ref = O.search(A, B)
    hits = np.zeros(len(ref["ia"]), dtype=D.HIT_DTYPE)
    for k in ("ia", "ib", "s", "t", "a", "b"):
        hits[k] = ref[k]
    want = isect.hits_to_records(A, sa, B, sb, hits)
    assert [r.to_line() for r in recs] == [w.to_line() for w in want]


@pytest.mark.parametrize("mode", ["brute", "cull"])
@pytest.mark.parametrize("name", ["C1", "C4i", "C4iii", "C5/8"])
def test_pair_candidates_spec_literal(name, mode):
    A, _, B, _ = config_pair(name)
    want, _ = S.pair_candidates(A, B)
    got = isect.pair_candidates(A, B, mode=mode)
    assert np.array_equal(got, want.astype(np.uint64))


@pytest.mark.parametrize("mode", ["brute", "cull"])
def test_pair_candidates_small_exhaustive(mode):
    A, _ = manifold_like(16, 5, 11)
    B = A + np.array([0.0, 0.0, 0.02, 0.0])[:, None, None]
    want, _ = S.pair_candidates(A, B)
    assert np.array_equal(isect.pair_candidates(A, B, mode=mode), want.astype(np.uint64))


def test_pair_candidates_mesh_counters_and_shards():
    A, _, B, _ = config_pair("C4i")
    want, n_pass = S.pair_candidates(A, B)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    gids, st = D.pair_candidates_mesh(Am, Bm)
    assert np.array_equal(gids, want.astype(np.uint64))
    assert st["n_aabb_pass"] == n_pass and st["n_hits"] == len(want)
    assert st["n_pairs"] == (Am.n_tri // 2) * (Bm.n_tri // 2) and st["n_tested"] < st["n_pairs"]
    parts = [D.pair_candidates_mesh(Am, Bm, shard=(g, 3))[0] for g in range(3)]
    assert np.array_equal(np.sort(np.concatenate(parts)), gids)
    nat = D.pair_candidates_mesh(D.DeviceMesh(A, 0, order=_lib.ORDER_NATURAL),
                                 D.DeviceMesh(B, 0, order=_lib.ORDER_NATURAL))[0]
    assert np.array_equal(nat, gids)


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("bad", [np.nan, np.inf, -np.inf])
def test_non_finite_rejected(mode, bad):
    """NaN/Inf inputs are flagged by the device packer and fail the search loudly."""
    from paper_2109_14814_b200.errors import BackendError
    A, _ = manifold_like(40, 7, 1)
    B = A.copy()
    B[2, 3, 17] = bad
    with pytest.raises(BackendError, match="non-finite"):
        D.search(A, B, mode=mode)
    with pytest.raises(BackendError, match="non-finite"):
        D.search_batch([(D.DeviceMesh(A, 0), D.DeviceMesh(A, 0)), (D.DeviceMesh(B, 0), D.DeviceMesh(A, 0))], mode=mode)
    assert len(D.search(A, A, mode=mode).hits) > 0  # finite inputs still fine


def test_bad_args_fail_loudly():
    A, _, B, _ = config_pair("C1")
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    with pytest.raises(Exception):
        D.search_device(Am, Bm, shard=(3, 2))
    with pytest.raises(Exception):
        D.search_device(Am, Bm, a_range=(10, 10 ** 9))


# ------------------------------------------------------------ batched tasks (one launch)
@pytest.mark.parametrize("mode", MODES)
def test_search_batch_equals_individual(mode):
    meshes = {}
    for name in ("C1", "C4i", "C4iii", "C5/8"):
        A, _, B, _ = config_pair(name)
        meshes[name] = (D.DeviceMesh(A, 0), D.DeviceMesh(B, 0))
    pairs = [(*meshes["C1"],), (*meshes["C4i"],), (*meshes["C4iii"],), (*meshes["C5/8"],),
             (*meshes["C4i"], (1000, 5000)), (meshes["C1"][1], meshes["C4i"][0]),
             (meshes["C4i"][0], meshes["C4i"][0])]  # meshes shared across tasks and within one
    batch = D.search_batch(pairs, mode=mode)
    for p, r in zip(pairs, batch):
        single = D.search_device(p[0], p[1], mode=mode, a_range=p[2] if len(p) > 2 else None)
        assert np.array_equal(r.hits, single.hits)
        for k in ("n_pairs", "n_aabb_pass", "n_singular", "n_hits"):
            assert r.stats[k] == single.stats[k], k


@pytest.mark.parametrize("mode", MODES)
def test_search_batch_sharded(mode):
    A, _, B, _ = config_pair("C4i")
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    full = D.search_batch([(Am, Bm), (Bm, Am)], mode=mode)
    parts = [D.search_batch([(Am, Bm), (Bm, Am)], mode=mode, shard=(g, 3)) for g in range(3)]
    for t in range(2):
        assert np.array_equal(D._merge([p[t] for p in parts]).hits, full[t].hits)


@pytest.mark.parametrize("mode,pipeline", [("cull", "triangle"), ("brute", "triangle"), ("prefilter", "triangle"),
                                           ("cull", "spec")])
def test_search_plan_matches_oracle(mode, pipeline):
    from paper_2109_14814_b200 import layers
    from paper_2109_14814_b200.mesh import half_layer, layered_mesh
    u = layered_mesh(96, "unstable", 3, 1.6, 0.1, 1)
    s = layered_mesh(96, "stable", 3, 1 / 1.6, 0.1, 2)
    plan = layers.enumerate_layer_pairs(u, s, 3)
    res = layers.search_plan(u, s, plan, mode=mode, pipeline=pipeline, text=True)
    recs, stats = res
    want = []
    for (n1, s1, n2, s2), tof in zip(plan.tasks, plan.tof):
        hu, hs = half_layer(u, n1, 1 if s1 == "+" else -1), half_layer(s, n2, 1 if s2 == "+" else -1)
        ca, cb = np.ascontiguousarray(hu.coords), np.ascontiguousarray(hs.coords)
        ref = O.search(ca, cb) if pipeline == "triangle" else S.find_intersections(ca, cb)
        h = np.zeros(len(ref["ia"]), dtype=D.HIT_DTYPE)
        for k in ("ia", "ib", "s", "t", "a", "b"):
            h[k] = ref[k]
        want.extend(isect.hits_to_records(ca, hu.s_values, cb, hs.s_values, h, layer=(n1, s1, n2, s2), tof=tof))
    assert [r.to_line() for r in recs] == [w.to_line() for w in want]
    assert res.text == "".join(w.to_line() + "\n" for w in want).encode()  # device-formatted records file
    assert len(stats) == len(plan) == 20
    assert len(want) > 0


def test_cli_intersect(tmp_path):
    from paper_2109_14814_b200 import cli, layers
    from paper_2109_14814_b200.mesh import layered_mesh, write_mesh
    u = layered_mesh(64, "unstable", 2, 1.6, 0.1, 1)
    s = layered_mesh(64, "stable", 2, 1 / 1.6, 0.1, 2)
    write_mesh(tmp_path / "u.mnf", u)
    write_mesh(tmp_path / "s.mnf", s)
    assert cli.main(["layers", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                     "--nmax", "2", "--plan", str(tmp_path / "plan.txt")]) == 0
    assert cli.main(["intersect", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                     "--plan", str(tmp_path / "plan.txt"), "--backend", "cuda", "--out", str(tmp_path / "rec.txt"),
                     "--manifest", str(tmp_path / "m.json")]) == 0
    recs, _ = layers.search_plan(u, s, layers.read_plan(tmp_path / "plan.txt"))
    assert (tmp_path / "rec.txt").read_text().splitlines() == [r.to_line() for r in recs]
    tri = None
    for mode in ("cull", "brute", "prefilter"):  # every search mode writes the identical records file
        out = tmp_path / f"rec_{mode}.txt"
        assert cli.main(["intersect", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                         "--plan", str(tmp_path / "plan.txt"), "--backend", "cuda", "--out", str(out),
                         "--mode", mode, "--pipeline", "triangle", "--devices", "0,0"]) == 0
        tri = tri or out.read_text()
        assert out.read_text() == tri
    assert cli.main(["intersect", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                     "--plan", str(tmp_path / "plan.txt"), "--backend", "cuda", "--out", str(tmp_path / "x"),
                     "--mode", "brute"]) == 2  # the spec pipeline runs on the culling kernels only


# ------------------------------------------------------------ device record fields (§8(f) row 4)
@pytest.mark.parametrize("name", ["C1", "C4ii", "C5/4"])
def test_device_record_fields_bit_exact(name):
    A, sa, B, sb = config_pair(name)
    hits = D.search(A, B, mode=_lib.MODE_CULL).hits
    g1, p1, q1 = isect.record_fields(A, sa, B, sb, hits)
    g2, p2, q2 = isect.record_fields_device(A, sa, B, sb, hits)
    assert np.array_equal(g1, g2)
    assert np.array_equal(_bits(p1), _bits(p2)) and np.array_equal(_bits(q1), _bits(q2))


def test_find_intersections_device_records_equal_host():
    A, sa, B, sb = config_pair("C4ii")
    recs = isect.find_intersections(A, B, pipeline="triangle")
    hits = D.search(A, B).hits
    want = isect.hits_to_records(A, np.linspace(-1.0, 1.0, A.shape[1]), B, np.linspace(-1.0, 1.0, B.shape[1]), hits)
    assert [r.to_line() for r in recs] == [w.to_line() for w in want]
    assert len(recs) < len(hits)  # shared-vertex hits collapse under the 1e-9 dedup


@pytest.mark.slow
@pytest.mark.parametrize("kind", ["same", "tangent"])
def test_parity_stress_large(kind, oracle_lib):
    """Near-degenerate stress pairs at 512×257 (262k triangles each): B = A (shared edges and
    vertices everywhere) and near-tangent sheets — every mode vs the C oracle's exact sweep."""
    from paper_2109_14814_b200.mesh import stress_pair
    A, B, _ = stress_pair(kind, N=512, M=257, seed=3)
    ref = oracle_lib.search(A, B, sweep=True, cap=1 << 22)
    for mode in MODES:
        r = D.search(A, B, mode=mode)
        assert_same_hits(ref, r.hits, r.stats)
    assert len(ref["ia"]) > (1000 if kind == "same" else 100)


def test_c_host_example():
    """The C ABI driven from plain C (no Python/torch): brute, cull and prefilter agree."""
    import subprocess
    d = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "tools", "c_example")
    subprocess.run(["make", "-s", "-C", d], check=True)
    out = subprocess.run([os.path.join(d, "mcx_example"), "200", "65"], capture_output=True, text=True, check=True)
    rows = [ln.split() for ln in out.stdout.strip().splitlines()]
    assert [r[0] for r in rows] == ["brute", "cull", "prefilter", "runtime"]
    brute, cull, pre, rt = rows
    assert rt[1] == rt[2] == brute[5] and rt[4] == brute[6]  # host runtime: same hits, one record each
    assert int(rt[3]) > 0
    assert pre[1:7] == brute[1:7]
    assert brute[1] == cull[1]                      # logical pairs
    assert brute[2] == brute[1] and int(cull[2]) < int(cull[1])  # executed tests
    assert brute[3:7] == cull[3:7]                  # aabb pass, singular, hits, checksum
    assert int(brute[5]) > 0


@pytest.mark.parametrize("mode", MODES)
@pytest.mark.parametrize("case", ["cross5", "cross6", "adversarial"])
def test_acceptance6_exact_oracle(case, mode):
    """SPEC acceptance 6: on synthetic meshes of (N1, N2, M1, M2) = (32, 32, 9, 9) the hit set
    equals a brute-force all-pairs EXACT (fractions) precise-test oracle.  Dyadic lattice
    inputs make the exact answer well defined at touching configurations."""
    from oracle import exact as X
    from paper_2109_14814_b200.mesh import dyadic, stress_pair
    if case == "adversarial":
        A, B, _ = stress_pair("dyadic", N=32, M=9, seed=4)
    else:
        seed = int(case[-1])
        A = dyadic(manifold_like(32, 9, seed)[0])
        B = dyadic(manifold_like(32, 9, seed + 10)[0])
    pA, pB = O.pack(A), O.pack(B)
    ov = O.aabb_overlap(pA["lo"][:, None], pA["hi"][:, None], pB["lo"][None], pB["hi"][None])
    want = set()
    for a, b in zip(*np.nonzero(ov)):
        sol = X.solve_exact(pA["p"][a], pA["e1"][a], pA["e2"][a], pB["p"][b], pB["e1"][b], pB["e2"][b])
        if X.accepted(sol):
            want.add((int(a), int(b)))
    r = D.search(A, B, mode=mode)
    got = set(zip(r.hits["ia"].tolist(), r.hits["ib"].tolist()))
    assert got == want
    assert r.stats["n_aabb_pass"] == int(ov.sum())


@pytest.mark.parametrize("name", ["C1", "C2", "C4i"])
def test_prefilter_counts(name):
    """MCX_MODE_PREFILTER: every pair is tested (n_tested == n_pairs); the exact FP64 box
    test runs only on quantised passes, a superset of the exact AABB passes."""
    A, _, B, _ = config_pair(name)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    rb = D.search_device(Am, Bm, mode=_lib.MODE_BRUTE)
    rp = D.search_device(Am, Bm, mode=_lib.MODE_PREFILTER)
    assert_same_hits(rb.hits, rp.hits)
    sp = rp.stats
    assert sp["n_tested"] == sp["n_pairs"] == rb.stats["n_pairs"]
    assert sp["n_aabb_pass"] == rb.stats["n_aabb_pass"] and sp["n_singular"] == rb.stats["n_singular"]
    assert sp["n_aabb_pass"] <= sp["n_exact_tests"] < sp["n_pairs"]
    assert rb.stats["n_exact_tests"] == rb.stats["n_pairs"]


def test_prefilter_frames_exact(oracle_lib):
    """Quantisation frames that make the integer test weak or degenerate never change
    the result: a far outlier column (coarse frame), a constant coordinate (κ = 0),
    huge magnitudes (frame extent overflows to inf → κ = 0), tiny magnitudes."""
    A, _, B, _ = config_pair("C4iii")
    cases = []
    A1 = A.copy(); A1[:, -1, :] += 1.0e6  # one far column in A
    cases.append((A1, B))
    A2 = A.copy(); B2 = B.copy(); A2[3] = 0.25; B2[3] = 0.25  # py constant on both meshes
    cases.append((A2, B2))
    cases.append((A * 1.0e300, B * 1.0e300))
    A4 = A.copy(); A4[0, 0, 0] = -1.7e308; B4 = B.copy(); B4[1, 0, 0] = 1.7e308  # extent overflows
    cases.append((A4, B4))
    cases.append((A * 1.0e-300, B * 1.0e-300))
    for Ax, Bx in cases:
        ref = oracle_lib.search(Ax, Bx, sweep=True)
        r = D.search(Ax, Bx, mode=_lib.MODE_PREFILTER)
        assert_same_hits(ref, r.hits, r.stats)


@pytest.fixture(scope="module")
def c5hd(oracle_lib):
    A, _, B, _ = config_pair("C5hd")
    return A, B, oracle_lib.search(A, B, sweep=True), D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)


@pytest.mark.parametrize("mode", MODES)
def test_parity_c5hd_full(mode, c5hd):
    """configs[4] at full scale, high-hit-density variant: 4.2M × 65k triangles,
    13,226 hits clustered in A's first quarter — hit compaction under load."""
    A, B, ref, Am, Bm = c5hd
    assert len(ref["ia"]) == 13226
    assert_same_hits(ref, D.search_device(Am, Bm, mode=mode).hits)
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)


@pytest.mark.parametrize("mode", [_lib.MODE_PREFILTER, _lib.MODE_CULL])
def test_c5hd_cyclic_shards_balance_hits(mode, c5hd):
    """8 cyclic A-block shards (the 8-GPU partition, run one after another here): their
    union is the full hit set and the clustered hits spread evenly over the shards."""
    A, B, ref, Am, Bm = c5hd
    parts = [D.search_device(Am, Bm, shard=(g, 8), mode=mode).hits for g in range(8)]
    got = np.concatenate(parts)
    got = got[np.lexsort((got["ib"], got["ia"]))]
    assert_same_hits(ref, got)
    counts = np.array([len(p) for p in parts])
    assert counts.max() <= 1.5 * counts.mean(), counts


@pytest.mark.parametrize("case", range(24))
def test_random_meshes_all_modes(case, oracle_lib):
    """Randomised parity sweep: random grid shapes (ragged, odd, tiny, tall), surfaces,
    affine scalings (1e-8 .. 1e8), translations and near-coincident copies, each
    searched in all three modes against the C oracle's exact sweep."""
    rng = np.random.default_rng(1000 + case)
    na, ma = int(rng.integers(1, 160)), int(rng.integers(2, 70))
    nb, mb = int(rng.integers(1, 160)), int(rng.integers(2, 70))
    A, _ = manifold_like(na, ma, int(rng.integers(0, 50)))
    kind = case % 3
    if kind == 0:    # independent surfaces
        B, _ = manifold_like(nb, mb, int(rng.integers(0, 50)))
    elif kind == 1:  # the same surface resampled, slightly perturbed (dense contacts)
        B, _ = manifold_like(nb, mb, 7)
        A, _ = manifold_like(na, ma, 7)
        B = B + rng.normal(0, 1e-3, (4, 1, 1))
    else:            # a copy of A shifted by a fraction of a cell (many touching boxes)
        B = A + rng.normal(0, 1e-2, (4, 1, 1))
    scale = 10.0 ** rng.uniform(-8, 8)
    shift = rng.normal(0, 10, (4, 1, 1)) * scale
    A, B = A * scale + shift + 0.0, B * scale + shift + 0.0
    ref = oracle_lib.search(A, B, sweep=True)
    for mode in MODES:
        r = D.search(A, B, mode=mode)
        assert_same_hits(ref, r.hits, r.stats)


@pytest.mark.parametrize("tool", ["memcheck", "racecheck", "synccheck", "initcheck"])
def test_compute_sanitizer_clean(tool):
    """Every libmcx kernel (pack, levels, three search modes, batches, shards, the
    capacity-regrow path, pair_candidates, records) under compute-sanitizer: no errors."""
    import shutil
    import subprocess
    exe = shutil.which("compute-sanitizer") or "/usr/local/cuda/bin/compute-sanitizer"
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([exe, "--tool", tool, "--error-exitcode", "7", sys.executable,
                          os.path.join(root, "tools", "sanitize_run.py")],
                         capture_output=True, text=True, timeout=600)
    assert out.returncode == 0, out.stdout[-3000:] + out.stderr[-3000:]
    assert "sanitize workload ok" in out.stdout


@pytest.mark.slow
def test_parity_4m_x_4m_vs_oracle(oracle_lib):
    """Beyond the BASELINE sizes: 4.2M x 4.2M triangles (1.76e13 pairs) in prefilter and
    cull mode against the C oracle's exact sweep."""
    A, _ = manifold_like(2048, 1025, 1)
    B, _ = manifold_like(2048, 1025, 2)
    ref = oracle_lib.search(A, B, sweep=True)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    for mode in (_lib.MODE_PREFILTER, _lib.MODE_CULL):
        r = D.search_device(Am, Bm, mode=mode)
        assert_same_hits(ref, r.hits, r.stats)


def test_bench_json_contract():
    """bench.py (our arm) on a small config: one JSON line with the keys the driver reads."""
    import json
    import subprocess
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    out = subprocess.run([sys.executable, os.path.join(root, "bench.py"), "--config", "C2", "--steps", "3",
                          "--warmup", "3", "--no-cpu-baseline", "--no-paper", "--no-c5"],
                         capture_output=True, text=True, check=True, timeout=600, cwd=root).stdout
    lines = [ln for ln in out.strip().splitlines() if ln.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    for k in ("metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better", "scaling",
              "vs_baseline", "dtype", "data", "config", "roofline", "e2e", "clocks", "gpu_launches"):
        assert k in d, k
    assert d["steps"] == 3 and d["warmup"] == 3 and d["n_gpus"] == 1 and d["value"] > 0
    assert d["config"]["pairs_per_step"] == 130560 * 130560 and "workload" in d["config"]
    for k in ("bound", "achieved", "peak", "unit", "frac", "traffic"):
        assert k in d["roofline"], k
    assert 0 < d["roofline"]["frac"] < 1.2
    for k in ("value", "unit", "h2d_bytes_per_step", "d2h_bytes_per_step"):
        assert k in d["e2e"], k
    assert d["e2e"]["h2d_bytes_per_step"] > 0 and d["gpu_launches"] > 0
    assert d["e2e"]["h2d_floor_ms"] > 0 and d["e2e"]["records"] == 4
    assert d["e2e"]["other_modes"]["cull_spec"]["records"] == 4
    # every e2e leg's rate is pairs per step / its own per-step time (the legs run different step counts)
    for leg in (d["e2e"], *d["e2e"]["other_modes"].values()):
        assert leg["value"] == pytest.approx(d["config"]["pairs_per_step"] / (leg["ms_per_step"] * 1e-3), rel=1e-6)
    assert d["hits"] == d["cull"]["hits"] == 4


# ------------------------------------------------------------ SPEC-literal pipeline on the GPU
def _as_hits(ref):
    h = np.zeros(len(ref["ia"]), dtype=D.HIT_DTYPE)
    for k in ("ia", "ib", "s", "t", "a", "b"):
        h[k] = ref[k]
    return h


@pytest.mark.parametrize("name", ["C1", "C4i", "C4ii", "C4iii", "C5/8", "C5/4"])
def test_spec_pipeline_records_equal_serial_backend(name):
    """find_intersections(pipeline="spec") on the GPU equals the SPEC-literal serial
    backend (oracle/serial.py: quad AABB + Moller + 4 precise tests per survivor) record
    for record, text byte for byte."""
    A, sa, B, sb = config_pair(name)
    want = isect.hits_to_records(A, sa, B, sb, _as_hits(S.find_intersections(A, B)))
    from paper_2109_14814_b200 import runtime
    recs, text, st = runtime.context(0).find(A, sa, B, sb, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC, text=True)
    got = isect.records_to_objects(recs, A.shape[2], B.shape[2])
    assert [r.to_line() for r in got] == [w.to_line() for w in want]
    assert text == "".join(w.to_line() + "\n" for w in want).encode()
    gids, n_pass = S.pair_candidates(A, B)
    assert st["n_candidates"] == len(gids) and st["n_aabb_pass"] == n_pass
    assert [r.to_line() for r in isect.find_intersections(A, B)] == [w.to_line() for w in want]  # the default


def test_spec_pipeline_acceptance_set():
    """(N1, N2, M1, M2) = (32, 32, 9, 9) dyadic meshes (SPEC acceptance 6 sizes): spec pipeline
    hits equal the serial backend's, and are a subset of the exact all-pairs answer."""
    from oracle import exact as X
    from paper_2109_14814_b200.mesh import dyadic
    for seed in (5, 6):
        A = dyadic(manifold_like(32, 9, seed)[0])
        B = dyadic(manifold_like(32, 9, seed + 10)[0])
        ref = S.find_intersections(A, B)
        r = D.search(A, B, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC)
        assert_same_hits(ref, r.hits)
        pA, pB = O.pack(A), O.pack(B)
        for a, b in zip(r.hits["ia"], r.hits["ib"]):
            sol = X.solve_exact(pA["p"][a], pA["e1"][a], pA["e2"][a], pB["p"][b], pB["e1"][b], pB["e2"][b])
            assert X.accepted(sol)


# ------------------------------------------------------------ device records pipeline (§8(f) row 4)
@pytest.mark.parametrize("name", ["C1", "C4i", "C4ii", "C5/8", "self-small"])
@pytest.mark.parametrize("dedup", [True, False])
def test_runtime_records_and_text_equal_host(name, dedup):
    """Device records (fields, (gid, τ_A, τ_B) order, 1e-9 dedup) and the device-formatted
    records text equal the host path (isect.hits_to_records + to_line) byte for byte.
    C1 / C5/8 / self-small take the single-kernel path (≤ 1024 hits; self-small = a small
    mesh against itself, up to 36 hits per shared vertex, which overflows its 8-predecessor
    lists and falls back), C4i / C4ii the general one."""
    from paper_2109_14814_b200 import runtime
    if name == "self-small":
        A, sa = manifold_like(12, 6, 3)
        B, sb = A.copy(), sa
    else:
        A, sa, B, sb = config_pair(name)
    hits = D.search(A, B, mode=_lib.MODE_CULL).hits
    want = isect.hits_to_records(A, sa, B, sb, hits, layer=(3, "-", 2, "+"), dedup=dedup)
    recs, text, st = runtime.context(0).find(A, sa, B, sb, (3, "-", 2, "+"), mode=_lib.MODE_CULL,
                                             pipeline=_lib.PIPE_TRIANGLE, dedup=dedup, text=True)
    got = isect.records_to_objects(recs, A.shape[2], B.shape[2], layer=(3, "-", 2, "+"))
    assert [r.to_line() for r in got] == [w.to_line() for w in want]
    assert text == "".join(w.to_line() + "\n" for w in want).encode()
    assert st["n_hits"] == len(hits)


@pytest.mark.parametrize("name,swap", [("C5", False), ("C5/4", True), ("C5hd", False), ("C5hd", True)])
def test_runtime_stepped_search_equals_unstepped(name, swap, monkeypatch):
    """mcx_find_intersections searches a large mesh chunk by chunk during its upload
    (find_stepped): records, text and stats equal the single-batch search (MCX_NO_STEPS)
    in both pipelines, with the larger mesh passed as A or as B (oriented: the solve
    un-swaps).  Fresh contexts also take the regrow path on C5hd (2.4M box survivors >
    the default 1M candidate capacity: the stepped attempt overflows and reruns)."""
    from paper_2109_14814_b200 import runtime
    A, sa, B, sb = config_pair(name)
    if swap:
        A, sa, B, sb = B, sb, A, sa
    keys = ("n_hits", "n_aabb_pass", "n_tested", "n_pairs", "n_candidates", "n_singular")
    for pipe in (_lib.PIPE_SPEC, _lib.PIPE_TRIANGLE):
        ctx = runtime.Context(0)
        got = ctx.find(A, sa, B, sb, (1, "+", 2, "-"), pipeline=pipe, text=True)
        again = ctx.find(A, sa, B, sb, (1, "+", 2, "-"), pipeline=pipe, text=True)  # capacities now sufficient
        monkeypatch.setenv("MCX_NO_STEPS", "1")
        want = runtime.Context(0).find(A, sa, B, sb, (1, "+", 2, "-"), pipeline=pipe, text=True)
        monkeypatch.delenv("MCX_NO_STEPS")
        for g in (got, again):
            assert g[1] == want[1] and len(want[1]) > 0
            assert np.array_equal(g[0], want[0])
            assert {k: g[2][k] for k in keys} == {k: want[2][k] for k in keys}
        ctx.close()


def test_runtime_batch_and_finish_hits():
    """mcx_intersect over several resident jobs equals one find per job; mcx_finish_hits
    (host hit list, e.g. gathered from several GPUs) equals find."""
    from paper_2109_14814_b200 import runtime
    ctx = runtime.context(0)
    cfgs = [config_pair(n) for n in ("C1", "C4ii", "C5/8")]
    meshes = [(ctx.mesh(A, sa), ctx.mesh(B, sb)) for A, sa, B, sb in cfgs]
    layers_ = [(1, "+", 1, "-"), (2, "-", 1, "+"), (0, "+", 0, "+")]
    jobs = [(ma, mb, L) for (ma, mb), L in zip(meshes, layers_)]
    recs, text, stats = ctx.intersect(jobs, pipeline=_lib.PIPE_TRIANGLE, text=True)
    parts, ptext = [], b""
    for (A, sa, B, sb), L in zip(cfgs, layers_):
        r, t, _ = ctx.find(A, sa, B, sb, L, pipeline=_lib.PIPE_TRIANGLE, text=True)
        parts.append(r)
        ptext += t
    assert text == ptext
    cat = np.concatenate(parts)
    for f in ("gid", "ia", "ib"):
        assert np.array_equal(recs[f], cat[f])
    assert np.array_equal(recs["task"], np.repeat(np.arange(3), [len(p) for p in parts]))
    A, sa, B, sb = cfgs[2]
    hits = D.search(A, B, devices=(0, 0), mode=_lib.MODE_CULL).hits
    r2, t2 = ctx.finish_hits(hits, meshes[2][0], meshes[2][1], layers_[2], text=True)
    assert t2 == ctx.find(A, sa, B, sb, layers_[2], pipeline=_lib.PIPE_TRIANGLE, text=True)[1]
    for ma, mb in meshes:
        ma.free()
        mb.free()


@pytest.mark.slow
def test_runtime_dense_records_equal_host():
    """Dense cases: C5hd (13,226 hits) and a 512×257 mesh against itself (every triangle
    touches its neighbours): device records and text equal the host path."""
    from paper_2109_14814_b200 import runtime
    for name in ("C5hd", "dense-self"):
        if name == "C5hd":
            A, sa, B, sb = config_pair("C5hd")
        else:
            A, sa = manifold_like(512, 257, 3)
            B, sb = A, sa
        hits = D.search(A, B, mode=_lib.MODE_CULL).hits
        want = isect.hits_to_records(A, sa, B, sb, hits)
        recs, text, _ = runtime.context(0).find(A, sa, B, sb, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_TRIANGLE,
                                                text=True)
        assert text == "".join(w.to_line() + "\n" for w in want).encode(), name
        assert len(recs) == len(want) and len(hits) > 10000


def test_search_plan_multi_device_equals_single():
    from paper_2109_14814_b200 import layers
    from paper_2109_14814_b200.mesh import layered_mesh
    u = layered_mesh(64, "unstable", 3, 1.6, 0.1, 1)
    s = layered_mesh(64, "stable", 3, 1 / 1.6, 0.1, 2)
    plan = layers.enumerate_layer_pairs(u, s, 3, include_core=True)
    a = layers.search_plan(u, s, plan, text=True)
    b = layers.search_plan(u, s, plan, devices=(0, 0, 0), text=True)
    assert a.text == b.text and len(a.records) == len(b.records) > 0
    assert [x["layer"] for x in b.stats] == plan.tasks


def test_concurrent_host_threads_one_device():
    """Two host threads searching concurrently on one device (contexts and workspaces are
    per thread; SPEC.md:504 tasks run concurrently) get the single-thread results."""
    import threading
    A, sa, B, sb = config_pair("C4i")
    ref = D.search(A, B, mode=_lib.MODE_CULL).hits
    out = [None] * 4
    from paper_2109_14814_b200 import runtime

    def work(k):
        if k % 2:
            out[k] = D.search(A, B, mode=_lib.MODE_PREFILTER).hits
        else:
            out[k] = runtime.context(0).find(A, sa, B, sb, pipeline=_lib.PIPE_TRIANGLE, dedup=False)[0]
    th = [threading.Thread(target=work, args=(k,)) for k in range(4)]
    for t in th:
        t.start()
    for t in th:
        t.join()
    for k in range(4):
        o = out[k]
        assert np.array_equal(np.sort(o["ia"].astype(np.int64) << 32 | o["ib"]), np.sort(ref["ia"].astype(np.int64) << 32 | ref["ib"]))


def test_device_guard_preserves_current_device():
    t = D.torch()
    before = t.cuda.current_device()
    A, sa, B, sb = config_pair("C1")
    isect.find_intersections(A, B, devices=(0,))
    D.search(A, B, devices=(0,))
    assert t.cuda.current_device() == before


# ------------------------------------------------------------ SPEC.md:485 geometric oracle
@pytest.mark.parametrize("pipeline", ["spec", "triangle"])
def test_ruled_surfaces_cross_along_known_curve(pipeline):
    """Two ruled-surface meshes constructed to cross along a known curve: every returned
    point lies within one mesh-cell diameter of the analytic curve, the hits
    cover the whole curve, and the records' parameter estimates (Eqs. 28-29) agree with the
    analytic parametrisations: θ_u ≈ θ_s ≈ the point's angle, s_u ≈ px, s_s ≈ 0 (t at py = 0)."""
    from paper_2109_14814_b200.mesh import ruled_curve, ruled_pair
    A, sa, B, sb = ruled_pair()
    from paper_2109_14814_b200.mesh import HalfLayer, ManifoldMesh
    ua = HalfLayer.whole(ManifoldMesh(coords=A, s_values=sa), 1, 1)
    sbh = HalfLayer.whole(ManifoldMesh(coords=B, s_values=sb, kind="stable"), 1, -1)
    recs = isect.find_intersections(ua, sbh, pipeline=pipeline)
    assert len(recs) > 50
    pts = np.array([r.point for r in recs])
    ang = np.arctan2(pts[:, 1], pts[:, 0]) % (2 * np.pi)
    phi = np.linspace(0.0, 2 * np.pi, 400001)
    curve = ruled_curve(phi)
    cellA = np.hypot(2 * np.pi / A.shape[2], sa[1] - sa[0])
    cellB = np.hypot(2 * np.pi / B.shape[2] * 1.2, np.hypot(0.5, 1.0) * (sb[1] - sb[0]))
    cell = max(cellA, cellB)
    for p, g in zip(pts, ang):
        k = int(g / (2 * np.pi) * 400000)
        idx = np.arange(k - 4000, k + 4000) % len(phi)
        assert np.min(np.linalg.norm(curve[idx] - p, axis=1)) <= cell
    gaps = np.diff(np.sort(ang))
    assert max(gaps.max(), 2 * np.pi - ang.max() + ang.min()) <= 3 * 2 * np.pi / B.shape[2]
    par = np.array([r.params for r in recs])  # θ_u, s_u, θ_s, s_s
    wrap = lambda x: (x + np.pi) % (2 * np.pi) - np.pi
    assert np.max(np.abs(wrap(par[:, 0] - ang))) <= 2 * np.pi / A.shape[2]
    assert np.max(np.abs(wrap(par[:, 2] - ang))) <= 2 * np.pi / B.shape[2]
    assert np.max(np.abs(par[:, 1] - pts[:, 2])) <= sa[1] - sa[0]
    assert np.max(np.abs(par[:, 3])) <= sb[1] - sb[0]


# ------------------------------------------------------------ full-scale parity (C5, C5hd, C3)
@pytest.fixture(scope="module")
def c5_full(oracle_lib):
    A, sa, B, sb = config_pair("C5")
    return A, sa, B, sb, oracle_lib.search(A, B, sweep=True, cap=1 << 20)


@pytest.mark.parametrize("mode", MODES)
def test_parity_c5_full(mode, c5_full):
    """The survey-frozen configs[4] pair at full scale (A 4,194,304 x B 65,536 triangles):
    hit set, s/t/a/b bits and counters equal the C oracle's exact sweep in every mode."""
    A, _, B, _, ref = c5_full
    r = D.search(A, B, mode=mode)
    assert_same_hits(ref, r.hits, r.stats)
    assert len(ref["ia"]) == 645


@pytest.mark.parametrize("name", ["C5", "C5hd", "C3"])
def test_spec_pipeline_full_scale(name, oracle_lib):
    """SPEC-literal pipeline at full scale against the C restatement of the serial backend
    (quad AABB sweep + Moller + 4 precise tests, bit-identical to oracle/serial.py on the
    reduced configs): hits, s/t/a/b bits, quad-AABB and candidate counts, and the records
    built from them."""
    A, sa, B, sb = config_pair(name)
    ref = oracle_lib.spec_search(A, B)
    r = D.search(A, B, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC)
    assert_same_hits(ref, r.hits)
    assert r.stats["n_aabb_pass"] == ref["n_quad_aabb_pass"] and r.stats["n_candidates"] == ref["n_candidates"]
    assert r.stats["n_singular"] == ref["n_singular"] and r.stats["n_pairs"] == ref["n_quad_pairs"]
    want = isect.hits_to_records(A, sa, B, sb, _as_hits(ref))
    got = isect.find_intersections(A, B)
    assert [g.to_line() for g in got] == [w.to_line() for w in want]


# ------------------------------------------------------------ orientation
@pytest.mark.parametrize("mode", MODES)
def test_orientation_swap_bit_identical(mode, oracle_lib):
    """A small A against a large B: with MCX_ORIENT_LARGER_A the sweep blocks and shards B
    (the larger mesh) and replicates A, but the precise test still runs as (A, B), so hits,
    s/t/a/b bits and counters equal the as-given search and the oracle — unsharded and over
    3 cyclic shards of B's blocks."""
    B, _, A, _ = config_pair("C5/8")  # A: 32x17 grid, B: 256x129 grid
    ref = oracle_lib.search(A, B, sweep=True)
    Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
    for orient in (_lib.ORIENT_AS_GIVEN, _lib.ORIENT_LARGER_A):
        r = D.search_device(Am, Bm, mode=mode, orient=orient)
        assert_same_hits(ref, r.hits, r.stats)
        parts = [D.search_device(Am, Bm, mode=mode, orient=orient, shard=(g, 3)) for g in range(3)]
        assert_same_hits(ref, D._merge(parts).hits)
    spec = D.search_device(Am, Bm, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC, orient=_lib.ORIENT_AS_GIVEN)
    spec2 = D.search_device(Am, Bm, mode=_lib.MODE_CULL, pipeline=_lib.PIPE_SPEC, orient=_lib.ORIENT_LARGER_A)
    assert np.array_equal(spec.hits, spec2.hits) and spec.stats["n_candidates"] == spec2.stats["n_candidates"]


def test_prefilter_size_rule(monkeypatch):
    """By default MCX_MODE_PREFILTER runs the FP64 sweep for calls below 2^28 pairs (C1:
    6.5e7; every pair then gets the exact test) and the quantised sweep above (C2: 1.7e10,
    exact tests only on quantised passes); hits are identical either way."""
    monkeypatch.delenv("MCX_PREFILTER_MIN_PAIRS", raising=False)
    for name, quantised in (("C1", False), ("C2", True)):
        A, _, B, _ = config_pair(name)
        Am, Bm = D.DeviceMesh(A, 0), D.DeviceMesh(B, 0)
        rp = D.search_device(Am, Bm, mode=_lib.MODE_PREFILTER)
        rb = D.search_device(Am, Bm, mode=_lib.MODE_BRUTE)
        assert np.array_equal(rp.hits, rb.hits)
        assert (rp.stats["n_exact_tests"] < rp.stats["n_pairs"]) == quantised


def test_column_views_equal_copied_half_layers():
    """A half-layer as a zero-copy column view of its resident mesh (plane stride = the
    parent's M) gives exactly the records of the same columns copied to a contiguous grid —
    both pipelines, both roles, ragged ranges."""
    from paper_2109_14814_b200 import runtime
    from paper_2109_14814_b200.mesh import layered_mesh
    u = layered_mesh(96, "unstable", 3, 1.6, 0.1, 1)
    s = layered_mesh(80, "stable", 3, 1 / 1.6, 0.1, 2)
    ctx = runtime.context(0)
    gu, gs = ctx.grid(u.coords, u.s_values), ctx.grid(s.coords, s.s_values)
    for (a0, a1), (b0, b1) in (((3, 17), (0, 9)), ((20, u.M - 1), (5, s.M - 3)), ((0, 1), (s.M - 6, s.M - 1))):
        va, vb = ctx.view(gu, a0, a1), ctx.view(gs, b0, b1)
        ca, cb = np.ascontiguousarray(u.coords[:, a0:a1 + 1]), np.ascontiguousarray(s.coords[:, b0:b1 + 1])
        ma, mb = ctx.mesh(ca, u.s_values[a0:a1 + 1]), ctx.mesh(cb, s.s_values[b0:b1 + 1])
        for pipe in (_lib.PIPE_SPEC, _lib.PIPE_TRIANGLE):
            r1, t1, st1 = ctx.intersect([(va, vb, (1, "+", 2, "-")), (vb, va, (2, "-", 1, "+"))], pipeline=pipe,
                                        text=True)
            r2, t2, st2 = ctx.intersect([(ma, mb, (1, "+", 2, "-")), (mb, ma, (2, "-", 1, "+"))], pipeline=pipe,
                                        text=True)
            assert t1 == t2 and np.array_equal(r1, r2)
            assert [x["n_aabb_pass"] for x in st1] == [x["n_aabb_pass"] for x in st2]
        for m in (va, vb, ma, mb):
            m.free()
    gu.free()
    gs.free()


def test_plan_failure_names_the_layer_pair():
    """a device failure surfaces as a task error carrying the layer-pair id —
    a NaN in one half-layer of a plan names that task, not the whole plan."""
    from paper_2109_14814_b200 import errors, layers
    from paper_2109_14814_b200.mesh import half_layer, layered_mesh
    u = layered_mesh(48, "unstable", 2, 1.6, 0.1, 1)
    s = layered_mesh(48, "stable", 2, 1 / 1.6, 0.1, 2)
    plan = layers.enumerate_layer_pairs(u, s, 2)
    c0, c1 = half_layer(s, 2, -1).col_range
    s.coords[1, (c0 + c1) // 2, 7] = np.nan  # only S_2^- is poisoned
    with pytest.raises(errors.BackendError) as exc:
        layers.search_plan(u, s, plan)
    assert exc.value.task is not None and exc.value.task[2:] == (2, "-")
    assert "non-finite" in str(exc.value)


@pytest.mark.parametrize("shape", [((333, 701), (257, 129)), ((1024, 257), (96, 257)), ((512, 513), (384, 385))])
def test_pageable_staged_upload_identical(shape, monkeypatch):
    """Grids of >= 2 MB from pageable NumPy memory go through the pinned staging ring
    (host copy threads, non-temporal stores, pieces of the 4 planes per slot); the results
    must equal those of pinned sources and of the driver's own pageable copy
    (MCX_NO_STAGE), for the plain and the stepped (unbalanced) search and for grid loads."""
    import torch
    from paper_2109_14814_b200 import runtime
    (na, ma), (nb, mb) = shape
    A, sa = manifold_like(na, ma, 1)
    B, sb = manifold_like(nb, mb, 2)
    ctx = runtime.context(0)
    got = ctx.find(A, sa, B, sb, pipeline=_lib.PIPE_TRIANGLE, text=True)
    pa, pb = torch.from_numpy(A).pin_memory(), torch.from_numpy(B).pin_memory()
    pinned = ctx.find(pa, sa, pb, sb, pipeline=_lib.PIPE_TRIANGLE, text=True)
    monkeypatch.setenv("MCX_NO_STAGE", "1")
    driver = ctx.find(A, sa, B, sb, pipeline=_lib.PIPE_TRIANGLE, text=True)
    monkeypatch.delenv("MCX_NO_STAGE")
    for other in (pinned, driver):
        assert np.array_equal(got[0], other[0]) and got[1] == other[1]
    assert len(got[0]) > 0
    g = ctx.grid(A, sa)  # unpacked grid load (the plan path) through the staging ring
    try:
        v = ctx.view(g, 0, ma - 1)
        try:
            w = ctx.mesh(A, sa)
            try:
                rb = ctx.mesh(B, sb)
                try:
                    r1 = ctx.intersect([(v, rb, (1, "+", 1, "-"))], pipeline=_lib.PIPE_TRIANGLE, text=True)
                    r2 = ctx.intersect([(w, rb, (1, "+", 1, "-"))], pipeline=_lib.PIPE_TRIANGLE, text=True)
                    assert r1[1] == r2[1] and np.array_equal(r1[0]["gid"], r2[0]["gid"])
                finally:
                    rb.free()
            finally:
                w.free()
        finally:
            v.free()
    finally:
        g.free()


@pytest.mark.parametrize("sizes", [((64, 200), (48, 120)), ((512, 900), (300, 400)), ((1024, 700), (96, 300))])
def test_strided_half_layers_read_in_place(sizes):
    """mcx_find_intersections_strided: column ranges of larger host meshes (the reference's
    HalfLayer views, plane stride > N·M) give the records and text of their contiguous
    copies — small (driver copy), staged (>= 2 MB pageable) and stepped (unbalanced) — and
    isect.find_intersections passes HalfLayers without a host copy."""
    from paper_2109_14814_b200 import runtime
    from paper_2109_14814_b200.mesh import ManifoldMesh, HalfLayer
    (na, ma), (nb, mb) = sizes
    A, sa = manifold_like(na, ma, 1)
    B, sb = manifold_like(nb, mb, 2)
    ha = HalfLayer(ManifoldMesh(A, sa), n=2, sign=1, col_range=(ma // 5, ma - ma // 7))
    hb = HalfLayer(ManifoldMesh(B, sb), n=3, sign=-1, col_range=(mb // 9, mb - 2))
    va, vb = ha.coords, hb.coords
    assert not va.flags.c_contiguous and runtime._host_grid(va)[2] == ma * na
    ctx = runtime.context(0)
    texts = {}
    for pipe in (_lib.PIPE_SPEC, _lib.PIPE_TRIANGLE):
        got = ctx.find(va, ha.s_values, vb, hb.s_values, (2, "+", 3, "-"), pipeline=pipe, text=True)
        ref = ctx.find(np.ascontiguousarray(va), ha.s_values, np.ascontiguousarray(vb), hb.s_values,
                       (2, "+", 3, "-"), pipeline=pipe, text=True)
        assert np.array_equal(got[0], ref[0]) and got[1] == ref[1]
        texts[pipe] = got[1]
    recs = isect.find_intersections(ha, hb)  # the plugin call on HalfLayers (spec pipeline)
    assert [r.to_line() for r in recs] == texts[_lib.PIPE_SPEC].decode().splitlines()
