"""CPU tests of the host side: the C ABI library's exports and struct layout, the
reference-facing API's error behaviour, mesh / records I/O and record building."""
import ctypes
import os
import re
import subprocess
import sys

import numpy as np
import pytest

from oracle import canonical as O
from paper_2109_14814_b200 import _lib, errors, isect
from paper_2109_14814_b200.mesh import (HalfLayer, ManifoldMesh, config_pair, half_layer, manifold_like,
                                        read_mesh, write_mesh)

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
HEADER = os.path.join(ROOT, "include", "mcx.h")


def _header_functions():
    txt = open(HEADER).read()
    return sorted(set(re.findall(r"^\s*(?:[a-z_0-9]+\s*\*?\s+)+\**(mcx_[a-z_0-9]+)\s*\(", txt, re.M)))


def test_library_exports_every_header_symbol():
    L = _lib.load()  # loads without a GPU (cudart is linked statically)
    funcs = _header_functions()
    assert set(funcs) == set(_lib.EXPORTS)
    for f in funcs:
        assert hasattr(L, f), f
    assert L.mcx_version() == 3
    assert L.mcx_a_block() == 1024
    assert isinstance(L.mcx_last_error(), bytes)


LAYOUT = [  # (C expression, ctypes value)
    ("sizeof(mcx_mesh_dev)", ctypes.sizeof(_lib.MeshDev)), ("offsetof(mcx_mesh_dev, N)", _lib.MeshDev.N.offset),
    ("offsetof(mcx_mesh_dev, box)", _lib.MeshDev.box.offset), ("offsetof(mcx_mesh_dev, status)", _lib.MeshDev.status.offset),
    ("sizeof(mcx_hit)", ctypes.sizeof(_lib.Hit)), ("offsetof(mcx_hit, s)", _lib.Hit.s.offset),
    ("sizeof(mcx_stats)", ctypes.sizeof(_lib.Stats)), ("offsetof(mcx_stats, n_candidates)", _lib.Stats.n_candidates.offset),
    ("sizeof(mcx_opts)", ctypes.sizeof(_lib.Opts)), ("offsetof(mcx_opts, mode)", _lib.Opts.mode.offset),
    ("offsetof(mcx_opts, workspace)", _lib.Opts.workspace.offset), ("offsetof(mcx_opts, pipeline)", _lib.Opts.pipeline.offset),
    ("offsetof(mcx_opts, cand_cap)", _lib.Opts.cand_cap.offset), ("offsetof(mcx_opts, orient)", _lib.Opts.orient.offset),
    ("sizeof(mcx_task)", ctypes.sizeof(_lib.Task)), ("sizeof(mcx_record)", ctypes.sizeof(_lib.Record)),
    ("offsetof(mcx_record, point)", _lib.Record.point.offset), ("offsetof(mcx_record, params)", _lib.Record.params.offset),
    ("offsetof(mcx_record, task)", _lib.Record.task.offset), ("sizeof(mcx_layer)", ctypes.sizeof(_lib.Layer)),
    ("sizeof(mcx_job)", ctypes.sizeof(_lib.Job)), ("offsetof(mcx_job, layer)", _lib.Job.layer.offset),
    ("sizeof(mcx_find_opts)", ctypes.sizeof(_lib.FindOpts)),
    ("offsetof(mcx_find_opts, shard_count)", _lib.FindOpts.shard_count.offset),
    ("offsetof(mcx_find_opts, orient)", _lib.FindOpts.orient.offset),
]


def test_struct_layout_matches_header(tmp_path):
    src = tmp_path / "layout.c"
    body = "".join(f'printf("%zu\\n", (size_t)({expr}));' for expr, _ in LAYOUT)
    src.write_text('#include <stdio.h>\n#include <stddef.h>\n#include "mcx.h"\nint main(void){' + body + "return 0;}\n")
    exe = tmp_path / "layout"
    subprocess.run(["gcc", "-I", os.path.join(ROOT, "include"), "-o", str(exe), str(src)], check=True)
    got = [int(v) for v in subprocess.run([str(exe)], capture_output=True, text=True, check=True).stdout.split()]
    assert got == [v for _, v in LAYOUT]


def test_device_formatter_matches_python_g17():
    """mcx_format_g17 is the host build of the device records formatter (mcx_format.cuh):
    it must print every double exactly like Python's f"{v:.17g}" (SPEC.md:507 records)."""
    L = _lib.load()
    rng = np.random.default_rng(7)
    vals = [0.0, -0.0, np.inf, -np.inf, np.nan, 1e16, 1e17, 0.0001, 1e-5, 0.1, 2.0 ** 60, 5e-324,
            1.7976931348623157e308, 1e-310, 6.283185307179586, 123456789012345650.0]
    for e in range(-324, 309, 7):
        x = float(f"1e{e}")
        vals += [x, np.nextafter(x, 0.0), np.nextafter(x, np.inf)]
    vals += list(rng.integers(0, 2 ** 64, size=20000, dtype=np.uint64).view(np.float64))
    vals += list(rng.normal(size=20000)) + list(rng.uniform(0, 1, 20000))
    # dyadic rationals (terminating decimal expansions: exact ties at the 17th digit occur)
    vals += list(rng.integers(1, 2 ** 53, 20000) / 2.0 ** rng.integers(0, 80, 20000))
    vals += [float(v) for v in rng.integers(0, 2 ** 63, 2000, dtype=np.int64)]  # integers (gid-sized)
    buf = ctypes.create_string_buffer(64)
    for v in vals:
        n = L.mcx_format_g17(float(v), buf)
        assert buf.value.decode() == f"{float(v):.17g}", repr(v)
        assert n == len(buf.value)


def test_formatter_integers_match_printf(tmp_path):
    """put_u64 (the gid field and exponents of the device records text) against printf
    %llu over edge and random 64-bit values: the header compiled as plain C++ (g++)."""
    import shutil
    import subprocess
    if not shutil.which("g++"):
        pytest.skip("g++ not available")
    src = tmp_path / "fmt.cpp"
    src.write_text(
        '#include <cstdio>\n#include <cstdint>\n#include "mcx_format.cuh"\n'
        "int main() {\n"
        "  uint64_t x = 88172645463325252ull;\n"
        "  uint64_t edge[] = {0, 1, 9, 10, 999999999ull, 1000000000ull, 1000000001ull, 4294967295ull,\n"
        "                     4294967296ull, 999999999999999999ull, 1000000000000000000ull,\n"
        "                     10000000000000000000ull, 18446744073709551615ull};\n"
        "  char buf[32], ref[32];\n"
        "  for (int i = 0; i < 200000 + 13; ++i) {\n"
        "    uint64_t v;\n"
        "    if (i < 13) v = edge[i];\n"
        "    else { x ^= x << 13; x ^= x >> 7; x ^= x << 17; v = x >> (x % 64); }\n"
        "    int n = mcx::fmt::put_u64(buf, v);\n"
        "    buf[n] = 0;\n"
        "    snprintf(ref, sizeof ref, \"%llu\", (unsigned long long)v);\n"
        "    for (int k = 0; ; ++k) { if (buf[k] != ref[k]) { printf(\"bad %s %s\\n\", buf, ref); return 1; }\n"
        "                            if (!ref[k]) break; }\n"
        "  }\n"
        "  printf(\"ok\\n\");\n"
        "  return 0;\n"
        "}\n")
    exe = tmp_path / "fmt"
    subprocess.run(["g++", "-O1", "-I", os.path.join(ROOT, "paper_2109_14814_b200", "csrc"), "-o", str(exe), str(src)],
                   check=True)
    out = subprocess.run([str(exe)], capture_output=True, text=True)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stdout


def test_only_cuda_backend():
    A, _ = manifold_like(8, 3, 1)
    for bad in ("serial", "parallel", "cpu"):
        with pytest.raises(errors.ConfigError):
            isect.find_intersections(A, A, backend=bad)
        with pytest.raises(errors.ConfigError):
            isect.pair_candidates(A, A, backend=bad)


def test_no_silent_cpu_fallback():
    torch = pytest.importorskip("torch")
    if torch.cuda.is_available():
        pytest.skip("GPU present")
    A, _ = manifold_like(8, 3, 1)
    with pytest.raises(errors.BackendError):
        isect.find_intersections(A, A)


def test_error_hierarchy_exit_codes():
    assert issubclass(errors.CapacityError, errors.BackendError)
    assert issubclass(errors.BackendError, errors.ManiconnError)
    assert errors.exit_code(errors.ConfigError("x")) == 2
    assert errors.exit_code(errors.NumericsError("x")) == 3
    assert errors.exit_code(errors.SingularSystemError("x", condition=1e13)) == 3
    assert errors.exit_code(errors.FileFormatError("x")) == 4
    assert errors.exit_code(errors.BackendError("x")) == 3
    e = errors.BackendError("boom", task=(3, "+", 2, "-"), status=2)
    assert "layer pair (3, '+', 2, '-')" in str(e)


REF_SRC = "/root/reference/pkg/src"


@pytest.mark.skipif(not os.path.isdir(REF_SRC), reason="reference sources not present (GPU box)")
def test_errors_are_the_reference_classes_when_importable():
    """With the reference package on the path, a reference caller's except clauses catch
    this backend's errors: the shared classes ARE maniconn.errors' (errors.py:4-53)."""
    code = (
        "import maniconn.errors as R\n"
        "from paper_2109_14814_b200 import errors as E, isect\n"
        "assert E.REFERENCE_CLASSES\n"
        "for n in ('ManiconnError', 'ConfigError', 'NumericsError', 'SingularSystemError', 'FileFormatError'):\n"
        "    assert getattr(E, n) is getattr(R, n), n\n"
        "assert issubclass(E.BackendError, R.ManiconnError) and issubclass(E.CapacityError, R.ManiconnError)\n"
        "import numpy as np\n"
        "try:\n"
        "    isect.find_intersections(np.zeros((4, 3, 8)), np.zeros((4, 3, 8)), backend='serial')\n"
        "except R.ConfigError:\n"
        "    pass\n"
        "else:\n"
        "    raise SystemExit('not caught')\n"
        "print('ok')\n")
    env = dict(os.environ, PYTHONPATH=os.pathsep.join([REF_SRC, ROOT, os.environ.get("PYTHONPATH", "")]))
    out = subprocess.run([sys.executable, "-c", code], env=env, capture_output=True, text=True, cwd=ROOT)
    assert out.returncode == 0 and out.stdout.strip() == "ok", out.stderr


def _mesh():
    N, K, n_max, lam, D = 16, 3, 2, 2.0, 0.1
    s = sorted({k * D / K for k in range(-K, K + 1)} | {sg * D * lam ** n for n in range(1, n_max + 1)
                                                         for sg in (1, -1)} | {sg * D * lam ** n * 0.7
                                                                               for n in range(1, n_max + 1) for sg in (1, -1)})
    s = np.array(s)
    coords, _ = manifold_like(N, len(s), 4)
    return ManifoldMesh(coords=coords, s_values=s, kind="unstable", omega=1.3, lam=lam, D=D, n_max=n_max,
                        boundary_cols=(0, len(s) - 1))


def test_mnf1_roundtrip(tmp_path):
    m = _mesh()
    p = tmp_path / "m.mnf"
    write_mesh(p, m)
    r = read_mesh(p)
    assert np.array_equal(r.coords, m.coords) and np.array_equal(r.s_values, m.s_values)
    assert (r.kind, r.omega, r.lam, r.D, r.n_max, r.boundary_cols) == (m.kind, m.omega, m.lam, m.D, m.n_max,
                                                                      m.boundary_cols)
    raw = p.read_bytes()
    (tmp_path / "bad").write_bytes(b"XXXX" + raw[4:])
    with pytest.raises(errors.FileFormatError):
        read_mesh(tmp_path / "bad")
    (tmp_path / "trail").write_bytes(raw + b"\0")
    with pytest.raises(errors.FileFormatError):
        read_mesh(tmp_path / "trail")
    (tmp_path / "trunc").write_bytes(raw[:100])
    with pytest.raises(errors.FileFormatError):
        read_mesh(tmp_path / "trunc")


def test_half_layer_columns():
    m = _mesh()
    h = half_layer(m, 1, +1)
    assert h.s_values[0] == pytest.approx(m.D) and h.s_values[-1] == pytest.approx(m.D * m.lam)
    assert h.M >= 2 and h.n_triangles == 2 * m.N * (h.M - 1)
    hn = half_layer(m, 2, -1)
    assert hn.s_values[0] == pytest.approx(-m.D * m.lam ** 2) and hn.s_values[-1] == pytest.approx(-m.D * m.lam)
    assert np.array_equal(h.coords, m.coords[:, h.col_range[0]:h.col_range[1] + 1])
    with pytest.raises(errors.ConfigError):
        half_layer(m, 3, +1)
    with pytest.raises(errors.ConfigError):
        HalfLayer(mesh=m, col_range=(2, 2))


def test_from_planes_layout():
    coords, s = manifold_like(6, 4, 2)
    m = ManifoldMesh.from_planes(coords[0].T, coords[1].T, coords[2].T, coords[3].T, s)
    assert np.array_equal(m.coords, coords)
    # paper's storage: entry (i, k) of plane c at linear index i + N·k (column-major)
    flat = m.coords[1].ravel()
    assert flat[3 + 6 * 2] == m.plane(1)[3, 2]


def test_records_from_oracle_hits(tmp_path):
    A, sa, B, sb = config_pair("C1")
    r = O.search(A, B)
    hits = np.zeros(len(r["ia"]), dtype=[("ia", "<u4"), ("ib", "<u4"), ("s", "<f8"), ("t", "<f8"),
                                         ("a", "<f8"), ("b", "<f8")])
    for k in ("ia", "ib", "s", "t", "a", "b"):
        hits[k] = r[k]
    recs = isect.hits_to_records(A, sa, B, sb, hits, layer=(3, "+", 2, "-"))
    assert len(recs) == 4
    pts_o = O.hit_points(A, r["ia"], r["s"], r["t"])
    gids = [rc.pair.gid for rc in recs]
    assert gids == sorted(gids)
    for rc in recs:
        a, b, c, d = rc.bary
        assert min(a, b, c, d) >= 0 and a + b <= 1 and c + d <= 1
        n = np.nonzero((r["ia"] == rc.tri_index[0]) & (r["ib"] == rc.tri_index[1]))[0][0]
        assert np.array_equal(rc.point, pts_o[n])
        # the B side gives the same point within 1e-10·scale
        pB = O.take(O.pack(B), np.array([rc.tri_index[1]]))
        qpt = (pB["p"][0] + c * pB["e1"][0]) + d * pB["e2"][0]
        assert np.max(np.abs(qpt - rc.point)) < 1e-10
        # parameter estimates are inside the quad's parameter cell
        thA = 2 * np.pi * np.arange(64) / 64
        assert thA[rc.pair.i] - 1e-12 <= rc.params[0] <= thA[rc.pair.i] + 2 * np.pi / 64 + 1e-12
        assert min(sa[rc.pair.k - 1], sa[rc.pair.k]) - 1e-12 <= rc.params[1] <= max(sa[rc.pair.k - 1], sa[rc.pair.k]) + 1e-12
    p = tmp_path / "rec.txt"
    isect.write_records(p, recs)
    lines = p.read_text().splitlines()
    assert len(lines) == 4 and all(len(ln.split()) == 17 for ln in lines)
    back = isect.read_records(p)
    for a, b in zip(recs, back):
        assert np.array_equal(a.point, b.point) and a.bary == b.bary and a.params == b.params
        assert a.pair.gid == b.pair.gid and a.layer == b.layer
    (tmp_path / "bad.txt").write_text("1 + 2\n")
    with pytest.raises(errors.FileFormatError):
        isect.read_records(tmp_path / "bad.txt")


def test_param_estimates_t2_vertices():
    """The T² barycentric→(θ,s) map hits the T² vertices exactly (SPEC.md:499 design decision)."""
    N, M = 8, 3
    coords, s = manifold_like(N, M, 1)
    i, k1 = 5, 1
    tA = 2 * (i + N * k1) + 1
    th = 2 * np.pi * np.arange(N) / N
    for (x, y), want in (((0.0, 0.0), (th[i], s[k1 + 1])), ((1.0, 0.0), (th[i] + 2 * np.pi / N, s[k1])),
                         ((0.0, 1.0), (th[i] + 2 * np.pi / N, s[k1 + 1]))):
        hits = np.zeros(1, dtype=[("ia", "<u4"), ("ib", "<u4"), ("s", "<f8"), ("t", "<f8"), ("a", "<f8"), ("b", "<f8")])
        hits["ia"], hits["ib"], hits["s"], hits["t"] = tA, 0, x, y
        rc = isect.hits_to_records(coords, s, coords, s, hits, dedup=False)[0]
        assert rc.params[0] == pytest.approx(want[0]) and rc.params[1] == pytest.approx(want[1])


def test_dedup_within_tolerance():
    pts = np.array([[0, 0, 0, 0], [5e-10, 0, 0, 0], [2e-9, 0, 0, 0], [1, 1, 1, 1], [1, 1, 1, 1 + 1e-10]], float)
    keep = isect._dedup_mask(pts, 1e-9)
    assert keep.tolist() == [True, False, True, True, False]


def test_dedup_greedy_chain():
    """a~b, b~c, not a~c: the greedy rule keeps a, drops b, keeps c (record order)."""
    pts = np.array([[0, 0, 0, 0], [8e-10, 0, 0, 0], [1.6e-9, 0, 0, 0]], float)
    assert isect._dedup_mask(pts, 1e-9).tolist() == [True, False, True]
    rng = np.random.default_rng(0)
    base = rng.normal(size=(50, 4))
    pts = np.concatenate([base, base + 1e-12, base[::-1]])
    keep = isect._dedup_mask(pts, 1e-9)
    assert keep.sum() == 50 and keep[:50].all()


def test_host_grid_plane_stride():
    """runtime._host_grid: a HalfLayer view (column range of its mesh) is passed in place
    with the mesh's plane stride; dense grids get stride 0; other layouts are copied."""
    from paper_2109_14814_b200 import runtime
    from paper_2109_14814_b200.mesh import HalfLayer, ManifoldMesh, manifold_like
    A, s = manifold_like(16, 40, 1)
    h = HalfLayer(ManifoldMesh(A, s), col_range=(5, 20))
    p, keep, plane = runtime._host_grid(h.coords)
    assert plane == 40 * 16 and p == A.ctypes.data + 5 * 16 * 8 and keep is h.coords or keep.base is not None
    assert runtime._host_grid(A)[2] == 0                      # dense
    assert runtime._host_grid(HalfLayer.whole(ManifoldMesh(A, s)).coords)[2] == 0
    T = np.ascontiguousarray(A.transpose(0, 2, 1)).transpose(0, 2, 1)  # rows not contiguous
    p2, keep2, plane2 = runtime._host_grid(T)
    assert plane2 == 0 and keep2.flags.c_contiguous and np.array_equal(keep2, A)
