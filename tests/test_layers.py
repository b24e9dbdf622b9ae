"""Layer-pair plan: enumeration counts, TOF, plan file, CLI."""
import math

import pytest

from paper_2109_14814_b200 import cli, errors, layers
from paper_2109_14814_b200.mesh import half_layer, layered_mesh, write_mesh


def _meshes(n_max=3, N=32):
    return (layered_mesh(N, "unstable", n_max, 1.6, 0.1, 1), layered_mesh(N, "stable", n_max, 1 / 1.6, 0.1, 2))


@pytest.mark.parametrize("n_max,count", [(1, 4), (2, 12), (5, 36)])
def test_enumeration_counts(n_max, count):  # SPEC.md:388-389, acceptance 5
    u, s = _meshes(n_max, 8)
    plan = layers.enumerate_layer_pairs(u, s, n_max)
    assert len(plan) == count == 4 * (2 * n_max - 1)
    assert len(set(plan.tasks)) == count
    assert all(n2 in (n1, n1 - 1) and n2 >= 1 for n1, _, n2, _ in plan.tasks)


def test_tof():  # TOF of a hit in (U3, S2) = 2π·5/Ω_p
    u, s = _meshes(3, 8)
    plan = layers.enumerate_layer_pairs(u, s, 3, omega_p=2.5)
    for (n1, _, n2, _), tof in zip(plan.tasks, plan.tof):
        assert tof == pytest.approx(2 * math.pi * (n1 + n2) / 2.5)


def test_plan_file_roundtrip(tmp_path):
    u, s = _meshes(2, 8)
    plan = layers.enumerate_layer_pairs(u, s, 2)
    p = tmp_path / "plan.txt"
    layers.write_plan(p, plan)
    back = layers.read_plan(p)
    assert back.tasks == plan.tasks and back.tof == plan.tof
    (tmp_path / "bad.txt").write_text("1 + 1\n")
    with pytest.raises(errors.FileFormatError):
        layers.read_plan(tmp_path / "bad.txt")


def test_half_layers_cover_columns():  # SPEC.md:381 telescoping union
    u, _ = _meshes(3, 8)
    cols = set()
    for n in range(1, 4):
        h = half_layer(u, n, +1)
        cols |= set(range(h.col_range[0], h.col_range[1] + 1))
        assert h.s_values[0] == pytest.approx(u.D * u.lam ** (n - 1))
    assert cols == {k for k in range(u.M) if u.s_values[k] >= u.D - 1e-15}


def test_cli_layers_and_errors(tmp_path):
    u, s = _meshes(2, 8)
    write_mesh(tmp_path / "u.mnf", u)
    write_mesh(tmp_path / "s.mnf", s)
    rc = cli.main(["layers", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"), "--nmax", "2",
                   "--plan", str(tmp_path / "plan.txt")])
    assert rc == 0 and len(layers.read_plan(tmp_path / "plan.txt")) == 12
    assert cli.main(["layers", "--umesh", str(tmp_path / "nope.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                     "--nmax", "2", "--plan", str(tmp_path / "p2.txt")]) == 4
    assert cli.main(["layers", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                     "--nmax", "9", "--plan", str(tmp_path / "p3.txt")]) == 2
    assert cli.main(["intersect", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"),
                     "--plan", str(tmp_path / "plan.txt"), "--backend", "serial", "--out", str(tmp_path / "r")]) == 2
    assert cli.main(["bogus"]) == 2


def test_include_core():  # --include-core re-enables the fundamental-domain cores
    u, s = _meshes(2, 8)
    plan = layers.enumerate_layer_pairs(u, s, 2, omega_p=2.0, include_core=True)
    assert len(plan) == 12 + 3
    assert plan.tasks[:3] == [(0, "+", 0, "+"), (1, "+", 0, "+"), (1, "-", 0, "+")]
    assert plan.tof[:3] == [0.0, pytest.approx(math.pi), pytest.approx(math.pi)]
    core = half_layer(u, 0, +1)
    lo, hi = core.col_range
    assert u.s_values[lo] == pytest.approx(-u.D) and u.s_values[hi] == pytest.approx(u.D)
    with pytest.raises(errors.ConfigError):
        half_layer(u, 0, -1)  # the core is one half-layer


def test_cli_layers_include_core(tmp_path):
    u, s = _meshes(2, 8)
    write_mesh(tmp_path / "u.mnf", u)
    write_mesh(tmp_path / "s.mnf", s)
    assert cli.main(["layers", "--umesh", str(tmp_path / "u.mnf"), "--smesh", str(tmp_path / "s.mnf"), "--nmax", "2",
                     "--plan", str(tmp_path / "plan.txt"), "--include-core"]) == 0
    assert layers.read_plan(tmp_path / "plan.txt").tasks[0] == (0, "+", 0, "+")


def test_read_plan_rejects_malformed_signs(tmp_path):  # '+-' used to pass a substring test
    p = tmp_path / "plan.txt"
    p.write_text("1 +- 1 + 6.28\n")
    with pytest.raises(errors.FileFormatError):
        layers.read_plan(p)


def test_assign_tasks_is_balanced_and_deterministic():
    costs = [9.0, 1.0, 5.0, 5.0, 3.0, 3.0, 2.0, 8.0]
    parts = layers.assign_tasks(costs, 3)
    assert sorted(k for p in parts for k in p) == list(range(8))
    assert parts == layers.assign_tasks(costs, 3)
    loads = [sum(costs[k] for k in p) for p in parts]
    assert max(loads) - min(loads) <= max(costs)
