"""Pin the CPU oracle (oracle/hvb_oracle.py) against the LIVE reference's
outputs recorded in tests/golden/golden.npz (make_golden.py)."""

import numpy as np
import pytest

from conftest import CASES
from oracle import hvb_oracle as ora

FULL = ["sphere2", "cap2", "floatshell1", "diel1", "diel2", "gap2", "cfg3mini", "plates"]


@pytest.mark.parametrize("name", FULL)
def test_oracle_matrix(golden, cases, name):
    m = cases(name)
    A = ora.assemble_dense(m)
    assert ora.entry_error(A, golden[name + "_A"]) <= 1e-10
    np.testing.assert_array_equal(ora.rhs(m), golden[name + "_rhs"])


def test_oracle_rodmini_rows(golden, cases):
    m = cases("rodmini")
    rows = golden["rodmini_rows"]
    A = ora.row_equations(m, rows)
    assert ora.entry_error(A, golden["rodmini_Arows"]) <= 1e-10


@pytest.mark.parametrize("name", CASES)
def test_oracle_near_pairs(golden, cases, name):
    m = cases(name)
    want = {tuple(p) for p in golden[name + "_nearpairs"].tolist()}
    rows = sorted({p[0] for p in want})[:40] or [0]
    _, got = ora.kernel_rows(m, m.colloc_points[rows], rows, "sl")
    got = {(rows[r], t) for r, t in got}
    want = {p for p in want if p[0] in set(rows)}
    assert got == want


def test_oracle_charge(golden, cases):
    m = cases("sphere2")
    q = ora.charge_vector(m, np.arange(m.n_collocation), ora.EPS0, 0.5 * ora.EPS0)
    ref = golden["sphere2_charge"]
    assert np.max(np.abs(q - ref)) <= 1e-10 * np.max(np.abs(ref))


@pytest.mark.parametrize("name", ["sphere2", "cap2", "diel1", "gap2", "plates"])
def test_oracle_fields(golden, cases, name):
    m = cases(name)
    u = golden[name + "_u"]
    pts = golden[name + "_pts"]
    E = ora.efield_points(m, u, pts)
    Eref = golden[name + "_E"]
    scale = max(np.max(np.abs(Eref)), 1e-300)
    assert np.max(np.abs(E - Eref)) <= 1e-9 * scale
    phi = ora.potential_points(m, u, pts)
    assert np.max(np.abs(phi - golden[name + "_phi"])) <= 1e-10 * np.max(np.abs(golden[name + "_phi"]))


def test_oracle_surface_field(golden, cases):
    m = cases("sphere2")
    s = ora.surface_field(m, golden["sphere2_u"], indices=np.arange(0, 162, 7))
    np.testing.assert_allclose(s, golden["sphere2_surfE"][::7], rtol=1e-10)


@pytest.mark.parametrize("name", ["sphere2", "cap2", "floatshell1", "diel2", "gap2", "cfg3mini"])
def test_oracle_gmres_semantics(golden, name):
    A = golden[name + "_A"]
    b = golden[name + "_rhs"]
    x, it, res = ora.gmres(A, b, rel_tol=1e-12, max_iters=600)
    it_ref, conv = golden[name + "_iters"]
    assert conv == 1 and it == it_ref
    u = golden[name + "_u"]
    assert np.max(np.abs(x[: len(u)] - u)) <= 1e-8 * np.max(np.abs(u))


def test_oracle_rules(golden):
    for c in range(3):
        uv, w = ora.duffy(c, 6)
        np.testing.assert_array_equal(uv, golden[f"duffy{c}_nodes"])
        np.testing.assert_array_equal(w, golden[f"duffy{c}_weights"])
    uv, w = ora.graded(3, 8, 8)
    np.testing.assert_array_equal(uv, golden["graded_nodes"])
    np.testing.assert_array_equal(w, golden["graded_weights"])


def test_oracle_closest_point_decisions(golden):
    cases = golden["closest_cases"]
    for row in cases[:1500]:
        cs = row[:9].reshape(3, 3)
        x = row[9:12]
        assert ora.closest_point_flat(x, *cs) == (row[12], row[13])


def test_oracle_near_rule(golden):
    corners = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    nodes6 = np.vstack([corners, 0.5 * (corners[0] + corners[1]), 0.5 * (corners[1] + corners[2]),
                        0.5 * (corners[2] + corners[0])])
    R = np.sqrt(0.5)
    for frac in (0.1, 0.3, 0.6, 1.0):
        x = corners.mean(axis=0) + np.array([0.0, 0.0, frac * R])
        uv, w = ora.near_rule(x, nodes6, R, ora.DEFAULT_CFG)
        np.testing.assert_allclose(uv, golden[f"near_{frac}_nodes"], rtol=0, atol=1e-15)
        np.testing.assert_allclose(w, golden[f"near_{frac}_weights"], rtol=1e-14)
