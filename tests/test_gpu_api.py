"""Drop-in conformance: the reference test-suite's API semantics (errors,
structure, invariants, analytic electrostatics) exercised through the
B200 package (reference tests/test_assembly.py, test_solver.py,
test_postprocess.py, test_kernels.py, test_acceptance.py)."""

import numpy as np
import pytest

from conftest import gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a CUDA device")]

from paper_2003_12663_b200 import fixtures  # noqa: E402
from paper_2003_12663_b200.mesh import EPS0  # noqa: E402


@pytest.fixture(scope="module")
def sphere2_solved():
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.solver import solve

    m = fixtures.sphere_mesh(2)
    A, b = assemble(m)
    return m, A, b, solve(A, b)


@pytest.fixture(scope="module")
def capacitor2():
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.solver import solve

    m = fixtures.concentric_mesh(2, [(0.5, "electrode 1.0"), (1.0, "electrode 0.0")])
    A, b = assemble(m)
    return m, solve(A, b)


# -- assembly ---------------------------------------------------------------


def test_missing_floating_surface_errors():
    from paper_2003_12663_b200.assembly import AssemblyError, assemble

    v, tris = fixtures.sphere_mesh_parts(1)
    ids = np.array([t[0] for t in tris])
    m = fixtures.mesh_from_parts(v, ids, np.zeros(len(ids), int), ["patch 0 electrode 1.0", "patch 1 floating 0"])
    with pytest.raises(AssemblyError, match="floating surface 0"):
        assemble(m)


def test_floating_structure_and_pair_completeness():
    from paper_2003_12663_b200.assembly import assemble

    m = fixtures.concentric_mesh(1, [(0.5, "electrode 1.0"), (0.75, f"sheet 0 {EPS0!r} {EPS0!r}"),
                                     (1.0, "electrode 0.0")])
    A, rhs = assemble(m)
    n = m.n_collocation
    dense = A.toarray()
    mem = m.floating_collocation(0)
    assert np.all(dense[mem, n] == -1.0)
    others = np.setdiff1d(np.arange(n), mem)
    assert np.all(dense[others, n] == 0.0) and np.all(rhs[mem] == 0.0)
    d = A.diagnostics
    assert d["pairs_regular"] + d["pairs_singular"] + d["pairs_near_singular"] == d["rows_with_integrals"] * d["n_triangles"]


def test_dirichlet_rows_on_constant_density_converge():
    from paper_2003_12663_b200.assembly import assemble, matvec

    errs = []
    for level in (1, 2):
        A, _ = assemble(fixtures.sphere_mesh(level))
        errs.append(np.max(np.abs(matvec(A, np.ones(A.size)) - 1.0)))
    assert errs[1] < errs[0] and errs[0] / errs[1] > 3.0


def test_dielectric_constant_density_limit():
    from paper_2003_12663_b200.assembly import assemble, matvec

    errs = []
    for level in (1, 2):
        v, tris = fixtures.sphere_mesh_parts(level)
        ids = np.array([t[0] for t in tris])
        m = fixtures.mesh_from_parts(v, ids, np.zeros(len(ids), int), ["patch 0 dielectric 2.0 5.0"])
        A, _ = assemble(m)
        got = matvec(A, np.ones(A.size))
        errs.append(np.max(np.abs(got - 2.0)) / 2.0)  # (e+ + e-)/2 + (e+ - e-)/2 = e+
    assert errs[1] < errs[0] and errs[1] < 0.01


def test_kprime_identity_and_efield_rows():
    from paper_2003_12663_b200.assembly import KERNEL_ADL, KERNEL_E, assemble_kernel_row

    m = fixtures.sphere_mesh(2)
    i = 17
    adl, _ = assemble_kernel_row(m, None, m.colloc_points[i], int(m.colloc_vertex_ids[i]), KERNEL_ADL,
                                 n_x=m.colloc_normals[i])
    assert abs(adl.sum() - 0.5) < 0.02
    e_rows, c = assemble_kernel_row(m, None, m.colloc_points[i], int(m.colloc_vertex_ids[i]), KERNEL_E)
    assert e_rows.shape == (m.n_collocation, 3)
    np.testing.assert_allclose(e_rows @ m.colloc_normals[i], adl, rtol=1e-12, atol=1e-15)
    assert c["singular"] == 6


def test_matrix_dump_roundtrip(tmp_path):
    from paper_2003_12663_b200.assembly import assemble, load_matrix, save_matrix

    A, _ = assemble(fixtures.sphere_mesh(1), n_blocks=3)
    p = tmp_path / "m.bin"
    save_matrix(A, p)
    B = load_matrix(p)
    assert B.n == A.n and len(B.blocks) == 3
    np.testing.assert_array_equal(B.toarray(), A.toarray())


def test_capacitance_of_unit_sphere(sphere2_solved):
    from paper_2003_12663_b200.assembly import charge_row

    m, _, _, sol = sphere2_solved
    q = charge_row(m, np.arange(m.n_collocation), eps_plus=EPS0)
    exact = 4.0 * np.pi * EPS0
    assert abs(float(q @ sol.u) - exact) / exact < 0.01


# -- solver -------------------------------------------------------------------


def test_gmres_small_systems():
    from oracle.hvb_oracle import gmres as ora_gmres
    from paper_2003_12663_b200.solver import SolverConfig, SolverError, residual, solve

    s = solve(np.diag([2.0, 4.0]), np.array([2.0, 4.0]))
    np.testing.assert_allclose(s.u, [1.0, 1.0], rtol=1e-12)
    assert s.iterations == 1
    a = np.array([[4.0, 1.0, -0.5], [0.3, 3.0, 0.8], [-0.2, 0.6, 5.0]])
    b = np.array([1.0, -2.0, 0.7])
    s = solve(a, b, SolverConfig(rel_tol=1e-12))
    assert np.max(np.abs(s.u - np.linalg.solve(a, b))) < 1e-10
    z = solve(np.diag([1.0, 2.0]), np.zeros(2))
    assert z.iterations == 0 and np.all(z.u == 0)
    with pytest.raises(SolverError) as err:
        solve(np.array([[0.0, 1.0], [-1.0, 0.0]]), np.array([1.0, 1.0]),
              SolverConfig(restart=1, max_iters=3, rel_tol=1e-14))
    assert err.value.best_residual >= 0.0 and err.value.iterations <= 3
    rng = np.random.default_rng(12)
    for n in (10, 30, 50):
        a = rng.standard_normal((n, n)) + n * np.eye(n)
        b = rng.standard_normal(n)
        s = solve(a, b, SolverConfig(restart=n, rel_tol=1e-12, max_iters=n))
        assert s.iterations <= n and residual(a, s.u, b) <= 1e-12
        _, it, _ = ora_gmres(a, b, restart=n, rel_tol=1e-12, max_iters=n)
        assert abs(s.iterations - it) <= 1
    with pytest.raises(ValueError):
        residual(np.eye(3), np.ones(3), np.ones(4))


def test_solution_invariant_under_block_count():
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.solver import solve

    m = fixtures.sphere_mesh(2)
    u1 = solve(*assemble(m, n_blocks=1)).u
    u4 = solve(*assemble(m, n_blocks=4)).u
    np.testing.assert_array_equal(u1, u4)


# -- postprocess ----------------------------------------------------------------


def test_potential_field_analytic(sphere2_solved):
    from paper_2003_12663_b200.postprocess import eval_efield, eval_potential

    m, _, _, sol = sphere2_solved
    assert abs(eval_potential(sol, m, [2.0, 0.0, 0.0]) - 0.5) / 0.5 < 0.01
    e = eval_efield(sol, m, [0.0, 2.0, 0.0])
    assert abs(np.linalg.norm(e) - 0.25) / 0.25 < 0.01
    assert np.linalg.norm(e / np.linalg.norm(e) - [0, 1, 0]) < 1e-3


def test_eval_at_vertex_rejected(sphere2_solved):
    from paper_2003_12663_b200.postprocess import eval_potential

    m, _, _, sol = sphere2_solved
    with pytest.raises(ValueError, match="coincides"):
        eval_potential(sol, m, m.colloc_points[5])


def test_batch_with_one_coincident_point_rejected(sphere2_solved):
    """Large batches run the coincidence check beside the device evaluation;
    one coincident point (a midside node) still raises and returns nothing."""
    from paper_2003_12663_b200.postprocess import eval_efield_batch

    m, _, _, sol = sphere2_solved
    X = np.random.default_rng(3).uniform(-2, 2, (5000, 3))
    X[4321] = m.vertices[-1]
    with pytest.raises(ValueError, match="coincides"):
        eval_efield_batch(sol, m, X)
    X[4321] = [2.5, 0.0, 0.0]
    assert np.all(np.isfinite(eval_efield_batch(sol, m, X)))


def test_field_is_gradient_and_linear(sphere2_solved):
    from paper_2003_12663_b200.postprocess import eval_efield, eval_potential
    from paper_2003_12663_b200.solver import Solution

    m, _, _, sol = sphere2_solved
    x = np.array([1.3, 0.9, -0.6])
    h = 1e-4
    grad = np.array([(eval_potential(sol, m, x + h * e) - eval_potential(sol, m, x - h * e)) / (2 * h)
                     for e in np.eye(3)])
    np.testing.assert_allclose(eval_efield(sol, m, x), -grad, rtol=1e-4)
    rng = np.random.default_rng(8)
    u1, u2 = rng.standard_normal((2, m.n_collocation))

    def phi(u):
        return eval_potential(Solution(u=u, V=np.zeros(0), iterations=0, residual=0.0), m, [1.4, -0.3, 0.8])

    assert phi(u1 + u2) == pytest.approx(phi(u1) + phi(u2), rel=1e-12)


def test_surface_field_and_seeds(sphere2_solved):
    from paper_2003_12663_b200.postprocess import pick_start_points, surface_field_magnitudes

    m, _, _, sol = sphere2_solved
    se = surface_field_magnitudes(m, sol)
    assert np.max(np.abs(se - 1.0)) < 0.02
    starts, idx, _ = pick_start_points(m, sol, 3, surface_e=se)
    assert starts.shape == (3, 3) and all(np.linalg.norm(s) > 1.0 for s in starts)


def test_tracing_semantics(sphere2_solved, capacitor2):
    from paper_2003_12663_b200.postprocess import TraceError, trace_fieldline
    from paper_2003_12663_b200.solver import Solution

    m, _, _, sol = sphere2_solved
    line = trace_fieldline(sol, m, np.array([1.05, 0.0, 0.0]), +1)
    assert line.termination in ("MaxLength", "LeftDomain")
    assert np.abs(line.points[:, 1:]).max() < 1e-3 * np.abs(line.points[:, 0]).max()
    zero = Solution(u=np.zeros_like(sol.u), V=np.zeros(0), iterations=0, residual=0.0)
    with pytest.raises(TraceError):
        trace_fieldline(zero, m, np.array([2.0, 0.0, 0.0]), +1)
    mc, solc = capacitor2
    line = trace_fieldline(solc, mc, np.array([0.504, 0.0, 0.0]), +1)
    assert line.termination == "SurfaceHit" and np.linalg.norm(line.points[-1]) > 0.95
    assert abs(line.length - 0.496) / 0.496 < 0.02
    line = trace_fieldline(solc, mc, np.array([0.45, 0.35, 0.2]), +1)
    assert line.length >= np.linalg.norm(line.points[-1] - line.points[0]) - 1e-12


def test_floating_conductor_gate_opt_in():
    """Reference semantics: closed floating conductors never pass the true-
    residual gate (SolverError); the opt-in scaled gate converges to the
    direct solution."""
    from conftest import _cfg3_parts
    from paper_2003_12663_b200 import fixtures as F
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.solver import SolverConfig, SolverError, solve

    v, tris = _cfg3_parts(F, 2, 1)
    m = F.mesh_from_parts(v, np.array([t[0] for t in tris]), np.array([t[1] for t in tris]),
                          ["patch 0 electrode 1.0", "patch 1 floating 0", "patch 2 electrode 0.0"])
    A, rhs = assemble(m)
    x = np.linalg.solve(A.toarray(), rhs)
    with pytest.raises(SolverError) as ei:
        solve(A, rhs, SolverConfig(max_iters=300))
    assert ei.value.iterations >= 300 and ei.value.best_residual > 1e-8
    sol = solve(A, rhs, SolverConfig(true_residual_gate=False))
    assert np.max(np.abs(sol.u - x[: m.n_collocation])) <= 1e-6 * np.max(np.abs(x))
    assert abs(sol.V[0] - x[-1]) <= 1e-6 * abs(x[-1])


def test_case_outputs_bitwise_across_blockings(cases, tmp_path):
    """solution.json and surface_field.csv from the device path are
    byte-identical for any row blocking (reference
    tests/test_cli.py:96-108: workers {1, 4}, blocks 3)."""
    from paper_2003_12663_b200 import outputs
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.config import Config
    from paper_2003_12663_b200.postprocess import surface_field_magnitudes
    from paper_2003_12663_b200.solver import solve

    m = cases("diel2")
    got = []
    for blocks in (1, 3):
        out = tmp_path / f"b{blocks}"
        out.mkdir()
        A, rhs = assemble(m, n_blocks=blocks)
        sol = solve(A, rhs)
        e = surface_field_magnitudes(m, sol)
        outputs.write_solution(out, "/case/mesh.bemesh", m, sol, e, Config(), {}, 1, blocks)
        outputs.write_surface_csv(out / "surface_field.csv", m, e)
        got.append(out)
    for name in ("solution.json", "surface_field.csv"):
        assert (got[0] / name).read_bytes() == (got[1] / name).read_bytes()
