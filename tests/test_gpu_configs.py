"""BASELINE.json configs 1-3 at their full sizes on the GPU against the CPU
oracle (pinned to the reference, tests/test_oracle_golden.py): sampled
matrix rows (including dielectric ADL rows and the floating neutrality
structure), the solve, and the config-1 capacitance.

cfg1: unit sphere, icosphere L4 (5,120 panels, N = 2,562).
cfg2: concentric 0.5 / 0.75 (dielectric shell) / 1.0, L4 (15,360 panels).
cfg3: driven + floating spheres in a grounded enclosure (46,080 panels,
      N = 23,047; the reference's own GMRES cannot pass its true-residual
      gate here -- SURVEY 0.4 -- so the solve uses the opt-in scaled gate and
      is checked by its residual)."""

import numpy as np
import pytest

from conftest import _cfg3_parts, gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a CUDA device")]


def _rows_vs_oracle(m, A, rows):
    from oracle import hvb_oracle as ora

    got = np.array([A.row(int(r)) for r in rows])
    ref = ora.row_equations(m, [int(r) for r in rows])
    return ora.entry_error(got, ref)


def test_cfg1_sphere_capacitance():
    from oracle import hvb_oracle as ora
    from paper_2003_12663_b200 import fixtures
    from paper_2003_12663_b200.assembly import assemble, charge_row
    from paper_2003_12663_b200.mesh import EPS0
    from paper_2003_12663_b200.solver import SolverConfig, solve

    m = fixtures.sphere_mesh(4)
    assert m.n_triangles == 5120 and m.n_collocation == 2562
    A, rhs = assemble(m)
    assert _rows_vs_oracle(m, A, np.linspace(0, m.n_collocation - 1, 24).astype(int)) <= 1e-10
    sol = solve(A, rhs)  # reference defaults
    assert sol.iterations > 0 and abs(np.mean(sol.u) - 1.0) < 1e-3  # sigma = V0 / R (kernel 1 / 4 pi r)
    q = charge_row(m, np.arange(m.n_collocation), eps_plus=EPS0)
    C = float(q @ sol.u) / 1.0
    assert abs(C - 4 * np.pi * EPS0) / (4 * np.pi * EPS0) < 1e-3  # discretisation error at L4
    idx = np.linspace(0, m.n_collocation - 1, 8).astype(int)
    qref = ora.charge_vector(m, idx, EPS0, 0.5 * EPS0)
    qsub = charge_row(m, idx, eps_plus=EPS0)
    assert np.max(np.abs(qsub - qref)) <= 1e-10 * np.max(np.abs(qref))
    tight = solve(A, rhs, SolverConfig(rel_tol=1e-12))
    x = np.linalg.solve(A.toarray(), rhs)
    assert np.max(np.abs(tight.u - x)) <= 1e-8 * np.max(np.abs(x))


def test_cfg2_dielectric_shell():
    from paper_2003_12663_b200 import fixtures
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.mesh import EPS0
    from paper_2003_12663_b200.solver import residual, solve

    m = fixtures.concentric_mesh(4, [(0.5, "electrode 1.0"), (0.75, f"dielectric {EPS0!r} {2 * EPS0!r}"),
                                     (1.0, "electrode 0.0")])
    assert m.n_triangles == 15360
    A, rhs = assemble(m)
    diel = np.nonzero(m.row_kind_code == 2)[0]
    rows = np.concatenate([np.linspace(0, m.n_collocation - 1, 12).astype(int), diel[:: len(diel) // 8][:8]])
    assert _rows_vs_oracle(m, A, rows) <= 1e-10
    sol = solve(A, rhs)
    assert residual(A, np.concatenate([sol.u, sol.V]), rhs) <= 1e-8


def test_cfg3_floating_conductor():
    from paper_2003_12663_b200 import fixtures
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.solver import SolverConfig, solve

    v, tris = _cfg3_parts(fixtures, 5, 4)
    m = fixtures.mesh_from_parts(v, np.array([t[0] for t in tris]), np.array([t[1] for t in tris]),
                                 ["patch 0 electrode 1.0", "patch 1 floating 0", "patch 2 electrode 0.0"])
    assert m.n_triangles == 46080 and m.n_collocation + m.n_floating == 23047
    A, rhs = assemble(m)
    n = m.n_collocation
    fl = np.nonzero(m.row_kind_code == 1)[0]
    rows = np.concatenate([np.linspace(0, n - 1, 10).astype(int), fl[:: len(fl) // 6][:6]])
    assert _rows_vs_oracle(m, A, rows) <= 1e-10
    # floating rows carry -1 in the floating column; the neutrality row sums
    # weighted ADL rows of the floating surface's members (reference 441-468)
    for r in fl[:3]:
        assert A.row(int(r))[n] == -1.0
    neut = A.row(n)
    assert np.count_nonzero(neut[:n]) > 0 and neut[n] == 0.0
    sol = solve(A, rhs, SolverConfig(true_residual_gate=False, max_iters=400))
    Ad = A.toarray()
    res = np.linalg.norm(rhs - Ad @ np.concatenate([sol.u, sol.V])) / np.linalg.norm(rhs)
    assert res <= 1e-6
    assert 0.2 < sol.V[0] < 0.5  # the floating sphere settles between 1 V and ground


def test_cfg4_full_size_sampled_rows_and_solve():
    """Config 4 at the benchmark size (199,104 panels, N = 99,558, 79 GB):
    evenly spaced rows, dielectric (ADL) rows and rows with deferred near
    pairs against the oracle (the oracle cannot hold the matrix: SURVEY
    8c), and the reference-semantics solve's true residual."""
    from paper_2003_12663_b200 import assembly, fixtures
    from paper_2003_12663_b200.solver import solve

    m = fixtures.rod_plane_mesh(1.0)
    assert m.n_triangles == 199104 and m.n_collocation == 99558
    A, rhs = assembly.assemble(m)
    near = assembly.LAST_NEAR_ROWS
    n = m.n_collocation
    diel = np.nonzero(m.row_kind_code == 2)[0]
    rows = [np.linspace(0, n - 1, 48).astype(int), diel[:: max(1, len(diel) // 12)][:12]]
    if near is not None and np.any(near > 0):
        nr = np.nonzero(near > 0)[0]
        rows.append(nr[:: max(1, len(nr) // 12)][:12])
    rows = np.unique(np.concatenate(rows))
    assert _rows_vs_oracle(m, A, rows) <= 1e-10
    sol = solve(A, rhs)
    assert sol.iterations > 0 and sol.residual <= 1e-8
