"""Config-4 geometry (rod-plane + insulator, scaled to ~18k panels) on the
GPU against the CPU oracle (oracle/hvb_oracle.py, pinned to the reference in
tests/test_oracle_golden.py and tests/test_trace.py): sampled matrix rows
(SL, dielectric ADL and rows with deferred near pairs), the solve's
residual, fields at random and near-surface points, and traced lines
(termination, point count, streamer verdict)."""

import numpy as np
import pytest

from conftest import gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a CUDA device")]

SCALE = 0.3


@pytest.fixture(scope="module")
def rp():
    from paper_2003_12663_b200 import assembly, fixtures
    from paper_2003_12663_b200.solver import SolverConfig, solve

    m = fixtures.rod_plane_mesh(SCALE)
    A, rhs = assembly.assemble(m)
    near_rows = assembly.LAST_NEAR_ROWS
    sol = solve(A, rhs, SolverConfig())
    return m, A, rhs, sol, near_rows


def test_rows_vs_oracle(rp):
    from oracle import hvb_oracle as ora

    m, A, _, _, near_rows = rp
    n = m.n_collocation
    diel = np.nonzero(m.row_kind_code == 2)[0]
    rows = list(np.linspace(0, n - 1, 10).astype(int)) + list(diel[:: max(1, len(diel) // 6)][:6])
    if near_rows is not None:
        rows += list(np.nonzero(near_rows > 0)[0][:6])
    rows = sorted(set(int(r) for r in rows))
    got = np.array([A.row(r) for r in rows])
    ref = ora.row_equations(m, rows)
    assert ora.entry_error(got, ref) <= 1e-10


def test_solution_residual(rp):
    from paper_2003_12663_b200.solver import residual

    m, A, rhs, sol, _ = rp
    assert sol.iterations > 0
    assert residual(A, np.concatenate([sol.u, sol.V]), rhs) <= 1e-8


def test_fields_vs_oracle(rp):
    from oracle import hvb_oracle as ora
    from paper_2003_12663_b200.postprocess import eval_efield_batch

    m, _, _, sol, _ = rp
    rng = np.random.default_rng(7)
    lo, hi = m.bounding_box()
    P = 0.5 * (lo + hi) + rng.uniform(-0.6, 0.6, (6, 3)) * (hi - lo)
    i = rng.integers(0, m.n_collocation, 4)
    P = np.vstack([P, m.colloc_points[i] + 0.004 * m.colloc_normals[i]])  # near-surface: deferred pairs
    E = eval_efield_batch(sol, m, P)
    Eref = ora.efield_points(m, sol.u, P)
    scale = np.maximum(np.linalg.norm(Eref, axis=1), 1e-3 * np.max(np.linalg.norm(Eref, axis=1)))
    assert np.max(np.linalg.norm(E - Eref, axis=1) / scale) <= 1e-8


def test_traced_lines_vs_oracle(rp):
    from oracle import hvb_oracle as ora
    from paper_2003_12663_b200.postprocess import (eval_efield_batch, load_ionization_model, pick_start_points,
                                                   streamer_integral, trace_fieldlines)

    m, _, _, sol, _ = rp
    import os

    gas = load_ionization_model(os.path.join(os.path.dirname(__file__), "..", "paper_2003_12663_b200", "data",
                                             "air_demo.gas"))
    starts, idx, _ = pick_start_points(m, sol, 64)
    pick = [0, 21, 42]
    starts, idx = starts[pick], idx[pick]
    E0 = eval_efield_batch(sol, m, starts)
    orient = np.where(np.einsum("ij,ij->i", E0, m.colloc_normals[idx]) >= 0, 1, -1)
    lines = trace_fieldlines(sol, m, starts, orient)
    diag = float(np.linalg.norm(np.ptp(m.vertices, axis=0)))
    for ln, x0, o in zip(lines, starts, orient):
        pts, mags, arcs, term = ora.trace_line(m, sol.u, x0, int(o))
        assert ln.termination == term
        assert len(ln.arc_lengths) == len(arcs)
        assert np.max(np.abs(ln.points - pts)) <= 1e-8 * diag
        v, inc = streamer_integral(ln, gas)
        vr, ir = ora.streamer(arcs, mags, gas.e_values, gas.alpha_values, gas.k_str)
        assert inc == ir and abs(v - vr) <= 1e-8 * max(abs(vr), 1e-300)
