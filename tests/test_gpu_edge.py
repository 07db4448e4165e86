"""Edge cases of the device path: empty batches, dimension mismatches,
bad arguments through the C ABI, the LeftDomain / MaxLength terminations,
a one-panel-per-surface mesh, and determinism of repeated launches."""

import numpy as np
import pytest

from conftest import build_case, gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a CUDA device")]


@pytest.fixture(scope="module")
def sphere():
    from paper_2003_12663_b200 import fixtures
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.solver import SolverConfig, solve

    m = fixtures.sphere_mesh(2)
    A, rhs = assemble(m)
    return m, A, rhs, solve(A, rhs, SolverConfig(rel_tol=1e-12))


def test_empty_batches(sphere):
    from paper_2003_12663_b200.postprocess import eval_efield_batch, eval_potential_batch, surface_distance_batch

    m, _, _, sol = sphere
    assert eval_efield_batch(sol, m, np.zeros((0, 3))).shape == (0, 3)
    assert eval_potential_batch(sol, m, np.zeros((0, 3))).shape == (0,)
    d, r = surface_distance_batch(m, np.zeros((0, 3)))
    assert d.shape == (0,) and r.shape == (0,)


def test_dimension_mismatches(sphere):
    from paper_2003_12663_b200.assembly import AssemblyError, assemble, matvec
    from paper_2003_12663_b200.solver import residual, solve

    m, A, rhs, _ = sphere
    with pytest.raises(ValueError):
        matvec(A, np.ones(A.size + 1))
    with pytest.raises(ValueError):
        solve(A, rhs[:-1])
    with pytest.raises(ValueError):
        residual(A, np.ones(3), rhs)
    with pytest.raises(ValueError):
        solve(np.ones((3, 4)), np.ones(3))
    with pytest.raises(AssemblyError):
        assemble(m, precision="half")


def test_c_abi_bad_arguments_raise_value_error():
    import torch

    from paper_2003_12663_b200 import _lib

    with pytest.raises(ValueError, match="split"):
        _lib.call("hvb_field", None, None, None, None, 10, 12, None, None, 1, 0, 0, None, None, None, 0,
                  _lib.stream_ptr())
    with pytest.raises(ValueError, match="nt/nq"):
        _lib.call("hvb_build_table", None, 5, 7, None, None, _lib.stream_ptr())
    torch.cuda.synchronize()


def test_left_domain_and_max_length(sphere):
    from paper_2003_12663_b200.postprocess import TraceParams, trace_fieldlines

    m, _, _, sol = sphere
    lines = trace_fieldlines(sol, m, np.array([[1.3, 0.1, 0.0], [1.3, 0.1, 0.0]]), [1, 1],
                             params=None)
    assert lines[0].termination == "LeftDomain"
    np.testing.assert_array_equal(lines[0].points, lines[1].points)  # identical lines in one batch
    short = trace_fieldlines(sol, m, np.array([[1.3, 0.1, 0.0]]), [1], params=TraceParams(max_length_frac=0.05))[0]
    assert short.termination == "MaxLength"
    # inward orientation from outside the sphere ends on the surface
    hit = trace_fieldlines(sol, m, np.array([[1.3, 0.1, 0.0]]), [-1])[0]
    assert hit.termination == "SurfaceHit" and abs(np.linalg.norm(hit.points[-1]) - 1.0) < 0.02


def test_minimal_mesh_one_panel_per_surface():
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.mesh import parse_mesh
    from paper_2003_12663_b200.solver import SolverConfig, solve

    text = ("bemesh 1\nvertex 0 0 0 0\nvertex 1 1 0 0\nvertex 2 0 1 0\nvertex 3 0.5 0 0\n"
            "vertex 4 0.5 0.5 0\nvertex 5 0 0.5 0\ntriangle 0 1 2 3 4 5 0\npatch 0 electrode 1.0\n")
    m = parse_mesh(text)
    A, rhs = assemble(m)
    sol = solve(A, rhs, SolverConfig(rel_tol=1e-12))
    assert A.shape == (3, 3) and np.all(np.isfinite(sol.u)) and np.all(sol.u > 0)


def test_repeated_launches_bitwise(sphere):
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.postprocess import eval_efield_batch

    m, A, _, sol = sphere
    np.testing.assert_array_equal(A.toarray(), assemble(m)[0].toarray())
    P = np.random.default_rng(4).uniform(-2, 2, (257, 3))
    np.testing.assert_array_equal(eval_efield_batch(sol, m, P), eval_efield_batch(sol, m, P))
    # a point evaluated alone equals the same point inside a batch
    np.testing.assert_array_equal(eval_efield_batch(sol, m, P[100:101])[0], eval_efield_batch(sol, m, P)[100])


def test_surface_field_subset_matches_full(sphere):
    from paper_2003_12663_b200.postprocess import surface_field_magnitudes

    m, _, _, sol = sphere
    full = surface_field_magnitudes(m, sol)
    idx = np.array([5, 0, 77, m.n_collocation - 1])
    np.testing.assert_array_equal(surface_field_magnitudes(m, sol, indices=idx), full[idx])
    assert surface_field_magnitudes(m, sol, indices=np.zeros(0, dtype=int)).shape == (0,)


def test_max_steps_budget_extension(sphere):
    from paper_2003_12663_b200.postprocess import TraceParams, trace_fieldlines

    m, _, _, sol = sphere
    # the inward line from 1.3 R takes many small steps towards the surface
    free = trace_fieldlines(sol, m, np.array([[1.3, 0.1, 0.0]]), [-1])[0]
    assert free.termination == "SurfaceHit" and len(free.points) > 4
    capped = trace_fieldlines(sol, m, np.array([[1.3, 0.1, 0.0]]), [-1], params=TraceParams(max_steps=2))[0]
    assert capped.termination == "MaxSteps" and len(capped.points) <= 3
    np.testing.assert_array_equal(capped.points, free.points[: len(capped.points)])
    # a budget the line never reaches changes nothing (reference semantics)
    big = trace_fieldlines(sol, m, np.array([[1.3, 0.1, 0.0]]), [-1], params=TraceParams(max_steps=10 ** 6))[0]
    np.testing.assert_array_equal(big.points, free.points)
    assert big.termination == free.termination


def test_target_batching_is_invisible(sphere, monkeypatch):
    """Batches larger than TARGET_BATCH run as several launches with the same
    per-target results (including the near pairs of near-surface points)."""
    from paper_2003_12663_b200 import postprocess

    m, _, _, sol = sphere
    rng = np.random.default_rng(9)
    d = rng.standard_normal((300, 3))
    P = np.vstack([rng.uniform(-2, 2, (300, 3)), 1.01 * d / np.linalg.norm(d, axis=1)[:, None]])
    ref = postprocess.eval_efield_batch(sol, m, P)
    monkeypatch.setattr(postprocess, "TARGET_BATCH", 128)
    np.testing.assert_array_equal(postprocess.eval_efield_batch(sol, m, P), ref)


@pytest.mark.parametrize("maker", ["sphere", "rod_plane", "one_panel"])
def test_device_panel_data_matches_host_statement(maker):
    """k_panel_data (ccr, cls, 32-panel group bounds) equals the host
    statement device.py:panel_groups and the numpy bracket bit for bit,
    including a ragged last group; k_build_stream's window slots equal
    l % WINDOW (dump slot WINDOW for corners owned by another tile)."""
    import torch

    from paper_2003_12663_b200 import device, fixtures
    from paper_2003_12663_b200.mesh import parse_mesh
    from paper_2003_12663_b200.quadrature import QuadConfig

    if maker == "sphere":
        m = fixtures.sphere_mesh(2)
    elif maker == "rod_plane":
        m = fixtures.rod_plane_mesh(0.1)
    else:
        m = parse_mesh("bemesh 1\nvertex 0 0 0 0\nvertex 1 1 0 0\nvertex 2 0 1 0\nvertex 3 0.5 0 0\n"
                       "vertex 4 0.5 0.5 0\nvertex 5 0 0.5 0\ntriangle 0 1 2 3 4 5 0\npatch 0 electrode 1.0\n")
    cfg = QuadConfig()
    dm = device.DeviceMesh(m, cfg, torch.device("cuda:0"))
    thr = cfg.eta * m.circumradii
    cls = np.column_stack([m.circumcenters, thr, thr * thr * (1 - 1e-13), thr * thr * (1 + 1e-13)])
    assert np.array_equal(dm.cls.cpu().numpy(), cls)
    assert np.array_equal(dm.ccr.cpu().numpy(), np.column_stack([m.circumcenters, m.circumradii]))
    assert np.array_equal(dm.groups.cpu().numpy(), device.panel_groups(m.circumcenters, m.circumradii, thr))
    # record tails (both stream formats): circumcircle bracket and window slots
    loc = dm.tiling.ent_meta[:, 1:4].astype(np.int64)
    real = dm.tiling.ent_tri >= 0                     # dummy records (-1) pad short stages
    ent = dm.tiling.ent_tri[real].astype(np.int64)
    for mode in (0, 1):
        rec = dm.stream_for(mode).cpu().numpy()
        assert np.array_equal(rec[real][:, -8:-5], m.circumcenters[ent])
        tail = np.ascontiguousarray(rec[:, -2:])
        offs = tail.view(np.uint16).reshape(len(rec), 8)[:, 4:7].astype(np.int64)
        assert np.array_equal(offs, np.where(loc >= 0, loc % dm.window, dm.window) * dm.window_stride * 8)
        flags = tail.view(np.uint16).reshape(len(rec), 8)[:, 7]
        assert not np.any(flags[~real])
    # SL stream nodes: x'.Y + |x'|^2 Q + P = |x - y|^2 / w^2 (csrc/assemble.cu)
    nq = dm.nq
    tab = dm.table.cpu().numpy()[ent]                     # (ne, nq, 6): y, w hat_c
    y, w = tab[:, :, :3], tab[:, :, 3:].sum(axis=2)
    rec = dm.stream_for(0).cpu().numpy()[real]
    pairs = rec[:, :5 * ((nq + 1) & ~1)].reshape(len(rec), -1, 10)
    Y = np.concatenate([pairs[:, :, None, 0:3], pairs[:, :, None, 6:9]], axis=2).reshape(len(rec), -1, 3)[:, :nq]
    P = np.stack([pairs[:, :, 3], pairs[:, :, 9]], axis=2).reshape(len(rec), -1)[:, :nq]
    Q = np.stack([pairs[:, :, 4], pairs[:, :, 5]], axis=2).reshape(len(rec), -1)[:, :nq]
    x = m.vertices.max(axis=0) + 0.5 * np.ptp(m.vertices, axis=0)   # a far point
    xc = x[None, :] - m.circumcenters[ent]
    r2 = np.einsum("ed,eqd->eq", xc, Y) + np.sum(xc * xc, axis=1)[:, None] * Q + P
    ref = np.sum((x[None, None, :] - y) ** 2, axis=2) / (w * w)
    assert np.max(np.abs(r2 - ref) / ref) <= 1e-13
    assert dm.h2d_bytes > m.tri_nodes.nbytes


@pytest.mark.parametrize("n,j", [(1, 0), (1000, 5), (99558, 40), (16 * 1024 * 8, 3), (16 * 1024 * 8 + 7, 3)])
def test_mgs_matches_host_gram_schmidt(n, j):
    """hvb_mgs (cluster kernel up to 16*1024*8 entries, cooperative kernel
    beyond) against modified Gram-Schmidt in float64 numpy, with the
    re-orthogonalisation pass (accumulate) and a bitwise repeat."""
    import torch

    from paper_2003_12663_b200 import _lib

    rng = np.random.default_rng(n + j)
    Q, _ = np.linalg.qr(rng.standard_normal((n, j + 1))) if n > j else (np.eye(n, j + 1), None)
    V = torch.tensor(np.ascontiguousarray(Q.T), device="cuda:0")
    w0 = rng.standard_normal(n)
    partial = torch.empty(_lib.lib().hvb_mgs_partial_size(), dtype=torch.float64, device="cuda:0")

    def run(accumulate, w, h):
        norms = torch.empty(2, dtype=torch.float64, device="cuda:0")
        _lib.call("hvb_mgs", _lib.ptr(V), n, j, _lib.ptr(w), n, _lib.ptr(h), _lib.ptr(norms), _lib.ptr(partial),
                  accumulate, _lib.stream_ptr())
        return norms.cpu().numpy()

    w = torch.tensor(w0, device="cuda:0")
    h = torch.zeros(j + 1, dtype=torch.float64, device="cuda:0")
    nrm = run(0, w, h)
    nrm2 = run(1, w, h)
    # host statement
    wh = w0.copy()
    hh = np.zeros(j + 1)
    for _ in range(2):
        for i in range(j + 1):
            c = Q[:, i] @ wh
            hh[i] += c
            wh -= c * Q[:, i]
    scale = np.linalg.norm(w0)
    assert np.allclose(h.cpu().numpy(), hh, rtol=0, atol=1e-12 * scale)
    assert np.allclose(w.cpu().numpy(), wh, rtol=0, atol=1e-12 * scale)
    assert abs(nrm[0] - scale) <= 1e-13 * scale and abs(nrm2[1] - np.linalg.norm(wh)) <= 1e-12 * scale
    # bitwise repeat
    w2 = torch.tensor(w0, device="cuda:0")
    h2 = torch.zeros(j + 1, dtype=torch.float64, device="cuda:0")
    run(0, w2, h2)
    run(1, w2, h2)
    assert torch.equal(w2, w) and torch.equal(h2, h)


def test_host_block_replacement_reuploads():
    """A host-backed SystemMatrix re-uploads a block whose data was replaced
    (the reference reads its blocks on every matvec)."""
    from paper_2003_12663_b200.assembly import RowBlock, SystemMatrix, matvec

    rng = np.random.default_rng(5)
    A = rng.standard_normal((6, 6))
    m = SystemMatrix(n=6, n_floating=0, blocks=[RowBlock(0, 3, A[:3].copy()), RowBlock(3, 6, A[3:].copy())])
    v = rng.standard_normal(6)
    np.testing.assert_allclose(matvec(m, v), A @ v, rtol=1e-13)
    B = rng.standard_normal((3, 6))
    m.blocks[1].data = B
    np.testing.assert_allclose(matvec(m, v), np.concatenate([A[:3] @ v, B @ v]), rtol=1e-13)


def test_field_sources_follow_in_place_density_edits(cases):
    """Editing solution.u in place (past index 2) re-uploads u AND rebuilds
    the density-contracted sources: the far field and the near pass both
    use the new density (a stale source cache mixed densities)."""
    from paper_2003_12663_b200.assembly import assemble
    from paper_2003_12663_b200.postprocess import eval_efield_batch
    from paper_2003_12663_b200.solver import Solution, SolverConfig, solve

    m = cases("cap2")
    A, rhs = assemble(m)
    sol = solve(A, rhs, SolverConfig(rel_tol=1e-12))
    P = np.array([[0.7, 0.1, 0.05], [0.0, 0.62, 0.1]])
    eval_efield_batch(sol, m, P)
    sol.u[7:] *= 1.5
    got = eval_efield_batch(sol, m, P)
    fresh = eval_efield_batch(Solution(u=sol.u.copy(), V=sol.V, iterations=0, residual=0.0), m, P)
    np.testing.assert_array_equal(got, fresh)
