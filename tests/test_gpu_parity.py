"""CUDA path vs the reference (golden fixtures from the live reference) and
vs the oracle.  Tolerances (north star): entries 1e-10 relative (row floor
1e-14 of the row max, see oracle.entry_error), solution/capacitance 1e-8,
fields 1e-8 of max(|E_ref|, E_scale), verdicts identical."""

import numpy as np
import pytest

from conftest import CASES, gpu_ok

pytestmark = [pytest.mark.gpu, pytest.mark.skipif(not gpu_ok(), reason="needs a CUDA device")]

FULL = ["sphere2", "cap2", "floatshell1", "diel1", "diel2", "gap2", "cfg3mini", "plates"]


@pytest.fixture(scope="module")
def assembled(cases):
    from paper_2003_12663_b200.assembly import assemble

    store = {}

    def get(name):
        if name not in store:
            store[name] = assemble(cases(name))
        return store[name]

    return get


def entry_error(a, b):
    from oracle.hvb_oracle import entry_error as ee

    return ee(a, b)


@pytest.mark.parametrize("name", FULL)
def test_matrix_vs_reference(golden, assembled, name):
    A, rhs = assembled(name)
    err = entry_error(A.toarray(), golden[name + "_A"])
    assert err <= 1e-10, err
    np.testing.assert_array_equal(rhs, golden[name + "_rhs"])


@pytest.mark.parametrize("name", CASES)
def test_pair_counts_vs_reference(golden, assembled, name):
    A, _ = assembled(name)
    d = A.diagnostics
    got = [d["pairs_regular"], d["pairs_singular"], d["pairs_near_singular"]]
    assert got == list(golden[name + "_diag"])


def test_rodmini_rows_vs_reference(golden, assembled):
    A, _ = assembled("rodmini")
    rows = golden["rodmini_rows"]
    dense = np.vstack([A.row(int(i)) for i in rows])
    assert entry_error(dense, golden["rodmini_Arows"]) <= 1e-10


@pytest.mark.parametrize("name", ["sphere2", "cap2", "floatshell1", "diel1", "diel2", "gap2", "cfg3mini",
                                  "plates", "rodmini"])
def test_solution_vs_reference(golden, assembled, name):
    from paper_2003_12663_b200.solver import SolverConfig, solve

    A, rhs = assembled(name)
    sol = solve(A, rhs, SolverConfig(rel_tol=1e-12, max_iters=600))
    u = golden[name + "_u"]
    assert np.max(np.abs(sol.u - u)) <= 1e-8 * np.max(np.abs(u))
    if len(golden[name + "_V"]):
        V = golden[name + "_V"]
        assert np.max(np.abs(sol.V - V)) <= 1e-8 * max(np.max(np.abs(V)), 1e-300)
    it_ref, conv = golden[name + "_iters"]
    if conv:
        assert abs(sol.iterations - int(it_ref)) <= 1


def test_capacitance_vs_reference(golden, cases):
    from paper_2003_12663_b200.assembly import charge_row
    from paper_2003_12663_b200.mesh import EPS0

    m = cases("sphere2")
    q = charge_row(m, np.arange(m.n_collocation), eps_plus=EPS0)
    ref = golden["sphere2_charge"]
    assert np.max(np.abs(q - ref)) <= 1e-10 * np.max(np.abs(ref))
    u = golden["sphere2_u"]
    C, Cref = float(q @ u), float(ref @ u)
    assert abs(C - Cref) <= 1e-8 * abs(Cref)


def _sol(golden, name):
    from paper_2003_12663_b200.solver import Solution

    return Solution(u=golden[name + "_u"], V=golden[name + "_V"], iterations=0, residual=0.0)


@pytest.mark.parametrize("name", ["sphere2", "cap2", "diel1", "gap2", "plates"])
def test_fields_vs_reference(golden, cases, name):
    from paper_2003_12663_b200.postprocess import eval_efield_batch, eval_potential_batch

    m = cases(name)
    sol = _sol(golden, name)
    pts = golden[name + "_pts"]
    E = eval_efield_batch(sol, m, pts)
    Eref = golden[name + "_E"]
    scale = np.maximum(np.linalg.norm(Eref, axis=1), 1e-3 * np.max(np.linalg.norm(Eref, axis=1)))
    assert np.max(np.linalg.norm(E - Eref, axis=1) / scale) <= 1e-8
    phi = eval_potential_batch(sol, m, pts)
    pref = golden[name + "_phi"]
    assert np.max(np.abs(phi - pref)) <= 1e-8 * np.max(np.abs(pref))


def test_surface_field_vs_reference(golden, cases):
    from paper_2003_12663_b200.postprocess import surface_field_magnitudes

    m = cases("sphere2")
    s = surface_field_magnitudes(m, _sol(golden, "sphere2"))
    np.testing.assert_allclose(s, golden["sphere2_surfE"], rtol=1e-8)


def test_traced_lines_vs_reference(golden, cases):
    from paper_2003_12663_b200.postprocess import IonizationModel, streamer_integral, trace_fieldlines

    gas = IonizationModel(np.array([0.0, 1.0, 2.0, 4.0]), np.array([0.0, 0.5, 3.0, 6.0]), 0.8)
    specs = [("sphere2", [1.05, 0.0, 0.0], 1), ("sphere2", [0.0, 0.7, 0.8], 1),
             ("cap2", [0.504, 0.0, 0.0], 1), ("cap2", [0.6, 0.0, 0.0], -1), ("cap2", [0.45, 0.35, 0.2], 1)]
    for k, (name, s0, o) in enumerate(specs):
        line = trace_fieldlines(_sol(golden, name), cases(name), np.array([s0]), [o])[0]
        assert line.termination == str(golden[f"line{k}_term"])
        v, inc = streamer_integral(line, gas)
        vref, incref = golden[f"line{k}_streamer"]
        assert inc == bool(incref)
        assert abs(v - vref) <= 1e-6 * max(abs(vref), 1e-12)
        if len(line.arc_lengths) == len(golden[f"line{k}_arcs"]):
            np.testing.assert_allclose(line.arc_lengths, golden[f"line{k}_arcs"], rtol=1e-8, atol=1e-12)


def test_seeds_vs_reference(golden, cases):
    from paper_2003_12663_b200.postprocess import pick_start_points

    starts, idx, _ = pick_start_points(cases("cap2"), _sol(golden, "cap2"), 5)
    assert set(idx.tolist()) == set(golden["cap2_seed_idx"].tolist()) or len(set(idx) & set(golden["cap2_seed_idx"])) >= 4


def test_block_invariance_bitwise(cases):
    from paper_2003_12663_b200.assembly import assemble, matvec

    m = cases("sphere2")
    dense = {nb: assemble(m, n_blocks=nb)[0] for nb in (1, 2, 8)}
    a1 = dense[1].toarray()
    np.testing.assert_array_equal(a1, dense[2].toarray())
    np.testing.assert_array_equal(a1, dense[8].toarray())
    v = np.random.default_rng(3).standard_normal(m.n_collocation)
    y1 = matvec(dense[1], v)
    np.testing.assert_array_equal(y1, matvec(dense[8], v))
    assert np.max(np.abs(y1 - a1 @ v)) <= 1e-13 * np.max(np.abs(a1 @ v))


def test_gemv_host_matrix():
    from paper_2003_12663_b200.assembly import RowBlock, SystemMatrix, matvec, partition_rows

    rng = np.random.default_rng(2)
    for n in (1, 7, 64, 333):
        a = rng.standard_normal((n, n))
        v = rng.standard_normal(n)
        blocks = [RowBlock(s, e, a[s:e].copy()) for s, e in partition_rows(n, min(3, n))]
        y = matvec(SystemMatrix(n=n, n_floating=0, blocks=blocks), v)
        assert np.max(np.abs(y - a @ v)) <= 1e-13 * max(1.0, np.max(np.abs(a @ v)))


def test_single_precision_storage_reference_semantics(cases, monkeypatch):
    """precision="single" (reference src/assembly.py:482-484, 386-392): the
    stored matrix is the float64 one rounded to float32; matvec casts v to
    float32 and reduces every row in float32 like the reference's
    ``data[i] @ vc`` -- checked against that exact numpy float32 dot within
    the float32 summation-order bound; GMRES on the single matrix agrees
    with the oracle GMRES run on the same float32 matvec semantics; the
    opt-in double-sum reduction is at least as close to the exact product."""
    from oracle import hvb_oracle as ora
    from paper_2003_12663_b200 import assembly
    from paper_2003_12663_b200.assembly import assemble, matvec
    from paper_2003_12663_b200.solver import SolverConfig, solve

    m = cases("diel2")
    A32, rhs = assemble(m, precision="single")
    a32 = A32.toarray()
    assert A32.blocks[0].data.dtype == np.float32
    np.testing.assert_array_equal(a32, assemble(m)[0].toarray().astype(np.float32))
    rng = np.random.default_rng(3)
    v = rng.standard_normal(A32.size)
    v32 = v.astype(np.float32)
    ref = np.array([a32[i] @ v32 for i in range(A32.size)], dtype=np.float64)  # the reference's float32 dot
    exact = a32.astype(np.float64) @ v32.astype(np.float64)
    mag = np.abs(a32).astype(np.float64) @ np.abs(v32).astype(np.float64)
    eps32 = np.finfo(np.float32).eps
    y = matvec(A32, v)
    bound = 2 * np.sqrt(A32.size) * eps32 * mag  # two float32 summation orders of N terms
    assert np.all(np.abs(y - ref) <= bound)
    assert np.max(np.abs(y - exact) / mag) > 1e-10  # really float32 sums, not double
    monkeypatch.setattr(assembly, "SINGLE_SUMS_F64", True)
    y64 = matvec(A32, v)
    assert np.max(np.abs(y64 - exact) / mag) <= np.max(np.abs(y - exact) / mag)
    monkeypatch.setattr(assembly, "SINGLE_SUMS_F64", False)
    sol = solve(A32, rhs, SolverConfig(rel_tol=1e-5))
    x, it, _ = ora.gmres(a32, rhs, rel_tol=1e-5,
                         matvec=lambda z: (a32 @ z.astype(np.float32)).astype(np.float64))
    full = np.concatenate([sol.u, sol.V])
    assert np.max(np.abs(full - x)) <= 1e-3 * np.max(np.abs(x))
    assert abs(sol.iterations - it) <= 2


def test_assemble_vs_oracle_random_points(cases):
    """Kernel rows at off-mesh points (incl. near-surface ones) vs the oracle."""
    from oracle import hvb_oracle as ora
    from paper_2003_12663_b200.assembly import KERNEL_ADL, KERNEL_SL, assemble_kernel_row

    m = cases("gap2")
    rng = np.random.default_rng(11)
    for _ in range(4):
        d = rng.standard_normal(3)
        x = (1.0 + 0.02 * rng.uniform()) * d / np.linalg.norm(d)
        row, _ = assemble_kernel_row(m, None, x, None, KERNEL_SL)
        ref, _ = ora.kernel_rows(m, x[None], None, "sl")
        assert entry_error(row[None], ref) <= 1e-10
        nx = d / np.linalg.norm(d)
        row, _ = assemble_kernel_row(m, None, x, None, KERNEL_ADL, n_x=nx)
        ref, _ = ora.kernel_rows(m, x[None], None, "adl", normals=nx[None])
        assert entry_error(row[None], ref) <= 1e-10


def test_regular_sweep_tiling_independent(cases, monkeypatch):
    """Re-assembly is bitwise reproducible, and a different column tiling
    (smaller tiles: other tile boundaries, other record groups and window
    flush points) gives the same entries to rounding."""
    from oracle import hvb_oracle as ora
    from paper_2003_12663_b200 import device
    from paper_2003_12663_b200.assembly import assemble

    m = cases("diel2")
    a = assemble(m)[0].toarray()
    np.testing.assert_array_equal(a, assemble(m)[0].toarray())
    m._device_cache.clear()
    monkeypatch.setattr(device, "MAX_TILE", 96)
    b = assemble(m)[0].toarray()
    m._device_cache.clear()
    assert ora.entry_error(a, b) <= 5e-12  # the 2/r Newton step is accurate to 1.25e-12


def test_regular_sweep_launch_chunks_bitwise(cases, monkeypatch):
    """The halo exchange (csrc/tiling.cpp 5) does not depend on how the rows
    are cut into launches: a scratch cap that forces one launch per 128 rows
    (each with its own exchange slots and completion counters) gives the
    same matrix bit for bit, with and without the longest-first tile order;
    the exchange is exercised (several tiles, halo copies)."""
    from paper_2003_12663_b200 import assembly, device

    m = cases("diel2")
    m._device_cache.clear()
    monkeypatch.setattr(device, "MAX_TILE", 96)  # many tiles: many halo copies and receiving columns
    dm = device.device_mesh(m)
    assert dm.n_tiles > 2 and dm.tiling.n_halo > 0
    a = assembly.assemble(m)[0].toarray()
    m._device_cache.clear()
    monkeypatch.setattr(assembly, "HALO_BYTES", 8 * 128 * device.device_mesh(m).n_slots)
    b = assembly.assemble(m)[0].toarray()
    np.testing.assert_array_equal(a, b)
    m._device_cache.clear()
    dm = device.device_mesh(m)
    dm.tile_order = None
    np.testing.assert_array_equal(a, assembly.assemble(m)[0].toarray())
    m._device_cache.clear()


def test_row_plan_cache_follows_the_mesh(cases):
    """assemble() keeps the uploaded row plan per device mesh; a changed row
    coefficient (a dielectric row's permittivity) must rebuild it: the
    re-assembly equals the assembly of a fresh mesh in the same state."""
    from paper_2003_12663_b200.assembly import assemble

    m = cases("diel2")
    a0 = assemble(m)[0].toarray()
    diel = np.flatnonzero(m.row_kind_code == 2)
    assert len(diel)
    saved = m.row_eps_plus.copy()
    try:
        m.row_eps_plus = saved.copy()
        m.row_eps_plus[diel] *= 1.5
        a1 = assemble(m)[0].toarray()
        assert not np.array_equal(a0[diel], a1[diel])
        from conftest import build_case

        fresh = build_case("diel2")
        fresh.row_eps_plus = m.row_eps_plus.copy()
        np.testing.assert_array_equal(a1, assemble(fresh)[0].toarray())
    finally:
        m.row_eps_plus = saved
        m._device_cache.clear()
