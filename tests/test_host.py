"""CPU tests of the host layer: C-ABI library, config, row partition,
column tiling invariants, quadrature rules and decisions, mesh validation,
streamer / ionization / CSV (reference semantics, tests/test_*.py)."""

import math
import os
import re

import numpy as np
import pytest

from paper_2003_12663_b200 import config, fixtures, quadrature
from paper_2003_12663_b200.mesh import EPS0, MeshError, parse_mesh

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


# ---------------------------------------------------------------------------
# C ABI
# ---------------------------------------------------------------------------


def _header_functions():
    text = open(os.path.join(ROOT, "include", "hvb.h")).read()
    return sorted(set(re.findall(r"^(?:int|long long|const char\*)\s+(hvb_\w+)\(", text, flags=re.M)))


def test_library_exports_every_header_symbol():
    import ctypes

    import __graft_entry__

    __graft_entry__.build()
    lib = ctypes.CDLL(__graft_entry__.LIB)
    names = _header_functions()
    assert len(names) >= 20
    for name in names:
        assert hasattr(lib, name), name
    lib.hvb_version.restype = ctypes.c_int
    assert lib.hvb_version() == 1


def test_binding_signatures_cover_header():
    from paper_2003_12663_b200 import _lib

    declared = set(_header_functions()) - {"hvb_last_error", "hvb_version", "hvb_line_state_bytes",
                                           "hvb_mgs_partial_size", "hvb_ipc_handle_bytes",
                                           "hvb_stream_record_doubles", "hvb_sweep_sched_ints"}
    assert declared == set(_lib.SIGNATURES)


def test_device_entry_points_fail_loudly_without_gpu():
    import torch

    from paper_2003_12663_b200 import _lib
    from paper_2003_12663_b200.assembly import assemble

    if torch.cuda.is_available():
        pytest.skip("GPU present")
    with pytest.raises(_lib.DeviceUnavailable):
        assemble(fixtures.sphere_mesh(1))


# ---------------------------------------------------------------------------
# config / partition
# ---------------------------------------------------------------------------


def test_config_defaults_and_overrides(tmp_path):
    c = config.Config()
    assert c["quad.eta"] == 1.2 and c["solver.restart"] == 100
    p = tmp_path / "run.cfg"
    p.write_text("# comment\nquad.eta = 1.5\nsolver.row_equilibrate = off\n")
    c = config.Config.load(p, overrides=["solver.rel_tol=1e-10"])
    assert c["quad.eta"] == 1.5 and c["solver.row_equilibrate"] is False and c["solver.rel_tol"] == 1e-10
    assert c.quad().eta == 1.5
    assert c.solver().rel_tol == 1e-10
    assert c.trace_params().rel_tol == 1e-6
    with pytest.raises(KeyError):
        config.Config({"quad.nope": 1})
    with pytest.raises(ValueError):
        c.set("solver.verbose", "maybe")


def test_partition_rows_reference_semantics():
    from paper_2003_12663_b200.assembly import partition_rows

    assert partition_rows(10, 3) == [(0, 4), (4, 7), (7, 10)]
    assert partition_rows(10, 1) == [(0, 10)]
    assert partition_rows(5, 5) == [(i, i + 1) for i in range(5)]
    with pytest.raises(ValueError):
        partition_rows(4, 5)


def test_solver_config_validation():
    from paper_2003_12663_b200.solver import SolverConfig

    with pytest.raises(ValueError):
        SolverConfig(restart=0)
    with pytest.raises(ValueError):
        SolverConfig(rel_tol=2.0)


# ---------------------------------------------------------------------------
# column tiling (device column order) invariants
# ---------------------------------------------------------------------------


# ---------------------------------------------------------------------------
# quadrature (reference tests/test_quadrature.py semantics)
# ---------------------------------------------------------------------------


@pytest.mark.parametrize("order", [2, 4, 6, 8])
def test_rules_exact(order):
    r = quadrature.regular_rule(order)
    assert abs(r.weights.sum() - 0.5) < 5e-15
    u, v = r.nodes[:, 0], r.nodes[:, 1]
    for i in range(order + 1):
        for j in range(order + 1 - i):
            exact = math.factorial(i) * math.factorial(j) / math.factorial(i + j + 2)
            assert abs(np.sum(r.weights * u ** i * v ** j) - exact) < 5e-15
    assert np.all(u >= 0) and np.all(v >= 0) and np.all(u + v <= 1)


def test_unsupported_order():
    with pytest.raises(quadrature.QuadratureError):
        quadrature.regular_rule(5)
    with pytest.raises(quadrature.QuadratureError):
        quadrature.duffy_rule(0, 1)
    with pytest.raises(quadrature.QuadratureError):
        quadrature.duffy_rule(3, 6)


def test_duffy_corner_singular_reference_value():
    # CORNER_SINGULAR_REF of the reference tests: int 1/|y| over the unit
    # right triangle from corner 0 = sqrt(2) asinh(1)
    r = quadrature.duffy_rule(0, 8)
    got = float(np.sum(r.weights / np.hypot(r.nodes[:, 0], r.nodes[:, 1])))
    assert abs(got - math.sqrt(2.0) * math.asinh(1.0)) < 1e-8
    assert abs(r.weights.sum() - 0.5) < 1e-14


def test_rules_match_reference_golden(golden):
    for c in range(3):
        r = quadrature.duffy_rule(c, 6)
        np.testing.assert_array_equal(r.nodes, golden[f"duffy{c}_nodes"])
        np.testing.assert_array_equal(r.weights, golden[f"duffy{c}_weights"])
    g = quadrature.graded_rule(3, 8, 8)
    np.testing.assert_array_equal(g.nodes, golden["graded_nodes"])
    np.testing.assert_array_equal(g.weights, golden["graded_weights"])


def test_closest_point_decisions_match_reference(golden):
    for row in golden["closest_cases"]:
        cs = row[:9].reshape(3, 3)
        assert quadrature.closest_point_flat(row[9:12], cs) == (row[12], row[13])


NEAR_REFS = {0.1: 2.006576943826, 0.3: 1.437278726277, 0.6: 0.959761111114, 1.0: 0.645094888525}


def test_near_singular_rule_accuracy_and_reference_nodes(golden):
    corners = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    from paper_2003_12663_b200.mesh import _flat_circumcircle

    c, R = _flat_circumcircle(corners)

    class Tri:
        nodes = np.vstack([corners, 0.5 * (corners[0] + corners[1]), 0.5 * (corners[1] + corners[2]),
                           0.5 * (corners[2] + corners[0])])
        circumradius = R

    for frac, ref in NEAR_REFS.items():
        x = corners.mean(axis=0) + np.array([0.0, 0.0, frac * R])
        rule = quadrature.near_singular_rule(x, Tri)
        pts = corners[0] + np.outer(rule.nodes[:, 0], corners[1]) + np.outer(rule.nodes[:, 1], corners[2])
        got = float(np.sum(rule.weights / np.linalg.norm(pts - x, axis=1)))
        assert abs(got - ref) / ref <= 1e-5
        np.testing.assert_allclose(rule.nodes, golden[f"near_{frac}_nodes"], atol=1e-15, rtol=0)


def test_subdivide_partitions_area():
    rng = np.random.default_rng(0)
    for _ in range(200):
        u, v = rng.uniform(0, 1, 2)
        if u + v > 1:
            u, v = 1 - u, 1 - v
        subs = quadrature.subdivide_at((u, v))
        area = sum(0.5 * abs((s.corners[1][0] - s.corners[0][0]) * (s.corners[2][1] - s.corners[0][1])
                             - (s.corners[1][1] - s.corners[0][1]) * (s.corners[2][0] - s.corners[0][0]))
                   for s in subs)
        assert abs(area - 0.5) < 1e-12
    assert len(quadrature.subdivide_at((0.0, 0.0))) == 1
    assert len(quadrature.subdivide_at((0.5, 0.0))) == 2
    assert len(quadrature.subdivide_at((0.2, 0.3))) == 3


def test_classify_pair_conformance():
    rng = np.random.default_rng(123)
    from paper_2003_12663_b200.mesh import CurvedTriangle, flat_circumcircles

    for _ in range(2000):
        cs = rng.uniform(-1, 1, (3, 3))
        cc, r = flat_circumcircles(cs[None])
        tri = CurvedTriangle(0, (0, 1, 2), (3, 4, 5), 0, np.vstack([cs, cs]), cc[0], float(r[0]))
        if rng.uniform() < 0.3:
            vid = int(rng.integers(0, 3))
            assert quadrature.classify_pair(cs[vid], vid, tri).is_singular
        else:
            p = rng.uniform(-2, 2, 3)
            want = "regular" if np.linalg.norm(p - cc[0]) > 1.2 * r[0] else "near_singular"
            got = quadrature.classify_pair(p, 999, tri).kind
            d = np.linalg.norm(p - cc[0])
            if abs(d - 1.2 * r[0]) > 1e-12:
                assert got == want


# ---------------------------------------------------------------------------
# mesh parsing / validation (reference tests/test_mesh.py messages)
# ---------------------------------------------------------------------------

FLAT = ("bemesh 1\nvertex 0 0 0 0\nvertex 1 1 0 0\nvertex 2 0 1 0\nvertex 3 0.5 0 0\n"
        "vertex 4 0.5 0.5 0\nvertex 5 0 0.5 0\ntriangle 0 1 2 3 4 5 0\npatch 0 electrode 1.0\n")


def test_parse_smallest_mesh():
    m = parse_mesh(FLAT)
    assert m.n_collocation == 3 and m.n_triangles == 1
    assert abs(m.total_area() - 0.5) < 1e-14


@pytest.mark.parametrize("text,frag", [
    (FLAT.replace("triangle 0 1 2 3 4 5 0", "triangle 0 1 2 3 4 999 0"), "references vertex 999"),
    ("vertex 0 0 0 0\n", "bemesh 1"),
    (FLAT.replace("patch 0 electrode 1.0", "patch 7 electrode 1.0"), "unknown patch tag 0"),
    (FLAT.replace("vertex 2 0 1 0", "vertex 2 2 0 0"), "degenerate triangle"),
    (FLAT + "vertex 6 3 3 3\n", "belongs to no triangle"),
    (FLAT.replace("patch 0 electrode 1.0", "patch 0 bogus 1.0"), "unknown patch kind"),
])
def test_parse_errors(text, frag):
    with pytest.raises(MeshError, match=frag):
        parse_mesh(text)


def test_triple_junction_rejected():
    v, tris = fixtures.sphere_mesh_parts(1)
    ids = np.array([t[0] for t in tris])
    tags = np.array([0 if k < len(tris) // 2 else 1 for k in range(len(tris))])
    with pytest.raises(MeshError, match="triple junctions"):
        fixtures.mesh_from_parts(v, ids, tags, ["patch 0 dielectric 1.0 2.0", "patch 1 dielectric 1.0 3.0"])


def test_priority_electrode_over_dielectric():
    v, tris = fixtures.sphere_mesh_parts(1)
    ids = np.array([t[0] for t in tris])
    tags = np.array([0 if k < len(tris) // 2 else 1 for k in range(len(tris))])
    m = fixtures.mesh_from_parts(v, ids, tags, ["patch 0 electrode 2.0", "patch 1 dielectric 1.0 3.0"])
    from paper_2003_12663_b200.mesh import Dirichlet, DielectricJump

    kinds = m.row_kinds
    assert any(isinstance(k, Dirichlet) for k in kinds) and any(isinstance(k, DielectricJump) for k in kinds)


def test_relative_permittivity_and_roundtrip(tmp_path):
    from paper_2003_12663_b200.mesh import load_mesh, save_mesh

    m = parse_mesh(FLAT.replace("patch 0 electrode 1.0", "permittivity relative\npatch 0 dielectric 2.0 1.0"))
    assert m.patches[0].eps_plus == 2.0 * EPS0
    p = tmp_path / "m.bemesh"
    save_mesh(fixtures.sphere_mesh(1), p)
    again = load_mesh(p)
    np.testing.assert_array_equal(again.vertices, fixtures.sphere_mesh(1).vertices)


def test_lumped_weights_partition_area():
    m = fixtures.sphere_mesh(2)
    assert abs(m.total_area() - 4 * math.pi) / (4 * math.pi) < 5e-3
    assert np.all(m.lumped_weights > 0)
    assert np.allclose(np.linalg.norm(m.colloc_normals, axis=1), 1.0)


def test_rod_plane_generator_config4():
    m = fixtures.rod_plane_mesh(1.0)
    assert 1.9e5 <= m.n_triangles <= 2.1e5
    assert m.n_floating == 0
    kinds = np.bincount(m.row_kind_code, minlength=3)
    assert kinds[0] > 0 and kinds[2] > 0 and kinds[1] == 0


# ---------------------------------------------------------------------------
# streamer / ionization / field lines / CSV
# ---------------------------------------------------------------------------


def _straight(length=2.0, n=5, e=7.0):
    from paper_2003_12663_b200.postprocess import FieldLine

    s = np.linspace(0, length, n)
    return FieldLine(np.column_stack([s, 0 * s, 0 * s]), np.full(n, e), s, "MaxLength")


def test_streamer_integral():
    from paper_2003_12663_b200.postprocess import IonizationModel, streamer_integral

    line = _straight()
    v, inc = streamer_integral(line, IonizationModel(np.array([0.0, 100.0]), np.array([5.0, 5.0]), 9.99))
    assert abs(v - 10.0) < 1e-12 and inc
    _, inc = streamer_integral(line, IonizationModel(np.array([0.0, 100.0]), np.array([5.0, 5.0]), 10.01))
    assert not inc
    with pytest.raises(ValueError):
        IonizationModel(np.array([1.0, 1.0]), np.array([0.0, 1.0]), 1.0)


def test_fieldline_validation_and_csv(tmp_path):
    from paper_2003_12663_b200.postprocess import FieldLine, IonizationModel, load_ionization_model, write_fieldline_csv

    with pytest.raises(ValueError):
        FieldLine(np.zeros((2, 3)), np.zeros(2), np.zeros(2), "MaxLength")
    p = tmp_path / "gas.txt"
    p.write_text("# gas\n0.0 0.0\n2e6 10.0\nkstr 9.15\n")
    model = load_ionization_model(p)
    assert model.k_str == 9.15 and model.alpha(1e6) == pytest.approx(5.0) and model.alpha(4e6) == 10.0
    q = tmp_path / "line.csv"
    write_fieldline_csv(_straight(), IonizationModel(np.array([0.0, 100.0]), np.array([5.0, 5.0]), 1.0), q)
    rows = q.read_text().strip().splitlines()
    assert rows[0] == "x,y,z,s,E,alpha,cumulative_integral" and float(rows[-1].split(",")[6]) == pytest.approx(10.0)


def test_demo_gas_file_shipped():
    from paper_2003_12663_b200.postprocess import load_ionization_model

    m = load_ionization_model(os.path.join(ROOT, "paper_2003_12663_b200", "data", "air_demo.gas"))
    assert m.k_str == 9.15 and len(m.e_values) == 9


def test_line_state_layout_matches_library():
    import ctypes

    import __graft_entry__
    from paper_2003_12663_b200.tracer import LINE_STATE_DTYPE

    __graft_entry__.build()
    lib = ctypes.CDLL(__graft_entry__.LIB)
    lib.hvb_line_state_bytes.restype = ctypes.c_int
    assert lib.hvb_line_state_bytes() == LINE_STATE_DTYPE.itemsize


def test_public_api_mirrors_reference_init():
    """Every name the reference package exports (src/__init__.py:8-64) is
    importable from the drop-in package root."""
    import paper_2003_12663_b200 as pkg

    names = ["EPS0", "CurvedTriangle", "DielectricJump", "Dirichlet", "FloatingDirichlet", "MeshError", "PatchSpec",
             "SurfaceMesh", "Vertex", "classify_vertex", "load_mesh", "map_reference", "parse_mesh", "save_mesh",
             "surface_frame", "PairClass", "QuadConfig", "Rule", "classify_pair", "closest_point", "duffy_rule",
             "near_singular_rule", "regular_rule", "subdivide_at", "SingularEvaluation", "adl_kernel",
             "efield_kernel", "sl_kernel", "AssemblyError", "Neutrality", "SystemMatrix", "assemble", "charge_row",
             "load_matrix", "matvec", "partition_rows", "save_matrix", "Solution", "SolverConfig", "SolverError",
             "residual", "solve", "FieldLine", "IonizationModel", "TraceError", "TraceParams", "eval_efield",
             "eval_potential", "load_ionization_model", "pick_start_points", "streamer_integral",
             "surface_field_magnitudes", "trace_fieldline", "Config"]
    missing = [n for n in names if not hasattr(pkg, n)]
    assert not missing, missing
    assert pkg.__version__ == "0.1.0"


def test_import_alias_drop_in():
    """INTEGRATION.md's alias: `hvbem` and its submodules resolve to the
    drop-in, with the names the reference's tests import."""
    import importlib
    import sys

    saved = {k: v for k, v in sys.modules.items() if k == "hvbem" or k.startswith("hvbem.")}
    try:
        sys.modules["hvbem"] = importlib.import_module("paper_2003_12663_b200")
        for sub in ("mesh", "quadrature", "kernels", "assembly", "solver", "postprocess", "fixtures", "config", "cli"):
            sys.modules[f"hvbem.{sub}"] = importlib.import_module(f"paper_2003_12663_b200.{sub}")
        from hvbem.assembly import (KERNEL_ADL, KERNEL_SL, AssemblyError, RowBlock, SystemMatrix,  # noqa: F401
                                    assemble, assemble_kernel_row, charge_row, load_matrix, matvec,
                                    partition_rows, save_matrix)
        from hvbem.fixtures import concentric_mesh, sphere_mesh  # noqa: F401
        from hvbem.mesh import CurvedTriangle, _flat_circumcircle  # noqa: F401
        from hvbem.postprocess import (FieldLine, IonizationModel, TraceError, TraceParams,  # noqa: F401
                                       eval_efield, eval_potential, load_ionization_model, pick_start_points,
                                       streamer_integral, surface_field_magnitudes, trace_fieldline,
                                       write_fieldline_csv)
        from hvbem.quadrature import (PairClass, QuadConfig, QuadratureError, classify_pair,  # noqa: F401
                                      closest_point, closest_point_flat, duffy_rule, near_singular_rule,
                                      regular_rule, subdivide_at)
        from hvbem.solver import Solution, SolverConfig, SolverError, residual, solve  # noqa: F401
    finally:
        for k in [k for k in sys.modules if k == "hvbem" or k.startswith("hvbem.")]:
            del sys.modules[k]
        sys.modules.update(saved)


@pytest.mark.parametrize("maker", [lambda: fixtures.sphere_mesh(3), lambda: fixtures.close_gap_mesh(2),
                                   lambda: fixtures.rod_plane_mesh(0.12), lambda: fixtures.rod_plane_mesh(0.4)])
def test_column_tiling_invariants(maker):
    """csrc/tiling.cpp (host C++, no GPU): the device column order is a
    permutation of contiguous owned tiles; every panel has exactly one
    record, in the lowest-numbered tile owning one of its corners, whose
    corners are that tile's local columns (owned -> device column or the
    partial slot of a receiving column, halo -> a copy slot); stages of
    `group` records have pairwise disjoint corners within the band (window
    - flush) of their first record, whose first column is the stage
    minimum; stage starts never decrease within a tile; dummies (-1) only
    pad stages; the receiving columns of a tile are numbered last and their
    exchange entries are partial then copies in producer order."""
    from paper_2003_12663_b200 import device

    m = maker()
    win, flush, grp, _ = device.sweep_geometry()
    band = win - flush
    T = device.column_tiling(m.colloc_points, m.tri_corner_cols, max_tile=2048)
    n, nt = m.n_collocation, m.n_triangles
    ntile = len(T.tile_width)
    assert np.array_equal(np.sort(T.perm), np.arange(n))
    assert np.array_equal(T.tile_col0, np.concatenate([[0], np.cumsum(T.tile_width)[:-1]]))
    assert T.tile_col0[-1] + T.tile_width[-1] == n
    home = np.repeat(np.arange(ntile), T.tile_width)[T.inv]          # original col -> owning tile
    primary = home[m.tri_corner_cols].min(axis=1)
    copies = {}                                                      # original col -> [(slot, producer)]
    partial = {}                                                     # original col -> partial slot
    seen = np.zeros(nt, dtype=int)
    for k in range(ntile):
        lc = T.lcol[T.tile_lptr[k]:T.tile_lptr[k + 1]]
        a, b = int(T.tile_ptr[k]), int(T.tile_ptr[k + 1])
        assert (b - a) % grp == 0
        prev = -1
        for s0 in range(a, b, grp):
            st = range(s0, s0 + grp)
            cols = [c for e in st for c in T.ent_meta[e, 1:4] if c >= 0]
            assert len(cols) == len(set(cols))                       # disjoint corners
            start = T.ent_meta[s0, 0]
            assert T.ent_tri[s0] >= 0 and start >= prev
            prev = start
            for e in st:
                t = int(T.ent_tri[e])
                if t < 0:
                    assert np.all(T.ent_meta[e, 1:4] == -1) and T.ent_meta[e, 4] == 0
                    continue
                assert primary[t] == k and T.ent_meta[e, 4] == 1
                loc = T.ent_meta[e, 1:4]
                assert min(loc) == T.ent_meta[e, 0] >= start and max(loc) <= start + band
                seen[t] += 1
        # local columns: every owned column, plus the halo
        owned = set(T.perm[T.tile_col0[k]:T.tile_col0[k] + T.tile_width[k]].tolist())
        for e in range(a, b):
            if T.ent_tri[e] >= 0:
                for c, l in zip(m.tri_corner_cols[T.ent_tri[e]], T.ent_meta[e, 1:4]):
                    d = int(lc[l])
                    if home[c] == k:
                        assert (d >= 0 and T.perm[d] == c) or (d < 0 and partial.setdefault(int(c), ~d) == ~d)
                    else:
                        assert d < 0 and home[c] > k and ~d < T.n_halo
                        if (~d, k) not in copies.setdefault(int(c), []):
                            copies[int(c)].append((~d, k))
        assert sum(1 for d in lc if d >= 0 or ~d >= T.n_halo) == len(owned)
    assert np.all(seen == 1)
    # partial slots per receiving column, from the exchange entries (a column
    # whose own tile has no panel on it is reached through them only)
    first = T.xent[T.xent[:, 2] == 1]
    px = {int(T.perm[d]): int(sl) for sl, d, _, _ in first}
    assert all(px[c] == sl for c, sl in partial.items())
    partial = px
    assert set(partial) == set(copies) and len(set(partial.values())) == len(partial)
    assert all(T.n_halo <= p < T.n_slots for p in partial.values())
    assert sum(len(v) for v in copies.values()) == T.n_halo
    for k in range(ntile):
        x = T.xent[T.tile_xptr[k]:T.tile_xptr[k + 1]]
        recv = [c for c in T.perm[T.tile_col0[k]:T.tile_col0[k] + T.tile_width[k]] if int(c) in partial]
        dev = T.inv[recv]
        assert np.array_equal(dev, np.arange(T.tile_col0[k] + T.tile_width[k] - len(recv),
                                             T.tile_col0[k] + T.tile_width[k]))  # receiving columns last
        want = []
        for c in recv:
            cp = sorted(copies[int(c)], key=lambda sp: sp[1])
            want.append([partial[int(c)], T.inv[c], 1, 0])
            want += [[sl, T.inv[c], 0, int(i + 1 == len(cp))] for i, (sl, _) in enumerate(cp)]
        assert np.array_equal(x, np.array(want, dtype=np.int32).reshape(-1, 4))
        prods = sorted({p for c in recv for _, p in copies[int(c)]})
        assert list(T.prods[T.tile_pptr[k]:T.tile_pptr[k + 1]]) == prods and all(p < k for p in prods)
        for p in prods:
            assert k in T.cons[T.tile_cptr[p]:T.tile_cptr[p + 1]]
    assert len(T.cons) == len(T.prods)


# ---------------------------------------------------------------------------
# case outputs (reference src/cli.py:172-235): byte-compatible writers
# ---------------------------------------------------------------------------


def test_case_outputs_match_reference_bytes(tmp_path):
    """solution.json, surface_field.csv and surface_field.vtk written by
    paper_2003_12663_b200.outputs equal, byte for byte, the files the
    reference's own writers produced on the same inputs
    (tests/golden/make_outputs_golden.py), and load_solution reads them."""
    import importlib.util

    from paper_2003_12663_b200 import outputs
    from paper_2003_12663_b200.config import Config
    from paper_2003_12663_b200.solver import Solution

    spec = importlib.util.spec_from_file_location("mog", os.path.join(ROOT, "tests", "golden",
                                                                       "make_outputs_golden.py"))
    src = open(spec.origin).read()
    ns = {}
    exec(src[src.index("MESH_PATH ="):src.index('if __name__ == "__main__":')], {"np": np}, ns)
    mesh = fixtures.sphere_mesh(1)
    u, e = ns["inputs"](mesh.n_collocation)
    sol = Solution(u=u, V=np.zeros(0), iterations=7, residual=3.25e-9)
    outputs.write_solution(tmp_path, ns["MESH_PATH"], mesh, sol, e, Config(), {"total": 1.0}, 1, 1)
    outputs.write_surface_csv(tmp_path / "surface_field.csv", mesh, e)
    outputs.write_surface_vtk(tmp_path / "surface_field.vtk", mesh, e)
    gold = os.path.join(ROOT, "tests", "golden", "outputs")
    for name in ("solution.json", "surface_field.csv", "surface_field.vtk"):
        assert (tmp_path / name).read_bytes() == open(os.path.join(gold, name), "rb").read(), name
    doc, back = outputs.load_solution(gold)
    assert doc["format"] == outputs.SOLUTION_FORMAT and back.iterations == 7
    np.testing.assert_array_equal(back.u, u)
    with pytest.raises(ValueError, match="unknown solution format"):
        (tmp_path / "solution.json").write_text('{"format": "x"}')
        outputs.load_solution(tmp_path)


@pytest.mark.parametrize("maker", [lambda: fixtures.sphere_mesh(3), lambda: fixtures.rod_plane_mesh(0.12)])
def test_halo_exchange_schedule_sums_every_column(maker):
    """The sweep's data flow over the host schedule (csrc/assemble.cu +
    csrc/tiling.cpp 5), emulated with one random value per (panel, corner):
    window sums per tile in record order, owned columns written, halo copies
    and receiving partials to slots, then each tile's exchange entries summed
    in order -- every device column ends up with the sum of its panels'
    contributions, each written exactly once."""
    from paper_2003_12663_b200 import device

    m = maker()
    T = device.column_tiling(m.colloc_points, m.tri_corner_cols, max_tile=512)
    n, nt = m.n_collocation, m.n_triangles
    val = np.random.default_rng(7).standard_normal((nt, 3))
    A = np.full(n, np.nan)
    written = np.zeros(n, dtype=int)
    slots = np.full(T.n_slots, np.nan)
    for k in range(len(T.tile_width)):
        lc = T.lcol[T.tile_lptr[k]:T.tile_lptr[k + 1]]
        win = np.zeros(len(lc))
        for e in range(T.tile_ptr[k], T.tile_ptr[k + 1]):
            t = T.ent_tri[e]
            if t >= 0:
                for c in range(3):
                    win[T.ent_meta[e, 1 + c]] += val[t, c]
        for i, d in enumerate(lc):
            if d >= 0:
                A[d] = win[i]
                written[d] += 1
            else:
                assert np.isnan(slots[~d])
                slots[~d] = win[i]
    for k in range(len(T.tile_width)):
        acc = None
        for sl, d, first, last in T.xent[T.tile_xptr[k]:T.tile_xptr[k + 1]]:
            acc = slots[sl] if first else acc + slots[sl]
            if last:
                A[d] = acc
                written[d] += 1
    assert np.all(written == 1) and not np.any(np.isnan(slots))
    ref = np.zeros(n)
    np.add.at(ref, T.inv[m.tri_corner_cols.ravel()], val.ravel())
    np.testing.assert_allclose(A, ref, rtol=1e-12, atol=1e-12)
