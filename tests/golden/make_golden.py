"""Generate the golden fixtures from the LIVE reference (hvbem 0.1.0).

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_golden.py

Writes tests/golden/*.npz.  Inputs are built with the reference's own
fixtures (bit-identical to paper_2003_12663_b200.fixtures, checked here and
in tests/test_mesh_parity.py through the recorded hashes); outputs are the
reference's own assemble / solve / charge_row / eval_* /
surface_field_magnitudes / trace_fieldline / near_singular_rule results.
"""

from __future__ import annotations

import hashlib
import os
import sys

import numpy as np

REF = os.environ.get("HVBEM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

import hvbem  # noqa: E402
from hvbem import assembly as RA  # noqa: E402
from hvbem import fixtures as RF  # noqa: E402
from hvbem import postprocess as RP  # noqa: E402
from hvbem import quadrature as RQ  # noqa: E402
from hvbem import solver as RS  # noqa: E402
from hvbem.mesh import EPS0, parse_mesh  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.abspath(os.path.join(OUT, "..", "..")))
from paper_2003_12663_b200 import fixtures as MF  # noqa: E402  (our generator, for cfg4-mini only)


def h(a) -> str:
    return hashlib.sha256(np.ascontiguousarray(a).tobytes()).hexdigest()


def mesh_record(m, prefix, rec):
    rec[prefix + "vertices_sha"] = h(m.vertices)
    rec[prefix + "cc_sha"] = h(m.circumcenters)
    rec[prefix + "cr_sha"] = h(m.circumradii)
    rec[prefix + "weights"] = m.lumped_weights
    rec[prefix + "normals"] = m.colloc_normals


def cfg3_mesh(level_sph, level_encl):
    v1, t1 = RF.sphere_mesh_parts(level_sph, radius=0.5, center=(-0.6, 0.0, 0.0), tag=0)
    v2, t2 = RF.sphere_mesh_parts(level_sph, radius=0.5, center=(0.6, 0.0, 0.0), tag=1, id_offset=len(v1))
    v3, t3 = RF.sphere_mesh_parts(level_encl, radius=3.0, flip=True, tag=2, id_offset=len(v1) + len(v2))
    text = RF.mesh_text(np.vstack([v1, v2, v3]), t1 + t2 + t3,
                        ["patch 0 electrode 1.0", "patch 1 floating 0", "patch 2 electrode 0.0"])
    return parse_mesh(text, name="<cfg3>")


def plates_mesh():
    """Two parallel flat slabs 4 mm apart (coplanar panels + near pairs)."""
    pa, ta = MF._box_grid((0.2, 0.2, 0.01), (6, 6, 1))
    pb, tb = MF._box_grid((0.2, 0.2, 0.01), (6, 6, 1))
    pb = pb + np.array([0.013, 0.0, 0.024])
    verts = np.vstack([pa, pb])
    tris = [(tuple(int(k) for k in r), 0) for r in ta] + [(tuple(int(k) + len(pa) for k in r), 1) for r in tb]
    text = RF.mesh_text(verts, tris, ["patch 0 electrode 1.0", "patch 1 electrode -1.0"])
    return parse_mesh(text, name="<plates>")


def rodplane_mini():
    v, ids, tags, lines = MF.rod_plane_parts(scale=0.12)
    tris = [(tuple(int(k) for k in r), int(t)) for r, t in zip(ids, tags)]
    return parse_mesh(RF.mesh_text(v, tris, lines), name="<rodplane-mini>")


def solve_tight(matrix, rhs):
    try:
        s = RS.solve(matrix, rhs, RS.SolverConfig(rel_tol=1e-12, max_iters=600))
        return s.u, s.V, s.iterations, True
    except RS.SolverError:
        x = np.linalg.solve(matrix.toarray(), rhs)
        return x[: matrix.n], x[matrix.n:], -1, False


def case(name, mesh, rec, rows=None, fields=None, surface=False):
    A, b = RA.assemble(mesh)
    dense = A.toarray()
    if rows is None:
        rec[name + "_A"] = dense
    else:
        rec[name + "_rows"] = np.asarray(rows)
        rec[name + "_Arows"] = dense[rows]
    rec[name + "_rhs"] = b
    rec[name + "_diag"] = np.array([A.diagnostics["pairs_regular"], A.diagnostics["pairs_singular"],
                                    A.diagnostics["pairs_near_singular"]])
    u, V, it, conv = solve_tight(A, b)
    rec[name + "_u"] = u
    rec[name + "_V"] = V
    rec[name + "_iters"] = np.array([it, int(conv)])
    mesh_record(mesh, name + "_mesh_", rec)
    sol = RS.Solution(u=u, V=V, iterations=0, residual=0.0)
    if fields is not None:
        pts = np.asarray(fields, dtype=float)
        rec[name + "_pts"] = pts
        rec[name + "_E"] = np.array([RP.eval_efield(sol, mesh, p) for p in pts])
        rec[name + "_phi"] = np.array([RP.eval_potential(sol, mesh, p) for p in pts])
    if surface:
        rec[name + "_surfE"] = RP.surface_field_magnitudes(mesh, sol)
    # near pairs of the first rows, as the reference defers them
    tab = mesh.tables(6)
    nl = []
    for i in range(min(mesh.n_collocation, 400)):
        _, deferred, _ = RA.row_pass1(mesh, tab, mesh.colloc_points[i], int(mesh.colloc_vertex_ids[i]),
                                      RA.KERNEL_SL)
        nl += [(i, t) for t in deferred]
    rec[name + "_nearpairs"] = np.array(nl, dtype=np.int64).reshape(-1, 2)
    return A, b, sol


def main():
    rec: dict = {}
    # mesh hashes of the fixture ladder
    for L in (1, 2, 3, 4):
        m = RF.sphere_mesh(L)
        rec[f"sphere{L}_vertices_sha"] = h(m.vertices)
        rec[f"sphere{L}_cc_sha"] = h(m.circumcenters)
        rec[f"sphere{L}_cr_sha"] = h(m.circumradii)

    pts = np.array([[2.0, 0.0, 0.0], [0.0, 0.0, 2.0], [1.3, 0.9, -0.6], [0.3, -0.2, 0.1],
                    [1.02, 0.05, 0.0], [0.0, 1.01, 0.02]])
    sphere2 = RF.sphere_mesh(2)
    A, b, sol = case("sphere2", sphere2, rec, fields=pts, surface=True)
    rec["sphere2_charge"] = RA.charge_row(sphere2, np.arange(sphere2.n_collocation), eps_plus=EPS0)
    # traced lines on the solved sphere and capacitor
    lines = []
    for s0, o in (([1.05, 0.0, 0.0], 1), ([0.0, 0.7, 0.8], 1)):
        ln = RP.trace_fieldline(sol, sphere2, np.array(s0, float), o)
        lines.append(ln)
    cap = RF.concentric_mesh(2, [(0.5, "electrode 1.0"), (1.0, "electrode 0.0")])
    Ac, bc, solc = case("cap2", cap, rec, fields=np.array([[0.7, 0.1, 0.05], [0.1, 0.6, 0.2], [0.503, 0.01, 0.0]]))
    for s0, o in (([0.504, 0.0, 0.0], 1), ([0.6, 0.0, 0.0], -1), ([0.45, 0.35, 0.2], 1)):
        lines.append(RP.trace_fieldline(solc, cap, np.array(s0, float), o))
    gas = RP.IonizationModel(np.array([0.0, 1.0, 2.0, 4.0]), np.array([0.0, 0.5, 3.0, 6.0]), 0.8)
    for k, ln in enumerate(lines):
        rec[f"line{k}_points"] = ln.points
        rec[f"line{k}_mags"] = ln.e_magnitudes
        rec[f"line{k}_arcs"] = ln.arc_lengths
        rec[f"line{k}_term"] = np.array(ln.termination)
        v, inc = RP.streamer_integral(ln, gas)
        rec[f"line{k}_streamer"] = np.array([v, float(inc)])
    rec["n_lines"] = np.array(len(lines))
    sp = RP.pick_start_points(cap, solc, 5)
    rec["cap2_seeds"] = sp[0]
    rec["cap2_seed_idx"] = sp[1]

    case("floatshell1", RF.concentric_mesh(1, [(0.5, "electrode 1.0"), (0.75, f"sheet 0 {EPS0!r} {EPS0!r}"),
                                                (1.0, "electrode 0.0")]), rec)
    case("diel1", RF.concentric_mesh(1, [(0.5, "electrode 1.0"), (0.75, f"dielectric {EPS0!r} {2 * EPS0!r}"),
                                         (1.0, "electrode 0.0")]), rec,
         fields=np.array([[0.7, 0.1, 0.05], [0.0, 0.6, 0.1]]))
    case("diel2", RF.concentric_mesh(2, [(0.5, "electrode 1.0"), (0.75, f"dielectric {EPS0!r} {2 * EPS0!r}"),
                                         (1.0, "electrode 0.0")]), rec)
    case("gap2", RF.concentric_mesh(2, [(1.0, "electrode 1.0"), (1.02, "electrode 0.0")]), rec,
         fields=np.array([[1.01, 0.0, 0.0], [0.0, 0.3, 1.005]]))
    case("cfg3mini", cfg3_mesh(1, 0), rec)
    case("plates", plates_mesh(), rec, fields=np.array([[0.0, 0.0, 0.017], [0.05, 0.03, 0.0105]]))
    rp = rodplane_mini()
    n = rp.n_collocation
    diel = [i for i, k in enumerate(rp.row_kinds) if isinstance(k, hvbem.DielectricJump)]
    rows = np.unique(np.concatenate([np.linspace(0, n - 1, 48).astype(int), np.array(diel[:16], dtype=int)]))
    case("rodmini", rp, rec, rows=rows)

    # quadrature golden values (reference tests/test_quadrature.py, test_acceptance.py)
    from hvbem.mesh import CurvedTriangle, _flat_circumcircle

    corners = np.array([[0.0, 0.0, 0.0], [1.0, 0.0, 0.0], [0.0, 1.0, 0.0]])
    nodes = np.vstack([corners, 0.5 * (corners[0] + corners[1]), 0.5 * (corners[1] + corners[2]),
                       0.5 * (corners[2] + corners[0])])
    c, r = _flat_circumcircle(corners)
    tri = CurvedTriangle(0, (0, 1, 2), (3, 4, 5), 0, nodes, c, r)
    for frac in (0.1, 0.3, 0.6, 1.0):
        x = corners.mean(axis=0) + np.array([0.0, 0.0, frac * r])
        rule = RQ.near_singular_rule(x, tri)
        rec[f"near_{frac}_nodes"] = rule.nodes
        rec[f"near_{frac}_weights"] = rule.weights
    for cn in range(3):
        d = RQ.duffy_rule(cn, 6)
        rec[f"duffy{cn}_nodes"] = d.nodes
        rec[f"duffy{cn}_weights"] = d.weights
    g = RQ._graded_rule(3, 8, 8)
    rec["graded_nodes"] = g.nodes
    rec["graded_weights"] = g.weights
    # random closest-point / subdivision decisions
    rng = np.random.default_rng(5)
    cp = []
    for _ in range(3000):
        cs = rng.uniform(-1, 1, (3, 3))
        x = rng.uniform(-1.5, 1.5, 3)
        cp.append((*cs.ravel(), *x, *RQ.closest_point_flat(x, cs)))
    rec["closest_cases"] = np.array(cp)

    np.savez_compressed(os.path.join(OUT, "golden.npz"), **rec)
    print("wrote", os.path.join(OUT, "golden.npz"), len(rec), "arrays")


if __name__ == "__main__":
    main()
