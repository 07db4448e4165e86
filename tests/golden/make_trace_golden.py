"""Golden field lines, seeds and surface distances from the LIVE reference.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_trace_golden.py

Writes tests/golden/trace_golden.npz: for the concentric capacitor (level 2)
and the 2 % gap shells (level 2) -- the reference's own solution
(rel_tol 1e-12), pick_start_points seeds with orientation sign(E.n) (the
CLI's rule, src/cli.py:276-283), every traced line (points, |E|, arcs,
termination), streamer values for a toy gas, and _surface_distance at
random points near the surfaces.
"""

from __future__ import annotations

import os
import sys

import numpy as np

REF = os.environ.get("HVBEM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from hvbem import assembly as RA  # noqa: E402
from hvbem import fixtures as RF  # noqa: E402
from hvbem import postprocess as RP  # noqa: E402
from hvbem import solver as RS  # noqa: E402

OUT = os.path.dirname(os.path.abspath(__file__))
GAS = RP.IonizationModel(np.array([0.0, 1.0, 2.0, 4.0, 40.0]), np.array([0.0, 0.5, 3.0, 6.0, 60.0]), 0.8)
CASES = {
    "cap2": lambda: RF.concentric_mesh(2, [(0.5, "electrode 1.0"), (1.0, "electrode 0.0")]),
    "gap2": lambda: RF.concentric_mesh(2, [(1.0, "electrode 1.0"), (1.02, "electrode 0.0")]),
}
SEEDS = {"cap2": 24, "gap2": 0}  # gap2: surface distances only (lines in a 2 % gap are
#                                   hours of reference near-singular Python loops)


def main():
    rec = {}
    rng = np.random.default_rng(11)
    for name, make in CASES.items():
        mesh = make()
        A, b = RA.assemble(mesh)
        s = RS.solve(A, b, RS.SolverConfig(rel_tol=1e-12, max_iters=600))
        sol = RS.Solution(u=s.u, V=s.V, iterations=0, residual=0.0)
        rec[f"{name}_u"] = s.u
        rec[f"{name}_V"] = s.V
        print(name, "solved", flush=True)
        if SEEDS[name] == 0:
            starts, idx, se = np.zeros((0, 3)), np.zeros(0, dtype=np.int64), np.zeros(0)
        else:
            starts, idx, se = RP.pick_start_points(mesh, sol, SEEDS[name])
        orient = np.array([1 if RP.eval_efield(sol, mesh, x) @ mesh.colloc_normals[i] >= 0 else -1
                           for x, i in zip(starts, idx)])
        rec[f"{name}_surfE"] = se
        rec[f"{name}_starts"] = starts
        rec[f"{name}_seed_idx"] = idx
        rec[f"{name}_orient"] = orient
        for k, (x0, o) in enumerate(zip(starts, orient)):
            ln = RP.trace_fieldline(sol, mesh, x0, int(o))
            rec[f"{name}_l{k}_points"] = ln.points
            rec[f"{name}_l{k}_mags"] = ln.e_magnitudes
            rec[f"{name}_l{k}_arcs"] = ln.arc_lengths
            rec[f"{name}_l{k}_term"] = np.array(ln.termination)
            v, inc = RP.streamer_integral(ln, GAS)
            rec[f"{name}_l{k}_streamer"] = np.array([v, float(inc)])
            print(name, k, ln.termination, len(ln.points), flush=True)
        # surface distance at random points near the collocation points
        i = rng.integers(0, mesh.n_collocation, 200)
        X = mesh.colloc_points[i] + rng.normal(0.0, 0.03, (200, 3))
        sd = np.array([RP._surface_distance(mesh, x) for x in X])
        rec[f"{name}_sd_pts"] = X
        rec[f"{name}_sd"] = sd
    rec["gas_e"] = GAS.e_values
    rec["gas_a"] = GAS.alpha_values
    rec["gas_k"] = np.array(GAS.k_str)
    np.savez_compressed(os.path.join(OUT, "trace_golden.npz"), **rec)
    print("wrote", os.path.join(OUT, "trace_golden.npz"), len(rec), "arrays")


if __name__ == "__main__":
    main()
