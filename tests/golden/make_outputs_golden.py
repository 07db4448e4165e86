"""Golden case-directory files written by the LIVE reference's own writers
(reference src/cli.py:172-221) for tests/test_host.py::test_case_outputs_*.

Run in the build container (the only place /root/reference exists):

    PYTHONDONTWRITEBYTECODE=1 python tests/golden/make_outputs_golden.py

Inputs: the reference's sphere_mesh(1) (bit-identical to ours,
tests/test_mesh_parity.py), a deterministic synthetic density / surface
field, the default Config and a fixed absolute mesh path.  Writes
tests/golden/outputs/{solution.json, surface_field.csv, surface_field.vtk}.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = os.environ.get("HVBEM_REF", "/root/reference/pkg/src")
sys.path.insert(0, REF)
sys.dont_write_bytecode = True

from hvbem import cli as RC  # noqa: E402
from hvbem import fixtures as RF  # noqa: E402
from hvbem.config import Config  # noqa: E402
from hvbem.solver import Solution  # noqa: E402

OUT = Path(os.path.dirname(os.path.abspath(__file__))) / "outputs"
MESH_PATH = "/hvb/case/sphere1.bemesh"


def inputs(n):
    u = np.sin(np.arange(n) * 0.37) * 1e-3 + 1.0 / 3.0
    e = np.cos(np.arange(n) * 0.11) ** 2 * 7.5e5 + np.pi
    return u, e


if __name__ == "__main__":
    OUT.mkdir(exist_ok=True)
    mesh = RF.sphere_mesh(1)
    u, e = inputs(mesh.n_collocation)
    sol = Solution(u=u, V=np.zeros(0), iterations=7, residual=3.25e-9)
    RC._write_solution(OUT, MESH_PATH, mesh, sol, e, Config(), {"total": 1.0}, 1, 1)
    (OUT / "run.json").unlink()
    RC._write_surface_csv(OUT / "surface_field.csv", mesh, e)
    RC._write_surface_vtk(OUT / "surface_field.vtk", mesh, e)
    print("wrote", sorted(p.name for p in OUT.iterdir()))
