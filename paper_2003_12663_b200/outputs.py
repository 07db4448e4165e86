"""Case-directory outputs of a solve: the files the reference's CLI writes
and its ``trace`` command reads back (reference src/cli.py:172-235).  The
CLI itself is out of scope; these writers and the loader keep
the on-disk formats byte-compatible, so a case solved here can be traced by
the reference and vice versa, and solution.json is bit-identical for any
row blocking / worker count (reference tests/test_cli.py:96-108).

* ``solution.json`` -- format "hvbem-solution 1": mesh path, n, n_floating,
  u, V, iterations, residual, surface |E|, config snapshot (indent 1; run
  metadata goes to run.json so the solution file is deterministic);
* ``surface_field.csv`` -- vertex_id,x,y,z,E per collocation point, floats
  as repr();
* ``surface_field.vtk`` -- legacy-VTK polydata of the corner triangles with
  |E| point data.
"""

from __future__ import annotations

import json
from pathlib import Path

import numpy as np

from .solver import Solution

__all__ = ["SOLUTION_FORMAT", "write_solution", "write_surface_csv", "write_surface_vtk", "load_solution"]

SOLUTION_FORMAT = "hvbem-solution 1"


def _floats(a) -> list:
    return [float(v) for v in np.asarray(a, dtype=np.float64).ravel()]


def write_solution(out_dir, mesh_path, mesh, solution, surface_e, cfg, timings=None, workers=1, blocks=1) -> None:
    """solution.json (deterministic) + run.json (timings, worker counts)."""
    out = Path(out_dir)
    doc = {
        "format": SOLUTION_FORMAT,
        "mesh_path": str(Path(mesh_path).resolve()),
        "n": int(mesh.n_collocation),
        "n_floating": int(mesh.n_floating),
        "u": _floats(solution.u),
        "V": _floats(solution.V),
        "iterations": int(solution.iterations),
        "residual": float(solution.residual),
        "surface_e": _floats(surface_e),
        "config": cfg.snapshot(),
    }
    (out / "solution.json").write_text(json.dumps(doc, indent=1), encoding="utf-8")
    (out / "run.json").write_text(json.dumps({"workers": workers, "blocks": blocks, "timings": timings or {}},
                                             indent=1), encoding="utf-8")


def write_surface_csv(path, mesh, surface_e) -> None:
    e = _floats(surface_e)
    rows = ["vertex_id,x,y,z,E"]
    for i, (vid, p) in enumerate(zip(np.asarray(mesh.colloc_vertex_ids).tolist(),
                                     np.asarray(mesh.colloc_points, dtype=np.float64).tolist())):
        rows.append(f"{int(vid)},{p[0]!r},{p[1]!r},{p[2]!r},{e[i]!r}")
    Path(path).write_text("\n".join(rows) + "\n", encoding="utf-8")


def write_surface_vtk(path, mesh, surface_e) -> None:
    pts = np.asarray(mesh.colloc_points, dtype=np.float64).tolist()
    cols = np.asarray(mesh.tri_corner_cols).tolist()
    n, nt = len(pts), len(cols)
    parts = ["# vtk DataFile Version 3.0", "hvbem surface field", "ASCII", "DATASET POLYDATA", f"POINTS {n} double"]
    parts += [f"{p[0]!r} {p[1]!r} {p[2]!r}" for p in pts]
    parts.append(f"POLYGONS {nt} {4 * nt}")
    parts += [f"3 {c[0]} {c[1]} {c[2]}" for c in cols]
    parts += [f"POINT_DATA {n}", "SCALARS E_magnitude double 1", "LOOKUP_TABLE default"]
    parts += [repr(v) for v in _floats(surface_e)]
    Path(path).write_text("\n".join(parts) + "\n", encoding="utf-8")


def load_solution(case_dir):
    """(payload dict, Solution) from a case directory's solution.json."""
    doc = json.loads((Path(case_dir) / "solution.json").read_text(encoding="utf-8"))
    if doc.get("format") != SOLUTION_FORMAT:
        raise ValueError(f"{case_dir}: unknown solution format")
    sol = Solution(u=np.array(doc["u"], dtype=float), V=np.array(doc["V"], dtype=float),
                   iterations=doc["iterations"], residual=doc["residual"])
    return doc, sol
