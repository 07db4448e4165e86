"""Minimal command line over the drop-in: ``solve`` only (the
reference's CLI is OUT OF SCOPE).  It exists so callers of the reference's
``hvbem.cli.main(["solve", ...])`` -- its acceptance tests among them
(tests/reference_suite/test_acceptance.py, criterion 7) -- find the same
entry point: mesh file in, case directory out (outputs.py formats,
byte-compatible with reference src/cli.py:172-221), the reference's exit
codes (src/cli.py:34-38).  ``fit_scaling_exponent`` is the bench ladder's
log-log slope (src/cli.py:385-392)."""

from __future__ import annotations

import argparse
import sys
import time
from pathlib import Path

import numpy as np

from .assembly import AssemblyError, assemble, save_matrix
from .config import Config, default_workers
from .mesh import MeshError, load_mesh
from .outputs import write_solution, write_surface_csv, write_surface_vtk
from .postprocess import surface_field_magnitudes
from .solver import SolverError, solve

__all__ = ["main", "fit_scaling_exponent", "EXIT_OK", "EXIT_PARSE", "EXIT_ASSEMBLY", "EXIT_SOLVER"]

EXIT_OK, EXIT_PARSE, EXIT_ASSEMBLY, EXIT_SOLVER = 0, 1, 2, 3


def fit_scaling_exponent(pairs):
    """Least-squares slope of log(time) against log(N); None if < 2 points."""
    pts = np.array([(n, t) for n, t in pairs if t > 0.0], dtype=float)
    if len(pts) < 2:
        return None
    return float(np.polyfit(np.log(pts[:, 0]), np.log(pts[:, 1]), 1)[0])


def _solve(args) -> int:
    cfg = Config.load(args.config, args.set)
    workers = args.workers or default_workers()
    out = Path(args.out)
    out.mkdir(parents=True, exist_ok=True)
    clock = time.perf_counter
    t = [clock()]
    mesh = load_mesh(args.mesh)
    t.append(clock())
    matrix, rhs = assemble(mesh, cfg.quad(), n_blocks=args.blocks, workers=workers,
                           precision=cfg["assembly.precision"])
    t.append(clock())
    sol = solve(matrix, rhs, cfg.solver(workers=workers))
    t.append(clock())
    surface_e = surface_field_magnitudes(mesh, sol, cfg=cfg.quad(), workers=workers)
    t.append(clock())
    names = ("mesh_load", "assembly", "solve", "surface_field")
    timings = {k: t[i + 1] - t[i] for i, k in enumerate(names)}
    timings["total"] = t[-1] - t[0]
    write_solution(out, args.mesh, mesh, sol, surface_e, cfg, timings, workers, args.blocks)
    write_surface_csv(out / "surface_field.csv", mesh, surface_e)
    write_surface_vtk(out / "surface_field.vtk", mesh, surface_e)
    if args.dump_matrix:
        save_matrix(matrix, out / "matrix.bin")
    print(f"solved {Path(args.mesh).name}: n={mesh.n_collocation} floating={mesh.n_floating} "
          f"iters={sol.iterations} residual={sol.residual:.2e}")
    return EXIT_OK


def main(argv=None) -> int:
    ap = argparse.ArgumentParser(prog="hvbem", description="B200 drop-in for hvbem: solve a mesh")
    sub = ap.add_subparsers(dest="command", required=True)
    p = sub.add_parser("solve", help="assemble, solve and write the surface field")
    p.add_argument("--mesh", required=True)
    p.add_argument("--config", default=None)
    p.add_argument("--out", required=True)
    p.add_argument("--workers", type=int, default=None)
    p.add_argument("--blocks", type=int, default=1)
    p.add_argument("--set", action="append", default=[], metavar="KEY=VALUE")
    p.add_argument("--dump-matrix", action="store_true")
    args = ap.parse_args(argv)
    try:
        return _solve(args)
    except (MeshError, FileNotFoundError, ValueError, KeyError) as exc:
        print(f"error: {exc}", file=sys.stderr)
        return EXIT_PARSE
    except AssemblyError as exc:
        print(f"assembly error: {exc}", file=sys.stderr)
        return EXIT_ASSEMBLY
    except SolverError as exc:
        print(f"solver did not converge: {exc} (best residual {exc.best_residual:.3e})", file=sys.stderr)
        return EXIT_SOLVER


if __name__ == "__main__":
    sys.exit(main())
