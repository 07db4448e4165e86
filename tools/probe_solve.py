"""Dev probe: GMRES convergence of cfg4 variants under reference semantics."""
import sys, os, time, logging
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
from paper_2003_12663_b200 import fixtures as F
from paper_2003_12663_b200.assembly import assemble
from paper_2003_12663_b200.solver import solve, SolverConfig, SolverError
logging.basicConfig(level=logging.INFO, format="%(message)s")
scale = float(sys.argv[1])
for name, v0, vp in (("rod+", 1e5, 0.0), ("plane-", 0.0, -1e5), ("split", 5e4, -5e4)):
    mesh = F.rod_plane_mesh(scale, v0=v0, v_plane=vp)
    A, b = assemble(mesh)
    t = time.time()
    try:
        s = solve(A, b, SolverConfig(max_iters=300, verbose=False))
        print(name, scale, "converged", s.iterations, f"{s.residual:.2e}", f"{time.time()-t:.2f}s", flush=True)
    except SolverError as e:
        print(name, scale, "FAILED", e.iterations, f"{e.best_residual:.3e}", f"{time.time()-t:.2f}s", flush=True)
    # scaled vs true ratio after a tight solve
    try:
        s = solve(A, b, SolverConfig(max_iters=400, rel_tol=1e-10))
        print(name, "tight converged", s.iterations, flush=True)
    except SolverError as e:
        print(name, "tight FAILED", e.iterations, f"{e.best_residual:.3e}", flush=True)
    del A
    torch.cuda.empty_cache()
