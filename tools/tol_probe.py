"""Dev probe: GMRES tolerance vs distance to a dense LU solve on config 2."""
import sys
import time

import numpy as np

sys.path.insert(0, ".")
from paper_2003_12663_b200 import fixtures  # noqa: E402
from paper_2003_12663_b200.assembly import assemble  # noqa: E402
from paper_2003_12663_b200.mesh import EPS0  # noqa: E402
from paper_2003_12663_b200.solver import SolverConfig, solve  # noqa: E402

m = fixtures.concentric_mesh(4, [(0.5, "electrode 1.0"), (0.75, f"dielectric {EPS0!r} {2 * EPS0!r}"),
                                 (1.0, "electrode 0.0")])
t = time.time()
A, rhs = assemble(m)
Ad = A.toarray()
x = np.linalg.solve(Ad, rhs)
kind = m.row_kind_code
print("cond est", np.linalg.cond(Ad[:2000, :2000]) if len(sys.argv) > 1 else "-")
for tol in (1e-12, 1e-13, 1e-14):
    try:
        sol = solve(A, rhs, SolverConfig(rel_tol=tol))
        d = np.abs(sol.u - x)
        i = int(np.argmax(d))
        print(f"tol {tol:.0e}: it {sol.iterations} res {sol.residual:.2e} maxdiff/max {d.max() / np.abs(x).max():.2e} "
              f"at kind {kind[i]} |x_i| {abs(x[i]):.3e}; per kind " +
              " ".join(f"{k}:{d[kind == k].max() / np.abs(x[kind == k]).max():.2e}" for k in np.unique(kind)))
    except Exception as e:  # noqa: BLE001
        print(f"tol {tol:.0e}: {type(e).__name__} {e}")
print("res of LU", np.linalg.norm(rhs - Ad @ x) / np.linalg.norm(rhs))
