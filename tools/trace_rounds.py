"""Dev probe: per-round device time vs outstanding field requests of the
config-5 tracer (8,192 strongest seeds by default): where the trace phase
spends its time (N-body-bound rounds vs the lockstep tail)."""
import os
import sys

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_12663_b200 import fixtures, tracer  # noqa: E402
from paper_2003_12663_b200.assembly import assemble  # noqa: E402
from paper_2003_12663_b200.postprocess import TraceParams, eval_efield_batch, pick_start_points  # noqa: E402
from paper_2003_12663_b200.quadrature import QuadConfig  # noqa: E402
from paper_2003_12663_b200.solver import solve  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
k = int(sys.argv[2]) if len(sys.argv) > 2 else 8192
mesh = fixtures.rod_plane_mesh(scale)
A, b = assemble(mesh)
sol = solve(A, b)
del A
starts, idx, _ = pick_start_points(mesh, sol, k)
E = eval_efield_batch(sol, mesh, starts)
orient = np.where(np.einsum("ij,ij->i", E, mesh.colloc_normals[idx]) >= 0, 1, -1)
torch.cuda.synchronize()
tracer.ROUND_PROBE = []
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
res = tracer.trace_device(sol, mesh, starts, orient, TraceParams(), QuadConfig())
e1.record()
torch.cuda.synchronize()
total = e0.elapsed_time(e1) / 1e3
rows = [(p, a.elapsed_time(b) / 1e3) for p, a, b in tracer.ROUND_PROBE]
tracer.ROUND_PROBE = None
pend = np.array([r[0] for r in rows])
ts = np.array([r[1] for r in rows])
print(f"lines {k} rounds {len(rows)} total {total:.3f}s sum-of-rounds {ts.sum():.3f}s evals {res.field_points}")
for lo, hi in ((0, 16), (16, 128), (128, 1024), (1024, 4096), (4096, 1 << 30)):
    sel = (pend >= lo) & (pend < hi)
    print(f"pending [{lo},{hi}): rounds {sel.sum():5d} time {ts[sel].sum():.3f}s requests {pend[sel].sum():9d} "
          f"us/request {1e6 * ts[sel].sum() / max(1, pend[sel].sum()):.2f}")
