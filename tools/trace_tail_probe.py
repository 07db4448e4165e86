"""Dev probe (GPU): trace a handful of cfg4 lines (every round is a tail
round) after assemble + solve; run under ncu's launch list to see which
kernel of a round dominates its latency."""
import os
import sys
import time

import numpy as np
import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2003_12663_b200 import fixtures, tracer  # noqa: E402
from paper_2003_12663_b200.assembly import assemble  # noqa: E402
from paper_2003_12663_b200.postprocess import TraceParams, eval_efield_batch, pick_start_points  # noqa: E402
from paper_2003_12663_b200.quadrature import QuadConfig  # noqa: E402
from paper_2003_12663_b200.solver import solve  # noqa: E402

k = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mesh = fixtures.rod_plane_mesh(1.0)
A, b = assemble(mesh)
sol = solve(A, b)
del A
starts, idx, _ = pick_start_points(mesh, sol, k)
E = eval_efield_batch(sol, mesh, starts)
orient = np.where(np.einsum("ij,ij->i", E, mesh.colloc_normals[idx]) >= 0, 1, -1)
for rep in range(int(os.environ.get("REPS", "2"))):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    res = tracer.trace_device(sol, mesh, starts, orient, TraceParams(), QuadConfig())
    torch.cuda.synchronize()
    dt = time.perf_counter() - t0
    print(f"{k} lines: {res.rounds} rounds in {dt:.3f} s = {1e6 * dt / max(1, res.rounds):.0f} us/round, "
          f"{res.field_points} evals", flush=True)

# host time inside the round call vs the whole trace
if os.environ.get("NOHOST"):
    sys.exit(0)
from paper_2003_12663_b200 import _lib  # noqa: E402

orig = _lib.call
acc = {"t": 0.0, "n": 0}


def timed(name, *a):
    t = time.perf_counter()
    r = orig(name, *a)
    if name == "hvb_trace_round":
        acc["t"] += time.perf_counter() - t
        acc["n"] += 1
    return r


_lib.call = timed
torch.cuda.synchronize()
t0 = time.perf_counter()
res = tracer.trace_device(sol, mesh, starts, orient, TraceParams(), QuadConfig())
torch.cuda.synchronize()
dt = time.perf_counter() - t0
print(f"host inside hvb_trace_round: {1e6 * acc['t'] / max(1, acc['n']):.0f} us/call over {acc['n']} calls; "
      f"wall {1e6 * dt / max(1, res.rounds):.0f} us/round")
