"""Dev: cfg-scale tracer phase alone (for ncu launch lists).
python tools/trace_phase.py [scale] [lines]"""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2003_12663_b200 import fixtures
from paper_2003_12663_b200.assembly import assemble
from paper_2003_12663_b200.postprocess import TraceParams, eval_efield_batch, pick_start_points
from paper_2003_12663_b200.quadrature import QuadConfig
from paper_2003_12663_b200.solver import solve
from paper_2003_12663_b200.tracer import trace_device

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
torch.cuda.cudart().cudaProfilerStart()
t = time.time()
res = trace_device(sol, mesh, starts, orient, TraceParams(), QuadConfig())
torch.cuda.synchronize()
torch.cuda.cudart().cudaProfilerStop()
print(f"trace {k} lines {time.time() - t:.3f}s rounds {res.rounds} evals {res.field_points}", flush=True)
