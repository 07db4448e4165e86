"""Dev probe: device tracer on the rod-plane config at a given scale.
python tools/trace_probe.py [scale] [lines]"""
import sys, time, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2003_12663_b200 import fixtures
from paper_2003_12663_b200.assembly import assemble
from paper_2003_12663_b200.solver import solve
from paper_2003_12663_b200.postprocess import (pick_start_points, eval_efield_batch, load_ionization_model,
                                               TraceParams, surface_field_magnitudes)
from paper_2003_12663_b200.quadrature import QuadConfig
from paper_2003_12663_b200.tracer import trace_device, streamer_device, TERMINATIONS, line_states

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 0.3
k = int(sys.argv[2]) if len(sys.argv) > 2 else 2000
t0 = time.time()
mesh = fixtures.rod_plane_mesh(scale)
print("mesh", mesh.n_triangles, mesh.n_collocation, f"{time.time()-t0:.1f}s", flush=True)
A, b = assemble(mesh)
sol = solve(A, b)
del A
torch.cuda.synchronize()
print("solved", sol.iterations, f"{time.time()-t0:.1f}s", flush=True)
se = surface_field_magnitudes(mesh, sol)
starts, idx, _ = pick_start_points(mesh, sol, k, surface_e=se)
E = eval_efield_batch(sol, mesh, starts)
orient = np.where(np.einsum("ij,ij->i", E, mesh.colloc_normals[idx]) >= 0, 1, -1)
torch.cuda.synchronize()
print("seeds", len(starts), f"{time.time()-t0:.1f}s", flush=True)
gas = load_ionization_model(os.path.join(os.path.dirname(fixtures.__file__), "data", "air_demo.gas"))
maxr = int(os.environ.get('MAXR', '0')) or None
for rep in range(int(os.environ.get("REPS", "1"))):
    torch.cuda.synchronize()
    t1 = time.time()
    res = trace_device(sol, mesh, starts, orient, TraceParams(), QuadConfig(), max_rounds=maxr)
    val, ver = streamer_device(res, gas)
    torch.cuda.synchronize()
    dt = time.time() - t1
    terms = np.bincount(res.info[:, 1], minlength=4)
    print(f"trace {len(starts)} lines: {dt:.3f}s rounds {res.rounds} evals {res.field_points} "
          f"({res.field_points/len(starts):.1f}/line) pts/line {res.info[:,0].mean():.1f} max {res.info[:,0].max()} "
          f"terms {dict(zip(TERMINATIONS, terms.tolist()))} status {np.bincount(res.info[:,2]).tolist()} "
          f"inception {int(ver.sum())} lines/s {len(starts)/dt:.1f}", flush=True)
    ls = line_states(res)
    run = np.nonzero(ls["status"] == 0)[0]
    diag = float(np.linalg.norm(np.ptp(mesh.vertices, axis=0)))
    for i in run[:8]:
        L = ls[i]
        print(f"  running line {i}: seed idx {idx[i]} x {L['x']} h/diag {L['h']/diag:.3e} s/diag {L['s']/diag:.3e} "
              f"d/R {L['d_surf']/L['local_r']:.3e} R {L['local_r']:.3e} armed {L['armed']} npts {L['npts']} "
              f"patch {mesh.tri_tags[mesh.vc_tri[mesh.vc_ptr[idx[i]]]] if hasattr(mesh,'tri_tags') else '?'} "
              f"start {starts[i]}", flush=True)
    if len(run):
        break
