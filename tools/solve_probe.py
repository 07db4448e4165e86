"""Dev: where the GMRES time goes on cfg4 (device time of GEMV / MGS launches
vs wall time of the solve)."""
import os
import sys
import time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import __graft_entry__
__graft_entry__.build()
from paper_2003_12663_b200 import _lib, fixtures
from paper_2003_12663_b200.assembly import assemble
from paper_2003_12663_b200.solver import solve

mesh = fixtures.rod_plane_mesh(float(sys.argv[1]) if len(sys.argv) > 1 else 1.0)
A, b = assemble(mesh)
solve(A, b)
rec = []
orig = _lib.call


def timed(name, *a):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig(name, *a)
    e1.record()
    rec.append((name, e0, e1))
    return r


_lib.call = timed
torch.cuda.synchronize()
t = time.perf_counter()
sol = solve(A, b)
torch.cuda.synchronize()
wall = time.perf_counter() - t
_lib.call = orig
tot = {}
for n, e0, e1 in rec:
    tot.setdefault(n, [0, 0.0])
    tot[n][0] += 1
    tot[n][1] += e0.elapsed_time(e1)
first, last = rec[0][1], rec[-1][2]
print(f"solve wall {wall * 1e3:.1f} ms, iterations {sol.iterations}, device span {first.elapsed_time(last):.1f} ms")
for n, (c, ms) in sorted(tot.items(), key=lambda x: -x[1][1]):
    print(f"  {n:20s} {c:5d} calls {ms:9.2f} ms")
