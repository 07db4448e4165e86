"""Dev probe (GPU): where the cfg4 GMRES solve spends its time -- device time
of the C-ABI kernels (CUDA events around each call) vs the solve's wall."""
import sys
import time
from collections import defaultdict

import torch

sys.path.insert(0, ".")
from paper_2003_12663_b200 import _lib, fixtures  # noqa: E402
from paper_2003_12663_b200.assembly import assemble  # noqa: E402
from paper_2003_12663_b200.solver import solve  # noqa: E402

m = fixtures.rod_plane_mesh(1.0)
A, b = assemble(m)
solve(A, b)
orig = _lib.call
ev = []


def timed(name, *a):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    r = orig(name, *a)
    e1.record()
    ev.append((name, e0, e1))
    return r


_lib.call = timed
torch.cuda.synchronize()
t0 = time.perf_counter()
sol = solve(A, b)
torch.cuda.synchronize()
wall = time.perf_counter() - t0
tot = defaultdict(float)
cnt = defaultdict(int)
for name, e0, e1 in ev:
    tot[name] += e0.elapsed_time(e1)
    cnt[name] += 1
print(f"solve wall {wall * 1e3:.1f} ms, {sol.iterations} iterations")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"  {k:24s} {cnt[k]:4d} calls {tot[k]:8.2f} ms")
print(f"  rest (torch elementwise, host, syncs) {wall * 1e3 - sum(tot.values()):.1f} ms")
