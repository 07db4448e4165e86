"""Dev probe (GPU): the bench step's field phase on config 4, piece by piece
(u upload, source contraction, N-body + near pairs), CUDA events + host
clock, after one assemble + solve."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_12663_b200 import fixtures, postprocess  # noqa: E402
from paper_2003_12663_b200.assembly import assemble  # noqa: E402
from paper_2003_12663_b200.device import device_mesh  # noqa: E402
from paper_2003_12663_b200.solver import SolverConfig, solve  # noqa: E402

m = fixtures.rod_plane_mesh(1.0)
lo, hi = m.bounding_box()
P = 0.5 * (lo + hi) + np.random.default_rng(1234).uniform(-0.6, 0.6, (100000, 3)) * (hi - lo)
dev = torch.device("cuda:0")
P_dev = torch.as_tensor(P, device=dev)
A, rhs = assemble(m)
sol = solve(A, rhs, SolverConfig())
del A
for it in range(4):
    ev = [torch.cuda.Event(enable_timing=True) for _ in range(5)]
    torch.cuda.synchronize()
    h0 = time.perf_counter()
    ev[0].record()
    dm = device_mesh(m)
    u_dev, key = postprocess._u_device(sol, dm)
    ev[1].record()
    src = postprocess._sources(dm, u_dev, key)
    ev[2].record()
    E = postprocess.field_points_device(dm, u_dev, src, P_dev, False)
    ev[3].record()
    torch.cuda.synchronize()
    h1 = time.perf_counter()
    t = [ev[i].elapsed_time(ev[i + 1]) for i in range(3)]
    print(f"it {it}: u {t[0]:.2f} ms  sources {t[1]:.2f} ms  field {t[2]:.2f} ms  (host {1e3 * (h1 - h0):.1f} ms, "
          f"near pairs {getattr(E, 'near_pairs', -1)})", flush=True)
