"""Dev probe: field evaluation at uniform cfg4 points (device time, best of 3)
and at small batches (the tracer's tail sizes)."""
import sys

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_12663_b200 import fixtures, postprocess  # noqa: E402
from paper_2003_12663_b200.device import device_mesh  # noqa: E402
from paper_2003_12663_b200.solver import Solution  # noqa: E402

m = fixtures.rod_plane_mesh(1.0)
dm = device_mesh(m)
sol = Solution(u=np.random.default_rng(1).standard_normal(m.n_collocation), V=np.zeros(0), iterations=0, residual=0)
u_dev, key = postprocess._u_device(sol, dm)
src = postprocess._sources(dm, u_dev, key)
lo, hi = m.bounding_box()
for npts in (100000, 1000, 32, 4):
    P = torch.as_tensor(0.5 * (lo + hi) + np.random.default_rng(0).uniform(-0.6, 0.6, (npts, 3)) * (hi - lo),
                        device=dm.device)
    best = 1e9
    for _ in range(3):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        postprocess.field_points_device(dm, u_dev, src, P, False)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"{npts} points: {best:.3f} ms  ({npts / best * 1e3:.0f} evals/s)")
