"""Dev probe: config-3 neutrality row (10,242 floating members) through the
fused charge-reduce path; device time of _weighted_adl_sum."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
sys.path.insert(0, "tests")
from conftest import _cfg3_parts  # noqa: E402
from paper_2003_12663_b200 import assembly, fixtures  # noqa: E402
from paper_2003_12663_b200.device import device_mesh  # noqa: E402

v, tris = _cfg3_parts(fixtures, 5, 4)
m = fixtures.mesh_from_parts(v, np.array([t[0] for t in tris]), np.array([t[1] for t in tris]),
                             ["patch 0 electrode 1.0", "patch 1 floating 0", "patch 2 electrode 0.0"])
dm = device_mesh(m)
mem = m.floating_collocation(0)
adl, ids = assembly._neutrality_scales(m, 0)
assembly._weighted_adl_sum(m, dm, mem, adl, ids)
torch.cuda.synchronize()
ts = []
for _ in range(3):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    row = assembly._weighted_adl_sum(m, dm, mem, adl, ids)
    e1.record()
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1) / 1e3)
print(f"cfg3 neutrality row: {len(mem)} members x {m.n_triangles} panels, fused charge-reduce "
      f"{min(ts) * 1e3:.2f} ms (best of 3), {len(mem) * m.n_triangles / min(ts):.3e} pairs/s")
