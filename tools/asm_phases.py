"""Dev probe (GPU): config-4 assembly phases (PROFILE spans, wall time) over
a few repeats."""
import sys
import time

sys.path.insert(0, ".")

import torch

from paper_2003_12663_b200 import assembly, fixtures
from paper_2003_12663_b200.device import device_mesh

m = fixtures.rod_plane_mesh(1.0)
dm = device_mesh(m)
dm.stream_for(1)
for it in range(4):
    prof = []
    assembly.PROFILE = prof
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    A, _ = assembly.assemble(m)
    torch.cuda.synchronize()
    wall = time.perf_counter() - t0
    assembly.PROFILE = None
    spans = {}
    for lab, e0, e1 in prof:
        spans[lab] = spans.get(lab, 0.0) + e0.elapsed_time(e1)
    print(f"it {it} wall {wall * 1e3:.1f} ms  " + "  ".join(f"{k} {v:.1f}" for k, v in spans.items()), flush=True)
    del A
