"""Dev probe (GPU): host-side time of assemble()'s pieces on config 4
(cProfile of the third call, after two warm-ups)."""
import cProfile
import pstats
import sys

import torch

sys.path.insert(0, ".")
from paper_2003_12663_b200 import assembly, fixtures  # noqa: E402
from paper_2003_12663_b200.device import device_mesh  # noqa: E402

m = fixtures.rod_plane_mesh(1.0)
dm = device_mesh(m)
for _ in range(2):
    A, _ = assembly.assemble(m)
    torch.cuda.synchronize()
    del A
pr = cProfile.Profile()
pr.enable()
A, _ = assembly.assemble(m)
torch.cuda.synchronize()
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
