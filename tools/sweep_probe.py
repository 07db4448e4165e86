"""Dev probe: regular-sweep kernel time on config 4 (SL + ADL launches),
best of 3 assemblies, plus the geometry of the built library."""
import sys
import time

import numpy as np
import torch

sys.path.insert(0, ".")
from paper_2003_12663_b200 import assembly, fixtures  # noqa: E402
from paper_2003_12663_b200.device import device_mesh, sweep_geometry  # noqa: E402

scale = float(sys.argv[1]) if len(sys.argv) > 1 else 1.0
m = fixtures.rod_plane_mesh(scale)
dm = device_mesh(m)
dm.stream_for(1)
best = None
for _ in range(3):
    prof = []
    assembly.PROFILE = prof
    A, _ = assembly.assemble(m)
    torch.cuda.synchronize()
    assembly.PROFILE = None
    reg = sum(e0.elapsed_time(e1) for lab, e0, e1 in prof if lab == "regular") / 1e3
    best = reg if best is None else min(best, reg)
    del A
print(f"geometry {sweep_geometry()} tiles {dm.n_tiles} records {dm.n_entries} local/n {dm.tiling.redundancy:.3f} halo {dm.tiling.n_halo} slots {dm.n_slots} "
      f"regular {best * 1e3:.1f} ms")
if len(sys.argv) > 2 and sys.argv[2] == "order":  # A/B: identity launch order of the tiles
    for label, order in (("identity order", None), ("longest first", dm.tile_order)):
        dm.tile_order = order
        best = None
        for _ in range(3):
            prof = []
            assembly.PROFILE = prof
            A, _ = assembly.assemble(m)
            torch.cuda.synchronize()
            assembly.PROFILE = None
            reg = sum(e0.elapsed_time(e1) for lab, e0, e1 in prof if lab == "regular") / 1e3
            best = reg if best is None else min(best, reg)
            del A
        print(f"{label}: regular {best * 1e3:.1f} ms")
