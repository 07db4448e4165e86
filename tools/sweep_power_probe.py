"""Dev probe (GPU): SM clock and board power while config-4 assemblies run
back to back (nvidia-smi sampled every 50 ms) -- is the sweep power-capped?"""
import subprocess
import sys
import threading
import time

import torch

sys.path.insert(0, ".")
from paper_2003_12663_b200 import assembly, fixtures  # noqa: E402
from paper_2003_12663_b200.device import device_mesh  # noqa: E402

m = fixtures.rod_plane_mesh(1.0)
dm = device_mesh(m)
dm.stream_for(1)
A, _ = assembly.assemble(m)
del A
samples = []
stop = False


def sample():
    while not stop:
        out = subprocess.run(["nvidia-smi", "--query-gpu=clocks.sm,power.draw,temperature.gpu,clocks_throttle_reasons.active",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True).stdout.strip()
        samples.append((time.perf_counter(), out))
        time.sleep(0.05)


th = threading.Thread(target=sample)
th.start()
times = []
for _ in range(12):
    prof = []
    assembly.PROFILE = prof
    A, _ = assembly.assemble(m)
    torch.cuda.synchronize()
    assembly.PROFILE = None
    times.append(sum(e0.elapsed_time(e1) for lab, e0, e1 in prof if lab == "regular"))
    del A
stop = True
th.join()
print("regular ms:", [round(t, 1) for t in times])
clk = [float(s.split(",")[0]) for _, s in samples if s]
pw = [float(s.split(",")[1]) for _, s in samples if s]
tmp = [float(s.split(",")[2]) for _, s in samples if s]
rs = sorted(set(s.split(",")[3].strip() for _, s in samples if s))
import numpy as np  # noqa: E402
print(f"sm MHz: min {min(clk):.0f} median {np.median(clk):.0f} max {max(clk):.0f}; power W: median {np.median(pw):.0f} "
      f"max {max(pw):.0f}; temp C: max {max(tmp):.0f}; throttle reasons: {rs}")
