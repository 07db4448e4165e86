"""Accuracy of the MUFU.RSQ64H + Newton refinements (dev probe)."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import __graft_entry__
__graft_entry__.build()
from paper_2003_12663_b200 import _lib
rng = np.random.default_rng(0)
r2 = np.exp(rng.uniform(np.log(1e-12), np.log(1e4), 1 << 22))
d = torch.as_tensor(r2, device="cuda")
out = torch.empty((len(r2), 3), dtype=torch.float64, device="cuda")
_lib.call("hvb_bench_rsqrt", _lib.ptr(d), len(r2), _lib.ptr(out), _lib.stream_ptr())
o = out.cpu().numpy()
ref = 1.0 / np.sqrt(r2)
e2 = np.abs(o[:, 0] * 0.5 - ref) / ref
e1 = np.abs(o[:, 1] - ref) / ref
e3 = np.abs(o[:, 2] - ref ** 3) / ref ** 3
print(f"rinv3: max rel err {e3.max():.3e} mean {e3.mean():.3e}")
print(f"rsqrt2_newton: max rel err {e2.max():.3e} mean {e2.mean():.3e}; rsqrt_full: max {e1.max():.3e} mean {e1.mean():.3e}")
