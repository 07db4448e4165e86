"""Node-loop throughput probe (dev tool): lane-nodes/s and FP64-op rate for
different occupancies, with and without the rsqrt."""
import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12663_b200 import _lib
out = torch.zeros(8, dtype=torch.float64, device="cuda")
st = _lib.stream_ptr()
iters = 2000
for var, name, ops in ((0, "cubic", 14), (2, "quadratic", 13), (3, "rsqrt2", 12), (1, "no-rsqrt", 9)):
    for warps_per_sm in (4, 8, 12, 16, 32):
        threads = 128
        blocks = 148 * warps_per_sm // 4
        _lib.call("hvb_bench_nodes", _lib.ptr(out), var, blocks, threads, 10, st)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(); _lib.call("hvb_bench_nodes", _lib.ptr(out), var, blocks, threads, iters, st); e1.record()
        torch.cuda.synchronize()
        t = e0.elapsed_time(e1) / 1e3
        nodes = blocks * threads * iters * 12 * 2
        print(f"{name:10s} warps/SM={warps_per_sm:2d}: {nodes/t/1e12:6.3f} Tnode/s  fp64-lane-ops {nodes*ops/t/1e12:6.2f} T/s "
              f"({nodes*ops/t/(148*64*1.965e9)*100:5.1f}% of pipe @1965MHz)")
