import sys, os
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2003_12663_b200 import _lib
out = torch.zeros(8, dtype=torch.float64, device="cuda")
_lib.call("hvb_bench_latency", _lib.ptr(out), 4096, _lib.stream_ptr())
torch.cuda.synchronize()
o = out.cpu().tolist()
print("latency cycles/op: DFMA %.1f DADD %.1f MUFU.RSQ64H(+DADD) %.1f rsqrt_full(+DADD) %.1f LDS-DADD-STS %.1f" % tuple(o[:5]))
